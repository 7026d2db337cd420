mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parareal.py -x -q --timeout=200 -k pipelining > gpurun_out/dbg_trace.log 2>&1
PSWIM_BENCH_LARGE_RODS=4 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --wire gloo --fine-steps 4 --no-cpu > gpurun_out/dbg_multi.out 2> gpurun_out/dbg_multi.err
