# full GPU suite + N=1 bench + the N>1 bench code path as 4 ranks on one GPU (gloo wire)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout=600 > gpurun_out/rc_gputest.log 2>&1
python bench.py > gpurun_out/rc_bench.json 2> gpurun_out/rc_bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 3 --warmup 3 --wire gloo --fine-steps 100 --coarse-steps 10 --large-fine-steps 2 --no-cpu > gpurun_out/rc_bench4.json 2> gpurun_out/rc_bench4.err
