for c in 25 34 50 100; do echo "== chunks $c"; PSWIM_MRS_CHUNKS=$c python tools/probe_fused.py 2>&1 | head -9; done > gpurun_out/r2_chunks.txt
python tools/probe_engine.py > gpurun_out/r2_eng_probe2.txt 2>&1
