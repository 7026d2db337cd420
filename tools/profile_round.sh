#!/bin/bash
# GPU-side profiling recipe (run under gpurun): launch list of bench.py + one ncu --set full
# capture of each hot kernel.  Summaries are extracted here by tools/ncu_summary.py.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-steps > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mrs_kernel -s 3 -c 1 -o gpurun_out/mrs_full -f \
    python tools/probe_mrs.py 16384 > gpurun_out/ncu_mrs.log 2>&1
for k in sqrt_tma rod_loads_wtma advance_tma; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/${k}_full -f \
      python tools/probe_rod.py > gpurun_out/ncu_$k.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"fused_kernel" -s 1 -c 1 -o gpurun_out/fused_full -f \
    python tools/flag16.py > gpurun_out/ncu_fused.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lj_launches.csv \
    python tools/probe_lj.py > gpurun_out/ncu_lj.log 2>&1
# round-end extras (this round): e2e breakdown, per-CTA MRS timeline (needs
# `python tools/probe_mrs_trace.py build` here first), sanitizers
python tools/probe_e2e.py 16384 4096 > gpurun_out/e2e.txt 2>&1
[ -f tools/libpswim_trace.so ] && python tools/probe_mrs_trace.py 16384 > gpurun_out/trace.txt 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_smoke.py > gpurun_out/san_$tool.txt 2>&1
done
