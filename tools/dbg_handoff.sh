# dev: run the threads + peer hand-off case; if it hangs, dump host threads and device kernels
mkdir -p gpurun_out
export PSWIM_COMM_TIMEOUT_S=20
python tools/debug_handoff.py ${1:-0} 1 > gpurun_out/dbg_h.log 2>&1 &
PY=$!
for i in $(seq 1 50); do sleep 1; kill -0 $PY 2>/dev/null || break; done
if kill -0 $PY 2>/dev/null; then
  timeout 60 cuda-gdb -batch -p $PY -ex "info cuda kernels" -ex "thread apply all bt 40" > gpurun_out/dbg_gdb.log 2>&1
  kill -9 $PY
fi
wait $PY
