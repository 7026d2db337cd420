# Dev sweep (run under gpurun): MRS at N = 16384 over tail-split (PSWIM_MRS_TAIL) and chunk
# (PSWIM_MRS_CHUNKS) settings; the defaults measured best (DESIGN §10 item 3).
mkdir -p gpurun_out
out=gpurun_out/tail_sweep.txt; : > $out
for rep in 1 2; do
for t in "" "6,4" "8,4" "4,8" "8,8" "12,4" "8,2" "16,2" "6,6"; do
  for c in "" 34 40; do
    r=$(PSWIM_MRS_TAIL=$t PSWIM_MRS_CHUNKS=$c python tools/probe_mrs.py 16384 2>&1 | grep "N=16384")
    echo "tail=[$t] chunks=[$c] $r" >> $out
  done
done
done
