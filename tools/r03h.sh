# r03h: compute-sanitizer on the current kernels (memcheck / racecheck / synccheck)
OUT=gpurun_out; mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_drive.py > $OUT/sanitize_${tool}_r03h.log 2>&1; echo "$tool rc=$?"; tail -3 $OUT/sanitize_${tool}_r03h.log
done
WT_SWEEP_DEDUP=0 timeout 1500 compute-sanitizer --tool memcheck python tools/sanitize_drive.py > $OUT/sanitize_memcheck_dedup0_r03h.log 2>&1; echo "memcheck dedup0 rc=$?"; tail -2 $OUT/sanitize_memcheck_dedup0_r03h.log
