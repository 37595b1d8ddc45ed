# r03r: full state of the tree: parity, smoke, bench + reference arm, ncu evidence
OUT=gpurun_out; mkdir -p $OUT
timeout 1800 python -m pytest tests -q -m gpu > $OUT/gpu_tests_r03r.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/gpu_tests_r03r.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_r03r.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_r03r.log
timeout 900 python bench.py > $OUT/bench_r03r.json 2> $OUT/bench_r03r.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $OUT/bench_ref_r03r.json 2>&1; echo "ref rc=$?"
bash tools/profile_round.sh r03r
timeout 1200 compute-sanitizer --tool racecheck python tools/sanitize_drive.py > $OUT/sanitize_racecheck_r03r.log 2>&1; tail -1 $OUT/sanitize_racecheck_r03r.log; timeout 1200 compute-sanitizer --tool memcheck python tools/sanitize_drive.py > $OUT/sanitize_memcheck_r03r.log 2>&1; tail -1 $OUT/sanitize_memcheck_r03r.log; timeout 1200 compute-sanitizer --tool synccheck python tools/sanitize_drive.py > $OUT/sanitize_synccheck_r03r.log 2>&1; tail -1 $OUT/sanitize_synccheck_r03r.log
