# r04r: full state of the tree after the r04 changes: parity, smoke, bench + reference arm, ncu evidence, sanitizers
OUT=gpurun_out; mkdir -p $OUT
timeout 1800 python -m pytest tests -q -m gpu > $OUT/gpu_tests_r04r.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/gpu_tests_r04r.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_r04r.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_r04r.log
timeout 900 python bench.py > $OUT/bench_r04r.json 2> $OUT/bench_r04r.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $OUT/bench_ref_r04r.json 2>&1; echo "ref rc=$?"
bash tools/profile_round.sh r04r
timeout 1200 compute-sanitizer --tool racecheck python tools/sanitize_drive.py > $OUT/sanitize_racecheck_r04r.log 2>&1; tail -1 $OUT/sanitize_racecheck_r04r.log; timeout 1200 compute-sanitizer --tool memcheck python tools/sanitize_drive.py > $OUT/sanitize_memcheck_r04r.log 2>&1; tail -1 $OUT/sanitize_memcheck_r04r.log; timeout 1200 compute-sanitizer --tool synccheck python tools/sanitize_drive.py > $OUT/sanitize_synccheck_r04r.log 2>&1; tail -1 $OUT/sanitize_synccheck_r04r.log
python tools/summarize_ncu.py $OUT/r04r_ncu_summary.md $OUT/ncu_{gather,eval4,escatter,sweepw,qfit,prune}_r04r.ncu-rep > /dev/null 2>&1; mkdir -p $OUT/reps; mv $OUT/ncu_{eval4,escatter,sweepw,prune}_r04r.ncu-rep $OUT/../ 2>/dev/null; ls -la $OUT | head -60
