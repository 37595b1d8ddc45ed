# r02k: re-entry check of HEAD on a fresh box: parity, smoke, bench, reference arm
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/gpu_tests_r02k.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/gpu_tests_r02k.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_r02k.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke_r02k.log
timeout 900 python bench.py > $OUT/bench_r02k.json 2> $OUT/bench_r02k.err; echo "bench rc=$?"; tail -c 4000 $OUT/bench_r02k.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref_r02k.json 2>&1; echo "ref rc=$?"; tail -c 600 $OUT/bench_ref_r02k.json
