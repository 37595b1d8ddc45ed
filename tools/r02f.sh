# GPU round trip r02f: verify HEAD (device-resident build, quad-lane fit, CPU baselines in bench)
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu_r02f.txt
./tools/bin/fp64_peak > $OUT/fp64_peak_r02f.json 2>&1; echo "fp64 rc=$?"; cat $OUT/fp64_peak_r02f.json
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_r02f.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke_r02f.log
timeout 1800 python -m pytest tests -q -m gpu --timeout 1500 > $OUT/gpu_tests_r02f.log 2>&1; echo "tests rc=$?"
tail -8 $OUT/gpu_tests_r02f.log
timeout 900 python bench.py > $OUT/bench_r02f.json 2> $OUT/bench_r02f.err; echo "bench rc=$?"
tail -c 6000 $OUT/bench_r02f.json; tail -5 $OUT/bench_r02f.err
