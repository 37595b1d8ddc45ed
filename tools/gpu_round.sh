#!/bin/bash
# One GPU round trip: parity tests, bench, launch list, ncu captures.
# Usage (from the repo root, under gpurun): bash tools/gpu_round.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
python -m pytest tests -x -q -m gpu > $OUT/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"
tail -3 $OUT/gpu_tests_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
python bench.py --steps 5 --warmup 3 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
tail -c 3000 $OUT/bench_$TAG.json
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref_$TAG.json 2>&1; echo "ref rc=$?"
tail -c 600 $OUT/bench_ref_$TAG.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --queries 20000000 --skip-cpu > /dev/null 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_gather -s 3 -c 1 -o $OUT/prof_gather_$TAG -f \
    python bench.py --steps 1 --warmup 1 --queries 20000000 --skip-cpu --skip-secondary > /dev/null 2>&1; echo "ncu gather rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 3 -c 1 -o $OUT/prof_sweep_$TAG -f \
    python bench.py --steps 1 --warmup 1 --queries 1000000 --skip-cpu > /dev/null 2>&1; echo "ncu sweep rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_eval -s 2 -c 1 -o $OUT/prof_eval_$TAG -f \
    python bench.py --steps 1 --warmup 1 --queries 20000000 --skip-cpu --skip-secondary > /dev/null 2>&1; echo "ncu eval rc=$?"
ls -la $OUT
