#!/bin/bash
# ncu evidence for profiles/: launch list of the bench command + full captures
# of the hot kernels (one GPU, short commands).  Usage: bash tools/profile_round.sh TAG
TAG=${1:-r01}
O=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --skip-cpu > $O/bench_under_ncu_$TAG.log 2>&1; echo "launches $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_step_$TAG.csv \
    python tools/prof_kernels.py step 100000000 > /dev/null 2>&1; echo "step launches $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_fit_$TAG.csv \
    python tools/prof_kernels.py fit > /dev/null 2>&1; echo "fit launches $?"
# the bench step's kernels, captured on the bench's own 1e8-query stream
ncu --set full --clock-control none --import-source on -k regex:k_gather_h -s 2 -c 1 -o $O/ncu_gather_$TAG -f \
    python tools/prof_kernels.py step 100000000 > /dev/null 2>&1; echo "gather $?"
ncu --set full --clock-control none --import-source on -k regex:k_eval4 -s 2 -c 1 -o $O/ncu_eval4_$TAG -f \
    python tools/prof_kernels.py step 100000000 > /dev/null 2>&1; echo "eval4 $?"
ncu --set full --clock-control none --import-source on -k regex:k_escatter -s 2 -c 1 -o $O/ncu_escatter_$TAG -f \
    python tools/prof_kernels.py step 100000000 > /dev/null 2>&1; echo "escatter $?"
ncu --set full --clock-control none --import-source on -k regex:k_sweep2 -s 2 -c 1 -o $O/ncu_sweep2_$TAG -f \
    python tools/prof_kernels.py sweep3 > /dev/null 2>&1; echo "sweep2 $?"
ncu --set full --clock-control none --import-source on -k regex:k_fit -s 1 -c 1 -o $O/ncu_fit_$TAG -f \
    python tools/prof_kernels.py fit > /dev/null 2>&1; echo "fit $?"
