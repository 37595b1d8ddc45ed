#!/bin/bash
# ncu evidence for profiles/: launch lists of the bench step / the build and
# full captures of the hot kernels (one GPU, short commands).
# Usage: bash tools/profile_round.sh TAG
TAG=${1:-r01}
O=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --skip-cpu > $O/bench_under_ncu_$TAG.log 2>&1; echo "launches $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_step_$TAG.csv \
    python tools/prof_kernels.py step 100000000 > /dev/null 2>&1; echo "step launches $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_build_$TAG.csv \
    python tools/prof_kernels.py build > /dev/null 2>&1; echo "build launches $?"
# the bench step's kernels, captured on the bench's own 1e8-query stream
ncu --set full --clock-control none --import-source on -k regex:k_gather_h -s 2 -c 1 -o $O/ncu_gather_$TAG -f \
    python tools/prof_kernels.py step 100000000 > /dev/null 2>&1; echo "gather $?"
ncu --set full --clock-control none --import-source on -k regex:k_eval4 -s 2 -c 1 -o $O/ncu_eval4_$TAG -f \
    python tools/prof_kernels.py step 100000000 > /dev/null 2>&1; echo "eval4 $?"
ncu --set full --clock-control none --import-source on -k regex:k_escatter -s 2 -c 1 -o $O/ncu_escatter_$TAG -f \
    python tools/prof_kernels.py step 100000000 > /dev/null 2>&1; echo "escatter $?"
# the build (config 3/4, records in HBM -> grid): representative sweep, bucket fit, pruning masks
ncu --set full --clock-control none --import-source on -k regex:k_sweep_w -s 1 -c 1 -o $O/ncu_sweepw_$TAG -f \
    python tools/prof_kernels.py build > /dev/null 2>&1; echo "sweep_w $?"
ncu --set full --clock-control none --import-source on -k regex:k_qfit -s 3 -c 1 -o $O/ncu_qfit_$TAG -f \
    python tools/prof_kernels.py build > /dev/null 2>&1; echo "qfit $?"
ncu --set full --clock-control none --import-source on -k regex:k_img_prune -s 1 -c 1 -o $O/ncu_prune_$TAG -f \
    python tools/prof_kernels.py build > /dev/null 2>&1; echo "prune $?"
