#!/bin/bash
# Quick GPU iteration: decide/prune tests, step launch list, ncu of one kernel, bench.
# usage: bash tools/gpu_quick.sh KERNEL_REGEX [TAG]   (every step under its own timeout)
K=${1:-k_eval3}; T=${2:-q}; O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_decide.py tests/test_gpu_prune.py -x -q > $O/t_$T.log 2>&1; echo "tests rc=$?" >> $O/t_$T.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_$T.csv python tools/prof_kernels.py step 100000000 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o $O/ncu_$T -f python tools/prof_kernels.py step 100000000 > /dev/null 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --skip-cpu --skip-secondary > $O/bench_$T.json 2>&1
