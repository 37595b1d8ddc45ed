#!/bin/bash
# r04j: batched latency gathers in k_select_k / k_samples_k: fit parity, build launches, bench secondary
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_fit.py tests/test_gpu_build_device.py tests/test_gpu_config3.py tests/test_gpu_baselines.py tests/test_gpu_sharded_build.py tests/test_gpu_dropin.py -x -q > $O/r04j_tests.log 2>&1; echo "rc=$?" >> $O/r04j_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r04j_launches_build.csv python tools/prof_kernels.py build > /dev/null 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --skip-cpu > $O/r04j_bench.json 2> $O/r04j_bench.err
