#!/bin/bash
# r04n: k_mpos_dense warp-aggregated atomicMin: fit / build parity, build launches
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_fit.py tests/test_gpu_build_device.py tests/test_gpu_config3.py tests/test_gpu_baselines.py tests/test_gpu_sharded_build.py tests/test_gpu_dropin.py -x -q > $O/r04n_tests.log 2>&1; echo "rc=$?" >> $O/r04n_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r04n_launches_build.csv python tools/prof_kernels.py build > /dev/null 2>&1
timeout 300 python tools/probe_fit.py 6 > $O/r04n_probe_fit.log 2>&1
