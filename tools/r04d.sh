#!/bin/bash
# r04d: k_qfit with the quad-parallel reflector division + batched sample loads
O=gpurun_out; mkdir -p $O
timeout 300 python tools/probe_fit.py 6 > $O/r04d_probe_fit.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fit.py tests/test_gpu_build_device.py tests/test_gpu_config3.py tests/test_gpu_baselines.py tests/test_gpu_sharded_build.py -x -q > $O/r04d_tests.log 2>&1; echo "rc=$?" >> $O/r04d_tests.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qfit -s 3 -c 1 -o $O/ncu_qfit_r04d -f \
    python tools/prof_kernels.py build > /dev/null 2>&1; echo "qfit $?" >> $O/r04d_tests.log
