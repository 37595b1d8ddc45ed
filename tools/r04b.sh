#!/bin/bash
# r04b: k_qfit at 7 CTAs/SM -- fit timing, fit parity, bench (with the e2e copy ceiling)
O=gpurun_out; mkdir -p $O
timeout 300 python tools/probe_fit.py 6 > $O/r04b_probe_fit.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fit.py tests/test_gpu_build_device.py -x -q > $O/r04b_tests.log 2>&1; echo "rc=$?" >> $O/r04b_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --skip-cpu > $O/r04b_bench.json 2> $O/r04b_bench.err
