#!/bin/bash
# r04l: k_img_prune leaders in shared memory (54 registers): image / prune / build parity, build launches, bench secondary
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_image.py tests/test_gpu_prune.py tests/test_gpu_build_device.py tests/test_gpu_config3.py tests/test_gpu_decide.py tests/test_gpu_sharded_build.py -x -q > $O/r04l_tests.log 2>&1; echo "rc=$?" >> $O/r04l_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r04l_launches_build.csv python tools/prof_kernels.py build > /dev/null 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --skip-cpu > $O/r04l_bench.json 2> $O/r04l_bench.err
