#!/bin/bash
# r04i: pinned plan upload + lazy engine info: build timeline, engine/build tests, bench secondary
O=gpurun_out; mkdir -p $O
timeout 300 python tools/probe_build_timeline.py > $O/r04i_timeline.log 2>&1
WT_TRACE_ENGINE=1 timeout 300 python tools/probe_build_timeline.py > $O/r04i_timeline_trace.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_build_device.py tests/test_gpu_image.py tests/test_gpu_dropin.py tests/test_gpu_decide.py tests/test_gpu_sharded_build.py -x -q > $O/r04i_tests.log 2>&1; echo "rc=$?" >> $O/r04i_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --skip-cpu > $O/r04i_bench.json 2> $O/r04i_bench.err
