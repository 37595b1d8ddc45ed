#!/bin/bash
# r04z: final tree: full GPU suite, smoke, default bench + reference arm, launch lists
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu > $O/r04z_gpu_tests.log 2>&1; echo "rc=$?" >> $O/r04z_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r04z_smoke.log 2>&1; echo "rc=$?" >> $O/r04z_smoke.log
timeout 900 python bench.py > $O/r04z_bench.json 2> $O/r04z_bench.err
timeout 600 python bench.py --impl reference > $O/r04z_bench_reference.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r04z_launches_build.csv python tools/prof_kernels.py build > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r04z_launches_step.csv python tools/prof_kernels.py step 100000000 > /dev/null 2>&1
