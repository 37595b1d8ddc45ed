#!/bin/bash
# r04g: k_eval4 at 4 CTAs/SM (RPT 2) + k_escatter batched global atomics: step time, digest, decide tests
O=gpurun_out; mkdir -p $O
timeout 300 python tools/probe_overlap.py > $O/r04g_step.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_decide.py tests/test_gpu_prune.py tests/test_gpu_config3.py -x -q > $O/r04g_tests.log 2>&1; echo "rc=$?" >> $O/r04g_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r04g_launches_step.csv python tools/prof_kernels.py step 100000000 > /dev/null 2>&1
