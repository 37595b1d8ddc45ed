#!/bin/bash
# r04m: k_escatter on 1024-slot chunks, up to 8 CTAs / SM: step time + digest, decide tests, step launches
O=gpurun_out; mkdir -p $O
timeout 300 python tools/probe_overlap.py > $O/r04m_step.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r04m_launches_step.csv python tools/prof_kernels.py step 100000000 > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_decide.py tests/test_gpu_prune.py tests/test_gpu_config3.py tests/test_gpu_wide.py -x -q > $O/r04m_tests.log 2>&1; echo "rc=$?" >> $O/r04m_tests.log
