#!/bin/bash
# r04a: gather / off-grid evaluation overlap sweep (config-2 step)
O=gpurun_out; mkdir -p $O
for v in "1 2" "2 2" "4 2" "4 1" "4 3" "8 2" "8 1" "16 2" "4 4"; do
  set -- $v
  WT_GATHER_OVERLAP=$1 WT_OVERLAP_GATHER_CTAS=$2 timeout 300 python tools/probe_overlap.py >> $O/r04a_overlap.jsonl 2>> $O/r04a_err.log
done
timeout 900 python -m pytest tests/test_gpu_decide.py tests/test_gpu_prune.py -x -q > $O/r04a_tests.log 2>&1; echo "rc=$?" >> $O/r04a_tests.log
