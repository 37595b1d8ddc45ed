#!/bin/bash
# r04k: pruning survival vs table structure (config-2 step); full GPU suite + smoke on the final tree
O=gpurun_out; mkdir -p $O
timeout 900 python tools/probe_survival.py > $O/r04k_survival.jsonl 2> $O/r04k_survival.err
timeout 1800 python -m pytest tests -q -m gpu > $O/r04k_gpu_tests.log 2>&1; echo "rc=$?" >> $O/r04k_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r04k_smoke.log 2>&1; echo "rc=$?" >> $O/r04k_smoke.log
