#!/bin/bash
# r04o: ncu captures of the build kernels changed in r04 (k_img_prune after r04l, k_select_k, k_qfit), summarised
O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_img_prune -s 1 -c 1 -o $O/ncu_prune_r04o -f python tools/prof_kernels.py build > /dev/null 2>&1; echo "prune $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_select_k -s 1 -c 1 -o $O/ncu_selectk_r04o -f python tools/prof_kernels.py build > /dev/null 2>&1; echo "select $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qfit -s 3 -c 1 -o $O/ncu_qfit_r04o -f python tools/prof_kernels.py build > /dev/null 2>&1; echo "qfit $?"
python tools/summarize_ncu.py $O/r04o_ncu_summary.md $O/ncu_prune_r04o.ncu-rep $O/ncu_selectk_r04o.ncu-rep $O/ncu_qfit_r04o.ncu-rep; echo "sum $?"
