#!/bin/bash
# r04c: k_qfit source-level capture (where the bucket fit's time goes)
O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qfit -s 3 -c 1 -o $O/ncu_qfit_r04c -f \
    python tools/prof_kernels.py build > /dev/null 2>&1; echo "qfit $?"
ncu -i $O/ncu_qfit_r04c.ncu-rep --page source --csv > $O/r04c_qfit_source.csv 2>/dev/null
ncu -i $O/ncu_qfit_r04c.ncu-rep --page raw --csv > $O/r04c_qfit_raw.csv 2>/dev/null
ls -la $O
