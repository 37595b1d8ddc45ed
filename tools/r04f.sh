#!/bin/bash
# r04f: source-level captures of the off-grid pipeline (k_eval4, k_escatter) on the bench's stream
O=gpurun_out; mkdir -p $O
for k in k_eval4 k_escatter; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $O/ncu_${k}_r04f -f \
    python tools/prof_kernels.py step 100000000 > /dev/null 2>&1; echo "$k $?"
done
