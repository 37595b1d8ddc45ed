# r02m: off-grid pipeline A/B (grouping on/off, rows per thread) + k_eval4 source-level capture
OUT=gpurun_out; mkdir -p $OUT
for v in "" "WT_EVAL_KEY_MODE=3" "WT_EVAL4_RPT=1" "WT_EVAL_KEY_MODE=3 WT_EVAL4_RPT=1" "WT_EVAL_KEY_BITS=14"; do
  env $v timeout 300 python bench.py --skip-cpu --skip-secondary --steps 10 --warmup 3 > $OUT/ab.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$OUT/ab.json').read().strip().splitlines()[-1]); o=d['offgrid_eval']; print('$v', 'step', round(d['ms_per_step'],4), 'offgrid', round(o['ms'],4), 'gather', round(d['roofline']['launch_ms'],4))"
done
ncu --set full --clock-control none --import-source on -k regex:k_eval4 -s 2 -c 1 -o $OUT/ncu_eval4_r02m -f \
    python bench.py --steps 1 --warmup 1 --skip-cpu --skip-secondary > /dev/null 2>&1; echo "ncu eval4 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_step_r02m.csv \
    python bench.py --steps 2 --warmup 1 --skip-cpu --skip-secondary > /dev/null 2>&1; echo "launches rc=$?"
