# r02y: hand-written u32 exclusive scan replaces the library scans on the decision path
OUT=gpurun_out; mkdir -p $OUT
timeout 1800 python -m pytest tests -q -m gpu -x > $OUT/gpu_tests_r02y.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/gpu_tests_r02y.log
timeout 600 python bench.py --skip-cpu --steps 10 --warmup 3 > $OUT/ab.json 2>/dev/null
python -c "
import json; d=json.loads(open('$OUT/ab.json').read().strip().splitlines()[-1]); o=d['offgrid_eval']; s=d['secondary']; print('step', round(d['ms_per_step'],4), 'value %.3e'%d['value'], 'offgrid', round(o['ms'],4), 'gather', round(d['roofline']['launch_ms'],4), 'launches', d['gpu_launches'], 'build', round(s['full_build']['ms_wall'],3))"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_step_r02y.csv python tools/prof_kernels.py step 100000000 > /dev/null 2>&1; echo "launches rc=$?"
