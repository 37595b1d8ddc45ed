# r02p: representative (M-interval) sweep: parity + timing
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_decide.py tests/test_gpu_config3.py tests/test_gpu_prune.py tests/test_gpu_sharded_build.py tests/test_gpu_fused_sweep.py tests/test_gpu_build_device.py tests/test_gpu_wide.py -x -q > $OUT/tests_r02p.log 2>&1; echo "tests rc=$?"; tail -5 $OUT/tests_r02p.log
for v in "" "WT_SWEEP_DEDUP=0"; do
  env $v timeout 600 python bench.py --skip-cpu --steps 5 --warmup 3 > $OUT/ab.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$OUT/ab.json').read().strip().splitlines()[-1]); s=d['secondary']; print('$v', 'build', round(s['full_build']['ms_wall'],3), round(s['full_build']['ms_device_events'],3), s['full_build']['stages_ms_wall_synced'], 'c3 sweep', round(s['config3_sweep']['ms'],4), s['config3_sweep']['roofline']['physical_evals'], 'c1 sweep', round(s['config1_sweep']['ms'],4))"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_build_r02p.csv python tools/probe_build_stages.py > /dev/null 2>&1; echo "launches rc=$?"
