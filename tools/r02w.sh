# r02w: K2 sort buffers swapped (no copy back), group flags / meta from the sorted keys, k_ranges full grid
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_fit.py tests/test_gpu_build_device.py tests/test_gpu_dropin.py tests/test_gpu_sharded_build.py tests/test_gpu_baselines.py tests/test_gpu_config3.py tests/test_gpu_prune.py -x -q > $OUT/tests_r02w.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests_r02w.log
timeout 1500 python -m pytest tests/test_gpu_decide.py -x -q -k "variants" > $OUT/tests_r02w_var.log 2>&1; echo "variants rc=$?"; tail -3 $OUT/tests_r02w_var.log
timeout 600 python bench.py --skip-cpu --steps 5 --warmup 3 > $OUT/ab.json 2>/dev/null
python -c "
import json; d=json.loads(open('$OUT/ab.json').read().strip().splitlines()[-1]); s=d['secondary']; print('build', round(s['full_build']['ms_wall'],3), round(s['full_build']['ms_device_events'],3), {k: round(v,3) for k,v in s['full_build']['stages_ms_wall_synced'].items()}, 'fit dev', round(s['config4_fit']['ms_device'],3))"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_build_r02w.csv python tools/prof_kernels.py build > /dev/null 2>&1; echo "launches rc=$?"
