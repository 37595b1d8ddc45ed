OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_fit.py tests/test_gpu_build_device.py tests/test_gpu_dropin.py tests/test_gpu_sharded_build.py tests/test_gpu_baselines.py tests/test_gpu_config3.py tests/test_oracle.py -x -q > $OUT/tests_r03f.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/tests_r03f.log
for i in 1 2; do timeout 600 python bench.py --skip-cpu --steps 5 --warmup 3 > $OUT/ab.json 2>/dev/null
python -c "
import json; d=json.loads(open('$OUT/ab.json').read().strip().splitlines()[-1]); s=d['secondary']; print('build', round(s['full_build']['ms_wall'],3), round(s['full_build']['ms_device_events'],3), 'fit dev', round(s['config4_fit']['ms_device'],3))"; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_build_r03f.csv python tools/prof_kernels.py build > /dev/null 2>&1; echo "launches rc=$?"
