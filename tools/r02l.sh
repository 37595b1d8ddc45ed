# r02l: stream-ordered grid create, device build exchange (pack / all-gather / merge), N=2 rehearsal
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_sharded_build.py tests/test_gpu_fused_sweep.py tests/test_gpu_build_device.py -x -q > $OUT/tests_r02l.log 2>&1; echo "tests rc=$?"; tail -15 $OUT/tests_r02l.log
timeout 300 python tools/probe_build_stages.py > $OUT/stages_sync_r02l.log 2>&1; echo "stages rc=$?"; tail -2 $OUT/stages_sync_r02l.log
GRID_ASYNC=1 timeout 300 python tools/probe_build_stages.py > $OUT/stages_async_r02l.log 2>&1; echo "stages async rc=$?"; tail -2 $OUT/stages_async_r02l.log
WT_DIST_REHEARSAL=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --skip-cpu > $OUT/bench_n2_rehearsal_r02l.json 2> $OUT/bench_n2_rehearsal_r02l.err; echo "n2 rc=$?"; tail -c 2500 $OUT/bench_n2_rehearsal_r02l.json; tail -20 $OUT/bench_n2_rehearsal_r02l.err
timeout 900 python bench.py --skip-cpu > $OUT/bench_r02l.json 2> $OUT/bench_r02l.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('$OUT/bench_r02l.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step']); print(json.dumps(d['secondary']['full_build'])[:1500])"
