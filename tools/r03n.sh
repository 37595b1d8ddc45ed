# r03n: N=2 code-path rehearsal on one GPU (gloo), sharded and fused sweeps
OUT=gpurun_out; mkdir -p $OUT
WT_DIST_REHEARSAL=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --skip-cpu > $OUT/bench_n2_r03n.json 2> $OUT/bench_n2_r03n.err; echo "n2 rc=$?"
python -c "
import json; d=json.loads(open('$OUT/bench_n2_r03n.json').read().strip().splitlines()[-1]); s=d['secondary']; print('n', d['n_gpus'], 'value %.3e'%d['value'], json.dumps(s['full_build'])[:300], s['config3_sweep']['sharding'], s['config4_fit'])"
tail -3 $OUT/bench_n2_r03n.err
WT_DIST_REHEARSAL=1 WT_FUSED_SWEEP=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 3 --skip-cpu > $OUT/bench_n2f_r03n.json 2> $OUT/bench_n2f_r03n.err; echo "n2 fused rc=$?"
python -c "
import json; d=json.loads(open('$OUT/bench_n2f_r03n.json').read().strip().splitlines()[-1]); s=d['secondary']; print('n', d['n_gpus'], s['config3_sweep']['sharding'], round(s['full_build']['ms_wall'],3))"
tail -3 $OUT/bench_n2f_r03n.err
timeout 600 python -m pytest tests/test_gpu_sharded_build.py tests/test_gpu_fused_sweep.py -q 2>&1 | tail -1
