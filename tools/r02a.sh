set -x
lscpu | head -20 > gpurun_out/lscpu.txt; nproc >> gpurun_out/lscpu.txt
nvidia-smi > gpurun_out/nvsmi_r02a.txt
python -m pytest tests -q -m gpu -x --timeout 1500 > gpurun_out/gpu_tests_r02a.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests_r02a.log
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_r02a.json
