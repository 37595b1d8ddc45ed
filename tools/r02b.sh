python -m pytest tests -q -m gpu --timeout 1500 > gpurun_out/gpu_tests_r02b.log 2>&1; echo "tests rc=$?"
tail -8 gpurun_out/gpu_tests_r02b.log
