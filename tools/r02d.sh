python -m pytest tests -q -m gpu -x --timeout 1500 -s -k "build_device or image" > gpurun_out/gpu_tests_r02d_new.log 2>&1; echo "new tests rc=$?"
tail -5 gpurun_out/gpu_tests_r02d_new.log
grep -E "wall ms|engine creation" gpurun_out/gpu_tests_r02d_new.log
python -m pytest tests -q -m gpu --timeout 1500 > gpurun_out/gpu_tests_r02d.log 2>&1; echo "tests rc=$?"
tail -8 gpurun_out/gpu_tests_r02d.log
