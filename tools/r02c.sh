python -m pytest tests -q -m gpu -x --timeout 1500 -s -k "image" > gpurun_out/gpu_tests_r02c_img.log 2>&1; echo "img tests rc=$?"
tail -5 gpurun_out/gpu_tests_r02c_img.log
python -m pytest tests -q -m gpu --timeout 1500 > gpurun_out/gpu_tests_r02c.log 2>&1; echo "tests rc=$?"
tail -8 gpurun_out/gpu_tests_r02c.log
