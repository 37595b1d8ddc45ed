python -m pytest tests -q -m gpu -x --timeout 1500 -s -k "fit or build_device or dropin or baselines" > gpurun_out/gpu_tests_r02e_fit.log 2>&1; echo "fit tests rc=$?"
tail -5 gpurun_out/gpu_tests_r02e_fit.log
grep -E "wall ms" gpurun_out/gpu_tests_r02e_fit.log
WT_FIT_TRACE=1 python tools/prof_kernels.py build > gpurun_out/trace_build_r02e.log 2>&1; tail -30 gpurun_out/trace_build_r02e.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_build_r02e.csv python tools/prof_kernels.py build > /dev/null 2>&1; echo "launches $?"
ncu --set full --clock-control none --import-source on -k regex:k_qfit -s 2 -c 1 -o gpurun_out/ncu_qfit_r02e -f python tools/prof_kernels.py build > /dev/null 2>&1; echo "qfit $?"
python -m pytest tests -q -m gpu --timeout 1500 > gpurun_out/gpu_tests_r02e.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/gpu_tests_r02e.log
