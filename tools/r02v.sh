# r02v: K2 streaming kernels captured (ranges / pack / group_flags / select / samples / mpos / radix)
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_prune.py -x -q > $OUT/tests_r02v.log 2>&1; echo "prune tests rc=$?"; tail -2 $OUT/tests_r02v.log
ncu --set full --clock-control none -k "regex:k_ranges|k_pack|k_group_flags|k_select|k_samples|k_mpos|k_group_meta" -s 7 -c 7 -o $OUT/ncu_k2_r02v -f python tools/prof_kernels.py build > /dev/null 2>&1; echo "k2 rc=$?"
