# r02g: hand-written tcgen05 GEMM family: tests, SASS, probe, config-5 validation with CUTLASS cross-check
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x > $OUT/gemm_tests_r02g.log 2>&1; echo "gemm tests rc=$?"; tail -3 $OUT/gemm_tests_r02g.log
timeout 300 python tools/probe_tc_gemm.py > $OUT/probe_tc_r02g.log 2>&1; echo "probe rc=$?"; grep -v "bad=0" $OUT/probe_tc_r02g.log | tail -12
timeout 2400 python tools/validate_gemm.py --out $OUT/gemm_validation_r02g.json > $OUT/gemm_validation_r02g.log 2>&1; echo "validate rc=$?"; tail -60 $OUT/gemm_validation_r02g.log
