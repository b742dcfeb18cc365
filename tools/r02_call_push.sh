set -u
OUT=gpurun_out/r02u; mkdir -p $OUT
L=paper_2412_12308_b200/libfftpde.so
cp tools/ab/lib_push.so $L
timeout 300 python tools/solve_once.py c3 0 > $OUT/push_solve.log 2>&1; echo "push solve $?"; tail -2 $OUT/push_solve.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -m gpu -q -x -k "wave or c3" > $OUT/push_pytest.log 2>&1; echo "push pytest $?"; tail -2 $OUT/push_pytest.log
bash tools/ab_variants.sh $OUT c3 2 tools/ab/lib_base.so tools/ab/lib_push.so
