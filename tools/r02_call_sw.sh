set -u
OUT=gpurun_out/r02s; mkdir -p $OUT
L=paper_2412_12308_b200/libfftpde.so
cp tools/ab/lib_sw128.so $L
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_sw128.log 2>&1; echo "sw128 pytest $?"; tail -2 $OUT/pytest_sw128.log
bash tools/ab_variants.sh $OUT c4 2 tools/ab/lib_sw64.so tools/ab/lib_sw128.so
cp tools/ab/lib_w3s.so $L
FFTPDE_VERBOSE=1 timeout 300 python tools/solve_once.py c3 0 > $OUT/w3s_solve.log 2>&1; echo "w3s solve $?"; tail -3 $OUT/w3s_solve.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "wave or c3" > $OUT/w3s_pytest.log 2>&1; echo "w3s pytest $?"; tail -2 $OUT/w3s_pytest.log
cp tools/ab/lib_sw128.so $L
bash tools/ab_variants.sh $OUT c3 1 tools/ab/lib_sw128.so tools/ab/lib_w3s.so
