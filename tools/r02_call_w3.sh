set -u
OUT=gpurun_out/r02r; mkdir -p $OUT
L=paper_2412_12308_b200/libfftpde.so
cp $L /tmp/keep.so; cp tools/ab/lib_w3.so $L
timeout 300 python tools/solve_once.py c3 0 > $OUT/w3_solve.log 2>&1; echo "w3 solve $?"; tail -2 $OUT/w3_solve.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "wave or c3" > $OUT/w3_pytest.log 2>&1; echo "w3 pytest $?"; tail -3 $OUT/w3_pytest.log
cp /tmp/keep.so $L
bash tools/ab_variants.sh $OUT c3 2 tools/ab/lib_base.so tools/ab/lib_w3.so
