set -u
OUT=gpurun_out/r02x; mkdir -p $OUT
timeout 300 python tools/solve_once.py c3 0 > $OUT/solve.log 2>&1; echo "solve $?"; tail -3 $OUT/solve.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -m gpu -q -x -k "wave or c3" > $OUT/pytest.log 2>&1; echo "pytest $?"; tail -15 $OUT/pytest.log
bash tools/ab_variants.sh $OUT c3 1 tools/ab/lib_base.so tools/ab/lib_wavet.so
