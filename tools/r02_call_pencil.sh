set -u
OUT=gpurun_out/r02v; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_sharded.py -m gpu -q -x > $OUT/pencil_pytest.log 2>&1; echo "sharded pytest $?"; tail -15 $OUT/pencil_pytest.log
