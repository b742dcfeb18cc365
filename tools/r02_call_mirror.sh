set -u
OUT=gpurun_out/r02m; mkdir -p $OUT
L=paper_2412_12308_b200/libfftpde.so
cp tools/ab/lib_mirror.so $L
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "wave or c3" > $OUT/pytest.log 2>&1; echo "mirror pytest $?"; tail -1 $OUT/pytest.log
for r in 1 2; do for v in base mirror; do cp tools/ab/lib_$v.so $L
  timeout 900 python bench.py --workload c3 --no-cpu-baseline --no-e2e --no-parity 2>/dev/null | tail -1 > $OUT/ab_$v.json
  python -c "import json; d=json.load(open('$OUT/ab_$v.json')); print('$v', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {k: v['ms_per_launch'] for k, v in d['roofline']['per_kernel'].items()})"
done; done
cp tools/ab/lib_base.so $L
