set -u
OUT=gpurun_out/r02s3; mkdir -p $OUT
L=paper_2412_12308_b200/libfftpde.so
cp tools/ab/lib_split.so $L
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "wave or c3 or c2 or diffus" > $OUT/pytest.log 2>&1; echo "split pytest $?"; tail -1 $OUT/pytest.log
for r in 1 2; do for v in base split; do cp tools/ab/lib_$v.so $L
  for w in c3 c2; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > $OUT/ab_${w}_$v.json
  python -c "import json; d=json.load(open('$OUT/ab_${w}_$v.json')); p=d.get('parity') or {}; print('$w $v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k: v['ms_per_launch'] for k, v in d['roofline']['per_kernel'].items()}, {k: p[k] for k in p if 'rel' in k})"
  done
done; done
cp tools/ab/lib_base.so $L
