set -u
OUT=gpurun_out/r02c4; mkdir -p $OUT
L=paper_2412_12308_b200/libfftpde.so
for v in s1m4 s1m5; do cp tools/ab/lib_$v.so $L
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c4 or poisson or batch or tma" > $OUT/pytest_$v.log 2>&1; echo "$v pytest $?"; tail -1 $OUT/pytest_$v.log
done
for r in 1 2; do for v in base s1m4 s1m5; do cp tools/ab/lib_$v.so $L
  timeout 900 python bench.py --workload c4 --no-cpu-baseline --no-e2e --no-parity 2>/dev/null | tail -1 > $OUT/ab_$v.json
  python -c "import json; d=json.load(open('$OUT/ab_$v.json')); print('$v', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], {k: v['ms_per_launch'] for k, v in d['roofline']['per_kernel'].items()})"
done; done
cp tools/ab/lib_base.so $L
