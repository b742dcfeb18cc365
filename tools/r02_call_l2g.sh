set -u
OUT=gpurun_out/r02g; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c4 or poisson or batch" > $OUT/pytest.log 2>&1; echo "pytest $?"; tail -1 $OUT/pytest.log
for r in 1 2; do for g in 0 -1 8 16 32 64; do
  if [ $g = -1 ]; then unset FFTPDE_L2GROUP; else export FFTPDE_L2GROUP=$g; fi
  timeout 600 python bench.py --workload c4 --no-cpu-baseline --no-e2e --no-parity 2>/dev/null | tail -1 > $OUT/ab_$g.json
  python -c "import json; d=json.load(open('$OUT/ab_$g.json')); print('L2GROUP=$g', round(d['ms_per_step'],4), d['gpu_launches'], {k: v['ms_per_launch'] for k, v in d['roofline']['per_kernel'].items()})"
done; done
