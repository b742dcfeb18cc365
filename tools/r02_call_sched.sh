# A/B: cluster scheduling policy of the C3 wave pass (FFTPDE_WAVE2_SCHED = 0 default, 1 spread, 2 load balancing)
set -u
OUT=gpurun_out/r02s; mkdir -p $OUT
for r in 1 2 3; do for v in 0 1 2; do
  FFTPDE_WAVE2_SCHED=$v timeout 600 python bench.py --workload c3 --no-cpu-baseline --no-e2e --no-parity 2>/dev/null | tail -1 > $OUT/ab_c3_sched${v}_$r.json
  python -c "import json; d=json.loads(open('$OUT/ab_c3_sched${v}_$r.json').read()); print('c3 sched=$v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k: v['ms_per_launch'] for k, v in d['roofline']['per_kernel'].items()})"
done; done
FFTPDE_WAVE2_SCHED=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "wave or c3" > $OUT/pytest_sched1.log 2>&1; echo "sched1 pytest $?"; tail -1 $OUT/pytest_sched1.log
