set -u
OUT=gpurun_out/r02y; mkdir -p $OUT
for v in 0 1; do
  FFTPDE_WAVET=$v timeout 600 python bench.py --workload c3 --no-cpu-baseline --no-e2e --no-parity 2>/dev/null | tail -1 > $OUT/ab_wavet$v.json
  python -c "import json; d=json.load(open('$OUT/ab_wavet$v.json')); print('WAVET=$v', round(d['ms_per_step'],3), {k: v['ms_per_launch'] for k, v in d['roofline']['per_kernel'].items()})"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wavet -s 3 -c 3 -o $OUT/wavet python tools/solve_once.py c3 0 > $OUT/ncu.log 2>&1; echo "ncu $?"
