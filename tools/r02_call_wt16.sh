set -u
OUT=gpurun_out/r02z; mkdir -p $OUT
L=paper_2412_12308_b200/libfftpde.so
cp tools/ab/lib_wt16.so $L
FFTPDE_WAVET=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "wave or c3" > $OUT/pytest16.log 2>&1; echo "wt16 pytest $?"; tail -1 $OUT/pytest16.log
for r in 1 2; do for v in wt32:0 wt32:1 wt16:1; do lib=${v%%:*}; w=${v#*:}; cp tools/ab/lib_$lib.so $L
  FFTPDE_WAVET=$w timeout 600 python bench.py --workload c3 --no-cpu-baseline --no-e2e --no-parity 2>/dev/null | tail -1 > $OUT/ab_${lib}_$w.json
  python -c "import json; d=json.load(open('$OUT/ab_${lib}_$w.json')); print('$lib WAVET=$w', round(d['ms_per_step'],2), {k: v['ms_per_launch'] for k, v in d['roofline']['per_kernel'].items()})"
done; done
cp tools/ab/lib_wt32.so $L
