#!/bin/bash
# GPU session: pytest -m gpu, smoke, bench lines c1-c4, ncu instruction/DRAM counts per workload
set -u
TAG=${1:-r02k}; STAGES=${2:-tsbc}
OUT=gpurun_out/$TAG
mkdir -p $OUT
KRE='regex:aa_kernel|line_kernel|by_kernel|bx_kernel|pipe_kernel|tma_cols_kernel|tma_wave2_cols_kernel|col2_kernel|row2d_kernel|small_solve_kernel|col_wave_kernel'
if [[ $STAGES == *t* ]]; then
  timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > $OUT/pytest_gpu.log 2>&1
  echo "pytest -m gpu exit $?"; tail -25 $OUT/pytest_gpu.log
fi
if [[ $STAGES == *s* ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?"; tail -2 $OUT/smoke.log
fi
if [[ $STAGES == *b* ]]; then
  for w in c1 c2 c3 c4; do
    timeout 900 python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err; echo "bench $w exit $?"
  done
fi
if [[ $STAGES == *c* ]]; then
  M=$(python -c "import sys; sys.path.insert(0,'tools'); import kernel_counts as k; print(k.METRICS)")
  for w in c5 c2 c3 c4 c1; do
    python tools/solve_once.py $w 0 > $OUT/solve_$w.log 2>&1 && \
    timeout 900 ncu --metrics $M --clock-control none -k "$KRE" --csv --log-file $OUT/counts_$w.csv python tools/solve_once.py $w 0 > $OUT/ncu_counts_$w.log 2>&1
    echo "ncu counts $w exit $?"
  done
fi
