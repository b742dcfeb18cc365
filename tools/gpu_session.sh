#!/bin/bash
# One gpurun session: GPU parity tests, bench lines, ncu launch list and one
# ncu --set full capture of the top kernel.  Usage (from the repo root, on the box):
#   bash tools/gpu_session.sh [tag] [stages]
# stages: any of  t (pytest -m gpu)  b (bench c2)  a (bench all workloads)
#                 l (ncu launch list)  f (ncu full, c3 wave column pass)  c (ncu full c2 rows)
set -u
TAG=${1:-r01}
STAGES=${2:-tblf}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/smi.txt" 2>&1
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { echo "build failed"; exit 1; }
if [[ $STAGES == *t* ]]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest -m gpu exit $?" ; tail -3 "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
  echo "smoke exit $?"; tail -2 "$OUT/smoke.log"
fi
if [[ $STAGES == *b* ]]; then
  timeout 600 python bench.py > "$OUT/bench_c2.json" 2> "$OUT/bench_c2.err"
  echo "bench c2 exit $?"; cat "$OUT/bench_c2.json"
fi
if [[ $STAGES == *a* ]]; then
  for w in c1 c3 c4 c5; do
    timeout 900 python bench.py --workload $w > "$OUT/bench_$w.json" 2> "$OUT/bench_$w.err"
    echo "bench $w exit $?"; cat "$OUT/bench_$w.json"
  done
  timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > "$OUT/bench_ref_c2.json" 2> "$OUT/bench_ref.err"
  echo "bench ref exit $?"
fi
if [[ $STAGES == *l* ]]; then
  CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
  $CMD > "$OUT/plain_launches.log" 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file "$OUT/launches_c2.csv" $CMD > "$OUT/ncu_launches.log" 2>&1
  echo "ncu launch list exit $?"
fi
if [[ $STAGES == *f* ]]; then
  CMD="python tools/prof_case.py wave4096"
  $CMD > "$OUT/plain_full.log" 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:col2_kernel -s 1 -c 1 \
      -o "$OUT/prof_c3_wavecol" $CMD > "$OUT/ncu_full.log" 2>&1
  echo "ncu full exit $?"
fi
if [[ $STAGES == *c* ]]; then
  CMD="python tools/prof_case.py c2"
  $CMD > "$OUT/plain_full_c2.log" 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 4 -c 2 \
      -o "$OUT/prof_c2_rows" $CMD > "$OUT/ncu_full_c2.log" 2>&1
  echo "ncu full c2 exit $?"
fi
