#!/bin/bash
# Round evidence: all bench lines, reference arm, ncu launch list (default bench
# command) and one ncu --set full capture per dominant kernel class.
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { echo "build failed"; exit 1; }
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke $?"
for w in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --workload $w > "$OUT/bench_$w.json" 2> "$OUT/bench_$w.err"; echo "bench $w $?"
done
timeout 600 python bench.py --impl reference > "$OUT/bench_ref_c2.json" 2> "$OUT/bench_ref.err"; echo "ref $?"
# launch list of the default bench command (short)
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > "$OUT/plain_launches.log" 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches_c2.csv" $CMD > "$OUT/ncu_launches.log" 2>&1
echo "launch list $?"
CMD="python tools/prof_case.py c2"
$CMD > "$OUT/plain_c2.log" 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 4 -c 2 -o "$OUT/full_c2" $CMD > "$OUT/ncu_full_c2.log" 2>&1
echo "full c2 $?"
CMD="python tools/prof_case.py wave4096"
$CMD > "$OUT/plain_c3.log" 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"col2_kernel|pipe_kernel" -s 2 -c 2 -o "$OUT/full_c3" $CMD > "$OUT/ncu_full_c3.log" 2>&1
echo "full c3 $?"
CMD="python tools/prof_case.py c4"
$CMD > "$OUT/plain_c4.log" 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:line_kernel -s 3 -c 2 -o "$OUT/full_c4" $CMD > "$OUT/ncu_full_c4.log" 2>&1
echo "full c4 $?"
