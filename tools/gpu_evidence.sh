#!/bin/bash
# Round evidence, part 1 (no profiler): build, smoke, every bench line, the
# reference arm.  The ncu captures run as separate gpurun calls
# (tools/ncu_launches.sh, tools/ncu_full.sh), one profiler run per call.
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { echo "build failed"; exit 1; }
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke $?"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > "$OUT/smi.txt" 2>&1
for w in c2 c1 c3 c4 c5 c2r c3r c4r rk4 rk4big dsrc p3d d3d; do
  timeout 900 python bench.py --workload $w > "$OUT/bench_$w.json" 2> "$OUT/bench_$w.err"; echo "bench $w $?"
done
for ex in lib peer nccl fused; do
  timeout 600 python bench.py --workload c5 --sharded --exchange $ex > "$OUT/bench_c5_sharded_p1_$ex.json" 2> "$OUT/bench_c5_sh_$ex.err"; echo "c5 sharded $ex $?"
done
for w in d3d p3d; do
  timeout 600 python bench.py --workload $w --sharded > "$OUT/bench_${w}_sharded_p1.json" 2> "$OUT/bench_${w}_sh.err"; echo "$w sharded $?"
done
timeout 600 python bench.py --impl reference > "$OUT/bench_ref_c2.json" 2> "$OUT/bench_ref.err"; echo "ref $?"
