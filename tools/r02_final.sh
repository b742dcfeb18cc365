#!/bin/bash
# Round-2 final evidence: GPU suite, smoke, every BASELINE config's bench line with the
# driver's flags (--steps 20 --warmup 5), the reference arm on C5, 3D pencil line.
set -u
OUT=gpurun_out/${1:-r02w}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest -m gpu exit $?"; tail -2 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $OUT/smoke.log
for w in c5 c1 c2 c3 c4; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > $OUT/bench_$w.json 2> $OUT/bench_$w.err; echo "bench $w $?"
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_ref_c5.json 2> $OUT/bench_ref_c5.err; echo "ref $?"
timeout 600 python bench.py --workload d3d --pencil 1x1 > $OUT/bench_d3d_pencil.json 2> $OUT/bench_d3d_pencil.err; echo "d3d pencil $?"
timeout 600 python bench.py --workload d3d --sharded > $OUT/bench_d3d_sharded.json 2> $OUT/bench_d3d_sharded.err; echo "d3d slab $?"
