#!/bin/bash
OUT=gpurun_out/${1:-r02n}; mkdir -p $OUT
for ex in fused nccl lib peer; do
  timeout 600 python bench.py --sharded --exchange $ex --steps 2 --warmup 3 > $OUT/bench_c5_sharded_$ex.json 2> $OUT/bench_c5_sharded_$ex.err; echo "sharded $ex exit $?"
done
for w in d3d rk4 c2r dsrc; do
  timeout 600 python bench.py --workload $w --steps 2 --warmup 3 > $OUT/bench_$w.json 2> $OUT/bench_$w.err; echo "$w exit $?"
done
timeout 600 python bench.py --workload d3d --sharded --steps 2 --warmup 3 > $OUT/bench_d3d_sharded.json 2> $OUT/bench_d3d_sharded.err; echo "d3d sharded exit $?"
timeout 300 python bench.py --impl reference --gpus 1 --steps 2 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref exit $?"
