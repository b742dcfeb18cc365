#!/bin/bash
# bench default line, reference arm, ncu counts of the C5 solve, host memory
set -u
OUT=gpurun_out/${1:-r02j}
mkdir -p $OUT
free -g > $OUT/free.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?"
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref exit $?"
M=$(python -c "import sys; sys.path.insert(0,'tools'); import kernel_counts as k; print(k.METRICS)")
python tools/solve_once.py c5 1 > $OUT/solve_plain.log 2>&1 && \
ncu --metrics $M --clock-control none -s 61 --csv --log-file $OUT/counts_c5.csv python tools/solve_once.py c5 1 > $OUT/ncu_counts.log 2>&1; echo "ncu exit $?"
