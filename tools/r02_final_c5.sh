#!/bin/bash
# final C5 evidence: bench line, reference arm, ncu launch list of the bench command, ncu --set full of the three passes
OUT=gpurun_out/${1:-r02o}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
timeout 900 python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench exit $?"
timeout 600 python bench.py --impl reference > $OUT/bench_ref_c5.json 2> $OUT/bench_ref_c5.err; echo "ref exit $?"
KRE='regex:aa_kernel|line_kernel|by_kernel|b3_kernel|bx_kernel'
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-parity"
$CMD > $OUT/plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" --csv --log-file $OUT/launches_c5.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "launch list exit $?"
python tools/solve_once.py c5 0 > $OUT/solve.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "$KRE" -s 3 -c 3 -o $OUT/c5_full python tools/solve_once.py c5 0 > $OUT/ncu_full.log 2>&1; echo "ncu full exit $?"
