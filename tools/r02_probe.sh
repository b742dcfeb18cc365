#!/bin/bash
# round-2 first probe: FP64/FP32 ALU roof with clocks sampled, then the current C5 bench line
set -u
OUT=gpurun_out/r02a
mkdir -p $OUT
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > $OUT/fp64_clocks.csv &
SMI=$!
./tools/fp64_peak 6 > $OUT/fp64_peak.jsonl 2>&1
kill $SMI
lscpu > $OUT/lscpu.txt; nproc > $OUT/nproc.txt
timeout 900 python bench.py --workload c5 --steps 2 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err
echo "bench c5 exit $?"
cat $OUT/fp64_peak.jsonl; cat $OUT/bench_c5.json
