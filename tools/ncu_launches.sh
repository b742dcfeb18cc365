#!/bin/bash
# Launch list (gpu__time_duration per launch) of the default bench command.
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > "$OUT/plain_launches.log" 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches_c2.csv" $CMD \
  > "$OUT/ncu_launches.log" 2>&1
echo "launch list $?"
