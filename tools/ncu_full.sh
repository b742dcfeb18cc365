#!/bin/bash
# One `ncu --set full` capture of the kernels matching REGEX in the bench
# program of WORKLOAD (after the same command has exited 0 without ncu).
# usage: tools/ncu_full.sh TAG WORKLOAD REGEX [SKIP] [COUNT]
set -u
TAG=$1; W=$2; RE=$3; SKIP=${4:-4}; COUNT=${5:-4}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
CMD="python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > "$OUT/plain_full_$W.log" 2>&1 || { echo "plain run failed"; exit 1; }
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:"$RE" -s $SKIP -c $COUNT \
  -o "$OUT/full_$W" $CMD > "$OUT/ncu_full_$W.log" 2>&1
echo "full $W $?"
