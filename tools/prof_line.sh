#!/bin/bash
# ncu --set full on single variants of tools/exp_line (filter strings), one report each
mkdir -p gpurun_out/exp
i=0
for f in "$@"; do
  i=$((i+1))
  ./tools/exp_line "$f" 3 > gpurun_out/exp/plain_$i.txt 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -s 3 -c 1 -o gpurun_out/exp/prof_$i ./tools/exp_line "$f" 3 > gpurun_out/exp/ncu_$i.log 2>&1
  echo "$i [$f] exit $?"; cat gpurun_out/exp/plain_$i.txt
done
