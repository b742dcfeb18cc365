#!/bin/bash
# A/B of library builds on one workload, alternating: tools/ab_variants.sh OUT WORKLOAD ROUNDS base.so variant1.so ...
# each run: bench.py --workload W (no e2e / cpu baseline / parity), ms_per_step and per-class ms per launch
OUT=$1; W=$2; R=$3; shift 3
L=paper_2412_12308_b200/libfftpde.so
mkdir -p $OUT; cp $L /tmp/ab_keep.so
for r in $(seq $R); do
  for v in "$@"; do
    cp $v $L
    timeout 600 python bench.py --workload $W --no-cpu-baseline --no-e2e --no-parity 2>/dev/null | tail -1 > $OUT/ab_${W}_$(basename $v .so)_$r.json
    python -c "import json,sys; d=json.loads(open('$OUT/ab_${W}_$(basename $v .so)_$r.json').read()); print('$W', '$(basename $v)', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k: v['ms_per_launch'] for k, v in d['roofline']['per_kernel'].items()})"
  done
done
cp /tmp/ab_keep.so $L
