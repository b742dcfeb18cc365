#!/bin/bash
# A/B of two library builds: tools/ab_lib.sh <variant.so> <workload>...  (swaps libfftpde.so)
L=paper_2412_12308_b200/libfftpde.so
V=$1; shift
cp $L /tmp/ab_base.so
for tag in base variant; do
  if [ $tag = variant ]; then cp $V $L; else cp /tmp/ab_base.so $L; fi
  for w in "$@"; do
    timeout 500 python bench.py --workload $w --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w $tag', round(d['ms_per_step'],4), d['roofline'].get('per_kernel_ms_per_step'))"
  done
done
cp /tmp/ab_base.so $L
