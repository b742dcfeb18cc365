#!/bin/bash
# A/B of library builds on the C5 solve (alternating, twice each; the first run of a
# call is often slower): tools/ab_c5.sh variant.so ...
L=paper_2412_12308_b200/libfftpde.so
cp $L /tmp/ab_base.so
python tools/c5_prof.py 4 > /dev/null   # warm the box
for rep in 1 2; do
  cp /tmp/ab_base.so $L; echo "base: $(python tools/c5_prof.py 20 | sed 's/"launches".*//')"
  for v in "$@"; do cp $v $L; echo "$v: $(python tools/c5_prof.py 20 | sed 's/"launches".*//')"; done
done
cp /tmp/ab_base.so $L
