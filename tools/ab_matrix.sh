#!/bin/bash
# tools/ab_matrix.sh "ENV=..." lib1.so lib2.so ... : every (env, lib) pair, alternating, twice
L=paper_2412_12308_b200/libfftpde.so
cp $L /tmp/ab_base.so
ENVS="$1"; shift
python tools/c5_prof.py 4 > /dev/null
for rep in 1 2; do
  for v in "$@"; do for e in $ENVS; do cp $v $L; echo "$v [$e]: $(env $e python tools/c5_prof.py 20 | sed 's/"launches".*//; s/"env": {[^}]*}, //')"; done; done
done
cp /tmp/ab_base.so $L
