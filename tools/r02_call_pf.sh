# A/B: the C3 wave column pass with its propagator rows prefetched (FFTPDE_WAVE2_PF=1: L2, 2: L1) or read past L1
# (FFTPDE_WAVE2_NA=1) vs the base build; usage: tools/r02_call_pf.sh OUT variant...
set -u
OUT=gpurun_out/$1; shift; mkdir -p $OUT
L=paper_2412_12308_b200/libfftpde.so
libs="tools/ab/lib_base.so"
for v in "$@"; do
  cp tools/ab/lib_$v.so $L
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "wave or c3" > $OUT/pytest_$v.log 2>&1; echo "$v pytest $?"; tail -1 $OUT/pytest_$v.log
  libs="$libs tools/ab/lib_$v.so"
done
bash tools/ab_variants.sh $OUT c3 3 $libs
cp tools/ab/lib_base.so $L
