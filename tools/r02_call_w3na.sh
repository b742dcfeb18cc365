set -u
OUT=gpurun_out/r02t; mkdir -p $OUT
L=paper_2412_12308_b200/libfftpde.so
bash tools/ab_variants.sh $OUT c3 1 tools/ab/lib_base.so tools/ab/lib_w3.so tools/ab/lib_w3na.so
cp tools/ab/lib_w3na.so $L
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tma_wave3 -s 2 -c 1 -o $OUT/w3na python tools/solve_once.py c3 0 > $OUT/ncu_w3na.log 2>&1; echo "ncu w3na $?"
cp tools/ab/lib_base.so $L
