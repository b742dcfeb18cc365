set -u
OUT=gpurun_out/r02q; mkdir -p $OUT
bash tools/ab_variants.sh $OUT c3 2 tools/ab/lib_base.so tools/ab/lib_tws.so
bash tools/ncu_full.sh r02q c3 'tma_wave2|pipe_kernel' 4 4
M=$(python -c "import sys; sys.path.insert(0,'tools'); import kernel_counts as k; print(k.METRICS)")
KRE='regex:aa_kernel|b3_kernel'
python tools/solve_once.py c5 0 > $OUT/solve_c5.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -k "$KRE" --csv --log-file $OUT/counts_c5.csv python tools/solve_once.py c5 0 > $OUT/ncu_counts_c5.log 2>&1
echo "counts c5 $?"
