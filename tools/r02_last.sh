# last check of round 2: GPU suite, smoke, C3 and C5 lines with the driver's flags
set -u
OUT=gpurun_out/${1:-r02z}; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest -m gpu exit $?"; tail -1 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $OUT/smoke.log
for w in c3 c5; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > $OUT/bench_$w.json 2> $OUT/bench_$w.err; echo "bench $w $?"
done
