#!/bin/bash
# Round evidence on one box: GPU tests, smoke, C5 bench + reference + ncu (tools/r02_final_c5.sh)
set -u
TAG=${1:-r02p}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest -m gpu exit $?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?"; tail -2 $OUT/smoke.log
bash tools/r02_final_c5.sh $TAG
