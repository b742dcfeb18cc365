#!/bin/bash
# distributed four-step (R28): GPU test, single-GPU C5 regression check, sharded P=1 (lib) timing
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
tag=${1:-fsd}
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q -k "distributed_fourstep" > gpurun_out/${tag}_test.log 2>&1
echo "test exit $?" >> gpurun_out/${tag}_test.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/${tag}_c5.json 2> gpurun_out/${tag}_c5.err
timeout 600 python bench.py --sharded --exchange lib --steps 3 --warmup 3 > gpurun_out/${tag}_c5_lib.json 2> gpurun_out/${tag}_c5_lib.err
tail -3 gpurun_out/${tag}_test.log
python - <<'P'
import json,glob,os
for f in sorted(glob.glob("gpurun_out/%s_c5*.json" % os.environ.get("TAG","fsd"))):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d["ms_per_step"], d.get("clocks",{}).get("sm_mhz"))
    except Exception as e: print(f, "ERR", e)
P
