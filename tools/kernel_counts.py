"""Per-launch DRAM bytes and FP instruction counts per kernel class from an ncu CSV.

usage (GPU box):
  ncu --metrics <METRICS> --clock-control none --csv --log-file gpurun_out/x.csv \
      python tools/solve_once.py <workload>
  python tools/kernel_counts.py gpurun_out/x.csv <workload-name>   # -> profiles/counts_<name>.json

Classes are the ones fftpde_read_profile / bench.py use (tools/traffic.py
classify, plus aa_pass for the four-step kernel).  dp_inst / sp_inst are thread
instructions (sass_thread_inst_executed DADD + DMUL + DFMA, FADD + FMUL + FFMA):
bench.py divides them by the measured FP64 / FP32 instruction rate for the ALU roof."""
import collections
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from traffic import classify  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ("dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
           "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,"
           "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,"
           "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum")


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3,
            "ms": 1.0, "s": 1e3, "inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9}.get(u, 1)


def main():
    path, name = sys.argv[1], sys.argv[2]
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    h = rows[hdr]
    ki, mi, ui, vi, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    kname = {}
    for r in rows[hdr + 1:]:
        try:
            v = float(r[vi].replace(",", "")) * unit_scale(r[ui])
        except ValueError:
            continue
        per[r[idi]][r[mi]] = v
        kname[r[idi]] = r[ki]
    acc = collections.defaultdict(lambda: collections.Counter())
    for lid, m in per.items():
        k = kname[lid]
        cls = ("aa_pass" if "aa_kernel" in k else "col_pass" if "by_kernel" in k or "b3_kernel<1>" in k or "b3_kernel<true>" in k
               else "row_pass" if "bx_kernel" in k or "b3_kernel<0>" in k or "b3_kernel<false>" in k else classify(k))
        a = acc[cls]
        a["launches"] += 1
        a["dram_bytes"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        a["ncu_ms"] += m.get("gpu__time_duration.sum", 0)
        a["dp_inst"] += sum(m.get(f"smsp__sass_thread_inst_executed_op_d{o}_pred_on.sum", 0) for o in ("add", "mul", "fma"))
        a["sp_inst"] += sum(m.get(f"smsp__sass_thread_inst_executed_op_f{o}_pred_on.sum", 0) for o in ("add", "mul", "fma"))
    out = {cls: {"launches": a["launches"], "dram_bytes": a["dram_bytes"] / a["launches"],
                 "dp_inst": a["dp_inst"] / a["launches"], "sp_inst": a["sp_inst"] / a["launches"],
                 "ncu_ms_per_launch": a["ncu_ms"] / a["launches"]} for cls, a in acc.items()}
    out["_source"] = {"csv": "profiles/r02/ncu/" + os.path.basename(path) + ".gz", "metrics": METRICS,
                      "note": "ncu replays with caches flushed: cold-cache DRAM bytes; per-launch means per class"}
    dst = os.path.join(ROOT, "profiles", f"counts_{name}.json")
    json.dump(out, open(dst, "w"), indent=1)
    print(dst, json.dumps({k: v for k, v in out.items() if k != "_source"}))


if __name__ == "__main__":
    main()
