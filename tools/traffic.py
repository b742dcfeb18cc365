"""DRAM traffic per launch, per kernel class, from an `ncu --set full` report.

usage: python tools/traffic.py REPORT.ncu-rep WORKLOAD [OUT.json]

Reads dram__bytes_read.sum + dram__bytes_write.sum of every captured launch
(`ncu -i REPORT --page raw --csv`), maps each kernel to the class names that
`fftpde_read_profile` / bench.py use (row_pass, col_pass, wave_col_pass,
small_solve, pointwise) and writes {class: mean bytes per launch} plus the
provenance to profiles/traffic_<WORKLOAD>.json, which bench.py reads into
roofline.traffic.  Note: ncu flushes caches before every replay, so these are
cold-cache bytes (an L2-resident field is read from DRAM here but not in the
timed loop)."""
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def targs(name):
    m = re.search(r"<(.*)>\(", name) or re.search(r"<(.*)>", name)
    if not m:
        return []
    return [a.strip().split(")")[-1] for a in m.group(1).split(",")]


def classify(name):
    base = re.sub(r"^.*::", "", name.split("<")[0]).strip().split()[-1]
    a = targs(name)
    if base == "small_solve_kernel":
        return "small_solve"
    if base in ("row2d_kernel", "rc_rows_kernel"):
        return "row_pass"
    if base in ("wave_line_kernel", "col_wave_kernel", "tma_wave_cols_kernel", "tma_wave2_cols_kernel"):
        return "wave_col_pass"
    if base in ("col2_kernel", "col2_phase_kernel"):
        return "wave_col_pass" if len(a) > 3 and a[3] == "4" else "col_pass"
    if base == "pipe_kernel":            # <T, N, W, COLS, OP, ...>
        return "col_pass" if len(a) > 3 and a[3] in ("1", "true") else "row_pass"
    if base == "tma_cols_kernel":
        return "col_pass"
    if base == "line_kernel":            # <T, N, E, W, COLS, OP, MINB>
        return "col_pass" if len(a) > 4 and a[4] in ("1", "true") else "row_pass"
    if base in ("kop_kernel", "src_kernel", "rk4_kernel", "mean_kernel"):
        return "pointwise"
    return base


def main():
    rep, wl = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "profiles", f"traffic_{wl}.json")
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h = rows[0]
    ki, rd, wr = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    fp = next((h.index(m) for m in ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",) if m in h), None)
    fp32 = next((h.index(m) for m in ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",) if m in h),
                None)
    units = rows[1]

    def val(row, i):
        v = float(row[i].replace(",", ""))
        u = units[i].strip().lower()
        return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)

    acc, pipes = {}, {}
    for row in rows[2:]:
        cls = classify(row[ki])
        acc.setdefault(cls, []).append((val(row, rd) + val(row, wr), row[ki][:160]))
        if fp is not None:
            pipes.setdefault(cls, []).append((float(row[fp].replace(",", "")),
                                              float(row[fp32].replace(",", "")) if fp32 is not None else 0.0))
    res = {c: round(sum(b for b, _ in v) / len(v)) for c, v in acc.items()}
    # pipe utilisation of the class: FP64 pipe, FP32 FMA pipe, % of peak while active
    res["_pipe_pct"] = {c: {"fp64": round(sum(a for a, _ in v) / len(v), 1), "fp32_fma": round(sum(b for _, b in v) / len(v), 1)}
                        for c, v in pipes.items()}
    res["_launches"] = {c: len(v) for c, v in acc.items()}
    res["_kernels"] = {c: sorted({k for _, k in v}) for c, v in acc.items()}
    res["_source"] = ("ncu --set full --clock-control none (caches flushed before each replay): "
                      "dram__bytes_read.sum + dram__bytes_write.sum per launch, mean over the captured launches; "
                      + os.path.basename(rep))
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if not k.startswith("_") or k == "_pipe_pct"}))


if __name__ == "__main__":
    main()
