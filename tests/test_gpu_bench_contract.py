"""bench.py's JSON line (the driver's contract) on the B200: the keys, their
types, and the invariants the judge checks (W >= 3, one line, e2e with its byte
counts, roofline against the measured peak, clocks sampled, our kernels counted).
The reference arm (the oracle) must print the same metric with impl=reference."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench(*args):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_native_line():
    d = bench("--workload", "c2", "--steps", "2", "--warmup", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "cpu_baseline", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["dtype"] == "f64"
    assert d["config"]["workload"].startswith("c2") and "l2" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 1024 * 1024 * 16 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "l2", "alu") and r["unit"] == ("GFP64inst/s" if r["bound"] == "alu" else "GB/s")
    assert 0 < r["frac"] < 1.2 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    st = r["step"]                                     # the whole step against the method's own bytes
    assert st["alg_bytes"] == 2 * 200 * 1024 * 1024 * 16 and 0 < st["alg_frac"] <= st["design_frac"]
    for k in r["per_kernel"].values():
        assert k["bound"] in ("hbm", "l2", "alu") and k["ms_per_launch"] > 0
    p = d["parity"]                                     # the oracle on the same input (cpu_baseline leg)
    assert p["rel_l2"] <= 1e-12 and p["mean_drift"] <= 1e-12
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    assert d["clocks"]["sm_mhz"] > 0 and isinstance(d["clocks"]["reasons"], list)
    assert d["gpu_launches"] == 2 * 200 * 2           # 2 steps x 200 solve steps x (row + column pass)


def test_reference_line():
    d = bench("--impl", "reference", "--workload", "c2", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["config"]["workload"] == "c2_diffusion_1024" and d["metric"].startswith("2D FFT-PDE")
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_default_is_c5_with_parity_and_same_config_reference():
    """The default line is C5 (the largest single-GPU config), with the closed-form
    parity and a reference arm carrying the identical config."""
    d = bench("--steps", "1", "--warmup", "3", "--no-e2e", "--no-cpu-baseline")
    assert d["config"]["workload"] == "c5_diffusion_32768" and d["n_gpus"] == 1
    assert d["parity"]["rel_l2"] <= 1e-12 and d["parity"]["mean_drift"] <= 1e-12 and d["parity"]["pass"]
    assert d["roofline"]["kernel"] in d["roofline"]["per_kernel"]
    ref = bench("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert ref["config"] == d["config"] and "c5_diffusion_32768" in ref["cpu_baseline"]["sample"]
