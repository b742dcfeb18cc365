"""bench.py host logic on CPU (no GPU): the self-launch of --gpus N, the reference
arm's config, and the roofline arithmetic (bound choice, per-pass vs method bytes)."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2412_12308_b200 import inputs as I  # noqa: E402


def test_gpus_n_self_launches_torchrun(monkeypatch):
    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2", "--warmup", "3"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert e.value.code == 0 and len(calls) == 1
    cmd = calls[0]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"] and "--nproc-per-node=4" in cmd
    assert "127.0.0.1" in cmd and cmd[-6:] == ["--gpus", "4", "--steps", "2", "--warmup", "3"]


def test_world_size_must_match_gpus(monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2"])
    monkeypatch.setenv("WORLD_SIZE", "4")
    with pytest.raises(SystemExit, match="WORLD_SIZE=4"):
        bench.main()


def test_reference_config_is_the_native_config():
    wl = I.WORKLOADS["c5"]
    sub, host = bench.c5_sample_workload(wl)
    assert sub.nx == 8192 and sub.D == wl.D and sub.dt == wl.dt   # the bounded sample keeps D and dt
    cfg = bench.workload_config(wl, 1)
    assert cfg["workload"] == "c5_diffusion_32768" and cfg["nx"] == 32768 and cfg["nsteps"] == 20


def test_roofline_bound_and_byte_accounting():
    # C5 four-step: three classes; the step's method bytes are counted once
    wl = I.WORKLOADS["c5"]
    prof = {"row_pass": (20 * 8.0, 20), "col_pass": (20 * 8.4, 20), "aa_pass": (21 * 11.0, 21)}
    r = bench.roofline_block(wl, prof, 20 * 8.0 + 20 * 8.4 + 21 * 11.0, 1)
    field = 32768 * 32768 * 16
    assert r["kernel"] == "aa_pass" and r["unit"] == "GB/s" and not r["l2_resident"]
    assert r["per_kernel"]["row_pass"]["pass_bytes_per_launch"] == 2 * field
    assert abs(r["per_kernel"]["aa_pass"]["pass_bytes_per_launch"] - (4 + 3 * 19) / 21 * field) < 1
    assert r["step"]["alg_bytes"] == 2 * field * 20
    assert abs(r["step"]["design_round_trips"] - (61 / 21 * 21 + 40 + 40) / 40) < 1e-3
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    # an L2-resident field (C2) is measured against the L2 roof, and is ALU-bound with the counts
    wl2 = I.WORKLOADS["c2"]
    r2 = bench.roofline_block(wl2, {"row_pass": (200 * 0.0106, 200), "col_pass": (200 * 0.0108, 200)},
                              200 * 0.0214, 1)
    assert r2["l2_resident"] and r2["bound"] in ("l2", "alu")
    if os.path.exists(os.path.join(ROOT, "profiles", "counts_c2_diffusion_1024.json")):
        assert r2["bound"] == "alu" and r2["unit"] == "GFP64inst/s"
