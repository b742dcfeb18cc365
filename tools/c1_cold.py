"""Cold-L2 cost of one C1 solve: events around single solves after an L2 flush,
with and without the flush, and the flush itself."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_12308_b200 import fftpde as F, inputs as I
d = I.c1_inputs(64)
p = F.Plan(64, 64)
x = torch.from_numpy(d.rho).cuda(); o = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for mode in ("flush", "warm", "flush+sync", "partial-flush-16MiB"):
    ts = []
    for i in range(30):
        if mode != "warm":
            if mode == "partial-flush-16MiB":
                flush[: 16 << 20].zero_()
            else:
                flush.zero_()
        if mode == "flush+sync":
            torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); p.poisson(x, out=o); b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    print(f"{mode:22s} median {ts[len(ts)//2]:.1f} us  min {ts[0]:.1f} us")

# bench-like: steps back to back, one sync at the end
for rep in range(3):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
    torch.cuda.synchronize()
    for a, b in ev:
        flush.zero_()
        a.record(s); p.poisson(x, out=o); b.record(s)
    torch.cuda.synchronize()
    print("bench-like steps:", " ".join(f"{a.elapsed_time(b) * 1e3:.1f}" for a, b in ev), "us")
