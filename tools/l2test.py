import torch, time
for mb in (4, 16):
    n = mb * 2**20 // 16
    a = torch.randn(n, dtype=torch.complex128, device="cuda"); b = torch.empty_like(a)
    for _ in range(5): b.copy_(a)
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); s.record()
    t0 = time.perf_counter()
    for _ in range(100): b.copy_(a)
    t1 = time.perf_counter()
    e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e) / 100
    print(f"eager copy {mb:4d} MiB: {t*1e3:8.2f} us/launch (host issue {1e6*(t1-t0)/100:.2f} us/launch)")
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3): b.copy_(a)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            for _ in range(100): b.copy_(a)
    torch.cuda.synchronize()
    g.replay(); torch.cuda.synchronize()
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    print(f"graph copy {mb:4d} MiB: {s.elapsed_time(e)/100*1e3:8.2f} us/launch")
