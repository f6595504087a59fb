import time, torch
torch.cuda.set_device(0)
for mb in (0.25, 0.75, 1.5, 3, 12, 48):
    n = int(mb * (1 << 20))
    h = torch.empty(n, dtype=torch.uint8).pin_memory(); d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s): d.copy_(h, non_blocking=True)
    s.synchronize()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        with torch.cuda.stream(s): d.copy_(h, non_blocking=True)
        b.record(s); s.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); t = ts[len(ts)//2]
    # two halves on two streams
    s2 = torch.cuda.Stream(); half = n // 2
    ts2 = []
    for _ in range(20):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        with torch.cuda.stream(s): d[:half].copy_(h[:half], non_blocking=True)
        with torch.cuda.stream(s2): d[half:].copy_(h[half:], non_blocking=True)
        torch.cuda.synchronize(); ts2.append(time.perf_counter() - t0)
    ts2.sort()
    print(f"{mb:6.2f} MB: 1 copy {t*1e3:7.1f} us ({n/t/1e6:6.1f} GB/s) | 2 streams wall {ts2[10]*1e6:7.1f} us")
