"""PCIe per-step copy pattern of the persistent runner: a 448 KB H2D per step
on one stream with (a) nothing else, (b) a 72 KB D2H per step on a second
stream, (c) the D2H split to 20 KB (compact outputs) -- us per step."""
import time

import torch
from cuda.bindings import runtime as rt

dev = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
host = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
hout = torch.empty(16 << 20, dtype=torch.uint8).pin_memory()
_, s0 = rt.cudaStreamCreateWithFlags(1)
_, s1 = rt.cudaStreamCreateWithFlags(1)
H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost
for h2d, d2h in ((458752, 0), (458752, 72448), (458752, 20480), (393216, 0), (0, 72448)):
    N = 3000
    for rep in range(2):
        rt.cudaDeviceSynchronize()
        t0 = time.perf_counter()
        for k in range(N):
            off = (k % 8) * 524288
            if h2d:
                rt.cudaMemcpyAsync(dev.data_ptr() + off, host.data_ptr() + off, h2d, H2D, s0)
            if d2h:
                rt.cudaMemcpyAsync(hout.data_ptr() + (k % 8) * 81920,
                                   dev.data_ptr() + (32 << 20) + (k % 8) * 81920, d2h, D2H, s1)
        rt.cudaDeviceSynchronize()
        dt = (time.perf_counter() - t0) / N
    print(f"H2D {h2d / 1024:.0f} KB + D2H {d2h / 1024:.0f} KB per step: {1e6 * dt:.2f} us/step")
