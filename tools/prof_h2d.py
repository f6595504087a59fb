"""H2D throughput of a stream of per-step copies (pinned -> device), the
persistent runner's upload pattern: one cudaMemcpyAsync (+ event) per step
issued from C (cuda-python bindings), on 1 or 2 streams."""
import sys
import time

import torch
from cuda.bindings import runtime as rt

sizes = [int(x) for x in (sys.argv[1:] or ["458752", "2490368"])]
dev = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
host = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
_, s0 = rt.cudaStreamCreateWithFlags(1)
_, s1 = rt.cudaStreamCreateWithFlags(1)
_, ev = rt.cudaEventCreateWithFlags(2)
H2D = rt.cudaMemcpyKind.cudaMemcpyHostToDevice
for nbytes in sizes:
    for ns in (1, 2):
        N = 4000
        for rep in range(2):
            rt.cudaDeviceSynchronize()
            t0 = time.perf_counter()
            for k in range(N):
                s = s0 if ns == 1 or k % 2 == 0 else s1
                off = (k % 8) * nbytes % (48 << 20)
                rt.cudaMemcpyAsync(dev.data_ptr() + off, host.data_ptr() + off, nbytes, H2D, s)
                rt.cudaEventRecord(ev, s)
            rt.cudaDeviceSynchronize()
            dt = (time.perf_counter() - t0) / N
        print(f"{nbytes / 1024:.0f} KB x {N} on {ns} stream(s): {1e6 * dt:.2f} us/copy, "
              f"{nbytes / dt / 1e9:.1f} GB/s")
