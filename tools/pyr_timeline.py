"""Summarise an FT_DEBUG_PYR_TIMELINE dump: per mark, min / median / max
offset (us) from the earliest block start."""
import sys
import numpy as np
rows = [list(map(int, l.split()[1:])) for l in open(sys.argv[1]) if not l.startswith("launch")]
a = np.array(rows, dtype=np.float64)
t0 = a[:, 0].min()
for k in range(a.shape[1]):
    v = a[:, k]
    v = v[v > 0]
    if len(v):
        d = (v - t0) / 1e3
        print(f"mark {k:2d}: n={len(v):4d} min={d.min():7.2f} med={np.median(d):7.2f} max={d.max():7.2f} us")
