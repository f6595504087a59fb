"""Per-block phase timeline of one steady-state step of the persistent track
kernel (the last of N back-to-back steps, 4 slots, no H2D):
    python tools/persist_timeline.py [N] [empty|ranges]"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
tl_path = "/tmp/persist_tl.txt"
os.environ["FT_DEBUG_TIMELINE"] = tl_path
os.environ["FT_DEBUG_PERSIST"] = "/tmp/persist_ts.txt"
if os.path.exists(tl_path):
    os.remove(tl_path)
sys.argv = [sys.argv[0], sys.argv[1] if len(sys.argv) > 1 else "3000", "4"] + sys.argv[2:]
mode = sys.argv[3] if len(sys.argv) > 3 else "empty"

import runpy  # noqa: E402

os.environ["PERSIST_TL_ONLY"] = mode
runpy.run_path(str(ROOT / "tools" / "prof_persist.py"), run_name="__main__")

lines = open(tl_path).read().strip().split("\n")
starts = [i for i, ln in enumerate(lines) if ln.startswith("launch")]
hdr = lines[starts[-1]]
T = np.array([[int(x) for x in ln.split()[1:]] for ln in lines[starts[-1] + 1:]],
             dtype=np.float64)
print(hdr)
Gs = int(hdr.split("Gs=")[1].split()[0])
Gm = int(hdr.split("Gm=")[1].split()[0])
per = Gs + Gm
t0 = T[:, 0][T[:, 0] > 0].min()
names = {"stereo": ["start", "staged+csr", "phase1/2 done", "barrier", "end", "-", "table landed",
                    "-", "w0 kp loaded", "w0 phase1", "w0 right strip", "w0 sweep", "w0 out",
                    "gathered", "median"],
         "map": ["start", "staged+csr+hash", "projected", "searched", "barrier", "end",
                 "table landed", "points landed"]}
for role, sel in (("stereo", [i for i in range(len(T)) if i % per < Gs]),
                  ("map", [i for i in range(len(T)) if i % per >= Gs])):
    R = T[sel]
    print(f"== {role}: {len(sel)} blocks (us since first block start)")
    for k, name in enumerate(names[role]):
        col = R[:, k]
        col = col[col > 0]
        if len(col) == 0:
            continue
        rel = (col - t0) / 1e3
        print(f"  {name:18s} min {rel.min():7.2f}  med {np.median(rel):7.2f}  max {rel.max():7.2f}")
