"""profiles/traffic.json entries from ncu --set full captures of the ring
kernel (tools/r2_capture.sh): DRAM bytes per launch / per frame, duration.

    python tools/traffic_update.py PREFIX   (reads gpurun_out/PREFIX_ring_g*_k*.ncu-rep)
"""
import csv
import glob
import io
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
prefix = sys.argv[1]
tf = ROOT / "profiles" / "traffic.json"
d = json.loads(tf.read_text()) if tf.exists() else {}
for rep in sorted(glob.glob(str(ROOT / "gpurun_out" / f"{prefix}_ring_g*_k*.ncu-rep"))):
    g, k = map(int, re.search(r"_g(\d+)_k(\d+)\.ncu-rep", rep).groups())
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]

    def get(name):
        i = hdr.index(name)
        v = float(vals[i].replace(",", ""))
        u = units[i]
        return v * {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1, "usecond": 1,
                    "msecond": 1e3, "nsecond": 1e-3}.get(u, 1)
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    dur = get("gpu__time_duration.sum")
    d[f"track_persist_kernel_ring_g{g}_k{k}"] = {
        "config": f"bench.py value region: ft_track_frames_ring over the resident cfg2 pipelines "
                  f"(> 2x L2), K={k} steps in one launch, {g} step group(s)",
        "dram_bytes_read_per_launch": int(rd), "dram_bytes_write_per_launch": int(wr),
        "steps_per_launch": k, "dram_bytes_per_frame": (rd + wr) / k, "ncu_duration_us": dur,
        "source": f"ncu --set full --clock-control none --import-source on -k "
                  f"regex:track_persist_kernel -s 1 -c 1 python tools/ncu_ring.py {g} {k} "
                  f"({prefix})"}
    print(g, k, int(rd), int(wr), dur)
tf.write_text(json.dumps(d, indent=1) + "\n")
