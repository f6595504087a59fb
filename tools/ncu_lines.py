"""Per-source-line warp-stall samples of a kernel from an ncu report: the
SASS page of `ncu -i REP --page source --csv --print-source sass` joined
with the line table of `nvdisasm -gi` of the same cubin (offsets from the
kernel's first instruction).

    python tools/ncu_lines.py REP CUBIN KERNEL_MANGLED [top]
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, cubin, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
sass = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout
line_of, cur, inside, fresh = {}, None, False, True
for ln in sass.splitlines():
    if re.match(r"\s*\.text\.", ln) or ln.startswith(".text."):
        inside = kern in ln
    if not inside and f"{kern}:" in ln:
        inside = True
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', ln)
    if m:
        if not fresh:  # innermost location first, then the sites it is inlined at
            continue
        fresh = False
        f = m.group(1).split("/")[-1]
        inl = re.search(r'inlined at "([^"]+)", line (\d+)', m.group(3))
        cur = f"{f}:{m.group(2)}" + (f" <- {inl.group(1).split('/')[-1]}:{inl.group(2)}" if inl else "")
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m:
        line_of[int(m.group(1), 16)] = cur
        fresh = True
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isamp, iexe = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(rows[2][ia], 16)
agg = defaultdict(lambda: [0, 0, defaultdict(int)])
tot = 0
for r in rows[2:]:
    if len(r) <= isamp or not r[ia].startswith("0x"):
        continue
    off = int(r[ia], 16) - base
    key = line_of.get(off, "?")
    s = int(r[isamp] or 0)
    agg[key][0] += s
    agg[key][1] += int(r[iexe] or 0)
    for i in stall_cols:
        v = int(r[i] or 0)
        if v:
            agg[key][2][hdr[i][6:]] += v
    tot += s
print(f"total samples {tot}")
for key, (s, e, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    tops = ", ".join(f"{k} {v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
    print(f"{100 * s / tot:5.1f}% {s:6d} inst {e:9d}  {key}  [{tops}]")
