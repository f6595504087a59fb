"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
launches, median and total time per kernel, share of the process's GPU time
and of our kernels' time.   python tools/launch_summary.py list.csv out.txt "header" """
import collections
import csv
import statistics
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path, out, header=""):
    rows = list(csv.reader(open(path)))
    i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[i]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                           "Metric Unit"))
    d = collections.defaultdict(list)
    for r in rows[i + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            d[r[ki]].append(float(r[vi].replace(",", "")) * UNIT[r[ui]])
    tot = sum(sum(v) for v in d.values())
    ours = {k: v for k, v in d.items() if "ft::" in k or "unnamed" in k or "bench_popc" in k}
    tot_ours = sum(sum(v) for v in ours.values())
    lines = [header, "", f"{'kernel':60s} {'launches':>8s} {'median us':>10s} {'total us':>10s} "
             f"{'share':>6s}"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1]))[:14]:
        lines.append(f"{k[:60]:60s} {len(v):8d} {statistics.median(v):10.2f} {sum(v):10.1f} "
                     f"{100 * sum(v) / tot:5.1f}%")
    lines += ["", "share of our kernels' time: " + ", ".join(
        f"{k.split('(')[0]} {100 * sum(v) / tot_ours:.1f}%"
        for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])))]
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:])
