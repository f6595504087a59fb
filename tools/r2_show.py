"""Print the headline fields of bench lines (round-2 checks)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001
        print(f, "unreadable:", exc)
        continue
    e = d["e2e"]
    r = d["roofline"]
    print(f, "value", round(d["value"]), "G", d.get("value_ring_groups"), "graph",
          round(d["value_graph_replays"]), "e2e", round(e["value"]), e["method"],
          "lat_us", round(1e3 * (e.get("latency_ms_per_frame_e2e") or 0), 1),
          "iso_us", round(1e3 * d["latency_ms_per_frame"], 1), "frac", round(r["frac"], 4),
          "ring_ms", {k: round(v, 3) for k, v in (json.loads(
              d["value_method"].split("ring ms per G: ")[1].split(")")[0].replace("'", '"'))
              if "ring ms per G" in d["value_method"] else {}).items()})
