"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list into per-kernel
launch counts, mean durations and shares of device time (written as JSON for profiles/)."""
import collections
import csv
import json
import sys


def summarise(path, command, by_grid=False):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    gi = h.index("Grid Size") if "Grid Size" in h else None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        name = r[ki].split("(")[0].strip()
        if by_grid and gi is not None:
            name += f" grid{r[gi]}"
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) / 1e3
    tot = sum(v[1] for v in agg.values())
    ks = {k: {"launches": n, "mean_us": t / n, "share": t / tot}
          for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])}
    return {"command": command, "note": "cold-cache, serialised per-launch device times; compare shares, not absolutes",
            "total_us": tot, "kernels": ks}


if __name__ == "__main__":
    out = summarise(sys.argv[1], sys.argv[2], by_grid=len(sys.argv) > 3)
    print(json.dumps(out, indent=1))
