"""Print the sweep results (gpurun_out/sweep/*.json): value, iters/s, last residual."""
import glob
import json
import os

for p in sorted(glob.glob(os.path.join(os.path.dirname(__file__), "..", "gpurun_out", "sweep", "*.json"))):
    try:
        d = [json.loads(l) for l in open(p) if l.startswith("{")][-1]
        print(f"{os.path.basename(p):32s} {d['value']:9.2f} Gpts/s  {d['iters_per_s']:10.1f} it/s  "
              f"res {d['residuals']['last']!r}")
    except Exception as e:  # noqa: BLE001
        print(os.path.basename(p), "FAILED", open(p.replace('.json', '.err')).read()[-300:])
