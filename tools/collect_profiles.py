"""Turn the outputs of tools/measure_all.sh (gpurun_out/m/) into the judged profiles/<round>/
files: bench lines, per-kernel launch shares, ncu --set full summaries, and
profiles/traffic.json (DRAM bytes per launch of each dominant kernel).

    python tools/collect_profiles.py r01 [SRC [DST_ROOT]]

On the GPU box measure_all.sh runs it with DST_ROOT=gpurun_out/m/collected (the .ncu-rep
files are summarised there and then deleted: gpurun copies back at most 64 MiB); here,
`python tools/collect_profiles.py r01 gpurun_out/m/collected/profiles/r01 .` is not needed —
copy gpurun_out/m/collected/profiles/ over profiles/.
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

from launch_share import summarise  # noqa: E402
from ncu_summary import summary  # noqa: E402

SRC = os.path.join(ROOT, "gpurun_out", "m")


def last_json(path):
    try:
        lines = [ln for ln in open(path).read().strip().splitlines() if ln.startswith("{")]
        return json.loads(lines[-1]) if lines else None
    except OSError:
        return None


def main(rnd, src=None, dst_root=None):
    global SRC
    if src:
        SRC = os.path.abspath(src)
    dst_root = os.path.abspath(dst_root) if dst_root else ROOT
    dst = os.path.join(dst_root, "profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    W = ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "p4", "imp2")
    for w in W:
        for arm in ("bench", "bench_reference"):
            d = last_json(os.path.join(SRC, f"{arm}_{w}.json"))
            if d is not None:
                json.dump(d, open(os.path.join(dst, f"{arm}_{w}.json"), "w"))
    for w in W:
        p = os.path.join(SRC, f"launches_{w}.csv")
        if os.path.exists(p):
            steps = "--steps 1" if w in ("cfg4", "cfg5", "p4", "imp2") else "--steps 2"
            out = summarise(p, f"ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --workload "
                               f"{w} {steps} --warmup 1 --no-e2e --no-cpu-baseline")
            json.dump(out, open(os.path.join(dst, f"launches_{w}.json"), "w"), indent=1)
    traffic_path = os.path.join(dst_root, "profiles", "traffic.json")
    if not os.path.exists(traffic_path) and os.path.exists(os.path.join(ROOT, "profiles", "traffic.json")):
        traffic_path_src = os.path.join(ROOT, "profiles", "traffic.json")
        os.makedirs(os.path.dirname(traffic_path), exist_ok=True)
        open(traffic_path, "w").write(open(traffic_path_src).read())
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    lib_sha = None
    try:
        lib_sha = open(os.path.join(SRC, "lib.sha")).read().split()[0][:16]
    except (OSError, IndexError):
        pass
    for w in W:
        name = f"ncu_{w}"
        rep = os.path.join(SRC, name + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        s = summary(rep)
        json.dump(s, open(os.path.join(dst, name + ".json"), "w"), indent=1)
        k = s[0]
        rd = float(k["dram__bytes_read.sum"][0]) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[
            k["dram__bytes_read.sum"][1]]
        wr = float(k["dram__bytes_write.sum"][0]) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[
            k["dram__bytes_write.sum"][1]]
        traffic[w] = {"bytes_per_launch": rd + wr, "kernel": k["kernel"][:60], "lib_sha16": lib_sha,
                      "source": f"profiles/{rnd}/{name}.json (ncu --set full, cold cache): "
                                "dram__bytes_read.sum + dram__bytes_write.sum"}
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    print("collected into", dst)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01", *sys.argv[2:4])
