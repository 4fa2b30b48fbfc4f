"""Slab decomposition on ONE GPU: K slabs of a BASELINE workload in one process
(paper_2504_03074_b200.slab.LocalHalo, device-to-device halo copies), timed
against the whole-grid context.  What it measures is the cost of the slab
schedule itself — region-split launches (boundary planes first, then the
interior), the per-pass halo copies and host-driven passes without a CUDA
graph — i.e. the per-GPU efficiency of the multi-GPU path before the NVLink
transfer (which the multi-GPU schedule overlaps with the interior planes).

    python tools/slab_local_bench.py --workload cfg4 --slabs 1 2 4 8 --iters 3
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--slabs", type=int, nargs="+", default=[1, 2])
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--no-whole", action="store_true")
    ap.add_argument("--graph", action="store_true", help="with --halo peer: one CUDA graph per slab iteration")
    ap.add_argument("--halo", choices=["local", "peer"], default="local",
                    help="local: LocalHalo (event-ordered device copies); peer: PeerHalo.local_group "
                         "(copies into the neighbours' ghost planes on each slab's stream, stream flags)")
    a = ap.parse_args()

    import torch

    import bench
    from paper_2504_03074_b200 import _native
    from paper_2504_03074_b200.slab import DeviceShard, LocalHalo, exchange_forcing, run_local_solve, slab_ranges

    g, f, corr, cfg, _ = bench.build_workload(a.workload)
    fv = np.asarray(f.values)
    sched = __import__("paper_2504_03074_b200").time_schedule(corr, cfg)
    n_t = sched["n_total"]
    out = {"workload": a.workload, "grid": list(g.shape), "N_t": n_t, "iters": a.iters, "runs": []}

    if not a.no_whole:
        from paper_2504_03074_b200.grid import operator_coefficients

        ctx = _native.Context(g.shape)
        ctx.set_operator(*operator_coefficients(g, 2, 1.0))
        ctx.set_schedule(0, sched)
        ctx.upload(_native.F, fv)
        ctx.zero(_native.V)
        ctx.fpi(1)
        ctx.synchronize()
        t0 = time.perf_counter()
        r = ctx.fpi(a.iters)
        ctx.synchronize()
        dt = time.perf_counter() - t0
        out["runs"].append({"slabs": "whole-grid whb_fpi (graph)", "gpts": g.size * n_t * a.iters / dt / 1e9,
                            "resid_sq_last": float(np.asarray(r).ravel()[-1])})
        ref_v = ctx.download(_native.V)
        ctx.close()
        del ctx
    for k in a.slabs:
        ranges = slab_ranges(g.shape[0], k)
        shards = [DeviceShard(g, rr) for rr in ranges]
        for sh, (p0, p1) in zip(shards, ranges):
            sh.set_schedule(sched)
            sh.upload(_native.F, np.ascontiguousarray(fv[p0:p1]))
            sh.zero(_native.V)
        if a.halo == "peer":
            from paper_2504_03074_b200.slab import PeerHalo, run_peer_local_solve

            halo = PeerHalo.local_group(shards)
            solve = lambda: run_peer_local_solve(shards, halo)  # noqa: E731
            if a.graph:
                from paper_2504_03074_b200.slab import PeerSlabGraphs

                exchange_forcing(shards, halo)
                for h, sh in zip(halo, shards):
                    h.epoch_end(sh)
                pg = PeerSlabGraphs(shards, halo)  # warm-up + capture (the warm-up is the first iterate)
                solve = pg.iterate
        else:
            halo = LocalHalo(shards)
            solve = lambda: run_local_solve(shards, halo)  # noqa: E731
        if not (a.halo == "peer" and a.graph):
            exchange_forcing(shards, halo)
            solve()  # warm-up pass (also the first FPI iterate)
        for sh in shards:
            sh.synchronize()
        l0 = sum(sh.ctx.launch_count() for sh in shards)
        t0 = time.perf_counter()
        sums = [sum(solve()) for _ in range(a.iters)]
        for sh in shards:
            sh.synchronize()
        dt = time.perf_counter() - t0
        launches = sum(sh.ctx.launch_count() for sh in shards) - l0
        row = {"slabs": k, "halo": a.halo + ("+graph" if a.graph else ""), "steps_per_pass": shards[0].pass_steps, "gpts": g.size * n_t * a.iters / dt / 1e9,
               "launches_per_iter": launches / a.iters, "resid_sq_last": sums[-1]}
        if not a.no_whole:
            v = np.concatenate([sh.download(_native.V) for sh in shards], axis=0)
            row["bitwise_equal_whole_grid"] = bool(np.array_equal(v, ref_v))
        out["runs"].append(row)
        for sh in shards:
            sh.ctx.close()
        del shards, halo
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
