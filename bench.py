"""Benchmark: explicit WaveHoltz fixed-point iterations on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4] [--impl ours|reference]

A "step" is one WaveHoltz fixed-point iteration v <- W(v, f) (N_t fused
leapfrog+filter steps over the whole grid + the residual reduction).  The
default workload, at every N, is BASELINE config 4 -- the north-star config:
3D 1025^3 fp64, omega = 150.3, 16 seeded Gaussians, CFL 0.9, N_t = 83 -- and
the default K = 10 is that config's iteration count (the timed region is the
solve from v = 0).  N = 1 runs the whole grid on one GPU; N > 1 splits it into
z-slabs (axis-0 plane ranges, one per GPU, halo exchange overlapped with the
interior planes, strong scaling).  Inputs are resident in HBM when timing
starts; the 1025^3 working set (7 x 8.6 GB) is far above L2 (an L2 flush still
runs before every timed iteration on one GPU, outside the timed span).

value      = grid-point updates / s (N stored points x N_t x K / device time), Gpts/s
e2e        = the same through the reference-facing C-ABI call with HOST buffers:
             whb_iterate_host (paper_2504_03074_b200.HostFPIStep), v copied in from pinned
             host memory and v_new copied out every step (the reference's _iterate loop body,
             driver.py:222-226; on the three-step plan the copies move in bands of rows behind
             the passes); e2e_solve = whb_upload(f) + whb_fpi(K) +
             whb_download(v) (the fpi_solve call: f in once, residual out every step, v out
             once); e2e_seam = wave_solve_filtered(GridField, ...) -> GridField, the Python seam
             the reference's drivers call (C ABI whb_solve_host)
roofline   = the dominant (multi-step) kernel: bytes per launch / average launch duration
             (CUDA events on the launching stream) against the measured HBM peak.  ``frac``
             uses the kernel's DRAM bytes per launch from the ncu capture of THIS build
             (profiles/traffic.json, matched by the library's sha256) and falls back to the
             kernel's compulsory bytes (56/T per update for a T-step pass) when no capture of
             this build exists; ``frac_48B`` is SURVEY 8(d)'s 48 B/update figure (> 1 for
             temporally blocked kernels by construction).
cpu_baseline = numpy restatement of the reference (1 core), bounded sample
--impl reference: the C OpenMP restatement of the reference on all host cores
             (the reference is pure numpy; oracle/ holds its bitwise restatement)

--gpus N without torchrun: bench.py re-launches itself through torch.distributed.run
(one process per GPU, 127.0.0.1 rendezvous); rank 0 prints the line.

--workload imp2: the implicit (trapezoidal) path of SURVEY 8(f) rank 4 -- 2D 2049^2,
omega = 50.5, N_t = 20, 8 seeded Gaussians; each step is one implicit WaveHoltz
iteration (20 implicit steps, each a multigrid-preconditioned CG solve).

N > 1: configs 3/4 -- z-slabs ("strong"; --decomp replicas for independent copies);
config 5 -- the 64 frequencies LPT-sharded across ranks ("strong"); configs 1/2 --
every rank solves its own copy ("weak").  Time is the max over ranks.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused wave-step+filter Gpts/s and WaveHoltz iters/s; % of HBM roofline"
BYTES_PER_UPDATE = 48  # read W^n, W^{n-1}, f, acc; write W^{n+1}, acc (fp64)

WORKLOADS = {
    # name: (dim, cells, omega, forcing, iterations)
    "cfg1": (2, 128, 20.3, ("single", 100.0, 200.0, (0.4, 0.6)), 100),
    "cfg2": (2, 2048, 100.5, ("multi", 8), 50),
    "cfg3": (3, 256, 40.7, ("single", 100.0, 300.0, (0.45, 0.5, 0.55)), 30),
    "cfg4": (3, 1024, 150.3, ("multi", 16), 10),
    # SURVEY 8(f) rank 2 (not a BASELINE config): config 2 with the order-4 stencil, on the
    # general-operator kernel
    "p4": (2, 2048, 100.5, ("multi", 8), 20),
}
ORDER = {"p4": 4}  # stencil order per workload (default 2)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------------------------------
# distributed plumbing


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def init_dist(ws):
    if ws <= 1:
        return None
    import torch.distributed as dist

    backend = "nccl"
    try:
        import torch

        if not torch.cuda.is_available():
            backend = "gloo"
    except Exception:
        backend = "gloo"
    dist.init_process_group(backend=backend)
    return dist


def barrier(dist):
    if dist is not None:
        dist.barrier()


def max_over_ranks(dist, x: float) -> float:
    if dist is None:
        return x
    import torch

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]


class ClockSampler:
    def __init__(self, gpu_index: int, interval_ms: int = 100):
        q = "clocks.sm,clocks.max.sm," + ",".join(f"clocks_event_reasons.{r}" for r in REASONS)
        self.cmd = ["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                    f"-lms", str(interval_ms)]
        self.proc = None
        self.lines = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(self.cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return self
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, active = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 2 + len(REASONS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for r, v in zip(REASONS, parts[2:]):
                if v.lower().startswith("active"):
                    active.add(r)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(active), "samples": len(sm)}


# ------------------------------------------------------------------------------------------
# workload construction


def build_workload(name):
    import paper_2504_03074_b200 as wh
    from paper_2504_03074_b200 import timestep as ts

    dim, n, omega, forcing, iters = WORKLOADS[name]
    ts._COURANT[2] = 0.9  # BASELINE "CFL 0.9"
    g = wh.build_grid(dim, [(0.0, 1.0)] * dim, [n] * dim, "dirichlet")
    if forcing[0] == "single":
        f = wh.gaussian_source(g, omega, forcing[1], forcing[2], forcing[3])
    else:
        f = wh.multi_gaussian_source(g, omega, forcing[1], seed=0, slab_planes=16 if dim == 3 else 64)
    corr = wh.correct_explicit(omega, g, ORDER.get(name, 2), 1.0)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    return g, f, corr, cfg, iters


def forcing_desc(name):
    if name == "cfg5":
        return "sum of 4 Gaussians, amp U(-100,100), centre U(0.1,0.9)^2, width U(100,1000), seed 0 (shared)"
    dim, n, omega, forcing, iters = WORKLOADS[name]
    if forcing[0] == "single":
        return f"{forcing[1]}*exp(-{forcing[2]}|x-{forcing[3]}|^2)"
    return f"sum of {forcing[1]} Gaussians, amp U(-100,100), centre U(0.1,0.9)^{dim}, width U(100,1000), seed 0"


def config_for(name, iterations, ws, decomp="slab", halo="nccl", g=None, cfg=None, n_t=None):
    """The workload description both arms print (identical dicts: same_config)."""
    if name == "cfg5":
        desc = {"workload": "cfg5", "grid": [1025, 1025], "omegas": "np.linspace(10.3, 200.3, 64)",
                "N_t_sum": 10522, "iterations": iterations, "cfl": 0.9, "forcing": forcing_desc(name),
                "parallelism": (f"frequencies LPT-sharded over {ws} GPUs (batch.lpt_shard)" if ws > 1
                                else "single GPU, 64 frequencies batched"),
                "l2": "flushed before every timed iteration (256 MiB write, outside the timed span)"}
        return desc
    dim, n, omega, forcing, _ = WORKLOADS[name]
    if ws > 1 and name in ("cfg3", "cfg4") and decomp == "slab":
        par = (f"z-slab decomposition over {ws} GPUs (slab_ranges: contiguous axis-0 plane ranges), "
               + {"peer": "peer-memory halo exchange (CUDA IPC copies on the exchange stream + stream flags), "
                          "one CUDA graph per iteration",
                  "nccl": "NCCL send/recv halo exchange in the C ABI on the exchange stream, overlapped with "
                          "the interior planes, one CUDA graph per iteration",
                  "torch": "torch.distributed NCCL P2P halo exchange overlapped with the interior planes"}[halo])
    elif ws > 1:
        par = f"independent replicas x{ws}"
    else:
        par = "single GPU"
    l2 = ("working set (7 fields x 8.6 GB) far above L2; flushed before every timed iteration anyway"
          if name == "cfg4" else "flushed before every timed iteration (256 MiB write, outside the timed span)")
    return {"workload": name, "grid": [n + 1] * dim, "omega": omega, "N_t": n_t, "iterations": iterations,
            "cfl": 0.9, "order": ORDER.get(name, 2), "forcing": forcing_desc(name), "parallelism": par, "l2": l2}


def lib_sha16():
    """The build being measured: sha256 (16 hex digits) of the library's build inputs (CUDA
    sources, header, nvcc flags; _build.source_sha16 -- nvcc output itself is not byte-stable)."""
    from paper_2504_03074_b200 import _build

    try:
        return _build.source_sha16()
    except OSError:
        return None


# ------------------------------------------------------------------------------------------
# CPU baseline (numpy restatement = the reference's own numpy call sequence, 1 core)


def cpu_baseline_numpy(g, f, corr, target_s=12.0, order=2):
    from oracle import waveholtz_oracle as O

    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    fv = np.array(f.values)
    if fv.size > (1 << 25):  # 1025^3: time a slab of axis-0 planes (same per-point work, bounded RAM)
        fv = np.ascontiguousarray(fv[: max(3, (1 << 25) // fv[0].size)])
    v = np.zeros_like(fv)

    def run(nsteps):
        s = dict(sc)
        s["n_total"] = nsteps
        t0 = time.perf_counter()
        O.wave_solve_filtered(v, fv, g.spacing, s, 1.0, ["dirichlet"] * g.dim, order)
        return time.perf_counter() - t0

    t3 = run(3)
    nsteps = int(max(3, min(corr.steps_per_period, target_s / max(t3 / 3, 1e-6))))
    dt = run(nsteps)
    gpts = fv.size * nsteps / dt / 1e9
    return {"value": gpts, "unit": "Gpts/s", "cores": 1, "kind": "port",
            "sample": f"{nsteps} fused leapfrog+filter steps of a {'x'.join(map(str, fv.shape))} grid through "
                      f"oracle/waveholtz_oracle.py (the reference's numpy ufunc sequence, bitwise identical to it; "
                      f"numpy elementwise ufuncs run on 1 core); {dt:.2f} s"}


# ------------------------------------------------------------------------------------------
# our arm


def load_traffic(workload):
    """ncu DRAM bytes per launch of the workload's dominant kernel, only if captured from the
    library this process loaded (profiles/traffic.json "lib_sha16"); else None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None, "no profiles/traffic.json"
    d = json.load(open(p)).get(workload)
    if d is None:
        return None, f"no ncu capture for {workload}"
    if d.get("lib_sha16") != lib_sha16():
        return None, f"ncu capture is of another build ({d.get('lib_sha16')})"
    return d.get("bytes_per_launch"), d.get("source")


class SingleRun:
    """One problem (configs 1-4) on this rank's GPU."""

    def __init__(self, args, local):
        import paper_2504_03074_b200 as wh
        from paper_2504_03074_b200.device import DeviceProblem

        g, f, corr, cfg, _ = build_workload(args.workload)
        self.g, self.f, self.corr, self.cfg = g, f, corr, cfg
        self.order = ORDER.get(args.workload, 2)
        self.prob = wh.HelmholtzProblem(g, self.order, 1.0, cfg.omega, f)
        sched = wh.time_schedule(corr, cfg)
        self.dp = DeviceProblem(g, c=1.0, order=self.order, device=local)
        self.dp.set_schedule(sched)
        self.dp.set_forcing(f.values)
        self.ctx = self.dp.ctx
        self.n_t = sched["n_total"]
        self.npts = g.size
        self.units_per_step = self.npts * self.n_t
        self.members = 1
        self.n_t_config = self.n_t
        self.f_sha = hashlib.sha256(np.ascontiguousarray(f.values).data).hexdigest()

    def reset(self):
        from paper_2504_03074_b200 import _native

        self.ctx.zero(_native.V)

    def e2e(self, K, W, dist):
        import torch

        import paper_2504_03074_b200 as wh
        from paper_2504_03074_b200 import _native

        stepper = wh.HostFPIStep(self.prob, self.cfg, device_state=self.dp)
        bufs = [_native.PinnedBuffer(self.g.shape), _native.PinnedBuffer(self.g.shape)]
        bufs[0].array[...] = 0.0
        for i in range(W):
            stepper(bufs[i % 2].array, bufs[(i + 1) % 2].array)
        bufs[0].array[...] = 0.0
        barrier(dist)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(K):
            stepper(bufs[i % 2].array, bufs[(i + 1) % 2].array)
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        for b in bufs:
            b.free()
        return te, {"h2d_bytes_per_step": self.npts * 8, "d2h_bytes_per_step": self.npts * 8 + 8,
                    "api": "paper_2504_03074_b200.HostFPIStep (C ABI whb_iterate_host), pinned host buffers; on the "
                           "three-step plan v moves in bands of rows on copy streams behind the (pass, band) launches"}

    def e2e_seam(self, K, dist):
        """The reference-facing Python seam: v = wave_solve_filtered(v, f, cfg, corr, op) with host
        GridFields, the call the reference's _iterate makes (driver.py:222) once the seam is rebound
        (INTEGRATION.md section 1): v in and W(v, f) out through host memory every call."""
        import torch

        import paper_2504_03074_b200 as wh
        from paper_2504_03074_b200 import timestep as ts

        op = wh.DiscreteOperator(self.g, self.order, 1.0)
        v = wh.GridField.zeros(self.g)
        for _ in range(2):  # warm: forcing cached by generation, two page-locked fields in the pool
            v = wh.wave_solve_filtered(v, self.f, self.cfg, self.corr, op)
        barrier(dist)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(K):
            v = ts.wave_solve_filtered(v, self.f, self.cfg, self.corr, op)
        te = time.perf_counter() - t0
        return te, {"h2d_bytes_per_step": self.npts * 8, "d2h_bytes_per_step": self.npts * 8,
                    "api": "paper_2504_03074_b200.wave_solve_filtered(GridField v, GridField f, ...) -> new "
                           "GridField (C ABI whb_solve_host; the fields' buffers are recycled page-locked memory, "
                           "copied in bands of rows behind the passes on the three-step plan)"}

    def e2e_solve(self, K, dist):
        """The fpi_solve call through the C ABI with host buffers: f copied in from pinned memory,
        K device-resident iterations, the residual history and v copied out."""
        import torch

        from paper_2504_03074_b200 import _native

        fb, vb = _native.PinnedBuffer(self.g.shape), _native.PinnedBuffer(self.g.shape)
        fb.array[...] = self.f.values
        barrier(dist)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        self.ctx.upload(_native.F, fb.array)
        self.ctx.zero(_native.V)
        rs = self.ctx.fpi(K)
        self.ctx.download(_native.V, out=vb.array)
        te = time.perf_counter() - t0
        assert rs.shape[0] == K
        fb.free()
        vb.free()
        return te, {"h2d_bytes_per_step": self.npts * 8 / K, "d2h_bytes_per_step": self.npts * 8 / K + 8,
                    "api": "C ABI whb_upload(F) + whb_fpi(K) + whb_download(V), pinned host buffers (f in "
                           "once, v out once, the K residuals read at the end)"}


class BatchRun:
    """Config 5: the rank's LPT share of the 64 frequencies, batched on its GPU."""

    def __init__(self, args, local, ws, rank):
        import paper_2504_03074_b200 as wh
        from paper_2504_03074_b200 import timestep as ts
        from paper_2504_03074_b200.batch import BatchedFPI, lpt_shard

        ts._COURANT[2] = 0.9
        g = wh.build_grid(2, [(0.0, 1.0)] * 2, [1024, 1024], "dirichlet")
        f = wh.multi_gaussian_source(g, 150.3, 4, seed=0)
        omegas = np.linspace(10.3, 200.3, 64)
        nts = [wh.correct_explicit(w, g, 2, 1.0).steps_per_period for w in omegas]
        mine = lpt_shard(nts, ws)[rank]
        self.g = g
        self.solver = BatchedFPI(g, f, omegas[mine], device=local)
        self.ctx = self.solver.ctx
        self.npts = g.size
        self.members = len(mine)
        self.units_per_step = self.solver.updates_per_iteration
        self.n_t = sum(self.solver.steps)
        self.n_t_config = None
        self.f_sha = hashlib.sha256(np.ascontiguousarray(f.values).tobytes()).hexdigest()
        self.desc = {"grid": list(g.shape), "omegas": "np.linspace(10.3, 200.3, 64)", "N_t_sum_rank0": self.n_t,
                     "members_rank0": self.members, "sharding": "LPT over N_t (batch.lpt_shard)"}

    def reset(self):
        self.solver.reset()

    def e2e(self, K, W, dist):
        import torch

        from paper_2504_03074_b200 import _native

        B = self.members
        host = [_native.PinnedBuffer(self.g.shape) for _ in range(B)]
        for h in host:
            h.array[...] = 0.0

        def step():
            for b in range(B):
                self.ctx.upload(_native.V, host[b].array, b)
            self.ctx.fpi(1)
            for b in range(B):
                self.ctx.download(_native.V, b, out=host[b].array)

        for _ in range(W):
            step()
        for h in host:
            h.array[...] = 0.0
        barrier(dist)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(K):
            step()
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        for h in host:
            h.free()
        return te, {"h2d_bytes_per_step": B * self.npts * 8, "d2h_bytes_per_step": B * self.npts * 8 + 8 * B,
                    "api": "C ABI whb_upload / whb_fpi / whb_download per member, pinned host buffers"}


def run_slab(args, dist, ws, rank, local):
    """Configs 3/4 at N > 1: one z-slab per GPU (slab.SlabFPI; halo exchange overlapped with the
    interior planes).  Strong scaling: the grid is fixed.  --emulate-cpu runs the same driver with
    the numpy stand-in shard over gloo (CPU test of the launcher; the numbers mean nothing)."""
    from paper_2504_03074_b200 import _native
    from paper_2504_03074_b200.slab import NcclHalo, PeerHalo, SlabFPI, TorchHalo, slab_ranges

    g, f, corr, cfg, _ = build_workload(args.workload)
    rng = slab_ranges(g.shape[0], ws)[rank]
    emulate = args.emulate_cpu
    if emulate:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from slab_numpy import NumpyShard

        shard = NumpyShard(g, rng)
        halo = TorchHalo(dist, rank, ws)
    else:
        import torch

        from paper_2504_03074_b200.slab import DeviceShard

        shard = DeviceShard(g, rng, device=local)
        if args.halo == "peer":
            halo = PeerHalo.from_dist(shard, dist, rank, ws)
        elif args.halo == "nccl":
            halo = NcclHalo(shard, dist, rank, ws)
        else:
            halo = TorchHalo(dist, rank, ws)
    solver = SlabFPI(shard, halo, corr, cfg, f, graph=args.halo in ("peer", "nccl"))
    n_t = solver.shard.n_total
    K, W = args.steps, args.warmup
    for _ in range(W):
        solver.iterate()
    solver.reset()
    if not emulate:
        shard.synchronize()
    barrier(dist)
    sampler = ClockSampler(local).start() if not emulate else None
    if emulate:
        t0 = time.perf_counter()
        res = [solver.iterate() for _ in range(K)]
        dev_s = max_over_ranks(dist, time.perf_counter() - t0)
        clocks, launches = None, 0
    else:
        l0 = shard.ctx.launch_count()
        stream = torch.cuda.ExternalStream(shard.ctx.stream_ptr(), device=f"cuda:{local}")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = [solver.iterate() for _ in range(K)]
        e1.record(stream)
        e1.synchronize()
        clocks = sampler.stop()
        launches = shard.ctx.launch_count() - l0
        dev_s = max_over_ranks(dist, e0.elapsed_time(e1) / 1e3)
    units = g.size * n_t * K
    value = units / dev_s / 1e9
    peak, peak_src = peaks()
    e2e = None
    if not args.no_e2e and not emulate:
        # the reference-facing call with host buffers, every step: each rank copies its owned
        # planes of v in from pinned memory, runs one slab iteration, copies v_new out
        host = _native.PinnedBuffer(shard.ctx.local_shape)
        host.array[...] = 0.0
        solver.reset()
        shard.synchronize()
        barrier(dist)
        t0 = time.perf_counter()
        for _ in range(K):
            shard.upload(_native.V, host.array)
            solver.iterate()
            shard.ctx.download(_native.V, out=host.array)
        te = max_over_ranks(dist, time.perf_counter() - t0)
        e2e = {"value": units / te / 1e9, "unit": "Gpts/s", "h2d_bytes_per_step": g.size * 8,
               "d2h_bytes_per_step": g.size * 8 + 8 * ws, "iters_per_s": K / te,
               "api": "slab.SlabFPI with per-rank whb_upload / whb_download of the owned planes (pinned)"}
        host.free()
    if rank == 0:
        kp = getattr(shard, "pass_steps", None) or shard.steps_per_pass  # steps per pass all slabs agreed on
        own_bpu = 56.0 / kp if kp > 1 else float(BYTES_PER_UPDATE)
        per_gpu = units / ws / dev_s
        line = {
            "metric": METRIC, "value": value, "unit": "Gpts/s", "n_gpus": ws, "steps": K, "warmup": W,
            "ms_per_step": dev_s * 1e3 / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (BASELINE forcing recipe, SURVEY 8(d)); f sha256 "
                    + hashlib.sha256(np.ascontiguousarray(f.values).data).hexdigest()[:16],
            "config": config_for(args.workload, K, ws, args.decomp, args.halo, n_t=n_t),
            "iters_per_s": K / dev_s,
            "roofline": {"bound": "hbm", "achieved": own_bpu * per_gpu / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": own_bpu * per_gpu / 1e9 / peak, "traffic": None, "peak_source": peak_src,
                         "bytes_per_update": own_bpu, "steps_per_pass": kp,
                         "frac_48B": BYTES_PER_UPDATE * per_gpu / 1e9 / peak,
                         "frac_source": "compulsory bytes of the slab's multi-step passes per GPU / device wall "
                                        "time of the timed iterations (exchange and region split included)"},
            "cpu_baseline": None, "e2e": e2e, "clocks": clocks, "gpu_launches": launches,
            "residuals": {"first": res[0], "last": res[-1]}, "impl": "ours",
            **({"emulated_cpu": "numpy stand-in shard over gloo: a launcher test, not a measurement"}
               if emulate else {}),
        }
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# implicit path

IMP2 = {"cells": 2048, "omega": 50.5, "n_t": 20, "gauss": 8, "iterations": 5}


def mg_vcycle_bytes(cells):
    """Algorithmic HBM bytes of one V-cycle (nu1 = nu2 = 2) summed over the levels above the
    single-CTA coarse sub-cycle: per point of a level, 8 red-black colour sweeps x 12 B (read b and
    the other colour's u, write u; each over half the points), residual + restriction 20 B (read u,
    b; write coarse b, u), prolongation 18 B (read coarse e, read/write u)."""
    n, total = cells, 0.0
    while n > 64:
        total += (n + 1) ** 2 * (8 * 12 + 20 + 18)
        n //= 2
    return total


def build_imp2():
    import paper_2504_03074_b200 as wh

    g = wh.build_grid(2, [(0.0, 1.0)] * 2, [IMP2["cells"]] * 2, "dirichlet")
    f = wh.multi_gaussian_source(g, IMP2["omega"], IMP2["gauss"], seed=0)
    cfg = wh.FilterConfig(omega=IMP2["omega"], periods=1, steps_per_period=IMP2["n_t"], mode="implicit")
    corr = wh.correct_implicit(IMP2["omega"], IMP2["n_t"])
    return g, f, cfg, corr


def cpu_baseline_implicit(g, f, target_s=12.0):
    from oracle import implicit_oracle as IO

    fv = np.array(f.values)
    v = np.zeros_like(fv)
    bcs = ["dirichlet"] * 2
    t0 = time.perf_counter()
    _, solver = IO.wave_solve_implicit(v, fv, g.spacing, bcs, 2, IMP2["omega"], IMP2["n_t"], max_steps=1)
    t1 = time.perf_counter() - t0
    m = int(max(1, min(IMP2["n_t"], target_s / max(t1, 1e-6))))
    t0 = time.perf_counter()
    _, solver = IO.wave_solve_implicit(v, fv, g.spacing, bcs, 2, IMP2["omega"], IMP2["n_t"], max_steps=m)
    dt = time.perf_counter() - t0
    return {"value": g.size * m / dt / 1e9, "unit": "Gpts/s", "cores": 1, "kind": "port",
            "sample": f"the first {m} of {IMP2['n_t']} implicit steps of one WaveHoltz iteration on the "
                      f"{'x'.join(map(str, g.shape))} grid through oracle/implicit_oracle.py (bitwise restatement of "
                      f"the reference's MG-preconditioned CG, numpy, 1 core); {solver.inner} CG iterations, {dt:.2f} s"}


def run_implicit(args, dist, ws, rank, local):
    import torch

    import paper_2504_03074_b200 as wh
    from paper_2504_03074_b200 import _native
    from paper_2504_03074_b200.device import device_problem
    from paper_2504_03074_b200.implicit import implicit_solver_for

    torch.cuda.set_device(local)
    g, f, cfg, corr = build_imp2()
    prob = wh.HelmholtzProblem(g, 2, 1.0, IMP2["omega"], f)
    dp = device_problem(g, device=local)
    ctx = dp.ctx
    K, W = args.steps, args.warmup
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=f"cuda:{local}")
    for _ in range(max(1, W)):
        wh.fpi_solve(prob, cfg, tol=-1.0, maxit=1)
    torch.cuda.synchronize()
    barrier(dist)
    sampler = ClockSampler(local).start()
    l0 = ctx.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    v, run = wh.fpi_solve(prob, cfg, tol=-1.0, maxit=K)  # K implicit iterations from v = 0
    e1.record(stream)
    e1.synchronize()
    clocks = sampler.stop()
    launches = ctx.launch_count() - l0
    dev_s = max_over_ranks(dist, e0.elapsed_time(e1) / 1e3)
    units = g.size * IMP2["n_t"] * K * max(1, ws)
    value = units / dev_s / 1e9
    # dominant unit: the multigrid V-cycle graph (timed alone with events on the context stream)
    solver = implicit_solver_for(dp, g, 2, 1.0, corr.dt)
    ctx.vec_upload(solver.r, np.random.default_rng(0).standard_normal(g.shape))
    for _ in range(3):
        ctx.mg_vcycle(solver.r, solver.z)
    reps = 30
    v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    v0.record(stream)
    for _ in range(reps):
        ctx.mg_vcycle(solver.r, solver.z)
    v1.record(stream)
    v1.synchronize()
    vc_s = v0.elapsed_time(v1) / 1e3 / reps
    vbytes = mg_vcycle_bytes(IMP2["cells"])
    peak, peak_src = peaks()
    achieved = vbytes / vc_s / 1e9
    cg_per_step = run.inner_iterations / (K * IMP2["n_t"])
    e2e = None
    if not args.no_e2e:
        # through the public surface with host fields: wave_solve_filtered(v, f) per iteration
        op = wh.DiscreteOperator(g, 2, 1.0)
        vf = wh.GridField.zeros(g)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(K):
            vf = wh.wave_solve_filtered(vf, f, cfg, corr, op)
        torch.cuda.synchronize()
        te = max_over_ranks(dist, time.perf_counter() - t0)
        e2e = {"value": units / te / 1e9, "unit": "Gpts/s", "h2d_bytes_per_step": g.size * 8,
               "d2h_bytes_per_step": g.size * 8, "iters_per_s": K / te,
               "api": "paper_2504_03074_b200.wave_solve_filtered (implicit mode) with host GridFields"}
    cpu = None if (rank != 0 or ws != 1 or args.no_cpu_baseline) else cpu_baseline_implicit(g, f)
    if rank == 0:
        line = {
            "metric": "implicit WaveHoltz Gpts/s (grid-point updates per s) and iters/s", "value": value,
            "unit": "Gpts/s", "n_gpus": ws, "steps": K, "warmup": W, "ms_per_step": dev_s * 1e3 / K,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE forcing recipe, 8 Gaussians, seed 0)",
            "config": {"workload": "imp2", "grid": list(g.shape), "omega": IMP2["omega"], "N_t": IMP2["n_t"],
                       "mode": "implicit (trapezoidal), MG-preconditioned CG to 1e-12 per step",
                       "iterations": K, "cg_iterations_per_step": cg_per_step,
                       "l2": "working set (~15 fields of 33.6 MB) far above L2",
                       "parallelism": f"independent replicas x{ws}" if ws > 1 else "single GPU"},
            "iters_per_s": K / dev_s,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                         "kernel": "multigrid V-cycle (CUDA graph: red-black GS sweeps, fused residual+restriction, "
                                   "prolongation per level; levels <= 64 cells in one shared-memory CTA)",
                         "bytes_per_vcycle": vbytes, "vcycle_us": vc_s * 1e6,
                         "note": "algorithmic bytes of one V-cycle (see bench.mg_vcycle_bytes) / its device time "
                                 "(CUDA events around graph replays); the V-cycle is the preconditioner of every "
                                 "CG iteration"},
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "gpu_launches": launches,
            "residuals": {"first": run.residuals[0], "last": run.residuals[-1]}, "impl": "ours",
        }
        print(json.dumps(line))


def run_reference_implicit(args, ws, rank):
    if rank != 0:
        return
    g, f, cfg, corr = build_imp2()
    cpu = cpu_baseline_implicit(g, f, target_s=20.0)
    line = {
        "metric": "implicit WaveHoltz Gpts/s (grid-point updates per s) and iters/s", "value": cpu["value"],
        "unit": "Gpts/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE forcing recipe, 8 Gaussians, seed 0)",
        "config": {"workload": "imp2", "grid": list(g.shape), "omega": IMP2["omega"], "N_t": IMP2["n_t"]},
        "impl": "reference", "cpu_baseline": cpu,
        "e2e": {"value": cpu["value"], "unit": "Gpts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_ours(args, dist, ws, rank, local):
    import torch

    from paper_2504_03074_b200 import _native

    if args.emulate_cpu:
        if not (ws > 1 and args.workload in ("cfg3", "cfg4") and args.decomp == "slab"):
            raise SystemExit("--emulate-cpu runs the z-slab path only (configs 3/4 at N > 1)")
        return run_slab(args, dist, ws, rank, local)
    torch.cuda.set_device(local)
    if ws > 1 and args.workload in ("cfg3", "cfg4") and args.decomp == "slab":
        return run_slab(args, dist, ws, rank, local)
    wl = BatchRun(args, local, ws, rank) if args.workload == "cfg5" else SingleRun(args, local)
    ctx = wl.ctx
    ctx.set_l2_flush(256 << 20)
    ctx.set_timing(True)
    K, W = args.steps, args.warmup

    # warm-up (same code path), then reset to v = 0 so the timed K iterations are the solve itself
    wl.reset()
    if W > 0:
        ctx.fpi(W)
    wl.reset()
    torch.cuda.synchronize()
    barrier(dist)
    sampler = ClockSampler(local).start()
    l0 = ctx.launch_count()
    torch.cuda.synchronize()
    t_wall0 = time.perf_counter()
    rs = ctx.fpi(K)  # K passes back-to-back on the context stream, events around each pass
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall0
    launches = ctx.launch_count() - l0
    clocks = sampler.stop()
    step_ms_total, step_launches, solve_ms = ctx.last_timing()
    barrier(dist)
    dev_s = max_over_ranks(dist, solve_ms / 1e3)
    residuals = np.sqrt(rs[:, 0]) / math.sqrt(wl.npts)

    units_rank = wl.units_per_step * K
    units = units_rank
    if dist is not None:
        t = torch.tensor([float(units_rank)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        units = float(t.item())
    value = units / dev_s / 1e9
    ms_per_step = dev_s * 1e3 / K
    peak, peak_src = peaks()
    kern, steps_per_pass = ctx.plan()
    # compulsory bytes of the kernel's algorithm: a pass of T fused steps reads W^s, W^{s-1}, f, acc
    # and writes W^{s+T-1}, W^{s+T}, acc (56 B per T updates); the cluster-resident kernel (plan
    # kernel 4) reads v and f and writes v once per fpi call
    if kern == 4:
        own_bpu = 24.0 * wl.npts / units_rank
    else:
        own_bpu = BYTES_PER_UPDATE if steps_per_pass == 1 else 56 / steps_per_pass
    step_s = step_ms_total / 1e3
    avg_launch_s = step_s / max(1, step_launches)
    bytes_per_launch_comp = own_bpu * units_rank / max(1, step_launches)
    traffic, traffic_src = load_traffic(args.workload)
    if traffic and getattr(wl, "members", 1) > 1:
        # a batched run's launches carry the members still active (64 down to 1): the capture, one
        # launch of all members, is not the average launch
        traffic, traffic_src = None, "batched launches differ in member count; the ncu capture is one launch of all members"
    if traffic:
        achieved, frac_source = traffic / avg_launch_s / 1e9, (
            "ncu DRAM bytes per launch of this build (profiles/traffic.json: " + str(traffic_src) + ")")
    else:
        achieved, frac_source = bytes_per_launch_comp / avg_launch_s / 1e9, (
            f"compulsory bytes per launch ({own_bpu:g} B/update; {traffic_src})")
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "frac_source": frac_source,
            "kernel": ("cluster-resident solve kernel (the whole grid in the shared memory of one thread-block "
                       "cluster, DSMEM halo rows, one cluster barrier per leapfrog step; all K fixed-point "
                       "iterations in one launch)" if kern == 4 else
                       (f"{steps_per_pass}-step fused kernel (temporal blocking: Laplacian + leapfrog + filter for "
                        f"{steps_per_pass} consecutive steps per HBM pass)" if steps_per_pass > 1
                        else "fused step kernel (Laplacian + leapfrog + filter accumulate)")
                       + (", TMA tensor boxes" if kern == 2 else ", cp.async.bulk rows" if kern == 1 else "")),
            "avg_launch_us": avg_launch_s * 1e6, "launches_timed": step_launches,
            "bytes_per_update": own_bpu,
            "achieved_compulsory": bytes_per_launch_comp / avg_launch_s / 1e9,
            "frac_compulsory": bytes_per_launch_comp / avg_launch_s / 1e9 / peak,
            "frac_48B": BYTES_PER_UPDATE * units_rank / step_s / 1e9 / peak,
            "peak_source": peak_src, "lib_sha16": lib_sha16(),
            "note": "avg_launch_us = CUDA events on the context stream bracketing every pass of the timed "
                    "iterations / passes (includes the per-pass residual reduction and inter-launch gaps). "
                    "frac_48B uses SURVEY 8(d)'s 48 B per update and exceeds 1 for multi-step kernels by "
                    "construction (they move 56/T B per update)."}

    e2e = e2e_solve = e2e_seam = None
    if not args.no_e2e:
        te, info = wl.e2e(K, W, dist)
        te = max_over_ranks(dist, te)
        e2e = {"value": units / te / 1e9, "unit": "Gpts/s", **info, "iters_per_s": K / te}
        if hasattr(wl, "e2e_solve"):
            ts_, info_s = wl.e2e_solve(K, dist)
            ts_ = max_over_ranks(dist, ts_)
            e2e_solve = {"value": units / ts_ / 1e9, "unit": "Gpts/s", **info_s, "iters_per_s": K / ts_}
        if hasattr(wl, "e2e_seam"):
            ks = K if wl.npts < (1 << 28) else min(K, 3)  # 1025^3: 17 GB of pageable copies per call
            tss, info_m = wl.e2e_seam(ks, dist)
            tss = max_over_ranks(dist, tss)
            e2e_seam = {"value": wl.units_per_step * ks / tss / 1e9, "unit": "Gpts/s", "calls": ks, **info_m,
                        "iters_per_s": ks / tss}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        if args.workload == "cfg5":
            import paper_2504_03074_b200 as wh

            corr = wh.correct_explicit(100.0, wl.g, 2, 1.0)
            f = wh.multi_gaussian_source(wl.g, 150.3, 4, seed=0)
            cpu = cpu_baseline_numpy(wl.g, f, corr)
        else:
            cpu = cpu_baseline_numpy(wl.g, wl.f, wl.corr, order=ORDER.get(args.workload, 2))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gpts/s", "n_gpus": ws, "steps": K, "warmup": W,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if args.workload == "cfg5" else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (BASELINE forcing recipe, SURVEY 8(d)); f sha256 " + wl.f_sha[:16],
            "config": config_for(args.workload, K, ws, args.decomp, args.halo, n_t=getattr(wl, "n_t_config", None)),
            "iters_per_s": K / dev_s,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "e2e_solve": e2e_solve, "e2e_seam": e2e_seam,
            "clocks": clocks,
            "gpu_launches": launches,
            "residuals": {"first": float(residuals[0]), "last": float(residuals[-1])},
            "wall_s_timed_region": t_wall, "impl": "ours",
        }
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# reference arm: C OpenMP restatement of the reference on all host cores


def run_reference(args, ws, rank):
    if rank != 0:
        return
    from oracle import native as ON
    from oracle import waveholtz_oracle as O

    if args.workload == "cfg5":
        return run_reference_cfg5(args, ws)
    if ORDER.get(args.workload, 2) != 2:  # the C restatement is order 2: the numpy one (1 core)
        g, f, corr, cfg, _ = build_workload(args.workload)
        cpu = cpu_baseline_numpy(g, f, corr, target_s=20.0, order=ORDER[args.workload])
        line = {"metric": METRIC, "value": cpu["value"], "unit": "Gpts/s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (BASELINE forcing recipe, SURVEY 8(d)); f sha256 "
                        + hashlib.sha256(np.ascontiguousarray(f.values).data).hexdigest()[:16],
                "config": config_for(args.workload, args.steps, ws, args.decomp, args.halo, n_t=corr.steps_per_period),
                "impl": "reference", "cpu_baseline": cpu,
                "e2e": {"value": cpu["value"], "unit": "Gpts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return
    g, f, corr, cfg, _ = build_workload(args.workload)
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    fv = np.array(f.values)
    npts = g.size
    # all host cores, except where OpenMP fork/join per step costs more than it saves (config 1's
    # 16.6K points): the thread count the C restatement runs fastest with (oracle/native.py)
    threads = ON.max_threads() if npts >= (1 << 20) else ON.auto_threads(npts)
    v = np.zeros_like(fv)
    # sample size: full iterations when one takes <= ~3 s, else a truncated pass of m steps
    t0 = time.perf_counter()
    s5 = dict(sc)
    s5["n_total"] = 5
    ON.wave_solve(v, fv, g.spacing, s5, nthreads=threads)
    per_step = (time.perf_counter() - t0) / 5
    n_t = sc["n_total"]
    m = n_t if per_step * n_t <= 3.0 else max(5, int(3.0 / per_step))
    sm = dict(sc)
    sm["n_total"] = m
    for _ in range(min(args.warmup, 1)):
        v = ON.wave_solve(v, fv, g.spacing, sm, nthreads=threads)
    v[...] = 0.0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vn = ON.wave_solve(v, fv, g.spacing, sm, nthreads=threads)
        # the reference's per-iteration residual ||v_new - v||_2 / sqrt(N) (driver.py:225)
        _ = np.linalg.norm(vn - v) / math.sqrt(npts)
        v = vn
    dt = time.perf_counter() - t0
    value = npts * m * args.steps / dt / 1e9
    sample = (f"{'full WaveHoltz iteration' if m == n_t else f'{m} of {n_t} leapfrog steps'} per step of "
              f"the {'x'.join(map(str, g.shape))} grid through oracle/whb_oracle.c (bitwise restatement of the "
              f"reference, -O2 -ffp-contract=off, OpenMP {threads} threads)")
    line = {
        "metric": METRIC, "value": value, "unit": "Gpts/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "strong" if (ws > 1 and args.workload in ("cfg3", "cfg4") and args.decomp == "slab") else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE forcing recipe, SURVEY 8(d)); f sha256 "
                + hashlib.sha256(np.ascontiguousarray(fv).data).hexdigest()[:16],
        "config": config_for(args.workload, args.steps, ws, args.decomp, args.halo, n_t=n_t),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "Gpts/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "Gpts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_reference_cfg5(args, ws):
    """Config 5 on the host: every step is one full W pass of each of the 64 omegas
    (the reference's per-omega loop), C restatement on all host cores."""
    import paper_2504_03074_b200 as wh
    from paper_2504_03074_b200 import timestep as ts
    from oracle import native as ON
    from oracle import waveholtz_oracle as O

    ts._COURANT[2] = 0.9
    g = wh.build_grid(2, [(0.0, 1.0)] * 2, [1024, 1024], "dirichlet")
    fv = np.array(wh.multi_gaussian_source(g, 150.3, 4, seed=0).values)
    omegas = np.linspace(10.3, 200.3, 64)
    scs = [O.step_scalars(*O.correct_explicit(w, g.spacing, 2, 1.0, 0.9)) for w in omegas]
    threads = ON.max_threads()
    vs = [np.zeros_like(fv) for _ in omegas]
    steps = min(args.steps, 3)  # bounded sample: ~1.1e10 updates per step
    for _ in range(min(args.warmup, 1)):
        ON.wave_solve(vs[0], fv, g.spacing, scs[0], nthreads=threads)
    t0 = time.perf_counter()
    for _ in range(steps):
        for b, sc in enumerate(scs):
            vs[b] = ON.wave_solve(vs[b], fv, g.spacing, sc, nthreads=threads)
    dt = time.perf_counter() - t0
    units = g.size * sum(sc["n_total"] for sc in scs) * steps
    value = units / dt / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "Gpts/s", "n_gpus": ws, "steps": steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3 / steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (BASELINE forcing recipe)",
        "config": config_for("cfg5", args.steps, ws),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "Gpts/s", "cores": threads, "kind": "port",
                         "sample": f"{steps} WaveHoltz iteration(s) of all 64 omegas through oracle/whb_oracle.c "
                                   f"(OpenMP {threads} threads)"},
        "e2e": {"value": value, "unit": "Gpts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch(n: int) -> int:
    """--gpus N outside torchrun: one process per GPU through torch.distributed.run on this
    node (127.0.0.1 rendezvous).  Rank 0's stdout carries the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg4", choices=sorted(WORKLOADS) + ["cfg5", "imp2"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--decomp", default="slab", choices=["slab", "replicas"],
                    help="N > 1 on configs 3/4: z-slab decomposition (default) or independent replicas")
    ap.add_argument("--halo", choices=["nccl", "torch", "peer"], default="nccl",
                    help="z-slab halo exchange at N > 1: NCCL send/recv inside the C ABI on the exchange "
                         "stream, one CUDA graph per iteration (default); torch.distributed P2P; or peer "
                         "memory (CUDA IPC mappings of the neighbours' ghost planes, stream flags, graph)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--emulate-cpu", action="store_true",
                    help="TEST ONLY: the z-slab driver with a numpy stand-in shard over gloo (no GPU)")
    ap.add_argument("--cells", type=int, default=None,
                    help="TEST ONLY: override the workload's cells per axis (CPU launcher test)")
    args = ap.parse_args()
    if args.cells:
        d, _, om, fo, it = WORKLOADS[args.workload]
        WORKLOADS[args.workload] = (d, args.cells, om, fo, it)
    if args.steps is None:
        args.steps = {"cfg5": 20, "imp2": IMP2["iterations"]}.get(args.workload) or WORKLOADS[args.workload][4]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    ws, rank, local = dist_env()
    if ws != args.gpus and rank == 0:
        sys.stderr.write(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}; using WORLD_SIZE\n")
    if args.impl == "reference":
        if args.workload == "imp2":
            run_reference_implicit(args, ws, rank)
        else:
            run_reference(args, ws, rank)
        return
    dist = init_dist(ws) if not args.emulate_cpu else _init_gloo(ws)
    try:
        if args.workload == "imp2":
            run_implicit(args, dist, ws, rank, local)
        else:
            run_ours(args, dist, ws, rank, local)
    finally:
        if dist is not None:
            dist.destroy_process_group()


def _init_gloo(ws):
    if ws <= 1:
        return None
    import torch.distributed as dist

    dist.init_process_group(backend="gloo")
    return dist


if __name__ == "__main__":
    main()
