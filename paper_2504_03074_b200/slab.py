"""Slab (axis-0) domain decomposition of the explicit WaveHoltz iteration across
GPUs — SURVEY §8(e).

Each rank owns a contiguous range of axis-0 planes (``slab_ranges``) in one
whb context (include/whb200.h: plane_begin/plane_end) whose allocation carries
G = 3 ghost planes on each side.  The stencil radius is 1, so a single
leapfrog step needs one ghost plane of W^s; a pass of k fused steps (temporal
blocking: the two-step 2D/3D kernels, the three-step 3D kernel) needs k planes
of W^s and k - 1 of W^{s-1} and f.  Per pass (s, ..., s+k-1):

    1. compute the k first and k last owned update planes     (region 1 of whb_step/pair/triple)
    2. post the exchange of what the NEXT pass (k' steps) reads: k' planes of
       W^{s+k} and k' - 1 of W^{s+k-1} per side                 (``halo_items``)
    3. compute the remaining interior planes                   (region 2)
    4. join the exchange before the next pass                  (stream wait)

so the halo traffic, (2k - 1) x (n1 x n2 x 8 B) per side per k steps, overlaps
the interior update.  ``pass_plan`` orders the passes like the whole-grid solve
(three-step passes then a 2/1-step remainder; pairs then a single step; single
steps for the general operator and 1D), with k agreed over all slabs
(``agreed_pass_steps``: the smallest plan, capped by the smallest slab).  f is
exchanged once (it is static).  Per FPI pass the residual sum of squares is
all-reduced (one fp64).

The exchange goes through ``torch.distributed`` (NCCL on GPUs, gloo on CPUs)
on the context's own CUDA stream (``torch.cuda.ExternalStream``); device
buffers are wrapped zero-copy through ``__cuda_array_interface__`` (a halo of
several planes is one contiguous message).  The in-process ``LocalHalo`` runs
several slabs in one process (one GPU or several) with device-to-device
copies, which is how the multi-slab kernels are checked on a single GPU.
"""

from __future__ import annotations

import contextlib
import math

import numpy as np

from . import _native
from .filters import mode_name
from .grid import operator_coefficients
from .timestep import time_schedule

__all__ = ["slab_ranges", "pass_plan", "run_pass", "agreed_pass_steps", "DeviceShard", "TorchHalo", "NcclHalo", "LocalHalo", "PeerHalo", "PeerSlabGraphs", "run_peer_local_solve", "SlabFPI", "SlabKrylov", "ShardedVectors",
           "run_filtered_solve", "run_local_solve", "halo_items", "exchange_forcing"]


def slab_ranges(n0: int, nranks: int):
    """Contiguous, near-equal [p0, p1) ranges of the n0 axis-0 planes (1025 / 8 -> 128 or 129)."""
    if nranks < 1 or nranks > n0:
        raise ValueError("need 1 <= nranks <= number of planes")
    base, extra = divmod(n0, nranks)
    out, p = [], 0
    for r in range(nranks):
        q = p + base + (1 if r < extra else 0)
        out.append((p, q))
        p = q
    return out


class _CudaArray:
    """Minimal __cuda_array_interface__ exporter for a raw device pointer."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": (int(n),), "typestr": "<f8",
                                         "strides": None, "version": 3}


def level(L: int):
    """Halo item naming time level L (level 0 = V)."""
    return ("level", int(L))


def field(fid: int):
    """Halo item naming a field slot (e.g. _native.F)."""
    return ("field", int(fid))


def halo_planes(shard, side: str, depth: int):
    """(send_first, recv_first) local plane indices of a depth-plane halo on one side."""
    g, n = shard.gh, shard.nloc
    if side == "lo":
        return g, g - depth
    return g + n - depth, g + n


def pass_plan(n_total: int, steps_per_pass: int):
    """The passes [(s, k), ...] of a solve, k leapfrog steps each, in the order the whole-grid
    solve runs them (whb200.cu enqueue_solve): with 3 steps per pass (and n_total > 3) three-step
    passes while >= 3 steps remain, then one pass of the remaining 2 or 1; with 2, passes
    (0, 1), (2, 3), ... and a last single step when n_total is odd; else single steps."""
    if steps_per_pass >= 3 and n_total > 3:
        out, s = [], 0
        while n_total - s >= 3:
            out.append((s, 3))
            s += 3
        if s < n_total:
            out.append((s, n_total - s))
        return out
    if steps_per_pass >= 2:
        return [(s, min(2, n_total - s)) for s in range(0, n_total, 2)]
    return [(s, 1) for s in range(n_total)]


def halo_items(s: int, k: int, k_next: int):
    """What a pass of k_next steps needs from the neighbours after the pass (s, k): k_next ghost
    planes of W^{s+k} and k_next - 1 of W^{s+k-1} per side (the pass reads W^{s-1} one plane less
    deep than W^s)."""
    e = s + k
    items = [(level(e), k_next)]
    if k_next > 1:
        items.append((level(e - 1), k_next - 1))
    return items


def run_pass(shard, s: int, k: int, region: int):
    """Region 0/1/2 of the k-step pass starting at step s (whb_step / whb_pair / whb_triple)."""
    (shard.step, shard.pair, shard.triple)[k - 1](s, region)


def agreed_pass_steps(shards, halo=None) -> int:
    """Steps per pass every slab of the decomposition runs: the smallest plan (whb_plan: 1, 2
    or 3) over the slabs, capped by the smallest slab (a pass of k steps takes k ghost planes
    from ONE neighbour).  Across processes this is an all-reduce (MIN) over the halo's process
    group, done once per shard and cached (every rank reaches it in the same solve)."""
    k = min(min(sh.steps_per_pass, sh.nloc) for sh in shards)
    dist = getattr(halo, "dist", None)
    if dist is not None and halo is not None and halo.nranks > 1:
        import torch

        dev = "cpu" if dist.get_backend() == "gloo" else f"cuda:{shards[0].device}"
        t = torch.tensor([k], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        k = int(t.item())
    return max(1, k)


def _pass_steps(shards, halo):
    k = getattr(shards[0], "pass_steps", None)
    if k is None:
        k = agreed_pass_steps(shards, halo)
        for sh in shards:
            sh.pass_steps = k
    return k


class DeviceShard:
    """One rank's slab on its GPU: a whb context owning planes [p0, p1)."""

    def __init__(self, grid, plane_range, c=1.0, order=2, device=0):
        clo, cmid, c2 = operator_coefficients(grid, order, c)
        self.grid = grid
        self.plane_range = tuple(plane_range)
        self.ctx = _native.Context(grid.shape, device=device, plane_range=plane_range)
        self.ctx.set_operator(clo, cmid, c2)
        self.nloc = self.plane_range[1] - self.plane_range[0]
        self.gh = self.ctx.ghost_planes()
        self.steps_per_pass = self.ctx.plan()[1]
        self.device = device

    # schedule / fields
    def set_schedule(self, sched):
        self.ctx.set_schedule(0, sched)
        self.n_total = sched["n_total"]

    def upload(self, field, local_values):
        self.ctx.upload(field, local_values)

    def download(self, field):
        return self.ctx.download(field)

    def zero(self, field):
        self.ctx.zero(field)

    # step-level control
    def solve_begin(self, out_mode, zero_forcing=False):
        self.ctx.solve_begin(out_mode, zero_forcing)

    def step(self, s, region):
        self.ctx.step(s, region)

    def pair(self, s, region):
        self.ctx.pair(s, region)

    def triple(self, s, region):
        self.ctx.triple(s, region)

    def solve_end(self) -> float:
        return self.ctx.solve_end()

    # halo plumbing
    def plane_ptr(self, item, plane):
        kind, ident = item
        if kind == "level":
            return self.ctx.level_plane_ptr(ident, plane)
        return self.ctx.field_plane_ptr(ident, plane)

    def planes(self, item, first, count):
        """Zero-copy torch view of `count` consecutive local planes of a level/field."""
        import torch

        ptr, n = self.plane_ptr(item, first)
        return torch.as_tensor(_CudaArray(ptr, n * count), device=f"cuda:{self.device}")

    def stream(self):
        import torch

        return torch.cuda.stream(torch.cuda.ExternalStream(self.ctx.stream_ptr(), device=f"cuda:{self.device}"))

    def synchronize(self):
        self.ctx.synchronize()


class TorchHalo:
    """Halo exchange between ranks with torch.distributed point-to-point ops."""

    def __init__(self, dist, rank: int, world: int):
        self.dist = dist
        self.rank = rank
        self.world = world

    @property
    def nranks(self):
        return self.world

    def start(self, shard, items):
        """Post the exchange of [(item, depth), ...]; every rank passes the same list."""
        d = self.dist
        ops = []
        with shard.stream():
            for item, depth in items:
                if self.rank > 0:
                    snd, rcv = halo_planes(shard, "lo", depth)
                    ops.append(d.P2POp(d.isend, shard.planes(item, snd, depth), self.rank - 1))
                    ops.append(d.P2POp(d.irecv, shard.planes(item, rcv, depth), self.rank - 1))
                if self.rank < self.world - 1:
                    snd, rcv = halo_planes(shard, "hi", depth)
                    ops.append(d.P2POp(d.isend, shard.planes(item, snd, depth), self.rank + 1))
                    ops.append(d.P2POp(d.irecv, shard.planes(item, rcv, depth), self.rank + 1))
            works = d.batch_isend_irecv(ops) if ops else []
        return shard, works

    def finish(self, handle):
        shard, works = handle
        with shard.stream():
            for w in works:
                w.wait()

    def allreduce_sum(self, x: float, shard) -> float:
        import torch

        dev = "cpu" if self.dist.get_backend() == "gloo" else f"cuda:{shard.device}"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t)
        return float(t.item())


class LocalHalo:
    """All slabs live in this process: plane copies between contexts (same or peer GPU)."""

    def __init__(self, shards):
        self.shards = list(shards)

    @property
    def nranks(self):
        return len(self.shards)

    def exchange(self, items):
        sh = self.shards
        for item, depth in items:
            for r in range(len(sh) - 1):
                lo, hi = sh[r], sh[r + 1]
                nbytes = depth * lo.plane_ptr(item, 0)[1] * 8
                lo_send, lo_recv = halo_planes(lo, "hi", depth)
                hi_send, hi_recv = halo_planes(hi, "lo", depth)
                lo.ctx.copy_device_to(lo.plane_ptr(item, lo_send)[0], hi.ctx, hi.plane_ptr(item, hi_recv)[0], nbytes)
                hi.ctx.copy_device_to(hi.plane_ptr(item, hi_send)[0], lo.ctx, lo.plane_ptr(item, lo_recv)[0], nbytes)


class NcclHalo:
    """Halo exchange with NCCL inside the C ABI (whb_nccl_*): the boundary planes of every item go
    to the neighbours as one ncclSend/ncclRecv group on the context's exchange stream, forked
    after the boundary planes (whb_comm_begin) and joined before the next pass (whb_comm_join),
    so the interior planes run while the planes are on NVLink -- and, unlike the torch.distributed
    path, the exchange is capturable: SlabFPI(graph=True) replays one CUDA graph per iteration
    (kernels + NCCL transfers) and all-reduces the residual once (whb_nccl_allreduce_sum)."""

    def __init__(self, shard, dist, rank: int, world: int):
        self.shard, self.rank, self.world = shard, rank, world
        self.dist = dist
        uid = [_native.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(uid, src=0)
        shard.ctx.nccl_init(world, rank, uid[0])

    @property
    def nranks(self):
        return self.world

    def start(self, shard, items):
        sends, recvs, counts, peers = [], [], [], []
        for item, depth in items:
            for q, side in ((self.rank - 1, "lo"), (self.rank + 1, "hi")):
                if 0 <= q < self.world:
                    snd, rcv = halo_planes(shard, side, depth)
                    sp, n = shard.plane_ptr(item, snd)
                    rp, _ = shard.plane_ptr(item, rcv)
                    sends.append(sp)
                    recvs.append(rp)
                    counts.append(n * depth)
                    peers.append(q)
        shard.ctx.comm_begin()
        shard.ctx.nccl_exchange(sends, recvs, counts, peers)
        shard.ctx.comm_end()
        return shard

    def finish(self, shard):
        shard.ctx.comm_join()

    def allreduce_sum(self, x: float, shard) -> float:
        return shard.ctx.nccl_allreduce_sum(x)


_PEER_LEVELS = 9  # levels 0..8 cover V and every ring slot (nring <= 6)


def _buffer_table(shard):
    """Plane-0 device address of every buffer a halo item can name: level L (0..8) and field F."""
    tab = {level(L): shard.plane_ptr(level(L), 0)[0] for L in range(_PEER_LEVELS)}
    tab[field(_native.F)] = shard.plane_ptr(field(_native.F), 0)[0]
    return tab


def _ring_size(tab):
    """Time-level ring length of a shard from its buffer table (level L >= 1 lives in slot L mod n)."""
    for n in range(1, _PEER_LEVELS - 1):
        if tab[level(1 + n)] == tab[level(1)]:
            return n
    raise RuntimeError("time-level ring longer than the buffer table")


def _canon(item, nring):
    kind, ident = item
    if kind != "level" or ident == 0:
        return item
    return level((ident - 1) % nring + 1)


class PeerHalo:
    """Halo exchange through peer memory: after the boundary planes are computed, this rank copies
    them straight into its neighbours' ghost planes (NVLink copy engines on the context stream;
    the neighbours' buffers are mapped with CUDA IPC across processes, or used directly when the
    slabs share a process), then bumps a flag in each neighbour's memory with a stream write; a
    rank waits for its own flags with a stream wait before the pass that reads the ghosts.  No
    NCCL on the data path, no host round trip per pass, no kernel spinning on the device.

    Ordering: ``start`` after region 1 of pass s (copy levels s+2, s+1; flag := seq), ``finish``
    after region 2 (wait until my flags >= seq).  A rank enters ``start`` of exchange e only after
    its ``finish`` of exchange e-1, i.e. after each neighbour completed region 1 of the pass that
    produced e-1, hence the whole pass before it — the last pass that read the ghost planes being
    overwritten (region 2 never reads ghosts).  Every rank runs the same exchange sequence, so
    the sequence numbers agree.

    Flags: flags[0] is written by the lower neighbour (rank - 1), flags[1] by the upper one."""

    def __init__(self, shard, rank: int, world: int, nlocs, peers, dist=None, opened=None):
        self.shard, self.rank, self.world = shard, rank, world
        self.nlocs = list(nlocs)
        self.peers = peers          # {neighbour rank: {"buf": {item: base}, "flags": ptr, "plane_bytes": b}}
        self.dist = dist
        self.opened = opened or []  # IPC mappings to close
        self.seq = 0
        self.nring = _ring_size(_buffer_table(shard))
        # exchange stream: one process per GPU (from_dist).  Slabs sharing one GPU in one process
        # (local_group) keep the exchange on their context streams: their stream waits would
        # otherwise share the GPU's hardware queues with the other slabs' exchange branches
        # (head-of-line blocking -- measured: a replayed in-process graph pair deadlocked)
        self.use_comm = dist is not None

    @property
    def nranks(self):
        return self.world

    # -- construction ----------------------------------------------------------------------
    @staticmethod
    def local_group(shards):
        """PeerHalos for slabs that all live in this process (direct device addresses)."""
        flags = [sh.ctx.flags_alloc(2) for sh in shards]
        tabs = [_buffer_table(sh) for sh in shards]
        pb = [sh.plane_ptr(level(0), 0)[1] * 8 for sh in shards]
        nlocs = [sh.nloc for sh in shards]
        out = []
        for r, sh in enumerate(shards):
            peers = {q: {"buf": tabs[q], "flags": flags[q], "plane_bytes": pb[q]}
                     for q in (r - 1, r + 1) if 0 <= q < len(shards)}
            h = PeerHalo(sh, r, len(shards), nlocs, peers)
            h.flags = flags[r]
            out.append(h)
        return out

    @staticmethod
    def from_dist(shard, dist, rank: int, world: int):
        """One PeerHalo per rank: IPC handles of the halo buffers and flags are all-gathered and
        the neighbours' allocations mapped into this process."""
        flags = shard.ctx.flags_alloc(2)
        mine = {"buf": {k: shard.ctx.ipc_handle(p) for k, p in _buffer_table(shard).items()},
                "flags": shard.ctx.ipc_handle(flags), "plane_bytes": shard.plane_ptr(level(0), 0)[1] * 8,
                "nloc": shard.nloc}
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        bases, peers, opened = {}, {}, []

        def mapped(h_off):
            h, off = h_off
            if h not in bases:
                bases[h] = shard.ctx.ipc_open(h)
                opened.append(bases[h])
            return bases[h] + off

        for q in (rank - 1, rank + 1):
            if 0 <= q < world:
                peers[q] = {"buf": {k: mapped(v) for k, v in allv[q]["buf"].items()},
                            "flags": mapped(allv[q]["flags"]), "plane_bytes": allv[q]["plane_bytes"]}
        h = PeerHalo(shard, rank, world, [a["nloc"] for a in allv], peers, dist=dist, opened=opened)
        h.flags = flags
        return h

    def epoch_end(self, shard=None):
        """Restart the exchange numbering: zero this rank's own flags (stream write, after every
        wait of the iteration) and the sequence counter.  Callers must separate epochs by a
        barrier that every rank passes only after its epoch_end (the residual all-reduce across
        processes; the host's residual read of every slab in one process), so no neighbour's
        next-epoch flag write can precede the reset."""
        sh = shard or self.shard
        sh.ctx.stream_write_u32(self.flags, 0)
        sh.ctx.stream_write_u32(self.flags + 4, 0)
        self.seq = 0

    def close(self):
        for b in self.opened:
            self.shard.ctx.ipc_close(b)
        self.opened = []
        if getattr(self, "flags", 0):
            self.shard.ctx.flags_free(self.flags)
            self.flags = 0

    # -- exchange --------------------------------------------------------------------------
    def _recv_plane(self, q, side_of_q, depth):
        """First ghost plane of neighbour q on its side `side_of_q` (its geometry: gh, nloc_q)."""
        g, n = self.shard.gh, self.nlocs[q]
        return g - depth if side_of_q == "lo" else g + n

    def start(self, shard, items):
        ctx = shard.ctx
        if self.use_comm:
            ctx.comm_begin()  # copies + flag writes on the exchange stream, after the boundary planes
        for item, depth in items:
            for q, my_side, q_side in ((self.rank - 1, "lo", "hi"), (self.rank + 1, "hi", "lo")):
                if q not in self.peers:
                    continue
                snd, _ = halo_planes(shard, my_side, depth)
                pq = self.peers[q]
                dst = pq["buf"][_canon(item, self.nring)] + self._recv_plane(q, q_side, depth) * pq["plane_bytes"]
                ctx.copy_async(shard.plane_ptr(item, snd)[0], dst, depth * pq["plane_bytes"])
        self.seq += 1
        for q, slot in ((self.rank - 1, 1), (self.rank + 1, 0)):  # I am q's upper / lower neighbour
            if q in self.peers:
                ctx.stream_write_u32(self.peers[q]["flags"] + 4 * slot, self.seq)
        if self.use_comm:
            ctx.comm_end()
        return self.seq

    def finish(self, seq):
        # my outgoing copies done (their source planes may be overwritten from the next pass on),
        # then the neighbours' copies into my ghost planes (their flags)
        if self.use_comm:
            self.shard.ctx.comm_join()
        for q, slot in ((self.rank - 1, 0), (self.rank + 1, 1)):
            if q in self.peers:
                self.shard.ctx.stream_wait_u32(self.flags + 4 * slot, seq)

    def allreduce_sum(self, x: float, shard) -> float:
        import torch

        dev = "cpu" if self.dist.get_backend() == "gloo" else f"cuda:{shard.device}"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t)
        return float(t.item())


def run_peer_local_solve(shards, halos, out_mode=_native.OUT_FPI, zero_forcing=False):
    """``run_filtered_solve``'s schedule for slabs of this process that exchange through
    ``PeerHalo.local_group`` (each op issued for every slab in turn, so the stream waits of one
    slab always follow the neighbour's enqueued flag writes).  Returns the residual sums."""
    for sh in shards:
        sh.solve_begin(out_mode, zero_forcing)
    plan = pass_plan(shards[0].n_total, _pass_steps(shards, None))

    def exchange_both(items, between=None):
        hs = [h.start(sh, items) for sh, h in zip(shards, halos)]
        if between:
            between()
        for h, q in zip(halos, hs):
            h.finish(q)

    exchange_both([(level(0), plan[0][1])])  # W^0 = v, as deep as the first pass reads it
    for n, (s, k) in enumerate(plan):
        if n + 1 == len(plan):
            for sh in shards:
                run_pass(sh, s, k, 0)
            continue
        for sh in shards:
            run_pass(sh, s, k, 1)
        exchange_both(halo_items(s, k, plan[n + 1][1]), lambda: [run_pass(sh, s, k, 2) for sh in shards])
    return [sh.solve_end() for sh in shards]


class PeerSlabGraphs:
    """In-process slabs exchanging through PeerHalo, one fixed-point iteration per slab captured
    as a CUDA graph (kernels, peer copies and the stream flag writes / waits that order them
    across the slabs' streams): an iteration costs one graph launch per slab and one residual
    read, instead of ~10 host calls per slab and pass.  Every epoch ends with epoch_end (flags
    back to 0), and the host reads every slab's residual before the next replay."""

    def __init__(self, shards, halos, out_mode=_native.OUT_FPI):
        self.shards, self.halos = list(shards), list(halos)
        self.out_mode = out_mode
        self._iterate_host()  # warm-up: device tables, plans and scratch exist before capture
        for sh in self.shards:
            sh.ctx.capture_begin()
        try:
            run_peer_local_solve(self.shards, self.halos, out_mode)
            for sh, h in zip(self.shards, self.halos):
                h.epoch_end(sh)
        finally:
            self.graphs = [sh.ctx.capture_end() for sh in self.shards]

    def _iterate_host(self):
        rs = run_peer_local_solve(self.shards, self.halos, self.out_mode)
        for sh, h in zip(self.shards, self.halos):
            h.epoch_end(sh)
        for sh in self.shards:
            sh.synchronize()
        return rs

    def iterate(self):
        """One replay per slab; returns the slabs' residual sums of squares."""
        for sh, gid in zip(self.shards, self.graphs):
            sh.ctx.graph_launch(gid)
        return [sh.ctx.resid_read() for sh in self.shards]


def _exchange_now(halo, shard, items):
    if halo.nranks > 1:
        halo.finish(halo.start(shard, items))


def run_filtered_solve(shard, halo, out_mode=_native.OUT_FPI, zero_forcing=False) -> float:
    """One W(v, f) pass of a slab with halo exchange (the schedule in the module docstring, with
    ``pass_plan``'s passes).  Returns this rank's residual sum of squares (FPI mode)."""
    shard.solve_begin(out_mode, zero_forcing)
    multi = halo.nranks > 1
    plan = pass_plan(shard.n_total, _pass_steps([shard], halo))
    _exchange_now(halo, shard, [(level(0), plan[0][1])])  # W^0 = v, as deep as the first pass reads it
    for n, (s, k) in enumerate(plan):
        if not multi or n + 1 == len(plan):
            run_pass(shard, s, k, 0)  # the last pass writes the output; no later step needs its halo
            continue
        run_pass(shard, s, k, 1)
        h = halo.start(shard, halo_items(s, k, plan[n + 1][1]))
        run_pass(shard, s, k, 2)
        halo.finish(h)
    return shard.solve_end()


def run_local_solve(shards, halo: LocalHalo, out_mode=_native.OUT_FPI, zero_forcing=False):
    """The same schedule for in-process slabs (each pass: boundary planes of every slab, plane
    copies, interior planes)."""
    for sh in shards:
        sh.solve_begin(out_mode, zero_forcing)
    plan = pass_plan(shards[0].n_total, _pass_steps(shards, None))
    halo.exchange([(level(0), plan[0][1])])
    for n, (s, k) in enumerate(plan):
        if n + 1 == len(plan):
            for sh in shards:
                run_pass(sh, s, k, 0)
            continue
        for sh in shards:
            run_pass(sh, s, k, 1)
        halo.exchange(halo_items(s, k, plan[n + 1][1]))
        for sh in shards:
            run_pass(sh, s, k, 2)
    return [sh.solve_end() for sh in shards]


def forcing_depth(shards, halo=None) -> int:
    """Ghost planes of f a k-step pass reads: k - 1 (at least 1), k agreed over the slabs."""
    return max(1, _pass_steps(list(shards), halo) - 1)


def exchange_forcing(shards_or_shard, halo):
    """f is read k - 1 planes beyond the owned range by a k-step pass: exchange it once (f is
    static)."""
    if isinstance(halo, LocalHalo):
        halo.exchange([(field(_native.F), forcing_depth(halo.shards))])
    elif isinstance(halo, (list, tuple)):  # PeerHalo.local_group
        items = [(field(_native.F), forcing_depth(shards_or_shard))]
        hs = [h.start(sh, items) for sh, h in zip(shards_or_shard, halo)]
        for h, q in zip(halo, hs):
            h.finish(q)
    else:
        _exchange_now(halo, shards_or_shard, [(field(_native.F), forcing_depth([shards_or_shard], halo))])


class ShardedVectors:
    """The vector interface ``linalg.device_gmres`` uses, over the slab contexts this process
    owns: element-wise operations act on every local slab, dot products are the sum of the
    slabs' owned-point dots completed by ``reduce`` (the cross-rank all-reduce for TorchHalo;
    identity when every slab is local).  The Krylov basis is thereby sharded like the grid —
    (restart + 1) vectors of 8.6 GB at 1025^3 do not fit one GPU."""

    def __init__(self, shards, reduce=None):
        self.shards = list(shards)
        self.reduce = reduce or (lambda x: x)

    def _each(self, name, *args):
        for sh in self.shards:
            getattr(sh.ctx, name)(*args)

    def vec_reserve(self, count):
        ids = [sh.ctx.vec_reserve(count) for sh in self.shards]
        if any(i != ids[0] for i in ids):
            raise RuntimeError("slab contexts disagree on vector ids")
        return ids[0]

    def dot(self, x, y) -> float:
        return self.reduce(sum(sh.ctx.dot(x, y) for sh in self.shards))

    def axpy(self, a, x, y):
        self._each("axpy", a, x, y)

    def scale_into(self, a, x, y):
        self._each("scale_into", a, x, y)

    def div_into(self, x, d, y):
        self._each("div_into", x, d, y)

    def sub_into(self, x, y, z):
        self._each("sub_into", x, y, z)

    def copy(self, x, y):
        self._each("copy", x, y)

    def lincomb(self, y, first, coef):
        self._each("lincomb", y, first, coef)


class SlabKrylov:
    """GMRES on A v = v - W(v, 0), b = W(0, f) (driver.py:247-300) over slab-decomposed
    grids: ``linalg.device_gmres`` (the reference's GMRES control flow, linalg.py:102-183)
    on ``ShardedVectors``; each mat-vec is one zero-forcing slab solve with halo exchange.

    ``shards`` / ``forcings``: this process's DeviceShards and their owned planes of f —
    one of each under TorchHalo (one rank per GPU), all of them under LocalHalo."""

    def __init__(self, shards, halo, corr, config, forcings):
        if mode_name(config.mode) != "explicit":
            raise NotImplementedError("the slab path runs the explicit scheme")
        self.shards = list(shards)
        self.halo = halo
        self.grid = self.shards[0].grid
        sched = time_schedule(corr, config)
        for sh, f in zip(self.shards, forcings):
            sh.set_schedule(sched)
            sh.upload(_native.F, np.ascontiguousarray(np.asarray(f, dtype=float)))
        self._local = isinstance(halo, LocalHalo)
        exchange_forcing(self.shards if self._local else self.shards[0], halo)
        reduce = None
        if not self._local and halo.nranks > 1:
            reduce = lambda x: halo.allreduce_sum(x, self.shards[0])  # noqa: E731
        self.vec = ShardedVectors(self.shards, reduce)

    def _solve(self, out_mode, zero_forcing):
        if self._local:
            run_local_solve(self.shards, self.halo, out_mode, zero_forcing)
        else:
            run_filtered_solve(self.shards[0], self.halo, out_mode, zero_forcing)

    def matvec(self, src, dst):
        """dst = src - W(src, 0)"""
        self.vec.copy(src, _native.V)
        self._solve(_native.OUT_AV, True)
        self.vec.copy(_native.OUT, dst)

    def solve(self, tol=1e-10, restart=50, maxit=500):
        """Returns (owned planes of x per local shard, report); residuals are scaled by
        1/sqrt(N) like driver.py:294."""
        from .linalg import device_gmres

        for sh in self.shards:
            sh.zero(_native.V)
        self._solve(_native.OUT_PLAIN, False)  # OUT = b = W(0, f)
        m = max(1, min(restart, maxit))
        ids = self.vec.vec_reserve(m + 4)
        b_id, x_id, work = ids[0], ids[1], ids[2:]
        self.vec.copy(_native.OUT, b_id)
        scale = math.sqrt(self.grid.size)
        rep = device_gmres(self.vec, self.matvec, b_id, x_id, tol=0.0, atol=tol * scale, restart=restart,
                           maxit=maxit, work_ids=work)
        rep.residual_history = [r / scale for r in rep.residual_history]
        return [sh.ctx.vec_download(x_id) for sh in self.shards], rep


class SlabFPI:
    """Fixed-point iteration (driver.py:211-230) over a slab-decomposed grid.

    ``shard`` is this rank's DeviceShard, ``halo`` a TorchHalo.  ``forcing``
    is either the full field (sliced here) or this rank's owned planes.
    """

    def __init__(self, shard, halo, corr, config, forcing, graph=False):
        if mode_name(config.mode) != "explicit":
            raise NotImplementedError("only the explicit path runs on the GPU")
        self.shard = shard
        self.halo = halo
        self.grid = shard.grid
        shard.set_schedule(time_schedule(corr, config))
        p0, p1 = shard.plane_range
        fv = np.asarray(forcing.values if hasattr(forcing, "values") else forcing, dtype=float)
        if fv.shape[0] == self.grid.shape[0] and fv.shape[0] != p1 - p0:
            fv = fv[p0:p1]
        if min(b - a for a, b in slab_ranges(self.grid.shape[0], halo.nranks)) < 2:
            raise ValueError("every slab needs at least 2 owned planes")
        shard.upload(_native.F, np.ascontiguousarray(fv))
        exchange_forcing(shard, halo)
        # graph=True (PeerHalo only): after one host-driven iteration, each iteration is one CUDA
        # graph replay (kernels, peer copies, flag writes / waits) + the residual all-reduce
        self.graph = bool(graph) and isinstance(halo, (PeerHalo, NcclHalo))
        self._peer = isinstance(halo, PeerHalo)
        self._gid = None
        if self.graph:
            if self._peer:
                halo.epoch_end(shard)
            shard.synchronize()
        self.reset()

    def reset(self):
        self.shard.zero(_native.V)

    def iterate(self) -> float:
        """One pass; returns the global scaled residual ||v_new - v||_2 / sqrt(N)."""
        if self.graph and self._gid is not None:
            self.shard.ctx.graph_launch(self._gid)
            rs = self.shard.ctx.resid_read()  # synchronises: the epoch's flag reset has executed
        else:
            rs = run_filtered_solve(self.shard, self.halo)
            if self.graph:
                if self._peer:
                    self.halo.epoch_end(self.shard)
                self.shard.synchronize()
        total = self.halo.allreduce_sum(rs, self.shard) if self.halo.nranks > 1 else rs
        if self.graph and self._gid is None:
            # capture the next iterations (nothing executes during capture)
            self.shard.ctx.capture_begin()
            try:
                run_filtered_solve(self.shard, self.halo)
                if self._peer:
                    self.halo.epoch_end(self.shard)
            finally:
                self._gid = self.shard.ctx.capture_end()
        return math.sqrt(total) / math.sqrt(self.grid.size)

    def local_iterate(self) -> np.ndarray:
        return self.shard.download(_native.V)
