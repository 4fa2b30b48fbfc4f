"""CPU: the peer-memory halo exchange (slab.PeerHalo) — which planes go to which neighbour
ghost planes, the flag protocol, the lockstep in-process driver — over NumpyShard stand-ins
whose "device addresses" index a simulated address space (copies and flag writes happen at
enqueue time, so a stream wait that is not yet satisfied is a protocol error).  Checked bitwise
against the single-domain oracle; tests/test_gpu_slab.py runs the same on the device."""

import numpy as np
import pytest

from paper_2504_03074_b200 import _native
from paper_2504_03074_b200.grid import build_grid
from paper_2504_03074_b200.slab import PeerHalo, exchange_forcing, run_peer_local_solve, slab_ranges
from paper_2504_03074_b200.timestep import correct_explicit, time_schedule
from paper_2504_03074_b200.filters import FilterConfig
from oracle import waveholtz_oracle as O

from test_slab_gloo import NumpyShard

SPAN = 1 << 40


class AddressSpace:
    def __init__(self):
        self.arrays = []

    def register(self, arr):
        self.arrays.append(arr)
        return len(self.arrays) * SPAN

    def resolve(self, addr):
        a = self.arrays[addr // SPAN - 1]
        return a, addr % SPAN


class PeerCtx:
    """The peer-exchange part of the whb context interface over an AddressSpace."""

    def __init__(self, space, shard):
        self.space, self.sh = space, shard
        self.log = []

    def flags_alloc(self, n):
        return self.space.register(np.zeros(n, dtype=np.uint32))

    def flags_free(self, ptr):
        pass

    def copy_async(self, src, dst, nbytes):
        a, o = self.space.resolve(src)
        b, p = self.space.resolve(dst)
        n = nbytes // 8
        b.reshape(-1)[p // 8:p // 8 + n] = a.reshape(-1)[o // 8:o // 8 + n]
        self.log.append(("copy", src, dst, nbytes))

    def stream_write_u32(self, ptr, value):
        a, o = self.space.resolve(ptr)
        a[o // 4] = value

    # the exchange stream protocol: copies and flag writes of an exchange between begin and end,
    # the join before the next exchange begins (synchronous here, so only the order is checked)
    def comm_begin(self):
        assert not getattr(self, "open", False), "whb_comm_begin while an exchange is open"
        assert getattr(self, "joined", True), "exchange started before the previous one was joined"
        self.open, self.joined = True, False

    def comm_end(self):
        assert getattr(self, "open", False), "whb_comm_end without whb_comm_begin"
        self.open = False

    def comm_join(self):
        assert not getattr(self, "open", False), "whb_comm_join inside an open exchange"
        self.joined = True

    def stream_wait_u32(self, ptr, value):
        a, o = self.space.resolve(ptr)
        assert np.int32(np.uint32(a[o // 4]) - np.uint32(value)) >= 0, "wait on a flag no neighbour has written"


class PeerNumpyShard(NumpyShard):
    def __init__(self, space, *a, **k):
        super().__init__(*a, **k)
        vecs = self.ctx
        self.ctx = PeerCtx(space, self)
        for name in ("vec_reserve", "dot"):
            setattr(self.ctx, name, getattr(vecs, name))
        self.base = {k: space.register(v) for k, v in self.buf.items()}
        self.plane_bytes = int(np.prod(self.buf["v"].shape[1:])) * 8

    def plane_ptr(self, item, plane):
        kind, ident = item
        key = ("v" if ident == 0 else ident % 6) if kind == "level" else self._field(ident)
        return self.base[key] + plane * self.plane_bytes, self.plane_bytes // 8


@pytest.mark.parametrize("use_comm", [False, True])
@pytest.mark.parametrize("dim,cells,omega,spp,world", [(2, (40, 24), 12.0, 2, 2), (3, (14, 10, 12), 6.5, 2, 3),
                                                       (2, (9, 30), 8.0, 2, 3), (2, (40, 24), 12.0, 1, 3),
                                                       (3, (20, 10, 12), 7.0, 3, 3), (2, (9, 30), 8.0, 3, 3)])
def test_peer_halo_lockstep_matches_single_domain(dim, cells, omega, spp, world, use_comm):
    """use_comm: the exchange-stream protocol of the one-process-per-GPU halos (begin / end around
    each exchange, join before the next begins) is followed on every exchange."""
    space = AddressSpace()
    g = build_grid(dim, [(0.0, 1.0)] * dim, cells, "dirichlet")
    f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 3, seed=7)
    corr = correct_explicit(omega, g, 2, 1.0)
    cfg = FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    shards = [PeerNumpyShard(space, g, r, steps_per_pass=spp) for r in slab_ranges(g.shape[0], world)]
    halos = PeerHalo.local_group(shards)
    for h in halos:
        h.use_comm = use_comm
    for sh in shards:
        sh.set_schedule(time_schedule(corr, cfg))
        p0, p1 = sh.plane_range
        sh.upload(_native.F, f[p0:p1])
    exchange_forcing(shards, halos)
    iters = 3
    res = []
    for _ in range(iters):
        rs = run_peer_local_solve(shards, halos)
        res.append(float(np.sqrt(sum(rs)) / np.sqrt(g.size)))
    v = np.concatenate([sh.download(_native.V) for sh in shards], axis=0)
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    vref, rref = O.fpi(f, g.spacing, sc, iters)
    assert np.array_equal(v, vref)
    np.testing.assert_allclose(res, rref, rtol=1e-12)
    # every copy lands in the neighbour's ghost planes, never in owned planes
    owner = {b // SPAN: q for q, sh in enumerate(shards) for b in sh.base.values()}
    for r, sh in enumerate(shards):
        for _, src, dst, nbytes in sh.ctx.log:
            q = owner[dst // SPAN]
            assert abs(q - r) == 1
            nb = shards[q]
            first = (dst % SPAN) // nb.plane_bytes
            last = first + nbytes // nb.plane_bytes - 1
            assert last < nb.gh or first >= nb.gh + nb.nloc
    # sequence numbers agree across ranks
    assert len({h.seq for h in halos}) == 1
