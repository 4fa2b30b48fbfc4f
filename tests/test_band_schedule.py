"""CPU: the launch schedule of the banded host solve (solve_host_banded, csrc/whb200.cu) orders
every data hazard.

The C++ code enqueues the (pass p, band b) launches by diagonals d = p + b (passes ascending),
diagonal d on stream d % NS; a launch waits for the upload event of band b+1 (pass 0) or for the
events of (p-1, b) and (p-1, b-1) (with one stream, stream order alone).  This test restates that
schedule, builds the happens-before relation it implies (stream FIFO order + event waits) and
checks that every pair of launches touching the same (level-ring slot or field, band) with at
least one write is ordered the way the pass-by-pass solve orders it -- for 3-step and 2-step
passes, 1-4 streams, and the 6-slot level ring (level L >= 1 in slot L mod 6, level 0 = v)."""

import itertools

import pytest


def passes_for(ns):
    """solve_host_banded: three-step passes while the remainder stays 0, 2 or 4; then two-step ones."""
    out, s = [], 0
    while ns - s >= 3 and (ns - s - 3) != 1:
        out.append((s, 3))
        s += 3
    while ns - s >= 2:
        out.append((s, 2))
        s += 2
    assert s == ns
    return out


def slot(level):
    return "v" if level <= 0 else f"ring{level % 6}"


def accesses(passes, p, b, nb, fpi):
    """(reads, writes) of launch (p, b) as sets of (buffer, band)."""
    s, k = passes[p]
    last = p == len(passes) - 1
    near = [c for c in (b - 1, b, b + 1) if 0 <= c < nb]  # a k-step pass reaches <= 3 rows past its band
    reads = {(slot(s), c) for c in near} | {(slot(s - 1), c) for c in near} | {("f", c) for c in near}
    if p > 0:
        reads.add(("acc", b))
    writes = set()
    if last:
        reads.add(("v", b))  # the residual / mat-vec reads v at the output points
        writes.add(("v" if fpi else "out", b))
    else:
        writes |= {(slot(s + k - 1), b), (slot(s + k), b), ("acc", b)}
    return reads, writes


def schedule(npass, nb, ns_streams):
    """Enqueue order and waits of solve_host_banded: [(p, b, stream, [awaited launches])]."""
    out = []
    for d in range(nb + npass - 1):
        for p in range(npass):
            b = d - p
            if not 0 <= b < nb:
                continue
            waits = []
            if p > 0 and ns_streams > 1:
                waits.append((p - 1, b))
                if b > 0:
                    waits.append((p - 1, b - 1))
            out.append((p, b, d % ns_streams, waits))
    return out


@pytest.mark.parametrize("ns_steps,nb,streams,fpi", [(83, 9, 2, True), (83, 9, 1, True), (82, 7, 3, False),
                                                     (84, 8, 4, True), (9, 5, 2, False), (35, 2, 2, True)])
def test_banded_schedule_orders_every_hazard(ns_steps, nb, streams, fpi):
    passes = passes_for(ns_steps)
    sched = schedule(len(passes), nb, streams)
    index = {(p, b): i for i, (p, b, _, _) in enumerate(sched)}
    assert len(index) == len(passes) * nb
    # happens-before: predecessor sets, closed transitively in enqueue order (every edge points backwards)
    before = [set() for _ in sched]
    last_on_stream = {}
    for i, (p, b, st, waits) in enumerate(sched):
        preds = [index[w] for w in waits]
        assert all(j < i for j in preds), "an awaited event is recorded before the wait is enqueued"
        if st in last_on_stream:
            preds.append(last_on_stream[st])
        last_on_stream[st] = i
        for j in preds:
            before[i] |= before[j] | {j}
    acc = [accesses(passes, p, b, nb, fpi) for (p, b, _, _) in sched]
    for i, j in itertools.combinations(range(len(sched)), 2):
        (pi, bi, _, _), (pj, bj, _, _) = sched[i], sched[j]
        ri, wi = acc[i]
        rj, wj = acc[j]
        if not (wi & (rj | wj) or wj & ri):
            continue
        assert pi != pj, f"launches of one pass never conflict: {sched[i][:2]} {sched[j][:2]}"
        first, second = (i, j) if pi < pj else (j, i)
        assert first in before[second], (f"hazard not ordered: {sched[first][:2]} -> {sched[second][:2]} "
                                         f"({(acc[first][1] & (acc[second][0] | acc[second][1])) or (acc[second][1] & acc[first][0])})")
