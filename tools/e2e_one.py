"""One (or a few) whb_iterate_host calls on a bench workload, for profiling the banded host
iteration: python tools/e2e_one.py [workload] [calls]   (WHB_PIPE_TRACE=1 prints the stage times)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import argparse  # noqa: E402

import bench  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 2
args = argparse.Namespace(workload=wl)
run = bench.SingleRun(args, 0)
import paper_2504_03074_b200 as wh  # noqa: E402
from paper_2504_03074_b200 import _native  # noqa: E402

step = wh.HostFPIStep(run.prob, run.cfg, device_state=run.dp)
bufs = [_native.PinnedBuffer(run.g.shape), _native.PinnedBuffer(run.g.shape)]
bufs[0].array[...] = 0.0
for i in range(calls):
    t0 = time.perf_counter()
    d = step(bufs[i % 2].array, bufs[(i + 1) % 2].array)
    print(f"call {i}: {time.perf_counter() - t0:.4f} s, residual {d:.6e}", flush=True)
