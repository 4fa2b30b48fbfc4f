"""Build variant libraries for tuning sweeps (compile-time kernel constants), e.g.

    python tools/variants.py wf_st12 -DWHB_WF_ST_EXTRA=8

writes paper_2504_03074_b200/lib/variants/libwhb200_<name>.so; select it at run time with
WHB_LIB=libwhb200_<name>.so.  The default build (build()) is what the product ships."""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_03074_b200 import _build  # noqa: E402


def build_variant(name, defines):
    out_dir = os.path.join(_build.LIB_DIR, "variants")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, f"libwhb200_{name}.so")
    cmd = [_build.nvcc(), *_build.NVCC_FLAGS, *defines, "-o", out, _build.SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stderr[-3000:])
        raise SystemExit(f"variant {name} failed")
    return out


if __name__ == "__main__":
    print(build_variant(sys.argv[1], sys.argv[2:]))
