"""Where the end-to-end call spends its time (developer tool): pageable numpy in, numpy out.

  python tools/e2e_breakdown.py [config]      (EMST_STAGE=0 for the plain cudaMemcpy path)
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_00514_b200 as E  # noqa: E402

cfg = {"blobs3d_37m": ("blobs", 37_000_000, 3), "normal3d_10m": ("normal", 10_000_000, 3)}[
    sys.argv[1] if len(sys.argv) > 1 else "blobs3d_37m"]
pts = E.generate(E.DatasetSpec(cfg[0], cfg[1], cfg[2], seed=0))
ctx = E.Context(0)
for it in range(4):
    t0 = time.perf_counter()
    res = E.boruvka_emst(pts, context=ctx)
    t1 = time.perf_counter()
    st = ctx.last_stats
    dev = 1e3 * (res.phase_timings["tree"] + res.phase_timings["mst"])
    print(f"stage={os.environ.get('EMST_STAGE', '1')} call {1e3 * (t1 - t0):.1f} ms, device tree+mst {dev:.1f} ms, "
          f"host/PCIe {1e3 * (t1 - t0) - dev:.1f} ms (in {st.host_in_ms:.1f} ms, out {st.host_out_ms:.1f} ms)", flush=True)
