import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2207_00514_b200 as E
from paper_2207_00514_b200 import mst as M, _lib
import ctypes
pts = E.generate(E.DatasetSpec("normal", 10_000_000, 3, seed=0))
bvh = E.build(pts)
state = E.ComponentState.initial(bvh, device="cuda")
r = 0
def T(): torch.cuda.synchronize(); return time.perf_counter()
while state.num_components > 1:
    r += 1
    E.reduce_labels(bvh, state)
    E.compute_upper_bounds(state, bvh.leaf_perm, pts)
    t0 = T()
    call = M._Call(bvh, pts, state); t1 = T()
    p = call.points(pts); t2 = T()
    lab = M._dev_array(state.labels, "int64", pts.shape[0], "labels"); reps = M._device_reps(lab); t3 = T()
    n = pts.shape[0]
    bu = torch.empty(n, dtype=torch.int64, device="cuda"); bv = torch.empty_like(bu); bw = torch.empty(n, dtype=torch.float64, device="cuda"); t4 = T()
    evals = ctypes.c_int64(0); e = _lib.err_buf()
    with call:
        ta = T()
        rc = _lib.load().emst_find_component_outgoing_edges(call.ctx.handle, None, n, 3, lab.data_ptr(), state.upper_bounds.data_ptr(), None, 3, bu.data_ptr(), bv.data_ptr(), bw.data_ptr(), ctypes.byref(evals), e, len(e))
        tb = T()
    assert rc == 0, e.value
    missing = reps[bv[reps] < 0]; ms = missing.shape[0]; t5 = T()
    out = E.OutgoingEdges(reps, bu, bv, bw, 0)
    E.merge_components(state, out)
    print(f"round {r}: call {1e3*(t1-t0):.2f} pts {1e3*(t2-t1):.2f} reps {1e3*(t3-t2):.2f} empty {1e3*(t4-t3):.2f} C {1e3*(tb-ta):.2f} missing {1e3*(t5-tb):.2f}", flush=True)
