"""Debug: GPU upper bounds vs a numpy restatement (developer tool)."""
import numpy as np
import paper_2207_00514_b200 as E

pts = E.generate(E.DatasetSpec("uniform", 1000, 2, seed=0))
tree = E.build(pts)
perm = np.asarray(tree.leaf_perm)
n = len(pts)
labels = np.arange(n, dtype=np.int64)
state = E.ComponentState(labels.copy(), np.full(n - 1, E.MIXED, np.int64), np.full(n, np.inf))
ub = E.compute_upper_bounds(state, perm, pts).copy()
want = np.full(n, np.inf)
p64 = pts.astype(np.float64)
for s in range(n - 1):
    a, b = perm[s], perm[s + 1]
    if labels[a] != labels[b]:
        w = np.sqrt(((p64[a] - p64[b]) ** 2).sum())
        want[labels[a]] = min(want[labels[a]], w)
        want[labels[b]] = min(want[labels[b]], w)
bad = np.nonzero(ub != want)[0]
print("mismatches", len(bad))
inv = np.argsort(perm)
for i in bad[:20]:
    print(i, "slot", inv[i], ub[i], want[i])
