"""Compare reconstruct_states of two engines on a small BASELINE config and
report where they differ (debugging aid)."""
import sys
import numpy as np
import paper_2401_16543_b200 as K

idx, n, e0, e1 = (int(x) for x in sys.argv[1:5])
w = K.baseline_config(idx, n=n)
U = K.initial_condition(w.grid, w.ic)
out = []
for e in (e0, e1):
    with K.Solver(w.grid) as s:
        s.set_option("engine", e)
        out.append(s.reconstruct_states(U))
A, B = out
d = np.argwhere(A != B)
print("shape", A.shape, "ndiff", len(d))
if len(d):
    cells = np.unique(d[:, 0])
    print("cells", cells[:40], "points", np.unique(d[:, 1]), "vars", np.unique(d[:, 2]))
    i = tuple(d[0]); print("first", i, A[i], B[i])
out = []
for e in (e0, e1):
    with K.Solver(w.grid) as s:
        s.set_option("engine", e)
        out.append(s.compute_rhs(U))
A, B = out
d = np.argwhere(A != B)
print("rhs ndiff", len(d), d[:10].tolist(), "maxabs", np.abs(A - B).max(), "scale", np.abs(A).max())
