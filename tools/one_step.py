"""Reconstruct / step a BASELINE config at small n (debugging aid:
KFVM_DEBUG_SYNC=1 reports the first failing kernel)."""
import sys
import paper_2401_16543_b200 as K

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
eng = int(sys.argv[3]) if len(sys.argv) > 3 else -1
w = K.baseline_config(idx, n=n)
U = K.initial_condition(w.grid, w.ic)
with K.Solver(w.grid) as s:
    if eng >= 0:
        s.set_option("engine", eng)
    St = s.reconstruct_states(U)
    print("states ok", St.shape, flush=True)
    print(s.advance(1))
