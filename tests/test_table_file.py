"""The hash-pinned table files and the oracle's IC restatement that let the
CPU reference arm of bench.py run without mapping libkfvm_b200.so."""
import numpy as np
import pytest

import paper_2401_16543_b200 as K
from oracle.kfvm_oracle import initial_condition as oracle_ic
from oracle.table_file import PINNED_HASH, TableFile, table_arrays


@pytest.mark.parametrize("dim,R", [(2, 2), (2, 3), (3, 2), (3, 3)])
def test_table_file_equals_live_precompute(dim, R):
    f = TableFile(dim, R)
    live = table_arrays(K.precompute(R, dim=dim).c_table.contents)
    for k, v in live.items():
        assert np.array_equal(f.arr[k].view(np.uint8), v.view(np.uint8)), k
    assert f.hash == PINNED_HASH[(dim, R)] == K.precompute(R, dim=dim).hash
    # the rebuilt struct reads back the same bytes
    again = table_arrays(f.c_table.contents)
    assert all(np.array_equal(again[k], live[k]) for k in live)


@pytest.mark.parametrize("idx,n", [(1, 32), (2, 40), (3, 12), (4, 14), (5, 12)])
def test_oracle_ic_bitwise_equals_product_ic(idx, n):
    w = K.baseline_config(idx, n=n)
    A = K.initial_condition(w.grid, w.ic)
    B = oracle_ic(w.grid, w.ic)
    assert np.array_equal(A.view(np.int64), B.view(np.int64))
    z0, nz = 2, 5
    S = oracle_ic(w.grid, w.ic, z0=z0, nz_local=nz, nthreads=3)
    assert np.array_equal(S, A[z0:z0 + nz])


def test_oracle_runs_on_table_file():
    """The oracle consumes the file table exactly like the live one."""
    from oracle import Oracle
    w = K.baseline_config(3, n=8)
    U = oracle_ic(w.grid, w.ic)
    a = Oracle(w.grid, K.precompute(2, dim=3)).compute_rhs(U)
    b = Oracle(w.grid, TableFile(3, 2)).compute_rhs(U)
    assert np.array_equal(a, b)
