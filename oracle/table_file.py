"""Hash-pinned reconstruction tables on disk (TEST INFRASTRUCTURE ONLY).

The table is the immutable ReconstructionSet of
proj/core/include/kfvm/kernel_recon.hpp:67-101 in the kfvm_table layout of
include/kfvm_b200.h.  oracle/tables/*.npz hold the canonical binary128
precompute rounded to FP64 (written by tools/export_tables.py).  load_table()
rebuilds a kfvm_table struct from those bytes with ctypes and numpy only —
no product library is mapped — and checks the FNV-1a hash against both the
stored value and PINNED_HASH, so the CPU reference arm of bench.py runs on
exactly the table the GPU consumes.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2401_16543_b200._abi import KfvmTable  # struct layout only (no library load)

_HERE = os.path.dirname(os.path.abspath(__file__))

# FNV-1a 64 of every table array (kfvm_table.hash), recorded in BASELINE.md §3
PINNED_HASH = {
    (2, 2): 0xf969e8f9b1ea6355,
    (2, 3): 0xf59bbd6a85a739de,
    (3, 2): 0x54cdaf1c17a1eb7c,
    (3, 3): 0x832dd6fa6b217913,
}

FIELDS = ("header", "size", "degree", "cell_offset", "offsets", "gather", "alpha", "face",
          "deriv", "gamma_lin", "face_weights", "points", "gl_nodes", "gl_weights",
          "ell_over_delta", "hash")


def _view(ptr, n, ct, dt):
    return np.frombuffer(C.cast(ptr, C.POINTER(ct * n)).contents, dtype=dt, count=n).copy()


def table_arrays(t: KfvmTable) -> dict:
    """Plain arrays of a kfvm_table (for export and byte comparisons)."""
    nf, npt, na, tot, R = t.n_full, t.n_points, t.n_alpha, t.total_cells, t.radius
    I, D = (C.c_int, np.int32), (C.c_double, np.float64)
    return {
        "header": np.array([t.dim, t.radius, t.n_stencils, t.n_points, t.n_alpha, t.n_full,
                            t.total_cells], dtype=np.int32),
        "size": np.array(t.size[:], dtype=np.int32),
        "degree": np.array(t.degree[:], dtype=np.int32),
        "cell_offset": np.array(t.cell_offset[:], dtype=np.int32),
        "offsets": _view(t.offsets, 3 * nf, *I),
        "gather": _view(t.gather, tot, *I),
        "alpha": _view(t.alpha, 3 * na, *I),
        "face": _view(t.face, tot * npt, *D),
        "deriv": _view(t.deriv, tot * na, *D),
        "gamma_lin": _view(t.gamma_lin, t.n_stencils, *D),
        "face_weights": _view(t.face_weights, npt, *D),
        "points": _view(t.points, 3 * npt, *D),
        "gl_nodes": _view(t.gl_nodes, R, *D),
        "gl_weights": _view(t.gl_weights, R, *D),
        "ell_over_delta": np.array([t.ell_over_delta]),
        "hash": np.array([t.hash], dtype=np.uint64),
    }


def fnv1a(arr: dict) -> int:
    """kfvm_table.hash: FNV-1a 64 over the header, size, degree, offsets,
    gather, alpha, face, deriv, gamma_lin, face_weights and ell/Delta bytes
    (the order of kfvm_table.cpp's build)."""
    parts = [arr["header"][[0, 1, 5, 3, 4]], arr["size"], arr["degree"], arr["offsets"],
             arr["gather"], arr["alpha"], arr["face"], arr["deriv"], arr["gamma_lin"],
             arr["face_weights"], arr["ell_over_delta"]]
    data = np.frombuffer(b"".join(np.ascontiguousarray(p).tobytes() for p in parts), np.uint8)
    h = 1469598103934665603
    m = (1 << 64) - 1
    for b in data.tolist():
        h = ((h ^ b) * 1099511628211) & m
    return h


class TableFile:
    """A kfvm_table rebuilt from oracle/tables/*.npz; keeps its arrays alive.
    Duck-types the parts of paper_2401_16543_b200.ReconstructionSet that the
    oracle wrapper uses (c_table, dim, R, n_face_points, n_derivs, counts)."""

    def __init__(self, dim: int, R: int, check_pin: bool = True):
        path = os.path.join(_HERE, "tables", f"kfvm_table_d{dim}_r{R}.npz")
        with np.load(path) as z:
            self.arr = {k: z[k] for k in FIELDS}
        a = self.arr
        h = fnv1a(a)
        if h != int(a["hash"][0]):
            raise ValueError(f"{path}: content hash {h:#x} != stored {int(a['hash'][0]):#x}")
        if check_pin and PINNED_HASH.get((dim, R)) not in (None, 0) and h != PINNED_HASH[(dim, R)]:
            raise ValueError(f"{path}: hash {h:#x} differs from the pinned {PINNED_HASH[(dim, R)]:#x}")
        self.hash = h
        t = KfvmTable()
        hd = a["header"]
        t.dim, t.radius, t.n_stencils, t.n_points, t.n_alpha, t.n_full, t.total_cells = map(int, hd)
        for q in range(8):
            t.size[q], t.degree[q], t.cell_offset[q] = (int(a["size"][q]), int(a["degree"][q]),
                                                         int(a["cell_offset"][q]))
        self._keep = {}
        for name, ct in (("offsets", C.c_int), ("gather", C.c_int), ("alpha", C.c_int),
                         ("face", C.c_double), ("deriv", C.c_double), ("gamma_lin", C.c_double),
                         ("face_weights", C.c_double), ("points", C.c_double),
                         ("gl_nodes", C.c_double), ("gl_weights", C.c_double)):
            buf = np.ascontiguousarray(a[name])
            self._keep[name] = buf
            setattr(t, name, buf.ctypes.data_as(C.POINTER(ct)))
        t.ell_over_delta = float(a["ell_over_delta"][0])
        t.hash = h
        self._t = t
        self.dim, self.R = int(hd[0]), int(hd[1])
        self.n_stencils = int(hd[2])
        self.counts = [int(x) for x in a["size"][:self.n_stencils]]

    @property
    def c_table(self):
        return C.pointer(self._t)

    def n_face_points(self) -> int:
        return self._t.n_points

    def n_derivs(self) -> int:
        return self._t.n_alpha


def load_table(dim: int, R: int) -> TableFile:
    return TableFile(dim, R)
