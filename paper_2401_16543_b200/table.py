"""Reconstruction table: mirror of kfvm::ReconstructionSet / StencilVectors.

Reference: proj/core/include/kfvm/kernel_recon.hpp:14-110 (KernelConfig,
StencilVectors, ReconstructionSet, precompute, evaluate) and
proj/core/include/kfvm/geometry.hpp:50-61 (StencilGeometry).  The arrays are
views of the immutable table built once by ``kfvm_table_build`` in binary128
(SURVEY.md §0.6); both the GPU and the CPU oracle consume these exact bytes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi


@dataclass(frozen=True)
class KernelConfig:
    """kernel_recon.hpp:14-16 — squared-exponential length scale in cell units."""
    ell_over_delta: float = 5.0


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    ct = C.c_int if dtype == np.int32 else C.c_double
    buf = C.cast(ptr, C.POINTER(ct * n)).contents
    return np.frombuffer(buf, dtype=dtype, count=n).copy()


@dataclass
class StencilVectors:
    """kernel_recon.hpp:69-86: vectors of one (sub)stencil, rows aligned with
    the stencil's lexicographic cell order."""
    count: int
    degree: int
    gather: np.ndarray  # position of each cell within the full stencil
    face: np.ndarray    # [n_face_points][count]
    deriv: np.ndarray   # [n_derivs][count]

    def face_row(self, s: int) -> np.ndarray:
        return self.face[s]

    def deriv_row(self, a: int) -> np.ndarray:
        return self.deriv[a]


class ReconstructionSet:
    """kernel_recon.hpp:88-101 (plus 3-D).  Owns the C table handle."""

    def __init__(self, R: int, kernel: KernelConfig = KernelConfig(), dim: int = 2):
        L = _abi.lib()
        p = C.POINTER(_abi.KfvmTable)()
        rc = L.kfvm_table_build(int(dim), int(R), float(kernel.ell_over_delta), C.byref(p))
        if rc == _abi.KFVM_ERR_CONFIG:
            raise ValueError("unsupported stencil radius (must be 2 or 3) or dimension")
        if rc != _abi.KFVM_OK:
            raise RuntimeError(f"precompute failed (code {rc}): block solve residual > 1e-9")
        self._ptr = p
        t = p.contents
        self.R = t.radius
        self.dim = t.dim
        self.kernel = kernel
        self.n_stencils = t.n_stencils
        nfull, npts, nal = t.n_full, t.n_points, t.n_alpha
        self.offsets = _arr(t.offsets, 3 * nfull, np.int32).reshape(nfull, 3)
        self.alphas = _arr(t.alpha, 3 * nal, np.int32).reshape(nal, 3)
        self.points = _arr(t.points, 3 * npts, np.float64).reshape(npts, 3)
        self.face_weights = _arr(t.face_weights, npts, np.float64)
        self.gamma = _arr(t.gamma_lin, t.n_stencils, np.float64)
        self.gl_nodes = _arr(t.gl_nodes, self.R, np.float64)
        self.gl_weights = _arr(t.gl_weights, self.R, np.float64)
        self.hash = int(t.hash)
        gather = _arr(t.gather, t.total_cells, np.int32)
        face = _arr(t.face, t.total_cells * npts, np.float64)
        deriv = _arr(t.deriv, t.total_cells * nal, np.float64)
        self.st = []
        for q in range(t.n_stencils):
            n, o = t.size[q], t.cell_offset[q]
            self.st.append(StencilVectors(
                count=n, degree=t.degree[q], gather=gather[o:o + n],
                face=face[o * npts:(o + n) * npts].reshape(npts, n),
                deriv=deriv[o * nal:(o + n) * nal].reshape(nal, n)))

    # kernel_recon.hpp:97-99
    def n_face_points(self) -> int:
        return self._ptr.contents.n_points

    def n_derivs(self) -> int:
        return self._ptr.contents.n_alpha

    def cells(self, q: int) -> np.ndarray:
        """Offsets of (sub)stencil q (geometry.hpp:57-60)."""
        return self.offsets[self.st[q].gather]

    @property
    def c_table(self):
        return self._ptr

    def __del__(self):
        try:
            if getattr(self, "_ptr", None):
                _abi.lib().kfvm_table_free(self._ptr)
                self._ptr = None
        except Exception:
            pass


_CACHE: dict = {}


def precompute(R: int, kernel: KernelConfig = KernelConfig(), dim: int = 2) -> ReconstructionSet:
    """kernel_recon.hpp:107 — deterministic, so results are cached per key."""
    key = (int(dim), int(R), float(kernel.ell_over_delta))
    if key not in _CACHE:
        _CACHE[key] = ReconstructionSet(R, kernel, dim)
    return _CACHE[key]


def evaluate(r: np.ndarray, g: np.ndarray) -> float:
    """kernel_recon.hpp:64-65: r . g; raises on length mismatch (std::length_error)."""
    if len(r) != len(g):
        raise ValueError("length mismatch")
    return float(np.dot(r, g))
