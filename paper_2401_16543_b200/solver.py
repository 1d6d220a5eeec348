"""GPU solver handle: mirror of the SPEC solver/driver API.

Every call goes through the C-ABI of include/kfvm_b200.h into
libkfvm_b200.so; there is no CPU path.  State arrays use the reference AoS
layout (x fastest, nvar conservative components per cell).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _abi
from .config import GridConfig, ICSpec
from .table import KernelConfig, ReconstructionSet, precompute


class KfvmRuntimeError(RuntimeError):
    """Runtime abort: NaN, inadmissible average or limiter abort (exit code 2)."""


class KfvmDeviceError(RuntimeError):
    """CUDA / NCCL / I/O failure (exit code 3)."""


class Solver:
    """One GPU (one rank of a slab decomposition).

    Parameters mirror the reference: ``grid`` (Grid2D + controls),
    ``rset`` the immutable ReconstructionSet.  ``rank``/``nranks``
    select this process's slab of the last axis; ``nccl_id`` is the 128-byte
    unique id from :func:`nccl_unique_id` (rank 0) when nranks > 1.
    """

    def __init__(self, grid: GridConfig, rset: Optional[ReconstructionSet] = None,
                 rank: int = 0, nranks: int = 1, device: int = 0,
                 nccl_id: Optional[bytes] = None):
        self.L = _abi.lib()
        self.grid = grid
        self.rset = rset or precompute(grid.radius, KernelConfig(grid.ell_over_delta), grid.dim)
        if self.rset.dim != grid.dim or self.rset.R != grid.radius:
            raise ValueError("ReconstructionSet does not match the grid")
        self._cfg = grid.c_config()
        dist = None
        if nranks > 1:
            dist = _abi.KfvmDist()
            dist.rank, dist.nranks, dist.device = rank, nranks, device
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("nccl_id (128 bytes) required for nranks > 1")
            C.memmove(dist.nccl_id, nccl_id, 128)
        elif device:
            dist = _abi.KfvmDist()
            dist.rank, dist.nranks, dist.device = 0, 1, device
        h = C.c_void_p()
        rc = self.L.kfvm_gpu_create(C.byref(self._cfg), self.rset.c_table,
                                    C.byref(dist) if dist is not None else None, C.byref(h))
        if rc == _abi.KFVM_ERR_CONFIG:
            raise ValueError("invalid solver configuration")
        if rc != _abi.KFVM_OK:
            raise KfvmDeviceError(f"kfvm_gpu_create failed (code {rc})")
        self.h = h
        p0, npl = C.c_int(), C.c_int()
        self.L.kfvm_slab_range(grid.slab_extent, nranks, rank, C.byref(p0), C.byref(npl))
        self.p0, self.np_local = p0.value, npl.value
        self.rank, self.nranks = rank, nranks
        plane = grid.nx * (grid.ny if grid.dim == 3 else 1)
        self.local_cells = plane * self.np_local
        self.local_shape = ((self.np_local, grid.ny, grid.nx) if grid.dim == 3
                            else (self.np_local, grid.nx)) + (grid.nvar,)

    # ----------------------------------------------------------- plumbing
    def _check(self, rc: int, what: str):
        if rc == _abi.KFVM_OK:
            return
        buf = C.create_string_buffer(512)
        self.L.kfvm_gpu_last_error(self.h, buf, 512)
        msg = f"{what}: {buf.value.decode(errors='replace')}"
        if rc == _abi.KFVM_ERR_RUNTIME:
            raise KfvmRuntimeError(msg)
        if rc == _abi.KFVM_ERR_CONFIG:
            raise ValueError(msg)
        raise KfvmDeviceError(msg)

    def close(self):
        if getattr(self, "h", None):
            self.L.kfvm_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ------------------------------------------------------------- state
    def set_state(self, U: np.ndarray):
        U = np.ascontiguousarray(U, dtype=np.float64)
        if U.size != self.local_cells * self.grid.nvar:
            raise ValueError("state size does not match the rank's slab")
        self._check(self.L.kfvm_gpu_set_state(self.h, U.ctypes.data), "set_state")

    def get_state(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        """The rank's state (AoS); into ``out`` (C-contiguous float64, e.g. a
        pinned buffer) when given."""
        if out is None:
            U = np.empty(self.local_shape, dtype=np.float64)
        else:
            if (out.dtype != np.float64 or not out.flags.c_contiguous
                    or out.size != self.local_cells * self.grid.nvar):
                raise ValueError("out must be a C-contiguous float64 array of the slab's size")
            U = out
        self._check(self.L.kfvm_gpu_get_state(self.h, U.ctypes.data), "get_state")
        return U

    def _host_buf(self, U: np.ndarray, what: str) -> np.ndarray:
        if (U.dtype != np.float64 or not U.flags.c_contiguous
                or U.size != self.local_cells * self.grid.nvar):
            raise ValueError(f"{what}: needs a C-contiguous float64 array of the slab's size")
        return U

    def set_state_async(self, U: np.ndarray):
        """Upload on the handle's stream without waiting; ``U`` (ideally
        pinned) must stay unchanged until :meth:`sync`."""
        U = self._host_buf(U, "set_state_async")
        self._check(self.L.kfvm_gpu_set_state_async(self.h, U.ctypes.data), "set_state_async")

    def get_state_async(self, out: np.ndarray):
        """Read back into ``out`` on the handle's stream; valid after :meth:`sync`."""
        out = self._host_buf(out, "get_state_async")
        self._check(self.L.kfvm_gpu_get_state_async(self.h, out.ctypes.data), "get_state_async")

    def set_state_device(self, ptr: int):
        self._check(self.L.kfvm_gpu_set_state_device(self.h, C.c_void_p(ptr)), "set_state_device")

    def get_state_device(self, ptr: int):
        self._check(self.L.kfvm_gpu_get_state_device(self.h, C.c_void_p(ptr)), "get_state_device")

    def generate_ic(self, ic: ICSpec):
        """Seeded IC generated on the device (bit-identical to initial_condition)."""
        p = ic.c_params()
        self._check(self.L.kfvm_gpu_ic_generate(self.h, C.byref(p)), "ic_generate")

    # -------------------------------------------------- reference API mirror
    def compute_rhs(self, U: Optional[np.ndarray] = None) -> np.ndarray:
        """compute_rhs: dU/dt of the state."""
        if U is not None:
            self.set_state(U)
        out = np.empty(self.local_shape, dtype=np.float64)
        self._check(self.L.kfvm_gpu_rhs(self.h, out.ctypes.data), "compute_rhs")
        return out

    def reconstruct_states(self, U: Optional[np.ndarray] = None) -> np.ndarray:
        """reconstruct_states (KXRCF off): limited face states,
        shape (cells, n_face_points, nvar)."""
        if U is not None:
            self.set_state(U)
        npts = self.rset.n_face_points()
        out = np.empty((self.local_cells, npts, self.grid.nvar), dtype=np.float64)
        self._check(self.L.kfvm_gpu_states(self.h, out.ctypes.data), "reconstruct_states")
        return out

    def kxrcf_flags(self, U: Optional[np.ndarray] = None) -> np.ndarray:
        """KXRCF troubled-cell flags (1 = WENO) of the rank's cells
        for the state (grid must have kxrcf=True)."""
        if U is not None:
            self.set_state(U)
        shape = self.local_shape[:-1]
        out = np.zeros(shape, dtype=np.uint8)
        self._check(self.L.kfvm_gpu_kxrcf_flags(self.h, out.ctypes.data), "kxrcf_flags")
        return out

    def select_dt(self, U: Optional[np.ndarray] = None) -> float:
        """select_dt, fixed-CFL rule."""
        if U is not None:
            self.set_state(U)
        dt = C.c_double()
        self._check(self.L.kfvm_gpu_select_dt(self.h, C.byref(dt)), "select_dt")
        return dt.value

    def ssp_rk3_stage(self, stage: int, dt: float):
        self._check(self.L.kfvm_gpu_stage(self.h, int(stage), float(dt)), "stage")

    def ssp_rk3_step(self) -> float:
        dt = C.c_double()
        self._check(self.L.kfvm_gpu_step(self.h, C.byref(dt)), "step")
        return dt.value

    def advance(self, nsteps: int) -> np.ndarray:
        """nsteps SSP-RK3 steps (graph-captured); returns the dt sequence."""
        dts = np.empty(max(nsteps, 1), dtype=np.float64)
        self._check(self.L.kfvm_gpu_run(self.h, int(nsteps), dts.ctypes.data), "advance")
        return dts[:nsteps]

    def advance_to(self, t_final: float, max_steps: int = 1 << 30) -> tuple:
        """advance_to: fixed-CFL SSP-RK3 steps until t_final (last step
        clipped); returns (steps launched, time reached)."""
        n, t = C.c_int(), C.c_double()
        self._check(self.L.kfvm_gpu_advance_to(self.h, float(t_final), int(max_steps),
                                               C.byref(n), C.byref(t)), "advance_to")
        return n.value, t.value

    def step_stats(self) -> tuple:
        """(accepted, rejected) steps of the last SSP(4,3) advance_to."""
        a, r = C.c_int(), C.c_int()
        self._check(self.L.kfvm_gpu_step_stats(self.h, C.byref(a), C.byref(r)), "step_stats")
        return a.value, r.value

    def run_async(self, nsteps: int):
        self._check(self.L.kfvm_gpu_run_async(self.h, int(nsteps)), "run_async")

    def sync(self):
        self._check(self.L.kfvm_gpu_sync(self.h), "sync")

    def dt_sequence(self, nsteps: int) -> np.ndarray:
        dts = np.empty(nsteps, dtype=np.float64)
        self._check(self.L.kfvm_gpu_dt_sequence(self.h, dts.ctypes.data, nsteps), "dt_sequence")
        return dts

    @property
    def stream(self) -> int:
        return self.L.kfvm_gpu_stream(self.h) or 0

    @property
    def launch_count(self) -> int:
        return int(self.L.kfvm_gpu_launch_count(self.h))

    def set_option(self, name: str, value: int):
        self._check(self.L.kfvm_gpu_set_option(self.h, name.encode(), int(value)), "set_option")

    def kernel_times(self) -> dict:
        v = [C.c_double() for _ in range(4)]
        self.L.kfvm_gpu_kernel_times(self.h, *[C.byref(x) for x in v])
        return dict(zip(("states", "flux", "update", "other"), (x.value for x in v)))


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    rc = _abi.lib().kfvm_nccl_unique_id(buf)
    if rc:
        raise KfvmDeviceError("ncclGetUniqueId failed (libnccl.so.2 not loadable?)")
    return bytes(buf)


def loopback_id() -> bytes:
    """Group id of the in-process loopback transport (kfvm_loopback_id): the
    nranks Solver handles created with it in this process (same device, one
    host thread per rank) exchange halos and reductions by device copies."""
    buf = (C.c_ubyte * 128)()
    _abi.lib().kfvm_loopback_id(buf)
    return bytes(buf)
