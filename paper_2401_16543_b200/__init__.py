"""B200-native KFVM-WENO FP64 stage update (arXiv 2401.16543).

Host-side mirror of the reference's operator API for the hot path
(SURVEY.md §8(b)), over the C-ABI library libkfvm_b200.so:

* :func:`precompute` / :class:`ReconstructionSet` / :class:`StencilVectors`
  mirror ``kfvm::precompute`` and the table types of
  proj/core/include/kfvm/kernel_recon.hpp:67-110 (generalised to 3-D).
* :class:`Solver` mirrors the SPEC solver module:
  ``compute_rhs``, ``reconstruct_states``, ``select_dt``
  (S:607), ``ssp_rk3_stage``/``ssp_rk3_step`` (BASELINE's SSP-RK3 in place of
  ``ssp43_step`` S:598) and ``advance`` (fixed-step ``advance_to`` S:616).

Errors follow the reference: bad radius / configuration raise ValueError
(``std::invalid_argument``, geometry.hpp:64), runtime aborts (NaN,
inadmissible averages) raise :class:`KfvmRuntimeError` (exit code 2),
device failures raise :class:`KfvmDeviceError` (exit code 3).
"""
from .table import KernelConfig, ReconstructionSet, StencilVectors, precompute  # noqa: F401
from .config import GridConfig, BASELINE_CONFIGS, baseline_config, initial_condition  # noqa: F401
from .solver import Solver, KfvmRuntimeError, KfvmDeviceError  # noqa: F401
from ._abi import lib as _lib  # noqa: F401

__all__ = [
    "KernelConfig", "ReconstructionSet", "StencilVectors", "precompute",
    "GridConfig", "BASELINE_CONFIGS", "baseline_config", "initial_condition",
    "Solver", "KfvmRuntimeError", "KfvmDeviceError",
]
