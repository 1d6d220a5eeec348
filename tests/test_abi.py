"""The C-ABI library loads on a CPU-only host and exports every function the
public header declares; the oracle is a separate library the product never
links."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2401_16543_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "kfvm_b200.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kfvm_[a-z0-9_]+)\s*\(", src)))


def test_header_functions_exported():
    names = declared_functions()
    assert len(names) >= 25
    L = C.CDLL(_abi.LIB_PATH)
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # every ctypes binding in the package refers to a declared function
    bound = {n for n, _, _ in _abi.EXPORTS}
    assert bound <= set(names), bound - set(names)


def test_library_is_sm100a_and_standalone():
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    nm = subprocess.run(["nm", "-D", "--undefined-only", _abi.LIB_PATH], capture_output=True,
                        text=True).stdout
    assert "kfo_" not in nm  # never links the oracle


def test_config_errors_without_gpu():
    """Invalid configurations are rejected with code 1 before touching a GPU."""
    L = _abi.lib()
    cfg = _abi.KfvmConfig()
    L.kfvm_config_defaults(C.byref(cfg), 2, 2, 16, 16, 1, 0)
    assert cfg.eps == 1e-40 and cfg.kappa == 0.4 and cfg.gamma == 1.4
    p = C.POINTER(_abi.KfvmTable)()
    assert L.kfvm_table_build(2, 5, 5.0, C.byref(p)) == _abi.KFVM_ERR_CONFIG
    assert L.kfvm_table_build(2, 2, 5.0, C.byref(p)) == _abi.KFVM_OK
    bad = _abi.KfvmConfig()
    L.kfvm_config_defaults(C.byref(bad), 3, 2, 16, 16, 16, 0)  # dim 3 vs 2-D table
    h = C.c_void_p()
    assert L.kfvm_gpu_create(C.byref(bad), p, None, C.byref(h)) == _abi.KFVM_ERR_CONFIG
    visc = _abi.KfvmConfig()
    L.kfvm_config_defaults(C.byref(visc), 2, 2, 16, 16, 1, 0)
    assert visc.viscous == 0 and visc.prandtl == 0.71 and visc.inv_froude2 == 0.0
    visc.viscous, visc.reynolds = 1, 0.0  # Re must be positive
    assert L.kfvm_gpu_create(C.byref(visc), p, None, C.byref(h)) == _abi.KFVM_ERR_CONFIG
    L.kfvm_table_free(p)


def test_slab_range_partition():
    L = _abi.lib()
    for n, P in ((256, 8), (10, 3), (7, 7)):
        total, prev = 0, 0
        for r in range(P):
            p0, np_ = C.c_int(), C.c_int()
            L.kfvm_slab_range(n, P, r, C.byref(p0), C.byref(np_))
            assert p0.value == prev
            prev = p0.value + np_.value
            total += np_.value
        assert total == n


def test_oracle_is_separate():
    from oracle import kfvm_oracle
    assert os.path.dirname(kfvm_oracle.LIB_PATH).endswith("oracle")
    assert kfvm_oracle.LIB_PATH != _abi.LIB_PATH


def test_no_cpu_fallback_when_library_missing(tmp_path, monkeypatch):
    """The product path fails loudly if libkfvm_b200.so is absent."""
    import importlib
    monkeypatch.setenv("KFVM_LIB", str(tmp_path / "missing.so"))
    mod = importlib.reload(_abi)
    try:
        with pytest.raises(RuntimeError):
            mod.lib()
    finally:
        monkeypatch.delenv("KFVM_LIB")
        importlib.reload(_abi)
