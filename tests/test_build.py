"""Register/spill budget of the hot kernels, from the ptxas report the build
writes (build/ptxas_kfvm_gpu.txt, make -Xptxas -v; no GPU needed).  The
documented budgets (kfvm_gpu.cu / kfvm_recon_u.cuh comments,
profiles/r02/README.md) are asserted so a comment cannot drift from the
compiled code again."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LOG = os.path.join(ROOT, "build", "ptxas_kfvm_gpu.txt")


def kernels():
    if not os.path.exists(LOG):
        pytest.skip("no ptxas report (library not built with make)")
    txt = open(LOG).read()
    out = {}
    for b in re.split(r"ptxas info    : Compiling entry function ", txt)[1:]:
        name = b.split("'")[1]
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", b)
        r = re.search(r"Used (\d+) registers", b)
        out[dem] = (int(r.group(1)), int(m.group(1)), int(m.group(2)))
    return out


def pick(ks, pat):
    hits = {k: v for k, v in ks.items() if re.search(pat, k)}
    assert hits, pat
    return hits


def test_3d_hot_kernels_do_not_spill():
    ks = kernels()
    for pat in [r"k_flux<3, 2>", r"k_flux<3, 3>", r"k_update<3, false>", r"k_bounds<3>"]:
        for k, (regs, st, ld) in pick(ks, re.escape(pat)).items():
            assert st == 0 and ld == 0, (k, regs, st, ld)


def test_3d_tensor_engine_fits_four_ctas_per_sm():
    """3-D R=2 tensor engine: 128 registers (4 x 128 threads per SM) with the
    documented small spill (kfvm_recon_u.cuh, KFVM_U_MINB32)."""
    ks = kernels()
    for k, (regs, st, ld) in pick(ks, re.escape("k_states_u<3, 2, false, false, ")).items():
        assert regs <= 128 and st <= 64 and ld <= 64, (k, regs, st, ld)


def test_3d_wide_engine_fits_one_cta_per_sm():
    """k_states_w<4>: 512 threads at 128 registers (the whole register file of
    an SM) with a small documented spill (kfvm_recon_w.cuh)."""
    ks = kernels()
    for k, (regs, st, ld) in pick(ks, re.escape("k_states_w<4, ")).items():
        assert regs <= 128 and st <= 64 and ld <= 64, (k, regs, st, ld)


def test_2d_flux_spill_budget_as_documented():
    """2-D k_flux runs at 64 registers (8 CTAs/SM) and spills a documented
    amount (kfvm_gpu.cu comment above k_flux)."""
    ks = kernels()
    for k, (regs, st, ld) in pick(ks, re.escape("k_flux<2, 2>")).items():
        assert regs == 64 and st <= 368, (k, regs, st, ld)
