"""Several live handles on one device: the constant banks
(c_k, c_t, c_gather, the generated weights) are per device, so a handle whose
constant image differs from a live handle's (different gamma, boundary
kinds, radius) must be refused with KFVM_ERR_CONFIG instead of silently
running with the other handle's constants; identical images share the bank,
and after the last handle of an image is destroyed a different image is
accepted (and computes the oracle's bits)."""
from dataclasses import replace

import numpy as np
import pytest

import paper_2401_16543_b200 as K
from oracle import Oracle

pytestmark = pytest.mark.gpu


def _grid(**over):
    w = K.baseline_config(1, n=16)
    return replace(w.grid, **over), w.ic


def test_different_images_refused(require_gpu):
    g, ic = _grid()
    with K.Solver(g):
        with pytest.raises(ValueError):
            K.Solver(replace(g, gamma=1.6))
        with pytest.raises(ValueError):
            K.Solver(replace(g, bc="outflow"))
        with K.Solver(g):  # same image: shared
            pass


def test_image_released_with_last_handle(require_gpu):
    g, ic = _grid()
    g2 = replace(g, gamma=1.6)
    with K.Solver(g):
        pass
    U = K.initial_condition(g2, ic)
    with K.Solver(g2) as s:  # the first image is gone: accepted
        s.set_state(U)
        d = s.advance(2)
        Ug = s.get_state()
    Uo, do = Oracle(g2, K.precompute(2)).run(U, 2)
    assert np.array_equal(d, do) and np.array_equal(Ug, Uo)
