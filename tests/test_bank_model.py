"""The half-warp shared-memory bank model behind the 3-D R=2 tensor engines'
layout (tools/bank_model.py): the numbers quoted in the design
(and matched by the ncu wavefront counts in profiles/r02) follow from the
chunk tables, so a change of the stencil order that would undo the layout
choice shows up here."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _model():
    spec = importlib.util.spec_from_file_location("bank_model", os.path.join(ROOT, "tools", "bank_model.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_ring_load_wavefronts():
    m = _model()
    stride4 = m.ring(36, lambda r: 4 * r)
    contig36 = m.ring(36, lambda r: r)
    contig42 = m.ring(42, lambda r: r)
    # cells 4 apart, rows 36 words apart: ~4 wavefronts per 64-bit load (ncu: 4.0-4.6)
    assert 3.8 < m.wavefronts(m.ch1, stride4) < 4.2
    assert 3.9 < m.wavefronts(m.ch2, stride4) < 4.3
    # contiguous cells: 3.4-3.6; with rows 42 words apart: ~2.1 (2 is the minimum)
    assert 3.2 < m.wavefronts(m.ch1, contig36) < 3.7
    assert m.wavefronts(m.ch1, contig42) < 2.25
    assert m.wavefronts(m.ch2, contig42) < 2.25


def test_cache_rows_of_eight_cells_conflict():
    m = _model()
    f = lambda k4, e, r8: 8 * e + r8  # noqa: E731
    assert m.wavefronts(m.ch1[m.K0:], f) > 4.0  # why the cache is split by half-warp and coloured
