"""Graph transpose / CSR build (graphs.py:59-105).

CPU tier: the oracle restatement reproduces the reference's outputs
(tests/golden/golden_graphs.npz, made by make_golden_graphs.py from the
unmodified reference).  GPU tier: ss_graph_transpose / ss_csr_from_edges
reproduce the same fixtures byte for byte, plus the reference tests'
properties (involution, degree conservation, errors) at larger sizes.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden_graphs.npz"))
CASES = [str(c) for c in G["cases"]]


def _case(c):
    return int(G[f"{c}_n"][0]), G[f"{c}_src"], G[f"{c}_dst"]


@pytest.mark.parametrize("case", CASES)
def test_oracle_matches_reference(case):
    n, src, dst = _case(case)
    off, tgt = O.csr_from_edges(n, src, dst)
    assert np.array_equal(off, G[f"{case}_off"]) and np.array_equal(tgt, G[f"{case}_tgt"])
    toff, ttgt = O.graph_transpose(n, off, tgt)
    assert np.array_equal(toff, G[f"{case}_toff"]) and np.array_equal(ttgt, G[f"{case}_ttgt"])


# ---- GPU ------------------------------------------------------------------

@pytest.fixture(scope="module")
def S():
    import paper_2304_10078_b200 as S
    return S


def _np(t):
    return t.cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_from_edges_and_transpose_golden(S, case):
    n, src, dst = _case(case)
    g = S.from_edges(n, src, dst)
    assert np.array_equal(_np(g.offsets), G[f"{case}_off"])
    assert np.array_equal(_np(g.targets), G[f"{case}_tgt"])
    tel = S.Telemetry()
    t = S.transpose(g, telemetry=tel)
    assert np.array_equal(_np(t.offsets), G[f"{case}_toff"])
    assert np.array_equal(_np(t.targets), G[f"{case}_ttgt"])
    assert t.num_vertices == n and t.num_edges == len(src)
    assert tel.scratch_allocations == (1 if len(src) else tel.scratch_allocations)


@pytest.mark.gpu
def test_involution_and_degrees_large(S):
    rng = np.random.default_rng(7)
    n, m = 1 << 18, 1 << 22
    src = np.minimum(rng.zipf(1.3, m) - 1, n - 1).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    order = np.lexsort((dst, src))
    g = S.from_edges(n, src[order], dst[order])
    t = S.transpose(g)
    assert S.transpose(t) == g                                   # canonical input: involution
    in_deg = np.bincount(dst, minlength=n)
    assert np.array_equal(np.diff(_np(t.offsets).astype(np.int64)), in_deg)
    toff, ttgt = O.graph_transpose(n, _np(g.offsets), _np(g.targets))
    assert np.array_equal(_np(t.offsets), toff) and np.array_equal(_np(t.targets), ttgt)


@pytest.mark.gpu
def test_double_transpose_canonicalizes(S):
    rng = np.random.default_rng(23)
    g = S.from_edges(100, rng.integers(0, 100, 2000), rng.integers(0, 100, 2000))
    once = S.transpose(g)
    assert S.transpose(S.transpose(once)) == once


@pytest.mark.gpu
def test_graph_errors(S):
    with pytest.raises(S.InputFormatError):
        S.CsrGraph(2, 1, np.array([0, 2, 1], np.uint64), np.array([0], np.uint32)).validate()
    with pytest.raises(S.InputFormatError):
        S.CsrGraph(2, 1, np.array([0, 0, 1], np.uint64), np.array([5], np.uint32)).validate()
    with pytest.raises(S.InputFormatError):
        S.CsrGraph(2, 2, np.array([0, 1, 1], np.uint64), np.array([0], np.uint32)).validate()
    with pytest.raises(S.InputFormatError):
        S.from_edges(2, [0], [5])
    with pytest.raises(S.InputFormatError):
        S.transpose(S.CsrGraph(3, 1, np.array([0, 1, 1, 0], np.uint64), np.array([1], np.uint32)))
