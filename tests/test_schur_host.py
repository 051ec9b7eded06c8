"""The host Schur services of Krylov-Schur reproduce the reference's
(schur.py) bit for bit on golden inputs, so lock decisions match.  CPU."""

import numpy as np
import pytest

from conftest import golden


@pytest.mark.parametrize("i", range(10))
def test_schur_services_bitwise(i):
    from paper_2104_01253_b200.schur import (SchurForm, hessenberg_real_schur, hessenberg_reduce,
                                            move_blocks_front, schur_eigenvectors, sort_schur)

    g = golden("schur.npz")
    h, u = hessenberg_reduce(g[f"a{i}"])
    assert np.array_equal(h, g[f"h{i}"]) and np.array_equal(u, g[f"u{i}"])
    f = hessenberg_real_schur(h)
    assert np.array_equal(f.t, g[f"t{i}"]) and np.array_equal(f.z, g[f"z{i}"])
    m = SchurForm(f.t.copy(), f.z.copy())
    assert move_blocks_front(m, list(g[f"sel{i}"])) == g[f"moved{i}"]
    assert np.array_equal(m.t, g[f"mt{i}"]) and np.array_equal(m.z, g[f"mz{i}"])
    vals, vecs = schur_eigenvectors(m)
    assert np.array_equal(vals, g[f"vals{i}"]) and np.array_equal(vecs, g[f"vecs{i}"])
    s = SchurForm(f.t.copy(), f.z.copy())
    sort_schur(s, lambda lam: lam.real)
    assert np.array_equal(s.t, g[f"st{i}"]) and np.array_equal(s.z, g[f"sz{i}"])


def test_match_eigenvalues_and_ritz_residual():
    from paper_2104_01253_b200 import EigenvalueTable, match_eigenvalues, ritz_residual

    t = EigenvalueTable(values=np.array([1.0, 2.0, 2.0]), unique=np.array([1.0, 2.0]),
                        multiplicity=np.array([1, 2]))
    rep = match_eigenvalues([2.0, 2.0 + 1e-9, 2.0 - 1e-9, 1.0], t, 1e-7)
    assert rep.n_matched == 3 and rep.over_multiplicity
    assert ritz_residual(np.eye(3), [1, 0, 0]) == 0.0
    hb = np.zeros((3, 2))
    hb[2, :] = [0.5, -2.0]
    assert ritz_residual(hb, [0.0, 1.0]) == 2.0
