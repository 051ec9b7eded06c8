"""The host Schur services of Krylov-Schur reproduce the reference's
(schur.py) bit for bit on golden inputs, so lock decisions match — both the
C++ services (csrc/schur_host.cu, numpy's own OpenBLAS) and the numpy
restatement.  CPU."""

import numpy as np
import pytest

from conftest import golden


@pytest.fixture(params=["native", "numpy"])
def schur_path(request, monkeypatch):
    from paper_2104_01253_b200 import schur

    nat = schur._native()
    if request.param == "native":
        if not nat:
            pytest.skip("numpy carries no ILP64 OpenBLAS here")
    else:
        monkeypatch.setattr(schur, "_NATIVE", False)
    return request.param


@pytest.mark.parametrize("i", range(10))
def test_schur_services_bitwise(i, schur_path):
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


@pytest.mark.parametrize("seed", range(4))
def test_native_schur_matches_numpy_restatement(seed, monkeypatch):
    """Random dense, Hessenberg, integer and defective-ish matrices: the C++
    services and the numpy restatement agree to the bit (T, Z, moves,
    eigenvectors with arbitrary Z and block picks)."""
    from paper_2104_01253_b200 import schur

    nat = schur._native()
    if not nat:
        pytest.skip("numpy carries no ILP64 OpenBLAS here")
    rng = np.random.default_rng(100 + seed)

    def run():
        out = []
        h, u = schur.hessenberg_reduce(a)
        f = schur.hessenberg_real_schur(h)
        g = schur.SchurForm(f.t.copy(), u @ f.z)
        out += [h, u, f.t, f.z, schur.move_blocks_front(g, sel[:len(g.blocks())] +
                                                       [False] * (len(g.blocks()) - len(sel)))]
        out += [g.t, g.z, *schur.schur_eigenvectors(g, picks(len(g.blocks())))]
        return out

    for trial in range(25):
        n = int(rng.integers(1, 65))
        kind = trial % 4
        if kind == 0:
            a = rng.standard_normal((n, n))
        elif kind == 1:
            a = np.triu(rng.standard_normal((n, n)), -1)
        elif kind == 2:
            a = rng.integers(-2, 3, (n, n)).astype(float)
        else:
            a = np.diag(np.full(n, 4.0)) + 1e-3 * rng.standard_normal((n, n))
        sel = [bool(x) for x in rng.integers(0, 2, n)]

        def picks(nb):
            return None if trial % 2 else list(range(0, nb, 2))

        monkeypatch.setattr(schur, "_NATIVE", False)
        want = run()
        monkeypatch.setattr(schur, "_NATIVE", nat)
        got = run()
        for x, y in zip(want, got):
            assert np.array_equal(x, y)
