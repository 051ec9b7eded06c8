"""Pin the CPU oracle (oracle/) against golden vectors the reference itself
produced (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import oracle
from conftest import golden


def _csr_apply(ptr, idx, dat):
    return lambda x: oracle.csr_matvec(ptr, idx, dat, x)


def test_csr_matvec_ragged_bitwise():
    g = golden("csr_ragged.npz")
    y = oracle.csr_matvec(g["indptr"], g["indices"], g["data"], g["x"])
    assert np.array_equal(y, g["y"])


def test_stencil_bitwise_and_csr_assembly():
    g = golden("operators.npz")
    for dims in ((5, 4, 6), (1, 1, 1), (3, 1, 7), (8, 8, 8)):
        key = "x".join(map(str, dims))
        assert np.array_equal(oracle.stencil7_matvec(g[f"x_{key}"], dims), g[f"y_{key}"])
        ptr, idx, dat = oracle.laplace3d_csr(*dims)
        assert np.array_equal(ptr, g[f"csr_indptr_{key}"])
        assert np.array_equal(idx, g[f"csr_indices_{key}"])
        assert np.array_equal(dat, g[f"csr_data_{key}"])


@pytest.mark.parametrize("k,beta", [(1, 0.5), (2, 0.5), (4, 0.5), (7, 0.3), (10, 0.5), (6, 0.0)])
def test_manteuffel_assembly_bitwise(k, beta):
    g = golden("operators.npz")
    ptr, idx, dat = oracle.manteuffel_csr(k, beta)
    assert np.array_equal(ptr, g[f"mant_indptr_{k}_{beta}"])
    assert np.array_equal(idx, g[f"mant_indices_{k}_{beta}"])
    assert np.array_equal(dat, g[f"mant_data_{k}_{beta}"])


@pytest.mark.parametrize("scheme", ["dcgs2", "cgs2"])
def test_arnoldi_manteuffel10(scheme):
    g = golden("arnoldi_m10.npz")
    apply = _csr_apply(*oracle.manteuffel_csr(10, 0.5))
    V, H, cnt = getattr(oracle, f"{scheme}_arnoldi")(apply, g["start"], 40)
    assert np.array_equal(H, g[f"{scheme}_H"])
    assert np.array_equal(V, g[f"{scheme}_V"])
    assert cnt.reductions == g[f"{scheme}_reductions"]
    assert cnt.flops == g[f"{scheme}_flops"]
    assert cnt.napply == g[f"{scheme}_napply"]
    assert cnt.kernels["MvTransMv"] == g[f"{scheme}_mvtransmv"]
    assert cnt.kernels["MvTimesMatAddMv"] == g[f"{scheme}_mvtimes"]
    assert cnt.kernels["MvDot"] == g[f"{scheme}_mvdot"]


@pytest.mark.parametrize("scheme", ["dcgs2", "cgs2"])
def test_arnoldi_poisson100_config1(scheme):
    g = golden("arnoldi_poisson100.npz")
    apply = _csr_apply(*oracle.manteuffel_csr(100, 0.0))
    start = np.random.Generator(np.random.PCG64(1729)).standard_normal(10000)
    V, H, cnt = getattr(oracle, f"{scheme}_arnoldi")(apply, start, 50)
    assert np.array_equal(H, g[f"{scheme}_H"])
    assert np.array_equal(V[::97], g[f"{scheme}_Vsub"])
    assert cnt.reductions == g[f"{scheme}_reductions"]


@pytest.mark.parametrize("scheme", ["dcgs2", "cgs2"])
def test_arnoldi_laplace3d(scheme):
    g = golden("arnoldi_laplace3d.npz")
    V, H, _ = getattr(oracle, f"{scheme}_arnoldi")(
        lambda x: oracle.stencil7_matvec(x, (6, 5, 4)), g["start"], 30)
    assert np.array_equal(H, g[f"{scheme}_H"])
    assert np.array_equal(V, g[f"{scheme}_V"])


@pytest.mark.parametrize("scheme", ["dcgs2", "cgs2"])
def test_qr(scheme):
    g = golden("qr.npz")
    Q, R, cnt = getattr(oracle, f"{scheme}_qr")(g["A"])
    assert np.array_equal(Q, g[f"{scheme}_Q"])
    assert np.array_equal(R, g[f"{scheme}_R"])
    assert cnt.reductions == g[f"{scheme}_reductions"]
    assert cnt.flops == g[f"{scheme}_flops"]
    Q, R, _ = getattr(oracle, f"{scheme}_qr")(g["Akappa"])
    assert np.array_equal(R, g[f"kappa_{scheme}_R"])


def test_qr_hand_worked_known_answer():
    # SPEC.md:215 / tests/test_ortho.py:145-158: beta=26, c=1, alpha=5, q=[.6,.8,0]
    g = golden("qr.npz")
    assert g["hand_R"][1, 1] == 5.0
    assert np.allclose(g["hand_Q"][:, 1], [0.6, 0.8, 0.0], atol=1e-15)
    # the oracle on the same two columns (q0 = e3 from the first push of e3)
    Q, R, _ = oracle.dcgs2_qr(np.array([[0.0, 3.0, 1.0], [0.0, 4.0, 0.0], [1.0, 1.0, 0.0]]))
    assert R[1, 1] == 5.0 and np.allclose(Q[:, 1], [0.6, 0.8, 0.0], atol=1e-15)


@pytest.mark.parametrize("case,scheme", [("mant12", "dcgs2"), ("mant12", "cgs2"),
                                         ("lap8", "dcgs2"), ("lap8", "cgs2")])
def test_gmres(case, scheme):
    g = golden("gmres.npz")
    if case == "mant12":
        ptr, idx, dat = oracle.manteuffel_csr(12, 0.5)
        apply = _csr_apply(ptr, idx, dat)
        anorm = float(np.linalg.norm(dat))
        restart, rtol, iters = 10, 1e-8, 400
    else:
        dims = (8, 8, 8)
        apply = lambda x: oracle.stencil7_matvec(x, dims)  # noqa: E731
        edges = 3 * 7 * 8 * 8
        anorm = float(np.sqrt(36.0 * 512 + 2.0 * edges))
        restart, rtol, iters = 0, 0.0, 60
    res = oracle.gmres(apply, g[f"{case}_b"], anorm, iters, restart, rtol, scheme)
    p = f"{case}_{scheme}"
    assert res["iterations"] == g[f"{p}_iterations"]
    assert np.array_equal(res["residual_history"], g[f"{p}_residual_history"])
    assert np.array_equal(res["backward_errors"], g[f"{p}_backward_errors"])
    assert np.array_equal(res["reduction_history"], g[f"{p}_reduction_history"])
    assert np.array_equal(res["x"], g[f"{p}_x"])


@pytest.mark.parametrize("scheme", ["dcgs2", "cgs2"])
def test_arnoldi_config3_shape(scheme):
    """The oracle at config 3's expansion shape (laplace3d(62, 64, 64),
    m = 253,952, n = 100) against the reference's own run: H within 1e-13
    normwise (the BLAS thread count here may differ from the golden's)."""
    g = golden("arnoldi_config3_shape.npz")
    dims = (62, 64, 64)
    start = np.random.Generator(np.random.PCG64(1729)).standard_normal(int(np.prod(dims)))
    V, H, cnt = getattr(oracle, f"{scheme}_arnoldi")(
        lambda x: oracle.stencil7_matvec(x, dims), start, 100)
    ref = g[f"{scheme}_H"]
    assert np.max(np.abs(H - ref)) <= 1e-13 * np.max(np.abs(ref))
    assert cnt.reductions == g[f"{scheme}_reductions"]


@pytest.mark.parametrize("tag", ["small", "edge", "mid"])
def test_band_random_restatement_vs_reference_from_coo(tag):
    """oracle.band_random_coo through a CSR assembly equals the reference's
    CsrMatrix.from_coo (problems.py:99-117) of the same entries
    (tests/golden/band_random.npz): distinct ascending columns per row, so
    the CSR is the COO in row-major order."""
    g = golden("band_random.npz")
    m, band, d, seed = (int(v) for v in g[f"{tag}_shape"])
    r, c, v = oracle.band_random_coo(m, band, d, seed)
    indptr = np.arange(m + 1, dtype=np.int64) * d
    assert np.all(np.diff(c.reshape(m, d), axis=1) > 0)
    assert np.all(np.abs(c - r) <= band)
    if m <= 1000:
        assert np.array_equal(g[f"{tag}_indptr"], indptr)
        assert np.array_equal(g[f"{tag}_indices"], c)
        assert np.array_equal(g[f"{tag}_data"], v)
    else:
        keep = np.r_[0:7000, m * d - 7000 : m * d]
        assert np.array_equal(g[f"{tag}_indptr"], indptr[::97])
        assert np.array_equal(g[f"{tag}_indices"], c[keep])
        assert np.array_equal(g[f"{tag}_data"], v[keep])
        assert np.array_equal(g[f"{tag}_datasum"], [np.sum(v), np.sum(c)])
