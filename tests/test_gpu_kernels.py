"""Kernel-level parity on the GPU: every libklsgpu entry point against a
numpy fp64 reference or the oracle, including odd / empty / ragged shapes.
Integer-exact operators (CSR, stencil) must be bit-identical."""

import numpy as np
import pytest
import torch

import oracle
from conftest import golden

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2104_01253_b200 import _lib, runtime

    return _lib, runtime


def _colmajor(a):
    """Device copy of a host (m, k) array as a column-major block with a
    padded leading dimension; returns (buffer (k, ld), ld)."""
    from paper_2104_01253_b200 import runtime

    m, k = a.shape
    ld = runtime.pad_rows(m)
    buf = torch.zeros((max(k, 1), ld), dtype=torch.float64, device="cuda")
    if k:
        buf[:k, :m] = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()
    return buf, ld


def _dot_tol(a, b):
    """Forward error bound scale for sums of products: eps * n * sum|a b|."""
    return 1e-15 * max(a.shape[0], 1) * (np.abs(a).T @ np.abs(b))


@pytest.mark.parametrize("m", [1, 2, 3, 63, 64, 1000, 4097, 100003])
@pytest.mark.parametrize("k", [0, 1, 3, 4, 5, 17])
def test_gram_dcgs2_matches_numpy(cuda, rng, m, k):
    lib, rt = _lib()
    Q = rng.standard_normal((m, k))
    w = rng.standard_normal(m)
    aw = rng.standard_normal(m)
    qb, ld = _colmajor(Q)
    wd = torch.from_numpy(w).cuda()
    awd = torch.from_numpy(aw).cuda()
    out = torch.full((2 * k + 3,), np.nan, dtype=torch.float64, device="cuda")
    ws, wsb = rt.workspace(k + 1)
    lib.call("kls_gram_dcgs2", qb.data_ptr(), ld, m, k, wd.data_ptr(), awd.data_ptr(),
             out.data_ptr(), None, ws, wsb, rt.stream_handle())
    got = out.cpu().numpy()
    left = np.hstack([Q, w[:, None]])
    right = np.column_stack([w, aw])
    want = np.concatenate([(left.T @ right).T.ravel(), [aw @ aw]])
    tol = np.concatenate([_dot_tol(left, right).T.ravel(), _dot_tol(aw[:, None], aw[:, None]).ravel()])
    assert np.all(np.abs(got - want) <= tol + 1e-300)
    # bitwise reproducible
    out2 = torch.empty_like(out)
    lib.call("kls_gram_dcgs2", qb.data_ptr(), ld, m, k, wd.data_ptr(), awd.data_ptr(),
             out2.data_ptr(), None, ws, wsb, rt.stream_handle())
    assert torch.equal(out, out2)


@pytest.mark.parametrize("m", [7, 4097, 100003])
@pytest.mark.parametrize("j", [1, 5, 33])
@pytest.mark.parametrize("qr", [0, 1])
def test_gram_dcgs2_step_fuses_scalars(cuda, rng, m, j, qr):
    """kls_gram_dcgs2_step == kls_gram_dcgs2 followed by kls_dcgs2_scalars."""
    if m <= j:
        pytest.skip("needs a tall basis (alpha^2 = beta - c.c > 0)")
    lib, rt = _lib()
    Q = np.linalg.qr(rng.standard_normal((m, j)))[0]
    w = rng.standard_normal(m)
    aw = rng.standard_normal(m)
    qb, ld = _colmajor(Q)
    wd, awd = torch.from_numpy(w).cuda(), torch.from_numpy(aw).cuda()
    ws, wsb = rt.workspace(j + 2)
    st = rt.stream_handle()
    g1 = torch.empty(2 * j + 3, dtype=torch.float64, device="cuda")
    c1 = torch.empty(2 * j + 2, dtype=torch.float64, device="cuda")
    lib.call("kls_gram_dcgs2", qb.data_ptr(), ld, m, j, wd.data_ptr(), awd.data_ptr(), g1.data_ptr(),
             None, ws, wsb, st)
    lib.call("kls_dcgs2_scalars", g1.data_ptr(), j, qr, c1.data_ptr(), None, st)
    g2 = torch.empty_like(g1)
    c2 = torch.empty_like(c1)
    gh = torch.full((2 * j + 3,), np.nan, dtype=torch.float64, device="cuda")
    lib.call("kls_gram_dcgs2_step", qb.data_ptr(), ld, m, j, wd.data_ptr(), awd.data_ptr(),
             g2.data_ptr(), c2.data_ptr(), gh.data_ptr(), qr, None, ws, wsb, st)
    assert torch.equal(g1, g2) and torch.equal(gh, g2)
    a, b = c1.cpu().numpy(), c2.cpu().numpy()
    assert np.allclose(a, b, rtol=1e-14, atol=0.0)
    c = g1[:j].cpu().numpy()
    alpha = np.sqrt(g1[j].item() - c @ c)
    assert b[2 * j + 1] == pytest.approx(alpha, rel=1e-13)


@pytest.mark.parametrize("k", [0, 2, 7, 1030])
def test_mv_trans_mv_generic_panels(cuda, rng, k):
    """k > 1024 exercises the multi-panel path; nx=1 with xnorm."""
    lib, rt = _lib()
    m = 3001
    Q = rng.standard_normal((m, k))
    x = rng.standard_normal(m)
    qb, ld = _colmajor(Q)
    xd = torch.from_numpy(x).cuda()
    out = torch.full((k + 1,), np.nan, dtype=torch.float64, device="cuda")
    ws, wsb = rt.workspace(k + 1)
    lib.call("kls_mv_trans_mv", qb.data_ptr() if k else None, ld, m, k, None, xd.data_ptr(), None,
             1, 1, out.data_ptr(), None, ws, wsb, rt.stream_handle())
    got = out.cpu().numpy()
    want = np.concatenate([Q.T @ x, [x @ x]])
    assert np.allclose(got, want, rtol=1e-12, atol=1e-11)


@pytest.mark.parametrize("m", [1, 5, 64, 1001, 70001])
@pytest.mark.parametrize("j", [0, 1, 4, 9])
@pytest.mark.parametrize("divide", [0, 1])
def test_dcgs2_update_matches_numpy(cuda, rng, m, j, divide):
    lib, rt = _lib()
    Q = rng.standard_normal((m, j + 1))
    Q[:, j] = 0.0
    w = rng.standard_normal(m)
    aw = rng.standard_normal(m)
    c = rng.standard_normal(j)
    t = rng.standard_normal(j + 1)
    alpha = 1.7
    qb, ld = _colmajor(Q)
    wd = torch.from_numpy(w.copy()).cuda()
    awd = torch.from_numpy(aw).cuda()
    coef = torch.from_numpy(np.concatenate([c, t])).cuda()
    lib.call("kls_dcgs2_update", qb.data_ptr(), ld, m, j, wd.data_ptr(), awd.data_ptr(),
             coef.data_ptr(), alpha, divide, None, rt.stream_handle())
    u = w - Q[:, :j] @ c
    q = u / alpha
    a = aw / alpha if divide else aw
    wn = a - (Q[:, :j] @ t[:j] + q * t[j])
    got_q = qb[j, :m].cpu().numpy()
    assert np.allclose(got_q, q, rtol=1e-13, atol=1e-13)
    assert np.allclose(wd.cpu().numpy(), wn, rtol=1e-13, atol=1e-12)
    # untouched columns stay untouched
    if j:
        assert np.array_equal(qb[:j, :m].cpu().numpy(), Q[:, :j].T)


@pytest.mark.parametrize("l", [1, 2])
@pytest.mark.parametrize("k", [0, 3, 6])
def test_mv_times_mat_add_mv_with_fused_norm(cuda, rng, l, k):
    lib, rt = _lib()
    m = 5003
    B = rng.standard_normal((m, k))
    Y = rng.standard_normal((m, l))
    S = rng.standard_normal((k, l))
    bb, ldb = _colmajor(B)
    yb, ldy = _colmajor(Y)
    sd = torch.from_numpy(np.ascontiguousarray(S.T).ravel()).cuda()
    nrm = torch.zeros(1, dtype=torch.float64, device="cuda")
    ws, wsb = rt.workspace(8)
    lib.call("kls_mv_times_mat_add_mv", yb.data_ptr(), ldy, m, l, bb.data_ptr() if k else None, ldb,
             k, sd.data_ptr() if k else None, -1.0, 0.5, nrm.data_ptr(), None, ws, wsb,
             rt.stream_handle())
    want = 0.5 * Y - B @ S
    got = yb[:l, :m].cpu().numpy().T
    assert np.allclose(got, want, rtol=1e-13, atol=1e-12)
    assert np.isclose(nrm.item(), want[:, -1] @ want[:, -1], rtol=1e-12)


@pytest.mark.parametrize("m", [1, 7, 512, 5003, 200001])
@pytest.mark.parametrize("k", [1, 3, 4, 9, 20, 40, 100, 130, 200, 256, 1500])
@pytest.mark.parametrize("host", [0, 1])
def test_project_gram_matches_numpy(cuda, rng, m, k, host):
    """CGS2's fused w = v - Q s, c = Q^T w (+ w.w): reference ortho.py:149-151."""
    if m * k > 5e7:
        pytest.skip("size")
    lib, rt = _lib()
    Q = rng.standard_normal((m, k))
    v = rng.standard_normal(m)
    s = rng.standard_normal(k)
    qb, ld = _colmajor(Q)
    vd = torch.from_numpy(v.copy()).cuda()
    out = torch.full((k + 1,), np.nan, dtype=torch.float64, device="cuda")
    ws, wsb = rt.workspace(k + 1)
    sd = torch.from_numpy(s).cuda()
    sp = s.ctypes.data if host else sd.data_ptr()
    lib.call("kls_project_gram", qb.data_ptr(), ld, m, k, vd.data_ptr(), sp, host, 1,
             out.data_ptr(), None, ws, wsb, rt.stream_handle())
    w = v - Q @ s
    got_w = vd.cpu().numpy()
    assert np.allclose(got_w, w, rtol=1e-13, atol=1e-12 * np.sqrt(k))
    got = out.cpu().numpy()
    want = np.concatenate([Q.T @ got_w, [got_w @ got_w]])
    tol = np.concatenate([_dot_tol(Q, got_w[:, None]).ravel(), [1e-15 * m * (got_w @ got_w)]])
    assert np.all(np.abs(got - want) <= tol + 1e-300)
    # deterministic
    vd2 = torch.from_numpy(v.copy()).cuda()
    out2 = torch.empty_like(out)
    lib.call("kls_project_gram", qb.data_ptr(), ld, m, k, vd2.data_ptr(), sp, host, 1,
             out2.data_ptr(), None, ws, wsb, rt.stream_handle())
    assert torch.equal(out, out2) and torch.equal(vd, vd2)


def test_csr_spmv_bitwise_ragged(cuda):
    """Rows of 0..300 nonzeros: numpy's reduceat/pairwise order, bit for bit."""
    from paper_2104_01253_b200 import CsrMatrix, CsrOperator

    g = golden("csr_ragged.npz")
    nrows = len(g["indptr"]) - 1
    n = g["x"].size
    # square-ify: pad with empty rows so the operator is n x n
    indptr = np.concatenate([g["indptr"], np.full(n - nrows, g["indptr"][-1])])
    op = CsrOperator(CsrMatrix(n, n, indptr, g["indices"], g["data"]))
    y = op.apply(g["x"]).cpu().numpy()
    assert np.array_equal(y[:nrows], g["y"])
    assert np.all(y[nrows:] == 0.0)


@pytest.mark.parametrize("k,beta", [(1, 0.5), (4, 0.5), (10, 0.5), (6, 0.0)])
def test_manteuffel_operator_bitwise(cuda, rng, k, beta):
    from paper_2104_01253_b200 import CsrOperator, ManteuffelSpec, manteuffel_build

    csr = manteuffel_build(ManteuffelSpec(k=k, beta=beta))
    ptr, idx, dat = oracle.manteuffel_csr(k, beta)
    assert np.array_equal(csr.indptr, ptr) and np.array_equal(csr.indices, idx)
    assert np.array_equal(csr.data, dat)
    x = rng.standard_normal(k * k)
    y = CsrOperator(csr).apply(x).cpu().numpy()
    assert np.array_equal(y, oracle.csr_matvec(ptr, idx, dat, x))


@pytest.mark.parametrize("dims", [(5, 4, 6), (1, 1, 1), (3, 1, 7), (8, 8, 8)])
def test_stencil_bitwise(cuda, dims):
    from paper_2104_01253_b200 import laplace3d

    g = golden("operators.npz")
    key = "x".join(map(str, dims))
    op = laplace3d(*dims)
    y = op.apply(g[f"x_{key}"]).cpu().numpy()
    assert np.array_equal(y, g[f"y_{key}"])
    assert op.frobenius_norm() == g[f"fro_{key}"]
    assert op.napply == 1


def test_stencil_large_bitwise_against_oracle(cuda, rng):
    from paper_2104_01253_b200 import laplace3d

    dims = (61, 67, 129)
    x = rng.standard_normal(int(np.prod(dims)))
    y = laplace3d(*dims).apply(x).cpu().numpy()
    assert np.array_equal(y, oracle.stencil7_matvec(x, dims))


def test_tsgemm_inplace(cuda, rng):
    lib, rt = _lib()
    m, k = 10007, 37
    V = rng.standard_normal((m, k))
    Z = rng.standard_normal((k, k))
    vb, ld = _colmajor(V)
    zd = torch.from_numpy(np.ascontiguousarray(Z.T).ravel()).cuda()  # column-major
    lib.call("kls_tsgemm_inplace", vb.data_ptr(), ld, m, k, zd.data_ptr(), rt.stream_handle())
    assert np.allclose(vb[:k, :m].cpu().numpy().T, V @ Z, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("m,k,p", [(1, 1, 1), (127, 5, 3), (130, 60, 30), (10007, 37, 37),
                                   (100_003, 60, 33), (4099, 70, 65), (777, 100, 100),
                                   (100_003, 100, 100), (1_000_003, 60, 30), (257, 64, 32),
                                   (513, 41, 17), (300_001, 44, 32)])
def test_tsgemm_inplace_cols(cuda, rng, m, k, p):
    """Krylov-Schur rotation V(:, :p) <- V(:, :k) Z(:, :p): ragged row tiles,
    column passes beyond 32, columns p..k-1 untouched; bitwise equal to the
    sequential fma order over k (the square kernel's order)."""
    lib, rt = _lib()
    V = rng.standard_normal((m, k + 1))
    Z = rng.standard_normal((k, p))
    vb, ld = _colmajor(V)
    zd = torch.from_numpy(np.ascontiguousarray(Z.T).ravel()).cuda()  # k x p column-major
    lib.call("kls_tsgemm_inplace_cols", vb.data_ptr(), ld, m, k, p, zd.data_ptr(),
             rt.stream_handle())
    got = vb[: k + 1, :m].cpu().numpy().T
    ref = V[:, :k] @ Z
    assert np.allclose(got[:, :p], ref, rtol=1e-12, atol=1e-12 * np.sqrt(k))
    assert np.array_equal(got[:, p:], V[:, p:])  # untouched columns (and the guard column k)
    vb2, _ = _colmajor(V)
    z2 = torch.from_numpy(np.ascontiguousarray(np.pad(Z, ((0, 0), (0, k - p))).T).ravel()).cuda()
    lib.call("kls_tsgemm_inplace", vb2.data_ptr(), ld, m, k, z2.data_ptr(), rt.stream_handle())
    assert torch.equal(vb2[:p, :m], vb[:p, :m])  # same fma order as the square entry point


@pytest.mark.parametrize("n,off", [(1, 0), (2, 0), (3, 1), (12345, 0), (12345, 1), (1_000_001, 0)])
def test_resid_norms_and_scale(cuda, rng, n, off):
    """128-bit path (aligned operands, odd tail) and the scalar path (an
    operand at an odd element offset)."""
    lib, rt = _lib()
    b, ax, x = (rng.standard_normal(n) for _ in range(3))
    bd, axd, xd = (torch.from_numpy(v).cuda() for v in (b, ax, x))
    if off:
        axd = torch.cat([torch.zeros(off, dtype=torch.float64, device="cuda"), axd])[off:]
    out = torch.zeros(3, dtype=torch.float64, device="cuda")
    ws, wsb = rt.workspace(4)
    lib.call("kls_resid_norms", bd.data_ptr(), axd.data_ptr(), xd.data_ptr(), n, out.data_ptr(),
             None, ws, wsb, rt.stream_handle())
    want = [np.sum((b - ax) ** 2), x @ x, b @ b]
    assert np.allclose(out.cpu().numpy(), want, rtol=1e-12)
    y = torch.empty_like(xd)
    lib.call("kls_scale", xd.data_ptr(), y.data_ptr(), n, 3.0, 0, rt.stream_handle())
    assert np.array_equal(y.cpu().numpy(), x / 3.0)


def test_errors_surface_as_exceptions(cuda):
    from paper_2104_01253_b200 import _lib

    with pytest.raises(_lib.KlsGpuError):
        _lib.call("kls_gram_dcgs2", None, 1, 10, 3, None, None, None, None, None, 0, None)


@pytest.mark.parametrize("dims", [(5, 4, 6), (1, 1, 1), (3, 1, 7), (8, 8, 8), (17, 9, 33)])
def test_device_built_laplace_csr_matches_host(cuda, rng, dims):
    from paper_2104_01253_b200 import laplace3d, laplace3d_csr_operator

    dev = laplace3d_csr_operator(*dims)
    ptr, idx, dat = oracle.laplace3d_csr(*dims)
    assert np.array_equal(dev._rowptr.cpu().numpy(), ptr)
    assert np.array_equal(dev._col.cpu().numpy()[: ptr[-1]], idx)
    assert np.array_equal(dev._val.cpu().numpy()[: ptr[-1]], dat)
    x = rng.standard_normal(int(np.prod(dims)))
    # the CSR product sums in reduceat order (not the stencil's), like the
    # reference's CsrOperator(laplace3d(...).to_csr())
    assert np.array_equal(dev.apply(x).cpu().numpy(), oracle.csr_matvec(ptr, idx, dat, x))
    assert np.allclose(dev.apply(x).cpu().numpy(), laplace3d(*dims).apply(x).cpu().numpy(),
                       rtol=1e-13, atol=1e-13)
    assert dev.frobenius_norm() == pytest.approx(float(np.linalg.norm(dat)), rel=1e-14)


@pytest.mark.parametrize("k,beta", [(1, 0.5), (2, 0.5), (7, 0.3), (10, 0.5), (31, 0.0)])
def test_device_built_manteuffel_matches_host(cuda, rng, k, beta):
    from paper_2104_01253_b200 import ManteuffelSpec, manteuffel_operator

    dev = manteuffel_operator(ManteuffelSpec(k=k, beta=beta))
    ptr, idx, dat = oracle.manteuffel_csr(k, beta)
    assert np.array_equal(dev._rowptr.cpu().numpy(), ptr)
    assert np.array_equal(dev._col.cpu().numpy()[: ptr[-1]], idx)
    assert np.array_equal(dev._val.cpu().numpy()[: ptr[-1]], dat)
    x = rng.standard_normal(k * k)
    assert np.array_equal(dev.apply(x).cpu().numpy(), oracle.csr_matvec(ptr, idx, dat, x))


@pytest.mark.parametrize("k,beta", [(37, 0.5), (100, 0.0)])
def test_ell_resid_norms_fused(cuda, rng, k, beta):
    """kls_ell_resid_norms = kls_ell_spmv + the three norms of
    kls_resid_norms (A x not stored), on device-built Manteuffel ELL."""
    import paper_2104_01253_b200 as kls
    from paper_2104_01253_b200 import problems

    lib, rt = _lib()
    op = problems.manteuffel_operator(kls.ManteuffelSpec(k=k, beta=beta))
    assert op._ell is not None
    x = torch.from_numpy(rng.standard_normal(op.n)).cuda()
    b = torch.from_numpy(rng.standard_normal(op.n)).cuda()
    y = op.apply(x).cpu().numpy()
    ecol, evals, elen, width, ld = op._ell
    out = torch.zeros(3, dtype=torch.float64, device="cuda")
    ws, wsb = rt.workspace(4)
    lib.call("kls_ell_resid_norms", ecol.data_ptr(), evals.data_ptr(), elen.data_ptr(), width,
             op.n, ld, x.data_ptr(), b.data_ptr(), out.data_ptr(), None, ws, wsb, rt.stream_handle())
    xh, bh = x.cpu().numpy(), b.cpu().numpy()
    want = [np.sum((bh - y) ** 2), xh @ xh, bh @ bh]
    assert np.allclose(out.cpu().numpy(), want, rtol=1e-12, atol=0)
    # the same rows per thread and the same segment tree as kls_resid_norms:
    # bitwise the unfused product + norms (they used to differ)
    yd = torch.from_numpy(y).cuda()
    out2 = torch.zeros(3, dtype=torch.float64, device="cuda")
    lib.call("kls_resid_norms", b.data_ptr(), yd.data_ptr(), x.data_ptr(), op.n, out2.data_ptr(),
             None, ws, wsb, rt.stream_handle())
    assert torch.equal(out, out2)


@pytest.mark.parametrize("tag", ["small", "edge", "mid"])
def test_device_built_band_random_matches_reference(cuda, rng, tag):
    """kls_build_band_csr (config 5's Arnoldi operator) is bitwise the
    reference's CsrMatrix.from_coo of the restated generator
    (tests/golden/band_random.npz), and its product is CsrMatrix.matvec's."""
    from paper_2104_01253_b200 import band_random_operator

    g = golden("band_random.npz")
    m, band, d, seed = (int(v) for v in g[f"{tag}_shape"])
    dev = band_random_operator(m, band=band, per_row=d, seed=seed)
    ptr = dev._rowptr.cpu().numpy()
    col = dev._col.cpu().numpy()[: m * d]
    val = dev._val.cpu().numpy()[: m * d]
    if m <= 1000:
        assert np.array_equal(ptr, g[f"{tag}_indptr"])
        assert np.array_equal(col, g[f"{tag}_indices"])
        assert np.array_equal(val, g[f"{tag}_data"])
    else:
        keep = np.r_[0:7000, m * d - 7000 : m * d]
        assert np.array_equal(ptr[::97], g[f"{tag}_indptr"])
        assert np.array_equal(col[keep], g[f"{tag}_indices"])
        assert np.array_equal(val[keep], g[f"{tag}_data"])
        assert np.array_equal(g[f"{tag}_datasum"], [np.sum(val), np.sum(col)])
    r, c, v = oracle.band_random_coo(m, band, d, seed)
    x = rng.standard_normal(m)
    assert np.array_equal(dev.apply(x).cpu().numpy(), oracle.csr_matvec(ptr, c, v, x))


@pytest.mark.parametrize("scheme", ["dcgs2", "cgs2"])
def test_band_random_arnoldi_vs_reference(cuda, scheme):
    """Config 5's Arnoldi variant at m = 50,000 (band 1000, 7 per row, 60
    steps) against the reference's own run: H within 1e-10 relative, the same
    reduction count, basis rows within 1e-10."""
    import paper_2104_01253_b200 as K

    g = golden("band_random.npz")
    op = K.band_random_operator(50_000, band=1000, per_row=7, seed=2525)
    start = np.random.Generator(np.random.PCG64(1729)).standard_normal(50_000)
    led = K.SyncLedger()
    V, H = K.arnoldi_expand(op, start, scheme, steps=60, ledger=led)
    ref = g[f"arnoldi_{scheme}_H"]
    assert np.max(np.abs(H - ref)) <= 1e-10 * np.max(np.abs(ref))
    assert led.reductions == int(g[f"arnoldi_{scheme}_reductions"])
    assert np.max(np.abs(V.cpu().numpy()[::997] - g[f"arnoldi_{scheme}_Vrows"])) <= 1e-10
