"""Property-based checks of the kernels on random shapes (hypothesis): every
size regime — the small-m 64-row-block kernels, the chunked LDG / TMA
kernels and their ragged tails — against numpy (floating point, forward-error
bounds) or the oracle (integer-exact operator order, bitwise)."""

import numpy as np
import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle

pytestmark = pytest.mark.gpu

SIZES = st.one_of(st.integers(1, 300), st.integers(300, 40_000), st.integers(60_000, 140_000))


def _lib():
    from paper_2104_01253_b200 import _lib, runtime

    return _lib, runtime


def _colmajor(a):
    from paper_2104_01253_b200 import runtime

    m, k = a.shape
    ld = runtime.pad_rows(m)
    buf = torch.zeros((max(k, 1), ld), dtype=torch.float64, device="cuda")
    if k:
        buf[:k, :m] = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()
    return buf, ld


def _bound(a, b):
    return 1e-15 * max(a.shape[0], 1) * (np.abs(a).T @ np.abs(b)) + 1e-300


@settings(deadline=None, max_examples=40)
@given(m=SIZES, j=st.integers(1, 70), seed=st.integers(0, 2**31))
def test_fuzz_gram_step(m, j, seed):
    lib, rt = _lib()
    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((m, j))
    w, aw = rng.standard_normal(m), rng.standard_normal(m)
    qb, ld = _colmajor(Q)
    wd, awd = torch.from_numpy(w).cuda(), torch.from_numpy(aw).cuda()
    out = torch.empty(2 * j + 3, dtype=torch.float64, device="cuda")
    coef = torch.empty(2 * j + 2, dtype=torch.float64, device="cuda")
    ws, wsb = rt.workspace(j + 2)
    lib.call("kls_gram_dcgs2_step", qb.data_ptr(), ld, m, j, wd.data_ptr(), awd.data_ptr(),
             out.data_ptr(), coef.data_ptr(), None, 0, None, ws, wsb, rt.stream_handle())
    left = np.hstack([Q, w[:, None]])
    right = np.column_stack([w, aw])
    want = np.concatenate([(left.T @ right).T.ravel(), [aw @ aw]])
    tol = np.concatenate([_bound(left, right).T.ravel(), _bound(aw[:, None], aw[:, None]).ravel()])
    assert np.all(np.abs(out.cpu().numpy() - want) <= tol)


@settings(deadline=None, max_examples=40)
@given(m=SIZES, j=st.integers(1, 70), divide=st.integers(0, 1), seed=st.integers(0, 2**31))
def test_fuzz_update(m, j, divide, seed):
    lib, rt = _lib()
    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((m, j + 1))
    Q[:, j] = 0.0
    w, aw = rng.standard_normal(m), rng.standard_normal(m)
    c, t = rng.standard_normal(j), rng.standard_normal(j + 1)
    alpha = 0.5 + rng.random()
    qb, ld = _colmajor(Q)
    wd, awd = torch.from_numpy(w).cuda(), torch.from_numpy(aw).cuda()
    wo = torch.empty_like(wd)
    coef = torch.from_numpy(np.concatenate([c, t, [alpha]])).cuda()
    lib.call("kls_dcgs2_update_dev", qb.data_ptr(), ld, m, j, wd.data_ptr(), wo.data_ptr(),
             awd.data_ptr(), coef.data_ptr(), divide, None, rt.stream_handle())
    q = (w - Q[:, :j] @ c) / alpha
    a = aw / alpha if divide else aw
    wn = a - (Q[:, :j] @ t[:j] + q * t[j])
    scale = 1.0 + np.abs(Q[:, :j]) @ (np.abs(c) + np.abs(t[:j]))
    assert np.all(np.abs(qb[j, :m].cpu().numpy() - q) <= 1e-14 * j * scale / alpha + 1e-300)
    assert np.all(np.abs(wo.cpu().numpy() - wn) <= 1e-14 * j * (scale / alpha + scale) + 1e-300)
    assert torch.equal(wd, torch.from_numpy(w).cuda())  # w untouched (w' went to w_out)


@settings(deadline=None, max_examples=30)
@given(n=st.integers(1, 3000), density=st.floats(0.0005, 0.01), seed=st.integers(0, 2**31))
def test_fuzz_csr_operator_bitwise(n, density, seed):
    """Random sparsity (ELL copy when rows are short, warp-staged CSR when
    long): bit-identical to the reference's numpy reduceat order."""
    import paper_2104_01253_b200 as kls

    rng = np.random.default_rng(seed)
    nnz = max(1, int(density * n * n))
    rows, cols = rng.integers(0, n, nnz), rng.integers(0, n, nnz)
    csr = kls.CsrMatrix.from_coo(n, n, rows, cols, rng.standard_normal(nnz))
    x = rng.standard_normal(n)
    y = kls.CsrOperator(csr).apply(x).cpu().numpy()
    assert np.array_equal(y, oracle.csr_matvec(csr.indptr, csr.indices, csr.data, x))


@settings(deadline=None, max_examples=30)
@given(m=SIZES, k=st.integers(1, 260), host=st.integers(0, 1), seed=st.integers(0, 2**31))
def test_fuzz_project_gram(m, k, host, seed):
    if m * k > 6_000_000:
        k = max(1, 6_000_000 // m)
    lib, rt = _lib()
    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((m, k))
    v, s = rng.standard_normal(m), rng.standard_normal(k)
    qb, ld = _colmajor(Q)
    vd = torch.from_numpy(v.copy()).cuda()
    sd = torch.from_numpy(s).cuda()
    out = torch.empty(k, dtype=torch.float64, device="cuda")
    ws, wsb = rt.workspace(k + 1)
    lib.call("kls_project_gram", qb.data_ptr(), ld, m, k, vd.data_ptr(),
             s.ctypes.data if host else sd.data_ptr(), host, 0, out.data_ptr(), None, ws, wsb,
             rt.stream_handle())
    wgot = vd.cpu().numpy()
    assert np.allclose(wgot, v - Q @ s, rtol=1e-12, atol=1e-12 * np.sqrt(k))
    assert np.all(np.abs(out.cpu().numpy() - Q.T @ wgot) <= _bound(Q, wgot[:, None]).ravel())
