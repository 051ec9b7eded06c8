"""GMRES on the device against the reference's golden runs: identical
iteration counts, residual histories within 1e-8 (the reference's own
paired-curve tolerance, tests/test_gmres.py:34-41), identical cumulative
reduction histories."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def kls():
    import paper_2104_01253_b200 as k

    return k


def _op(name):
    K = kls()
    if name == "mant12":
        return K.CsrOperator(K.manteuffel_build(K.ManteuffelSpec(k=12))), 10, 1e-8, 400
    if name == "lap8":
        return K.laplace3d(8, 8, 8), 0, 0.0, 60
    return K.CsrOperator(K.manteuffel_build(K.ManteuffelSpec(k=100))), 50, 1e-6, 10000


@pytest.mark.parametrize("case,scheme", [("mant12", "dcgs2"), ("mant12", "cgs2"),
                                         ("lap8", "dcgs2"), ("lap8", "cgs2"),
                                         ("mant100", "dcgs2")])
def test_gmres_matches_reference(cuda, case, scheme):
    K = kls()
    g = golden("gmres.npz")
    op, restart, rtol, iters = _op(case)
    led = K.SyncLedger()
    res = K.gmres_solve(op, g[f"{case}_b"], K.GmresConfig(max_iters=iters, restart=restart,
                                                          rtol=rtol, scheme=scheme), ledger=led)
    p = f"{case}_{scheme}"
    assert res.iterations == g[f"{p}_iterations"]
    assert res.converged == bool(g[f"{p}_converged"])
    ref = g[f"{p}_residual_history"]
    assert res.residual_history.shape == ref.shape
    assert np.max(np.abs(res.residual_history - ref)) <= 1e-8
    assert np.array_equal(res.reduction_history, g[f"{p}_reduction_history"])
    be = g[f"{p}_backward_errors"]
    assert np.max(np.abs(res.backward_errors - be)) <= 1e-8
    x = res.x.cpu().numpy()
    xr = g[f"{p}_x"]
    if x.size != xr.size:
        x = x[::97]
    assert np.max(np.abs(x - xr)) <= 1e-6 * max(np.max(np.abs(xr)), 1.0)


def test_identity_and_zero_rhs(cuda):
    K = kls()
    op = K.DenseOperator(np.eye(9))
    b = np.arange(1.0, 10.0)
    res = K.gmres_solve(op, b, K.GmresConfig(max_iters=5))
    assert res.iterations == 1 and res.breakdown and res.converged
    assert np.allclose(res.x.cpu().numpy(), b, atol=1e-14)
    res = K.gmres_solve(op, np.zeros(9), K.GmresConfig(max_iters=5))
    assert res.iterations == 0 and res.converged


def test_backward_error_exact_solution(cuda):
    K = kls()
    op = K.laplace3d(4, 4, 4)
    x = np.random.Generator(np.random.PCG64(2)).standard_normal(op.n)
    b = op.apply(x).cpu().numpy()
    assert K.backward_error(op, x, b) <= 1e-15


def test_gmres_config2_full_size_iteration_parity(cuda):
    """BASELINE config 2 at full size (m = 1e6 convection-diffusion,
    GMRES(50), DCGS2, rtol 1e-6, 57 restart cycles): the same iteration
    count to convergence as the reference's CPU run (tests/golden/
    make_golden.py --only gmres_config2) and identical cumulative reduction
    counts.  Residual histories: through the slow phase (cycles < 42) the
    curves agree to ~1e-14; once convergence accelerates the restarted
    iteration amplifies rounding and the reference itself moves by up to
    1.1e-7 (1.7e-3 relative) under a BLAS thread-count change (one sample
    of that spread), so the whole curve must stay within 3x the reference's
    largest spread and each cycle within 1e-8 or 10x the spread in that
    cycle."""
    K = kls()
    try:
        g = golden("gmres_config2.npz")
    except FileNotFoundError:
        pytest.skip("gmres_config2.npz not generated")
    op = K.CsrOperator(K.manteuffel_build(K.ManteuffelSpec(k=1000, beta=0.5)))
    one = op.apply(np.ones(op.n)).cpu().numpy()
    b = one / np.linalg.norm(one)
    led = K.SyncLedger()
    res = K.gmres_solve(op, b, K.GmresConfig(max_iters=10000, restart=50, rtol=1e-6,
                                             scheme="dcgs2"), ledger=led)
    assert res.converged == bool(g["converged"])
    assert res.iterations == int(g["iterations"])
    ref = g["residual_history"]
    assert res.residual_history.shape == ref.shape
    assert int(g["iterations_threads8"]) == int(g["iterations"])
    spread = np.abs(g["residual_history_threads8"] - ref)
    dev = np.abs(res.residual_history - ref)
    for c0 in range(0, ref.size, 50):
        cyc = slice(c0, c0 + 50)
        assert dev[cyc].max() <= max(1e-8, 10.0 * spread[cyc].max()), c0 // 50
    assert dev.max() <= 3.0 * spread.max()
    assert dev[: 42 * 50].max() <= 1e-12
    assert np.array_equal(res.reduction_history, g["reduction_history"])
    assert led.reductions == int(g["reductions"])
