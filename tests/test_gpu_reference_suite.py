"""The reference's own test cases for the north-star schemes (dcgs2, cgs2),
re-run on the device path with the reference's thresholds.

Each test names the reference test it mirrors (pkg/tests/test_ortho.py,
pkg/tests/test_arnoldi.py).  Householder R factors and dense products that
the reference takes from kls.dense come from numpy here (test
infrastructure; nothing on the device path calls them).
"""

import numpy as np
import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st

pytestmark = pytest.mark.gpu

SCHEMES = ("dcgs2", "cgs2")


def kls():
    import paper_2104_01253_b200 as k

    return k


def kappa(m, n, kap, seed):
    from paper_2104_01253_b200.cli import synthetic_kappa

    return synthetic_kappa(m, n, kap, seed)


def householder_r(a):
    return np.linalg.qr(a, mode="r")


def host(t):
    return t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def mant(k, beta=0.5):
    K = kls()
    return K.CsrOperator(K.manteuffel_build(K.ManteuffelSpec(k=k, beta=beta)))


@pytest.fixture(scope="module")
def start100():
    return np.random.Generator(np.random.PCG64(77)).standard_normal(100)


# ---------------------------------------------------------------------------
# test_ortho.py


@pytest.mark.parametrize("scheme", SCHEMES)
def test_identity_input_exact(cuda, scheme):
    """test_ortho.py:18-22"""
    q, r = kls().qr_factorize(np.eye(3), scheme)
    assert np.allclose(host(q), np.eye(3), atol=1e-15)
    assert np.allclose(r, np.eye(3), atol=1e-15)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_against_householder_oracle(cuda, rng, scheme):
    """test_ortho.py:25-33 (and test_dcgs2_final_qr_matches_householder, :196-200)"""
    K = kls()
    a = rng.standard_normal((100, 10))
    q, r = K.qr_factorize(a, scheme)
    rh = householder_r(a)
    assert np.max(np.abs(np.abs(r) - np.abs(rh))) <= 1e-10 * np.max(np.abs(rh))
    assert K.loss_of_orthogonality(q) <= 1e-13
    assert np.all(np.diag(r) >= 0)
    assert np.allclose(np.tril(r, -1), 0.0)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_duplicate_column_breaks_down(cuda, rng, scheme):
    """test_ortho.py:36-46"""
    K = kls()
    a1 = rng.standard_normal(40)
    state = K.make_state(scheme, 40, 4)
    state.push(a1)
    with pytest.raises(K.BreakdownError):
        state.push(a1.copy())
        state.push(rng.standard_normal(40))
        state.finalize()


@pytest.mark.parametrize("scheme", SCHEMES)
def test_reduction_count_per_column(cuda, rng, scheme):
    """test_ortho.py:49-63"""
    K = kls()
    m, n = 60, 8
    state = K.make_state(scheme, m, n)
    counts = []
    for _ in range(n):
        before = state.ledger.reductions
        state.push(rng.standard_normal(m))
        counts.append(state.ledger.reductions - before)
    if scheme in K.DELAYED_SCHEMES:
        assert counts[0] == 0
        assert counts[1:] == [K.per_iteration_synchs(scheme, j) for j in range(2, n + 1)]
    else:
        assert counts == [K.per_iteration_synchs(scheme, j) for j in range(1, n + 1)]


@pytest.mark.parametrize("scheme", SCHEMES)
def test_totals_match_prediction(cuda, rng, scheme):
    """test_ortho.py:66-72"""
    K = kls()
    for n in (5, 17, 50, 100):
        a = rng.standard_normal((120, n))
        led = K.SyncLedger()
        K.qr_factorize(a, scheme, ledger=led)
        assert K.assert_matches(led, K.predicted_counts(scheme, n)).passed


@pytest.mark.parametrize("scheme", SCHEMES)
def test_representation_error_machine_level(cuda, scheme):
    """test_ortho.py:75-79"""
    K = kls()
    a = kappa(120, 25, 1e8, seed=4)
    q, r = K.qr_factorize(a, scheme)
    assert K.representation_error_qr(a, q, r) <= 1e-13


def test_capacity_and_shape_errors(cuda, rng):
    """test_ortho.py:87-97, for the device schemes"""
    K = kls()
    for scheme in SCHEMES:
        state = K.make_state(scheme, 10, 1)
        state.push(rng.standard_normal(10))
        with pytest.raises(K.DimensionError):
            state.push(rng.standard_normal(10))
            state.finalize()
        with pytest.raises(K.DimensionError):
            K.make_state(scheme, 10, 2).push(rng.standard_normal(11))
        with pytest.raises(ValueError):
            s = K.make_state(scheme, 3, 2)
            s.push(np.array([1.0, np.nan, 0.0]))
            s.finalize()
    with pytest.raises(K.UnknownSchemeError):
        K.make_state("qrx", 10, 2)


def test_cgs2_correction_zero_on_orthogonal_input(cuda):
    """test_ortho.py:103-110"""
    state = kls().make_state("cgs2", 3, 3)
    for j in range(3):
        e = np.zeros(3)
        e[j] = 2.0
        state.push(e)
    _, r = state.finalize()
    assert np.allclose(r, 2.0 * np.eye(3))


def test_dcgs2_orthogonal_input(cuda):
    """test_ortho.py:161-168 (against cgs2 here: single-pass cgs is not a
    device scheme)"""
    K = kls()
    q0, _ = np.linalg.qr(np.random.Generator(np.random.PCG64(3)).standard_normal((40, 6)))
    a = 3.0 * q0
    q1, r1 = K.qr_factorize(a, "dcgs2")
    q2, r2 = K.qr_factorize(a, "cgs2")
    assert np.max(np.abs(host(q1) - host(q2))) <= 1e-13
    assert np.max(np.abs(r1 - r2)) <= 1e-13 * np.max(np.abs(r1))
    assert np.allclose(np.abs(r1), 3.0 * np.eye(6), atol=1e-13)


def test_dcgs2_agrees_with_cgs2_moderate_kappa(cuda):
    """test_ortho.py:171-176"""
    K = kls()
    a = kappa(100, 10, 1e4, seed=17)
    q1, r1 = K.qr_factorize(a, "cgs2")
    q2, r2 = K.qr_factorize(a, "dcgs2")
    assert np.max(np.abs(r1 - r2)) <= 1e-10 * np.max(np.abs(r1))
    assert np.max(np.abs(host(q1) - host(q2))) <= 1e-10


def test_dcgs2_single_column(cuda):
    """test_ortho.py:179-185"""
    state = kls().make_state("dcgs2", 5, 1)
    v = np.arange(1.0, 6.0)
    state.push(v)
    q, r = state.finalize()
    assert np.allclose(host(q)[:, 0], v / np.linalg.norm(v))
    assert r[0, 0] == pytest.approx(np.linalg.norm(v))


def test_dcgs2_total_reductions(cuda, rng):
    """test_ortho.py:188-193"""
    K = kls()
    for n in (1, 2, 10, 30):
        a = rng.standard_normal((60, n))
        led = K.SyncLedger()
        K.qr_factorize(a, "dcgs2", ledger=led)
        assert n <= led.reductions <= n + 2


def test_dcgs2_pending_invariant(cuda, rng):
    """test_ortho.py:203-208"""
    state = kls().make_state("dcgs2", 20, 5)
    state.push(rng.standard_normal(20))
    assert state.npushed == 1 and state.ncols == 0 and state._w is not None
    state.push(rng.standard_normal(20))
    assert state.npushed == 2 and state.ncols == 1 and state._w is not None


@pytest.fixture(scope="module")
def kappa_sweep(cuda):
    """test_ortho.py:222-236 for the device schemes"""
    K = kls()
    m, n = 200, 50
    kappas = np.array([10.0**e for e in range(0, 15)])
    out = {}
    for scheme in SCHEMES:
        loos, rres = [], []
        for kap in kappas:
            a = kappa(m, n, kap, seed=1234)
            q, r = K.qr_factorize(a, scheme)
            loos.append(K.loss_of_orthogonality(q))
            rres.append(K.representation_error_qr(a, q, r))
        out[scheme] = (np.array(loos), np.array(rres))
    return kappas, out


def test_loo_stays_at_eps_level(kappa_sweep):
    """test_ortho.py:249-259: cgs2 and dcgs2 stay O(eps) across kappa 1..1e14"""
    kappas, data = kappa_sweep
    eps_level = 100 * 50 * np.finfo(float).eps
    for i in range(len(kappas)):
        assert data["cgs2"][0][i] <= eps_level
        assert data["dcgs2"][0][i] <= eps_level


def test_dcgs2_health_at_high_kappa(kappa_sweep):
    """test_ortho.py:268-276 (the dcgs2 half)"""
    kappas, data = kappa_sweep
    sel = (kappas >= 1e9) & (kappas <= 1e12)
    assert np.all(data["dcgs2"][0][sel] <= 1e-7)
    assert np.all(data["dcgs2"][1][sel] <= 1e-7)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_r_matches_oracle_at_kappa_1e6(cuda, scheme):
    """test_ortho.py:294-299"""
    a = kappa(150, 25, 1e6, seed=41)
    _, r = kls().qr_factorize(a, scheme)
    rh = householder_r(a)
    assert np.max(np.abs(np.abs(r) - np.abs(rh))) <= 1e-8 * np.max(np.abs(rh))


@settings(deadline=None, max_examples=15)
@given(
    n=st.integers(min_value=1, max_value=20),
    extra=st.integers(min_value=0, max_value=60),
    seed=st.integers(min_value=0, max_value=2**31),
    scheme=st.sampled_from(SCHEMES),
)
def test_scheme_property_well_conditioned(n, extra, seed, scheme):
    """test_ortho.py:305-320"""
    K = kls()
    m = n + extra
    a = np.random.Generator(np.random.PCG64(seed)).standard_normal((m, n))
    led = K.SyncLedger()
    q, r = K.qr_factorize(a, scheme, ledger=led)
    assert K.loss_of_orthogonality(q) <= 1e-12 * max(n, 1)
    assert K.representation_error_qr(a, q, r) <= 1e-13
    assert np.all(np.diag(r) >= 0)
    assert K.assert_matches(led, K.predicted_counts(scheme, n)).passed


# ---------------------------------------------------------------------------
# test_arnoldi.py


@pytest.mark.parametrize("scheme", SCHEMES)
def test_rre_invariant_on_manteuffel(cuda, scheme, start100):
    """test_arnoldi.py:29-35 and test_loo_machine_level_for_reorthogonalized, :38-41"""
    K = kls()
    op = mant(10)
    v, h = K.arnoldi_expand(op, start100, scheme, steps=40)
    assert v.shape == (100, 41) and h.shape == (41, 40)
    assert K.representation_error_arnoldi(op, v, h) <= 1e-12
    assert not np.any(np.tril(h, -2))
    assert np.all(np.diag(h, -1) >= 0)
    assert K.loss_of_orthogonality(v) <= 1e-13


def test_random_operator_rre(cuda, rng):
    """test_arnoldi.py:44-50"""
    K = kls()
    op = K.DenseOperator(rng.standard_normal((50, 50)))
    v, h = K.arnoldi_expand(op, rng.standard_normal(50), "dcgs2", steps=10)
    assert K.representation_error_arnoldi(op, v, h) <= 1e-12
    v, h = K.arnoldi_expand(op, rng.standard_normal(50), "cgs2", steps=5)
    assert K.representation_error_arnoldi(op, v, h) <= 1e-13
    assert K.loss_of_orthogonality(v) <= 1e-14


def test_h_agreement_dcgs2_vs_cgs2(cuda, start100):
    """test_arnoldi.py:53-57"""
    K = kls()
    op = mant(10)
    _, h1 = K.arnoldi_expand(op, start100, "cgs2", steps=10)
    _, h2 = K.arnoldi_expand(op, start100, "dcgs2", steps=10)
    assert np.max(np.abs(h1 - h2)) <= 1e-9 * np.linalg.norm(op.to_dense())


@pytest.mark.parametrize("scheme", SCHEMES)
def test_eigenvector_start_immediate_breakdown(cuda, scheme):
    """test_arnoldi.py:105-112 (cgs2 there).  The reference's dcgs2 finalizes
    the start column in its first step and sees the vanished direction one
    step later (True, then False), reaching the same final state."""
    K = kls()
    exp = K.arnoldi(K.DenseOperator(np.diag([1.0, 2.0, 3.0])), np.array([1.0, 0.0, 0.0]), scheme,
                    capacity=4)
    if scheme == "dcgs2":
        assert exp.step() is True and not exp.happy
    assert exp.step() is False
    v, h = exp.finalize()
    assert exp.happy
    assert h.shape == (1, 1) and h[0, 0] == pytest.approx(1.0)
    assert np.allclose(host(v)[:, 0], [1.0, 0.0, 0.0])


@pytest.mark.parametrize("scheme", SCHEMES)
def test_resume_keeps_expansion_valid(cuda, scheme, start100):
    """test_arnoldi.py:128-137"""
    K = kls()
    op = mant(10)
    v0, h0 = K.arnoldi_expand(op, start100, "cgs2", steps=10)
    v0 = host(v0)
    exp = K.resume_arnoldi(op, v0, h0, scheme, capacity=30)
    while exp.order < 25:
        exp.step()
    v, h = exp.finalize()
    assert v.shape == (100, 26) and h.shape == (26, 25)
    assert K.representation_error_arnoldi(op, v, h) <= 1e-12
    assert np.allclose(h[:11, :10], h0, atol=1e-14)


def test_arnoldi_flop_overhead_is_quadratic(cuda, start100):
    """test_arnoldi.py:171-186"""
    K = kls()
    op = mant(10)
    n = 40
    led_a = K.SyncLedger()
    K.arnoldi_expand(op, start100, "dcgs2", steps=n, ledger=led_a)
    led_q = K.SyncLedger()
    a = np.column_stack([start100] + [np.random.Generator(np.random.PCG64(j)).standard_normal(100)
                                      for j in range(n - 1)])
    K.qr_factorize(a, "dcgs2", ledger=led_q)
    diff = led_a.flops - led_q.flops
    cubic = sum(2 * (j + 1) * j for j in range(1, n + 1))
    assert 0.5 * cubic <= diff <= 2.0 * cubic + 4 * n * 100


def test_manteuffel50_long_run_curves(cuda):
    """test_arnoldi.py:195-208 (the cgs2 / dcgs2 bounds): 300 steps"""
    K = kls()
    op = mant(50)
    start = np.random.Generator(np.random.PCG64(5)).standard_normal(op.n)
    for scheme in SCHEMES:
        v, h = K.arnoldi_expand(op, start, scheme, steps=300)
        assert K.loss_of_orthogonality(v) <= 1e-12
        assert K.representation_error_arnoldi(op, v, h) <= 1e-13


# ---------------------------------------------------------------------------
# test_gmres.py


def _xh(res):
    return host(res.x)


def test_gmres_laplace_slab_matches_direct_solve(cuda):
    """test_gmres.py:23-31"""
    K = kls()
    op = K.laplace3d(32, 32, 1)
    a = op.to_dense()
    b = np.ones(op.n)
    x_direct = np.linalg.solve(a, b)
    res = K.gmres_solve(op, b, K.GmresConfig(max_iters=100, scheme="cgs2"))
    x = _xh(res)
    assert np.linalg.norm(b - a @ x) / np.linalg.norm(b) <= 1e-10
    assert np.linalg.norm(x - x_direct) <= 1e-8 * np.linalg.norm(x_direct)


def test_gmres_paired_residual_curves_cgs2_vs_dcgs2(cuda):
    """test_gmres.py:34-41"""
    K = kls()
    op = K.laplace3d(32, 32, 1)
    b = np.ones(op.n)
    r1 = K.gmres_solve(op, b, K.GmresConfig(max_iters=100, scheme="cgs2"))
    r2 = K.gmres_solve(op, b, K.GmresConfig(max_iters=100, scheme="dcgs2"))
    n = min(len(r1.residual_history), len(r2.residual_history))
    assert n == 100
    assert np.max(np.abs(r1.residual_history[:n] - r2.residual_history[:n])) <= 1e-8


@pytest.mark.parametrize("scheme", SCHEMES)
def test_gmres_residual_history_monotone(cuda, scheme):
    """test_gmres.py:44-50"""
    K = kls()
    op = K.laplace3d(8, 8, 8)
    b = op.apply(np.ones(op.n))
    res = K.gmres_solve(op, b, K.GmresConfig(max_iters=60, scheme=scheme))
    assert np.all(np.diff(res.residual_history) <= 1e-14)


def test_gmres_reduction_rates_one_vs_three(cuda):
    """test_gmres.py:53-61"""
    K = kls()
    op = K.laplace3d(10, 10, 10)
    b = op.apply(np.ones(op.n))
    led2 = K.SyncLedger()
    K.gmres_solve(op, b, K.GmresConfig(max_iters=50, scheme="cgs2"), ledger=led2)
    ledd = K.SyncLedger()
    K.gmres_solve(op, b, K.GmresConfig(max_iters=50, scheme="dcgs2"), ledger=ledd)
    assert led2.reductions == 3 * 50
    assert ledd.reductions <= 50 + 2


def test_gmres_reduction_history_cumulative(cuda):
    """test_gmres.py:64-71"""
    K = kls()
    op = K.laplace3d(6, 6, 6)
    b = op.apply(np.ones(op.n))
    led = K.SyncLedger()
    res = K.gmres_solve(op, b, K.GmresConfig(max_iters=20, scheme="dcgs2"), ledger=led)
    assert len(res.reduction_history) == len(res.residual_history)
    assert np.all(np.diff(res.reduction_history) >= 0)
    assert res.reduction_history[-1] <= led.reductions


@pytest.mark.parametrize("scheme", SCHEMES)
def test_gmres_restarted_converges(cuda, scheme):
    """test_gmres.py:74-80"""
    K = kls()
    op = K.laplace3d(10, 10, 1)
    b = np.ones(op.n)
    a = op.to_dense()
    res = K.gmres_solve(op, b, K.GmresConfig(max_iters=200, restart=25, rtol=1e-10, scheme=scheme))
    assert np.linalg.norm(b - a @ _xh(res)) / np.linalg.norm(b) <= 1e-9
    assert res.converged


def test_gmres_rtol_early_stop(cuda):
    """test_gmres.py:83-89"""
    K = kls()
    op = K.laplace3d(8, 8, 1)
    res = K.gmres_solve(op, np.ones(op.n), K.GmresConfig(max_iters=64, rtol=1e-6))
    assert res.converged and res.iterations < 64
    assert res.residual_history[-1] <= 1e-6


@pytest.mark.parametrize("scheme", SCHEMES)
def test_gmres_stagnation_flag_on_shift_operator(cuda, scheme):
    """test_gmres.py:92-103"""
    K = kls()
    n = 40
    a = np.zeros((n, n))
    a[0, n - 1] = 1.0
    a[np.arange(1, n), np.arange(0, n - 1)] = 1.0
    b = np.zeros(n)
    b[0] = 1.0
    res = K.gmres_solve(K.DenseOperator(a), b, K.GmresConfig(max_iters=30, scheme=scheme))
    assert res.stagnated
    assert res.residual_history[-1] == pytest.approx(1.0, abs=1e-12)


def test_gmres_zero_rhs(cuda):
    """test_gmres.py:106-109"""
    K = kls()
    op = K.laplace3d(3, 3, 3)
    res = K.gmres_solve(op, np.zeros(op.n), K.GmresConfig(max_iters=5))
    assert res.converged and np.all(_xh(res) == 0.0)


def test_backward_error_cases(cuda, rng):
    """test_gmres.py:116-133"""
    K = kls()
    op = K.laplace3d(6, 6, 1)
    x = np.ones(op.n)
    assert K.backward_error(op, x, op.apply(x)) <= 1e-15
    op = K.laplace3d(4, 4, 1)
    assert K.backward_error(op, np.zeros(op.n), np.ones(op.n)) == pytest.approx(1.0)
    a = rng.standard_normal((12, 12))
    x = rng.standard_normal(12)
    assert K.backward_error(a, x, a @ x) <= 1e-15


def test_matrix_free_frobenius_probe_used(cuda):
    """test_gmres.py:146-154"""
    K = kls()
    op = K.laplace3d(12, 12, 12)
    x = np.ones(op.n)
    b = host(op.apply(x))
    be = K.backward_error(op, x + 1e-3, b)
    exact_fro = np.sqrt(36.0 * op.n + 2.0 * (3 * 11 * 12 * 12))
    ref = np.linalg.norm(b - host(op.apply(x + 1e-3))) / (
        exact_fro * np.linalg.norm(x + 1e-3) + np.linalg.norm(b))
    assert be == pytest.approx(ref, rel=1e-10)


# ---------------------------------------------------------------------------
# test_kernels.py (device operands: CUDA tensors, column-major blocks)


def _dev(a):
    a = np.asarray(a, dtype=np.float64)
    t = torch.from_numpy(np.ascontiguousarray(a.T if a.ndim == 2 else a)).cuda()
    return t.T if a.ndim == 2 else t


def test_kernel_dot_cases(cuda, rng):
    """test_kernels.py:11-55"""
    from paper_2104_01253_b200 import kernels, ledger as L

    assert kernels.dot(_dev([1.0, 2.0, 3.0]), _dev([4.0, 5.0, 6.0])) == 32.0
    q = rng.standard_normal(50)
    q /= np.linalg.norm(q)
    assert abs(kernels.dot(_dev(q), _dev(q)) - 1.0) <= 1e-15
    x, y = rng.standard_normal(1000), rng.standard_normal(1000)
    acc = 0.0
    for a, b in zip(x, y):
        acc += a * b
    d = kernels.dot(_dev(x), _dev(y))
    assert d == pytest.approx(acc, rel=1e-15, abs=1e-15)
    assert d == kernels.dot(_dev(x.copy()), _dev(y.copy()))  # bitwise deterministic
    led = L.SyncLedger()
    kernels.dot(_dev(np.ones(8)), _dev(np.ones(8)), ledger=led)
    assert led.reductions == 1 and led.kernel_counts[L.MV_DOT] == 1 and led.flops == 16
    with pytest.raises(kls().DimensionError):
        kernels.dot(_dev(np.ones(3)), _dev(np.ones(4)))
    assert kernels.norm2(_dev([3.0, 4.0])) == 5.0
    assert kernels.norm2(_dev(np.zeros(10))) == 0.0
    x = rng.standard_normal(300)
    led = L.SyncLedger()
    assert kernels.norm2(_dev(x), ledger=led) == pytest.approx(
        np.sqrt(kernels.dot(_dev(x), _dev(x))), rel=1e-15)
    assert led.reductions == 1


def test_kernel_mv_trans_mv_cases(cuda, rng):
    """test_kernels.py:58-103"""
    from paper_2104_01253_b200 import kernels, ledger as L

    x = np.array([[1.0], [2.0], [3.0]])
    assert np.array_equal(kernels.mv_trans_mv(_dev(np.eye(3)), _dev(x)), x)
    q, _ = np.linalg.qr(np.random.Generator(np.random.PCG64(5)).standard_normal((40, 6)))
    assert np.linalg.norm(kernels.mv_trans_mv(_dev(q), _dev(q)) - np.eye(6)) <= 1e-14
    b = rng.standard_normal((50, 5))
    xx = rng.standard_normal((50, 2))
    got = kernels.mv_trans_mv(_dev(b), _dev(xx))
    for i in range(5):
        for j in range(2):
            assert got[i, j] == pytest.approx(float(np.dot(b[:, i], xx[:, j])), rel=1e-14, abs=1e-14)
    b = rng.standard_normal((30, 4))
    for width in (1, 2, 7):
        led = L.SyncLedger()
        kernels.mv_trans_mv(_dev(b), _dev(rng.standard_normal((30, width))), ledger=led)
        assert led.reductions == 1 and led.kernel_counts[L.MV_TRANS_MV] == 1
    led = L.SyncLedger()
    out = kernels.mv_trans_mv(_dev(np.zeros((10, 0))), _dev(np.ones((10, 1))), ledger=led)
    assert out.shape == (0, 1) and led.reductions == 1 and led.flops == 0
    with pytest.raises(kls().DimensionError):
        kernels.mv_trans_mv(_dev(np.ones((5, 2))), _dev(np.ones((6, 2))))


def test_kernel_mv_times_mat_add_mv_cases(cuda, rng):
    """test_kernels.py:106-158"""
    from paper_2104_01253_b200 import kernels, ledger as L

    y = _dev(np.array([[1.0], [1.0]]))
    out = kernels.mv_times_mat_add_mv(y, _dev(np.eye(2)), np.array([[1.0], [1.0]]), sign=-1.0)
    assert out is y and np.array_equal(host(out), np.zeros((2, 1)))
    y0 = rng.standard_normal((7, 1))
    y = _dev(y0)
    kernels.mv_times_mat_add_mv(y, _dev(rng.standard_normal((7, 3))), np.zeros((3, 1)))
    assert np.array_equal(host(y), y0)
    y0 = rng.standard_normal((100, 2))
    b = rng.standard_normal((100, 8))
    s = rng.standard_normal((8, 2))
    expected = y0.copy()
    for i in range(100):
        for j in range(2):
            acc = 0.0
            for k in range(8):
                acc += b[i, k] * s[k, j]
            expected[i, j] -= acc
    got = kernels.mv_times_mat_add_mv(_dev(y0), _dev(b), s, sign=-1.0)
    assert np.allclose(host(got), expected, rtol=1e-14, atol=1e-14)
    led = L.SyncLedger()
    kernels.mv_times_mat_add_mv(_dev(rng.standard_normal((20, 1))), _dev(rng.standard_normal((20, 3))),
                                rng.standard_normal((3, 1)), ledger=led)
    assert led.reductions == 0 and led.kernel_counts[L.MV_TIMES_MAT_ADD_MV] == 1
    assert led.flops == 2 * 20 * 3
    y = _dev(np.full((3, 1), 2.0))
    kernels.mv_times_mat_add_mv(y, _dev(np.zeros((3, 0))), np.zeros((0, 1)), scale=0.5)
    assert np.array_equal(host(y), np.ones((3, 1)))
    with pytest.raises(kls().DimensionError):
        kernels.mv_times_mat_add_mv(_dev(np.ones((5, 1))), _dev(np.ones((5, 2))), np.ones((3, 1)))


@settings(deadline=None, max_examples=25)
@given(
    m=st.integers(min_value=1, max_value=60),
    k=st.integers(min_value=0, max_value=8),
    l=st.integers(min_value=1, max_value=4),
    seed=st.integers(min_value=0, max_value=2**31),
)
def test_kernels_deterministic_and_consistent(m, k, l, seed):
    """test_kernels.py:160-172"""
    from paper_2104_01253_b200 import kernels

    gen = np.random.Generator(np.random.PCG64(seed))
    b = gen.standard_normal((m, k))
    x = gen.standard_normal((m, l))
    g1 = kernels.mv_trans_mv(_dev(b), _dev(x))
    g2 = kernels.mv_trans_mv(_dev(b.copy()), _dev(x.copy()))
    assert np.array_equal(g1, g2)
    assert np.allclose(g1, b.T @ x, rtol=1e-13, atol=1e-13)


# ---------------------------------------------------------------------------
# test_eig.py (the Krylov-Schur cases not already in test_gpu_eig.py)


def test_ritz_residual_matches_explicit_residual(cuda, rng):
    """test_eig.py:49-62"""
    K = kls()
    from paper_2104_01253_b200.schur import hessenberg_real_schur, schur_eigenvectors

    op = K.DenseOperator(rng.standard_normal((40, 40)))
    v, h = K.arnoldi_expand(op, rng.standard_normal(40), "cgs2", steps=15)
    v = host(v)
    k = h.shape[1]
    form = hessenberg_real_schur(np.triu(h[:k, :k], -1))
    vals, vecs = schur_eigenvectors(form)
    a = op.to_dense()
    for i in range(len(vals)):
        y = vecs[:, i]
        z = v[:, :k] @ y
        explicit = np.linalg.norm(a @ z - vals[i] * z)
        assert K.ritz_residual(h, y) == pytest.approx(explicit, rel=1e-6, abs=1e-8)


def test_ks_invariant_dim_monotone_across_restarts(cuda):
    """test_eig.py:140-148"""
    K = kls()
    op = mant(7)
    cfg = K.KrylovSchurConfig(max_basis=20, tol=1e-7, scheme="cgs2", max_restarts=15)
    res = K.krylov_schur_run(op, cfg, seed=5)
    assert all(b >= a for a, b in zip(res.lock_history, res.lock_history[1:]))
    assert res.lock_history[-1] == res.invariant_dim


@pytest.mark.parametrize("scheme", SCHEMES)
def test_ks_restart_budget_flags_incomplete(cuda, scheme):
    """test_eig.py:151-161"""
    K = kls()
    op = mant(10)
    res = K.krylov_schur_run(op, K.KrylovSchurConfig(max_basis=20, tol=1e-7, scheme=scheme,
                                                     max_restarts=2), seed=5)
    assert res.incomplete and res.invariant_dim < 20
    res2 = K.krylov_schur_run(op, K.KrylovSchurConfig(max_basis=20, tol=1e-7, scheme=scheme,
                                                      max_restarts=30), seed=5)
    assert res2.invariant_dim > res.invariant_dim


def test_ks_config_validation():
    """test_eig.py:184-191"""
    K = kls()
    with pytest.raises(ValueError):
        K.KrylovSchurConfig(max_basis=5, keep=5)
    with pytest.raises(ValueError):
        K.KrylovSchurConfig(max_basis=5, tol=0.0)
    assert K.KrylovSchurConfig(max_basis=10).keep == 5


# ---------------------------------------------------------------------------
# test_acceptance.py (criteria on the north-star schemes; SEED = 7)

ACC_SEED = 7


def test_acceptance_01_sync_count_exactness(cuda):
    """test_acceptance.py:48-69 (cgs2: 150, dcgs2: 50..52 on 5000 x 50)"""
    K = kls()
    a = np.random.Generator(np.random.PCG64(ACC_SEED)).standard_normal((5000, 50))
    for scheme, (lo, hi) in {"cgs2": (150, 150), "dcgs2": (50, 52)}.items():
        led = K.SyncLedger()
        K.qr_factorize(a, scheme, ledger=led)
        assert lo <= led.reductions <= hi


def test_acceptance_02_loo_ceiling(cuda):
    """test_acceptance.py:72-99: max LOO over kappa 1e0..1e12 <= 100 eps n"""
    K = kls()
    worst = 0.0
    for scheme in SCHEMES:
        for e in range(0, 13):
            a = kappa(200, 50, 10.0**e, seed=ACC_SEED)
            q, _ = K.qr_factorize(a, scheme)
            worst = max(worst, K.loss_of_orthogonality(q))
    assert worst <= 100 * np.finfo(float).eps * 50


def test_acceptance_07_krylov_schur_correctness(cuda):
    """test_acceptance.py:174-191"""
    K = kls()
    spec = K.ManteuffelSpec(k=10)
    op = K.CsrOperator(K.manteuffel_build(spec))
    table = K.manteuffel_eigenvalues(spec)
    cfg = K.KrylovSchurConfig(max_basis=100, tol=1e-7, scheme="cgs2")
    res = K.krylov_schur_run(op, cfg, seed=ACC_SEED, exact=table)
    rep = K.match_eigenvalues(res.values.real, table, cfg.tol)
    assert rep.n_matched == len(res.values)
    assert not res.over_multiplicity and not rep.over_multiplicity


def test_acceptance_08_arnoldi_equivalence(cuda):
    """test_acceptance.py:194-211"""
    K = kls()
    op = mant(20)
    start = np.random.Generator(np.random.PCG64(ACC_SEED)).standard_normal(op.n)
    v1, h1 = K.arnoldi_expand(op, start, "cgs2", steps=50)
    rre1 = K.representation_error_arnoldi(op, v1, h1)
    v2, h2 = K.arnoldi_expand(op, start, "dcgs2", steps=50)
    rre2 = K.representation_error_arnoldi(op, v2, h2)
    afro = np.linalg.norm(op.to_dense())
    assert np.max(np.abs(h1 - h2)) <= 1e-8 * afro
    assert rre1 <= 1e-12 and rre2 <= 1e-12


def test_acceptance_09_gmres_reduction_proxy(cuda):
    """test_acceptance.py:214-236: 24^3 Laplace, 100 iterations"""
    K = kls()
    op = K.laplace3d(24, 24, 24)
    b = host(op.apply(np.ones(op.n)))
    b /= np.linalg.norm(b)
    led2 = K.SyncLedger()
    r2 = K.gmres_solve(op, b, K.GmresConfig(max_iters=100, scheme="cgs2"), ledger=led2)
    ledd = K.SyncLedger()
    rd = K.gmres_solve(op, b, K.GmresConfig(max_iters=100, scheme="dcgs2"), ledger=ledd)
    n = min(len(r2.residual_history), len(rd.residual_history))
    assert n == 100
    assert np.max(np.abs(r2.residual_history[:n] - rd.residual_history[:n])) <= 1e-8
    assert ledd.reductions <= 102 and led2.reductions == 300


def test_acceptance_10_eigen_count_agreement(cuda):
    """test_acceptance.py:239-260 (the cgs2 / dcgs2 half: counts within 2)"""
    K = kls()
    spec = K.ManteuffelSpec(k=10)
    csr = K.manteuffel_build(spec)
    table = K.manteuffel_eigenvalues(spec)
    for restart in (25, 50, 75):
        counts = {}
        for scheme in SCHEMES:
            cfg = K.KrylovSchurConfig(max_basis=restart, tol=1e-7, scheme=scheme, max_restarts=250)
            res = K.krylov_schur_run(K.CsrOperator(csr), cfg, seed=ACC_SEED, exact=table)
            counts[scheme] = K.match_eigenvalues(res.values.real, table, 1e-7).n_matched
        assert abs(counts["cgs2"] - counts["dcgs2"]) <= 2, (restart, counts)


# ---------------------------------------------------------------------------
# test_problems.py (device products)


def test_csr_matvec_matches_dense(cuda, rng):
    """test_problems.py:47-57: CsrMatrix.matvec, now a device product"""
    K = kls()
    csr = K.CsrMatrix.from_coo(4, 4, [0, 1, 1, 3], [1, 0, 3, 2], [1.5, -2.0, 0.5, 4.0])
    x = rng.standard_normal(4)
    assert np.allclose(csr.matvec(x), csr.to_dense() @ x, atol=1e-15)
    csr = K.CsrMatrix.from_coo(3, 3, [2], [0], [7.0])
    assert csr.matvec(np.array([1.0, 2.0, 3.0])).tolist() == [0.0, 0.0, 7.0]
    rect = K.CsrMatrix.from_coo(3, 5, [0, 2, 2], [4, 1, 3], [1.0, 2.0, 3.0])
    x = rng.standard_normal(5)
    assert np.allclose(rect.matvec(x), rect.to_dense() @ x, atol=1e-15)


def test_laplace_stencil_cases(cuda, rng):
    """test_problems.py:134-185"""
    K = kls()
    assert host(K.laplace3d(1, 1, 1).apply(np.array([1.0])))[0] == pytest.approx(6.0)
    op = K.laplace3d(4, 4, 4)
    a = op.to_csr()
    for x in (np.ones(op.n), rng.standard_normal(op.n)):
        assert np.allclose(host(op.apply(x)), a.matvec(x), atol=1e-13)
    op = K.laplace3d(3, 4, 5)
    for _ in range(3):
        x, y = rng.standard_normal(op.n), rng.standard_normal(op.n)
        assert abs(host(op.apply(x)) @ y - x @ host(op.apply(y))) <= 1e-13 * (
            np.linalg.norm(x) * np.linalg.norm(y))
    op = K.laplace3d(5, 4, 3)
    assert op.frobenius_norm() == pytest.approx(np.linalg.norm(op.to_csr().to_dense()), rel=1e-14)
    op = K.laplace3d(6, 6, 6)
    exact = np.linalg.norm(op.to_csr().to_dense())
    assert K.LinearOperator.frobenius_norm(op, samples=64, seed=1) == pytest.approx(exact, rel=0.25)
    op = K.laplace3d(2, 2, 2)
    op.apply(np.ones(8))
    op.apply(np.ones(8))
    assert op.napply == 2
    with pytest.raises(K.DimensionError):
        op.apply(np.ones(9))


def test_square_operator_guard(cuda):
    """test_problems.py:276-283"""
    K = kls()
    rect = K.CsrMatrix.from_coo(2, 3, [0, 1], [2, 0], [1.0, 2.0])
    with pytest.raises(K.DimensionError):
        K.CsrOperator(rect)
    with pytest.raises(K.DimensionError):
        K.DenseOperator(np.ones((2, 3)))


def test_metric_device_paths(cuda, rng):
    """test_metrics.py:61-77 on device bases"""
    K = kls()
    op = mant(6)
    v, h = K.arnoldi_expand(op, rng.standard_normal(op.n), "cgs2", steps=12)
    assert K.representation_error_arnoldi(op, v, h) <= 1e-14
    h2 = h.copy()
    h2[0, 0] += 1.0
    assert K.representation_error_arnoldi(op, v, h2) == pytest.approx(
        1.0 / np.linalg.norm(op.to_dense()), rel=1e-6)
    v, h = K.arnoldi_expand(op, rng.standard_normal(op.n), "dcgs2", steps=15)
    a1 = K.representation_error_arnoldi(op, v, h)
    assert a1 == pytest.approx(K.representation_error_arnoldi(op, v.clone(), h.copy()), abs=1e-15)


def test_flop_lead_coefficients_at_scale(cuda):
    """test_ledger.py:120-134 for the device schemes (m = 1e5, n = 100)"""
    K = kls()
    m, n = 100_000, 100
    a = np.random.Generator(np.random.PCG64(8)).standard_normal((m, n))
    for scheme in SCHEMES:
        led = K.SyncLedger()
        K.qr_factorize(a, scheme, ledger=led)
        lead = led.flops / (m * n * n)
        expect = K.predicted_counts(scheme, n).flop_lead
        assert abs(lead - expect) <= 0.1 * expect, (scheme, lead, expect)
