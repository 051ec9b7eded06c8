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
