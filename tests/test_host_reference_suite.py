"""The reference's host-side test cases (pkg/tests/test_ledger.py,
test_problems.py, test_metrics.py) against this package's host mirror of
the reference interface: the synchronization ledger and cost model, the CSR
storage and test-problem generators, Matrix Market ingestion and the host
metric paths.  CPU only; the Matrix Market corpus comes from the committed
fixture tests/golden/mtx_corpus.json (generated from the reference's
pkg/tests/data by tests/golden/make_golden.py --only mtx).
"""

import io
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN


def kls():
    import paper_2104_01253_b200 as k

    return k


# ---------------------------------------------------------------------------
# test_ledger.py


def test_record_reductions_by_class():
    """test_ledger.py:16-25"""
    from paper_2104_01253_b200.ledger import MV_DOT, MV_TIMES_MAT_ADD_MV, MV_TRANS_MV

    led = kls().SyncLedger()
    led.record(MV_DOT, flops=10)
    assert led.reductions == 1
    led.record(MV_TIMES_MAT_ADD_MV, flops=5)
    assert led.reductions == 1
    led.record(MV_TRANS_MV, flops=20)
    assert led.reductions == 2 and led.flops == 35
    assert led.kernel_counts == {MV_TRANS_MV: 1, MV_TIMES_MAT_ADD_MV: 1, MV_DOT: 1}


def test_reductions_equal_reducing_kernel_counts():
    """test_ledger.py:28-36"""
    from paper_2104_01253_b200.ledger import MV_DOT, MV_TIMES_MAT_ADD_MV, MV_TRANS_MV

    led = kls().SyncLedger()
    for cls, n in ((MV_TRANS_MV, 7), (MV_DOT, 4), (MV_TIMES_MAT_ADD_MV, 9)):
        for _ in range(n):
            led.record(cls)
    assert led.reductions == led.kernel_counts[MV_TRANS_MV] + led.kernel_counts[MV_DOT]


def test_reset_local_flops_and_unknown_class():
    """test_ledger.py:39-51"""
    from paper_2104_01253_b200.ledger import MV_DOT

    led = kls().SyncLedger()
    led.record(MV_DOT, flops=4)
    led.add_flops(25)
    assert led.flops == 29
    led.reset()
    assert led.reductions == 0 and led.flops == 0
    assert all(v == 0 for v in led.kernel_counts.values())
    with pytest.raises(ValueError):
        kls().SyncLedger().record("Gemm")


def test_csv_row_schema():
    """test_ledger.py:54-61"""
    from paper_2104_01253_b200.ledger import CSV_HEADER, MV_DOT, MV_TRANS_MV

    led = kls().SyncLedger()
    led.record(MV_TRANS_MV, flops=100)
    led.record(MV_DOT, flops=10)
    assert CSV_HEADER == "run_id,scheme,n,m,reductions,mvtransmv,mvdot,mvtimes,flops"
    assert led.csv_row("r1", "cgs2", 50, 5000) == "r1,cgs2,50,5000,2,1,1,0,110"


@pytest.mark.parametrize("scheme,n,total", [
    ("cgs2", 50, 150), ("dcgs2", 50, 50), ("cgs", 50, 100), ("cgs2-lagged", 50, 100),
    ("icwy-mgs", 50, 50), ("mgs", 50, 1275), ("mgs", 20, 210), ("dcgs2-hrt", 50, 50)])
def test_predicted_totals(scheme, n, total):
    """test_ledger.py:64-78"""
    assert kls().predicted_counts(scheme, n).total_synchs == total


def test_per_iteration_formulas_and_unknown_scheme():
    """test_ledger.py:81-91"""
    K = kls()
    assert K.per_iteration_synchs("cgs2", 7) == 3
    assert K.per_iteration_synchs("cgs2-lagged", 7) == 2
    assert K.per_iteration_synchs("mgs", 7) == 7
    assert K.per_iteration_synchs("dcgs2", 7) == 1
    assert K.per_iteration_synchs("icwy-mgs", 7) == 1
    with pytest.raises(K.UnknownSchemeError):
        K.predicted_counts("gram", 10)


def test_assert_matches_exact_and_slack():
    """test_ledger.py:94-117"""
    from paper_2104_01253_b200.ledger import MV_DOT

    K = kls()

    def led_with(n):
        led = K.SyncLedger()
        for _ in range(n):
            led.record(MV_DOT)
        return led

    assert K.assert_matches(led_with(150), K.predicted_counts("cgs2", 50)).passed
    rep = K.assert_matches(led_with(52), K.predicted_counts("dcgs2", 50))
    assert rep.passed and rep.delta == 2
    rep = K.assert_matches(led_with(151), K.predicted_counts("cgs2", 50))
    assert not rep.passed and rep.delta == 1
    assert not K.assert_matches(led_with(49), K.predicted_counts("dcgs2", 50)).passed


# ---------------------------------------------------------------------------
# test_problems.py: CSR storage, generators, Matrix Market


def test_csr_from_coo_and_transpose(rng):
    """test_problems.py:29-44, 60-62 (the products, :47-57, run on the
    device: test_gpu_reference_suite.py)"""
    K = kls()
    csr = K.CsrMatrix.from_coo(2, 2, [0, 0, 1], [1, 1, 0], [2.0, 3.0, -1.0])
    assert csr.nnz == 2 and csr.to_dense().tolist() == [[0.0, 5.0], [-1.0, 0.0]]
    n = 30
    csr = K.CsrMatrix.from_coo(n, n, rng.integers(0, n, 200), rng.integers(0, n, 200),
                               rng.standard_normal(200))
    for i in range(n):
        assert np.all(np.diff(csr.indices[csr.indptr[i]:csr.indptr[i + 1]]) > 0)
    assert np.all(np.diff(csr.indptr) >= 0)
    csr = K.CsrMatrix.from_coo(3, 5, [0, 2, 2], [4, 1, 3], [1.0, 2.0, 3.0])
    assert np.array_equal(csr.transpose().to_dense(), csr.to_dense().T)


def test_manteuffel_family():
    """test_problems.py:69-127"""
    K = kls()
    spec = K.ManteuffelSpec(k=1)
    a = K.manteuffel_build(spec).to_dense()
    assert a.shape == (1, 1) and a[0, 0] == pytest.approx(4.0)
    assert np.allclose(K.manteuffel_eigenvalues(spec).values, [4.0])
    spec = K.ManteuffelSpec(k=2, beta=0.5)
    ev = np.sort(np.linalg.eigvals(K.manteuffel_build(spec).to_dense()).real)
    assert np.allclose(ev, [2.063508, 4.0, 4.0, 5.936492], atol=1e-6)
    table = K.manteuffel_eigenvalues(spec)
    assert np.max(np.abs(table.values - ev)) <= 1e-9
    assert table.multiplicity[np.argmin(np.abs(table.unique - 4.0))] == 2
    mm, nn = K.manteuffel_parts(K.ManteuffelSpec(k=6))
    assert np.array_equal(mm.to_dense(), mm.to_dense().T)
    assert np.array_equal(nn.to_dense(), -nn.to_dense().T)
    assert np.min(np.linalg.eigvalsh(mm.to_dense())) > 0
    for k in (1, 2, 3, 5, 8, 12):
        spec = K.ManteuffelSpec(k=k, beta=0.5)
        dense_ev = np.sort(np.linalg.eigvals(K.manteuffel_build(spec).to_dense()).real)
        table = K.manteuffel_eigenvalues(spec)
        assert len(table.values) == k * k and int(np.sum(table.multiplicity)) == k * k
        assert np.max(np.abs(dense_ev - table.values)) <= 1e-8
    table = K.manteuffel_eigenvalues(K.ManteuffelSpec(k=3, beta=0.0))
    theta = np.cos(np.arange(1, 4) * np.pi / 4)
    assert np.allclose(table.values, np.sort((2 * (2 - (theta[:, None] + theta[None, :]))).ravel()),
                       atol=1e-14)
    spec = K.ManteuffelSpec(k=4, beta=0.3, length=2.0)
    assert spec.h == pytest.approx(0.4)
    ev = np.sort(np.linalg.eigvals(K.manteuffel_build(spec).to_dense()).real)
    assert np.max(np.abs(ev - K.manteuffel_eigenvalues(spec).values)) <= 1e-8
    with pytest.raises(ValueError):
        K.manteuffel_eigenvalues(K.ManteuffelSpec(k=3, beta=2.5))
    with pytest.raises(ValueError):
        K.ManteuffelSpec(k=0)


def test_synthetic_kappa():
    """test_problems.py:188-210"""
    from paper_2104_01253_b200.cli import synthetic_kappa

    s = np.linalg.svd(synthetic_kappa(60, 10, 1.0, seed=2), compute_uv=False)
    assert s[0] / s[-1] == pytest.approx(1.0, rel=1e-12)
    s = np.linalg.svd(synthetic_kappa(80, 12, 1e8, seed=3), compute_uv=False)
    assert s[0] / s[-1] == pytest.approx(1e8, rel=0.05)
    assert np.array_equal(synthetic_kappa(40, 6, 1e4, seed=7), synthetic_kappa(40, 6, 1e4, seed=7))
    with pytest.raises(ValueError):
        synthetic_kappa(10, 2, 0.5, seed=0)


@pytest.fixture(scope="module")
def corpus():
    with open(os.path.join(GOLDEN, "mtx_corpus.json")) as f:
        return json.load(f)


def test_matrix_market_corpus_matches_reference(corpus):
    """test_problems.py:215-252: every good file parses to the reference's
    CSR arrays; every bad file raises MatrixMarketError at its line"""
    K = kls()
    assert len(corpus) == 14
    for name, ref in corpus.items():
        src = io.StringIO(ref["text"])
        if ref["ok"]:
            csr = K.parse_matrix_market(src)
            assert (csr.nrows, csr.ncols) == (ref["nrows"], ref["ncols"]), name
            assert csr.indptr.tolist() == ref["indptr"], name
            assert csr.indices.tolist() == ref["indices"], name
            assert csr.data.tolist() == ref["data"], name
        else:
            with pytest.raises(K.MatrixMarketError) as err:
                K.parse_matrix_market(src)
            assert err.value.line == ref["line"], name


def test_matrix_market_semantics(corpus):
    """test_problems.py:215-234"""
    K = kls()
    csr = K.parse_matrix_market(io.StringIO(corpus["good_identity2.mtx"]["text"]))
    assert csr.nnz == 2 and np.array_equal(csr.to_dense(), np.eye(2))
    d = K.parse_matrix_market(io.StringIO(corpus["good_symmetric.mtx"]["text"])).to_dense()
    assert np.array_equal(d, d.T) and d[0, 0] == 4.0 and d[1, 0] == -1.5 and d[0, 1] == -1.5
    d = K.parse_matrix_market(io.StringIO(corpus["good_skew.mtx"]["text"])).to_dense()
    assert np.array_equal(d, -d.T) and d[1, 0] == 1.5 and d[0, 1] == -1.5


def test_matrix_market_roundtrip_and_string(rng):
    """test_problems.py:255-273"""
    K = kls()
    n = 12
    csr = K.CsrMatrix.from_coo(n, n, rng.integers(0, n, 40), rng.integers(0, n, 40),
                               rng.standard_normal(40))
    buf = io.StringIO()
    K.write_matrix_market(csr, buf, comment="roundtrip")
    back = K.parse_matrix_market(io.StringIO(buf.getvalue()))
    assert np.array_equal(back.indptr, csr.indptr)
    assert np.array_equal(back.indices, csr.indices)
    assert np.array_equal(back.data, csr.data)
    csr = K.parse_matrix_market("%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 -3.5\n")
    assert csr.to_dense()[0, 0] == -3.5


# (text, line of the MatrixMarketError) -- each line number was obtained by
# running the reference's parse_matrix_market (problems.py:368-469) here:
# the first offending line in file order wins, whatever the failure kind
_MM_EDGE = [
    ("2 2 2\n1 1 x\n1 1 1\n1 1 1\n", "general", 3),     # unparsable before the extra entry
    ("2 2 1\n\n% c\n3 1 1\n", "general", 5),            # out of bounds after blank + comment
    ("2 2 2\n1 2 1\n2 2 1\n", "skew-symmetric", 4),     # nonzero skew diagonal
    ("2 2 3\n1 1 1\n% tail\n\n", "general", 5),         # too few entries: the last line
    ("2 2 1\n1 1 1 1\n", "general", 3),                 # four tokens
    ("% only comment\n", "general", 2),                 # no size line
    ("2 2 -1\n", "general", 2),                         # negative size
    ("2 x 1\n", "general", 2),                          # non-integer size
]


@pytest.mark.parametrize("body,sym,line", _MM_EDGE)
def test_matrix_market_error_lines(body, sym, line):
    K = kls()
    text = f"%%MatrixMarket matrix coordinate real {sym}\n" + body
    with pytest.raises(K.MatrixMarketError) as err:
        K.parse_matrix_market(io.StringIO(text))
    assert err.value.line == line


# ---------------------------------------------------------------------------
# test_metrics.py (host paths)


def test_metric_host_paths(rng):
    """test_metrics.py:21-58, 80-98"""
    K = kls()
    assert K.loss_of_orthogonality(np.eye(5)) == 0.0
    q = np.zeros((4, 2))
    q[0, 0] = q[0, 1] = 1.0
    assert K.loss_of_orthogonality(q) == pytest.approx(np.sqrt(2.0))
    q, _ = np.linalg.qr(np.random.Generator(np.random.PCG64(5)).standard_normal((500, 50)))
    assert K.loss_of_orthogonality(q) <= 1e-13
    a = rng.standard_normal((30, 6))
    q, r = np.linalg.qr(a)
    assert K.representation_error_qr(a, q, r) <= 1e-15
    assert K.representation_error_qr(a, q, np.zeros_like(r)) == pytest.approx(1.0)
    a = rng.standard_normal((40, 8))
    q, r = np.linalg.qr(a)
    signs = np.array([1, -1, 1, -1, -1, 1, 1, -1], dtype=float)
    assert K.loss_of_orthogonality(q * signs[None, :]) == pytest.approx(
        K.loss_of_orthogonality(q), abs=1e-15)
    assert K.representation_error_qr(a, q * signs[None, :], r * signs[:, None]) == pytest.approx(
        K.representation_error_qr(a, q, r), abs=1e-16)
    with pytest.raises(K.DimensionError):
        K.representation_error_arnoldi(np.eye(4), np.ones((4, 3)), np.ones((3, 3)))
    spec = K.ManteuffelSpec(k=3)
    table = K.manteuffel_eigenvalues(spec)
    assert K.forward_error_count(table.values.copy(), table, 1e-7) == 9
    assert K.forward_error_count(np.zeros(0), table, 1e-7) == 0


def test_stability_report_validation():
    """test_metrics.py:92-105"""
    K = kls()
    rep = K.StabilityReport(scheme="dcgs2", step=10, loo=1e-15, rre=1e-16)
    assert rep.n_forward_converged == -1
    with pytest.raises(ValueError):
        K.StabilityReport(scheme="cgs", step=5, loo=-1.0, rre=0.0)
