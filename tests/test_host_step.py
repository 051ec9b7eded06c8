"""The C++ host step (kls_dcgs2_host_step, numpy's own OpenBLAS entry points)
against the numpy host step (arnoldi.py:367-420 restated): identical bits in
every output, identical ledger, identical breakdown decisions — on random
steps including near-breakdown ones.  CPU only (host code of libklsgpu.so)."""

import importlib

import numpy as np
import pytest


def test_c_host_step_bitwise_matches_numpy():
    A = importlib.import_module("paper_2104_01253_b200.arnoldi")
    from paper_2104_01253_b200.ledger import SyncLedger

    if not A._host_blas():
        pytest.skip("numpy without scipy-openblas: the numpy host step is used")
    rng = np.random.default_rng(1)
    kinds = {"ok": 0, "happy": 0, "pyth": 0}
    for t in range(1500):
        j = int(rng.integers(0, 160))
        cap = j + 2 + int(rng.integers(0, 5))
        g = rng.standard_normal(2 * j + 3) * 10.0 ** rng.uniform(-3, 3)
        if t % 3:
            g[j] = float(g[:j] @ g[:j]) * (1 + 10.0 ** rng.uniform(-17, 1))
        if t % 7 == 0:
            g[j] = 1e-40
        g[2 * j + 2] = abs(g[2 * j + 2])
        kp = rng.standard_normal(j)
        h1 = rng.standard_normal((cap, cap - 1))
        h2 = h1.copy()
        l1, l2 = SyncLedger(), SyncLedger()
        out = []
        for f, h, led in ((A._host_step_numpy, h1, l1), (A.dcgs2_host_step, h2, l2)):
            try:
                out.append(("ok", f(g, j, 12345, 0.7, kp, h, led)))
            except A.BreakdownError as e:
                out.append(("pyth", str(e)))
        (k1, r1), (k2, r2) = out
        assert k1 == k2, t
        assert np.array_equal(h1, h2) and l1.flops == l2.flops, t
        assert l1.kernel_counts == l2.kernel_counts, t
        if k1 == "pyth":
            assert r1 == r2
            kinds["pyth"] += 1
        elif r1 is None:
            assert r2 is None
            kinds["happy"] += 1
        else:
            kinds["ok"] += 1
            for a, b in zip(r1, r2):
                assert np.array_equal(np.asarray(a), np.asarray(b)), t
    assert all(v > 0 for v in kinds.values()), kinds
