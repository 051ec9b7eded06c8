"""The fused DCGS2 step (csrc/fused.cu: update of step j -> banded ELL
product -> Gram pass of step j+1 with its reduction and scalar step, ONE
launch) against the three unfused launches it replaces: bitwise equal
Q(:, j), w', Aw', reduced g and next coefficients, on odd row counts (segment
tails), several widths and reaches; and end-to-end expansions through the
public API against the oracle."""

import ctypes

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _ops():
    import paper_2104_01253_b200 as kls
    from paper_2104_01253_b200 import problems

    return {
        "mant301": lambda: problems.manteuffel_operator(kls.ManteuffelSpec(k=301, beta=0.5)),
        "mant1000": lambda: problems.manteuffel_operator(kls.ManteuffelSpec(k=1000, beta=0.5)),
        "band200003": lambda: problems.band_random_operator(200_003, band=1000, per_row=7, seed=11),
        "band300000_wide": lambda: problems.band_random_operator(300_000, band=5000, per_row=5,
                                                                 seed=12),
    }


_cache = {}


def _op(name):
    if name not in _cache:
        _cache[name] = _ops()[name]()
    return _cache[name]


def _plan(lib, op, Q, ld, gdev, cdev, gout, ws, wsb, st):
    p = lib.KlsStepPlan()
    p.Q, p.ldq, p.m = Q.data_ptr(), ld, op.n
    p.segs = op.segs.c
    p.gdev, p.cdev = gdev.data_ptr(), cdev.data_ptr()
    p.gout[0] = p.gout[1] = gout.data_ptr()
    p.ws, p.ws_bytes, p.stream = ws, wsb, st
    p.divide, p.qr = 1, 0
    p.op = op.op_desc()
    return p


@pytest.mark.parametrize("name", ["mant301", "mant1000", "band200003", "band300000_wide"])
@pytest.mark.parametrize("j", [0, 1, 4, 7, 50, 101, 150])
def test_fused_step_bitwise_unfused(cuda, name, j):
    from paper_2104_01253_b200 import _lib as lib
    from paper_2104_01253_b200 import runtime as rt

    op = _op(name)
    m = op.n
    assert op._ell is not None
    ld = rt.pad_rows(m)
    g = torch.Generator(device="cuda").manual_seed(1000 + j)
    Q = torch.randn((j + 2, ld), dtype=torch.float64, device="cuda", generator=g) / np.sqrt(m)
    Q[:, m:] = 0
    w = torch.randn(m, dtype=torch.float64, device="cuda", generator=g)
    aw = op.apply(w)
    nres = 2 * (j + 1) + 3
    st = rt.stream_handle()
    ws, wsb = rt.workspace_for(st, j + 3, m)
    segp = op.segs.ptr
    gdev = torch.zeros(nres, dtype=torch.float64, device="cuda")
    cdev = torch.zeros(nres, dtype=torch.float64, device="cuda")
    gout = torch.zeros(nres, dtype=torch.float64, device="cuda")
    # the step's coefficients as the preceding Gram + scalar step makes them
    lib.call("kls_gram_dcgs2_step", Q.data_ptr(), ld, m, j, w.data_ptr(), aw.data_ptr(),
             gdev.data_ptr(), cdev.data_ptr(), gout.data_ptr(), 0, segp, ws, wsb, st)
    Q2, g2, c2, o2 = Q.clone(), gdev.clone(), cdev.clone(), gout.clone()
    # unfused: the three launches of kls_dcgs2_queue_step
    w1, a1 = torch.empty_like(w), torch.empty_like(w)
    ecol, evals, elen, width, eld = op._ell
    lib.call("kls_dcgs2_update_dev", Q.data_ptr(), ld, m, j, w.data_ptr(), w1.data_ptr(),
             aw.data_ptr(), cdev.data_ptr(), 1, segp, st)
    lib.call("kls_ell_spmv", ecol.data_ptr(), evals.data_ptr(), elen.data_ptr(), width, m, eld,
             w1.data_ptr(), a1.data_ptr(), st)
    lib.call("kls_gram_dcgs2_step", Q.data_ptr(), ld, m, j + 1, w1.data_ptr(), a1.data_ptr(),
             gdev.data_ptr(), cdev.data_ptr(), gout.data_ptr(), 0, segp, ws, wsb, st)
    # fused
    plan = _plan(lib, op, Q2, ld, g2, c2, o2, ws, wsb, st)
    assert lib.load().kls_dcgs2_fused_eligible(ctypes.byref(plan), j) == 1
    w2, a2 = torch.full_like(w, np.nan), torch.full_like(w, np.nan)
    lib.call("kls_dcgs2_fused_step", ctypes.byref(plan), j, w.data_ptr(), w2.data_ptr(),
             aw.data_ptr(), a2.data_ptr(), 0)
    assert lib.load().kls_dcgs2_fused_error(st) == 0
    torch.cuda.synchronize()
    assert torch.equal(Q2[j, :m], Q[j, :m])
    assert torch.equal(Q2[: j, :m], Q[: j, :m])
    assert torch.equal(w2, w1)
    assert torch.equal(a2, a1)
    assert torch.equal(g2, gdev)
    assert torch.equal(c2[: nres - 1], cdev[: nres - 1])
    assert torch.equal(o2, gout)


def test_fused_step_ineligible_cases(cuda):
    """Off the fused path: several ranks, small m, CSR-only or unknown reach
    -- eligibility says no and the entry point refuses loudly."""
    from paper_2104_01253_b200 import _lib as lib
    from paper_2104_01253_b200 import runtime as rt
    import paper_2104_01253_b200 as kls
    from paper_2104_01253_b200 import problems

    small = problems.manteuffel_operator(kls.ManteuffelSpec(k=100))  # m = 1e4
    big = _op("mant301")
    st = rt.stream_handle()
    ws, wsb = rt.workspace_for(st, 8, big.n)
    t = torch.zeros(max(big.n, 8) * 4, dtype=torch.float64, device="cuda")
    for op, ok in ((small, 0), (big, 1)):
        plan = _plan(lib, op, t, rt.pad_rows(op.n), t, t, t, ws, wsb, st)
        assert lib.load().kls_dcgs2_fused_eligible(ctypes.byref(plan), 2) == ok
    plan = _plan(lib, big, t, rt.pad_rows(big.n), t, t, t, ws, wsb, st)
    plan.op.reach = 0  # unknown reach
    assert lib.load().kls_dcgs2_fused_eligible(ctypes.byref(plan), 2) == 0
    with pytest.raises(lib.KlsGpuError):
        lib.call("kls_dcgs2_fused_step", ctypes.byref(plan), 2, t.data_ptr(), t.data_ptr(),
                 t.data_ptr(), t.data_ptr(), 0)


@pytest.mark.parametrize("name", ["mant301", "band200003"])
def test_fused_expansion_matches_oracle(cuda, name):
    """arnoldi_expand through the public API (the native lookahead loop, now
    one fused launch per step) against the oracle's DCGS2 expansion."""
    import paper_2104_01253_b200 as kls

    op = _op(name)
    ptr = op._rowptr.cpu().numpy()
    idx = op._col.cpu().numpy()[: ptr[-1]]
    dat = op._val.cpu().numpy()[: ptr[-1]]
    steps = 40
    start = np.random.Generator(np.random.PCG64(7)).standard_normal(op.n)
    led = kls.SyncLedger()
    n0 = op.napply
    V, H = kls.arnoldi_expand(op, start, "dcgs2", steps=steps, ledger=led)
    Vr, Hr, cnt = oracle.dcgs2_arnoldi(lambda x: oracle.csr_matvec(ptr, idx, dat, x), start, steps)
    assert np.max(np.abs(H - Hr)) <= 1e-12 * np.max(np.abs(Hr))
    assert np.max(np.abs(V.cpu().numpy() - Vr)) <= 1e-10
    assert led.reductions == cnt.reductions and op.napply - n0 == cnt.napply
