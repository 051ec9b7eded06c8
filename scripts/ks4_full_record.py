"""BASELINE config 4 at full size on the GPU, instrumented like the
reference run of tests/golden/make_golden.py --only ks_config4_full: every
restart's active Hessenberg block -> its sorted Ritz values and size, plus
the final lock history and locked values.  Writes gpurun_out/ks4_full_gpu.npz.

    python scripts/ks4_full_record.py [--restarts 240] [--operator host|device]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--restarts", type=int, default=240)
    ap.add_argument("--operator", default="host", choices=("host", "device"))
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "ks4_full_gpu.npz"))
    a = ap.parse_args()
    import paper_2104_01253_b200 as kls
    import paper_2104_01253_b200.eig as keig

    rec = {"ritz": [], "na": []}
    orig = keig._schur_of

    def spy(block):
        rec["na"].append(block.shape[0])
        rec["ritz"].append(np.sort_complex(np.linalg.eigvals(block)))
        return orig(block)

    keig._schur_of = spy
    spec = kls.ManteuffelSpec(k=3163, beta=0.5)
    op = (kls.CsrOperator(kls.manteuffel_build(spec)) if a.operator == "host"
          else kls.manteuffel_operator(spec))
    cfg = kls.KrylovSchurConfig(max_basis=60, tol=1e-7, scheme="dcgs2", max_restarts=a.restarts)
    t0 = time.perf_counter()
    res = kls.krylov_schur_run(op, cfg, seed=1729)
    sec = time.perf_counter() - t0
    ritz = np.zeros((len(rec["na"]), 60), dtype=np.complex128)
    for i, v in enumerate(rec["ritz"]):
        ritz[i, : v.size] = v
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    np.savez_compressed(a.out, ritz=ritz, na=np.array(rec["na"]), values=np.asarray(res.values),
                        lock_history=np.array(res.lock_history), restarts=res.restarts, seconds=sec)
    lh = [int(x) for x in res.lock_history]
    print(json.dumps({"restarts": res.restarts, "seconds": sec, "invariant_dim": res.invariant_dim,
                      "locks": [(i, v) for i, v in enumerate(lh) if i == 0 or lh[i] != lh[i - 1]]}))


if __name__ == "__main__":
    main()
