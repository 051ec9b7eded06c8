"""Bitwise check of schur.py against a saved earlier copy of it (SCHUR_ORIG,
e.g. `git show HEAD~1:paper_2104_01253_b200/schur.py > /tmp/schur_orig.py`)
on random Hessenberg problems: Hessenberg reduction, Schur form, block
reordering, sorted Schur form and eigenvectors must agree to the bit.

    SCHUR_ORIG=/tmp/schur_orig.py python scripts/schur_bitwise_check.py [seed]
"""

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2104_01253_b200 import schur as NEW  # noqa: E402


def load_old(path):
    src = open(path).read().replace("from .errors import", "from paper_2104_01253_b200.errors import")
    mod = {"__name__": "schur_orig"}
    exec(compile(src, path, "exec"), mod)
    return type("Old", (), {k: staticmethod(v) if callable(v) else v for k, v in mod.items()
                            if not k.startswith("__")})


def work(S, H, sel_seed):
    H1, U = S.hessenberg_reduce(H)
    f = S.hessenberg_real_schur(np.triu(H1, -1))
    nb = len(S.block_list(f.t))
    sel = np.random.default_rng(sel_seed).random(nb) < 0.5
    S.move_blocks_front(f, sel)
    vals, Y = S.schur_eigenvectors(f)
    f2 = S.hessenberg_real_schur(np.triu(H1, -1), sort_key=lambda z: -abs(z))
    return [H1, U, f.t, f.z, vals, Y, f2.t, f2.z]


def main():
    old = load_old(os.environ.get("SCHUR_ORIG", "/tmp/schur_orig.py"))
    rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
    t_old = t_new = 0.0
    for t in range(60):
        n = int(rng.integers(3, 61))
        kind = t % 3
        if kind == 0:
            A = rng.standard_normal((n, n))
        elif kind == 1:
            A = rng.standard_normal((n, n)) + np.diag(np.linspace(1, 8, n)) * 3
        else:
            A = np.triu(rng.standard_normal((n, n)), -1)
            A[np.arange(1, n), np.arange(n - 1)] *= 1e-3
        t0 = time.perf_counter()
        a = work(old, A, t)
        t_old += time.perf_counter() - t0
        t0 = time.perf_counter()
        b = work(NEW, A, t)
        t_new += time.perf_counter() - t0
        for x, y in zip(a, b):
            x, y = np.ascontiguousarray(x), np.ascontiguousarray(y)
            assert x.shape == y.shape and x.tobytes() == y.tobytes(), (t, n)
    print(f"bitwise identical; old {t_old:.2f}s new {t_new:.2f}s")


if __name__ == "__main__":
    main()
