"""Small end-to-end run for compute-sanitizer (memcheck / racecheck):
every kernel family on odd sizes, TMA paths included (m >= 1024)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01253_b200 as kls
rng = np.random.default_rng(0)
op = kls.laplace3d(13, 11, 17)             # m = 2431 (odd, > 1024: TMA path + ragged tail)
s = rng.standard_normal(op.n)
for scheme in ("dcgs2", "cgs2"):
    kls.arnoldi_expand(op, s, scheme, 12)
mop = kls.manteuffel_operator(kls.ManteuffelSpec(k=37))  # device-built CSR + ELL
kls.gmres_solve(mop, rng.standard_normal(mop.n), kls.GmresConfig(max_iters=30, restart=10, rtol=1e-12, scheme="dcgs2"))
kls.qr_factorize(rng.standard_normal((3001, 9)), "dcgs2")
kls.krylov_schur_run(kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=6))),
                     kls.KrylovSchurConfig(max_basis=12, scheme="dcgs2", max_restarts=3), seed=1)
# Krylov-Schur rotation kernel: ragged row tile, two column passes
import torch
from paper_2104_01253_b200 import _lib, runtime
m, k, p = 1001, 40, 35
ld = runtime.pad_rows(m)
V = torch.randn((k + 1, ld), dtype=torch.float64, device="cuda")
Z = torch.randn(k * p, dtype=torch.float64, device="cuda")
_lib.call("kls_tsgemm_inplace_cols", V.data_ptr(), ld, m, k, p, Z.data_ptr(), runtime.stream_handle())
# the 256-row rotation (p <= 32): ragged last tile, odd row count, two column stages
m, k, p = 3001, 44, 30
ld = runtime.pad_rows(m)
V = torch.randn((k + 1, ld), dtype=torch.float64, device="cuda")
Z = torch.randn(k * p, dtype=torch.float64, device="cuda")
_lib.call("kls_tsgemm_inplace_cols", V.data_ptr(), ld, m, k, p, Z.data_ptr(), runtime.stream_handle())
# GMRES with backward errors riding on the next step (combined update + dual
# ELL kernel): ELL operator above 65536 rows, odd m, restart 7
bop = kls.manteuffel_operator(kls.ManteuffelSpec(k=257))
kls.gmres_solve(bop, rng.standard_normal(bop.n),
                kls.GmresConfig(max_iters=16, restart=7, rtol=1e-14, scheme="dcgs2",
                                backward_errors=True))
# host Schur services (C++) on a 40 x 40 problem
from paper_2104_01253_b200 import schur
f = schur.hessenberg_real_schur(schur.hessenberg_reduce(rng.standard_normal((40, 40)))[0])
schur.move_blocks_front(f, [i % 3 == 0 for i in range(len(f.blocks()))])
schur.schur_eigenvectors(f)
torch.cuda.synchronize()
print("sanitize run ok")
