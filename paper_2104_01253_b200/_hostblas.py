"""numpy's own OpenBLAS (the ILP64 scipy-openblas numpy wheels carry), so the
C++ host services (kls_dcgs2_host_step, the kls_schur_* family) can issue
the very BLAS / LAPACK calls numpy's dot, matmul, linalg.solve and
linalg.qr issue, and reproduce numpy's results bit for bit.  None when this
numpy carries another BLAS (the callers then keep their numpy paths)."""

import ctypes
import glob
import os

import numpy as np

_SYMS = {"ddot": "scipy_cblas_ddot64_", "dgemv": "scipy_cblas_dgemv64_",
         "dgemm": "scipy_cblas_dgemm64_", "dgesv": "scipy_dgesv_64_",
         "dgeqrf": "scipy_dgeqrf_64_", "dorgqr": "scipy_dorgqr_64_",
         "zgemv": "scipy_cblas_zgemv64_", "zdotu_sub": "scipy_cblas_zdotu_sub64_"}
_PTRS = None


def pointers():
    """{name: address} of numpy's entry points, or None."""
    global _PTRS
    if _PTRS is None:
        _PTRS = False
        libs = glob.glob(os.path.join(os.path.dirname(np.__file__), os.pardir, "numpy.libs",
                                      "libscipy_openblas64_*.so"))
        if len(libs) == 1:
            try:
                lib = ctypes.CDLL(libs[0])
                _PTRS = {k: ctypes.cast(getattr(lib, v), ctypes.c_void_p).value
                         for k, v in _SYMS.items()}
            except (OSError, AttributeError):
                _PTRS = False
    return _PTRS or None
