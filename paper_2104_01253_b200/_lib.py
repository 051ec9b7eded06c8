"""ctypes binding of libklsgpu.so (the C-ABI declared in include/klsgpu.h).

There is no fallback: if the library or a GPU is missing, the first kernel
call raises.  Loading the library itself does not need a GPU, so the CPU
test suite can check that every declared symbol is exported.
"""

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libklsgpu.so")

c_dp = ctypes.c_void_p  # device pointers travel as integers
i32 = ctypes.c_int32
i64 = ctypes.c_int64
f64 = ctypes.c_double
sz = ctypes.c_size_t

# name -> (restype, argtypes); must match include/klsgpu.h
SIGNATURES = {
    "kls_version": (ctypes.c_int, []),
    "kls_last_error": (ctypes.c_char_p, []),
    "kls_device_sm_count": (ctypes.c_int, []),
    "kls_stream_sync": (ctypes.c_int, [c_dp]),
    "kls_host_device_ptr": (ctypes.c_int, [c_dp, ctypes.POINTER(ctypes.c_void_p)]),
    "kls_workspace_bytes": (sz, [i64, i32]),
    "kls_mv_trans_mv": (ctypes.c_int, [c_dp, i64, i64, i32, c_dp, c_dp, c_dp, i32, i32, c_dp, c_dp, c_dp, sz, c_dp]),
    "kls_project_gram": (ctypes.c_int, [c_dp, i64, i64, i32, c_dp, c_dp, i32, i32, c_dp, c_dp, c_dp, sz, c_dp]),
    "kls_ipc_handle_bytes": (sz, []),
    "kls_peer_buffer_alloc": (ctypes.c_int, [sz, ctypes.POINTER(ctypes.c_void_p), c_dp]),
    "kls_peer_buffer_open": (ctypes.c_int, [c_dp, ctypes.POINTER(ctypes.c_void_p)]),
    "kls_peer_buffer_close": (ctypes.c_int, [c_dp]),
    "kls_peer_buffer_free": (ctypes.c_int, [c_dp]),
    "kls_gram_dcgs2_step": (ctypes.c_int, [c_dp, i64, i64, i32, c_dp, c_dp, c_dp, c_dp, c_dp, i32,
                                           c_dp, c_dp, sz, c_dp]),
    "kls_gram_dcgs2_peer_step": (ctypes.c_int, [c_dp, i64, i64, i32, c_dp, c_dp, c_dp, c_dp, c_dp,
                                                i32, c_dp, c_dp, sz, c_dp, i32, i32, i32,
                                                ctypes.c_uint64, c_dp,
                                                c_dp]),
    "kls_dcgs2_host_step": (ctypes.c_int, [c_dp, i32, i64, f64, c_dp, c_dp, i64, c_dp, c_dp, c_dp,
                                           c_dp, c_dp]),
    "kls_dcgs2_queue_step": (ctypes.c_int, [c_dp, i32, c_dp, c_dp, c_dp, c_dp, c_dp, i32, i32]),
    "kls_dcgs2_queue_step_be": (ctypes.c_int, [c_dp, i32, c_dp, c_dp, c_dp, c_dp, c_dp, i32, i32,
                                               c_dp]),
    "kls_ell_apply_resid_norms": (ctypes.c_int, [c_dp, c_dp, c_dp, i32, i64, i64, c_dp, c_dp, c_dp,
                                                 c_dp, c_dp, c_dp, c_dp, sz, c_dp]),
    "kls_event_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p)]),
    "kls_event_destroy": (ctypes.c_int, [c_dp]),
    "kls_event_record": (ctypes.c_int, [c_dp, c_dp]),
    "kls_event_sync": (ctypes.c_int, [c_dp]),
    "kls_ell_spmv_peer": (ctypes.c_int, [c_dp, c_dp, c_dp, i32, i64, i64, c_dp, c_dp, i64, c_dp,
                                         c_dp, i64, i64, c_dp, i32, i32, ctypes.c_uint64, c_dp,
                                         c_dp]),
    "kls_dcgs2_run": (ctypes.c_int, [c_dp, i32, i32, i32, i32, c_dp]),
    "kls_hessenberg_reduce": (ctypes.c_int, [c_dp, c_dp, i64, c_dp]),
    "kls_ell_resid_norms": (ctypes.c_int, [c_dp, c_dp, c_dp, i32, i64, i64, c_dp, c_dp, c_dp,
                                           c_dp, c_dp, sz, c_dp]),
    "kls_schur_sweeps": (ctypes.c_int, [c_dp, c_dp, i64, i64, c_dp]),
    "kls_schur_swap": (ctypes.c_int, [c_dp, c_dp, i64, i64, i32, i32, c_dp]),
    "kls_schur_move_front": (i64, [c_dp, c_dp, i64, c_dp, i64, c_dp]),
    "kls_schur_eigenvectors": (ctypes.c_int, [c_dp, c_dp, i64, i64, c_dp, i64, c_dp, c_dp, c_dp]),
    "kls_gram_dcgs2": (ctypes.c_int, [c_dp, i64, i64, i32, c_dp, c_dp, c_dp, c_dp, c_dp, sz, c_dp]),
    "kls_dcgs2_update": (ctypes.c_int, [c_dp, i64, i64, i32, c_dp, c_dp, c_dp, f64, i32, c_dp, c_dp]),
    "kls_dcgs2_scalars": (ctypes.c_int, [c_dp, i32, i32, c_dp, c_dp, c_dp]),
    "kls_dcgs2_update_dev": (ctypes.c_int, [c_dp, i64, i64, i32, c_dp, c_dp, c_dp, c_dp, i32,
                                            c_dp, c_dp]),
    "kls_dcgs2_update_host": (ctypes.c_int, [c_dp, i64, i64, i32, c_dp, c_dp, c_dp, f64, i32, c_dp, c_dp]),
    "kls_mv_times_mat_add_mv": (
        ctypes.c_int,
        [c_dp, i64, i64, i32, c_dp, i64, i32, c_dp, f64, f64, c_dp, c_dp, c_dp, sz, c_dp],
    ),
    "kls_mv_times_mat_add_mv_host": (
        ctypes.c_int,
        [c_dp, i64, i64, i32, c_dp, i64, i32, c_dp, f64, f64, c_dp, c_dp, c_dp, sz, c_dp],
    ),
    "kls_csr_spmv": (ctypes.c_int, [c_dp, c_dp, c_dp, i64, c_dp, c_dp, c_dp]),
    "kls_csr_to_ell": (ctypes.c_int, [c_dp, c_dp, c_dp, i64, i32, i64, c_dp, c_dp, c_dp, c_dp]),
    "kls_ell_spmv": (ctypes.c_int, [c_dp, c_dp, c_dp, i32, i64, i64, c_dp, c_dp, c_dp]),
    "kls_stencil7": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, i64, i64, i64, c_dp]),
    "kls_dense_gemv": (ctypes.c_int, [c_dp, i64, i64, c_dp, c_dp, c_dp]),
    "kls_scale": (ctypes.c_int, [c_dp, c_dp, i64, f64, i32, c_dp]),
    "kls_sub": (ctypes.c_int, [c_dp, c_dp, c_dp, i64, c_dp]),
    "kls_resid_norms": (ctypes.c_int, [c_dp, c_dp, c_dp, i64, c_dp, c_dp, c_dp, sz, c_dp]),
    "kls_tsgemm_inplace": (ctypes.c_int, [c_dp, i64, i64, i32, c_dp, c_dp]),
    "kls_tsgemm_inplace_cols": (ctypes.c_int, [c_dp, i64, i64, i32, i32, c_dp, c_dp]),
    "kls_peer_buffer_bytes": (sz, [i32]),
    "kls_lap7_nnz": (i64, [i64, i64, i64, i64, i64]),
    "kls_build_lap7_csr": (ctypes.c_int, [i64, i64, i64, i64, i64, i64, c_dp, c_dp, c_dp, c_dp]),
    "kls_mant5_nnz": (i64, [i64, i64, i64]),
    "kls_build_mant5_csr": (ctypes.c_int, [i64, i64, i64, i64, f64, f64, c_dp, c_dp, c_dp, c_dp]),
    "kls_build_band_csr": (ctypes.c_int, [i64, i64, i32, ctypes.c_uint64, i64, i64, i64, c_dp,
                                          c_dp, c_dp, c_dp]),
    "kls_peer_seg_combine": (ctypes.c_int, [c_dp, i32, c_dp, c_dp, i32, i32, i32, ctypes.c_uint64,
                                            c_dp, c_dp]),
    "kls_gram_dcgs2_peer": (ctypes.c_int, [c_dp, i64, i64, i32, c_dp, c_dp, c_dp, c_dp, c_dp, sz,
                                           c_dp, i32, i32, i32, ctypes.c_uint64, c_dp, c_dp]),
    "kls_seg_rows": (ctypes.c_int, [c_dp, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
    "kls_seg_exports": (ctypes.c_int, [i32, i32, c_dp]),
    "kls_seg_combine": (ctypes.c_int, [c_dp, i32, i64, i32, c_dp, c_dp]),
    "kls_peer_signal": (ctypes.c_int, [c_dp, i32, i32, i32, ctypes.c_uint64, c_dp]),
    "kls_stencil7_peer": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, i64, i64, i64, c_dp, i32,
                                         ctypes.c_uint64, c_dp, c_dp]),
}

# entry points that launch no kernel (not counted as GPU launches)
_NO_LAUNCH = frozenset({"kls_version", "kls_last_error", "kls_device_sm_count", "kls_stream_sync",
                        "kls_host_device_ptr", "kls_workspace_bytes", "kls_peer_buffer_bytes",
                        "kls_lap7_nnz", "kls_mant5_nnz", "kls_ipc_handle_bytes",
                        "kls_peer_buffer_alloc", "kls_peer_buffer_open", "kls_peer_buffer_close",
                        "kls_peer_buffer_free", "kls_dcgs2_host_step", "kls_event_create",
                        "kls_seg_rows", "kls_seg_exports",
                        "kls_event_destroy", "kls_event_record", "kls_event_sync",
                        "kls_hessenberg_reduce", "kls_schur_sweeps", "kls_schur_swap",
                        "kls_schur_move_front", "kls_schur_eigenvectors",
                        "kls_dcgs2_run"})  # its kernels are counted by the caller


class KlsSegs(ctypes.Structure):
    """include/klsgpu.h KlsSegs: the rank-count-independent reduction layout."""

    _fields_ = [("m", i64), ("unit", i64), ("world", i32), ("rank", i32)]


class KlsOpDesc(ctypes.Structure):
    """include/klsgpu.h KlsOpDesc: an operator's apply as plain pointers."""

    _fields_ = [("kind", i32), ("width", i32), ("m", i64), ("n0", i64), ("n1", i64), ("n2", i64),
                ("p0", c_dp), ("p1", c_dp), ("p2", c_dp)]


class KlsHostBlas(ctypes.Structure):
    """include/klsgpu.h KlsHostBlas: numpy's own BLAS / LAPACK entry points."""

    _fields_ = [("ddot", c_dp), ("dgemv", c_dp), ("dgemm", c_dp), ("dgesv", c_dp),
                ("dgeqrf", c_dp), ("dorgqr", c_dp), ("zgemv", c_dp), ("zdotu_sub", c_dp)]


class KlsStepPlan(ctypes.Structure):
    """include/klsgpu.h KlsStepPlan (kls_dcgs2_queue_step)."""

    _fields_ = [("Q", c_dp), ("ldq", i64), ("m", i64), ("segs", KlsSegs), ("gdev", c_dp), ("cdev", c_dp),
                ("gout", c_dp * 2), ("ws", c_dp), ("ws_bytes", sz), ("stream", c_dp),
                ("event", c_dp * 2), ("divide", i32), ("qr", i32), ("op", KlsOpDesc)]


class KlsBeCol(ctypes.Structure):
    """include/klsgpu.h KlsBeCol (kls_dcgs2_queue_step_be)."""

    _fields_ = [("x", c_dp), ("xj", c_dp), ("q", i32), ("y", c_dp), ("b", c_dp), ("out", c_dp)]


class KlsRunState(ctypes.Structure):
    """include/klsgpu.h KlsRunState (kls_dcgs2_run)."""

    _fields_ = [("plan", ctypes.POINTER(KlsStepPlan)), ("w", c_dp * 2), ("wx", c_dp * 2),
                ("aw", c_dp * 2), ("gslot", c_dp * 2), ("h", c_dp), ("ldh", i64), ("k", c_dp),
                ("scratch", c_dp), ("ddot", c_dp), ("dgemv", c_dp), ("m", i64),
                ("capacity", i32)]


OP_ELL, OP_CSR, OP_STENCIL7, OP_DENSE = 1, 2, 3, 4

_lock = threading.Lock()
_lib = None
_launches = 0  # kernel-launching calls made through this binding


class KlsGpuError(RuntimeError):
    """A libklsgpu call returned a negative status."""


def load():
    """Load libklsgpu.so (building it first if nvcc is present and it is stale)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            try:
                from .csrc.build import build

                build()
            except Exception as exc:  # no toolkit on this host: report loudly
                raise RuntimeError(
                    f"libklsgpu.so is missing at {LIB_PATH} and could not be built: {exc}"
                ) from exc
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


_fns = {}


def call(name, *args):
    """Invoke a status-returning entry point; raise KlsGpuError on failure."""
    global _launches
    fn = _fns.get(name)
    if fn is None:
        fn = _fns[name] = getattr(load(), name)
    rc = fn(*args)
    if rc != 0:
        msg = load().kls_last_error().decode(errors="replace")
        raise KlsGpuError(f"{name} failed ({rc}): {msg}")
    if name not in _NO_LAUNCH:
        _launches += 1
    return rc


def count_launches(n):
    """Account for kernels a composite entry point launched beyond its first."""
    global _launches
    _launches += n


def launch_count():
    return _launches


def reset_launch_count():
    global _launches
    _launches = 0
