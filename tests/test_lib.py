"""The C-ABI library builds, loads without a GPU, and exports every entry
point include/klsgpu.h declares (no compute calls).  CPU only."""

import ctypes
import os
import re

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "klsgpu.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kls_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_path():
    names = declared()
    for must in ("kls_gram_dcgs2", "kls_dcgs2_update", "kls_mv_trans_mv", "kls_mv_times_mat_add_mv",
                 "kls_csr_spmv", "kls_stencil7", "kls_tsgemm_inplace"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2104_01253_b200 import _lib

    lib = _lib.load()
    handle = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared():
        assert hasattr(handle, name), name
    assert lib.kls_version() == 1


def test_binding_table_matches_header():
    from paper_2104_01253_b200 import _lib

    assert sorted(_lib.SIGNATURES) == declared()


def test_sm100a_cubin_embedded():
    """The fatbin carries sm_100a SASS (checked with cuobjdump when present)."""
    import shutil
    import subprocess

    from paper_2104_01253_b200 import _lib

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        return
    out = subprocess.run([exe, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
