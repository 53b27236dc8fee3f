"""CPU checks of the boundary: libseed.so builds for sm_100a, loads, and exports
every symbol include/seed.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "seed.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(seed_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_exports_header_symbols():
    from paper_1910_06591_b200 import build as B
    lib_path = B.build()
    lib = ctypes.CDLL(lib_path)
    syms = declared_symbols()
    assert "seed_vtrace" in syms and "seed_learner_step" in syms and "seed_infer" in syms
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in seed.h but not exported"
    from paper_1910_06591_b200 import _lib
    assert set(_lib.EXPORTED) == set(syms), set(_lib.EXPORTED) ^ set(syms)


def test_sass_is_sm100a_with_tcgen05():
    from paper_1910_06591_b200 import build as B
    lib_path = B.build()
    out = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out or "SM100" in out.upper()
    assert "UTCHMMA" in out, "tcgen05.mma (UTCHMMA) missing from the SASS"
    assert "LDTM" in out, "tcgen05.ld (LDTM) missing from the SASS"


def test_host_argument_errors_without_gpu():
    """Host-checkable errors return synchronously, before any CUDA call."""
    import paper_1910_06591_b200 as S
    lib = S.load()
    assert lib.seed_abi_version() == 1
    assert lib.seed_status_string(2) == b"unsupported shape"
    # T < 1 -> SEED_E_SHAPE; c_bar > rho_bar -> SEED_E_ARG
    p = ctypes.c_void_p(16)
    assert lib.seed_vtrace(0, 4, p, p, p, p, p, p, 1.0, 1.0, 1.0, p, p, None, None) == 2
    assert lib.seed_vtrace(4, 4, p, p, p, p, p, p, 0.5, 1.0, 1.0, p, p, None, None) == 1
    assert lib.seed_vtrace(4, 4, p, p, p, p, p, p, 1.0, 1.0, 1.5, p, p, None, None) == 1
