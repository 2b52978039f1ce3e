"""The C-ABI library: it loads, exports every symbol include/sa.h declares, and its host-side
argument checks behave as documented (no compute calls: these run without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_1303_3692_b200 as sa

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "sa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sa_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert header_functions() == sorted(sa.EXPORTED_SYMBOLS)


def test_library_exports_every_symbol():
    L = sa.lib()
    for name in header_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", sa.LIB_PATH], capture_output=True, text=True).stdout
    for name in header_functions():
        assert re.search(rf"\bT {name}$", out, flags=re.M), name


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", sa.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_string():
    assert sa.lib().sa_version() >= 100
    assert isinstance(sa.lib().sa_last_error(), bytes)


def _create(ref, n, k=0):
    h = ctypes.c_void_p()
    opts = sa._Opts(-1, k, 0, 0)
    rc = sa.lib().sa_index_create(ref, n, ctypes.byref(opts), ctypes.byref(h))
    return rc, h


def test_create_argument_errors_before_any_device_work():
    buf = ctypes.create_string_buffer(b"ACGT")
    assert _create(buf, 0)[0] == sa.SA_EEMPTY
    assert _create(None, 4)[0] == sa.SA_EINVAL
    assert _create(buf, 1 << 32)[0] == sa.SA_ETOOLONG
    assert b"2^32" in sa.lib().sa_last_error()
    assert _create(buf, 4, k=17)[0] == sa.SA_EINVAL
    opts = sa._Opts(-1, 0, 0, 0)
    assert sa.lib().sa_index_create(buf, 4, ctypes.byref(opts), None) == sa.SA_EINVAL


def test_no_device_is_a_loud_error():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(sa.SAError) as e:
        sa.Index("ACGTACGT")
    assert e.value.code == sa.SA_ECUDA


def test_match_argument_errors():
    L = sa.lib()
    # NULL index
    assert L.sa_match_batch(None, None, None, 0, 1, 0, None, None, None, 0, 0, None) == sa.SA_EINVAL
    assert L.sa_match_order(None, None, None, 0, 1, 0, 0, None, None, None, None, 0, None) == sa.SA_EINVAL
    ws = ctypes.c_size_t()
    assert L.sa_locate_workspace_size(10, ctypes.byref(ws)) in (sa.SA_OK, sa.SA_ECUDA)  # CUB asks the device
    assert L.sa_locate_workspace_size(10, None) == sa.SA_EINVAL
    assert L.sa_locate(None, None, None, 0, None, None) == sa.SA_EINVAL
