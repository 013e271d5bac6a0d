"""Host-side checks of the boundary (no GPU compute): libaci.so builds for sm_100a, loads, and
exports every symbol include/aci.h declares; the binding rejects bad calls loudly."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2604_00037_b200 import _build
    _build.build()
    import paper_2604_00037_b200 as aci
    return aci.load()


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "aci.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?(?:int|void|double|char|tt_t)\s*\*?\s*(\w+)\s*\(", txt, flags=re.M)
    return sorted(set(names))


def test_header_symbols_exported(lib):
    import paper_2604_00037_b200 as aci
    names = _header_symbols()
    assert set(names) == set(aci.EXPORTS), names
    nm = subprocess.run(["nm", "-D", "--defined-only", aci.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", nm, flags=re.M), n
        assert hasattr(lib, n)


def test_library_is_sm100a(lib):
    import paper_2604_00037_b200 as aci
    out = subprocess.run(["cuobjdump", "--list-elf", aci.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", aci.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA" in sass  # FP64 tensor-core path (mma.sync f64 -> DMMA.8x8x4)


def test_version_and_limits(lib):
    import paper_2604_00037_b200 as aci
    assert "sm_100a" in aci.version()
    rows, cols = aci.limits()
    assert rows >= 1024 and cols >= 1024


def test_no_device_fails_loudly(lib):
    """Without a GPU the compute calls return ACI_ERR_CUDA (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import numpy as np
    import paper_2604_00037_b200 as aci
    with pytest.raises(aci.AciError) as e:
        aci.TensorTrain.from_cores([np.ones((1, 2, 1)), np.ones((1, 2, 1))])
    assert "CUDA" in str(e.value)


def test_invalid_shapes_rejected(lib):
    import ctypes as C
    import numpy as np
    d = np.array([2, 2], np.int32)
    r = np.array([2, 1, 1], np.int32)  # boundary rank != 1
    h = C.c_void_p()
    c = np.ones(4)
    ptrs = (C.POINTER(C.c_double) * 2)(c.ctypes.data_as(C.POINTER(C.c_double)), c.ctypes.data_as(C.POINTER(C.c_double)))
    st = lib.tt_create(2, d.ctypes.data_as(C.POINTER(C.c_int)), r.ctypes.data_as(C.POINTER(C.c_int)), ptrs, C.byref(h))
    assert st == -1
    assert b"boundary" in lib.aci_last_error()


def test_c_example_builds_against_the_header():
    """examples/aci_example.c uses only include/aci.h and links against libaci.so."""
    from paper_2604_00037_b200 import _build
    exe = _build.build_example()
    assert os.path.exists(exe)
