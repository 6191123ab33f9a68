"""CPU-side checks of the C-ABI library: it builds, loads, exports every symbol
include/ifgf.h declares, and its host-only logic (partitioner, status strings,
argument validation) behaves.  No compute call needs a GPU here."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ifgf.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2010_02857_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ifgf_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("ifgf_plan", "ifgf_apply", "ifgf_plan_destroy", "ifgf_plan_stats", "ifgf_apply_host",
                 "ifgf_direct", "ifgf_partition", "ifgf_status_string", "ifgf_last_error_message"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (ifgf_\w+)", out))
    assert set(declared_functions()) <= exported


def test_library_is_sm100a_native(lib):
    """The fatbin carries sm_100a SASS (cuobjdump lists the ELF arch)."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib._name], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_binding_exports_match(lib):
    from paper_2010_02857_b200 import ifgf
    assert set(ifgf.EXPORTED) <= set(declared_functions())


def test_status_strings_and_version(lib):
    from paper_2010_02857_b200 import ifgf
    assert ifgf.version().startswith("ifgf-b200")
    lib.ifgf_status_string.restype = ctypes.c_char_p
    assert lib.ifgf_status_string(2) == b"IFGF_EDOMAIN"
    assert lib.ifgf_status_string(6) == b"IFGF_EINTERNAL"


def test_partition_contiguous_and_balanced():
    from paper_2010_02857_b200 import ifgf
    rng = np.random.default_rng(0)
    for R in (1, 2, 3, 4, 8):
        w = rng.uniform(0.5, 3.0, 10_000)
        b = ifgf.partition(w, R)
        assert b[0] == 0 and b[-1] == len(w) and np.all(np.diff(b) >= 0)
        loads = np.array([w[b[r]:b[r + 1]].sum() for r in range(R)])
        assert loads.max() - loads.min() <= 2 * w.max()
    assert list(ifgf.partition(np.ones(3), 5)) == [0, 0, 1, 2, 3, 3] or ifgf.partition(np.ones(3), 5)[-1] == 3
    b = ifgf.partition(np.zeros(0), 2)
    assert list(b) == [0, 0, 0]


def test_partition_rejects_bad_weights():
    from paper_2010_02857_b200 import ifgf
    with pytest.raises(ifgf.IfgfError):
        ifgf.partition(np.array([1.0, -1.0]), 2)
    with pytest.raises(ifgf.IfgfError):
        ifgf.partition(np.array([1.0, np.nan]), 2)


def test_plan_argument_validation_without_gpu(lib):
    """Invalid arguments are rejected before any device work (IFGF_EINVAL)."""
    from paper_2010_02857_b200 import ifgf
    h = ctypes.c_void_p()
    pts = np.zeros((4, 3))
    f = lib.ifgf_plan
    f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                  ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
    assert f(None, 4, 1.0, 3, 3, 5, None, ctypes.byref(h)) == 1
    assert f(pts.ctypes.data, 0, 1.0, 3, 3, 5, None, ctypes.byref(h)) == 1
    assert f(pts.ctypes.data, 4, -1.0, 3, 3, 5, None, ctypes.byref(h)) == 1
    assert f(pts.ctypes.data, 4, 1.0, 23, 3, 5, None, ctypes.byref(h)) == 1
    assert f(pts.ctypes.data, 4, 1.0, 3, 0, 5, None, ctypes.byref(h)) == 1
    assert f(pts.ctypes.data, 4, 1.0, 3, 3, 17, None, ctypes.byref(h)) == 1
    assert not h.value
    assert lib.ifgf_plan_destroy(None) == 0


def test_no_cpu_fallback_in_product_package():
    """The product package never imports the oracle (task rule ③)."""
    pkg = os.path.join(ROOT, "paper_2010_02857_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f
