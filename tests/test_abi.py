"""C-ABI library checks that need no GPU (-m "not gpu"): the library loads,
exports every symbol include/agr.h declares, and rejects calls cleanly when
no CUDA device is present (no compute calls are made here)."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

import paper_2503_01471_b200 as agr


def test_library_loads_and_exports_header_symbols():
    lib = agr.load()
    syms = agr.header_symbols()
    assert len(syms) >= 18
    for name in syms:
        assert hasattr(lib, name), name
    assert agr.abi_version() == 4


def test_exports_match_nm():
    """Every agr_* function in the header is a dynamic symbol of libagr.so."""
    out = subprocess.run(["nm", "-D", "--defined-only", agr.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(agr.header_symbols()) <= exported


def test_library_is_sm100a():
    """The fatbin carries sm_100a SASS (cuobjdump lists the arch)."""
    cuobjdump = "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump missing")
    out = subprocess.run([cuobjdump, "--list-elf", agr.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_create_rejects_bad_input_without_launching():
    """Argument errors return before any device work (EINVAL + message)."""
    lib = agr.load()
    h = ctypes.c_void_p()
    st = lib.agr_scene_create(0, None, 0, 1, None, None, ctypes.byref(h))
    assert st == agr.AGR_EINVAL and h.value is None
    assert "mesh" in agr.last_error()
    v = np.zeros((3, 3), np.float32)
    f = np.asarray([[0, 1, 5]], np.int32)  # index out of range
    m = (agr.agr_mesh * 1)(agr.agr_mesh(v.ctypes.data, 3, f.ctypes.data, 1))
    off = np.asarray([0, 0], np.int64)
    st = lib.agr_scene_create(0, m, 1, 1, off.ctypes.data, None, ctypes.byref(h))
    assert st == agr.AGR_EINVAL and "out of range" in agr.last_error()


def test_null_scene_calls_fail_cleanly():
    lib = agr.load()
    assert lib.agr_scene_destroy(None) == agr.AGR_OK
    assert lib.agr_build(None, None) == agr.AGR_EINVAL
    assert lib.agr_refit(None, None) == agr.AGR_EINVAL
    assert lib.agr_set_exact_mode(None, 1) == agr.AGR_EINVAL


def test_no_oracle_in_product_path():
    """The product package never references oracle/ (DESIGN.md §2)."""
    root = os.path.dirname(agr.__file__)
    for dirpath, _, files in os.walk(root):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in txt and "oracle.h" not in txt, fn
