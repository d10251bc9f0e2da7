"""CPU checks of the boundary: libmarconi.so loads, exports every symbol include/marconi.h
declares, fails loudly without a GPU, and the product path never touches the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

import __graft_entry__ as GE
from paper_2411_19379_b200 import marconi as M

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "marconi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mc_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    GE.build()
    lib = ctypes.CDLL(M.LIB_PATH)
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(M.EXPORTED)


def test_struct_sizes_match_header():
    assert ctypes.sizeof(M.mc_model) == 32
    assert ctypes.sizeof(M.mc_variant) == 56
    assert M.REQUEST_DTYPE.itemsize == 16
    assert M.SNAP_DTYPE.itemsize == 32
    assert ctypes.sizeof(M.mc_replay_args) == 128  # 11 pointers/u64 + 6 u32 (+pad), see include/marconi.h


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    arr = (M.mc_variant * 1)(M.make_variant(__import__("tracegen").MODEL_7B, 10 ** 12, 0))
    h = ctypes.c_void_p()
    rc = M.lib().mc_create(arr, 1, 1024, 0, ctypes.byref(h))
    assert rc != 0
    assert M.lib().mc_last_error()


def test_argument_validation_without_gpu():
    import tracegen as tg
    lib = M.lib()
    h = ctypes.c_void_p()
    bad = (M.mc_variant * 1)(M.make_variant(tg.Model(4, 24, 28, bytes_per_param=3), 10, 0))
    assert lib.mc_create(bad, 1, 1024, 0, ctypes.byref(h)) == -1          # MC_EINVAL
    zero = (M.mc_variant * 1)(M.make_variant(tg.Model(0, 4, 4), 10, 0))
    assert lib.mc_create(zero, 1, 1024, 0, ctypes.byref(h)) == -1
    ok = (M.mc_variant * 1)(M.make_variant(tg.MODEL_7B, 10, 0))
    assert lib.mc_create(ok, 1, 1000, 0, ctypes.byref(h)) == -1           # not a power of two


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2411_19379_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "liboracle" not in txt and "oracle.cpp" not in txt, f
    # and the oracle never includes product code
    txt = open(os.path.join(ROOT, "oracle", "oracle.cpp")).read()
    assert "marconi.h" not in txt and "replay.cuh" not in txt
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(import|from)\s+(paper_2411_19379_b200|\.\.)", txt, re.M), f
            assert "libmarconi" not in txt, f
