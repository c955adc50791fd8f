"""CPU-side checks of the C ABI boundary: the library loads, exports every symbol that
include/lattice_b200.h declares, and host-only contract checks (no GPU compute) behave like
the reference's UsageError paths (datasets.hpp:60-84)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "lattice_b200.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lattice_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2512_09200_b200 as L
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L.lib, s), s
    assert set(L.EXPORTS) >= set(syms)


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2512_09200_b200", "liblattice_b200.so")
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_zipper_validate_contract():
    import paper_2512_09200_b200 as L

    def v(d, p):
        d = np.array(d, np.int64)
        p = np.array(p, np.float64)
        return L.lib.lattice_zipper_validate(len(d), ctypes.c_void_p(d.ctypes.data),
                                             ctypes.c_void_p(p.ctypes.data))
    assert v([1, 2], [0.5, 0.5]) == L.OK
    assert v([], []) == L.USAGE
    assert v([2, 2], [0.5, 0.5]) == L.USAGE          # not strictly increasing
    assert v([0, 2], [0.5, 0.5]) == L.USAGE          # non-positive
    assert v([1, 2], [0.5, 0.6]) == L.USAGE          # sum != 1
    assert v([1, 2], [1.5, -0.5]) == L.USAGE         # negative
    assert v([1, 2], [float("nan"), 1.0]) == L.USAGE
    assert v([1, 2], [0.5, 0.5 + 5e-10]) == L.OK     # |sum-1| <= 1e-9
    assert v([1, 2], [0.5, 0.6]) == L.USAGE and b"sum to 1" in L.lib.lattice_last_error()


def test_usage_errors_raise_without_gpu():
    import paper_2512_09200_b200 as L
    a = L.BagArgs()
    a.features, a.batch, a.dim, a.table_dtype, a.out_dtype = 1, 1, 128, 7, 0
    assert L.lib.lattice_embedding_bag(ctypes.byref(a), None) == L.USAGE
    with pytest.raises(L.UsageError):
        L.check(L.USAGE)
