"""C-ABI library checks that need no GPU: the in-tree libgpfvm.so loads, exports
every symbol include/gpfvm.h declares, and validates problem descriptions."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import gpfvm_inputs as gi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2406_05020_b200.build import build
    build()
    from paper_2406_05020_b200 import _lib
    return _lib.load()


def test_exports_every_header_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "gpfvm.h")).read()
    names = set(re.findall(r"\b(gpfvm_[a-z_0-9]+)\s*\(", hdr))
    assert len(names) >= 12
    for n in sorted(names):
        assert hasattr(lib, n), n
    from paper_2406_05020_b200 import _lib
    assert names == set(_lib.EXPORTS), names ^ set(_lib.EXPORTS)


def test_sm100a_cubin_embedded():
    so = os.path.join(ROOT, "paper_2406_05020_b200", "libgpfvm.so")
    out = os.popen(f"cuobjdump --list-elf {so} 2>/dev/null").read()
    assert "sm_100a" in out


def test_dmma_in_sass():
    """The GEMM kernels really issue FP64 tensor-core instructions."""
    so = os.path.join(ROOT, "paper_2406_05020_b200", "libgpfvm.so")
    sass = os.popen(f"cuobjdump -sass -fun dgemm_dmma_kernel {so} 2>/dev/null | grep -c DMMA").read().strip()
    if not sass or sass == "0":
        sass = os.popen(f"cuobjdump -sass {so} 2>/dev/null | grep -c DMMA").read().strip()
    assert int(sass) > 0


def test_problem_create_and_size_on_cpu(lib):
    from paper_2406_05020_b200 import GpfvmProblem
    p = GpfvmProblem(gi.config0())
    assert p.N == 16 + 2 * 16 + 256
    p.close()


def test_invalid_descriptions_rejected(lib):
    from paper_2406_05020_b200 import GpfvmProblem
    from paper_2406_05020_b200._lib import GpfvmError
    bad = gi.config0()
    bad.blocks[3].terms[1].order = (0, 4)          # u_xxxx on Matérn-5/2 cells: order > q+1
    with pytest.raises(GpfvmError, match="smoothness"):
        GpfvmProblem(bad)
    bad = gi.config0()
    bad.blocks[0].sites[1].hi[3] = bad.blocks[0].sites[1].lo[3]  # empty interval
    with pytest.raises(GpfvmError, match="lo >= hi"):
        GpfvmProblem(bad)
    bad = gi.config0()
    bad.kernels[0][0].q = 5
    with pytest.raises(GpfvmError):
        GpfvmProblem(bad)


def test_last_error_is_set(lib):
    h = C.c_void_p()
    rc = lib.gpfvm_problem_create(None, 0, C.byref(h))
    assert rc != 0
    assert b"null" in lib.gpfvm_last_error()
