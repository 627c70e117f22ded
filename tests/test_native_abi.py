"""The C-ABI library builds for sm_100a, loads without a GPU and exports
every entry point include/sbr200.h declares."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT, has_cuda


def _declared():
    text = open(os.path.join(ROOT, "include", "sbr200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(sbr_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = _declared()
    for n in ("sbr_solve", "sbr_trace_grid", "sbr_closest_hit", "sbr_bvh_build",
              "sbr_accumulate", "sbr_solve_shard", "sbr_finalize"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2604_09243_b200 import _build, _native
    _build.build()
    lib = _native.load_library()
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing
    assert set(_native.EXPORTED) == set(_declared())
    assert lib.sbr_abi_version() == 3


def test_sass_is_sm100a():
    from paper_2604_09243_b200 import _build
    path = _build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


@pytest.mark.skipif(has_cuda(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly():
    from paper_2604_09243_b200 import _native
    import paper_2604_09243_b200 as sbr
    from paper_2604_09243_b200 import meshgen
    with pytest.raises((_native.NativeUnavailable, _native.CudaError, sbr.ValidationError)):
        sbr.build(meshgen.plate_mesh())
