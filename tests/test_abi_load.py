"""CPU-side checks of the boundary: libcyclicot.so builds for sm_100a, loads without a GPU, exports every
function declared in include/*.h, and its non-compute entry points answer. No kernel is launched."""
import ctypes
import glob
import os
import re
import subprocess

import pytest

import paper_2311_13147_b200 as cot
from paper_2311_13147_b200 import build as _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        src = re.sub(r"//[^\n]*", "", src)
        for mt in re.finditer(r"^[A-Za-z_][\w\s\*]*?\b([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M):
            name = mt.group(1)
            if name not in ("if", "while", "for", "sizeof", "defined"):
                names.append(name)
    return sorted(set(names))


@pytest.fixture(scope="module")
def L():
    _build.build()
    return cot.lib()


def test_header_declares_the_paper_entry_points():
    names = _declared_functions()
    for required in ("clot_aggregate", "clot_expand", "cerot_solve", "cerot_iter", "cerot_plan",
                     "cot_workspace_bytes", "cot_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol(L):
    names = _declared_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(L, name), f"libcyclicot.so does not export {name}"


def test_abi_version_and_workspace_sizing(L):
    assert L.cot_abi_version() == 1
    w = L.cot_workspace_bytes(1, 64, 1024, cot.COT_F32)
    # G (4 MiB) + argmin (4 MiB) + two fp64 partial buffers + state
    assert w > 8 * 1024 * 1024
    assert L.cot_workspace_bytes(0, 1, 1, cot.COT_F32) == 0


def test_argument_errors_without_gpu(L):
    # shape/dtype validation happens before any CUDA call
    assert L.clot_aggregate(None, 1, 0, 4, 0, None, None, None, None) == -1
    assert b"B, n, m" in L.cot_last_error()
    assert L.clot_expand(None, None, 1, 2, 4, 7, None, None) == -1
    assert L.cerot_iter(None, None, None, None, 1, 2, 4, 0, None, 1, 0.0, 1, 0, None, None, None, 0, None) == -1


def test_sass_is_sm100a_and_uses_bulk_copies(L):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", cot.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", cot.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "MUFU.EX2" in sass           # the Gibbs-kernel exponentials on the SFU
    assert "UBLKCP" in sass             # TMA bulk copies (expand stores)


def test_expand_path_query(L):
    """cot_expand_path reports the kernel clot_expand selects (no device work): the C3/C4 shapes take the TMA
    bulk-store kernel, C5 the whole-row kernel, ragged m the vector-store kernel."""
    assert L.cot_expand_path(4, 1024, cot.COT_F32) == 1
    assert L.cot_expand_path(64, 1024, cot.COT_F32) == 1
    assert L.cot_expand_path(16, 128, cot.COT_F32) == 2
    assert L.cot_expand_path(4, 130, cot.COT_F32) == 0
    assert L.cot_expand_path(0, 4, cot.COT_F32) == -1


def test_deterministic_flag_rejected_by_split_entry_points(L):
    """COT_DETERMINISTIC on the rows-only / NCCL entry points is an argument error before any device work."""
    det = cot.COT_DETERMINISTIC
    assert L.cerot_rows(None, None, None, 1, 4, 16, 0, None, det, None, None, None, 0, 0, None) == -1
    assert b"COT_DETERMINISTIC" in L.cot_last_error()
    assert L.cerot_iter_sharded(None, None, None, None, 4, 16, 0, 8, 0, None, 1, 0.0, 1, det, None, None, None, 0,
                                None, None) == -1
    assert b"COT_DETERMINISTIC" in L.cot_last_error()
