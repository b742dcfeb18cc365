"""C-ABI boundary checks that need no GPU: the library builds/loads, exports
every symbol include/fftpde.h declares, and validates arguments synchronously
(plan creation and status codes touch no device)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fftpde.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2412_12308_b200 import build, fftpde
    build.build()
    return fftpde.load_library()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fftpde_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ["fftpde_plan_2d", "fftpde_forward", "fftpde_inverse", "fftpde_poisson",
                     "fftpde_diffuse", "fftpde_wave_step", "fftpde_poisson_batched",
                     "fftpde_workspace_size", "fftpde_set_workspace", "fftpde_set_stream"]:
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2412_12308_b200 import fftpde
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert sorted(fftpde.EXPORTS) == declared_functions()


def plan(lib, nx, ny, batch=1, dtype=1, Lx=1.0, Ly=1.0):
    h = ctypes.c_void_p()
    st = lib.fftpde_plan_2d(ctypes.byref(h), nx, ny, batch, dtype, Lx, Ly, 0)
    return st, h


def test_plan_validation(lib):
    from paper_2412_12308_b200 import fftpde as F
    assert plan(lib, 64, 64)[0] == F.OK
    assert plan(lib, 0, 64)[0] == F.ERR_EMPTY
    assert plan(lib, 64, 64, batch=0)[0] == F.ERR_EMPTY
    assert plan(lib, 12, 64)[0] == F.ERR_NOT_POW2_X          # offending axis named
    assert plan(lib, 64, 48)[0] == F.ERR_NOT_POW2_Y
    assert plan(lib, 65536, 64)[0] == F.ERR_UNSUPPORTED          # longer than 2^15
    assert plan(lib, 32768, 64)[0] == F.OK                       # two-level row pass
    assert plan(lib, 4, 16384)[0] == F.ERR_UNSUPPORTED           # long columns need 8 columns (c128)
    assert plan(lib, 8, 16384)[0] == F.OK
    assert plan(lib, 64, 64, dtype=7)[0] == F.ERR_INVALID_ARG
    assert plan(lib, 64, 64, Lx=0.0)[0] == F.ERR_INVALID_ARG
    assert plan(lib, 64, 64, Ly=float("nan"))[0] == F.ERR_INVALID_ARG
    assert plan(lib, 64, 64, Lx=-1.0)[0] == F.ERR_INVALID_ARG
    st, h = plan(lib, 3, 64)
    assert h.value is None                                     # *plan NULL on error


def test_workspace_size_and_unset_workspace(lib):
    from paper_2412_12308_b200 import fftpde as F
    st, h = plan(lib, 256, 128, batch=4, dtype=F.C128)
    assert st == F.OK
    ws = lib.fftpde_workspace_size(h)
    # twiddles (nx+ny complex) + k^2 and diffusion tables per axis + 3 wave quadrant tables
    assert ws >= (256 + 128) * 16 + 2 * (256 + 128) * 8 + 3 * 129 * 65 * 8
    st32, h32 = plan(lib, 256, 128, batch=4, dtype=F.C64)
    assert lib.fftpde_workspace_size(h32) < ws
    # compute calls before a workspace is set fail synchronously, nothing enqueued
    buf = ctypes.create_string_buffer(256 * 128 * 16 + 64)
    ptr = (ctypes.addressof(buf) + 15) & ~15
    assert lib.fftpde_poisson(h, ptr, ptr) == F.ERR_WORKSPACE
    assert lib.fftpde_set_workspace(h, None, 0) == F.ERR_INVALID_ARG
    assert lib.fftpde_set_workspace(h, 256, ws - 1) == F.ERR_WORKSPACE
    assert lib.fftpde_launch_count(h) == 0
    for p in (h, h32):
        assert lib.fftpde_destroy(p) == F.OK


def test_status_strings(lib):
    from paper_2412_12308_b200 import fftpde as F
    assert F.status_string(F.ERR_NOT_POW2_X).startswith("nx is not a power of two")
    assert F.status_string(F.OK) == "ok"
    assert F.status_string(99) == "unknown status"


def test_product_package_does_not_reference_the_oracle():
    # the product path must never route through oracle/ 
    pkg = os.path.join(ROOT, "paper_2412_12308_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                bad = re.findall(r"(?:from|import)\s+oracle|liboracle|fftpde_oracle", text)
                assert not bad, (os.path.join(dirpath, f), bad)


def test_sharded_plan_validation(lib):
    # argument checks happen before NCCL or the device is touched
    from paper_2412_12308_b200 import fftpde as F
    h = ctypes.c_void_p()
    uid = ctypes.create_string_buffer(128)
    assert lib.fftpde_plan_2d_sharded(ctypes.byref(h), 64, 64, 1, 1.0, 1.0, 0, uid, 2, 2) == F.ERR_INVALID_ARG
    assert lib.fftpde_plan_2d_sharded(ctypes.byref(h), 64, 64, 1, 1.0, 1.0, 0, None, 0, 1) == F.ERR_INVALID_ARG
    assert lib.fftpde_plan_2d_sharded(ctypes.byref(h), 64, 64, 1, 1.0, 1.0, 0, uid, 0, 0) == F.ERR_INVALID_ARG
    assert lib.fftpde_nccl_unique_id(None) == F.ERR_INVALID_ARG
    assert h.value is None


def test_sharded_loopback_argument_forms(lib):
    from paper_2412_12308_b200 import fftpde as F
    h = ctypes.c_void_p()
    # loopback needs rank == FFTPDE_SHARDED_LOOPBACK and nranks >= 1
    assert lib.fftpde_plan_2d_sharded(ctypes.byref(h), 64, 64, 1, 1.0, 1.0, 0, None, -1, 0) == F.ERR_INVALID_ARG
    assert lib.fftpde_plan_3d_sharded(ctypes.byref(h), 64, 64, 8, 1, 1.0, 1.0, 1.0, 0, None, 1, 2) == F.ERR_INVALID_ARG
    assert F.SHARDED_LOOPBACK == -1
