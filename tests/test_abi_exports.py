"""CPU: the C-ABI library loads, exports every symbol include/softsphere_b200.h declares, and the
ctypes mirrors of the POD structs have the C layout.  No compute calls (no GPU here)."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from helpers import ROOT
from paper_2004_07484_b200 import _lib, build

HEADER = os.path.join(ROOT, "include", "softsphere_b200.h")


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_expected_entry_points():
    names = declared_functions()
    for required in ("ss_forward", "ss_backward", "ss_workspace_bytes", "ss_read_status", "ss_status_string",
                     "ss_debug_tile_lists", "ss_launch_count"):
        assert required in names
    assert set(names) == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), f"{name} declared in the header but not exported"


def test_abi_version_and_status_strings(lib):
    assert lib.ss_abi_version() == 2
    assert _lib.status_string(_lib.SS_OK) == "ok"
    assert "workspace" in _lib.status_string(_lib.SS_ERR_WORKSPACE)


def test_struct_layouts_match_the_c_header(tmp_path):
    prog = tmp_path / "sizes.c"
    prog.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "softsphere_b200.h"\n'
        'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(SsCamera), sizeof(SsDims), '
        'sizeof(SsBlend), sizeof(SsForwardArgs), sizeof(SsBackwardArgs), sizeof(SsStatus), '
        'offsetof(SsForwardArgs, workspace), offsetof(SsBackwardArgs, cam_grad));return 0;}\n')
    exe = tmp_path / "sizes"
    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    subprocess.run([cc, "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [C.sizeof(_lib.SsCamera), C.sizeof(_lib.SsDims), C.sizeof(_lib.SsBlend), C.sizeof(_lib.SsForwardArgs),
            C.sizeof(_lib.SsBackwardArgs), C.sizeof(_lib.SsStatus), _lib.SsForwardArgs.workspace.offset,
            _lib.SsBackwardArgs.cam_grad.offset]
    assert got == want


def test_workspace_bytes_and_argument_checks(lib):
    n = C.c_size_t()
    d = _lib.SsDims(1_000_000, 4_000_000, 3, 1024, 1024, 5)
    assert lib.ss_workspace_bytes(C.byref(d), C.byref(n)) == _lib.SS_OK
    assert 100e6 < n.value < 400e6
    bad = _lib.SsDims(10, 100, 0, 64, 64, 5)  # d = 0
    assert lib.ss_workspace_bytes(C.byref(bad), C.byref(n)) == _lib.SS_ERR_DIMS
    bad = _lib.SsDims(10, 100, 3, 64, 64, 0)  # K = 0 (blend.py:44)
    assert lib.ss_workspace_bytes(C.byref(bad), C.byref(n)) == _lib.SS_ERR_PARAMS
    # host-side argument validation happens before any CUDA call, so it is testable without a GPU
    a = _lib.SsForwardArgs()
    a.dims = _lib.SsDims(0, 16, 3, 32, 32, 5)
    a.cam.width, a.cam.height, a.cam.focal, a.cam.sensor_w, a.cam.near_, a.cam.far_ = 32, 32, 5.0, 2.0, 0.1, 45.0
    a.blend = _lib.SsBlend(0.1, -1.0, 0.0, 16, 256, 0, 0)  # eps <= 0 (blend.py:40)
    assert lib.ss_forward(C.byref(a), None) == _lib.SS_ERR_PARAMS
    a.blend = _lib.SsBlend(0.1, 0.01, 1.0, 16, 256, 0, 0)  # tau = 1 (blend.py:42)
    assert lib.ss_forward(C.byref(a), None) == _lib.SS_ERR_PARAMS
    a.blend = _lib.SsBlend(0.1, 0.01, 0.0, 8, 256, 0, 0)  # tile != 16
    assert lib.ss_forward(C.byref(a), None) == _lib.SS_ERR_UNSUPPORTED
    a.blend = _lib.SsBlend(0.1, 0.01, 0.0, 16, 256, 0, 0)
    a.cam.far_ = 0.05  # near >= far (camera.py:172)
    assert lib.ss_forward(C.byref(a), None) == _lib.SS_ERR_CAMERA
    a.cam.far_ = 45.0
    assert lib.ss_forward(C.byref(a), None) == _lib.SS_ERR_NULL  # no buffers given


def test_banded_forward_argument_checks_and_band_rows(lib):
    """ss_forward_banded / ss_band_rows: host-side checks and the band geometry (no CUDA call is reached)."""
    a = _lib.SsForwardArgs()
    a.dims = _lib.SsDims(0, 16, 3, 32, 32, 5)
    a.cam.width, a.cam.height, a.cam.focal, a.cam.sensor_w, a.cam.near_, a.cam.far_ = 32, 32, 5.0, 2.0, 0.1, 45.0
    a.blend = _lib.SsBlend(0.1, 0.01, 0.0, 16, 256, 0, 0)
    ev = (C.c_void_p * 2)(C.c_void_p(1), C.c_void_p(2))
    assert lib.ss_forward_banded(C.byref(a), 0, ev, None) == _lib.SS_ERR_PARAMS
    assert lib.ss_forward_banded(C.byref(a), 17, ev, None) == _lib.SS_ERR_PARAMS  # SS_MAX_BANDS = 16
    assert lib.ss_forward_banded(C.byref(a), 2, None, None) == _lib.SS_ERR_NULL
    missing = (C.c_void_p * 2)(C.c_void_p(1), C.c_void_p(None))
    assert lib.ss_forward_banded(C.byref(a), 2, missing, None) == _lib.SS_ERR_NULL
    assert lib.ss_forward_banded(C.byref(a), 2, ev, None) == _lib.SS_ERR_NULL  # (no buffers given, like ss_forward)
    r0, r1 = C.c_int(), C.c_int()
    # bands are whole tile rows, contiguous, top to bottom, and cover the image: 1080 rows = 68 tile rows
    for height, n in ((1080, 4), (100, 3), (16, 16), (1, 1), (1024, 2)):
        prev = 0
        for b in range(n):
            assert lib.ss_band_rows(height, n, b, C.byref(r0), C.byref(r1)) == _lib.SS_OK
            assert r0.value == prev and r0.value <= r1.value <= height
            assert r0.value % 16 == 0 or r0.value == height
            prev = r1.value
        assert prev == height
    assert lib.ss_band_rows(64, 2, 2, C.byref(r0), C.byref(r1)) == _lib.SS_ERR_PARAMS
    assert lib.ss_band_rows(64, 0, 0, C.byref(r0), C.byref(r1)) == _lib.SS_ERR_PARAMS
    assert lib.ss_band_rows(64, 2, 0, None, C.byref(r1)) == _lib.SS_ERR_NULL
