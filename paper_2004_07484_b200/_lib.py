"""ctypes binding of the C-ABI shared library (include/softsphere_b200.h).

There is NO CPU fallback: if the CUDA library is missing or a call fails, this raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SS_B200_LIB selects another build of the same library (kernel experiments); the default is the in-tree build
LIB_PATH = os.environ.get("SS_B200_LIB") or os.path.join(_HERE, "csrc", "libss_b200.so")

SS_OK = 0
SS_ERR_NULL, SS_ERR_DIMS, SS_ERR_PARAMS, SS_ERR_CAMERA = 1, 2, 3, 4
SS_ERR_WORKSPACE, SS_ERR_UNSUPPORTED, SS_ERR_CUDA = 5, 6, 7

FLAG_INVALID_INPUT = 1
FLAG_PAIR_OVERFLOW = 2
FLAG_LIST_FALLBACK = 4

OPT_STORE_BUFFER = 1
OPT_COLLECT_STATS = 2
OPT_NORMALIZE = 4
OPT_GATE = 8
OPT_CAMERA_GRADS = 16
OPT_ACCUMULATE = 32
OPT_REUSE_RECORDS = 64
OPT_SKIP_VALIDATE = 128
OPT_DETERMINISTIC = 256

MODE_PINHOLE, MODE_ORTHOGRAPHIC = 0, 1
MAX_FEATURE_DIM, MAX_TOP_K, TILE, MAX_CHUNK = 32, 64, 16, 256


class SsCamera(C.Structure):
    _fields_ = [("t", C.c_double * 3), ("R", C.c_double * 9), ("focal", C.c_double),
                ("sensor_w", C.c_double), ("near_", C.c_double), ("far_", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("mode", C.c_int32), ("pad_", C.c_int32)]


class SsDims(C.Structure):
    _fields_ = [("num_spheres", C.c_int64), ("max_pairs", C.c_int64), ("feature_dim", C.c_int32),
                ("width", C.c_int32), ("height", C.c_int32), ("top_k", C.c_int32)]


class SsBlend(C.Structure):
    _fields_ = [("gamma", C.c_double), ("eps", C.c_double), ("tau", C.c_double), ("tile", C.c_int32),
                ("chunk", C.c_int32), ("flags", C.c_uint32), ("pad_", C.c_uint32)]


_P = C.c_void_p


class SsForwardArgs(C.Structure):
    _fields_ = [("dims", SsDims), ("cam", SsCamera), ("blend", SsBlend),
                ("pos", _P), ("rad", _P), ("opa", _P), ("feat", _P), ("bg", _P),
                ("workspace", _P), ("workspace_bytes", C.c_size_t),
                ("image", _P), ("bg_weight", _P), ("ids", _P), ("z", _P), ("closeness", _P),
                ("log_denom", _P), ("rect", _P), ("on_sensor", _P), ("earliest", _P),
                ("proj_radius_px", _P)]


class SsBackwardArgs(C.Structure):
    _fields_ = [("dims", SsDims), ("cam", SsCamera), ("blend", SsBlend),
                ("pos", _P), ("rad", _P), ("opa", _P), ("feat", _P), ("bg", _P),
                ("workspace", _P), ("workspace_bytes", C.c_size_t),
                ("ids", _P), ("z", _P), ("closeness", _P), ("log_denom", _P), ("upstream", _P),
                ("d_pos", _P), ("d_rad", _P), ("d_opa", _P), ("d_feat", _P), ("pixel_count", _P),
                ("cam_grad", _P), ("det_workspace", _P), ("det_workspace_bytes", C.c_size_t)]


class SsFitStepArgs(C.Structure):
    _fields_ = [("num_spheres", C.c_int64), ("feature_dim", C.c_int32), ("pad_", C.c_int32),
                ("pos", _P), ("rad", _P), ("opa", _P), ("feat", _P),
                ("d_pos", _P), ("d_rad", _P), ("d_opa", _P), ("d_feat", _P),
                ("pixel_count", _P), ("visibility", _P),
                ("m_pos", _P), ("v_pos", _P), ("m_rad", _P), ("v_rad", _P), ("m_opa", _P), ("v_opa", _P),
                ("m_feat", _P), ("v_feat", _P),
                ("lr", C.c_double * 4), ("step", C.c_int64 * 4),
                ("beta1", C.c_double), ("beta2", C.c_double), ("adam_eps", C.c_double),
                ("radius_min", C.c_double), ("lambda_od", C.c_double), ("cam", SsCamera), ("energy", _P)]


class SsColumn(C.Structure):
    _fields_ = [("src", _P), ("dst", _P), ("row_bytes", C.c_int64), ("dst_stride_bytes", C.c_int64)]


class SsLight(C.Structure):
    _fields_ = [("direction", C.c_double * 3), ("intensity", C.c_double), ("ambient", C.c_double)]


class SsStatus(C.Structure):
    _fields_ = [("flags", C.c_int64), ("spheres_on_sensor", C.c_int64), ("num_pairs", C.c_int64),
                ("candidates_tested", C.c_int64), ("hits_blended", C.c_int64),
                ("pixels_early_stopped", C.c_int64), ("first_invalid", C.c_int64),
                ("reserved", C.c_int64 * 9)]


EXPORTS = ("ss_abi_version", "ss_status_string", "ss_last_cuda_error", "ss_workspace_bytes", "ss_workspace_init",
           "ss_forward", "ss_forward_banded", "ss_band_rows", "ss_backward", "ss_deterministic_workspace_bytes", "ss_read_status", "ss_photometric_loss", "ss_fit_step", "ss_adam_flat", "ss_debug_tile_lists", "ss_launch_count",
           "ss_prune_mask", "ss_prune_mask_f64", "ss_subdivide_f64", "ss_mask_nonzero_i32", "ss_compact_workspace_bytes", "ss_compact_rows", "ss_subdivide",
           "ss_psc1_unpack", "ss_psc1_pack", "ss_convert_f64_f32", "ss_convert_f32_f64",
           "ss_shade_identity", "ss_shade_identity_backward", "ss_shade_diffuse", "ss_shade_diffuse_backward",
           "ss_shade_linear", "ss_shade_linear_backward", "ss_view_directions",
           "ss_profile_enable", "ss_profile_enable_mask", "ss_profile_collect", "ss_profile_captured_reset",
           "ss_profile_collect_captured", "ss_profile_kernel_count", "ss_profile_kernel_name")

_lib = None


class NativeLibraryError(RuntimeError):
    """The sm_100a extension is missing or failed; there is no fallback path."""


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} not found: build it with `python -m paper_2004_07484_b200.build` "
            "(nvcc, sm_100a). This package has no CPU or PyTorch fallback.")
    lib = C.CDLL(LIB_PATH)
    lib.ss_abi_version.restype = C.c_int
    lib.ss_status_string.restype = C.c_char_p
    lib.ss_status_string.argtypes = [C.c_int]
    lib.ss_last_cuda_error.restype = C.c_char_p
    lib.ss_workspace_bytes.restype = C.c_int
    lib.ss_workspace_bytes.argtypes = [C.POINTER(SsDims), C.POINTER(C.c_size_t)]
    lib.ss_workspace_init.restype = C.c_int
    lib.ss_workspace_init.argtypes = [C.POINTER(SsDims), C.c_void_p, C.c_size_t, C.c_void_p]
    lib.ss_forward.restype = C.c_int
    lib.ss_forward.argtypes = [C.POINTER(SsForwardArgs), C.c_void_p]
    lib.ss_forward_banded.restype = C.c_int
    lib.ss_forward_banded.argtypes = [C.POINTER(SsForwardArgs), C.c_int, C.POINTER(C.c_void_p), C.c_void_p]
    lib.ss_band_rows.restype = C.c_int
    lib.ss_band_rows.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.ss_backward.restype = C.c_int
    lib.ss_backward.argtypes = [C.POINTER(SsBackwardArgs), C.c_void_p]
    lib.ss_deterministic_workspace_bytes.restype = C.c_int
    lib.ss_deterministic_workspace_bytes.argtypes = [C.POINTER(SsDims), C.POINTER(C.c_size_t)]
    lib.ss_photometric_loss.restype = C.c_int
    lib.ss_photometric_loss.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
    lib.ss_fit_step.restype = C.c_int
    lib.ss_fit_step.argtypes = [C.POINTER(SsFitStepArgs), C.c_void_p]
    lib.ss_adam_flat.restype = C.c_int
    lib.ss_adam_flat.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_double, C.c_double,
                                 C.c_double, C.c_double, C.c_int64, C.c_int, C.c_double, C.c_void_p]
    V, I64, I32, D = C.c_void_p, C.c_int64, C.c_int32, C.c_double
    for name, argtypes in (
            ("ss_prune_mask", [V, V, V, V, I64, I32, D, D, V, V]),
            ("ss_prune_mask_f64", [V, V, V, V, I64, I32, D, D, V, V]),
            ("ss_subdivide_f64", [V, V, V, V, I64, I32, D, V, V, V, V, V]),
            ("ss_mask_nonzero_i32", [V, I64, V, V]),
            ("ss_compact_workspace_bytes", [I64, C.POINTER(C.c_size_t)]),
            ("ss_compact_rows", [V, I64, C.POINTER(SsColumn), I32, V, C.c_size_t, V, V]),
            ("ss_subdivide", [V, V, V, V, I64, I32, D, V, V, V, V, V]),
            ("ss_psc1_unpack", [V, I64, I32, V, V, V, V, V]),
            ("ss_psc1_pack", [V, V, V, V, I64, I32, V, V]),
            ("ss_convert_f64_f32", [V, V, I64, V]),
            ("ss_convert_f32_f64", [V, V, I64, V]),
            ("ss_shade_identity", [V, I64, V, V]),
            ("ss_shade_identity_backward", [V, V, I64, V, V]),
            ("ss_shade_diffuse", [V, I64, C.POINTER(SsLight), I32, V, V]),
            ("ss_shade_diffuse_backward", [V, V, I64, C.POINTER(SsLight), I32, V, V]),
            ("ss_shade_linear", [V, V, I64, I32, V, V, V, V]),
            ("ss_shade_linear_backward", [V, V, I64, I32, V, V, V, V, V, V, V]),
            ("ss_view_directions", [C.POINTER(SsCamera), V, V])):
        fn = getattr(lib, name)
        fn.restype = C.c_int
        fn.argtypes = argtypes
    lib.ss_read_status.restype = C.c_int
    lib.ss_read_status.argtypes = [C.c_void_p, C.POINTER(SsStatus), C.c_void_p]
    lib.ss_debug_tile_lists.restype = C.c_int
    lib.ss_debug_tile_lists.argtypes = [C.POINTER(SsDims), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.ss_launch_count.restype = C.c_int64
    lib.ss_profile_enable.restype = None
    lib.ss_profile_enable.argtypes = [C.c_int]
    lib.ss_profile_enable_mask.restype = None
    lib.ss_profile_enable_mask.argtypes = [C.c_uint]
    lib.ss_profile_collect.restype = C.c_int
    lib.ss_profile_collect.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int]
    lib.ss_profile_captured_reset.restype = None
    lib.ss_profile_collect_captured.restype = C.c_int
    lib.ss_profile_collect_captured.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int]
    lib.ss_profile_kernel_count.restype = C.c_int
    lib.ss_profile_kernel_name.restype = C.c_char_p
    lib.ss_profile_kernel_name.argtypes = [C.c_int]
    if lib.ss_abi_version() != 2:
        raise NativeLibraryError("libss_b200.so ABI version mismatch")
    _lib = lib
    return lib


def status_string(code: int) -> str:
    lib = load()
    msg = lib.ss_status_string(code).decode()
    if code == SS_ERR_CUDA:
        msg += ": " + lib.ss_last_cuda_error().decode()
    return msg


def launch_count() -> int:
    return int(load().ss_launch_count())


def profile_enable(on: bool) -> None:
    load().ss_profile_enable(1 if on else 0)


def profile_enable_only(names) -> None:
    """Time only the named kernels (e.g. ['k_raster'])."""
    lib = load()
    n = lib.ss_profile_kernel_count()
    mask = 0
    for i in range(n):
        if lib.ss_profile_kernel_name(i).decode() in names:
            mask |= 1 << i
    lib.ss_profile_enable_mask(mask)


def profile_collect() -> dict:
    """{kernel name: (total ms, launches)} since the last enable/collect (synchronises the device)."""
    lib = load()
    n = lib.ss_profile_kernel_count()
    ms = (C.c_double * n)()
    cnt = (C.c_int64 * n)()
    rc = lib.ss_profile_collect(ms, cnt, n)
    if rc != SS_OK:
        raise NativeLibraryError(status_string(rc))
    return {lib.ss_profile_kernel_name(i).decode(): (float(ms[i]), int(cnt[i])) for i in range(n)}


def profile_captured_reset() -> None:
    load().ss_profile_captured_reset()


def profile_collect_captured() -> dict:
    """{kernel: (ms of the most recent graph replay, launches)} for launches captured into a CUDA graph while
    profiling was enabled (synchronises the device)."""
    lib = load()
    n = lib.ss_profile_kernel_count()
    ms = (C.c_double * n)()
    cnt = (C.c_int64 * n)()
    rc = lib.ss_profile_collect_captured(ms, cnt, n)
    if rc != SS_OK:
        raise NativeLibraryError(f"ss_profile_collect_captured failed: {rc}")
    return {lib.ss_profile_kernel_name(i).decode(): (float(ms[i]), int(cnt[i])) for i in range(n)}
