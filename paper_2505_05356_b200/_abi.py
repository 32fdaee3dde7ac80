"""ctypes binding of the C ABI in include/tsb.h (paper_2505_05356_b200/lib/libtsb.so).

The shared library is the product: hand-written sm_100a kernels behind a plain
C interface.  There is no CPU fallback -- importing this module without the
built library raises, and every entry point that touches the GPU returns an
error (raised here as TsbError) when no sm_100 device is present.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# TSB_LIB: an alternative in-tree build of the same ABI (A/B timing experiments)
LIB_PATH = Path(os.environ.get("TSB_LIB") or Path(__file__).resolve().parent / "lib" / "libtsb.so")
HEADER_PATH = Path(__file__).resolve().parent.parent / "include" / "tsb.h"

TSB_OK, TSB_ERR_INVALID, TSB_ERR_CUDA, TSB_ERR_NOMEM, TSB_ERR_UNSUPPORTED, TSB_ERR_NCCL = range(6)
TSB_HOST, TSB_DEVICE = 0, 1
CH_QUAD, CH_DEPTH, CH_WEIGHT, CH_TRANSM, CH_COUNTS, CH_FULL_LISTS = 1, 2, 4, 8, 16, 32
CH_PHASOR, CH_DISTORTION, CH_COLOR, CH_FLOW, CH_EXACT, CH_DETERMINISTIC = 64, 128, 256, 512, 1024, 2048
(OUT_QUAD, OUT_DEPTH_RAW, OUT_DEPTH, OUT_WEIGHT, OUT_TRANSM, OUT_N_CONTRIB, OUT_N_PROCESSED,
 OUT_D_QUAD, OUT_PHASOR, OUT_DISTORTION, OUT_COLOR, OUT_MOTION_FWD_ACC, OUT_MOTION_BWD_ACC, OUT_FLOW_FWD,
 OUT_FLOW_BWD, OUT_FLOW_VALID, OUT_D_MOTION_FWD_ACC, OUT_D_MOTION_BWD_ACC, OUT_F64, OUT_EXT_F64) = range(20)


STAGES = ["preprocess", "depth_sort", "scan", "binning", "tile_sort", "ranges", "raster_fwd", "fixup", "loss",
          "raster_bwd", "chain", "adam", "allreduce", "bin_count", "bin_emit"]


class TsbError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class Camera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("near_plane", C.c_double),
                ("far_plane", C.c_double), ("R", C.c_double * 9), ("t", C.c_double * 3)]


class RenderOptions(C.Structure):
    _fields_ = [("alpha_threshold", C.c_double), ("transmittance_floor", C.c_double), ("dilation", C.c_double),
                ("sigma_cutoff", C.c_double), ("coverage_eps", C.c_double), ("tile_size", C.c_int32),
                ("channels", C.c_uint32), ("bg_quad", C.c_double * 8),
                ("bg_phasor", C.c_double * 4), ("bg_color", C.c_double * 3)]


class SceneDesc(C.Structure):
    _fields_ = [("n", C.c_int32), ("n_keyframes", C.c_int32), ("sh_degree", C.c_int32), ("n_freq", C.c_int32),
                ("frequency", C.c_double * 2), ("source_intensity", C.c_double), ("speed_of_light", C.c_double),
                ("color", C.c_int32), ("_pad", C.c_int32)]


class Frame(C.Structure):
    _fields_ = [("key", C.c_int32), ("_pad", C.c_int32), ("w", C.c_double)]


class AdamConfig(C.Structure):
    _fields_ = [("position", C.c_double), ("log_scale", C.c_double), ("rotation", C.c_double),
                ("opacity", C.c_double), ("reflectivity", C.c_double), ("motion", C.c_double),
                ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double), ("color", C.c_double)]


_lib = None

_fp = C.POINTER(C.c_float)
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_vp = C.c_void_p


class DensifyConfigC(C.Structure):
    _fields_ = [("grad_threshold", C.c_double), ("opacity_floor", C.c_double), ("split_scale_fraction", C.c_double),
                ("split_shrink", C.c_double), ("min_count", C.c_int32)]


class DeformConfigC(C.Structure):
    _fields_ = [("hidden_layers", C.c_int32), ("width", C.c_int32), ("l_x", C.c_int32), ("l_t", C.c_int32),
                ("coord_scale", C.c_double)]

# name -> (restype, argtypes)
SIGNATURES = {
    "tsb_last_error": (C.c_char_p, []),
    "tsb_abi_version": (C.c_int, []),
    "tsb_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "tsb_ctx_destroy": (None, [_vp]),
    "tsb_ctx_synchronize": (C.c_int, [_vp]),
    "tsb_ctx_stream": (_vp, [_vp]),
    "tsb_ctx_join": (C.c_int, [_vp]),
    "tsb_pass_stream": (_vp, [_vp]),
    "tsb_ctx_launch_count": (C.c_int64, [_vp]),
    "tsb_ctx_redo_count": (C.c_int64, [_vp]),
    "tsb_ctx_raster_counts": (C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "tsb_ctx_scan_counts": (C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "tsb_ctx_set_profiling": (C.c_int, [_vp, C.c_int]),
    "tsb_ctx_stage_times": (C.c_int, [_vp, _dp, _lp]),
    "tsb_scene_create": (C.c_int, [_vp, C.POINTER(SceneDesc), C.POINTER(_vp)]),
    "tsb_scene_destroy": (None, [_vp]),
    "tsb_scene_set_params": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp]),
    "tsb_scene_get_params": (C.c_int, [_vp, _fp, _fp, _fp, _fp, _fp, _fp]),
    "tsb_scene_get_grads": (C.c_int, [_vp, _fp, _fp, _fp, _fp, _fp, _fp, _dp, _dp]),
    "tsb_scene_get_bg_grads": (C.c_int, [_vp, _dp, _dp]),
    "tsb_scene_zero_grads": (C.c_int, [_vp]),
    "tsb_scene_set_sh": (C.c_int, [_vp, C.c_int, _vp]),
    "tsb_scene_get_sh": (C.c_int, [_vp, _fp, C.c_int]),
    "tsb_scene_set_color": (C.c_int, [_vp, C.c_int, _vp]),
    "tsb_scene_get_color": (C.c_int, [_vp, _fp, C.c_int]),
    "tsb_scene_get_bg_color_grad": (C.c_int, [_vp, _dp]),
    "tsb_scene_get_adam_state": (C.c_int, [_vp, _fp, _fp]),
    "tsb_scene_get_densify_stat": (C.c_int, [_vp, _fp, _lp]),
    "tsb_scene_adam_step": (C.c_int, [_vp, C.POINTER(AdamConfig)]),
    "tsb_adam_step_flat": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, _vp, C.c_size_t, C.c_int64, C.c_double,
                                      C.c_double, C.c_double, C.c_double]),
    "tsb_adam_reindex_flat": (C.c_int, [_vp, C.c_int, _vp, _vp, C.c_size_t, _vp, C.c_size_t, C.c_int32, _vp, _vp]),
    "tsb_pass_create": (C.c_int, [_vp, C.POINTER(_vp)]),
    "tsb_pass_destroy": (None, [_vp]),
    "tsb_pass_prepare": (C.c_int, [_vp, _vp, C.POINTER(Camera), C.POINTER(RenderOptions), C.POINTER(Frame)]),
    "tsb_pass_visible_count": (C.c_int, [_vp, _ip]),
    "tsb_pass_num_keys": (C.c_int, [_vp, _lp]),
    "tsb_pass_forward": (C.c_int, [_vp]),
    "tsb_pass_forward_loss": (C.c_int, [_vp, C.c_int, _vp, _dp, _dp]),
    "tsb_pass_forward_image_loss": (C.c_int, [_vp, C.c_int, _vp, _dp, C.c_double, _dp]),
    "tsb_pass_output": (C.c_int, [_vp, C.c_int, C.POINTER(_vp), C.POINTER(C.c_size_t)]),
    "tsb_pass_download": (C.c_int, [_vp, C.c_int, _vp, C.c_size_t]),
    "tsb_pass_download_async": (C.c_int, [_vp, C.c_int, _vp, C.c_size_t]),
    "tsb_pass_wait": (C.c_int, [_vp]),
    "tsb_pass_backward": (C.c_int, [_vp, C.c_int, _vp]),
    "tsb_pass_backward_buffers": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp]),
    "tsb_pass_backward_ext": (C.c_int, [_vp, C.c_int] + [_vp] * 9),
    "tsb_pass_set_motion": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "tsb_pass_flow_loss": (C.c_int, [_vp, C.c_int, _vp, _vp, C.c_double, _dp, _lp, _ip]),
    "tsb_pass_get_motion_grads": (C.c_int, [_vp, _fp, _fp]),
    "tsb_pass_debug_keep_screen": (C.c_int, [_vp, C.c_int]),
    "tsb_pass_debug_set_list_capacity": (C.c_int, [_vp, C.c_uint32]),
    "tsb_scene_densify": (C.c_int, [_vp, _vp, C.c_double, C.POINTER(C.c_int32)]),
    "tsb_deform_create": (C.c_int, [_vp, _vp, C.POINTER(_vp)]),
    "tsb_deform_destroy": (None, [_vp]),
    "tsb_deform_param_count": (C.c_int64, [_vp]),
    "tsb_deform_set_params": (C.c_int, [_vp, C.c_int, _vp]),
    "tsb_deform_get_params": (C.c_int, [_vp, _vp]),
    "tsb_deform_get_grads": (C.c_int, [_vp, _vp]),
    "tsb_deform_zero_grads": (C.c_int, [_vp]),
    "tsb_deform_offsets": (C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_int64, C.c_double, _vp]),
    "tsb_deform_backward": (C.c_int, [_vp, C.c_int, C.c_int, _vp, _vp]),
    "tsb_deform_scene_offsets": (C.c_int, [_vp, C.c_int, _vp, C.c_int, C.c_double]),
    "tsb_deform_scene_backward": (C.c_int, [_vp, C.c_int, _vp, C.c_int]),
    "tsb_deform_debug_activation": (C.c_int, [_vp, C.c_int, C.c_int, _vp]),
    "tsb_deform_adam_step": (C.c_int, [_vp, C.c_double, C.c_double, C.c_double, C.c_double]),
    "tsb_debug_gemm": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, C.c_int64, C.c_int64, _vp, C.c_int64,
                                C.c_int64, _vp, C.c_int, _vp, _vp]),
    "tsb_pass_debug_prepared": (C.c_int, [_vp, _ip, _ip]),
    "tsb_pass_debug_tiles": (C.c_int, [_vp, _ip, _ip, _lp, _ip]),
    "tsb_pass_debug_records": (C.c_int, [_vp, _fp]),
    "tsb_pass_debug_screen_grads": (C.c_int, [_vp, _fp]),
    "tsb_pass_debug_fixups": (C.c_int, [_vp, _ip]),
    "tsb_pass_debug_fixup_list": (C.c_int, [_vp, _ip, C.c_int32, _ip]),
    "tsb_comm_unique_id": (C.c_int, [_vp]),
    "tsb_comm_create": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.POINTER(_vp)]),
    "tsb_comm_destroy": (None, [_vp]),
    "tsb_scene_allreduce_grads": (C.c_int, [_vp, _vp]),
    "tsb_write_pfm": (C.c_int, [C.c_char_p, _vp, C.c_int, C.c_int, C.c_int]),
    "tsb_read_pfm": (C.c_int, [C.c_char_p, _vp, C.c_size_t, _ip, _ip, _ip]),
    "tsb_pass_render_stack": (C.c_int, [_vp, C.c_char_p, C.c_int]),
    "tsb_unambiguous_range": (C.c_double, [C.c_double]),
    "tsb_quad_to_depth": (C.c_double, [C.c_double] * 5),
    "tsb_quad_basis": (None, [C.c_double, C.c_double, _dp]),
}


def lib():
    """Load libtsb.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    if rc != TSB_OK:
        raise TsbError(rc, lib().tsb_last_error().decode(errors="replace"))
