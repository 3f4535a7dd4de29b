"""ctypes binding of the in-tree C-ABI library (include/echoforge_b200.h).

There is no CPU fallback: if ``libechoforge_b200.so`` is missing or no CUDA
device is present, every compute entry point raises.  Errors from the
library map to ValueError (EF_EINVAL, the reference's contract-violation
convention) or RuntimeError (CUDA / unsupported).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EF_LIB_PATH", os.path.join(HERE, "libechoforge_b200.so"))

EF_OK, EF_EINVAL, EF_ECUDA, EF_ENOMEM, EF_EUNSUPPORTED, EF_ENCCL = 0, -1, -2, -3, -4, -5
ST_NAMES = ("paths", "segments", "reflections", "arrivals", "direct", "dropped", "escaped",
            "nodes", "tris")
EF_ST_COUNT = 10
P_NAMES = ("rt60", "gain", "drr_db", "total", "direct", "silent", "fit_n", "slope",
           "first_bin", "last_bin")
EF_P_COUNT = 10
EF_S_COUNT = 4

_lib = None


class TraceConfig(ctypes.Structure):
    """ef_trace_config (include/echoforge_b200.h)."""
    _fields_ = [("n_sources", ctypes.c_int32), ("order", ctypes.c_int32),
                ("n_bins", ctypes.c_int32), ("max_bounces", ctypes.c_int32),
                ("n_rays", ctypes.c_int64), ("ray0", ctypes.c_uint32),
                ("seed", ctypes.c_uint32), ("frame", ctypes.c_uint32),
                ("mode", ctypes.c_int32), ("bin_len", ctypes.c_double),
                ("listener", ctypes.c_double * 3), ("radius", ctypes.c_double),
                ("e0", ctypes.c_float), ("record_ids", ctypes.c_int32),
                ("clear_outputs", ctypes.c_int32), ("diffuse_rain", ctypes.c_int32),
                ("er_max_order", ctypes.c_int32), ("er_capacity", ctypes.c_int64),
                ("er_entries", ctypes.c_void_p), ("er_count", ctypes.c_void_p)]


# ef_er_entry (72 bytes)
ER_DTYPE = np.dtype([("src", "<i4"), ("order", "<i4"), ("tri0", "<i4"), ("tri1", "<i4"),
                     ("dist", "<f8"), ("dir", "<f4", 3), ("pad", "<f4"), ("energy", "<f4", 8)])


class AnalysisConfig(ctypes.Structure):
    """ef_analysis_config."""
    _fields_ = [("n_sources", ctypes.c_int32), ("n_bins", ctypes.c_int32),
                ("n_bands", ctypes.c_int32), ("order", ctypes.c_int32),
                ("bin_s", ctypes.c_double), ("max_rt", ctypes.c_double)]


EXPORTS = ("ef_abi_version", "ef_last_error", "ef_launch_count", "ef_scene_create",
           "ef_scene_destroy", "ef_scene_info", "ef_intersect_batch", "ef_occluded_batch",
           "ef_ray_triangles", "ef_eval_sh_batch", "ef_loudness_batch", "ef_trace", "ef_analyze", "ef_blend",
           "ef_audio_create", "ef_audio_destroy", "ef_audio_info", "ef_audio_process", "ef_audio_update",
           "ef_scene_refit", "ef_acoustic_metrics", "ef_scene_create_ex", "ef_scene_rebuild",
           "ef_trace_fused", "ef_peer_alloc", "ef_peer_free", "ef_peer_open", "ef_peer_close",
           "ef_nccl_unique_id", "ef_nccl_comm_create", "ef_nccl_comm_destroy", "ef_nccl_reduce_hist",
           "ef_obj_parse", "ef_mesh_info", "ef_mesh_arrays", "ef_mesh_destroy")


def lib():
    """Load the library once; raises RuntimeError when it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is not built; run `python -m paper_1803_00430_b200.build` "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    L.ef_abi_version.restype = ctypes.c_int
    L.ef_last_error.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
    L.ef_launch_count.restype = ctypes.c_uint64
    L.ef_scene_create.argtypes = [vp, vp, vp, vp, vp, i64, vp, vp, i32, i32,
                                  ctypes.POINTER(vp)]
    L.ef_scene_destroy.argtypes = [vp]
    L.ef_scene_info.argtypes = [vp, vp]
    L.ef_intersect_batch.argtypes = [vp, vp, vp, i64, f64, vp, i32, vp, vp, vp, vp]
    L.ef_occluded_batch.argtypes = [vp, vp, vp, i64, vp, vp]
    L.ef_ray_triangles.argtypes = [vp, vp, i64, vp, vp, vp, i64, f64, vp, vp, vp, vp]
    L.ef_eval_sh_batch.argtypes = [vp, i64, i32, vp, vp]
    L.ef_loudness_batch.argtypes = [vp, i64, i32, vp, i32, vp, vp]
    L.ef_trace.argtypes = [vp, ctypes.POINTER(TraceConfig), vp, vp, vp, vp, vp, vp, vp, vp,
                           vp, vp]
    L.ef_analyze.argtypes = [ctypes.POINTER(AnalysisConfig), vp, vp, vp, vp, vp, i32, vp,
                             vp, vp, vp, vp]
    L.ef_blend.argtypes = [vp, vp, i64, f64, vp, vp]
    L.ef_audio_create.argtypes = [vp] * 13
    L.ef_scene_refit.argtypes = [vp] * 6
    L.ef_scene_rebuild.argtypes = [vp] * 6
    L.ef_trace_fused.argtypes = [vp, ctypes.POINTER(TraceConfig), vp, vp, vp, vp, vp, i32, vp, vp,
                                 vp, vp, vp]
    L.ef_peer_alloc.argtypes = [i64, ctypes.POINTER(vp), vp]
    L.ef_peer_free.argtypes = [vp]
    L.ef_peer_open.argtypes = [vp, ctypes.POINTER(vp)]
    L.ef_peer_close.argtypes = [vp]
    L.ef_scene_create_ex.argtypes = [vp, vp, vp, vp, vp, i64, vp, vp, i32, i32, ctypes.c_uint32,
                                     ctypes.POINTER(vp)]
    L.ef_acoustic_metrics.argtypes = [vp, i64, i32, f64, vp, f64, f64, vp, vp]
    L.ef_audio_destroy.argtypes = [vp]
    L.ef_audio_info.argtypes = [vp, vp]
    L.ef_audio_process.argtypes = [vp, vp, vp, vp, vp]
    L.ef_audio_update.argtypes = [vp] * 10
    L.ef_nccl_unique_id.argtypes = [vp]
    L.ef_nccl_comm_create.argtypes = [i32, i32, vp, i32, ctypes.POINTER(vp)]
    L.ef_nccl_comm_destroy.argtypes = [vp]
    L.ef_nccl_reduce_hist.argtypes = [vp, vp, vp, i64, i32, vp]
    L.ef_obj_parse.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
    L.ef_mesh_info.argtypes = [vp, vp]
    L.ef_mesh_arrays.argtypes = [vp, vp, vp, vp, vp, i64]
    L.ef_mesh_destroy.argtypes = [vp]
    for name in EXPORTS:
        getattr(L, name).restype = ctypes.c_int if name != "ef_launch_count" else ctypes.c_uint64
    _lib = L
    return L


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    lib().ef_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(rc: int) -> None:
    if rc == EF_OK:
        return
    msg = last_error()
    if rc == EF_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"echoforge_b200 error {rc}: {msg}")


def launch_count() -> int:
    return int(lib().ef_launch_count())


# ------------------------------------------------------------------ torch glue
def torch():
    import torch as _t
    return _t


def device():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("echoforge_b200 needs a CUDA device (B200); there is no CPU fallback")
    return t.device("cuda", t.cuda.current_device())


def stream_handle(stream=None):
    t = torch()
    s = stream if stream is not None else t.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(x):
    if x is None:
        return None
    return ctypes.c_void_p(x.data_ptr())


def to_device(x, dtype, shape=None):
    """numpy / list / torch -> contiguous device tensor of `dtype`."""
    t = torch()
    if isinstance(x, t.Tensor):
        y = x.to(device=device(), dtype=dtype)
    else:
        y = t.as_tensor(np.asarray(x), dtype=dtype, device=device())
    if shape is not None:
        y = y.reshape(shape)
    return y.contiguous()


class DeviceArray:
    """A raw device pointer as a torch-importable array (CUDA array
    interface); keeps `owner` alive."""

    def __init__(self, address: int, shape, typestr: str = "<f4", owner=None):
        self.owner = owner
        self.__cuda_array_interface__ = {"shape": tuple(int(x) for x in shape), "typestr": typestr,
                                         "data": (int(address), False), "version": 3,
                                         "strides": None}

    def tensor(self):
        return torch().as_tensor(self, device=device())


def host_ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)
