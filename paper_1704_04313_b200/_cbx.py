"""ctypes binding of include/cbx.h (the C-ABI of _lib/libcbx.so)."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libcbx.so")


class CbxError(RuntimeError):
    """Base of all errors (cbinfer::error, error.hpp:9-12)."""
    code = -1


class ShapeError(CbxError):
    code = 1


class GeometryError(CbxError):
    code = 2


class BoundsError(CbxError):
    code = 3


class IoError(CbxError):
    code = 4


class SpecError(CbxError):
    code = 5


class CudaError(CbxError):
    code = 6


class ArgError(CbxError, ValueError):
    code = 7


_BY_CODE = {c.code: c for c in (ShapeError, GeometryError, BoundsError, IoError, SpecError, CudaError, ArgError)}


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA library first "
        "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_1704_04313_b200). "
        "There is no CPU fallback.")

lib = C.CDLL(LIB_PATH)


class Geom(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("kernelH", "kernelW", "strideH", "strideW", "padH", "padW",
                                       "inChannels", "outChannels")]


class LayerDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("geom", Geom), ("window", C.c_int), ("stride", C.c_int),
                ("threshold", C.c_float), ("fuseRelu", C.c_int)]


class NetDesc(C.Structure):
    _fields_ = [("inputChannels", C.c_int), ("inputHeight", C.c_int), ("inputWidth", C.c_int),
                ("numClasses", C.c_int), ("numLayers", C.c_int), ("layers", C.POINTER(LayerDesc))]


class LayerStats(C.Structure):
    _fields_ = [("changedInputPixels", C.c_int64), ("changedOutputPixels", C.c_int64),
                ("gemmMacs", C.c_uint64)]


class KernelTime(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("layer", C.c_int), ("ms", C.c_float)]


class Sprite(C.Structure):
    _fields_ = [("size", C.c_int), ("velocity", C.c_int), ("intensity", C.c_float)]


class SynthCfg(C.Structure):
    _fields_ = [("channels", C.c_int), ("height", C.c_int), ("width", C.c_int), ("frames", C.c_int),
                ("numSprites", C.c_int), ("sprites", C.POINTER(Sprite)),
                ("noiseAmplitude", C.c_float), ("seed", C.c_uint32)]


VP = C.c_void_p
lib.cbx_last_error.restype = C.c_char_p
lib.cbx_last_error.argtypes = [VP]
lib.cbx_version.restype = C.c_char_p
lib.cbx_stream.restype = VP
lib.cbx_stream.argtypes = [VP]
lib.cbx_last_launch_count.argtypes = [VP]
lib.cbx_op_extract_workspace.restype = C.c_size_t
lib.cbx_op_extract_workspace.argtypes = [C.c_int64]
lib.cbx_has_history.argtypes = [VP]
lib.cbx_submit_u8.argtypes = [VP, C.c_int, C.POINTER(C.c_uint8), C.POINTER(C.c_uint16), C.POINTER(C.c_int64)]
lib.cbx_get_input.argtypes = [VP, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]
lib.cbx_read_step_times.argtypes = [VP, C.POINTER(C.c_int64)]
for _name in ("cbx_load_layer", "cbx_set_thresholds", "cbx_get_thresholds", "cbx_set_option", "cbx_reset", "cbx_forward",
              "cbx_forward_device", "cbx_forward_device_u8", "cbx_profile_forward_u8", "cbx_sync", "cbx_read_labels", "cbx_read_stats", "cbx_labels_device",
              "cbx_get_activation", "cbx_get_trace", "cbx_destroy"):
    getattr(lib, _name).argtypes = None
lib.cbx_destroy.argtypes = [VP]
lib.cbx_submit.argtypes = [VP, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_uint16), C.POINTER(C.c_int64)]
lib.cbx_wait.argtypes = [VP, C.c_int64, VP, VP]
lib.cbx_worst_case_counts.argtypes = [VP, C.POINTER(C.c_int64)]
lib.cbx_num_lanes.argtypes = [VP]
lib.cbx_layer_operands.argtypes = [VP, C.c_int]

# exported symbols declared in include/cbx.h (checked by tests without a GPU)
EXPORTS = [
    "cbx_last_error", "cbx_version", "cbx_chain_dims", "cbx_create", "cbx_create_ex", "cbx_num_lanes", "cbx_layer_operands",
    "cbx_destroy",
    "cbx_load_layer",
    "cbx_set_thresholds", "cbx_get_thresholds", "cbx_set_option", "cbx_reset", "cbx_forward", "cbx_forward_device",
    "cbx_submit", "cbx_wait", "cbx_worst_case_counts", "cbx_sync", "cbx_read_labels", "cbx_read_stats", "cbx_labels_device", "cbx_stream",
    "cbx_last_launch_count", "cbx_profile_forward", "cbx_get_activation", "cbx_get_trace", "cbx_op_detect", "cbx_op_dilate",
    "cbx_op_extract_workspace", "cbx_op_extract", "cbx_op_maxpool", "cbx_op_argmax",
    "cbx_op_cbconv_update", "cbx_random_filters", "cbx_synth_frame", "cbx_synth_frame_device",
    "cbx_get_input", "cbx_has_history", "cbx_read_step_times", "cbx_op_relu", "cbx_op_gen_x", "cbx_op_gemm",
    "cbx_op_scatter", "cbx_forward_u8", "cbx_submit_u8", "cbx_op_decode_u8", "cbx_forward_device_u8",
    "cbx_profile_forward_u8",
]


def check(rc: int, msg: str | None = None) -> None:
    if rc == 0:
        return
    if msg is None:
        msg = (lib.cbx_last_error(None) or b"").decode()
    raise _BY_CODE.get(rc, CbxError)(msg)
