"""Op-level API on device tensors (torch CUDA tensors are used only as device
buffers and stream handles). Each op is one call into the C-ABI:

  detect_changes   cbx_op_detect    <- cbconv.cpp:57-71
  dilate_changes   cbx_op_dilate    <- cbconv.cpp:73-82
  extract_indexes  cbx_op_extract   <- cbconv.cpp:99-113
  maxpool          cbx_op_maxpool   <- baseline.cpp:119-145
  argmax_classify  cbx_op_argmax    <- baseline.cpp:147-163
  cbconv_update    cbx_op_cbconv_update <- gen_x_reduced+gemm+update_output, cbconv.cpp:115-155
"""
from __future__ import annotations

import ctypes as C

from ._cbx import Geom, GeometryError, ShapeError, check, lib


def _torch():
    import torch
    return torch


def _stream(t):
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _geom(g: dict) -> Geom:
    return Geom(*[int(g[f]) for f, _ in Geom._fields_])


def detect_changes(cur, prev, tau: float):
    """cur, prev: CUDA float32 [C,H,W]. Returns (uint8 [H,W] mask, count tensor)."""
    torch = _torch()
    if cur.shape != prev.shape:
        raise ShapeError("detect_changes: frame dimensions differ")
    Cc, H, W = cur.shape
    m = torch.zeros((H, W), dtype=torch.uint8, device=cur.device)
    cnt = torch.zeros(2, dtype=torch.int64, device=cur.device)
    check(lib.cbx_op_detect(_ptr(cur.contiguous()), _ptr(prev.contiguous()), Cc, H, W, C.c_float(tau),
                            _ptr(m), _ptr(cnt), _stream(cur)))
    return m, cnt[0]


def dilate_changes(mask, geom: dict):
    torch = _torch()
    H, W = mask.shape
    g = _geom(geom)
    if g.kernelH < 1 or g.kernelW < 1 or g.strideH < 1 or g.strideW < 1 or g.padH < 0 or g.padW < 0 \
            or H + 2 * g.padH < g.kernelH or W + 2 * g.padW < g.kernelW:
        raise GeometryError("invalid convolution geometry")
    Ho = (H + 2 * g.padH - g.kernelH) // g.strideH + 1
    Wo = (W + 2 * g.padW - g.kernelW) // g.strideW + 1
    out = torch.zeros((Ho, Wo), dtype=torch.uint8, device=mask.device)
    check(lib.cbx_op_dilate(_ptr(mask.contiguous()), H, W, C.byref(g), _ptr(out), _stream(mask)))
    return out


def extract_indexes(mask):
    """Ascending int32 linear indices of the set bytes of `mask` (any shape)."""
    torch = _torch()
    n = mask.numel()
    flat = torch.zeros(((n + 15) // 16) * 16 + 16, dtype=torch.uint8, device=mask.device)
    flat[:n] = mask.reshape(-1)
    idx = torch.empty(max(n, 1), dtype=torch.int32, device=mask.device)
    cnt = torch.zeros(1, dtype=torch.int32, device=mask.device)
    ws = torch.empty(int(lib.cbx_op_extract_workspace(n)), dtype=torch.uint8, device=mask.device)
    check(lib.cbx_op_extract(_ptr(flat), C.c_int64(n), _ptr(idx), _ptr(cnt), _ptr(ws), _stream(mask)))
    return idx[: int(cnt.item())]


def maxpool(t, window: int, stride: int):
    torch = _torch()
    Cc, H, W = t.shape
    if window < 1 or stride < 1 or window > H or window > W:
        raise GeometryError("maxpool: invalid window")
    out = torch.empty((Cc, (H - window) // stride + 1, (W - window) // stride + 1), dtype=torch.float32,
                      device=t.device)
    check(lib.cbx_op_maxpool(_ptr(t.contiguous()), Cc, H, W, window, stride, _ptr(out), _stream(t)))
    return out


def argmax_classify(t):
    torch = _torch()
    Cc, H, W = t.shape
    out = torch.empty((H, W), dtype=torch.int16, device=t.device)
    check(lib.cbx_op_argmax(_ptr(t.contiguous()), Cc, H, W, _ptr(out), _stream(t)))
    return out


def cbconv_update(inp, K, bias, geom: dict, idx, prev_out, fuse_relu: bool):
    """Reduced conv of the listed output pixels written over a copy of prev_out
    (exact fp32 order, bitwise equal to gen_x_reduced + gemm + update_output)."""
    out = prev_out.clone().contiguous()
    Cc, H, W = inp.shape
    g = _geom(geom)
    check(lib.cbx_op_cbconv_update(_ptr(inp.contiguous()), Cc, H, W, _ptr(K.contiguous()),
                                   _ptr(bias.contiguous()), C.byref(g), _ptr(idx.contiguous()),
                                   int(idx.numel()), int(fuse_relu), _ptr(out), _stream(inp)))
    return out
