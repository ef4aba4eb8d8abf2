"""B200-native change-based CNN inference (CBinfer, arXiv 1704.04313).

Python mirror of the reference's netspec-driven API (namespace ``cbinfer``,
/root/reference/proj/core/include/cbinfer/*.hpp) over the C-ABI in
``include/cbx.h``. Every call goes through the in-tree CUDA library
``_lib/libcbx.so`` (sm_100a); there is no CPU fallback: importing this package
without the built library raises ImportError, and a missing or unusable GPU
surfaces as :class:`CudaError` from the library.

Reference -> here:
  network_spec_from_json / load_network_spec / network_spec_to_json  (network.hpp:39-41)
  chain_dims                                                          (network.hpp:45)
  load_network / forward_frame / reset_state                          (network.hpp:88-97)
  Network.thresholds / Network.set_thresholds                         (network.hpp:66-67)
  read_weights_f32le / write_weights_f32le                            (io.hpp:29-30)
  random_filters / generate_weights / synth_frame / sprite_rect       (synth.hpp:42-85)
  detect_changes / dilate_changes / extract_indexes / maxpool /
  argmax_classify / cbconv_update (op level, device tensors)          (cbconv.hpp:87-113,
                                                                       baseline.hpp:58-79)
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from ._cbx import (BoundsError, CbxError, CudaError, GeometryError, IoError, ShapeError,
                   SpecError, check, lib, LayerDesc, NetDesc, LayerStats, Geom, SynthCfg, Sprite, KernelTime)
import ctypes as C

__all__ = [
    "LayerSpec", "NetworkSpec", "network_spec_from_json", "load_network_spec",
    "network_spec_to_json", "chain_dims", "read_weights_f32le", "write_weights_f32le",
    "random_filters", "generate_weights", "synth_frame", "Network", "load_network",
    "forward_frame", "reset_state", "ForwardResult", "CbxError", "ShapeError", "GeometryError",
    "BoundsError", "IoError", "SpecError", "CudaError", "ops",
]

KINDS = ("CBCONV", "CONV", "RELU", "MAXPOOL", "CLASSIFY")
ENGINES = {"baseline": 0, "cbinfer": 1}
PRECISIONS = {"exact": 0, "tf32": 1, "f16": 2}


@dataclass
class LayerSpec:
    """LayerSpec, network.hpp:17-27."""
    kind: str = "CONV"
    kernelH: int = 1
    kernelW: int = 1
    strideH: int = 1
    strideW: int = 1
    padH: int = 0
    padW: int = 0
    inChannels: int = 0
    outChannels: int = 1
    window: int = 0
    stride: int = 0
    threshold: float = 0.0
    fuseRelu: bool = False
    weightsFile: str = ""

    def is_conv(self) -> bool:
        return self.kind in ("CBCONV", "CONV")

    def geom(self) -> dict:
        return dict(kernelH=self.kernelH, kernelW=self.kernelW, strideH=self.strideH,
                    strideW=self.strideW, padH=self.padH, padW=self.padW,
                    inChannels=self.inChannels, outChannels=self.outChannels)


@dataclass
class NetworkSpec:
    """NetworkSpec, network.hpp:29-35."""
    inputChannels: int = 0
    inputHeight: int = 0
    inputWidth: int = 0
    numClasses: int = 0
    layers: List[LayerSpec] = field(default_factory=list)

    def cb_layers(self) -> List[int]:
        return [k for k, l in enumerate(self.layers) if l.kind == "CBCONV"]


def network_spec_from_json(text: str) -> NetworkSpec:
    """network_spec_from_json, network.cpp:43-85 (same defaults and errors)."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise SpecError(f"network spec: invalid JSON: {e}") from None
    try:
        spec = NetworkSpec(int(doc["inputChannels"]), int(doc["inputHeight"]),
                           int(doc["inputWidth"]), int(doc["numClasses"]))
        for jl in doc["layers"]:
            kind = jl["kind"]
            if kind not in KINDS:
                raise SpecError(f'unknown layer kind "{kind}"')
            l = LayerSpec(kind=kind)
            if l.is_conv():
                l.kernelH, l.kernelW = int(jl["kernelH"]), int(jl["kernelW"])
                l.strideH, l.strideW = int(jl.get("strideH", 1)), int(jl.get("strideW", 1))
                l.padH, l.padW = int(jl.get("padH", 0)), int(jl.get("padW", 0))
                l.outChannels = int(jl["outChannels"])
                l.weightsFile = str(jl["weightsFile"])
            if kind == "CBCONV":
                l.threshold = float(np.float32(jl.get("threshold", 0.0)))
                l.fuseRelu = bool(jl.get("fuseRelu", False))
                if l.threshold < 0:
                    raise SpecError("network spec: negative threshold")
            if kind == "MAXPOOL":
                l.window, l.stride = int(jl["window"]), int(jl["stride"])
            spec.layers.append(l)
        return spec
    except (KeyError, TypeError, ValueError) as e:
        raise SpecError(f"network spec: {e!r}") from None


def load_network_spec(path: str) -> NetworkSpec:
    try:
        with open(path) as f:
            return network_spec_from_json(f.read())
    except OSError:
        raise IoError(f"cannot open network spec {path}") from None


def network_spec_to_json(spec: NetworkSpec) -> str:
    """network_spec_to_json, network.cpp:95-126."""
    layers = []
    for l in spec.layers:
        jl = {"kind": l.kind}
        if l.is_conv():
            jl.update(kernelH=l.kernelH, kernelW=l.kernelW, strideH=l.strideH, strideW=l.strideW,
                      padH=l.padH, padW=l.padW, outChannels=l.outChannels, weightsFile=l.weightsFile)
        if l.kind == "CBCONV":
            jl.update(threshold=float(str(np.float32(l.threshold))), fuseRelu=l.fuseRelu)
        if l.kind == "MAXPOOL":
            jl.update(window=l.window, stride=l.stride)
        layers.append(jl)
    return json.dumps(dict(inputChannels=spec.inputChannels, inputHeight=spec.inputHeight,
                           inputWidth=spec.inputWidth, numClasses=spec.numClasses, layers=layers),
                      indent=2) + "\n"


def _net_desc(spec: NetworkSpec):
    arr = (LayerDesc * max(1, len(spec.layers)))()
    for k, l in enumerate(spec.layers):
        arr[k].kind = KINDS.index(l.kind)
        arr[k].geom = Geom(l.kernelH, l.kernelW, l.strideH, l.strideW, l.padH, l.padW,
                           l.inChannels, l.outChannels)
        arr[k].window, arr[k].stride = l.window, l.stride
        arr[k].threshold = l.threshold
        arr[k].fuseRelu = int(l.fuseRelu)
    d = NetDesc(spec.inputChannels, spec.inputHeight, spec.inputWidth, spec.numClasses,
                len(spec.layers), arr)
    return d, arr


def chain_dims(spec: NetworkSpec) -> List[Tuple[Tuple[int, int, int], Tuple[int, int, int]]]:
    """chain_dims, network.cpp:128-188. Fills inChannels of the spec's conv layers."""
    d, arr = _net_desc(spec)
    out = (LayerDesc * max(1, len(spec.layers)))()
    dims = (C.c_int * (6 * max(1, len(spec.layers))))()
    check(lib.cbx_chain_dims(C.byref(d), out, dims))
    shapes = []
    for k, l in enumerate(spec.layers):
        if l.is_conv():
            l.inChannels = out[k].geom.inChannels
        shapes.append(((dims[6 * k], dims[6 * k + 1], dims[6 * k + 2]),
                       (dims[6 * k + 3], dims[6 * k + 4], dims[6 * k + 5])))
    return shapes


# ---------------------------------------------------------------- weights I/O
def read_weights_f32le(path: str, geom: dict) -> Tuple[np.ndarray, np.ndarray]:
    """read_weights_f32le, io.cpp:121-139: exact byte length, k(o,c,j,i) then biases."""
    O = geom["outChannels"]
    cols = geom["inChannels"] * geom["kernelH"] * geom["kernelW"]
    expect = (O * cols + O) * 4
    try:
        with open(path, "rb") as f:
            buf = f.read()
    except OSError:
        raise IoError(f"cannot open {path}") from None
    if len(buf) != expect:
        raise IoError(f"{path}: expected {expect} bytes (kernel {O}x{geom['inChannels']}x"
                      f"{geom['kernelH']}x{geom['kernelW']} + bias), got {len(buf)}")
    a = np.frombuffer(buf, dtype="<f4").astype(np.float32)
    K, b = a[: O * cols].reshape(O, cols).copy(), a[O * cols:].copy()
    if not (np.isfinite(K).all() and np.isfinite(b).all()):
        raise IoError(f"non-finite value in {path}")
    return K, b


def write_weights_f32le(path: str, K: np.ndarray, bias: np.ndarray) -> None:
    with open(path, "wb") as f:
        f.write(np.ascontiguousarray(K, "<f4").tobytes())
        f.write(np.ascontiguousarray(bias, "<f4").tobytes())


def random_filters(geom: dict, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """random_filters, synth.cpp:188-196 (mt19937, fan-in scaled)."""
    cols = geom["inChannels"] * geom["kernelH"] * geom["kernelW"]
    K = np.zeros((geom["outChannels"], cols), np.float32)
    b = np.zeros(geom["outChannels"], np.float32)
    g = Geom(*[int(geom[f]) for f, _ in Geom._fields_])
    check(lib.cbx_random_filters(C.byref(g), C.c_uint32(seed & 0xFFFFFFFF),
                                 K.ctypes.data_as(C.POINTER(C.c_float)),
                                 b.ctypes.data_as(C.POINTER(C.c_float))))
    return K, b


def generate_weights(spec: NetworkSpec, dir: Optional[str], seed: int) -> Dict[int, Tuple[np.ndarray, np.ndarray]]:
    """generate_weights, synth.cpp:198-209: layer k (1-based over all layers) gets
    random_filters(geom, seed + k). Writes reference-format files when `dir` is
    given; returns {layer_index: (K, bias)}."""
    chain_dims(spec)
    out = {}
    if dir:
        os.makedirs(dir, exist_ok=True)
    for k, l in enumerate(spec.layers):
        if not l.is_conv():
            continue
        K, b = random_filters(l.geom(), seed + k + 1)
        out[k] = (K, b)
        if dir:
            write_weights_f32le(os.path.join(dir, l.weightsFile or f"layer{k + 1}.weights.f32le"), K, b)
    return out


def _synth_cfg(cfg: dict):
    sp = cfg.get("sprites", [])
    arr = (Sprite * max(1, len(sp)))()
    for k, s in enumerate(sp):
        arr[k] = Sprite(int(s[0]), int(s[1]), float(s[2]))
    return SynthCfg(int(cfg.get("channels", 3)), int(cfg.get("height", 64)), int(cfg.get("width", 64)),
                    int(cfg.get("frames", 10)), len(sp), arr, float(cfg.get("noise", 0.0)),
                    int(cfg.get("seed", 1)) & 0xFFFFFFFF), arr


def synth_frame(cfg: dict, f: int) -> np.ndarray:
    """synth_frame, synth.cpp:66-91. cfg: channels,height,width,sprites=[(size,vel,intensity)],noise,seed."""
    c, keep = _synth_cfg(cfg)
    out = np.zeros((c.channels, c.height, c.width), np.float32)
    check(lib.cbx_synth_frame(C.byref(c), f, out.ctypes.data_as(C.POINTER(C.c_float))))
    return out


def synth_frame_device(cfg: dict, f: int, out_ptr: int, stream: int = 0) -> None:
    """On-device noise-free synth frame into a device buffer (bench input source)."""
    c, keep = _synth_cfg(cfg)
    check(lib.cbx_synth_frame_device(C.byref(c), f, C.c_void_p(out_ptr), C.c_void_p(stream)))


def decode_u8_device(in_ptr: int, S: int, channels: int, height: int, width: int, out_ptr: int,
                     stream: int = 0) -> None:
    """cbx_op_decode_u8: S interleaved 8-bit frames on the device -> planar fp32 px / 255."""
    check(lib.cbx_op_decode_u8(C.c_void_p(in_ptr), S, channels, height, width, C.c_void_p(out_ptr),
                               C.c_void_p(stream)))


# ---------------------------------------------------------------- network
@dataclass
class ForwardResult:
    """ForwardResult, network.hpp:72-76 (one per stream)."""
    labels: np.ndarray
    stats: List[dict]
    macsTotal: int


class Network:
    """A loaded network on one B200 serving `streams` independent camera streams.

    Mirrors cbinfer::Network (network.hpp:54-68) + forward_frame/reset_state.
    Weights: dict {layer: (K, bias)} in the reference layout, or a directory
    of reference weight files (read_weights_f32le)."""

    def __init__(self, spec: NetworkSpec, weights, device: int = 0, streams: int = 1,
                 precision: str = "tf32", fuse_tail: bool = True, lanes: int = 0):
        self.spec = spec
        self.shapes = chain_dims(spec)
        self.streams = streams
        self.device = device
        self.precision = precision
        d, arr = _net_desc(spec)
        h = C.c_void_p()
        # lanes: independent engines over contiguous stream groups whose kernels
        # overlap on the GPU (0 = automatic: 2 when streams >= 2)
        check(lib.cbx_create_ex(C.byref(d), device, streams, PRECISIONS[precision], lanes, C.byref(h)))
        self._h = h
        self.nl = len(spec.layers)
        if isinstance(weights, str):
            wdir = weights
            weights = {}
            for k, l in enumerate(spec.layers):
                if l.is_conv():
                    try:
                        weights[k] = read_weights_f32le(os.path.join(wdir, l.weightsFile), l.geom())
                    except IoError as e:
                        raise IoError(f"layer {k + 1} ({l.kind}): {e}") from None
        for k, l in enumerate(spec.layers):
            if l.is_conv():
                if k not in weights:
                    raise IoError(f"layer {k + 1} ({l.kind}): missing weights")
                K, b = weights[k]
                K = np.ascontiguousarray(K, np.float32)
                b = np.ascontiguousarray(b, np.float32)
                if K.size != l.outChannels * l.inChannels * l.kernelH * l.kernelW or b.size != l.outChannels:
                    raise IoError(f"layer {k + 1} ({l.kind}): weight shape mismatch")
                self._chk(lib.cbx_load_layer(self._h, k, K.ctypes.data_as(C.POINTER(C.c_float)),
                                             b.ctypes.data_as(C.POINTER(C.c_float))))
        if not fuse_tail:
            self.set_fuse_tail(False)
        last = spec.layers[-1]
        self.label_hw = self.shapes[-1][0][1:] if last.kind == "CLASSIFY" else self.shapes[-1][1][1:]
        self._frame_elems = spec.inputChannels * spec.inputHeight * spec.inputWidth

    def _chk(self, rc):
        if rc:
            check(rc, lib.cbx_last_error(self._h).decode())

    def close(self):
        # (at interpreter shutdown the module global `lib` may already be gone)
        if getattr(self, "_h", None) and lib is not None:
            lib.cbx_destroy(self._h)
        self._h = None

    def __del__(self):
        self.close()

    # -- thresholds
    def thresholds(self) -> List[float]:
        n = len(self.spec.cb_layers())
        t = (C.c_float * max(1, n))()
        self._chk(lib.cbx_get_thresholds(self._h, t, n))
        return [t[i] for i in range(n)]

    def set_thresholds(self, taus: Sequence[float]) -> None:
        t = (C.c_float * max(1, len(taus)))(*taus)
        self._chk(lib.cbx_set_thresholds(self._h, t, len(taus)))
        for k, tau in zip(self.spec.cb_layers(), taus):
            self.spec.layers[k].threshold = float(tau)

    def reset_state(self) -> None:
        self._chk(lib.cbx_reset(self._h))

    def set_fuse_tail(self, on: bool) -> None:
        """CBX_OPT_FUSE_TAIL: run the network's per-pixel tail in the last
        tcgen05 conv's epilogue (default) or materialize every layer."""
        self._chk(lib.cbx_set_option(self._h, 0, int(bool(on))))

    def set_step_times(self, on: bool) -> None:
        """CBX_OPT_STEP_TIMES: event nodes at the kernel boundaries of the frame
        graph; step_times() then returns the reference's StepTimes per layer."""
        self._chk(lib.cbx_set_option(self._h, 2, int(bool(on))))

    def step_times(self) -> np.ndarray:
        """[S, layers, 5] ns (detect, extract, generate, multiply, update) of
        the last frame (StepTimes, cbconv.hpp:44-52; see cbx_read_step_times)."""
        out = np.zeros((self.streams, self.nl, 5), np.int64)
        self._chk(lib.cbx_read_step_times(self._h, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out

    def has_history(self) -> bool:
        return lib.cbx_has_history(self._h) == 1

    def layer_input(self, layer: int, s: int = 0, engine: str = "cbinfer") -> np.ndarray:
        """Input tensor of `layer` after the last frame (prevInput of a CBCONV)."""
        c, h, w = self.shapes[layer][0]
        out = np.zeros((c, h, w), np.float32)
        self._chk(lib.cbx_get_input(self._h, ENGINES[engine], layer, s, out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def set_tc_pair(self, mode: int) -> None:
        """CBX_OPT_TC_PAIR: -1 auto (single-CTA tiles), 0 single-CTA tiles,
        1 CTA pairs (cta_group::2) everywhere."""
        self._chk(lib.cbx_set_option(self._h, 1, int(mode)))

    # -- forward
    def forward(self, frames: np.ndarray, engine: str = "cbinfer") -> List[ForwardResult]:
        """frames: [S, C, H, W] float32 host array (or [C,H,W] when S == 1)."""
        f = np.ascontiguousarray(frames, np.float32)
        if f.size != self._frame_elems * self.streams:
            raise ShapeError("forward_frame: frame does not match network input dimensions")
        S = self.streams
        labels = np.zeros((S,) + tuple(self.label_hw), np.uint16)
        stats = (LayerStats * (S * self.nl))()
        macs = (C.c_uint64 * S)()
        self._chk(lib.cbx_forward(self._h, ENGINES[engine], f.ctypes.data_as(C.POINTER(C.c_float)),
                                  labels.ctypes.data_as(C.POINTER(C.c_uint16)), stats, macs))
        out = []
        for s in range(S):
            st = [dict(changedInputPixels=stats[s * self.nl + k].changedInputPixels,
                       changedOutputPixels=stats[s * self.nl + k].changedOutputPixels,
                       gemmMacs=stats[s * self.nl + k].gemmMacs) for k in range(self.nl)]
            out.append(ForwardResult(labels[s], st, macs[s]))
        return out

    def forward_u8(self, frames: np.ndarray, engine: str = "cbinfer") -> List[ForwardResult]:
        """cbx_forward_u8: 8-bit camera frames [S, H, W, C] (or [H, W, C]),
        interleaved like the binary PPM raster; decoded on the device as
        read_ppm does (px / 255, io.cpp:60-104)."""
        f = np.ascontiguousarray(frames, np.uint8)
        if f.size != self._frame_elems * self.streams:
            raise ShapeError("forward_frame: frame does not match network input dimensions")
        S = self.streams
        labels = np.zeros((S,) + tuple(self.label_hw), np.uint16)
        stats = (LayerStats * (S * self.nl))()
        macs = (C.c_uint64 * S)()
        self._chk(lib.cbx_forward_u8(self._h, ENGINES[engine], f.ctypes.data_as(C.POINTER(C.c_uint8)),
                                     labels.ctypes.data_as(C.POINTER(C.c_uint16)), stats, macs))
        return [ForwardResult(labels[s], [dict(changedInputPixels=stats[s * self.nl + k].changedInputPixels,
                                               changedOutputPixels=stats[s * self.nl + k].changedOutputPixels,
                                               gemmMacs=stats[s * self.nl + k].gemmMacs) for k in range(self.nl)],
                              macs[s]) for s in range(S)]

    def submit_u8(self, frames: np.ndarray, labels: np.ndarray) -> int:
        """cbx_submit_u8: as submit() with 8-bit interleaved frames [S, H, W, C]
        (4x fewer bytes over PCIe), decoded on the device."""
        if frames.dtype != np.uint8 or not frames.flags.c_contiguous or frames.size != self._frame_elems * self.streams:
            raise ShapeError("submit_u8: frames must be a contiguous uint8 [S, H, W, C] array of the network input")
        want = (self.streams,) + tuple(self.label_hw)
        if labels.dtype != np.uint16 or not labels.flags.c_contiguous or labels.shape != want:
            raise ShapeError(f"submit_u8: labels must be a contiguous uint16 array of shape {want}")
        t = C.c_int64()
        self._chk(lib.cbx_submit_u8(self._h, ENGINES["cbinfer"], frames.ctypes.data_as(C.POINTER(C.c_uint8)),
                                    labels.ctypes.data_as(C.POINTER(C.c_uint16)), C.byref(t)))
        return t.value

    def submit(self, frames: np.ndarray, labels: np.ndarray) -> int:
        """cbx_submit: enqueue the next frame of every stream ([S, C, H, W]
        float32 host array) without waiting; labels ([S, Hl, Wl] uint16 host
        array) is filled by the time wait(ticket) returns. Both must stay
        alive and unchanged until then; pinned host memory lets the copy of
        the next submission overlap this frame's kernels."""
        if frames.dtype != np.float32 or not frames.flags.c_contiguous or frames.size != self._frame_elems * self.streams:
            raise ShapeError("submit: frames must be a contiguous float32 [S, C, H, W] array of the network input")
        want = (self.streams,) + tuple(self.label_hw)
        if labels.dtype != np.uint16 or not labels.flags.c_contiguous or labels.shape != want:
            raise ShapeError(f"submit: labels must be a contiguous uint16 array of shape {want}")
        t = C.c_int64()
        self._chk(lib.cbx_submit(self._h, ENGINES["cbinfer"], frames.ctypes.data_as(C.POINTER(C.c_float)),
                                 labels.ctypes.data_as(C.POINTER(C.c_uint16)), C.byref(t)))
        return t.value

    def wait(self, ticket: int, with_stats: bool = True):
        """cbx_wait: block until submission `ticket` is done; returns its
        per-stream LayerStats lists (or None) and macsTotal per stream."""
        S = self.streams
        if not with_stats:
            self._chk(lib.cbx_wait(self._h, ticket, None, None))
            return None
        stats = (LayerStats * (S * self.nl))()
        macs = (C.c_uint64 * S)()
        self._chk(lib.cbx_wait(self._h, ticket, stats, macs))
        return [[dict(changedInputPixels=stats[s * self.nl + k].changedInputPixels,
                      changedOutputPixels=stats[s * self.nl + k].changedOutputPixels,
                      gemmMacs=stats[s * self.nl + k].gemmMacs) for k in range(self.nl)]
                for s in range(S)], list(macs)

    def worst_case_counts(self) -> np.ndarray:
        """cbench analyze-prop (cbench.cpp:242-302) on the device for the last
        change-based frame: [S, numCB-1] worst-case updated counts of CBCONV
        layers 1.. (the previous CB layer's updated set pushed through the
        layers in between, worst_case_propagation cbconv.cpp:84-97)."""
        ncb = len(self.spec.cb_layers())
        out = np.zeros((self.streams, max(0, ncb - 1)), np.int64)
        self._chk(lib.cbx_worst_case_counts(self._h, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out

    def forward_frame(self, frame: np.ndarray, engine: str = "cbinfer") -> ForwardResult:
        return self.forward(frame, engine)[0]

    def forward_device(self, frame_ptrs: Sequence[int], engine: str = "cbinfer") -> None:
        arr = (C.c_void_p * self.streams)(*frame_ptrs)
        self._chk(lib.cbx_forward_device(self._h, ENGINES[engine], arr))

    def forward_device_u8(self, frame_ptrs: Sequence[int], engine: str = "cbinfer") -> None:
        """cbx_forward_device_u8: 8-bit interleaved frames (H x W x C bytes) on the device."""
        arr = (C.c_void_p * self.streams)(*frame_ptrs)
        self._chk(lib.cbx_forward_device_u8(self._h, ENGINES[engine], arr))

    def set_u8_native(self, on: bool) -> None:
        """CBX_OPT_U8_NATIVE: 8-bit frames run natively (byte detection + kind::i8
        layer 1) or are decoded to fp32 planar frames first."""
        self._chk(lib.cbx_set_option(self._h, 3, int(bool(on))))

    def sync(self):
        self._chk(lib.cbx_sync(self._h))

    def read_labels(self, engine: str = "cbinfer") -> np.ndarray:
        labels = np.zeros((self.streams,) + tuple(self.label_hw), np.uint16)
        self._chk(lib.cbx_read_labels(self._h, ENGINES[engine], labels.ctypes.data_as(C.POINTER(C.c_uint16))))
        return labels

    def read_stats(self, engine: str = "cbinfer"):
        S = self.streams
        stats = (LayerStats * (S * self.nl))()
        macs = (C.c_uint64 * S)()
        self._chk(lib.cbx_read_stats(self._h, ENGINES[engine], stats, macs))
        return [[dict(changedInputPixels=stats[s * self.nl + k].changedInputPixels,
                      changedOutputPixels=stats[s * self.nl + k].changedOutputPixels,
                      gemmMacs=stats[s * self.nl + k].gemmMacs) for k in range(self.nl)]
                for s in range(S)], list(macs)

    def profile(self, frame_ptrs: Sequence[int], engine: str = "cbinfer", u8: bool = False) -> List[dict]:
        """One forward outside the CUDA graph with CUDA events around every
        kernel (cbx_profile_forward / cbx_profile_forward_u8 for 8-bit device
        frames). Returns [{name, layer, ms}]."""
        arr = (C.c_void_p * self.streams)(*frame_ptrs)
        cap = 256
        out = (KernelTime * cap)()
        n = C.c_int()
        fn = lib.cbx_profile_forward_u8 if u8 else lib.cbx_profile_forward
        self._chk(fn(self._h, ENGINES[engine], arr, out, cap, C.byref(n)))
        return [dict(name=out[i].name.decode(), layer=out[i].layer, ms=out[i].ms) for i in range(min(n.value, cap))]

    def num_lanes(self) -> int:
        return lib.cbx_num_lanes(self._h)

    def layer_operands(self, layer: int) -> str:
        """Operand format of a conv layer: 'fp32' (exact, CUDA cores), 'tf32' or 'f16' (tcgen05),
        'i8' (tcgen05 kind::i8 on 8-bit camera frames; fp32 frames take the exact path)."""
        return {0: "fp32", 1: "tf32", 2: "f16", 3: "i8"}.get(lib.cbx_layer_operands(self._h, layer), "none")

    def stream_handle(self) -> int:
        return lib.cbx_stream(self._h) or 0

    def last_launch_count(self) -> int:
        return lib.cbx_last_launch_count(self._h)

    # -- traces (ForwardTrace / CBConvTrace)
    def layer_output(self, layer: int, s: int = 0, engine: str = "cbinfer") -> np.ndarray:
        c, h, w = self.shapes[layer][1]
        out = np.zeros((c, h, w), np.float32)
        self._chk(lib.cbx_get_activation(self._h, ENGINES[engine], layer, s,
                                         out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def final_activation(self, s: int = 0, engine: str = "cbinfer") -> np.ndarray:
        k = self.nl - 2 if self.spec.layers[-1].kind == "CLASSIFY" else self.nl - 1
        if k < 0:
            raise SpecError("network has no activation layer before CLASSIFY")
        return self.layer_output(k, s, engine)

    def trace(self, cb: int, s: int = 0):
        """(detected input-grid mask or None on a full frame, ascending updated indices)."""
        k = self.spec.cb_layers()[cb]
        (_, h, w), (_, ho, wo) = self.shapes[k]
        det = np.zeros((h, w), np.uint8)
        upd = np.zeros(ho * wo, np.int32)
        n = C.c_int64()
        first = C.c_int()
        self._chk(lib.cbx_get_trace(self._h, cb, s, det.ctypes.data_as(C.POINTER(C.c_uint8)),
                                    upd.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(n), C.byref(first)))
        return (None if first.value else det), upd[: n.value].copy()


def load_network(spec: NetworkSpec, weights, **kw) -> Network:
    """load_network, network.cpp:207-235 (weights: directory or {layer: (K, bias)})."""
    return Network(spec, weights, **kw)


def forward_frame(net: Network, frame: np.ndarray, engine: str = "cbinfer") -> ForwardResult:
    return net.forward_frame(frame, engine)


def reset_state(net: Network) -> None:
    net.reset_state()


from . import ops  # noqa: E402  (op-level API over device tensors)
