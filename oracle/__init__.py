"""TEST INFRASTRUCTURE ONLY -- ctypes access to the CPU oracle.

Two back ends, same Python surface:

* ``Oracle``  -- oracle/_build/liboracle.so, the plain-C restatement of the
  reference path (cbinfer_oracle.c). Always buildable (gcc), travels to the GPU
  box, and is what the ``-m gpu`` parity tests compare the CUDA path with.
* ``Ref``     -- oracle/_ref/libcbinfer_ref.so, the UNMODIFIED reference
  library compiled from /root/reference sources (oracle/Makefile ``ref``). Used
  to pin the restatement and as bench.py's ``--impl reference`` arm.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package. The product never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcbinfer_ref.so")

KIND = {"CBCONV": 0, "CONV": 1, "RELU": 2, "MAXPOOL": 3, "CLASSIFY": 4}
ERR = {-1: "shape_error", -2: "geometry_error", -3: "bounds_error", -4: "io_error", -5: "spec_error"}


class OracleError(RuntimeError):
    def __init__(self, code, what=""):
        super().__init__(f"{ERR.get(code, 'error')}({code}) {what}")
        self.code = code
        self.kind = ERR.get(code, "error")


def build(ref: bool = False) -> None:
    """Compile the restatement (and, when /root/reference exists, the reference)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


class Geom(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("kernelH", "kernelW", "strideH", "strideW", "padH", "padW",
                                       "inChannels", "outChannels")]


class Layer(C.Structure):
    _fields_ = [("kind", C.c_int), ("geom", Geom), ("window", C.c_int), ("stride", C.c_int),
                ("threshold", C.c_float), ("fuseRelu", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("changedInputPixels", C.c_int64), ("changedOutputPixels", C.c_int64),
                ("gemmMacs", C.c_uint64)]


class Sprite(C.Structure):
    _fields_ = [("size", C.c_int), ("velocity", C.c_int), ("intensity", C.c_float)]


class SynthCfg(C.Structure):
    _fields_ = [("channels", C.c_int), ("height", C.c_int), ("width", C.c_int), ("frames", C.c_int),
                ("numSprites", C.c_int), ("sprites", C.POINTER(Sprite)),
                ("noiseAmplitude", C.c_float), ("seed", C.c_uint32)]


def _f32(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(C.POINTER(C.c_float))


def _u8(a):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return a, a.ctypes.data_as(C.POINTER(C.c_uint8))


def make_geom(k, stride=1, pad=0, inC=1, outC=1, kw=None, stride_w=None, pad_w=None):
    return dict(kernelH=k, kernelW=k if kw is None else kw, strideH=stride,
                strideW=stride if stride_w is None else stride_w, padH=pad,
                padW=pad if pad_w is None else pad_w, inChannels=inC, outChannels=outC)


def _geom(g: dict) -> Geom:
    return Geom(**{f: int(g.get(f, 1 if f.startswith(("kernel", "stride")) else 0))
                   for f, _ in Geom._fields_})


def out_hw(g: dict, h: int, w: int):
    return ((h + 2 * g["padH"] - g["kernelH"]) // g["strideH"] + 1,
            (w + 2 * g["padW"] - g["kernelW"]) // g["strideW"] + 1)


def spec_from_json(text: str) -> dict:
    """Minimal netspec reader with the reference defaults (network.cpp:43-85)."""
    doc = json.loads(text)
    layers = []
    for jl in doc["layers"]:
        l = {"kind": jl["kind"]}
        if jl["kind"] in ("CBCONV", "CONV"):
            l.update(kernelH=jl["kernelH"], kernelW=jl["kernelW"], strideH=jl.get("strideH", 1),
                     strideW=jl.get("strideW", 1), padH=jl.get("padH", 0), padW=jl.get("padW", 0),
                     outChannels=jl["outChannels"], weightsFile=jl["weightsFile"])
        if jl["kind"] == "CBCONV":
            l.update(threshold=float(jl.get("threshold", 0.0)), fuseRelu=bool(jl.get("fuseRelu", False)))
        if jl["kind"] == "MAXPOOL":
            l.update(window=jl["window"], stride=jl["stride"])
        layers.append(l)
    return dict(inputChannels=doc["inputChannels"], inputHeight=doc["inputHeight"],
                inputWidth=doc["inputWidth"], numClasses=doc["numClasses"], layers=layers)


def spec_to_json(spec: dict) -> str:
    return json.dumps(spec, indent=2)


def _layers_array(spec: dict):
    arr = (Layer * len(spec["layers"]))()
    for k, l in enumerate(spec["layers"]):
        arr[k].kind = KIND[l["kind"]]
        if l["kind"] in ("CBCONV", "CONV"):
            arr[k].geom = _geom(dict(l, inChannels=0))
        arr[k].window = int(l.get("window", 0))
        arr[k].stride = int(l.get("stride", 0))
        arr[k].threshold = float(l.get("threshold", 0.0))
        arr[k].fuseRelu = int(bool(l.get("fuseRelu", False)))
    return arr


class Oracle:
    """The C restatement (cbinfer_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = L = C.CDLL(path)
        L.orc_detect_changes.restype = C.c_int64
        L.orc_extract_indexes.restype = C.c_int64
        L.orc_unit_float.restype = C.c_float
        L.orc_mt_next.restype = C.c_uint32

    # ---- ops ---------------------------------------------------------
    def detect_changes(self, cur, prev, tau):
        cur, pc = _f32(cur)
        prev, pp = _f32(prev)
        if cur.shape != prev.shape:
            raise OracleError(-1, "detect_changes: frame dimensions differ")
        c, h, w = cur.shape
        m = np.zeros((h, w), np.uint8)
        self.lib.orc_detect_changes(pc, pp, c, h, w, C.c_float(tau), m.ctypes.data_as(C.POINTER(C.c_uint8)))
        return m

    def dilate_changes(self, m, g):
        m, pm = _u8(m)
        ho, wo = out_hw(g, *m.shape)
        out = np.zeros((max(ho, 0), max(wo, 0)), np.uint8)
        geom = _geom(g)
        rc = self.lib.orc_dilate_changes(pm, m.shape[0], m.shape[1], C.byref(geom),
                                         out.ctypes.data_as(C.POINTER(C.c_uint8)))
        if rc:
            raise OracleError(rc)
        return out

    def worst_case_propagation(self, idx, g, h, w):
        idx = np.ascontiguousarray(idx, np.int32)
        ho, wo = out_hw(g, h, w)
        out = np.zeros((ho, wo), np.uint8)
        geom = _geom(g)
        rc = self.lib.orc_worst_case_propagation(idx.ctypes.data_as(C.POINTER(C.c_int32)), C.c_int64(len(idx)),
                                                 C.byref(geom), h, w,
                                                 out.ctypes.data_as(C.POINTER(C.c_uint8)))
        if rc:
            raise OracleError(rc)
        return out

    def extract_indexes(self, m):
        m, pm = _u8(m)
        idx = np.zeros(m.size, np.int32)
        n = self.lib.orc_extract_indexes(pm, C.c_int64(m.size), idx.ctypes.data_as(C.POINTER(C.c_int32)))
        return idx[:n].copy()

    def gen_x_reduced(self, inp, idx, g):
        inp, pi = _f32(inp)
        idx = np.ascontiguousarray(idx, np.int32)
        rows = g["inChannels"] * g["kernelH"] * g["kernelW"]
        X = np.zeros((len(idx), rows), np.float32)  # column-major [n][rows]
        geom = _geom(g)
        rc = self.lib.orc_gen_x_reduced(pi, *inp.shape, idx.ctypes.data_as(C.POINTER(C.c_int32)),
                                        C.c_int64(len(idx)), C.byref(geom), X.ctypes.data_as(C.POINTER(C.c_float)))
        if rc:
            raise OracleError(rc)
        return X

    def gemm(self, K, bias, X):
        K, pk = _f32(K)
        bias, pb = _f32(bias)
        X, px = _f32(X)
        rows, cols = K.shape
        n = X.shape[0]
        Y = np.zeros((rows, n), np.float32)
        self.lib.orc_gemm(pk, pb, rows, cols, px, C.c_int64(n), Y.ctypes.data_as(C.POINTER(C.c_float)))
        return Y

    def update_output(self, prev, Y, idx, fuse):
        out = np.array(prev, np.float32, copy=True, order="C")
        Y, py = _f32(Y)
        idx = np.ascontiguousarray(idx, np.int32)
        if Y.shape[1] != len(idx) or Y.shape[0] != out.shape[0]:
            raise OracleError(-1, "update_output")
        rc = self.lib.orc_update_output(out.ctypes.data_as(C.POINTER(C.c_float)), *out.shape, py,
                                        idx.ctypes.data_as(C.POINTER(C.c_int32)), C.c_int64(len(idx)), int(fuse))
        if rc:
            raise OracleError(rc)
        return out

    def conv_full(self, inp, K, bias, g):
        inp, pi = _f32(inp)
        K, pk = _f32(K)
        bias, pb = _f32(bias)
        ho, wo = out_hw(g, inp.shape[1], inp.shape[2])
        out = np.zeros((g["outChannels"], ho, wo), np.float32)
        geom = _geom(g)
        rc = self.lib.orc_conv_full(pi, *inp.shape, pk, pb, C.byref(geom),
                                    out.ctypes.data_as(C.POINTER(C.c_float)))
        if rc:
            raise OracleError(rc)
        return out

    def relu(self, t):
        t, pt = _f32(t)
        out = np.empty_like(t)
        self.lib.orc_relu(pt, C.c_int64(t.size), out.ctypes.data_as(C.POINTER(C.c_float)))
        return out

    def maxpool(self, t, window, stride):
        t, pt = _f32(t)
        c, h, w = t.shape
        if window < 1 or stride < 1 or window > h or window > w:
            raise OracleError(-2, "maxpool")
        out = np.zeros((c, (h - window) // stride + 1, (w - window) // stride + 1), np.float32)
        rc = self.lib.orc_maxpool(pt, c, h, w, window, stride, out.ctypes.data_as(C.POINTER(C.c_float)))
        if rc:
            raise OracleError(rc)
        return out

    def argmax_classify(self, t):
        t, pt = _f32(t)
        c, h, w = t.shape
        out = np.zeros((h, w), np.uint16)
        self.lib.orc_argmax_classify(pt, c, h, w, out.ctypes.data_as(C.POINTER(C.c_uint16)))
        return out

    # ---- synth ---------------------------------------------------------
    @staticmethod
    def _cfg(cfg: dict):
        sp = cfg.get("sprites", [])
        arr = (Sprite * max(1, len(sp)))()
        for k, s in enumerate(sp):
            arr[k] = Sprite(int(s[0]), int(s[1]), float(s[2]))
        c = SynthCfg(cfg.get("channels", 3), cfg.get("height", 64), cfg.get("width", 64),
                     cfg.get("frames", 10), len(sp), arr, float(cfg.get("noise", 0.0)),
                     int(cfg.get("seed", 1)) & 0xFFFFFFFF)
        return c, arr

    def synth_frame(self, cfg: dict, f: int):
        c, keep = self._cfg(cfg)
        out = np.zeros((c.channels, c.height, c.width), np.float32)
        rc = self.lib.orc_synth_frame(C.byref(c), f, out.ctypes.data_as(C.POINTER(C.c_float)))
        if rc:
            raise OracleError(rc)
        return out

    def synth_labels(self, cfg: dict, f: int):
        c, keep = self._cfg(cfg)
        out = np.zeros((c.height, c.width), np.uint16)
        rc = self.lib.orc_synth_labels(C.byref(c), f, out.ctypes.data_as(C.POINTER(C.c_uint16)))
        if rc:
            raise OracleError(rc)
        return out

    def sprite_rect(self, cfg: dict, s: int, f: int):
        c, keep = self._cfg(cfg)
        r = (C.c_int * 4)()
        rc = self.lib.orc_sprite_rect(C.byref(c), s, f, r)
        if rc:
            raise OracleError(rc)
        return tuple(r)

    def random_filters(self, g: dict, seed: int):
        cols = g["inChannels"] * g["kernelH"] * g["kernelW"]
        K = np.zeros((g["outChannels"], cols), np.float32)
        b = np.zeros(g["outChannels"], np.float32)
        geom = _geom(g)
        self.lib.orc_random_filters(C.byref(geom), C.c_uint32(seed & 0xFFFFFFFF),
                                    K.ctypes.data_as(C.POINTER(C.c_float)),
                                    b.ctypes.data_as(C.POINTER(C.c_float)))
        return K, b

    def chain_dims(self, spec: dict):
        arr = _layers_array(spec)
        nl = len(spec["layers"])
        dims = (C.c_int * (6 * nl))()
        rc = self.lib.orc_chain_dims(spec["inputChannels"], spec["inputHeight"], spec["inputWidth"],
                                     spec["numClasses"], arr, nl, dims)
        if rc:
            raise OracleError(rc)
        shapes = [((dims[6 * k], dims[6 * k + 1], dims[6 * k + 2]),
                   (dims[6 * k + 3], dims[6 * k + 4], dims[6 * k + 5])) for k in range(nl)]
        in_ch = [arr[k].geom.inChannels for k in range(nl)]
        return shapes, in_ch

    def generate_weights(self, spec: dict, seed: int):
        """generate_weights (synth.cpp:198-209): layer k (1-based over ALL layers) uses seed+k.
        Returns {layer_index: (K, bias)} for the conv layers."""
        shapes, in_ch = self.chain_dims(spec)
        out = {}
        for k, l in enumerate(spec["layers"]):
            if l["kind"] in ("CBCONV", "CONV"):
                g = dict(_geom_dict(l), inChannels=in_ch[k])
                out[k] = self.random_filters(g, seed + k + 1)
        return out

    # ---- network -----------------------------------------------------
    def load_network(self, spec: dict, weights: dict) -> "OracleNet":
        return OracleNet(self, spec, weights)


def _geom_dict(l: dict) -> dict:
    return dict(kernelH=l["kernelH"], kernelW=l["kernelW"], strideH=l.get("strideH", 1),
                strideW=l.get("strideW", 1), padH=l.get("padH", 0), padW=l.get("padW", 0),
                inChannels=l.get("inChannels", 0), outChannels=l["outChannels"])


class OracleNet:
    def __init__(self, orc: Oracle, spec: dict, weights: dict):
        self.orc, self.lib, self.spec = orc, orc.lib, spec
        arr = _layers_array(spec)
        h = C.c_void_p()
        rc = self.lib.orc_net_create(spec["inputChannels"], spec["inputHeight"], spec["inputWidth"],
                                     spec["numClasses"], arr, len(spec["layers"]), C.byref(h))
        if rc:
            raise OracleError(rc)
        self.h = h
        self.nl = len(spec["layers"])
        self.shapes, _ = orc.chain_dims(spec)
        for k, (K, b) in weights.items():
            K, pk = _f32(K)
            b, pb = _f32(b)
            self.lib.orc_net_set_weights(self.h, k, pk, pb)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_net_free(self.h)
            self.h = None

    def reset_state(self):
        self.lib.orc_net_reset(self.h)

    def set_thresholds(self, taus):
        t = (C.c_float * len(taus))(*taus)
        rc = self.lib.orc_net_set_thresholds(self.h, t, len(taus))
        if rc:
            raise OracleError(rc)

    def forward_frame(self, frame, engine="cbinfer"):
        frame, pf = _f32(frame)
        hw = self.shapes[-1][0][1:] if self.spec["layers"][-1]["kind"] == "CLASSIFY" else self.shapes[-1][1][1:]
        labels = np.zeros(hw, np.uint16)
        st = (Stats * self.nl)()
        macs = C.c_uint64()
        rc = self.lib.orc_forward_frame(self.h, pf, 1 if engine == "cbinfer" else 0,
                                        labels.ctypes.data_as(C.POINTER(C.c_uint16)), st, C.byref(macs))
        if rc:
            raise OracleError(rc)
        stats = [dict(changedInputPixels=s.changedInputPixels, changedOutputPixels=s.changedOutputPixels,
                      gemmMacs=s.gemmMacs) for s in st]
        return dict(labels=labels, stats=stats, macsTotal=macs.value)

    def warm(self, frame, nthreads):
        frame, pf = _f32(frame)
        self.lib.orc_net_warm(self.h, pf, int(nthreads))

    def copy_state_from(self, other: "OracleNet"):
        self.lib.orc_net_copy_state(self.h, other.h)

    def layer_output(self, k):
        p = C.POINTER(C.c_float)()
        d = (C.c_int * 3)()
        self.lib.orc_net_layer_output(self.h, k, C.byref(p), d)
        n = d[0] * d[1] * d[2]
        return np.ctypeslib.as_array(p, shape=(n,)).reshape(d[0], d[1], d[2]).copy()

    def final_activation(self):
        p = C.POINTER(C.c_float)()
        d = (C.c_int * 3)()
        self.lib.orc_net_final_activation(self.h, C.byref(p), d)
        n = d[0] * d[1] * d[2]
        return np.ctypeslib.as_array(p, shape=(n,)).reshape(d[0], d[1], d[2]).copy()

    def trace(self, cb):
        det = C.POINTER(C.c_uint8)()
        d = (C.c_int * 2)()
        up = C.POINTER(C.c_int32)()
        n = C.c_int64()
        rc = self.lib.orc_net_trace(self.h, cb, C.byref(det), d, C.byref(up), C.byref(n))
        if rc:
            raise OracleError(rc)
        detected = None
        if det:
            detected = np.ctypeslib.as_array(det, shape=(d[0] * d[1],)).reshape(d[0], d[1]).copy()
        updated = np.ctypeslib.as_array(up, shape=(max(n.value, 1),))[: n.value].copy()
        return detected, updated


class Ref:
    """The unmodified reference library (oracle/_ref/libcbinfer_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = L = C.CDLL(path)
        L.ref_detect_changes.restype = C.c_int64
        L.ref_extract_indexes.restype = C.c_int64
        L.ref_last_error.restype = C.c_char_p

    def _chk(self, rc):
        if rc < 0:
            raise OracleError(rc, self.lib.ref_last_error().decode())
        return rc

    @staticmethod
    def _g(g):
        return (C.c_int * 8)(g["kernelH"], g["kernelW"], g["strideH"], g["strideW"], g["padH"],
                             g["padW"], g["inChannels"], g["outChannels"])

    def detect_changes(self, cur, prev, tau):
        cur, pc = _f32(cur)
        prev, pp = _f32(prev)
        c, h, w = cur.shape
        m = np.zeros((h, w), np.uint8)
        self._chk(self.lib.ref_detect_changes(pc, pp, c, h, w, C.c_float(tau),
                                              m.ctypes.data_as(C.POINTER(C.c_uint8))))
        return m

    def dilate_changes(self, m, g):
        m, pm = _u8(m)
        ho, wo = out_hw(g, *m.shape)
        out = np.zeros((max(ho, 0), max(wo, 0)), np.uint8)
        self._chk(self.lib.ref_dilate_changes(pm, m.shape[0], m.shape[1], self._g(g),
                                              out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out

    def extract_indexes(self, m):
        m, pm = _u8(m)
        idx = np.zeros(m.size, np.int32)
        n = self._chk(self.lib.ref_extract_indexes(pm, m.shape[0], m.shape[1],
                                                   idx.ctypes.data_as(C.POINTER(C.c_int32))))
        return idx[:n].copy()

    def conv_full(self, inp, K, bias, g):
        inp, pi = _f32(inp)
        K, pk = _f32(K)
        bias, pb = _f32(bias)
        ho, wo = out_hw(g, inp.shape[1], inp.shape[2])
        out = np.zeros((g["outChannels"], ho, wo), np.float32)
        self._chk(self.lib.ref_conv_full(pi, *inp.shape, pk, pb, self._g(g),
                                         out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def maxpool(self, t, window, stride):
        t, pt = _f32(t)
        c, h, w = t.shape
        out = np.zeros((c, (h - window) // stride + 1, (w - window) // stride + 1), np.float32)
        self._chk(self.lib.ref_maxpool(pt, c, h, w, window, stride, out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def synth_frame(self, cfg: dict, f: int):
        sp = cfg.get("sprites", [])
        n = len(sp)
        sizes = (C.c_int * max(1, n))(*[s[0] for s in sp])
        vels = (C.c_int * max(1, n))(*[s[1] for s in sp])
        ints = (C.c_float * max(1, n))(*[s[2] for s in sp])
        ch, h, w = cfg.get("channels", 3), cfg.get("height", 64), cfg.get("width", 64)
        out = np.zeros((ch, h, w), np.float32)
        self._chk(self.lib.ref_synth_frame(ch, h, w, n, sizes, vels, ints, C.c_float(cfg.get("noise", 0.0)),
                                           C.c_uint32(int(cfg.get("seed", 1)) & 0xFFFFFFFF), f,
                                           out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def random_filters(self, g, seed):
        cols = g["inChannels"] * g["kernelH"] * g["kernelW"]
        K = np.zeros((g["outChannels"], cols), np.float32)
        b = np.zeros(g["outChannels"], np.float32)
        self._chk(self.lib.ref_random_filters(self._g(g), C.c_uint32(seed & 0xFFFFFFFF),
                                              K.ctypes.data_as(C.POINTER(C.c_float)),
                                              b.ctypes.data_as(C.POINTER(C.c_float))))
        return K, b

    def load_network(self, spec: dict, seed: int, weights_dir: str | None = None) -> "RefNet":
        return RefNet(self, spec, seed, weights_dir)


def _spec_json_for_ref(spec: dict) -> str:
    doc = dict(inputChannels=spec["inputChannels"], inputHeight=spec["inputHeight"],
               inputWidth=spec["inputWidth"], numClasses=spec["numClasses"], layers=[])
    for k, l in enumerate(spec["layers"]):
        jl = {kk: vv for kk, vv in l.items() if kk != "inChannels"}
        if l["kind"] in ("CBCONV", "CONV") and "weightsFile" not in jl:
            jl["weightsFile"] = f"layer{k + 1}.weights.f32le"
        doc["layers"].append(jl)
    return json.dumps(doc)


class RefNet:
    """A reference Network loaded through its own JSON parser + weight files,
    driven through its own forward_frame (network.cpp:252-315)."""

    def __init__(self, ref: Ref, spec: dict, seed: int, weights_dir: str | None):
        self.ref, self.lib = ref, ref.lib
        self._tmp = None
        js = _spec_json_for_ref(spec).encode()
        if weights_dir is None:
            self._tmp = tempfile.TemporaryDirectory(prefix="cbx_ref_w_")
            weights_dir = self._tmp.name
            ref._chk(self.lib.ref_generate_weights(js, weights_dir.encode(), C.c_uint32(seed)))
        h = C.c_void_p()
        ref._chk(self.lib.ref_net_load(js, weights_dir.encode(), C.byref(h)))
        self.h = h
        self.spec = spec
        self.nl = len(spec["layers"])
        self.weights_dir = weights_dir

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_net_free(self.h)
            self.h = None

    def reset_state(self):
        self.lib.ref_net_reset(self.h)

    def set_thresholds(self, taus):
        t = (C.c_float * len(taus))(*taus)
        self.ref._chk(self.lib.ref_net_set_thresholds(self.h, t, len(taus)))

    def forward_frame(self, frame, engine="cbinfer", trace=True, labels_shape=None):
        frame, pf = _f32(frame)
        labels = np.zeros(labels_shape, np.uint16) if labels_shape else None
        st = (C.c_int64 * (3 * self.nl))()
        macs = C.c_uint64()
        self.ref._chk(self.lib.ref_forward_frame(
            self.h, pf, 1 if engine == "cbinfer" else 0,
            labels.ctypes.data_as(C.POINTER(C.c_uint16)) if labels is not None else None,
            st, C.byref(macs), int(trace)))
        stats = [dict(changedInputPixels=st[3 * k], changedOutputPixels=st[3 * k + 1],
                      gemmMacs=st[3 * k + 2]) for k in range(self.nl)]
        return dict(labels=labels, stats=stats, macsTotal=macs.value)

    def calibrate(self, frames, grid_size=16, budget=1.0):
        """Reference default_threshold_grids + calibrate_thresholds over one
        sequence (calibration.cpp:73-170): (thresholds, [(layer, tau, err)])."""
        fr = np.ascontiguousarray(np.stack(frames), np.float32)
        ncb = sum(l["kind"] == "CBCONV" for l in self.spec["layers"])
        th = (C.c_float * max(1, ncb))()
        n = ncb * grid_size
        lay, tau, err = (C.c_int * n)(), (C.c_float * n)(), (C.c_double * n)()
        self.ref._chk(self.lib.ref_calibrate(self.h, fr.ctypes.data_as(C.POINTER(C.c_float)), len(frames),
                                             int(grid_size), C.c_double(budget), th, lay, tau, err))
        return [th[k] for k in range(ncb)], [(lay[i], tau[i], err[i]) for i in range(n)]

    def sweep(self, frames, factors):
        """Reference sweep_threshold_factor over one sequence
        (calibration.cpp:172-240): [(errorIncrease, changedPixelsTotal, macsTotal)]."""
        fr = np.ascontiguousarray(np.stack(frames), np.float32)
        nf = len(factors)
        fa = (C.c_double * nf)(*factors)
        err, ch, macs = (C.c_double * nf)(), (C.c_int64 * nf)(), (C.c_uint64 * nf)()
        self.ref._chk(self.lib.ref_sweep(self.h, fr.ctypes.data_as(C.POINTER(C.c_float)), len(frames), fa, nf,
                                         err, ch, macs))
        return [(err[i], ch[i], macs[i]) for i in range(nf)]

    def warm(self, frame, nthreads):
        frame, pf = _f32(frame)
        self.ref._chk(self.lib.ref_net_warm(self.h, pf, int(nthreads)))

    def copy_state_from(self, other: "RefNet"):
        self.ref._chk(self.lib.ref_net_copy_state(self.h, other.h))

    def final_activation(self):
        p = C.POINTER(C.c_float)()
        d = (C.c_int * 3)()
        self.lib.ref_net_final_activation(self.h, C.byref(p), d)
        n = d[0] * d[1] * d[2]
        return np.ctypeslib.as_array(p, shape=(n,)).reshape(d[0], d[1], d[2]).copy()

    def trace(self, cb):
        det = C.POINTER(C.c_uint8)()
        d = (C.c_int * 2)()
        up = C.POINTER(C.c_int32)()
        n = C.c_int64()
        self.ref._chk(self.lib.ref_net_trace(self.h, cb, C.byref(det), d, C.byref(up), C.byref(n)))
        detected = None
        if det:
            detected = np.ctypeslib.as_array(det, shape=(d[0] * d[1],)).reshape(d[0], d[1]).copy()
        updated = np.ctypeslib.as_array(up, shape=(max(n.value, 1),))[: n.value].copy() if n.value else np.zeros(0, np.int32)
        return detected, updated
