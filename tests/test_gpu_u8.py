"""GPU: the native 8-bit camera path (CBX_OPT_U8_NATIVE, tensor-core
precisions): change detection on the frame bytes fused with the RGBX copy of
the frame, and layer 1 as a tcgen05 kind::i8 conv over those bytes with the
filters split into three 8-bit digits of a 22-bit fixed-point weight.

Parity bar (north star): layer-1 change masks and index lists bit-exact
against the oracle on read_ppm's tensors (px / 255.0f, io.cpp:60-104);
layer-1 outputs within 2^-16 * sum|w x| + 1e-6 of the reference (the exact
integer accumulation leaves only the 2^-23 weight quantization, far inside
the 2^-9 tensor-core bound of the deeper layers); final activations and
labels within the network tolerance; change-based == dense at tau = 0."""
import numpy as np
import pytest

from netutil import bits, paper_spec, stats_arr, to_pkg_spec

pytestmark = pytest.mark.gpu


def u8_clip(orc, h, w, frames, seed, sprites, noise=0.0):
    cfg = dict(channels=3, height=h, width=w, sprites=sprites, noise=noise, seed=seed)
    return [np.ascontiguousarray(np.clip(np.rint(orc.synth_frame(cfg, f).transpose(1, 2, 0) * 255.0), 0, 255)
                                 .astype(np.uint8)) for f in range(frames)]


def decode(x):
    """read_ppm: planar float32 px / 255.0f."""
    return np.ascontiguousarray((x.astype(np.float32) / np.float32(255.0)).transpose(2, 0, 1))


def im2col_abs(x, K, kh, kw, ph, pw):
    """sum_r |K[o, r]| * |X[r, p]| per output pixel (the error-bound scale)."""
    C, H, W = x.shape
    O = K.shape[0]
    xp = np.pad(np.abs(x), ((0, 0), (ph, ph), (pw, pw)))
    Ho, Wo = H + 2 * ph - kh + 1, W + 2 * pw - kw + 1
    Ka = np.abs(K).reshape(O, C, kh, kw)
    out = np.zeros((O, Ho, Wo), np.float64)
    for c in range(C):
        for j in range(kh):
            for i in range(kw):
                out += Ka[:, c, j, i][:, None, None] * xp[c, j:j + Ho, i:i + Wo][None]
    return out


@pytest.mark.parametrize("prec", ["f16", "tf32"])
@pytest.mark.parametrize("h,w,noise", [(48, 64, 0.01), (64, 96, 0.0), (40, 80, 0.03)])
def test_native_u8_layer1(gpu, orc, prec, h, w, noise):
    spec = paper_spec(h, w)
    wts = orc.generate_weights(spec, 1)
    onet = orc.load_network(spec, wts)
    net = gpu.Network(to_pkg_spec(gpu, spec), wts, precision=prec)
    assert net.layer_operands(0) == "i8"
    K0, b0 = wts[0]
    clip = u8_clip(orc, h, w, 5, 3, [(12, 2, 0.9), (7, 3, 0.6)], noise)
    for f, fr in enumerate(clip):
        want = onet.forward_frame(decode(fr))
        got = net.forward_u8(fr)[0]
        # layer 1: masks, index lists and counters bit-exact
        d1, u1 = net.trace(0)
        d2, u2 = onet.trace(0)
        assert (d1 is None) == (d2 is None)
        if d1 is not None:
            rows = np.nonzero((d1 != d2).any(axis=1))[0]
            assert np.array_equal(d1, d2), (f, rows.tolist(), int(d1.sum()), int(d2.sum()),
                                            np.array_equal(net.layer_input(0).view(np.uint32), decode(fr).view(np.uint32)))
        assert np.array_equal(u1, u2), f
        assert np.array_equal(stats_arr(got.stats)[0], stats_arr(want["stats"])[0]), f
        # layer-1 outputs: exact integer accumulation, 2^-23 weight quantization
        ref = onet.layer_output(0)
        scale = im2col_abs(decode(fr), K0, 7, 7, 3, 3) + np.abs(b0)[:, None, None]
        err = np.abs(net.layer_output(0).astype(np.float64) - ref)
        assert (err <= 2.0 ** -16 * scale + 1e-6).all(), (f, err.max())
        # the rest of the network within the tensor-core tolerance
        assert (got.labels != want["labels"]).sum() <= max(1, 1e-3 * got.labels.size), f


@pytest.mark.parametrize("prec", ["f16", "tf32"])
def test_native_u8_tau0_cb_equals_baseline(gpu, orc, prec):
    """test_network.cpp:176-199 on the 8-bit path: at tau = 0 the change-based
    engine equals the dense engine bitwise (same kernels), and both stay within
    the network tolerance of the reference."""
    h, w = 64, 96
    spec = paper_spec(h, w, (0.0, 0.0, 0.0))
    wts = orc.generate_weights(spec, 1)
    onet = orc.load_network(spec, wts)
    net = gpu.Network(to_pkg_spec(gpu, spec), wts, precision=prec)
    for f, fr in enumerate(u8_clip(orc, h, w, 4, 5, [(12, 2, 0.9)], 0.01)):
        want = onet.forward_frame(decode(fr))
        cb = net.forward_u8(fr)[0]
        act_cb = net.final_activation()
        dense = net.forward_u8(fr, engine="baseline")[0]
        assert np.array_equal(cb.labels, dense.labels), f
        assert np.array_equal(bits(act_cb), bits(net.final_activation(engine="baseline"))), f
        assert np.abs(act_cb - onet.final_activation()).max() <= 1e-3
        assert (cb.labels != want["labels"]).mean() <= 1e-3


def test_native_u8_matches_decoded_path(gpu, orc):
    """Native 8-bit path vs the decode path (CBX_OPT_U8_NATIVE = 0, bitwise the
    fp32 path): identical layer-1 masks / index lists / counters on every frame
    of a 2-lane 4-stream context; deeper layers differ only near tau
    (mismatch <= 1 % of the detected pixels)."""
    h, w, S = 64, 128, 4
    spec = paper_spec(h, w)
    wts = orc.generate_weights(spec, 1)
    a = gpu.Network(to_pkg_spec(gpu, spec), wts, streams=S, precision="f16", lanes=2)
    b = gpu.Network(to_pkg_spec(gpu, spec), wts, streams=S, precision="f16", lanes=2)
    b.set_u8_native(False)
    assert a.num_lanes() == 2
    clips = [u8_clip(orc, h, w, 5, 10 + s, [(14, 2 + s, 0.9)], 0.005 * s) for s in range(S)]
    for f in range(5):
        x = np.ascontiguousarray(np.stack([clips[s][f] for s in range(S)]))
        ra, rb = a.forward_u8(x), b.forward_u8(x)
        for s in range(S):
            assert np.array_equal(stats_arr(ra[s].stats)[0], stats_arr(rb[s].stats)[0]), (f, s)
            assert np.array_equal(a.trace(0, s)[1], b.trace(0, s)[1]), (f, s)
            for cb in (1, 2):
                da, _ = a.trace(cb, s)
                db, _ = b.trace(cb, s)
                if da is not None:
                    assert np.count_nonzero(da != db) <= max(1, 0.01 * np.count_nonzero(db)), (f, s, cb)
            assert (ra[s].labels != rb[s].labels).sum() <= max(1, 1e-3 * ra[s].labels.size)


def test_native_u8_format_switch_and_device_frames(gpu, orc):
    """History across frame formats: 8-bit (native), fp32, 8-bit, 8-bit from
    device buffers (cbx_forward_device_u8), pipelined submits -- the layer-1
    detection always equals the reference's on read_ppm's tensors."""
    import torch
    h, w = 48, 64
    spec = paper_spec(h, w)
    wts = orc.generate_weights(spec, 1)
    onet = orc.load_network(spec, wts)
    net = gpu.Network(to_pkg_spec(gpu, spec), wts, precision="f16")
    clip = u8_clip(orc, h, w, 8, 4, [(10, 3, 0.9)], 0.01)
    dev = [torch.from_numpy(fr).cuda() for fr in clip]
    for f, fr in enumerate(clip):
        want = onet.forward_frame(decode(fr))
        if f == 2:
            got = net.forward(decode(fr))[0]  # fp32 frame after 8-bit history
        elif f in (4, 5):
            net.forward_device_u8([dev[f].data_ptr()])
            net.sync()
            got = None
        else:
            got = net.forward_u8(fr)[0]
        d1, u1 = net.trace(0)
        d2, u2 = onet.trace(0)
        if d1 is not None:
            assert np.array_equal(d1, d2), f
        assert np.array_equal(u1, u2), f
        stats, _ = net.read_stats()
        assert np.array_equal(stats_arr(stats[0])[0], stats_arr(want["stats"])[0]), f
        if got is not None:
            assert (got.labels != want["labels"]).sum() <= max(1, 1e-3 * got.labels.size)
        # prevInput of layer 1 is the decoded frame whichever path ran
        assert np.array_equal(net.layer_input(0).view(np.uint32), decode(fr).view(np.uint32)), f
    # pipelined 8-bit submits equal synchronous native forwards bitwise
    p = gpu.Network(to_pkg_spec(gpu, spec), wts, precision="f16")
    q = gpu.Network(to_pkg_spec(gpu, spec), wts, precision="f16")
    labs = [np.zeros((1,) + tuple(p.label_hw), np.uint16) for _ in clip]
    tickets = []
    for f, fr in enumerate(clip):
        tickets.append(p.submit_u8(fr[None], labs[f]))
        if len(tickets) >= 2:
            p.wait(tickets[-2])
    p.wait(tickets[-1])
    for f, fr in enumerate(clip):
        r = q.forward_u8(fr)[0]
        assert np.array_equal(labs[f][0], r.labels), f


def test_native_u8_odd_width_falls_back(gpu, orc):
    """Widths not divisible by 16 decode to fp32 (layer 1 stays bitwise)."""
    h, w = 54, 74
    spec = paper_spec(h, w)
    wts = orc.generate_weights(spec, 1)
    net = gpu.Network(to_pkg_spec(gpu, spec), wts, precision="f16")
    assert net.layer_operands(0) == "fp32"
    onet = orc.load_network(spec, wts)
    for fr in u8_clip(orc, h, w, 3, 2, [(9, 2, 0.9)], 0.01):
        onet.forward_frame(decode(fr))
        net.forward_u8(fr)
        assert np.array_equal(bits(net.layer_output(0)), bits(onet.layer_output(0)))


def test_native_u8_weight_dynamic_range(gpu, orc):
    """Per-channel digit scaling: one output channel with weights ~1e3, one with
    ~1e-4, one all zero -- each within 2^-16 of its own scale."""
    h, w = 32, 48
    spec = paper_spec(h, w, (0.0, 0.0, 0.0))
    wts = orc.generate_weights(spec, 1)
    K0, b0 = wts[0]
    K0 = K0.copy()
    K0[0] *= 1.0e4
    K0[1] *= 1.0e-3
    K0[2] = 0.0
    wts = dict(wts)
    wts[0] = (K0, b0)
    onet = orc.load_network(spec, wts)
    net = gpu.Network(to_pkg_spec(gpu, spec), wts, precision="tf32", fuse_tail=False)
    for fr in u8_clip(orc, h, w, 2, 6, [(8, 2, 0.9)], 0.05):
        onet.forward_frame(decode(fr))
        net.forward_u8(fr)
        ref = onet.layer_output(0)
        scale = im2col_abs(decode(fr), K0, 7, 7, 3, 3) + np.abs(b0)[:, None, None]
        err = np.abs(net.layer_output(0).astype(np.float64) - ref)
        assert (err <= 2.0 ** -16 * scale + 1e-6).all(), err.max()


@pytest.mark.parametrize("tau", [0.0, 0.04, float(np.float32(10) / np.float32(255)), float(np.float32(3) / np.float32(255)), 0.5])
def test_native_u8_detect_any_tau(gpu, orc, tau):
    """The byte-difference shortcut of the 8-bit detection is exact for every
    tau, including taus that sit on a k / 255 boundary (the pairs with
    |a - b| = k then split by rounding and take the exact decode path):
    layer-1 masks, index lists and counters equal the oracle's."""
    h, w = 48, 96
    spec = paper_spec(h, w, (tau, 0.05, 0.05))
    wts = orc.generate_weights(spec, 1)
    onet = orc.load_network(spec, wts)
    net = gpu.Network(to_pkg_spec(gpu, spec), wts, precision="f16")
    # noisy clip: every byte difference class occurs
    for f, fr in enumerate(u8_clip(orc, h, w, 4, 8, [(10, 2, 0.9)], 0.06)):
        want = onet.forward_frame(decode(fr))
        got = net.forward_u8(fr)[0]
        d1, u1 = net.trace(0)
        d2, u2 = onet.trace(0)
        if d1 is not None:
            assert np.array_equal(d1, d2), (tau, f)
        assert np.array_equal(u1, u2), (tau, f)
        assert np.array_equal(stats_arr(got.stats)[0], stats_arr(want["stats"])[0]), (tau, f)
