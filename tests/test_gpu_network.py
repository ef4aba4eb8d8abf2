"""GPU: network-level parity of the CUDA engine (through the C-ABI) with the
oracle restatement, which is itself pinned to the reference (test_oracle.py).

Exact mode (CBX_PREC_EXACT) must be BIT-EXACT in everything: labels, stats,
every layer's activation, change masks and index lists. TF32 mode (tcgen05)
keeps layer-1 masks/indices/outputs bit-exact and stays within the stated
tolerance elsewhere (max-abs 1e-3 of final activations at tau=0, label
disagreement <= 0.1%)."""
import numpy as np
import pytest

from netutil import bits, c1_spec, generic_spec, paper_spec, stats_arr, tiny_spec, to_pkg_spec

pytestmark = pytest.mark.gpu


def run_pair(cbx, orc, spec, seed, cfg, frames, precision="exact", streams=1, check_layers=True):
    w = orc.generate_weights(spec, seed)
    onet = orc.load_network(spec, w)
    net = cbx.Network(to_pkg_spec(cbx, spec), w, streams=streams, precision=precision)
    ncb = sum(l["kind"] == "CBCONV" for l in spec["layers"])
    for f in range(frames):
        fr = orc.synth_frame(cfg, f)
        want = onet.forward_frame(fr)
        got = net.forward(np.stack([fr] * streams))
        for s in range(streams):
            yield f, s, want, got[s], onet, net, ncb


@pytest.mark.parametrize("name,spec,seed,cfg,frames", [
    ("c1", c1_spec(), 1, dict(channels=16, height=128, width=128, sprites=[(24, 7, 0.9)], seed=2), 8),
    ("paper48", paper_spec(48, 64), 1, dict(channels=3, height=48, width=64, sprites=[(10, 2, 0.9)], noise=0.01, seed=3), 5),
    # width not a multiple of 4 (scalar detection path), odd pooled sizes (27x37 -> 13x18)
    ("paper_odd", paper_spec(54, 74), 1, dict(channels=3, height=54, width=74, sprites=[(9, 2, 0.9)], noise=0.01, seed=5), 5),
    ("tiny_tau0", tiny_spec(), 42, dict(channels=2, height=16, width=16, sprites=[(5, 1, 0.9)], noise=0.03, seed=7), 5),
    ("generic", generic_spec(), 5, dict(channels=3, height=37, width=45, sprites=[(6, 2, 0.8)], noise=0.015, seed=9), 6),
])
def test_exact_bitwise(gpu, orc, name, spec, seed, cfg, frames):
    for f, s, want, got, onet, net, ncb in run_pair(gpu, orc, spec, seed, cfg, frames):
        assert np.array_equal(got.labels, want["labels"]), (name, f)
        assert np.array_equal(stats_arr(got.stats), stats_arr(want["stats"])), (name, f)
        assert got.macsTotal == want["macsTotal"]
        for k, l in enumerate(spec["layers"]):
            if l["kind"] == "CLASSIFY":
                continue
            assert np.array_equal(bits(net.layer_output(k)), bits(onet.layer_output(k))), (name, f, k)
        for cb in range(ncb):
            d1, u1 = net.trace(cb)
            d2, u2 = onet.trace(cb)
            assert (d1 is None) == (d2 is None)
            if d1 is not None:
                assert np.array_equal(d1, d2), (name, f, cb)
            assert np.array_equal(u1, u2), (name, f, cb)


def test_golden_c1_direct(gpu, orc, golden):
    """The CUDA path against the reference's own recorded outputs (no oracle)."""
    import json
    d = golden("c1.npz")
    spec = json.loads(str(d["spec"][0]))
    cfg = json.loads(str(d["synth"][0]))
    w = gpu.generate_weights(to_pkg_spec(gpu, spec), None, int(d["seed"][0]))
    net = gpu.Network(to_pkg_spec(gpu, spec), w, precision="exact")
    for f in range(8):
        r = net.forward_frame(gpu.synth_frame(cfg, f))
        assert np.array_equal(r.labels, d[f"f{f}_labels"])
        assert np.array_equal(stats_arr(r.stats), d[f"f{f}_stats"])
        det, upd = net.trace(0)
        assert np.array_equal(upd, d[f"f{f}_cb0_upd"])
        if det is not None:
            assert np.array_equal(np.packbits(det.reshape(-1)), d[f"f{f}_cb0_det"])


def test_tau0_cb_equals_baseline_gpu(gpu, orc):
    """test_network.cpp:176-199 on the GPU engine, both precisions: CB == Baseline bitwise."""
    spec = tiny_spec(0.0)
    w = orc.generate_weights(spec, 42)
    cfg = dict(channels=2, height=16, width=16, sprites=[(5, 1, 0.9)], noise=0.03, seed=7)
    for prec in ("exact", "tf32"):
        net = gpu.Network(to_pkg_spec(gpu, spec), w, precision=prec)
        for f in range(5):
            fr = orc.synth_frame(cfg, f)
            a = net.forward_frame(fr, "cbinfer")
            fa = net.final_activation(engine="cbinfer")
            b = net.forward_frame(fr, "baseline")
            fb = net.final_activation(engine="baseline")
            assert np.array_equal(bits(fa), bits(fb)), (prec, f)
            assert np.array_equal(a.labels, b.labels)


def test_static_scene_and_reset(gpu, orc):
    """test_network.cpp:163-174 and :236-257."""
    spec = paper_spec(32, 48, (0.02, 0.05, 0.05))
    w = orc.generate_weights(spec, 99)
    net = gpu.Network(to_pkg_spec(gpu, spec), w, precision="exact")
    fr = np.random.default_rng(71).random((3, 32, 48), dtype=np.float32)
    first = net.forward_frame(fr)
    assert first.macsTotal > 0
    second = net.forward_frame(fr)
    for cb in net.spec.cb_layers():
        assert second.stats[cb]["gemmMacs"] == 0
    assert np.array_equal(first.labels, second.labels)
    net.reset_state()
    again = net.forward_frame(fr)
    assert again.macsTotal == first.macsTotal
    assert np.array_equal(again.labels, first.labels)
    assert np.array_equal(stats_arr(again.stats), stats_arr(first.stats))


def test_baseline_leaves_cb_state(gpu, orc):
    """network.cpp:278-285: interleaved Baseline frames do not disturb the CB state."""
    spec = paper_spec(48, 64)
    w = orc.generate_weights(spec, 1)
    cfg = dict(channels=3, height=48, width=64, sprites=[(10, 2, 0.9)], noise=0.01, seed=3)
    onet = orc.load_network(spec, w)
    net = gpu.Network(to_pkg_spec(gpu, spec), w, precision="exact")
    for f in range(4):
        fr = orc.synth_frame(cfg, f)
        net.forward_frame(orc.synth_frame(cfg, f + 7), "baseline")
        got = net.forward_frame(fr, "cbinfer")
        want = onet.forward_frame(fr)
        assert np.array_equal(got.labels, want["labels"])
        assert np.array_equal(stats_arr(got.stats), stats_arr(want["stats"]))


def test_multistream_independent(gpu, orc):
    """Streams batched in one context behave like independent Networks."""
    spec = paper_spec(40, 56)
    w = orc.generate_weights(spec, 3)
    S = 3
    cfgs = [dict(channels=3, height=40, width=56, sprites=[(8, 1 + s, 0.9)], noise=0.005 * s, seed=10 + s)
            for s in range(S)]
    onets = [orc.load_network(spec, w) for _ in range(S)]
    net = gpu.Network(to_pkg_spec(gpu, spec), w, streams=S, precision="exact")
    for f in range(4):
        frames = [orc.synth_frame(c, f) for c in cfgs]
        got = net.forward(np.stack(frames))
        for s in range(S):
            want = onets[s].forward_frame(frames[s])
            assert np.array_equal(got[s].labels, want["labels"]), (f, s)
            assert np.array_equal(stats_arr(got[s].stats), stats_arr(want["stats"])), (f, s)
            for cb in range(3):
                assert np.array_equal(net.trace(cb, s)[1], onets[s].trace(cb)[1])


@pytest.mark.parametrize("prec", ["f16", "tf32"])
def test_tf32_tolerance(gpu, orc, prec):
    """Tensor-core modes at tau=0: layer-1 masks/indices/outputs bit-exact,
    final activations within 1e-3 max-abs, labels within 0.1% (tau > 0:
    test_tf32_mask_mismatch_counts). f16: layer 3 with fp16 operands; tf32:
    tf32 operands everywhere."""
    spec = paper_spec(64, 96, (0.0, 0.0, 0.0))
    w = orc.generate_weights(spec, 1)
    cfg = dict(channels=3, height=64, width=96, sprites=[(12, 2, 0.9)], noise=0.01, seed=3)
    onet = orc.load_network(spec, w)
    net = gpu.Network(to_pkg_spec(gpu, spec), w, precision=prec)
    for f in range(4):
        fr = orc.synth_frame(cfg, f)
        want = onet.forward_frame(fr)
        got = net.forward_frame(fr)
        assert np.array_equal(bits(net.layer_output(0)), bits(onet.layer_output(0)))
        d1, u1 = net.trace(0)
        d2, u2 = onet.trace(0)
        assert np.array_equal(u1, u2)
        err = np.abs(net.final_activation() - onet.final_activation()).max()
        assert err <= 1e-3, err
        assert (got.labels != want["labels"]).mean() <= 1e-3


@pytest.mark.parametrize("h,w,prec", [(96, 128, "f16"), (54, 74, "f16"), (96, 128, "tf32")])
def test_tf32_mask_mismatch_counts(gpu, orc, h, w, prec):
    """TF32 mode at the base taus (0.04, 0.05, 0.05) on a sprite clip: the
    per-CBCONV-layer changed-pixel mismatch counts against the oracle --
    popcount(detected_gpu XOR detected_ref) and |updated_gpu symdiff
    updated_ref| -- are 0 for layer 1 and bounded (<= 1% of the reference's
    count) for layers 2-3, where a tf32 activation can cross tau; labels within
    0.1% (at least one pixel). scripts/parity_report.py writes the same counts at 320x240 and 1080p
    against the compiled reference (profiles/r1_parity.json)."""
    spec = paper_spec(h, w, (0.04, 0.05, 0.05))
    wts = orc.generate_weights(spec, 1)
    cfg = dict(channels=3, height=h, width=w, sprites=[(16, 3, 0.9), (10, 2, 0.9)], noise=0.0, seed=3)
    onet = orc.load_network(spec, wts)
    net = gpu.Network(to_pkg_spec(gpu, spec), wts, precision=prec)
    counts = []
    for f in range(5):
        fr = orc.synth_frame(cfg, f)
        want = onet.forward_frame(fr)
        got = net.forward_frame(fr)
        if f == 0:
            continue
        for cb in range(3):
            dg, ug = net.trace(cb)
            dr, ur = onet.trace(cb)
            det_mis = int(np.count_nonzero(dg != dr))
            upd_mis = int(np.setxor1d(ug, ur).size)
            counts.append((f, cb, det_mis, int(np.count_nonzero(dr)), upd_mis, ur.size))
            if cb == 0:
                assert det_mis == 0 and upd_mis == 0, (f, det_mis, upd_mis)
            else:
                assert det_mis <= max(1, 0.01 * np.count_nonzero(dr)), (f, cb, det_mis)
                assert upd_mis <= max(1, 0.01 * ur.size), (f, cb, upd_mis)
        # 0.1 % of the label map, but at least one pixel (a 13x18 map has 234)
        assert (got.labels != want["labels"]).sum() <= max(1, 1e-3 * got.labels.size)
    assert any(c[3] > 0 for c in counts if c[1] == 2)  # the clip reaches layer 3


def test_layer_operands(gpu, orc):
    """Operand formats reported per conv layer: layer 1 kind::i8 for 8-bit
    frames (exact fp32 for planar fp32 frames), layer 2 tf32, layer 3 fp16 (fed by a MAXPOOL) under
    precision f16 and tf32 under precision tf32; the head's 1x1 convs exact;
    exact mode fp32 only."""
    spec = paper_spec(32, 48)
    w = orc.generate_weights(spec, 1)
    net = gpu.Network(to_pkg_spec(gpu, spec), w, precision="f16")
    # layer 1: kind::i8 for 8-bit frames (width 48 is a multiple of 16; fp32
    # frames take the exact path)
    assert [net.layer_operands(k) for k in (0, 2, 4, 5)] == ["i8", "tf32", "f16", "fp32"]
    assert net.layer_operands(1) == "none"  # MAXPOOL
    net2 = gpu.Network(to_pkg_spec(gpu, spec), w, precision="tf32")
    assert [net2.layer_operands(k) for k in (0, 2, 4, 5)] == ["i8", "tf32", "tf32", "fp32"]
    odd = paper_spec(32, 40)  # width not a multiple of 16: no 8-bit native path
    net3 = gpu.Network(to_pkg_spec(gpu, odd), orc.generate_weights(odd, 1), precision="tf32")
    assert net3.layer_operands(0) == "fp32"
    ex = gpu.Network(to_pkg_spec(gpu, spec), w, precision="exact")
    assert all(ex.layer_operands(k) == "fp32" for k in (0, 2, 4))


def test_f16_overflow_reported(gpu, orc):
    """Layer 3's fp16 operands only cover |x| <= 65504. The pool-2 shadow
    writer flags a larger value; the flag is sticky until a full evaluation,
    so the frame that overflowed AND every later change-based frame (whose
    outputs may still hold results computed from inf) fail when their stats
    are read, after which the next frame is evaluated in full and succeeds
    (tf32 operands take every frame). Weights are scaled so that pool-2
    peaks near 3e4 on frame A; frame B is A times 6."""
    h, w = 32, 48
    spec = paper_spec(h, w, (0.0, 0.0, 0.0))
    wts = orc.generate_weights(spec, 1)
    A = orc.synth_frame(dict(channels=3, height=h, width=w, sprites=[(6, 2, 0.9)], noise=0.0, seed=1), 0)
    probe = gpu.Network(to_pkg_spec(gpu, spec), wts, precision="tf32")
    probe.forward_frame(A)
    c = 3.0e4 / float(np.abs(probe.layer_output(3)).max())
    big = {k: ((K * c).astype(np.float32), (b * c).astype(np.float32)) if k == 0 else (K, b)
           for k, (K, b) in wts.items()}
    B = (A * 6.0).astype(np.float32)
    tf = gpu.Network(to_pkg_spec(gpu, spec), big, precision="tf32")
    tf.forward_frame(A)
    assert np.abs(tf.layer_output(3)).max() < 6.0e4
    tf.forward_frame(B)
    assert np.abs(tf.layer_output(3)).max() > 7.0e4  # B's pool-2 values leave the fp16 range
    net = gpu.Network(to_pkg_spec(gpu, spec), big, precision="f16")
    net.forward_frame(A)
    with pytest.raises(gpu.CbxError, match="fp16 operand overflow"):
        net.forward_frame(B)
    ok = net.forward_frame(A)  # evaluated in full after the error
    assert ok.stats[0]["changedInputPixels"] == h * w
    # pipelined: the overflowing frame and the incremental frame after it both report
    S = 1
    lab = [np.zeros((S,) + tuple(net.label_hw), np.uint16) for _ in range(4)]
    fr = [np.ascontiguousarray(x[None]) for x in (A, B, B, A)]
    t = [net.submit(fr[0], lab[0]), net.submit(fr[1], lab[1]), net.submit(fr[2], lab[2])]
    net.wait(t[0])
    with pytest.raises(gpu.CbxError, match="fp16 operand overflow"):
        net.wait(t[1])
    with pytest.raises(gpu.CbxError, match="fp16 operand overflow"):
        net.wait(t[2])
    t3 = net.submit(fr[3], lab[3])
    stats, _ = net.wait(t3)
    assert stats[0][0]["changedInputPixels"] == h * w  # full evaluation, no error
    fresh = gpu.Network(to_pkg_spec(gpu, spec), big, precision="f16")
    assert np.array_equal(fresh.forward_frame(A).labels, lab[3][0])
    with pytest.raises(gpu.CbxError, match="fp16 range"):
        gpu.Network(to_pkg_spec(gpu, spec), {k: (K * 1e7, b) for k, (K, b) in wts.items()}, precision="f16")


def test_errors(gpu, orc):
    spec = paper_spec(32, 48)
    w = orc.generate_weights(spec, 1)
    net = gpu.Network(to_pkg_spec(gpu, spec), w)
    with pytest.raises(gpu.ShapeError):
        net.forward_frame(np.zeros((3, 32, 47), np.float32))
    with pytest.raises(gpu.SpecError):
        net.set_thresholds([0.1, 0.1])
    with pytest.raises(gpu.SpecError):
        net.set_thresholds([0.1, -0.1, 0.1])
    net.set_thresholds([0.5, 0.25, 0.125])
    assert net.thresholds() == [0.5, 0.25, 0.125]


@pytest.mark.parametrize("precision", ["exact", "tf32"])
def test_submit_wait_pipelined(gpu, orc, precision):
    """cbx_submit / cbx_wait with two frames in flight reproduces the oracle
    frame by frame (exact mode bitwise; tf32 labels within tolerance) and
    matches the synchronous forward exactly."""
    spec = paper_spec(48, 64)
    w = orc.generate_weights(spec, 1)
    S = 2
    cfgs = [dict(channels=3, height=48, width=64, sprites=[(10, 2 + s, 0.9)], noise=0.01, seed=3 + s) for s in range(S)]
    onets = [orc.load_network(spec, w) for _ in range(S)]
    pipe = gpu.Network(to_pkg_spec(gpu, spec), w, streams=S, precision=precision)
    sync = gpu.Network(to_pkg_spec(gpu, spec), w, streams=S, precision=precision)
    F = 6
    frames = [np.ascontiguousarray(np.stack([orc.synth_frame(c, f) for c in cfgs])) for f in range(F)]
    labels = [np.zeros((S,) + tuple(pipe.label_hw), np.uint16) for _ in range(F)]
    tickets, results = [], []
    for f in range(F):
        tickets.append(pipe.submit(frames[f], labels[f]))
        if f >= 1:
            results.append(pipe.wait(tickets[f - 1]))
    results.append(pipe.wait(tickets[-1]))
    for f in range(F):
        ref = sync.forward(frames[f])
        stats, macs = results[f]
        for s in range(S):
            want = onets[s].forward_frame(frames[f][s])
            assert np.array_equal(labels[f][s], ref[s].labels), (f, s)
            assert np.array_equal(stats_arr(stats[s]), stats_arr(ref[s].stats)), (f, s)
            assert macs[s] == ref[s].macsTotal
            if precision == "exact":
                assert np.array_equal(labels[f][s], want["labels"]), (f, s)
                assert np.array_equal(stats_arr(stats[s]), stats_arr(want["stats"])), (f, s)
            else:
                assert (labels[f][s] != want["labels"]).mean() <= 1e-3
    with pytest.raises(gpu.CbxError):
        pipe.wait(tickets[0])  # expired: only the last 3 submissions can be waited on
    with pytest.raises(gpu.CbxError):
        pipe.wait(F + 5)


def _oracle_worst_counts(orc, spec, onet):
    """cbench analyze-prop (cbench.cpp:242-302) restated with the oracle's ops on
    the oracle's own trace of the last frame."""
    from oracle import make_geom
    dims, _ = orc.chain_dims(spec)
    cb = [k for k, l in enumerate(spec["layers"]) if l["kind"] == "CBCONV"]
    out = []
    for j in range(1, len(cb)):
        prev, nxt = cb[j - 1], cb[j]
        _, upd = onet.trace(j - 1)
        (_, h, w) = dims[prev][1]
        wave = np.zeros(h * w, np.uint8)
        wave[upd] = 1
        wave = wave.reshape(h, w)
        for li in range(prev + 1, nxt):
            l = spec["layers"][li]
            if l["kind"] == "MAXPOOL":
                wave = orc.dilate_changes(wave, make_geom(l["window"], l["stride"], 0))
            elif l["kind"] == "CONV":
                wave = orc.dilate_changes(wave, make_geom(l["kernelH"], l.get("strideH", 1), l.get("padH", 0),
                                                          kw=l["kernelW"], stride_w=l.get("strideW", 1),
                                                          pad_w=l.get("padW", 0)))
        l = spec["layers"][nxt]
        g = make_geom(l["kernelH"], l.get("strideH", 1), l.get("padH", 0), kw=l["kernelW"],
                      stride_w=l.get("strideW", 1), pad_w=l.get("padW", 0))
        out.append(int(orc.dilate_changes(wave, g).sum()))
    return out


@pytest.mark.parametrize("name,spec,cfg", [
    ("paper", paper_spec(64, 96), dict(channels=3, height=64, width=96, sprites=[(12, 3, 0.9)], noise=0.01, seed=3)),
    ("generic", generic_spec(), dict(channels=3, height=37, width=45, sprites=[(6, 2, 0.8)], noise=0.015, seed=9)),
])
def test_worst_case_counts(gpu, orc, name, spec, cfg):
    """analyze-prop worst-case counts on the device == the oracle restatement,
    and never below the actual updated counts (the superset property)."""
    w = orc.generate_weights(spec, 1)
    onet = orc.load_network(spec, w)
    net = gpu.Network(to_pkg_spec(gpu, spec), w, precision="exact")
    net.forward_frame(orc.synth_frame(cfg, 0))
    onet.forward_frame(orc.synth_frame(cfg, 0))
    with pytest.raises(gpu.CbxError):
        net.worst_case_counts()  # first frame: full evaluation, nothing propagated
    cb = net.spec.cb_layers()
    for f in range(1, 4):
        fr = orc.synth_frame(cfg, f)
        got_frame = net.forward_frame(fr)
        onet.forward_frame(fr)
        worst = net.worst_case_counts()
        assert worst.shape == (1, len(cb) - 1)
        assert list(worst[0]) == _oracle_worst_counts(orc, spec, onet), (name, f)
        for j in range(1, len(cb)):
            assert worst[0, j - 1] >= got_frame.stats[cb[j]]["changedOutputPixels"]


def test_lanes_equivalent(gpu, orc):
    """Splitting the streams over 1, 2 or 3 lanes (independent engines on their
    own CUDA streams) gives identical labels, stats, traces and activations."""
    spec = paper_spec(40, 56)
    w = orc.generate_weights(spec, 3)
    S = 5
    cfgs = [dict(channels=3, height=40, width=56, sprites=[(8, 1 + s, 0.9)], noise=0.004 * s, seed=30 + s)
            for s in range(S)]
    nets = [gpu.Network(to_pkg_spec(gpu, spec), w, streams=S, precision="tf32", lanes=l) for l in (1, 2, 3)]
    assert [n.num_lanes() for n in nets] == [1, 2, 3]
    for f in range(4):
        fr = np.stack([orc.synth_frame(c, f) for c in cfgs])
        outs = [n.forward(fr) for n in nets]
        for o in outs[1:]:
            for s in range(S):
                assert np.array_equal(o[s].labels, outs[0][s].labels), (f, s)
                assert np.array_equal(stats_arr(o[s].stats), stats_arr(outs[0][s].stats)), (f, s)
        for s in range(S):
            ref_act = nets[0].layer_output(3, s)
            for n in nets[1:]:
                assert np.array_equal(bits(n.layer_output(3, s)), bits(ref_act))
                assert np.array_equal(n.trace(1, s)[1], nets[0].trace(1, s)[1])
    if f:
        w1 = nets[0].worst_case_counts()
        for n in nets[1:]:
            assert np.array_equal(n.worst_case_counts(), w1)


def test_step_times(gpu, orc):
    """CBX_OPT_STEP_TIMES: per-layer StepTimes from event nodes inside the
    frame graph (cbconv.hpp:44-52): first CBCONV has a detection interval,
    every CBCONV an extract (dilate + compact) and a multiply interval (the
    fused gather-conv-scatter); generate / update are fused (0); non-CB layers
    have none; results are unchanged by the timing nodes; off -> zeros."""
    spec = paper_spec(48, 64)
    w = orc.generate_weights(spec, 1)
    cfg = dict(channels=3, height=48, width=64, sprites=[(10, 2, 0.9)], noise=0.01, seed=3)
    timed = gpu.Network(to_pkg_spec(gpu, spec), w, precision="tf32", streams=2)
    plain = gpu.Network(to_pkg_spec(gpu, spec), w, precision="tf32", streams=2)
    timed.set_step_times(True)
    cb = timed.spec.cb_layers()
    for f in range(3):
        fr = np.stack([orc.synth_frame(dict(cfg, seed=3 + s), f) for s in range(2)])
        a, b = timed.forward(fr), plain.forward(fr)
        for s in range(2):
            assert np.array_equal(a[s].labels, b[s].labels)
        t = timed.step_times()
        assert t.shape == (2, len(spec["layers"]), 5)
        for k in range(len(spec["layers"])):
            if k not in cb:
                assert not t[:, k].any(), k
        for k in cb:
            assert (t[:, k, 3] > 0).all(), (f, k)                # multiply
            assert not t[:, k, 2].any() and not t[:, k, 4].any()  # generate / update fused
            if f > 0:
                assert (t[:, k, 1] > 0).all(), (f, k)            # extract
        assert (t[:, cb[0], 0] > 0).all() == (f > 0)             # detection only on steady frames
        assert not t[:, cb[1:], 0].any()
        assert not plain.step_times().any()
    assert timed.has_history()
    x = timed.layer_input(0, 1)
    assert np.array_equal(x.view(np.uint32), fr[1].view(np.uint32))
    assert np.array_equal(timed.layer_input(2, 0).view(np.uint32), timed.layer_output(1, 0).view(np.uint32))
    timed.reset_state()
    assert not timed.has_history()


@pytest.mark.parametrize("precision", ["exact", "f16"])
def test_u8_ingest_equals_decoded_frames(gpu, orc, precision):
    """8-bit camera frames (the PPM raster, io.cpp:60-104) through
    cbx_forward_u8 / cbx_submit_u8 with CBX_OPT_U8_NATIVE = 0 give bitwise the labels, stats, traces and
    activations of cbx_forward on the planar px / 255.0f frames read_ppm would
    produce (numpy float32 division is the same IEEE-rounded division)."""
    spec = paper_spec(48, 64)
    w = orc.generate_weights(spec, 1)
    S = 2
    rng = np.random.default_rng(5)
    clips = []
    for s in range(S):
        cfg = dict(channels=3, height=48, width=64, sprites=[(10, 2 + s, 0.9)], noise=0.01, seed=3 + s)
        clips.append([np.clip(np.rint(orc.synth_frame(cfg, f).transpose(1, 2, 0) * 255.0), 0, 255).astype(np.uint8)
                      for f in range(5)])
    u8 = [np.ascontiguousarray(np.stack([clips[s][f] for s in range(S)])) for f in range(5)]
    dec = [np.ascontiguousarray((x.astype(np.float32) / np.float32(255.0)).transpose(0, 3, 1, 2)) for x in u8]
    a = gpu.Network(to_pkg_spec(gpu, spec), w, streams=S, precision=precision)
    b = gpu.Network(to_pkg_spec(gpu, spec), w, streams=S, precision=precision)
    p = gpu.Network(to_pkg_spec(gpu, spec), w, streams=S, precision=precision)
    # the decode path (bitwise the fp32 path); the native 8-bit path is
    # covered by tests/test_gpu_u8.py
    a.set_u8_native(False)
    p.set_u8_native(False)
    labs = [np.zeros((S,) + tuple(p.label_hw), np.uint16) for _ in range(5)]
    tickets = [p.submit_u8(u8[f], labs[f]) for f in range(3)]
    waited = {t: p.wait(t) for t in tickets}
    for f in range(3, 5):
        tickets.append(p.submit_u8(u8[f], labs[f]))
        waited[tickets[-1]] = p.wait(tickets[-1])
    for f in range(5):
        ra, rb = a.forward_u8(u8[f]), b.forward(dec[f])
        for s in range(S):
            assert np.array_equal(ra[s].labels, rb[s].labels), (f, s)
            assert np.array_equal(labs[f][s], rb[s].labels), (f, s)
            assert [x["changedOutputPixels"] for x in ra[s].stats] == [x["changedOutputPixels"] for x in rb[s].stats]
            assert [x["changedOutputPixels"] for x in waited[tickets[f]][0][s]] == \
                [x["changedOutputPixels"] for x in rb[s].stats]
            assert np.array_equal(a.layer_input(0, s).view(np.uint32), dec[f][s].view(np.uint32))
            assert np.array_equal(a.final_activation(s).view(np.uint32), b.final_activation(s).view(np.uint32))
            assert np.array_equal(a.trace(0, s)[1], b.trace(0, s)[1])
    _ = rng
