"""GPU: the tcgen05 gathered convolution against the exact oracle, one layer
at a time, with error bounds derived from the operand formats:

* kind::tf32: 10 mantissa bits, so |y_tc - y_exact| <= 2^-9 * sum_r |w_r x_r|
  (+ fp32 accumulation slack);
* kind::f16 (precision "f16": layers with > 128 outputs fed by a MAXPOOL):
  fp16 keeps the same 10 mantissa bits but a 5-bit exponent; operands below
  6.1e-5 are subnormal with an absolute rounding error <= 2^-25, so
  |y_tc - y_exact| <= 2^-9 * sum_r |w_r x_r| + 2^-24 * sum_r (|w_r| + |x_r|).

Shapes cover N split (304 = 128 + 176 with the split accumulator), N padding
(52 -> 64, 40 -> 48, 37 -> 48), channel padding (Cin % 4 != 0, and % 8 != 0
for fp16), stride, asymmetric kernels and K-blocks straddling taps; the fp16
cases also run on small-magnitude (subnormal) activations."""
import numpy as np
import pytest

from netutil import to_pkg_spec

pytestmark = pytest.mark.gpu


def two_layer(cin, h, w, layer):
    # layer 0: exact 1x1 CONV from the planar frame to a channels-last tensor of
    # `cin` channels; layer 1: the tcgen05 layer under test (tau=0, full frames).
    return dict(inputChannels=3, inputHeight=h, inputWidth=w, numClasses=layer["outChannels"], layers=[
        dict(kind="CONV", kernelH=1, kernelW=1, outChannels=cin, weightsFile="a"), layer])


def pooled_layer(cin, h, w, layer):
    # as two_layer, with a 2x2/2 MAXPOOL in front of the tested layer: the
    # pooling kernel writes the fp16 shadow a kind::f16 layer gathers from
    return dict(inputChannels=3, inputHeight=h, inputWidth=w, numClasses=layer["outChannels"], layers=[
        dict(kind="CONV", kernelH=1, kernelW=1, outChannels=cin, weightsFile="a"),
        dict(kind="MAXPOOL", window=2, stride=2), layer])


CASES = [
    (52, 30, 40, dict(kind="CBCONV", kernelH=7, kernelW=7, padH=3, padW=3, outChannels=304, threshold=0.0, fuseRelu=True, weightsFile="b")),
    (4, 60, 80, dict(kind="CBCONV", kernelH=7, kernelW=7, padH=3, padW=3, outChannels=52, threshold=0.0, fuseRelu=True, weightsFile="b")),
    (304, 20, 24, dict(kind="CONV", kernelH=1, kernelW=1, outChannels=40, weightsFile="b")),
    (6, 33, 47, dict(kind="CBCONV", kernelH=5, kernelW=3, strideH=2, strideW=1, padH=2, padW=1, outChannels=37, threshold=0.0, fuseRelu=False, weightsFile="b")),
    (13, 17, 19, dict(kind="CBCONV", kernelH=3, kernelW=3, padH=1, padW=1, outChannels=300, threshold=0.0, fuseRelu=True, weightsFile="b")),
]

# kind::f16 candidates (> 128 outputs); the input is the pooled tensor
F16_CASES = [
    (52, 60, 80, dict(kind="CBCONV", kernelH=7, kernelW=7, padH=3, padW=3, outChannels=304, threshold=0.0, fuseRelu=True, weightsFile="b")),
    (13, 34, 38, dict(kind="CBCONV", kernelH=3, kernelW=3, padH=1, padW=1, outChannels=300, threshold=0.0, fuseRelu=True, weightsFile="b")),
    (20, 40, 50, dict(kind="CBCONV", kernelH=5, kernelW=3, strideH=2, strideW=1, padH=2, padW=1, outChannels=160, threshold=0.0, fuseRelu=False, weightsFile="b")),
    (6, 26, 30, dict(kind="CONV", kernelH=1, kernelW=1, outChannels=136, weightsFile="b")),
    # packed fp16 gather (channels a multiple of 4, even padded row): 3 x 12
    # halves = 72 B per kernel row, the 5th chunk runs 8 B into the next
    # pixel, windows start on both 8-byte parities (24-byte pixels); 5 x 20
    # halves = 200 B (13 chunks) with stride 2; and 10 channels (20-byte
    # pixels: not 8-byte aligned, so the padded layout is kept)
    (12, 36, 44, dict(kind="CBCONV", kernelH=3, kernelW=3, padH=1, padW=1, outChannels=144, threshold=0.0, fuseRelu=True, weightsFile="b")),
    (20, 44, 52, dict(kind="CBCONV", kernelH=5, kernelW=5, strideH=2, strideW=2, padH=2, padW=2, outChannels=160, threshold=0.0, fuseRelu=False, weightsFile="b")),
    (10, 36, 44, dict(kind="CBCONV", kernelH=3, kernelW=3, padH=1, padW=1, outChannels=144, threshold=0.0, fuseRelu=True, weightsFile="b")),
]


def _geom(l, cin):
    return dict(kernelH=l["kernelH"], kernelW=l["kernelW"], strideH=l.get("strideH", 1),
                strideW=l.get("strideW", 1), padH=l.get("padH", 0), padW=l.get("padW", 0),
                inChannels=cin, outChannels=l["outChannels"])


def _check_layer(gpu, orc, net, onet, spec, wts, cfg, tested, cin, f16, frames=3, scale_in=None):
    """Runs `frames` frames; the tested layer's input must match the oracle
    bitwise (exact layers before it), its output within the operand bound."""
    l = spec["layers"][tested]
    g = _geom(l, cin)
    K, b = wts[tested]
    for f in range(frames):
        fr = orc.synth_frame(cfg, f)
        onet.forward_frame(fr)
        net.forward_frame(fr)
        x = onet.layer_output(tested - 1)
        assert np.array_equal(net.layer_output(tested - 1).view(np.uint32), x.view(np.uint32))
        want = onet.layer_output(tested)
        got = net.layer_output(tested)
        ho, wo = want.shape[1:]
        X = orc.gen_x_reduced(np.abs(x), np.arange(ho * wo, dtype=np.int32), g)
        scale = orc.gemm(np.abs(K), np.abs(b), X).reshape(want.shape).astype(np.float64)
        bound = 2.0 ** -9 * scale + 1e-6
        if f16:
            ones = np.ones_like(X)
            sum_w = orc.gemm(np.abs(K), np.zeros_like(b), ones).reshape(want.shape).astype(np.float64)
            sum_x = X.astype(np.float64).sum(axis=1).reshape(want.shape[1:])[None]
            bound = bound + 2.0 ** -24 * (sum_w + sum_x)
        err = np.abs(got.astype(np.float64) - want)
        assert np.all(err <= bound), (float((err / bound).max()), float(err.max()))


@pytest.mark.parametrize("pair", [-1, 0, 1])
@pytest.mark.parametrize("cin,h,w,layer", CASES)
def test_tc_layer_vs_exact(gpu, orc, cin, h, w, layer, pair):
    """pair: CBX_OPT_TC_PAIR (-1 auto = single CTA, 0 single CTA, 1 CTA pairs)."""
    check_tc_layer(gpu, orc, cin, h, w, layer, pair)


def test_all_cases_run_on_tcgen05(gpu, orc):
    """Every tf32 case above actually runs on the tensor cores (>= 32 outputs)."""
    for cin, h, w, layer in CASES:
        spec = two_layer(cin, h, w, layer)
        net = gpu.Network(to_pkg_spec(gpu, spec), orc.generate_weights(spec, 11), precision="tf32")
        assert net.layer_operands(1) == "tf32", layer


@pytest.mark.parametrize("pair", [0, 1])
@pytest.mark.parametrize("cin,h,w,layer", [c for c in CASES if c[3]["outChannels"] >= 52])
def test_tc_layer_many_tiles_per_cta(gpu, orc, monkeypatch, cin, h, w, layer, pair):
    """The persistent loop across tiles: the grid capped at 2 CTAs
    (CBX_TC_MAXCTAS, read at layer setup), so every CTA walks several tiles --
    stage-ring and accumulator-parity continuation, and for N > 256 the split
    accumulator's alternating tail columns and shared-column hand-off."""
    monkeypatch.setenv("CBX_TC_MAXCTAS", "2")
    check_tc_layer(gpu, orc, cin, h, w, layer, pair)


def check_tc_layer(gpu, orc, cin, h, w, layer, pair):
    spec = two_layer(cin, h, w, layer)
    wts = orc.generate_weights(spec, 11)
    onet = orc.load_network(spec, wts)
    net = gpu.Network(to_pkg_spec(gpu, spec), wts, precision="tf32")
    net.set_tc_pair(pair)
    cfg = dict(channels=3, height=h, width=w, sprites=[(5, 2, 0.9)], noise=0.02, seed=5)
    _check_layer(gpu, orc, net, onet, spec, wts, cfg, 1, cin, False)


@pytest.mark.parametrize("magnitude", ["unit", "subnormal"])
@pytest.mark.parametrize("maxctas,pair", [(None, -1), ("2", -1), (None, 1), ("4", 1)])
@pytest.mark.parametrize("cin,h,w,layer", F16_CASES)
def test_f16_layer_vs_exact(gpu, orc, monkeypatch, cin, h, w, layer, maxctas, pair, magnitude):
    """kind::f16 per-layer bound: a MAXPOOL-fed layer with > 128 outputs under
    precision "f16" (the headline operand format of the paper's layer 3),
    against the exact oracle on the same pooled input; 'subnormal' scales the
    first layer so the pooled activations are ~1e-5 (fp16 subnormal range);
    maxctas caps the persistent grid so every CTA walks several tiles; pair=1
    runs CTA pairs (cta_group::2, M = 256, each SM holding half the filters)."""
    if maxctas:
        monkeypatch.setenv("CBX_TC_MAXCTAS", maxctas)
    spec = pooled_layer(cin, h, w, layer)
    wts = orc.generate_weights(spec, 13)
    if magnitude == "subnormal":
        K0, b0 = wts[0]
        wts[0] = ((K0 * 4e-5).astype(np.float32), (b0 * 4e-5).astype(np.float32))
    onet = orc.load_network(spec, wts)
    net = gpu.Network(to_pkg_spec(gpu, spec), wts, precision="f16")
    net.set_tc_pair(pair)
    assert net.layer_operands(2) == "f16"
    cfg = dict(channels=3, height=h, width=w, sprites=[(5, 2, 0.9)], noise=0.02, seed=5)
    if magnitude == "subnormal":
        fr = orc.synth_frame(cfg, 0)
        onet.forward_frame(fr)
        x = onet.layer_output(1)
        assert 0 < np.abs(x).max() < 6.1e-5 * 4  # mostly below the fp16 normal range
        onet.reset_state()
    _check_layer(gpu, orc, net, onet, spec, wts, cfg, 2, cin, True)


@pytest.mark.parametrize("pack", ["0", "1"])
def test_f16_packed_and_padded_gather(gpu, orc, monkeypatch, pack):
    """The paper's layer 3 (52 -> 304, 7x7) with the packed fp16 gather
    (52 channels unpadded, 46 chunks per kernel row, odd-parity windows from
    the 8-byte-shifted shadow) and with CBX_TC_PACK=0 (channels padded to 56,
    49 chunks): both within the kind::f16 bound of the exact oracle."""
    monkeypatch.setenv("CBX_TC_PACK", pack)
    cin, h, w, layer = F16_CASES[0]
    spec = pooled_layer(cin, h, w, layer)
    wts = orc.generate_weights(spec, 17)
    onet = orc.load_network(spec, wts)
    net = gpu.Network(to_pkg_spec(gpu, spec), wts, precision="f16")
    assert net.layer_operands(2) == "f16"
    cfg = dict(channels=3, height=h, width=w, sprites=[(6, 3, 0.9)], noise=0.02, seed=9)
    _check_layer(gpu, orc, net, onet, spec, wts, cfg, 2, cin, True)


@pytest.mark.parametrize("maxctas,prec", [(None, "f16"), ("3", "f16"), (None, "tf32")])
def test_fused_tail_equals_unfused(gpu, orc, monkeypatch, maxctas, prec):
    """The per-pixel head (1x1 CONV, RELU, 1x1 CONV, CLASSIFY) run inside the
    last tcgen05 conv's epilogue gives bitwise the same labels, final
    activation and stats as running every layer separately (maxctas: grid
    capped so each CTA walks several tiles)."""
    from netutil import paper_spec, stats_arr
    if maxctas:
        monkeypatch.setenv("CBX_TC_MAXCTAS", maxctas)
    spec = paper_spec(72, 112)
    w = orc.generate_weights(spec, 1)
    fused = gpu.Network(to_pkg_spec(gpu, spec), w, precision=prec, fuse_tail=True)
    plain = gpu.Network(to_pkg_spec(gpu, spec), w, precision=prec, fuse_tail=False)
    cfg = dict(channels=3, height=72, width=112, sprites=[(14, 3, 0.9)], noise=0.01, seed=4)
    for f in range(4):
        fr = orc.synth_frame(cfg, f)
        a, b = fused.forward_frame(fr), plain.forward_frame(fr)
        assert np.array_equal(a.labels, b.labels)
        assert np.array_equal(stats_arr(a.stats), stats_arr(b.stats))
        assert np.array_equal(fused.final_activation().view(np.uint32), plain.final_activation().view(np.uint32))
    with pytest.raises(gpu.SpecError):
        fused.layer_output(5)  # the head's first 1x1 conv output is not materialized
    for engine in ("baseline",):
        a, b = fused.forward_frame(fr, engine), plain.forward_frame(fr, engine)
        assert np.array_equal(a.labels, b.labels)


# multi-pixel-row convs (conv_mpr.cu): precision "f16" with CBX_MPR_F16=1, a <= 4-channel input;
# groups of R adjacent output pixels per tensor-core row, fp16 operands
# converted while gathering. Widths not divisible by R, channel padding
# (3 -> 4 inputs, 37 -> 40 outputs), asymmetric kernels and a 1x1 kernel.
MPR_CASES = [
    (4, 60, 80, dict(kind="CBCONV", kernelH=7, kernelW=7, padH=3, padW=3, outChannels=52, threshold=0.0, fuseRelu=True, weightsFile="b")),
    (3, 33, 47, dict(kind="CBCONV", kernelH=3, kernelW=3, padH=1, padW=1, outChannels=37, threshold=0.0, fuseRelu=False, weightsFile="b")),
    (4, 29, 38, dict(kind="CBCONV", kernelH=5, kernelW=3, padH=2, padW=1, outChannels=64, threshold=0.0, fuseRelu=True, weightsFile="b")),
    (2, 21, 30, dict(kind="CONV", kernelH=1, kernelW=1, outChannels=48, weightsFile="b")),
]


@pytest.mark.parametrize("R", ["1", "2", "4"])
@pytest.mark.parametrize("maxctas", [None, "2"])
@pytest.mark.parametrize("magnitude", ["unit", "subnormal"])
@pytest.mark.parametrize("cin,h,w,layer", MPR_CASES)
def test_mpr_f16_layer_vs_exact(gpu, orc, monkeypatch, cin, h, w, layer, magnitude, maxctas, R):
    """The multi-pixel-row conv against the exact oracle under the fp16
    operand bound, full frames and change-based frames (tau = 0) alike;
    R = CBX_MPR_R (pixels per tensor-core row, clamped to N <= 256), maxctas
    caps the persistent grid so every CTA walks several tiles."""
    monkeypatch.setenv("CBX_MPR_R", R)
    monkeypatch.setenv("CBX_MPR_F16", "1")  # (opt-in for fp32-input layers)
    if maxctas:
        monkeypatch.setenv("CBX_TC_MAXCTAS", maxctas)
    spec = two_layer(cin, h, w, layer)
    wts = orc.generate_weights(spec, 17)
    if magnitude == "subnormal":
        K0, b0 = wts[0]
        wts[0] = ((K0 * 4e-5).astype(np.float32), (b0 * 4e-5).astype(np.float32))
    onet = orc.load_network(spec, wts)
    net = gpu.Network(to_pkg_spec(gpu, spec), wts, precision="f16")
    assert net.layer_operands(1) == "f16"
    cfg = dict(channels=3, height=h, width=w, sprites=[(5, 2, 0.9)], noise=0.02, seed=5)
    _check_layer(gpu, orc, net, onet, spec, wts, cfg, 1, cin, True, frames=4)
    if layer["kind"] == "CBCONV":  # change-based frames ran: the update lists were group lists
        d, u = net.trace(0)
        _, ou = onet.trace(0)
        assert np.array_equal(u, ou)


GROUP_CASES = [c for c in MPR_CASES if c[3].get("strideH", 1) == 1]


@pytest.mark.parametrize("R", ["2", "4"])
@pytest.mark.parametrize("maxctas", [None, "2"])
@pytest.mark.parametrize("cin,h,w,layer", GROUP_CASES)
def test_tc_pixel_groups_vs_exact(gpu, orc, monkeypatch, cin, h, w, layer, maxctas, R):
    """conv_tc with pixel groups (CBX_TC_GROUP: R adjacent output pixels per
    tensor-core row, kind::tf32) within the tf32 bound of the exact result,
    full and change-based frames; the change-based update lists are group
    lists, their traces equal the oracle's."""
    monkeypatch.setenv("CBX_TC_GROUP", R)
    if maxctas:
        monkeypatch.setenv("CBX_TC_MAXCTAS", maxctas)
    spec = two_layer(cin, h, w, layer)
    wts = orc.generate_weights(spec, 19)
    onet = orc.load_network(spec, wts)
    net = gpu.Network(to_pkg_spec(gpu, spec), wts, precision="tf32")
    assert net.layer_operands(1) == "tf32"
    cfg = dict(channels=3, height=h, width=w, sprites=[(5, 2, 0.9)], noise=0.02, seed=6)
    _check_layer(gpu, orc, net, onet, spec, wts, cfg, 1, cin, False, frames=4)
    if layer["kind"] == "CBCONV":
        _, u = net.trace(0)
        _, ou = onet.trace(0)
        assert np.array_equal(u, ou)
