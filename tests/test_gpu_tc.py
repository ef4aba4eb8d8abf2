"""GPU: the tcgen05 (tf32) gathered convolution against the exact oracle,
with an error bound derived from the operands: tf32 keeps 10 mantissa bits,
so |y_tc - y_exact| <= 2^-9 * sum_r |w_r x_r| (+ fp32 accumulation slack).
Shapes cover N split (304 = 128 + 176 with the split accumulator),
N padding (52 -> 64, 8 -> 16),
channel padding (Cin % 4 != 0), stride, asymmetric kernels and K-blocks
straddling taps."""
import numpy as np
import pytest

from netutil import to_pkg_spec

pytestmark = pytest.mark.gpu


def two_layer(cin, h, w, layer):
    # layer 0: exact 1x1 CONV from the planar frame to a channels-last tensor of
    # `cin` channels; layer 1: the tcgen05 layer under test (tau=0, full frames).
    return dict(inputChannels=3, inputHeight=h, inputWidth=w, numClasses=layer["outChannels"], layers=[
        dict(kind="CONV", kernelH=1, kernelW=1, outChannels=cin, weightsFile="a"), layer])


CASES = [
    (52, 30, 40, dict(kind="CBCONV", kernelH=7, kernelW=7, padH=3, padW=3, outChannels=304, threshold=0.0, fuseRelu=True, weightsFile="b")),
    (4, 60, 80, dict(kind="CBCONV", kernelH=7, kernelW=7, padH=3, padW=3, outChannels=52, threshold=0.0, fuseRelu=True, weightsFile="b")),
    (304, 20, 24, dict(kind="CONV", kernelH=1, kernelW=1, outChannels=8, weightsFile="b")),
    (6, 33, 47, dict(kind="CBCONV", kernelH=5, kernelW=3, strideH=2, strideW=1, padH=2, padW=1, outChannels=37, threshold=0.0, fuseRelu=False, weightsFile="b")),
    (13, 17, 19, dict(kind="CBCONV", kernelH=3, kernelW=3, padH=1, padW=1, outChannels=300, threshold=0.0, fuseRelu=True, weightsFile="b")),
]


@pytest.mark.parametrize("pair", [-1, 0, 1])
@pytest.mark.parametrize("cin,h,w,layer", CASES)
def test_tc_layer_vs_exact(gpu, orc, cin, h, w, layer, pair):
    """pair: CBX_OPT_TC_PAIR (-1 auto = CTA pairs for N > 128, 0 single CTA, 1 pairs)."""
    check_tc_layer(gpu, orc, cin, h, w, layer, pair)


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
    for f in range(3):
        fr = orc.synth_frame(cfg, f)
        onet.forward_frame(fr)
        net.forward_frame(fr)
        x = onet.layer_output(0)
        assert np.array_equal(net.layer_output(0).view(np.uint32), x.view(np.uint32))
        want = onet.layer_output(1)
        got = net.layer_output(1)
        l = spec["layers"][1]
        g = dict(kernelH=l["kernelH"], kernelW=l["kernelW"], strideH=l.get("strideH", 1),
                 strideW=l.get("strideW", 1), padH=l.get("padH", 0), padW=l.get("padW", 0),
                 inChannels=cin, outChannels=l["outChannels"])
        K, b = wts[1]
        ho, wo = want.shape[1:]
        X = orc.gen_x_reduced(np.abs(x), np.arange(ho * wo, dtype=np.int32), g)
        scale = orc.gemm(np.abs(K), np.abs(b), X).reshape(want.shape)
        err = np.abs(got.astype(np.float64) - want)
        bound = 2.0 ** -9 * scale + 1e-6
        assert np.all(err <= bound), (float((err / bound).max()), float(err.max()))


@pytest.mark.parametrize("maxctas,f16", [(None, "1"), ("3", "1"), (None, "0")])
def test_fused_tail_equals_unfused(gpu, orc, monkeypatch, maxctas, f16):
    """The per-pixel head (1x1 CONV, RELU, 1x1 CONV, CLASSIFY) run inside the
    last tcgen05 conv's epilogue gives bitwise the same labels, final
    activation and stats as running every layer separately (maxctas: grid
    capped so each CTA walks several tiles)."""
    from netutil import paper_spec, stats_arr
    if maxctas:
        monkeypatch.setenv("CBX_TC_MAXCTAS", maxctas)
    monkeypatch.setenv("CBX_TC_F16", f16)
    spec = paper_spec(72, 112)
    w = orc.generate_weights(spec, 1)
    fused = gpu.Network(to_pkg_spec(gpu, spec), w, precision="tf32", fuse_tail=True)
    plain = gpu.Network(to_pkg_spec(gpu, spec), w, precision="tf32", fuse_tail=False)
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
