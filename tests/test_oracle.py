"""CPU: pin the C restatement (oracle/) to the reference.

1. Known-answer tests restated from the reference's own suites
   (tests/test_cbconv.cpp, test_baseline.cpp, test_synth.cpp).
2. Golden fixtures produced by the UNMODIFIED reference (tests/golden/make_golden.py).
3. When oracle/_ref is built here: randomized bitwise comparison with it.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import REF_SO, OracleError, make_geom, spec_from_json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAPER = os.path.join(ROOT, "paper_1704_04313_b200", "netspecs", "paper_like.json")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# ---------------------------------------------------------------- KATs
def test_detect_identical_frames_empty(orc):  # test_cbconv.cpp:52-57
    a = np.random.default_rng(31).random((2, 5, 5), dtype=np.float32)
    assert orc.detect_changes(a, a, 0.0).sum() == 0
    assert orc.detect_changes(a, a, 0.5).sum() == 0


def test_detect_single_pixel_and_strict(orc):  # test_cbconv.cpp:59-71
    prev = np.full((1, 4, 4), 0.5, np.float32)
    cur = prev.copy()
    cur[0, 2, 1] += np.float32(0.05)
    m = orc.detect_changes(cur, prev, 0.04)
    assert m.sum() == 1 and m[2, 1] == 1
    eq = prev.copy()
    eq[0, 2, 1] = np.float32(0.54)
    assert orc.detect_changes(eq, prev, 0.04001).sum() == 0


def test_detect_or_oracle_and_monotone(orc):  # test_cbconv.cpp:73-105
    rng = np.random.default_rng(33)
    for _ in range(50):
        a = rng.random((2, 6, 6), dtype=np.float32)
        b = rng.random((2, 6, 6), dtype=np.float32)
        ta = float(rng.random() * 0.5)
        tb = ta + float(rng.random() * 0.5)
        ma, mb = orc.detect_changes(a, b, ta), orc.detect_changes(a, b, tb)
        d = a - b
        assert np.array_equal(ma, ((d > np.float32(ta)) | (-d > np.float32(ta))).any(0))
        assert not np.any(mb & ~ma)


@pytest.mark.parametrize("pos,count", [((10, 10), 49), ((0, 0), 16)])
def test_dilate_7x7(orc, pos, count):  # test_cbconv.cpp:107-133
    m = np.zeros((20, 20), np.uint8)
    m[pos] = 1
    d = orc.dilate_changes(m, make_geom(7, 1, 3))
    assert d.shape == (20, 20) and d.sum() == count


def test_two_dilations_169(orc):  # test_cbconv.cpp:118-124, acceptance c2
    m = np.zeros((30, 30), np.uint8)
    m[15, 15] = 1
    g = make_geom(7, 1, 3)
    assert orc.dilate_changes(orc.dilate_changes(m, g), g).sum() == 169


def test_dilate_bruteforce_strided(orc):  # test_cbconv.cpp:135-149
    rng = np.random.default_rng(37)
    for _ in range(30):
        k, s = int(rng.integers(1, 5)), int(rng.integers(1, 4))
        p = int(rng.integers(0, k + 1))
        h, w = k + int(rng.integers(0, 8)), k + int(rng.integers(0, 8))
        m = (rng.integers(0, 100, (h, w)) < 20).astype(np.uint8)
        got = orc.dilate_changes(m, make_geom(k, s, p))
        ho, wo = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        want = np.zeros((ho, wo), np.uint8)
        for y in range(ho):
            for x in range(wo):
                for kj in range(k):
                    for ki in range(k):
                        jj, ii = y * s + kj - p, x * s + ki - p
                        if 0 <= jj < h and 0 <= ii < w and m[jj, ii]:
                            want[y, x] = 1
        assert np.array_equal(got, want)


def test_worst_case_propagation(orc):  # test_cbconv.cpp:151-184
    g = make_geom(7, 1, 3)
    assert orc.worst_case_propagation([], g, 12, 12).sum() == 0
    assert orc.worst_case_propagation([10 * 20 + 10], g, 20, 20).sum() == 49
    with pytest.raises(OracleError):
        orc.worst_case_propagation([100], make_geom(3, 1, 1), 5, 5)


def test_extract_basic(orc):  # test_cbconv.cpp:187-204
    assert len(orc.extract_indexes(np.zeros((4, 4), np.uint8))) == 0
    two = np.zeros((4, 4), np.uint8)
    two[0, 1] = two[2, 3] = 1
    assert orc.extract_indexes(two).tolist() == [1, 11]
    assert orc.extract_indexes(np.ones((3, 5), np.uint8)).tolist() == list(range(15))


def test_gemm_kats(orc):  # test_baseline.cpp:90-125
    K = np.array([[1, 2], [3, 4]], np.float32)
    Y = orc.gemm(K, np.zeros(2, np.float32), np.array([[5, 6]], np.float32))
    assert Y[:, 0].tolist() == [17.0, 39.0]
    Y = orc.gemm(np.zeros((2, 3), np.float32), np.array([0.5, -1], np.float32), np.ones((4, 3), np.float32))
    assert np.all(Y[0] == 0.5) and np.all(Y[1] == -1)


def test_maxpool_kat(orc):  # test_baseline.cpp:221-231
    t = np.arange(1, 17, dtype=np.float32).reshape(1, 4, 4)
    assert orc.maxpool(t, 2, 2)[0].tolist() == [[6, 8], [14, 16]]


def test_argmax_ties_lowest(orc):  # test_baseline.cpp:274-286
    t = np.zeros((3, 2, 2), np.float32)
    t[1, 0, 0] = 1
    t[2, 0, 0] = 1
    lab = orc.argmax_classify(t)
    assert lab[0, 0] == 1 and lab[1, 1] == 0


def test_im2col_gemm_equals_conv_full(orc):  # test_baseline.cpp:153-185
    rng = np.random.default_rng(5)
    for _ in range(40):
        k, s = int(rng.integers(1, 6)), int(rng.integers(1, 3))
        p = int(rng.integers(0, k))
        ci, co = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        h, w = k + int(rng.integers(0, 9)), k + int(rng.integers(0, 9))
        g = make_geom(k, s, p, ci, co)
        x = rng.standard_normal((ci, h, w)).astype(np.float32)
        K = rng.standard_normal((co, ci * k * k)).astype(np.float32)
        b = rng.standard_normal(co).astype(np.float32)
        ho, wo = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        X = orc.gen_x_reduced(x, np.arange(ho * wo, dtype=np.int32), g)
        Y = orc.gemm(K, b, X).reshape(co, ho, wo)
        assert np.array_equal(bits(Y), bits(orc.conv_full(x, K, b, g)))


def test_synth_box_symmetric_difference(orc):  # test_synth.cpp:71-98
    cfg = dict(channels=3, height=64, width=80, sprites=[(12, 3, 0.9)], seed=11)
    for f in range(1, 6):
        a, b = orc.synth_frame(cfg, f - 1), orc.synth_frame(cfg, f)
        m = orc.detect_changes(b, a, 0.04)
        r0, r1 = orc.sprite_rect(cfg, 0, f - 1), orc.sprite_rect(cfg, 0, f)
        box = lambda r: {(j, i) for j in range(r[0], r[2]) for i in range(r[1], r[3])}
        assert m.sum() == len(box(r0) ^ box(r1))


# ---------------------------------------------------------------- golden fixtures
def test_golden_ops(orc, golden):
    d = golden("ops.npz")
    for k in range(3):
        for t, tau in enumerate((0.0, 0.04, 0.09)):
            assert np.array_equal(orc.detect_changes(d[f"det{k}_a"], d[f"det{k}_b"], tau), d[f"det{k}_m{t}"])
    for k in range(7):
        kk, s, p = d[f"dil{k}_g"].tolist()
        assert np.array_equal(orc.dilate_changes(d[f"dil{k}_in"], make_geom(kk, s, p)), d[f"dil{k}_out"])
    assert np.array_equal(orc.extract_indexes(d["ext_in"]), d["ext_out"])
    assert np.array_equal(bits(orc.maxpool(d["pool_in"], 2, 2)), bits(d["pool_2_2"]))
    assert np.array_equal(bits(orc.maxpool(d["pool_in"], 3, 2)), bits(d["pool_3_2"]))
    for k in range(4):
        kk, s, p, ci, co = d[f"conv{k}_g"].tolist()
        y = orc.conv_full(d[f"conv{k}_x"], d[f"conv{k}_K"], d[f"conv{k}_b"], make_geom(kk, s, p, ci, co))
        assert np.array_equal(bits(y), bits(d[f"conv{k}_y"]))
    cfg = json.loads(str(d["synth_cfg"][0]))
    for f in range(3):
        assert np.array_equal(bits(orc.synth_frame(cfg, f)), bits(d[f"synth_f{f}"]))
    K, b = orc.random_filters(make_geom(7, 1, 3, 52, 304), 4)
    assert [sha(K), sha(b)] == d["rf_sha"].tolist()


@pytest.mark.parametrize("name", ["c1.npz", "paper48.npz", "tiny_tau0.npz"])
def test_golden_network(orc, golden, name):
    d = golden(name)
    spec = json.loads(str(d["spec"][0]))
    cfg = json.loads(str(d["synth"][0]))
    net = orc.load_network(spec, orc.generate_weights(spec, int(d["seed"][0])))
    ncb = sum(l["kind"] == "CBCONV" for l in spec["layers"])
    f = 0
    while f"f{f}_labels" in d:
        fr = orc.synth_frame(cfg, f)
        assert sha(fr) == str(d[f"f{f}_frame_sha"][0])
        r = net.forward_frame(fr)
        assert np.array_equal(r["labels"], d[f"f{f}_labels"])
        st = np.array([[s["changedInputPixels"], s["changedOutputPixels"], s["gemmMacs"]] for s in r["stats"]])
        assert np.array_equal(st, d[f"f{f}_stats"])
        assert r["macsTotal"] == int(d[f"f{f}_macs"][0])
        assert sha(net.final_activation()) == str(d[f"f{f}_final_sha"][0])
        for cb in range(ncb):
            det, upd = net.trace(cb)
            assert np.array_equal(upd, d[f"f{f}_cb{cb}_upd"])
            if f"f{f}_cb{cb}_det" in d:
                assert np.array_equal(np.packbits(det.reshape(-1)), d[f"f{f}_cb{cb}_det"])
            else:
                assert det is None
        f += 1
    assert f >= 5


# ---------------------------------------------------------------- live reference
needs_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built (make -C oracle ref)")


@needs_ref
def test_restatement_matches_reference_random_nets(orc):
    """acceptance.cpp:71-120 style: random nets, oracle restatement == reference bitwise."""
    from oracle import Ref
    ref = Ref()
    rng = np.random.default_rng(20240001)
    for trial in range(12):
        inC, h, w = int(rng.integers(1, 5)), int(rng.integers(8, 17)), int(rng.integers(8, 17))
        layers, ch = [], inC
        for l in range(int(rng.integers(1, 4))):
            k = 7 if rng.integers(0, 2) else 3
            ch = int(rng.integers(1, 9))
            layers.append(dict(kind="CBCONV", kernelH=k, kernelW=k, padH=k // 2, padW=k // 2, outChannels=ch,
                               threshold=float(rng.choice([0.0, 0.02, 0.1])), fuseRelu=bool(rng.integers(0, 3)),
                               weightsFile=f"l{l}.w"))
            if l == 0:
                layers.append(dict(kind="MAXPOOL", window=2, stride=2))
        spec = dict(inputChannels=inC, inputHeight=h, inputWidth=w, numClasses=ch, layers=layers)
        seed = 1000 + trial
        on = orc.load_network(spec, orc.generate_weights(spec, seed))
        rn = ref.load_network(spec, seed)
        cfg = dict(channels=inC, height=h, width=w, sprites=[(3, 1, 0.9)], noise=0.02, seed=trial + 1)
        for f in range(4):
            fr = orc.synth_frame(cfg, f)
            a = on.forward_frame(fr)
            b = rn.forward_frame(fr, labels_shape=a["labels"].shape)
            assert np.array_equal(a["labels"], b["labels"])
            assert a["stats"] == b["stats"]
            assert np.array_equal(bits(on.final_activation()), bits(rn.final_activation()))
