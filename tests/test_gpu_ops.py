"""GPU: op-level parity of the CUDA kernels with the oracle / golden vectors.
All calls go through the C-ABI (cbx_op_*) on device buffers."""
import numpy as np
import pytest

from oracle import make_geom

pytestmark = pytest.mark.gpu


def T(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def H(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


def test_detect_kats(gpu):
    prev = np.full((1, 4, 4), 0.5, np.float32)
    cur = prev.copy()
    cur[0, 2, 1] += np.float32(0.05)
    m, n = gpu.ops.detect_changes(T(cur), T(prev), 0.04)
    assert H(m).sum() == 1 and H(m)[2, 1] == 1 and int(n) == 1
    eq = prev.copy()
    eq[0, 2, 1] = np.float32(0.54)
    m, _ = gpu.ops.detect_changes(T(eq), T(prev), 0.04001)
    assert H(m).sum() == 0
    with pytest.raises(gpu.ShapeError):
        gpu.ops.detect_changes(T(np.zeros((1, 2, 2), np.float32)), T(np.zeros((1, 2, 3), np.float32)), 0.0)


def test_detect_golden_and_large(gpu, orc, golden):
    d = golden("ops.npz")
    for k in range(3):
        for t, tau in enumerate((0.0, 0.04, 0.09)):
            m, n = gpu.ops.detect_changes(T(d[f"det{k}_a"]), T(d[f"det{k}_b"]), tau)
            assert np.array_equal(H(m), d[f"det{k}_m{t}"])
            assert int(n) == int(d[f"det{k}_m{t}"].sum())
    rng = np.random.default_rng(7)
    a = rng.random((3, 1080, 1920), dtype=np.float32)
    b = a.copy()
    sel = rng.random((1080, 1920)) < 0.03
    b[1][sel] += np.float32(0.1)
    m, n = gpu.ops.detect_changes(T(a), T(b), 0.04)
    want = orc.detect_changes(a, b, 0.04)
    assert np.array_equal(H(m), want) and int(n) == int(want.sum())


def test_dilate_kats_and_golden(gpu, golden):
    m = np.zeros((20, 20), np.uint8)
    m[10, 10] = 1
    assert H(gpu.ops.dilate_changes(T(m), make_geom(7, 1, 3))).sum() == 49
    m = np.zeros((16, 16), np.uint8)
    m[0, 0] = 1
    assert H(gpu.ops.dilate_changes(T(m), make_geom(7, 1, 3))).sum() == 16
    m = np.zeros((30, 30), np.uint8)
    m[15, 15] = 1
    g = make_geom(7, 1, 3)
    assert H(gpu.ops.dilate_changes(gpu.ops.dilate_changes(T(m), g), g)).sum() == 169
    d = golden("ops.npz")
    for k in range(7):
        kk, s, p = d[f"dil{k}_g"].tolist()
        assert np.array_equal(H(gpu.ops.dilate_changes(T(d[f"dil{k}_in"]), make_geom(kk, s, p))), d[f"dil{k}_out"])


def test_dilate_random_large(gpu, orc):
    rng = np.random.default_rng(3)
    for (h, w, k, s, p) in [(1080, 1920, 7, 1, 3), (270, 480, 7, 1, 3), (301, 257, 5, 2, 2), (64, 1000, 3, 3, 0)]:
        m = (rng.random((h, w)) < 0.01).astype(np.uint8)
        g = make_geom(k, s, p)
        assert np.array_equal(H(gpu.ops.dilate_changes(T(m), g)), orc.dilate_changes(m, g))


def test_extract(gpu, orc, golden):
    d = golden("ops.npz")
    assert np.array_equal(H(gpu.ops.extract_indexes(T(d["ext_in"]))), d["ext_out"])
    two = np.zeros((4, 4), np.uint8)
    two[0, 1] = two[2, 3] = 1
    assert H(gpu.ops.extract_indexes(T(two))).tolist() == [1, 11]
    assert H(gpu.ops.extract_indexes(T(np.zeros((4, 4), np.uint8)))).size == 0
    assert H(gpu.ops.extract_indexes(T(np.ones((3, 5), np.uint8)))).tolist() == list(range(15))
    rng = np.random.default_rng(11)
    for n, dens in [(2_073_600, 0.02), (2_073_600, 0.9), (123_457, 0.3), (4096 * 37 + 5, 0.0005)]:
        m = (rng.random(n) < dens).astype(np.uint8)
        assert np.array_equal(H(gpu.ops.extract_indexes(T(m))), orc.extract_indexes(m))


def test_maxpool_argmax(gpu, orc, golden):
    t = np.arange(1, 17, dtype=np.float32).reshape(1, 4, 4)
    assert H(gpu.ops.maxpool(T(t), 2, 2))[0].tolist() == [[6, 8], [14, 16]]
    d = golden("ops.npz")
    assert np.array_equal(H(gpu.ops.maxpool(T(d["pool_in"]), 2, 2)).view(np.uint32), d["pool_2_2"].view(np.uint32))
    assert np.array_equal(H(gpu.ops.maxpool(T(d["pool_in"]), 3, 2)).view(np.uint32), d["pool_3_2"].view(np.uint32))
    with pytest.raises(gpu.GeometryError):
        gpu.ops.maxpool(T(t), 5, 1)
    z = np.zeros((3, 2, 2), np.float32)
    z[1, 0, 0] = z[2, 0, 0] = 1
    lab = H(gpu.ops.argmax_classify(T(z))).astype(np.uint16)
    assert lab[0, 0] == 1 and lab[1, 1] == 0
    x = np.random.default_rng(2).standard_normal((8, 33, 47)).astype(np.float32)
    assert np.array_equal(H(gpu.ops.argmax_classify(T(x))).astype(np.uint16), orc.argmax_classify(x))


def test_cbconv_update_exact(gpu, orc, golden):
    """gen_x_reduced + gemm + update_output, bitwise (cbconv.cpp:115-155)."""
    d = golden("ops.npz")
    rng = np.random.default_rng(9)
    for k in range(4):
        kk, s, p, ci, co = d[f"conv{k}_g"].tolist()
        g = make_geom(kk, s, p, ci, co)
        x, K, b = d[f"conv{k}_x"], d[f"conv{k}_K"], d[f"conv{k}_b"]
        y = d[f"conv{k}_y"]
        ho, wo = y.shape[1:]
        full = np.arange(ho * wo, dtype=np.int32)
        out = gpu.ops.cbconv_update(T(x), T(K), T(b), g, T(full), T(np.zeros_like(y)), False)
        assert np.array_equal(H(out).view(np.uint32), y.view(np.uint32))
        # reduced list over a random previous output, fused ReLU
        prev = rng.standard_normal(y.shape).astype(np.float32)
        idx = np.sort(rng.choice(ho * wo, size=max(1, ho * wo // 5), replace=False)).astype(np.int32)
        want = orc.update_output(prev, orc.gemm(K, b, orc.gen_x_reduced(x, idx, g)), idx, True)
        out = gpu.ops.cbconv_update(T(x), T(K), T(b), g, T(idx), T(prev), True)
        assert np.array_equal(H(out).view(np.uint32), want.view(np.uint32))
