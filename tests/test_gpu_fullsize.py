"""GPU: size-independent properties at the benchmark's full size (1080p,
BASELINE configs[2]/[3]), where a full oracle run would be too slow:

* layer-1 change mask and updated index list of every steady frame are
  bit-exact against the oracle's detect_changes / dilate_changes /
  extract_indexes on the same frames (tf32 mode: layer 1 is exact fp32);
* at tau = 0 the change-based frame equals the dense (Baseline) frame
  bitwise -- labels and final activation -- on sparse sprite motion, in both
  precisions (test_network.cpp:176-199 at full size);
* the pipelined host API returns the same labels as the device-resident path.
"""
import json

import numpy as np
import pytest

from netutil import bits, paper_spec, to_pkg_spec

pytestmark = pytest.mark.gpu

H, W = 1080, 1920
CFG = dict(channels=3, height=H, width=W, sprites=[(128, 12, 0.9)] * 6, noise=0.0, seed=11)


def test_layer1_masks_and_indices_1080p(gpu, orc):
    from oracle import make_geom
    spec = paper_spec(H, W)
    w = orc.generate_weights(spec, 1)
    net = gpu.Network(to_pkg_spec(gpu, spec), w, precision="tf32", streams=1)
    g = make_geom(7, 1, 3)
    prev = None
    for f in range(4):
        fr = orc.synth_frame(CFG, f)
        net.forward_frame(fr)
        det, upd = net.trace(0)
        if prev is None:
            assert det is None
        else:
            want_det = orc.detect_changes(fr, prev, spec["layers"][0]["threshold"])
            assert np.array_equal(det, want_det), f
            want_idx = orc.extract_indexes(orc.dilate_changes(want_det, g))
            assert np.array_equal(upd, want_idx), f
            assert 0 < upd.size < H * W // 10
        prev = fr


@pytest.mark.parametrize("precision", ["tf32", "exact"])
def test_tau0_cb_equals_dense_1080p(gpu, orc, precision):
    spec = paper_spec(H, W, (0.0, 0.0, 0.0))
    w = orc.generate_weights(spec, 1)
    net = gpu.Network(to_pkg_spec(gpu, spec), w, precision=precision, streams=1)
    for f in range(3 if precision == "tf32" else 2):
        fr = orc.synth_frame(CFG, f)
        a = net.forward_frame(fr, "cbinfer")
        fa = net.final_activation(engine="cbinfer")
        b = net.forward_frame(fr, "baseline")
        fb = net.final_activation(engine="baseline")
        assert np.array_equal(a.labels, b.labels), (precision, f)
        assert np.array_equal(bits(fa), bits(fb)), (precision, f)


def test_submit_matches_device_path_1080p(gpu, orc):
    import torch
    spec = paper_spec(H, W)
    w = orc.generate_weights(spec, 1)
    S = 2
    a = gpu.Network(to_pkg_spec(gpu, spec), w, precision="tf32", streams=S)
    b = gpu.Network(to_pkg_spec(gpu, spec), w, precision="tf32", streams=S)
    frames = [np.ascontiguousarray(np.stack([orc.synth_frame(dict(CFG, seed=20 + s), f) for s in range(S)]))
              for f in range(4)]
    labels = [np.zeros((S,) + tuple(a.label_hw), np.uint16) for _ in frames]
    t = [a.submit(fr, lab) for fr, lab in zip(frames, labels)][-3:]
    for x in t:
        a.wait(x, with_stats=False)
    dev = torch.from_numpy(np.stack(frames)).cuda()
    for f in range(len(frames)):
        b.forward_device([dev[f, s].data_ptr() for s in range(S)])
        assert np.array_equal(b.read_labels(), labels[f]), f
