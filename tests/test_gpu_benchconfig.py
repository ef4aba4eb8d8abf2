"""GPU: output parity of the benchmark configuration itself (bench.py's
default workload) against the UNMODIFIED reference compiled from its sources
(oracle/_ref, the bench's --impl reference arm):

* paper_like.json at 1920x1080, S = 2 streams in 2 lanes, precision "f16"
  (the bench default: layer 1 kind::i8 on the 8-bit frames, layer 2
  kind::tf32, layer 3 kind::f16), base thresholds (0.04, 0.05, 0.05), the
  bench's sprite recipe (12 sprites x 128 px, 12 px/frame) with per-stream
  seeds (shard.stream_seed) quantized to 8-bit camera frames exactly as the
  bench does (bench.quantize_u8); the GPU takes the bytes (cbx_forward_u8,
  native path), the reference read_ppm's decode of them (bench.decode_u8);
  weights generate_weights(seed 1) written by the reference itself;
* frame 0 (full evaluation) and two steady frames, every stream checked:
  - layer-1 detected mask and updated index list bit-exact,
  - layers 2-3: popcount(detected XOR) and |updated symdiff| <= 1 % of the
    reference's count (a tensor-core activation may cross tau),
  - final activation (input of CLASSIFY) max-abs <= 1e-3,
  - labels disagree on <= 0.1 % of the pixels.

Reference: forward_frame network.cpp:252-315, cbconv_forward cbconv.cpp:157-228.
"""
import os
import threading

import numpy as np
import pytest

from netutil import paper_spec, to_pkg_spec

pytestmark = pytest.mark.gpu

H, W, S, LANES = 1080, 1920, 2, 2
RECIPE = [(128, 12, 0.9)] * 12


def test_bench_configuration_vs_reference(gpu):
    import bench
    import oracle
    from paper_1704_04313_b200 import shard
    if not os.path.exists(oracle.REF_SO):
        pytest.skip("oracle/_ref (the reference built from its sources) is not built")
    ref = oracle.Ref()
    spec = paper_spec(H, W)
    rnets = [ref.load_network(spec, 1)]
    rnets.append(ref.load_network(spec, 1, weights_dir=rnets[0].weights_dir))
    net = gpu.Network(to_pkg_spec(gpu, spec), rnets[0].weights_dir, streams=S, precision="f16", lanes=LANES)
    assert net.num_lanes() == LANES
    assert [net.layer_operands(k) for k in (0, 2, 4)] == ["i8", "tf32", "f16"]
    cfgs = [dict(channels=3, height=H, width=W, sprites=RECIPE, noise=0.0, seed=shard.stream_seed(g))
            for g in range(S)]
    nproc = os.cpu_count() or 1
    report = []
    for f in range(3):
        cams = [bench.quantize_u8(ref.synth_frame(c, f)) for c in cfgs]
        frames = [bench.decode_u8(x) for x in cams]
        got = net.forward_u8(np.stack(cams))
        if f == 0:
            for s in range(S):  # the reference's full first frame, its ops split over all cores
                rnets[s].warm(frames[s], nproc)
            want = None
        else:
            want = [None] * S

            def run(s):
                want[s] = rnets[s].forward_frame(frames[s], labels_shape=tuple(net.label_hw))
            ts = [threading.Thread(target=run, args=(s,)) for s in range(S)]
            for t in ts:
                t.start()
            for t in ts:
                t.join()
        if want is None:  # warm(): the reference's full frame 0 keeps no trace
            continue
        for s in range(S):
            fa_gpu, fa_ref = net.final_activation(s), rnets[s].final_activation()
            err = float(np.abs(fa_gpu.astype(np.float64) - fa_ref).max())
            assert err <= 1e-3, (f, s, err)
            lab = got[s].labels
            dis = int(np.count_nonzero(lab != want[s]["labels"]))
            assert dis <= max(1, 1e-3 * lab.size), (f, s, dis)
            for cb in range(3):
                dg, ug = net.trace(cb, s)
                dr, ur = rnets[s].trace(cb)
                det_mis = int(np.count_nonzero(dg != dr))
                upd_mis = int(np.setxor1d(ug, ur).size)
                report.append((f, s, cb, det_mis, int(np.count_nonzero(dr)), upd_mis, int(ur.size)))
                if cb == 0:
                    assert det_mis == 0 and upd_mis == 0, (f, s, det_mis, upd_mis)
                    assert np.array_equal(ug, ur)
                else:
                    assert det_mis <= max(1, 0.01 * np.count_nonzero(dr)), (f, s, cb, det_mis)
                    assert upd_mis <= max(1, 0.01 * ur.size), (f, s, cb, upd_mis)
            for field in ("changedInputPixels", "changedOutputPixels", "gemmMacs"):
                assert got[s].stats[0][field] == want[s]["stats"][0][field], (f, s, field)
    # the clip reaches layer 3 on every stream
    assert all(r[6] > 0 for r in report if r[2] == 2)
    print("bench-config parity (frame, stream, cb, det_mis, det_ref, upd_mis, upd_ref):", report)


def test_synth_frame_device_matches_reference():
    """cbx_synth_frame_device (the bench's on-device clip source) equals the
    reference's synth_frame (synth.cpp:66-91) bitwise on noise-free clips:
    the bench recipe at 1080p and odd sizes / channel counts."""
    import oracle
    import torch
    import paper_1704_04313_b200 as cbx
    gen = oracle.Ref() if os.path.exists(oracle.REF_SO) else oracle.Oracle()
    cases = [dict(channels=3, height=H, width=W, sprites=RECIPE, noise=0.0, seed=1),
             dict(channels=3, height=H, width=W, sprites=[(192, 20, 0.9)] * 16, noise=0.0, seed=7),
             dict(channels=16, height=128, width=128, sprites=[(24, 7, 0.9)], noise=0.0, seed=2),
             dict(channels=5, height=37, width=61, sprites=[(9, 3, 0.7), (30, 1, 0.95)], noise=0.0, seed=12345)]
    for cfg in cases:
        buf = torch.empty((cfg["channels"], cfg["height"], cfg["width"]), dtype=torch.float32, device="cuda")
        for f in (0, 1, 5, 11):
            cbx.synth_frame_device(cfg, f, buf.data_ptr(), torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            want = gen.synth_frame(cfg, f)
            assert np.array_equal(buf.cpu().numpy().view(np.uint32), want.view(np.uint32)), (cfg["seed"], f)
