"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs the reference library compiled from /root/reference sources
(oracle/_ref/libcbinfer_ref.so, built by `make -C oracle ref`) -- never the
restatement -- and stores its outputs as small .npz fixtures. Re-run here
(where /root/reference exists) with:

    python tests/golden/make_golden.py

Fixtures:
  ops.npz        detect/dilate/extract/maxpool/conv_full/synth/random_filters cases
  c1.npz         BASELINE config 1: CBCONV 3x3 16->32 @128x128, 8 frames, ~2% change
  paper48.npz    paper_like.json @48x64, 5 noisy frames, tau (0.04,0.05,0.05)
  tiny_tau0.npz  a 16x16 3-CBCONV net at tau=0 (CB == Baseline contract)
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import Ref, make_geom, spec_from_json  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ops(ref):
    rng = np.random.default_rng(1234)
    d = {}
    # detect: random frames, several taus
    for k, (c, h, w) in enumerate([(3, 17, 23), (16, 32, 32), (2, 5, 5)]):
        a = rng.random((c, h, w), dtype=np.float32)
        b = a + (rng.random((c, h, w), dtype=np.float32) - 0.5) * 0.2
        for t, tau in enumerate((0.0, 0.04, 0.09)):
            d[f"det{k}_a"], d[f"det{k}_b"] = a, b
            d[f"det{k}_m{t}"] = ref.detect_changes(a, b, tau)
    # dilate: random maps, strided geometries
    geoms = [(7, 1, 3), (3, 1, 1), (3, 2, 1), (4, 3, 2), (2, 2, 0), (1, 1, 0), (5, 2, 4)]
    for k, (kk, s, p) in enumerate(geoms):
        m = (rng.random((29, 37)) < 0.05).astype(np.uint8)
        g = make_geom(kk, s, p)
        d[f"dil{k}_in"] = m
        d[f"dil{k}_g"] = np.array([kk, s, p], np.int32)
        d[f"dil{k}_out"] = ref.dilate_changes(m, g)
    # extract across 256-pixel blocks
    m = (rng.random((40, 40)) < 0.3).astype(np.uint8)
    d["ext_in"], d["ext_out"] = m, ref.extract_indexes(m)
    # maxpool
    t = rng.standard_normal((5, 13, 17)).astype(np.float32)
    d["pool_in"] = t
    d["pool_2_2"] = ref.maxpool(t, 2, 2)
    d["pool_3_2"] = ref.maxpool(t, 3, 2)
    # conv_full
    for k, (kk, s, p, ci, co, h, w) in enumerate([(3, 1, 1, 2, 3, 9, 11), (7, 1, 3, 3, 4, 16, 20),
                                                  (3, 2, 0, 4, 5, 12, 12), (1, 1, 0, 8, 8, 6, 7)]):
        x = rng.standard_normal((ci, h, w)).astype(np.float32)
        K = rng.standard_normal((co, ci * kk * kk)).astype(np.float32) * 0.3
        b = rng.standard_normal(co).astype(np.float32) * 0.1
        d[f"conv{k}_x"], d[f"conv{k}_K"], d[f"conv{k}_b"] = x, K, b
        d[f"conv{k}_g"] = np.array([kk, s, p, ci, co], np.int32)
        d[f"conv{k}_y"] = ref.conv_full(x, K, b, make_geom(kk, s, p, ci, co))
    # synth + random_filters
    cfg = dict(channels=3, height=48, width=64, sprites=[(10, 2, 0.9), (6, 3, 0.7)], noise=0.01, seed=3)
    d["synth_cfg"] = np.array([json.dumps(cfg)])
    for f in range(3):
        d[f"synth_f{f}"] = ref.synth_frame(cfg, f)
    K, b = ref.random_filters(make_geom(7, 1, 3, 52, 304), 4)
    d["rf_sha"] = np.array([sha(K), sha(b)])
    d["rf_head"] = K[:2, :16]
    np.savez_compressed(os.path.join(OUT, "ops.npz"), **d)


def run_net(ref, spec, seed, frames, name, taus=None, synth=None):
    """Drive the reference Network through forward_frame and keep its outputs.
    Large tensors are stored as sha256 digests (the restatement must reproduce
    them bit for bit); small ones in full."""
    ncb = sum(l["kind"] == "CBCONV" for l in spec["layers"])
    d = {"spec": np.array([json.dumps(spec)]), "seed": np.array([seed])}
    if synth is not None:
        d["synth"] = np.array([json.dumps(synth)])
    net = ref.load_network(spec, seed)
    if taus is not None:
        net.set_thresholds(taus)
    net.forward_frame(frames[0])
    lab_shape = net.final_activation().shape[1:]
    net = ref.load_network(spec, seed)
    if taus is not None:
        net.set_thresholds(taus)
    small = lambda a: a.nbytes <= 64 * 1024
    for f, fr in enumerate(frames):
        r = net.forward_frame(fr, labels_shape=lab_shape)
        if small(fr):
            d[f"f{f}_frame"] = fr
        d[f"f{f}_frame_sha"] = np.array([sha(fr)])
        d[f"f{f}_labels"] = r["labels"]
        d[f"f{f}_stats"] = np.array([[s["changedInputPixels"], s["changedOutputPixels"], s["gemmMacs"]]
                                     for s in r["stats"]], np.int64)
        d[f"f{f}_macs"] = np.array([r["macsTotal"]], np.uint64)
        fa = net.final_activation()
        d[f"f{f}_final_sha"] = np.array([sha(fa)])
        if small(fa):
            d[f"f{f}_final"] = fa
        for cb in range(ncb):
            det, upd = net.trace(cb)
            d[f"f{f}_cb{cb}_upd"] = upd
            if det is not None:
                d[f"f{f}_cb{cb}_det"] = np.packbits(det.reshape(-1))
                d[f"f{f}_cb{cb}_detshape"] = np.array(det.shape, np.int32)
    np.savez_compressed(os.path.join(OUT, name), **d)


def main():
    ref = Ref()
    ops(ref)
    # C1: single CBCONV 3x3 16->32 on 128x128 (BASELINE.json configs[0])
    c1 = dict(inputChannels=16, inputHeight=128, inputWidth=128, numClasses=32,
              layers=[dict(kind="CBCONV", kernelH=3, kernelW=3, strideH=1, strideW=1, padH=1, padW=1,
                           outChannels=32, threshold=0.05, fuseRelu=True, weightsFile="l1.w")])
    cfg = dict(channels=16, height=128, width=128, sprites=[(24, 7, 0.9)], noise=0.0, seed=2)
    run_net(ref, c1, 1, [ref.synth_frame(cfg, f) for f in range(8)], "c1.npz", synth=cfg)
    # paper_like at 48x64 with noise
    spec = spec_from_json(open("/root/reference/proj/netspecs/paper_like.json").read())
    spec["inputHeight"], spec["inputWidth"] = 48, 64
    for l, t in zip([l for l in spec["layers"] if l["kind"] == "CBCONV"], (0.04, 0.05, 0.05)):
        l["threshold"] = t
    cfg = dict(channels=3, height=48, width=64, sprites=[(10, 2, 0.9)], noise=0.01, seed=3)
    run_net(ref, spec, 1, [ref.synth_frame(cfg, f) for f in range(5)], "paper48.npz", synth=cfg)
    # tiny tau=0 net (test_network.cpp:176-199 structure)
    tiny = dict(inputChannels=2, inputHeight=16, inputWidth=16, numClasses=3, layers=[
        dict(kind="CBCONV", kernelH=7, kernelW=7, padH=3, padW=3, outChannels=4, threshold=0.0, fuseRelu=True, weightsFile="a"),
        dict(kind="MAXPOOL", window=2, stride=2),
        dict(kind="CBCONV", kernelH=7, kernelW=7, padH=3, padW=3, outChannels=6, threshold=0.0, fuseRelu=True, weightsFile="b"),
        dict(kind="MAXPOOL", window=2, stride=2),
        dict(kind="CBCONV", kernelH=7, kernelW=7, padH=3, padW=3, outChannels=8, threshold=0.0, fuseRelu=True, weightsFile="c"),
        dict(kind="CONV", kernelH=1, kernelW=1, outChannels=4, weightsFile="d"),
        dict(kind="RELU"),
        dict(kind="CONV", kernelH=1, kernelW=1, outChannels=3, weightsFile="e"),
        dict(kind="CLASSIFY")])
    cfg = dict(channels=2, height=16, width=16, sprites=[(5, 1, 0.9)], noise=0.03, seed=7)
    run_net(ref, tiny, 42, [ref.synth_frame(cfg, f) for f in range(5)], "tiny_tau0.npz", synth=cfg)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
