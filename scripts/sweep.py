#!/usr/bin/env python
"""Change-rate / threshold sweeps of the change-based path on one B200
(BASELINE.json configs[1], [2], [4]).

  * rate:  frames/s vs the layer-1 input changed fraction, sprite recipes of
           SURVEY.md 8d, at 320x240 (configs[1]) and 1920x1080 (configs[2]),
           next to the dense per-frame comparator (Baseline engine, same
           kernels over every pixel) -> speed-up over dense.
  * tau:   threshold sweep (factor 0, 0.25 .. 2 of the base taus, cbench.cpp:393)
           at 320x240: frames/s and label disagreement against the dense
           engine on the same frames (calibration.cpp:56-58 pixel_disagreement).
  * worst: 100% change (noise on every pixel, tau = 0): change-based vs dense.

Timing: resident clips in HBM, CUDA events on the network's stream around K
steady frames (ping-pong playback), after warm-up; inputs per step exceed L2
at 1080p (4 streams x 2 frames x 24.9 MB), at 320x240 the S-stream clip
(S x 0.92 MB) does not, which the output records.

  python scripts/sweep.py [--which rate,tau,worst] [--out gpurun_out/sweep.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1704_04313_b200 as cbx  # noqa: E402

RECIPES_320 = [(2, 24, 3), (4, 24, 3), (4, 32, 4), (8, 32, 5), (10, 40, 6), (12, 40, 10), (32, 48, 16)]
RECIPES_1080 = [(8, 96, 8), (12, 128, 12), (16, 160, 16), (16, 192, 20), (20, 192, 20)]


def make_net(h, w, S, taus=bench.BASE_TAUS, precision="f16"):
    specd = bench.paper_spec_dict(h, w, taus)
    spec = cbx.network_spec_from_json(json.dumps(specd))
    return cbx.Network(spec, cbx.generate_weights(spec, None, 1), streams=S, precision=precision)


def sprite_clip(h, w, S, F, recipe):
    n, size, vel = recipe
    clip = torch.empty((F, S, 3, h, w), dtype=torch.float32, device="cuda")
    for s in range(S):
        cfg = dict(channels=3, height=h, width=w, sprites=[(size, vel, 0.9)] * n, noise=0.0, seed=s + 1)
        for f in range(F):
            cbx.synth_frame_device(cfg, f, clip[f, s].data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return clip


def timed_fps(net, clip, engine, K, warm=3):
    F, S = clip.shape[0], clip.shape[1]
    ptrs = lambda i: [clip[bench.pingpong(i, F), s].data_ptr() for s in range(S)]
    stream = torch.cuda.ExternalStream(net.stream_handle())
    net.reset_state()
    for i in range(warm + 1):
        net.forward_device(ptrs(i), engine)
    net.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(warm + 1, warm + 1 + K):
        net.forward_device(ptrs(i), engine)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return S * K / (ms / 1000.0), ms / K


def change_fractions(net, clip, frames=6):
    """Mean changed fractions over steady frames 1..frames-1 (from reset)."""
    F, S = clip.shape[0], clip.shape[1]
    cb = net.spec.cb_layers()
    net.reset_state()
    rows = []
    for i in range(frames):
        net.forward_device([clip[bench.pingpong(i, F), s].data_ptr() for s in range(S)])
        if i:
            rows.append(net.read_stats()[0])
    (c, h, w) = net.shapes[cb[0]][0]
    l1_in = float(np.mean([st[cb[0]]["changedInputPixels"] for r in rows for st in r])) / (h * w)
    outs = [float(np.mean([st[k]["changedOutputPixels"] for r in rows for st in r])) /
            (net.shapes[k][1][1] * net.shapes[k][1][2]) for k in cb]
    return l1_in, outs


def rate_sweep(h, w, S, recipes, K):
    net = make_net(h, w, S)
    clip = sprite_clip(h, w, S, 8, recipes[0])
    dense_fps, dense_ms = timed_fps(net, clip, "baseline", max(3, K // 4))
    rows = []
    for rc in recipes:
        clip = sprite_clip(h, w, S, 8, rc)
        fps, ms = timed_fps(net, clip, "cbinfer", K)
        l1, outs = change_fractions(net, clip)
        rows.append(dict(recipe=dict(sprites=rc[0], size=rc[1], velocity=rc[2]), l1_input_changed=l1,
                         layer_output_changed=outs, fps=fps, ms_per_step=ms, speedup_vs_dense=fps / dense_fps))
        print(f"  {w}x{h} S={S} recipe {rc}: L1 in {100 * l1:.2f}%  fps {fps:.0f}  x{fps / dense_fps:.2f} vs dense",
              flush=True)
        del clip
    return dict(height=h, width=w, streams=S, dense_fps=dense_fps, dense_ms_per_step=dense_ms, points=rows)


def tau_sweep(h, w, S, recipe, K, factors):
    out = []
    clip = sprite_clip(h, w, S, 8, recipe)
    F = clip.shape[0]
    ref_net = make_net(h, w, S)
    for fac in factors:
        taus = tuple(fac * t for t in bench.BASE_TAUS)
        net = make_net(h, w, S, taus)
        fps, ms = timed_fps(net, clip, "cbinfer", K)
        # accuracy: labels of every steady frame vs the dense engine on the same frame
        net.reset_state()
        dis, n = 0, 0
        for i in range(8):
            ptr = [clip[bench.pingpong(i, F), s].data_ptr() for s in range(S)]
            net.forward_device(ptr)
            lab = net.read_labels()
            ref_net.forward_device(ptr, "baseline")
            ref = ref_net.read_labels("baseline")
            if i:
                dis += int((lab != ref).sum())
                n += lab.size
        l1, outs = change_fractions(net, clip)
        out.append(dict(factor=fac, taus=list(taus), fps=fps, ms_per_step=ms, label_disagreement=dis / n,
                        l1_input_changed=l1, layer_output_changed=outs))
        print(f"  tau x{fac}: fps {fps:.0f}  label disagreement {100 * dis / n:.4f}%  L1 in {100 * l1:.2f}%",
              flush=True)
        net.close()
    return dict(height=h, width=w, streams=S, recipe=list(recipe), points=out)


def worst_case(h, w, S, K, noise=0.05):
    """tau = 0 and noise on every pixel: every input pixel changes every frame."""
    net = make_net(h, w, S, taus=(0.0, 0.0, 0.0))
    F = 4
    clip = torch.empty((F, S, 3, h, w), dtype=torch.float32, device="cuda")
    for s in range(S):
        cfg = dict(channels=3, height=h, width=w, sprites=[(24, 3, 0.9)], noise=noise, seed=s + 1)
        for f in range(F):
            clip[f, s].copy_(torch.from_numpy(cbx.synth_frame(cfg, f)))
    torch.cuda.synchronize()
    fps, ms = timed_fps(net, clip, "cbinfer", K)
    dfps, dms = timed_fps(net, clip, "baseline", K)
    l1, outs = change_fractions(net, clip, frames=4)
    print(f"  worst case {w}x{h}: L1 in {100 * l1:.1f}%  cb fps {fps:.0f}  dense fps {dfps:.0f}  ratio {fps / dfps:.2f}",
          flush=True)
    return dict(height=h, width=w, streams=S, noise=noise, l1_input_changed=l1, layer_output_changed=outs,
                cb_fps=fps, dense_fps=dfps, cb_over_dense=fps / dfps)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="rate,tau,worst")
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--s320", type=int, default=64, help="streams per GPU at 320x240")
    ap.add_argument("--s1080", type=int, default=8, help="streams per GPU at 1920x1080")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    args = ap.parse_args()
    res = dict(gpu=torch.cuda.get_device_name(0), when=time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
               precision="f16", base_taus=list(bench.BASE_TAUS))
    which = args.which.split(",")
    if "rate" in which:
        print("rate sweep 320x240", flush=True)
        res["rate_320x240"] = rate_sweep(240, 320, args.s320, RECIPES_320, args.steps)
        print("rate sweep 1920x1080", flush=True)
        res["rate_1920x1080"] = rate_sweep(1080, 1920, args.s1080, RECIPES_1080, args.steps)
    if "tau" in which:
        print("threshold sweep 320x240", flush=True)
        res["tau_320x240"] = tau_sweep(240, 320, args.s320, RECIPES_320[3], args.steps,
                                       [0.0, 0.25, 0.5, 0.75, 1.0, 1.25, 1.5, 1.75, 2.0])
    if "worst" in which:
        print("worst case", flush=True)
        res["worst_320x240"] = worst_case(240, 320, args.s320, args.steps)
        res["worst_1920x1080"] = worst_case(1080, 1920, args.s1080, max(5, args.steps // 4))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
