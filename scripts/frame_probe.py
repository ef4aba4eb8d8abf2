"""Probe: the bench workload (paper net, 1080p, S streams in one lane) for a
few steady frames, 8-bit native or fp32 frames -- a target for ncu
(--set full -k regex:...) and a per-kernel event profile.

  python scripts/frame_probe.py [--streams 8] [--input u8|f32] [--frames 6] [--profile]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1704_04313_b200 as cbx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--streams", type=int, default=8)
ap.add_argument("--lanes", type=int, default=1)
ap.add_argument("--recipe", default="2.2")
ap.add_argument("--input", default="u8", choices=["u8", "f32"])
ap.add_argument("--precision", default="f16")
ap.add_argument("--frames", type=int, default=6)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--engine", default="cbinfer", choices=["cbinfer", "baseline"])
args = ap.parse_args()

S, F, H, W = args.streams, 6, 1080, 1920
specd = bench.paper_spec_dict(H, W)
spec = cbx.network_spec_from_json(json.dumps(specd))
wts = cbx.generate_weights(spec, None, 1)
net = cbx.Network(spec, wts, streams=S, precision=args.precision, lanes=args.lanes)
clip = torch.empty((F, S, 3, H, W), dtype=torch.float32, device="cuda")
ns = argparse.Namespace(recipe=args.recipe, height=H, width=W)
for s in range(S):
    cfg = bench.clip_cfg(ns, s + 1)
    for f in range(F):
        cbx.synth_frame_device(cfg, f, clip[f, s].data_ptr(), torch.cuda.current_stream().cuda_stream)
clip8 = (clip * 255.0).round().clamp(0, 255).to(torch.uint8).permute(0, 1, 3, 4, 2).contiguous()
cbx.decode_u8_device(clip8.data_ptr(), F * S, 3, H, W, clip.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
u8 = args.input == "u8"
ptrs = (lambda i: [clip8[bench.pingpong(i, F), s].data_ptr() for s in range(S)]) if u8 else \
    (lambda i: [clip[bench.pingpong(i, F), s].data_ptr() for s in range(S)])
fwd = net.forward_device_u8 if u8 else net.forward_device
for i in range(args.frames):
    fwd(ptrs(i))
net.sync()
if args.profile:
    for i in range(args.frames, args.frames + 3):
        prof = net.profile(ptrs(i), engine=args.engine, u8=u8)
        print(" ".join(f"{p['name']}[{p['layer']}]={p['ms'] * 1000:.1f}us" for p in prof))
    st, _ = net.read_stats()
    print("changed out L1/L2/L3:", [st[0][k]["changedOutputPixels"] for k in (0, 2, 4)])
