"""Probe: per-kernel device times of the paper net at 1080p (S streams), for
each CBX_OPT_TC_PAIR mode, dense (Baseline engine) and steady change-based
frames. Graph-free pass with CUDA events around every kernel.

  python scripts/tc_probe.py [--modes 0,1] [--streams 4] [--frames 3]
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
ap.add_argument("--modes", default="0,1")
ap.add_argument("--streams", type=int, default=4)
ap.add_argument("--recipe", default="2.2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--only", default="", help="engine filter: cbinfer or baseline")
ap.add_argument("--precision", default="f16", choices=["f16", "tf32"])
ap.add_argument("--stages", default="", help="comma list of CBX_TC_STAGES values to sweep")
ap.add_argument("--nofuse", action="store_true", help="run the per-pixel head unfused (no tail in the L3 epilogue)")
ap.add_argument("--nsplit", default="", help="comma list of CBX_TC_NSPLIT values (1 even split, 0 256+rest)")
args = ap.parse_args()

S, F, H, W = args.streams, 6, 1080, 1920
specd = bench.paper_spec_dict(H, W)
spec = cbx.network_spec_from_json(json.dumps(specd))
wts = cbx.generate_weights(spec, None, 1)
net = cbx.Network(spec, wts, streams=S, precision=args.precision, fuse_tail=not args.nofuse, lanes=1)
clip = torch.empty((F, S, 3, H, W), dtype=torch.float32, device="cuda")
ns = argparse.Namespace(recipe=args.recipe, height=H, width=W)
for s in range(S):
    cfg = bench.clip_cfg(ns, s + 1)
    for f in range(F):
        cbx.synth_frame_device(cfg, f, clip[f, s].data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
ptrs = lambda i: [clip[bench.pingpong(i, F), s].data_ptr() for s in range(S)]

combos = [(int(m), st, sp) for m in args.modes.split(",") for st in (args.stages.split(",") if args.stages else [""])
          for sp in (args.nsplit.split(",") if args.nsplit else [""])]
for mode, st, sp in combos:
    if st:
        os.environ["CBX_TC_STAGES"] = st
    if sp:
        os.environ["CBX_TC_NSPLIT"] = sp
    net.set_tc_pair(mode)
    for engine in ("baseline", "cbinfer"):
        if args.only and engine != args.only:
            continue
        net.reset_state()
        for i in range(4):
            net.forward_device(ptrs(i), engine)
        net.sync()
        acc = {}
        for r in range(args.reps):
            for kt in net.profile(ptrs(4 + r), engine):
                acc.setdefault(f"{kt['name']}[{kt['layer']}]", []).append(kt["ms"])
        tot = sum(sum(v) / len(v) for v in acc.values())
        print(f"pair={mode} stages={st or 'auto'} nsplit={sp or 'auto'} {engine}: total {tot * 1000:.1f} us  " +
              "  ".join(f"{k}={1000 * sum(v) / len(v):.1f}" for k, v in acc.items()), flush=True)
