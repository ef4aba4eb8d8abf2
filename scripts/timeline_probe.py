"""Timeline of the two-lane bench step: kernel start/end times from CUPTI
(torch.profiler) for a few steady steps of 16 x 1080p streams in 2 lanes,
printed per lane (CUDA stream) with idle gaps, so the critical path of the
overlapped step can be read off. Tuning aid, not product.

  python scripts/timeline_probe.py [--streams 16] [--lanes 2] [--steps 3]
"""
import argparse
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_1704_04313_b200 as cbx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--streams", type=int, default=16)
ap.add_argument("--lanes", type=int, default=2)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "timeline.json"))
args = ap.parse_args()

S, F, H, W = args.streams, 6, 1080, 1920
specd = bench.paper_spec_dict(H, W)
spec = cbx.network_spec_from_json(json.dumps(specd))
net = cbx.Network(spec, cbx.generate_weights(spec, None, 1), streams=S, precision="f16", lanes=args.lanes)
clip = torch.empty((F, S, 3, H, W), dtype=torch.float32, device="cuda")
ns = argparse.Namespace(recipe="2.2", height=H, width=W)
for s in range(S):
    cfg = bench.clip_cfg(ns, s + 1)
    for f in range(F):
        cbx.synth_frame_device(cfg, f, clip[f, s].data_ptr(), torch.cuda.current_stream().cuda_stream)
clip8 = (clip * 255.0).round().clamp(0, 255).to(torch.uint8).permute(0, 1, 3, 4, 2).contiguous()
torch.cuda.synchronize()
ptrs = lambda i: [clip8[bench.pingpong(i, F), s].data_ptr() for s in range(S)]
for i in range(8):
    net.forward_device_u8(ptrs(i))
net.sync()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(8, 8 + args.steps):
        net.forward_device_u8(ptrs(i))
    net.sync()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
rows = []
for e in ev:
    rows.append((e.time_range.start, e.time_range.end, e.name, getattr(e, "device_resource_id", 0)))
rows.sort()
t0 = rows[0][0] if rows else 0
by_stream = defaultdict(list)
for s_, e_, n, sid in rows:
    by_stream[sid].append((s_ - t0, e_ - t0, n))
short = lambda n: n.split("(")[0].replace("void ", "").replace("cbx::", "").replace("(anonymous namespace)::", "")[:34]
for sid, lst in sorted(by_stream.items()):
    print(f"== stream {sid}: {len(lst)} kernels")
    prev = None
    for s_, e_, n in lst:
        gap = (s_ - prev) if prev is not None else 0.0
        print(f"  {s_:9.1f} {e_:9.1f} {e_ - s_:7.1f} us  gap {gap:6.1f}  {short(n)}")
        prev = e_
span = (rows[-1][1] - t0) if rows else 0
print(f"span {span:.1f} us for {args.steps} steps: {span / max(1, args.steps):.1f} us/step")
json.dump([dict(start=s_ - t0, end=e_ - t0, name=n, stream=sid) for s_, e_, n, sid in rows], open(args.out, "w"))
