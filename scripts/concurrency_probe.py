"""Probe: do two independent Networks on two CUDA streams (N streams each)
overlap on the GPU? Compares one Network with 2N camera streams against two
Networks with N each, both driven back to back with device-resident clips."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import argparse  # noqa: E402

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1704_04313_b200 as cbx  # noqa: E402

N, F, K = int(sys.argv[1]) if len(sys.argv) > 1 else 4, 8, 30
H, W = 1080, 1920
specd = bench.paper_spec_dict(H, W)
spec = cbx.network_spec_from_json(json.dumps(specd))
wts = cbx.generate_weights(spec, None, 1)
ns = argparse.Namespace(recipe="2.2", height=H, width=W)
clip = torch.empty((F, 2 * N, 3, H, W), dtype=torch.float32, device="cuda")
for s in range(2 * N):
    cfg = bench.clip_cfg(ns, s + 1)
    for f in range(F):
        cbx.synth_frame_device(cfg, f, clip[f, s].data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()


def timed(nets, splits):
    for n in nets:
        n.reset_state()
    for i in range(4):
        for n, (a, b) in zip(nets, splits):
            n.forward_device([clip[bench.pingpong(i, F), s].data_ptr() for s in range(a, b)])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for n in nets:
        torch.cuda.current_stream().wait_stream(torch.cuda.ExternalStream(n.stream_handle()))
    for i in range(4, 4 + K):
        for n, (a, b) in zip(nets, splits):
            n.forward_device([clip[bench.pingpong(i, F), s].data_ptr() for s in range(a, b)])
    for n in nets:
        torch.cuda.current_stream().wait_stream(torch.cuda.ExternalStream(n.stream_handle()))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return 2 * N * K / (ms / 1000.0), ms / K


one = cbx.Network(spec, wts, streams=2 * N)
fps1, ms1 = timed([one], [(0, 2 * N)])
one.close()
for lanes in (2, 4, 8):
    if (2 * N) % lanes:
        continue
    per = 2 * N // lanes
    nets = [cbx.Network(spec, wts, streams=per) for _ in range(lanes)]
    fps2, ms2 = timed(nets, [(l * per, (l + 1) * per) for l in range(lanes)])
    print(f"one net x{2 * N} streams: {fps1:.0f} fps ({ms1:.3f} ms/step); {lanes} nets x{per} on {lanes} CUDA streams: "
          f"{fps2:.0f} fps ({ms2:.3f} ms/step)")
    for n in nets:
        n.close()
