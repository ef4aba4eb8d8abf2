#!/usr/bin/env python
"""Parity report of the B200 path against the reference compiled from its own
sources (oracle/_ref; the C restatement when absent) on the same synthetic
clips -- the numbers north_star asks to report (SURVEY.md 8c parity plan):

  * layer-1 change masks and index lists: bit-exact (mismatch must be 0),
  * per-CBCONV-layer changed-pixel mismatch counts: popcount(detected_gpu XOR
    detected_ref) on the layer's input grid and |updated_gpu sym-diff
    updated_ref| on its output grid, next to the reference's own counts,
  * final activations (max-abs error) and segmentation maps (label
    disagreement) against the reference,

for precision=f16 (the bench's serving mode: layer 3 fp16 operands), tf32 and
exact (bitwise expected); each run records the per-layer operand formats,
at configs[1] (320x240) and configs[2] (1920x1080), base taus (0.04, 0.05,
0.05). Test/report infrastructure: runs the reference on the host as checker.

  python scripts/parity_report.py [--out profiles/r1_parity.json] [--frames 6]
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

import bench  # noqa: E402
import oracle  # noqa: E402
import paper_1704_04313_b200 as cbx  # noqa: E402


def ref_network(spec):
    if os.path.exists(oracle.REF_SO):
        r = oracle.Ref()
        return r.load_network(spec, 1), "reference (oracle/_ref, compiled from the reference sources)"
    orc = oracle.Oracle()
    return orc.load_network(spec, orc.generate_weights(spec, 1)), "oracle C restatement"


def run(h, w, recipe, frames, precision, nthreads):
    spec = bench.paper_spec_dict(h, w)
    ref, kind = ref_network(spec)
    wts = oracle.Oracle().generate_weights(spec, 1)
    net = cbx.Network(cbx.network_spec_from_json(json.dumps(spec)), wts, precision=precision)
    cfg = bench.clip_cfg(argparse.Namespace(recipe=recipe, height=h, width=w), 1)
    synth = oracle.Oracle().synth_frame
    ncb = len(net.spec.cb_layers())
    rows = []
    for f in range(frames):
        fr = synth(cfg, f)
        t0 = time.perf_counter()
        if f == 0 and hasattr(ref, "warm"):
            ref.warm(fr, nthreads)  # first frame is a full evaluation: reference ops over all cores
            want = None
        else:
            want = ref.forward_frame(fr, trace=True, labels_shape=tuple(net.label_hw)) \
                if hasattr(ref, "warm") else ref.forward_frame(fr)
        tref = time.perf_counter() - t0
        got = net.forward_frame(fr)
        if want is None:  # warm(): no labels/trace returned for frame 0
            continue
        layers = []
        for cb in range(ncb):
            dg, ug = net.trace(cb)
            dr, ur = ref.trace(cb)
            det_mis = None if (dg is None or dr is None) else int(np.count_nonzero(dg != dr))
            layers.append(dict(cb=cb + 1,
                               detected_ref=None if dr is None else int(np.count_nonzero(dr)),
                               detected_mismatch=det_mis,
                               updated_ref=int(ur.size), updated_gpu=int(ug.size),
                               updated_symdiff=int(np.setxor1d(ug, ur, assume_unique=True).size)))
        fa_g, fa_r = net.final_activation(), ref.final_activation()
        lab_r = want["labels"]
        rows.append(dict(frame=f, ref_seconds=round(tref, 2), layers=layers,
                         final_max_abs_err=float(np.abs(fa_g.astype(np.float64) - fa_r).max()),
                         label_disagreement=float((got.labels != lab_r).mean())))
        print(f"  {w}x{h} {precision} frame {f}: " +
              "  ".join(f"L{l['cb']} det {l['detected_mismatch']}/{l['detected_ref']} "
                        f"upd {l['updated_symdiff']}/{l['updated_ref']}" for l in layers) +
              f"  max|dy| {rows[-1]['final_max_abs_err']:.2e}  labels {100 * rows[-1]['label_disagreement']:.4f}%",
              flush=True)
    operands = {str(k): net.layer_operands(k) for k, l in enumerate(net.spec.layers) if l.is_conv()}
    net.close()
    return dict(height=h, width=w, recipe=recipe, precision=precision, operands=operands, checker=kind,
                frames=rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity.json"))
    ap.add_argument("--frames", type=int, default=6)
    ap.add_argument("--frames-1080", type=int, default=3)
    args = ap.parse_args()
    nthreads = os.cpu_count() or 1
    res = dict(when=time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), taus=list(bench.BASE_TAUS), runs=[])
    for precision in ("f16", "tf32", "exact"):
        res["runs"].append(run(240, 320, "2.2", args.frames, precision, nthreads))
    for precision in ("f16", "tf32"):
        res["runs"].append(run(1080, 1920, "2.2", args.frames_1080, precision, nthreads))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
