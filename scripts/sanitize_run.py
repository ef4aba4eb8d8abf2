"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): the paper net at 96x128 through every kernel family -- detect,
dilate+compact, the exact planar layer-1 conv, the tcgen05 convs (tf32, f16,
single CTA and CTA pairs, split accumulator, fused tail, persistent grid
capped so CTAs walk several tiles), the 8-bit camera path (byte detection +
RGBX copy, kind::i8 multi-pixel-row layer 1), the fp16 multi-pixel-row conv
(CBX_MPR_F16=1, R = 1 and 4), pooling, argmax, the op-level API -- a few
frames each. Test infrastructure (the oracle is not used).

  compute-sanitizer --tool memcheck python scripts/sanitize_run.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1704_04313_b200 as cbx  # noqa: E402

H, W = 96, 128
spec = json.load(open(os.path.join(ROOT, "paper_1704_04313_b200", "netspecs", "paper_like.json")))
spec["inputHeight"], spec["inputWidth"] = H, W
for l, t in zip([l for l in spec["layers"] if l["kind"] == "CBCONV"], (0.04, 0.05, 0.05)):
    l["threshold"] = t
sp = cbx.network_spec_from_json(json.dumps(spec))
w = cbx.generate_weights(sp, None, 1)
frames = [np.stack([cbx.synth_frame(dict(channels=3, height=H, width=W, sprites=[(14, 3, 0.9)], noise=0.01,
                                         seed=3 + s), f) for s in range(2)]) for f in range(4)]
u8s = [np.ascontiguousarray(np.clip(np.rint(fr * 255), 0, 255).astype(np.uint8).transpose(0, 2, 3, 1)) for fr in frames]
for prec, pair, maxctas, mpr in [("f16", -1, None, None), ("f16", 1, None, None), ("tf32", 0, "2", None),
                                 ("tf32", 1, "2", None), ("exact", -1, None, None), ("f16", -1, "3", "1"),
                                 ("f16", -1, None, "4")]:
    if maxctas:
        os.environ["CBX_TC_MAXCTAS"] = maxctas
    else:
        os.environ.pop("CBX_TC_MAXCTAS", None)
    if mpr:
        os.environ["CBX_MPR_F16"] = "1"
        os.environ["CBX_MPR_R"] = mpr
    else:
        os.environ.pop("CBX_MPR_F16", None)
    net = cbx.Network(sp, w, streams=2, precision=prec)
    net.set_tc_pair(pair)
    net.set_step_times(True)
    for f in range(4):
        net.forward(frames[f])
        net.forward(frames[f], "baseline")
    net.reset_state()
    for f in range(4):  # 8-bit frames: full, then steady native frames
        net.forward_u8(u8s[f])
        net.forward_u8(u8s[f], "baseline")
    net.step_times()
    net.close()
    print("ok", prec, pair, maxctas, flush=True)
print("sanitize workload done")
