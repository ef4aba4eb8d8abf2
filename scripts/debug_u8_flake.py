"""Debug: repeat the 40x80 8-bit native layer-1 check, report mismatching rows."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1704_04313_b200 as gpu
from oracle import Oracle
from netutil import paper_spec, to_pkg_spec
from test_gpu_u8 import u8_clip, decode
orc = Oracle()
h, w = int(sys.argv[1]), int(sys.argv[2])
prec = sys.argv[3]
spec = paper_spec(h, w)
wts = orc.generate_weights(spec, 1)
bad = 0
for rep in range(int(sys.argv[4])):
    onet = orc.load_network(spec, wts)
    net = gpu.Network(to_pkg_spec(gpu, spec), wts, precision=prec)
    clip = u8_clip(orc, h, w, 5, 3, [(12, 2, 0.9), (7, 3, 0.6)], 0.03)
    for f, fr in enumerate(clip):
        onet.forward_frame(decode(fr))
        net.forward_u8(fr)
        d1, u1 = net.trace(0)
        d2, u2 = onet.trace(0)
        if d1 is not None and not np.array_equal(d1, d2):
            rows = np.nonzero((d1 != d2).any(axis=1))[0]
            print(f"rep {rep} frame {f}: mismatch rows {rows.tolist()[:20]} gpu_ones={int(d1.sum())} ref_ones={int(d2.sum())}")
            x = net.layer_input(0)
            print("   layer_input(0) == decode(frame):", np.array_equal(x.view(np.uint32), decode(fr).view(np.uint32)))
            bad += 1
            break
    net.close()
print("bad", bad)
