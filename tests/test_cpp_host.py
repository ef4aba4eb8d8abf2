"""The C++ drop-in host API (include/cbinfer_b200.hpp) and its driver
tools/cbx_run (the counterpart of the reference's `cbench run`)."""
import json
import os
import subprocess

import numpy as np
import pytest

from netutil import paper_spec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "tools", "cbx_run")


@pytest.fixture(scope="module")
def tool():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools")], check=True)
    return TOOL


def write_case(tmp, orc, spec, seed, cfg, frames):
    import paper_1704_04313_b200 as cbx
    sp = cbx.network_spec_from_json(json.dumps(spec))
    cbx.generate_weights(sp, str(tmp / "w"), seed)
    (tmp / "net.json").write_text(cbx.network_spec_to_json(sp))
    seq = tmp / "seq"
    seq.mkdir()
    for f in range(frames):
        orc.synth_frame(cfg, f).astype("<f4").tofile(seq / f"frame_{f:04d}.f32le")
    (seq / "manifest.json").write_text(json.dumps(dict(channels=cfg["channels"], height=cfg["height"],
                                                       width=cfg["width"], frames=frames)))
    return str(tmp / "net.json"), str(tmp / "w"), str(seq)


def test_cpp_tool_usage_errors(tool, tmp_path):
    r = subprocess.run([tool], capture_output=True, text=True)
    assert r.returncode == 1 and "usage" in r.stderr
    r = subprocess.run([tool, "--net", str(tmp_path / "missing.json"), "--weights", str(tmp_path), "--seq", "x"],
                       capture_output=True, text=True)
    assert r.returncode == 2 and "cannot open network spec" in r.stderr


@pytest.mark.gpu
def test_cpp_tool_matches_oracle(tool, tmp_path, orc):
    spec = paper_spec(48, 64)
    cfg = dict(channels=3, height=48, width=64, sprites=[(10, 2, 0.9)], noise=0.01, seed=3)
    net, wdir, seq = write_case(tmp_path, orc, spec, 1, cfg, 5)
    r = subprocess.run([tool, "--net", net, "--weights", wdir, "--seq", seq, "--precision", "exact"],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    rows = [l.split(",") for l in r.stdout.strip().splitlines()]
    hdr, rows = rows[0], rows[1:]
    onet = orc.load_network(spec, orc.generate_weights(spec, 1))
    for f, row in enumerate(rows):
        want = onet.forward_frame(orc.synth_frame(cfg, f))
        assert int(row[2]) == want["macsTotal"]
        cb = [k for k, l in enumerate(spec["layers"]) if l["kind"] == "CBCONV"]
        got = [int(v) for v in row[3:3 + 2 * len(cb)]]
        exp = sum(([want["stats"][k]["changedInputPixels"], want["stats"][k]["changedOutputPixels"]] for k in cb), [])
        assert got == exp
        lab = want["labels"].reshape(-1).astype(np.uint64)
        assert int(row[-1]) == int((lab * (np.arange(lab.size) % 9973 + 1)).sum())
