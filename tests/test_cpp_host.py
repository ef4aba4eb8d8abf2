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


@pytest.mark.gpu
def test_cpp_tool_analyze_prop(tool, tmp_path, orc):
    """cbx_run --mode analyze-prop (cbench analyze-prop, cbench.cpp:242-302):
    one row per steady frame and CBCONV layer k >= 2; detected counts equal the
    oracle's updated counts, worst-case counts bound them."""
    spec = paper_spec(48, 64)
    cfg = dict(channels=3, height=48, width=64, sprites=[(10, 2, 0.9)], noise=0.01, seed=3)
    net, wdir, seq = write_case(tmp_path, orc, spec, 1, cfg, 4)
    r = subprocess.run([tool, "--net", net, "--weights", wdir, "--seq", seq, "--precision", "exact",
                        "--mode", "analyze-prop"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == "frameIndex,layer,detectedCount,worstCaseCount,detectedFraction,worstCaseFraction"
    rows = [l.split(",") for l in lines[1:]]
    assert [(int(a[0]), int(a[1])) for a in rows] == [(f, k) for f in (1, 2, 3) for k in (2, 3)]
    onet = orc.load_network(spec, orc.generate_weights(spec, 1))
    cb = [k for k, l in enumerate(spec["layers"]) if l["kind"] == "CBCONV"]
    stats = [onet.forward_frame(orc.synth_frame(cfg, f))["stats"] for f in range(4)]
    for row in rows:
        f, k = int(row[0]), int(row[1])
        assert int(row[2]) == stats[f][cb[k - 1]]["changedOutputPixels"]
        assert int(row[3]) >= int(row[2])
