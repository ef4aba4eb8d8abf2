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


needs_ref = pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libcbinfer_ref.so")),
                               reason="oracle/_ref not built")


@pytest.mark.gpu
@needs_ref
def test_cpp_tool_calibrate_and_sweep_match_reference(tool, tmp_path):
    """cbx_run --mode calibrate / sweep (cbench calibrate / sweep over the B200
    engine, exact mode) reproduce the reference's own calibrate_thresholds and
    sweep_threshold_factor on the same sequence: same grids, chosen thresholds,
    per-candidate error, changed-pixel and MAC totals."""
    from oracle import Ref
    spec = paper_spec(40, 56)
    cfg = dict(channels=3, height=40, width=56, sprites=[(9, 2, 0.9)], noise=0.004, seed=5)
    from oracle import Oracle
    orc = Oracle()
    net, wdir, seq = write_case(tmp_path, orc, spec, 1, cfg, 5)
    frames = [orc.synth_frame(cfg, f) for f in range(5)]
    ref = Ref()
    rnet = ref.load_network(spec, 1, weights_dir=wdir)
    want_th, want_sweep = rnet.calibrate(frames, grid_size=6, budget=0.5)
    r = subprocess.run([tool, "--net", net, "--weights", wdir, "--seq", seq, "--precision", "exact",
                        "--mode", "calibrate", "--grid", "6", "--budget", "0.5"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == "layer,threshold,errorIncrease"
    got = [l.split(",") for l in lines[1:-1]]
    assert [(int(a), np.float32(b)) for a, b, _ in got] == [(l, np.float32(t)) for l, t, _ in want_sweep]
    np.testing.assert_allclose([float(c) for _, _, c in got], [e for _, _, e in want_sweep], rtol=0, atol=1e-7)
    assert lines[-1] == "thresholds: " + ",".join("%.9g" % t for t in want_th)

    factors = [0.0, 0.5, 1.0, 2.0]
    rnet.set_thresholds([0.04, 0.05, 0.05])
    want = rnet.sweep(frames, factors)
    r = subprocess.run([tool, "--net", net, "--weights", wdir, "--seq", seq, "--precision", "exact",
                        "--mode", "sweep", "--thresholds", "0.04,0.05,0.05", "--factors", "0,0.5,1,2"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rows = [l.split(",") for l in r.stdout.strip().splitlines()[1:]]
    assert len(rows) == len(factors)
    for row, (err, ch, macs) in zip(rows, want):
        assert abs(float(row[2]) - err) <= 1e-7
        assert int(row[3]) == ch and int(row[5]) == macs
