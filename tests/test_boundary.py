"""CPU (no GPU needed): the C-ABI library loads, exports every symbol
include/cbx.h declares, and its host-side logic mirrors the reference
(spec parsing, chain_dims, weight-file checks, fixtures, error mapping)."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

import paper_1704_04313_b200 as cbx
from netutil import PAPER, generic_spec, paper_spec, tiny_spec, to_pkg_spec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_match_header():
    hdr = open(os.path.join(ROOT, "include", "cbx.h")).read()
    declared = set(re.findall(r"CBX_API\s+[\w\s\*]+?\b(cbx_\w+)\s*\(", hdr))
    assert declared == set(cbx._cbx.EXPORTS)
    lib = ctypes.CDLL(cbx._cbx.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name


def test_library_is_sm100a():
    data = open(cbx._cbx.LIB_PATH, "rb").read()
    assert b"sm_100a" in data


def test_spec_roundtrip_and_errors():
    spec = cbx.load_network_spec(PAPER)
    back = cbx.network_spec_from_json(cbx.network_spec_to_json(spec))
    assert back == spec
    with pytest.raises(cbx.SpecError):
        cbx.network_spec_from_json("{not json")
    with pytest.raises(cbx.IoError):
        cbx.load_network_spec("/nonexistent.json")


def test_chain_dims_paper_and_tiny():
    shapes = cbx.chain_dims(to_pkg_spec(cbx, paper_spec(1080, 1920)))
    assert shapes[0][1] == (4, 1080, 1920) and shapes[2][1] == (52, 540, 960)
    assert shapes[4][1] == (304, 270, 480) and shapes[-1][1] == (1, 270, 480)
    spec = to_pkg_spec(cbx, tiny_spec())
    shapes = cbx.chain_dims(spec)  # test_network.cpp:90-102
    assert shapes[0][1] == (4, 16, 16) and shapes[1][1] == (4, 8, 8) and shapes[2][1] == (6, 8, 8)
    assert shapes[3][1] == (6, 4, 4) and shapes[4][1] == (8, 4, 4) and shapes[5][1] == (4, 4, 4)
    assert shapes[7][1] == (3, 4, 4) and spec.layers[2].inChannels == 4


def test_chain_dims_rejects():
    spec = to_pkg_spec(cbx, tiny_spec())
    spec.numClasses = 5
    with pytest.raises(cbx.SpecError):
        cbx.chain_dims(spec)
    empty = cbx.NetworkSpec(4, 4, 4, 1, [])
    with pytest.raises(cbx.SpecError):
        cbx.chain_dims(empty)
    bad = to_pkg_spec(cbx, tiny_spec())
    bad.layers[0].kernelH = 40
    bad.layers[0].padH = 0
    with pytest.raises(cbx.GeometryError):
        cbx.chain_dims(bad)
    cls = to_pkg_spec(cbx, tiny_spec())
    cls.layers.insert(0, cbx.LayerSpec(kind="CLASSIFY"))
    with pytest.raises(cbx.SpecError):
        cbx.chain_dims(cls)


def test_weights_io(tmp_path):
    spec = to_pkg_spec(cbx, tiny_spec())
    w = cbx.generate_weights(spec, str(tmp_path), 5)
    l = spec.layers[4]
    K, b = cbx.read_weights_f32le(str(tmp_path / l.weightsFile), l.geom())
    assert np.array_equal(K, w[4][0]) and np.array_equal(b, w[4][1])
    f = tmp_path / l.weightsFile
    data = f.read_bytes()
    f.write_bytes(data[:-4])
    with pytest.raises(cbx.IoError):
        cbx.read_weights_f32le(str(f), l.geom())
    f.write_bytes(data + b"\0\0\0\0")
    with pytest.raises(cbx.IoError):
        cbx.read_weights_f32le(str(f), l.geom())
    f.write_bytes(data[:-4] + np.array([np.nan], "<f4").tobytes())
    with pytest.raises(cbx.IoError):
        cbx.read_weights_f32le(str(f), l.geom())


def test_fixtures_match_oracle(orc):
    for spec in (paper_spec(48, 64), tiny_spec(), generic_spec()):
        a = cbx.generate_weights(to_pkg_spec(cbx, spec), None, 17)
        b = orc.generate_weights(spec, 17)
        assert a.keys() == b.keys()
        for k in a:
            assert np.array_equal(a[k][0], b[k][0]) and np.array_equal(a[k][1], b[k][1])
    cfg = dict(channels=3, height=48, width=64, sprites=[(10, 2, 0.9), (7, 5, 0.6)], noise=0.01, seed=3)
    for f in range(4):
        assert np.array_equal(cbx.synth_frame(cfg, f).view(np.uint32), orc.synth_frame(cfg, f).view(np.uint32))


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    spec = to_pkg_spec(cbx, tiny_spec())
    w = cbx.generate_weights(spec, None, 1)
    with pytest.raises(cbx.CudaError):
        cbx.Network(spec, w)
