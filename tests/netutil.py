"""Shared helpers for the network-level parity tests."""
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAPER = os.path.join(ROOT, "paper_1704_04313_b200", "netspecs", "paper_like.json")


def paper_spec(h, w, taus=(0.04, 0.05, 0.05)):
    spec = json.load(open(PAPER))
    spec["inputHeight"], spec["inputWidth"] = h, w
    for l, t in zip([l for l in spec["layers"] if l["kind"] == "CBCONV"], taus):
        l["threshold"] = t
    return spec


def c1_spec(tau=0.05):
    return dict(inputChannels=16, inputHeight=128, inputWidth=128, numClasses=32,
                layers=[dict(kind="CBCONV", kernelH=3, kernelW=3, strideH=1, strideW=1, padH=1, padW=1,
                             outChannels=32, threshold=tau, fuseRelu=True, weightsFile="l1.w")])


def tiny_spec(tau=0.0):
    L = lambda k, o, f: dict(kind="CBCONV", kernelH=k, kernelW=k, padH=k // 2, padW=k // 2, outChannels=o,
                             threshold=tau, fuseRelu=True, weightsFile=f)
    return dict(inputChannels=2, inputHeight=16, inputWidth=16, numClasses=3, layers=[
        L(7, 4, "a"), dict(kind="MAXPOOL", window=2, stride=2), L(7, 6, "b"), dict(kind="MAXPOOL", window=2, stride=2),
        L(7, 8, "c"), dict(kind="CONV", kernelH=1, kernelW=1, outChannels=4, weightsFile="d"), dict(kind="RELU"),
        dict(kind="CONV", kernelH=1, kernelW=1, outChannels=3, weightsFile="e"), dict(kind="CLASSIFY")])


def generic_spec():
    """Every layer kind in unusual positions: non-CB 3x3 CONV feeding a CBCONV,
    standalone RELU, 3/2 pooling, strided CBCONV, no CLASSIFY (implicit argmax)."""
    return dict(inputChannels=3, inputHeight=37, inputWidth=45, numClasses=5, layers=[
        dict(kind="CONV", kernelH=3, kernelW=3, padH=1, padW=1, outChannels=6, weightsFile="a"),
        dict(kind="RELU"),
        dict(kind="CBCONV", kernelH=5, kernelW=3, strideH=2, strideW=1, padH=2, padW=1, outChannels=7,
             threshold=0.02, fuseRelu=False, weightsFile="b"),
        dict(kind="MAXPOOL", window=3, stride=2),
        dict(kind="CBCONV", kernelH=3, kernelW=3, padH=1, padW=1, outChannels=9, threshold=0.01,
             fuseRelu=True, weightsFile="c"),
        dict(kind="CBCONV", kernelH=1, kernelW=1, outChannels=12, threshold=0.0, fuseRelu=True, weightsFile="d"),
        dict(kind="CONV", kernelH=1, kernelW=1, outChannels=5, weightsFile="e")])


def to_pkg_spec(cbx, spec):
    return cbx.network_spec_from_json(json.dumps(spec))


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def stats_arr(stats):
    return np.array([[s["changedInputPixels"], s["changedOutputPixels"], s["gemmMacs"]] for s in stats], np.int64)
