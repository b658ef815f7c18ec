"""SURVEY sec 8f item 2, attention variants, against oracle compositions: the original HGT's
JOINT softmax over every relation into a target type (one softmax LJA over the union of the
relations, sources keyed by (relation, key) -- programs.HGTJointProgram) and HyGNN's double
attention (node-level then hyperedge-level softmax LJAs, PAPER.md:956 --
programs.HypergraphAttentionProgram)."""
import numpy as np
import pytest
import torch

import synth
from oracle import programs as op
from tests.util import FP32_TOL, assert_close, np_

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2605_24207_b200 import programs
    return programs


def test_hgt_joint_softmax(P):
    mag = synth.mag_like(5, scale=0.004)
    prog = P.HGTJointProgram(mag)
    prog.step()
    torch.cuda.synchronize()
    par = P.hgt_parameters(mag, 7)
    out, g = op.hgt_joint_step(mag, par, mag["heads"])
    d = mag["d"]
    for t in prog.targets:
        assert_close(np_(prog.Ht[t]), out[t], FP32_TOL, f"Ht[{t}]")
        assert_close(np_(prog.dWq[t]), g["dWq"][t], FP32_TOL, f"dWq[{t}]")
    for name in mag["rels"]:
        dW = np_(prog.dWkm[name])
        assert_close(dW[:d], g["dWk"][name], FP32_TOL, f"dWk[{name}]")
        assert_close(dW[d:], g["dWm"][name], FP32_TOL, f"dWm[{name}]")
    for t, ref in g["dH"].items():
        assert_close(np_(prog.dH[t]), ref, FP32_TOL, f"dH[{t}]")
    # the joint softmax differs from the per-relation one wherever a target has >= 2 relations
    per_rel = P.HGTProgram(mag)
    per_rel.forward()
    torch.cuda.synchronize()
    assert not np.allclose(np_(per_rel.Ht["paper"]), np_(prog.Ht["paper"]), atol=1e-3)


def test_hygnn_double_attention(P):
    hg = synth.hypergraph_like(6, n_nodes=20_000, n_hyper=3_000, n_inc=100_000, d=128)
    prog = P.HypergraphAttentionProgram(hg)
    prog.step()
    torch.cuda.synchronize()
    ref = op.hygnn_attention_step(hg, P.hygnn_attention_parameters(128, 13), 8)
    assert_close(np_(prog.Eh), ref["Eh"], FP32_TOL, "Eh (node-level attention)")
    assert_close(np_(prog.Xo), ref["Xo"], FP32_TOL, "Xo (hyperedge-level attention)")
    dWkv1, dWkv2 = np_(prog.dWkv1), np_(prog.dWkv2)
    scale = 1.0 / np.sqrt(128 / 8)
    # key maps carry the folded scale: d(scaled W) = d(W) / scale
    assert_close(dWkv2[:128], ref["dWk2"], FP32_TOL, "dWk2")
    assert_close(dWkv2[128:], ref["dWv2"], FP32_TOL, "dWv2")
    assert_close(dWkv1[:128], ref["dWk1"], FP32_TOL, "dWk1")
    assert_close(dWkv1[128:], ref["dWv1"], FP32_TOL, "dWv1")
    assert_close(np_(prog.dWq1), ref["dWq1"], FP32_TOL, "dWq1")
    assert_close(np_(prog.dWq2), ref["dWq2"], FP32_TOL, "dWq2")
    assert_close(np_(prog.dX), ref["dX"], FP32_TOL, "dX")
    assert_close(np_(prog.dE0), ref["dE0"], FP32_TOL, "dE0 (hyperedge embeddings)")
    del scale
