"""GPU parity of whole programs (the bench workloads) against the oracle.

Cora-shaped GCN: every output and gradient element by element.  arxiv-shaped GCN at
BASELINE.json's full size, in the launch configuration bench.py times: the join index
bit-exact, and each hot-path step checked on the same inputs the GPU consumed (sampled
groups for the forward, every source row for the backward, sampled rows for projections).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import programs as op
from tests.util import FP32_TOL, TF32_TOL, assert_close, np_

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2605_24207_b200 import programs
    return programs


@pytest.mark.parametrize("prec", ["3xtf32", "tf32"])
def test_gcn_cora_full(P, prec):
    g = synth.cora_like(42)
    prog = P.GCNProgram(g, prec=prec)
    prog.step()
    torch.cuda.synchronize()
    extra = {}
    H, dW, dX0 = op.gcn_step(g, out=extra)
    tol = FP32_TOL if prec == "3xtf32" else TF32_TOL
    assert_close(np_(prog.H[-1]), H[-1], tol, "out")
    assert_close(np_(prog.H[1]), H[1], tol, "H1 (bias + ReLU)")
    for l in range(len(dW)):
        assert_close(np_(prog.dW[l]), dW[l], tol, f"dW{l}")
        assert_close(np_(prog.db[l]), extra["db"][l], tol, f"db{l}")
    assert_close(np_(prog.dH[0]), dX0, tol, "dX0")


def test_gcn_cora_cuda_graph(P):
    """The step captured in a CUDA graph replays to the same bits as eager launches."""
    g = synth.cora_like(42)
    prog = P.GCNProgram(g)
    prog.step()
    torch.cuda.synchronize()
    ref = [t.clone() for t in prog.dW] + [prog.H[-1].clone()]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        prog.step()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        prog.step()
    graph.replay()
    torch.cuda.synchronize()
    for a, b in zip(ref, list(prog.dW) + [prog.H[-1]]):
        assert torch.equal(a, b)


@pytest.mark.slow
def test_gcn_arxiv_full_size_sampled(P):
    g = synth.arxiv_like(42)
    prog = P.GCNProgram(g)
    prog.step()
    torch.cuda.synchronize()
    key = g["nodes"]["key"]
    o1 = oracle.build_join_index(g["edges"]["src"], g["edges"]["dst"], key, key)
    for k in ("group_ptr", "group_key", "group_dst_row", "src_row", "edge_row", "src_ptr", "src_pos"):
        np.testing.assert_array_equal(np_(getattr(prog.idx1, k)), o1[k], err_msg=k)
    o2 = oracle.build_join_index(g["edges"]["src"], g["edges"]["dst"], o1["group_key"], o1["group_key"])
    np.testing.assert_array_equal(np_(prog.idx2.src_row), o2["src_row"])
    w1 = oracle.gcn_norm(o1, len(key))
    assert_close(np_(prog.w1), w1, FP32_TOL, "norm")
    rng = np.random.default_rng(0)
    sizes = np.diff(o1["group_ptr"])
    sel = np.unique(np.concatenate([rng.choice(o1["n_groups"], 3000, replace=False),
                                    np.argsort(sizes)[-20:]]))          # + the 20 largest hubs
    # layer 1 forward on the projection the GPU produced: the LJA, then the O7 epilogue
    # (bias + ReLU) fused into its store
    Z0 = np_(prog.Z[0])
    b0 = g["b"][0]
    ref, _ = oracle.lja_fwd(o1, "src", "sum", src=Z0, edge=w1, edge_mode=1, sel=sel)
    assert_close(np_(prog.H[1])[sel], oracle.epilogue_fwd(ref, b0, "relu"), FP32_TOL, "H1 sampled")
    # projection (tcgen05 3xTF32) on sampled rows
    rows = rng.choice(len(key), 2000, replace=False)
    assert_close(Z0[rows], oracle.project(g["nodes"]["x"][rows], g["W"][0]), FP32_TOL, "Z0 rows")
    # layer 1 backward: the layer-2 projection backward dH1 = dZ1 W1 (from the GPU's dZ1), the
    # epilogue backward on every row (fused into that projection on the GPU), then the LJA
    # backward on every source row from the GPU's d(pre-activation)
    # (the ReLU mask is a decision taken in floating point: both sides take it from the GPU's
    # fp32 output -- pre = H1 - b, which is the pre-activation where H1 > 0 and gives the
    # zero derivative where H1 = 0)
    dH1, _, _ = oracle.project_bwd(np_(prog.H[1]), g["W"][1], np_(prog.dZ[1]), want_db=False)
    dP0, db0, _, _ = oracle.epilogue_bwd(dH1, np_(prog.H[1]) - b0, b0, "relu")
    assert_close(np_(prog.dP[0]), dP0, FP32_TOL, "dP0 all rows")
    assert_close(np_(prog.db[0]), db0, FP32_TOL, "db0")
    dZ0 = oracle.lja_bwd(o1, np_(prog.dP[0]), "src", "sum", src=Z0, edge=w1, edge_mode=1,
                         want=("src",))["src"]
    assert_close(np_(prog.dZ[0]), dZ0, FP32_TOL, "dZ0 all rows")
    # dW of layer 1 on the GPU's own dZ
    _, dW0, _ = oracle.project_bwd(g["nodes"]["x"], g["W"][0], np_(prog.dZ[0]), want_dx=False, want_db=False)
    assert_close(np_(prog.dW[0]), dW0, FP32_TOL, "dW0")


def test_host_streamed_steps_cora(P):
    """HostStreamedSteps (the e2e path of bench.py): inputs streamed from pinned host memory
    with the next step's copy overlapping the current step, replayed through a CUDA graph;
    gradients read back to host equal the oracle's."""
    g = synth.cora_like(42)
    prog = P.GCNProgram(g)
    cs = P.CapturedStep(prog)
    ins, _ = prog.host_io()
    host = [x.cpu().pin_memory() for x in ins]
    for x in ins:                      # the step must really read what the pipeline copies
        x.zero_()
    pipe = P.HostStreamedSteps(prog, cs.replay)
    pipe.prefetch(host)
    for i in range(3):
        out = pipe.step(next_inputs=host if i < 2 else None)
    torch.cuda.synchronize()
    _, dW, _ = op.gcn_step(g)
    for l in range(len(dW)):
        assert_close(out[l].numpy(), dW[l], FP32_TOL, f"dW{l}")
