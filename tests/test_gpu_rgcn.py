"""GPU parity of the R-GCN program (per-relation maps moved above the per-relation mean by
linearity, selection pushdown per relation, one stacked tcgen05 GEMM) against the oracle's
per-join-row definition (no pushdown) -- SURVEY sec 8f item 1."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.util import FP32_TOL, assert_close, np_

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scale", [0.1, 1.0])
def test_rgcn_layer(scale):
    from paper_2605_24207_b200 import programs
    g = synth.rgcn_like(5, n_nodes=int(8285 * scale), n_pairs=int(29043 * scale))
    prog = programs.RGCNProgram(g)
    prog.step()
    torch.cuda.synchronize()
    keys = g["nodes"]["key"]
    idx = oracle.build_join_index(g["edges"]["src"], g["edges"]["dst"], keys, keys)
    ref = oracle.rgcn_fwd(idx, g["edges"]["rel"], g["nodes"]["x"], g["W"])
    out = np_(prog.out)                                  # dense, node-key order
    rank = np.argsort(np.argsort(keys, kind="stable"), kind="stable")
    rows = rank[idx["group_dst_row"]]
    assert_close(out[rows], ref, FP32_TOL, "out (groups)")
    lone = np.setdiff1d(np.arange(len(keys)), rows)     # no in-edges: the self term only
    if len(lone):
        x_lone = g["nodes"]["x"][np.argsort(keys, kind="stable")[lone]]
        assert_close(out[lone], oracle.project(x_lone, g["W"][0]), FP32_TOL, "out (self only)")
    # backward: the full upstream gradient over every node row (dense, key order)
    dO = np.asarray(g["d_out"], np.float64)
    full_idx_rows = rows
    dx, dW = oracle.rgcn_bwd(idx, g["edges"]["rel"], g["nodes"]["x"], g["W"], dO[full_idx_rows])
    # self terms of the nodes without in-edges (not groups of the oracle index)
    if len(lone):
        node_rows = np.argsort(keys, kind="stable")[lone]
        dx[node_rows] += dO[lone] @ np.asarray(g["W"][0], np.float64)
        dW[0] += dO[lone].T @ np.asarray(g["nodes"]["x"], np.float64)[node_rows]
    assert_close(np_(prog.dX), dx, FP32_TOL, "dX")
    d = prog.d
    dWst = np_(prog.dWst)
    for r in range(prog.R + 1):
        assert_close(dWst[:, r * d:(r + 1) * d], dW[r], FP32_TOL, f"dW[{r}]")
