"""SURVEY sec 8f item 4 on the GPU: selection sigma pushed into the join-index build
(rnn_select_mask + rnn_build_join_index_sel; the join rule's U(T(sigma(R1 |><| ...))),
PAPER.md:444, "selection pushdowns" :1031) and mini-batch streaming of an LJA whose source
embeddings stay in host memory (programs.MiniBatchLJA) -- against the
oracle on the filtered relation / the single-shot join-aggregate."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.util import FP32_TOL, assert_close, np_

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rnn():
    from paper_2605_24207_b200 import rnn
    return rnn


def cu(a):
    return torch.as_tensor(np.ascontiguousarray(a)).cuda()


OPS = {"==": np.equal, "!=": np.not_equal, "<": np.less, "<=": np.less_equal, ">": np.greater,
       ">=": np.greater_equal}


def test_select_mask_predicates(rnn):
    rng = np.random.default_rng(0)
    a = rng.integers(-5, 6, 10_000).astype(np.int64)
    f = rng.standard_normal(10_000).astype(np.float32)
    for op, fn in OPS.items():
        np.testing.assert_array_equal(np_(rnn.select_mask(cu(a), op, 2)), fn(a, 2).astype(np.uint8))
        np.testing.assert_array_equal(np_(rnn.select_mask(cu(f), op, 0.25)),
                                      fn(f, np.float32(0.25)).astype(np.uint8))
    m = rnn.select_mask(cu(a), ">=", -1)
    rnn.select_mask(cu(f), "<", 0.5, mask=m, combine="and")
    rnn.select_mask(cu(a), "==", 5, mask=m, combine="or")
    ref = ((a >= -1) & (f < np.float32(0.5))) | (a == 5)
    np.testing.assert_array_equal(np_(m), ref.astype(np.uint8))


@pytest.mark.parametrize("seed", range(6))
def test_index_with_selection(rnn, seed):
    """sigma(E) |><| S |><| T: the index of the masked build is the canonical index of the
    filtered relation (edge_row refers to rows of the unfiltered E), and the LJA over it
    equals the oracle's LJA over E[mask]."""
    rng = np.random.default_rng(seed)
    db = synth.random_db(rng, 300, 200, 8000, d_s=16)
    db["e_dst"][:2000] = db["t_key"][0]            # a hub
    etype = rng.integers(0, 5, 8000).astype(np.int64)
    ew = rng.random(8000).astype(np.float32)
    m = rnn.select_mask(cu(etype), "!=", 2)
    rnn.select_mask(cu(ew), ">", 0.3, mask=m, combine="and")
    mask = (etype != 2) & (ew > np.float32(0.3))
    np.testing.assert_array_equal(np_(m), mask.astype(np.uint8))
    gi = rnn.build_join_index(cu(db["e_src"]), cu(db["e_dst"]), cu(db["s_key"]), cu(db["t_key"]),
                              e_mask=m, rows_per_item=32)
    keep = np.nonzero(mask)[0]
    oi = oracle.build_join_index(db["e_src"][keep], db["e_dst"][keep], db["s_key"], db["t_key"])
    assert gi.n_join_rows == oi["n_join_rows"] and gi.n_groups == oi["n_groups"]
    for k in ("group_ptr", "group_key", "group_dst_row", "src_row", "src_ptr", "src_pos"):
        np.testing.assert_array_equal(np_(getattr(gi, k)), oi[k], err_msg=k)
    np.testing.assert_array_equal(np_(gi.edge_row), keep[oi["edge_row"]])
    z = db["z_s"]
    w = ew                                        # per-E-row weight, selected rows only
    q = rnn.make_query("src", "sum", src=cu(z), edge=cu(w))
    out = rnn.join_aggregate_fwd(gi, q)
    ref, _ = oracle.lja_fwd(oi, "src", "sum", src=z, edge=w[keep])
    assert_close(np_(out), ref, FP32_TOL, "fwd over sigma(E)")
    dO = rng.standard_normal(ref.shape).astype(np.float32)
    g = rnn.join_aggregate_bwd(gi, q, cu(dO))
    rg = oracle.lja_bwd(oi, dO, "src", "sum", src=z, edge=w[keep])
    assert_close(np_(g["src"]), rg["src"], FP32_TOL, "d_src")
    dw = np.zeros(8000)
    dw[keep] = rg["edge"][:, 0]
    assert_close(np_(g["edge"]).reshape(-1), dw, FP32_TOL, "d_w (0 on unselected rows)")


@pytest.mark.parametrize("agg,batch", [("sum", 4000), ("mean", 1500), ("sum", 100000)])
def test_minibatch_streaming(rnn, agg, batch):
    """Source embeddings in pinned host memory, target keys in batches: the streamed forward
    and the scattered source gradient equal the single-shot join-aggregate (oracle)."""
    from paper_2605_24207_b200 import programs
    hg = synth.hypergraph_like(4, n_nodes=30_000, n_hyper=8_000, n_inc=150_000, d=64)
    nk, hk = hg["nodes"]["key"], hg["hyperedges"]["key"]
    iv, ih = hg["inc"]["node"], hg["inc"]["hyper"]
    z = hg["nodes"]["x"]
    mb = programs.MiniBatchLJA(iv, ih, nk, hk, z, agg=agg, batch_groups=batch)
    assert len(mb.batches) == -(-len(hk) // batch)
    out = mb.forward().numpy()
    o = oracle.build_join_index(iv, ih, nk, hk)
    ref, _ = oracle.lja_fwd(o, "src", agg, src=z)
    rows = np.searchsorted(np.sort(hk), o["group_key"])          # dense T-key order
    assert_close(out[rows], ref, FP32_TOL, "streamed forward")
    empty = np.setdiff1d(np.arange(len(hk)), rows)
    assert np.all(out[empty] == 0)
    rng = np.random.default_rng(1)
    dO = rng.standard_normal((len(hk), 64)).astype(np.float32)
    d_src = np_(mb.backward(torch.from_numpy(dO).pin_memory()))
    rg = oracle.lja_bwd(o, dO[rows], "src", agg, src=z, want=("src",))["src"]
    assert_close(d_src, rg, FP32_TOL, "streamed d_src")
