"""GPU parity of the hypergraph (config 4) and HGT (config 3) programs against the oracle,
element by element, at reduced scale with the configs' structure (power-law incidence with
hub hyperedges; four node relations and four edge relations with dense target groups)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import programs as op
from tests.util import FP32_TOL, assert_close, np_

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2605_24207_b200 import programs
    return programs


def test_hypergraph_two_hop(P):
    hg = synth.hypergraph_like(3, n_nodes=20000, n_hyper=3000, n_inc=120000, d=128)
    prog = P.HypergraphProgram(hg)
    prog.step()
    torch.cuda.synchronize()
    ref = op.hypergraph_step(hg)
    np.testing.assert_array_equal(np_(prog.idx1.group_key), ref["o1"]["group_key"])
    np.testing.assert_array_equal(np_(prog.idx2.src_row), ref["o2"]["src_row"])
    assert_close(np_(prog.Xo), ref["Xo"], FP32_TOL, "Xo")
    assert_close(np_(prog.dTheta), ref["dTheta"], FP32_TOL, "dTheta")
    assert_close(np_(prog.dX), ref["dX"], FP32_TOL, "dX")


def test_hgt_layer(P):
    mag = synth.mag_like(5, scale=0.004)
    prog = P.HGTProgram(mag)
    prog.step()
    torch.cuda.synchronize()
    d = prog.d
    Ht_ref = {t: np.zeros((prog.n[t], d)) for t in prog.targets}
    dY_ref = {t: np.zeros((prog.n[t], len(b) * d)) for t, b in prog.blocks.items()}
    for name, r in prog.rels.items():
        ts, tt = r["src_type"], r["dst_type"]
        W_s, W_t = np_(prog.W[ts]), np_(prog.W[tt])
        ik = prog.col[("k", name)][1]
        im = prog.col[("m", name)][1]
        iq = prog.col[("q", tt)][1]
        res = op.hgt_relation(mag["h"][ts], mag["h"][tt], W_s[ik * d:(ik + 1) * d],
                              W_s[im * d:(im + 1) * d], W_t[iq * d:(iq + 1) * d],
                              mag["key"][ts], mag["key"][tt], r["src"], r["dst"], prog.h,
                              np_(prog.d_out[tt]))
        O = np_(prog.O[name])
        rows = res["dense_rows"]
        assert_close(O[rows], res["out"], FP32_TOL, f"O[{name}]")
        empty = np.setdiff1d(np.arange(prog.n[tt]), rows)
        assert np.all(O[empty] == 0.0), name                     # empty groups aggregate to 0
        assert_close(np_(prog.lse[name])[rows], res["lse"], FP32_TOL, f"lse[{name}]")
        Ht_ref[tt][rows] += res["out"]
        dY_ref[ts][:, ik * d:(ik + 1) * d] = res["dK"]
        dY_ref[ts][:, im * d:(im + 1) * d] = res["dM"]
        dY_ref[tt][:, iq * d:(iq + 1) * d] += res["dQ"]     # shared Q: dQ summed over phi
    for t in prog.targets:                                   # Ht rows: dense, T-key order
        assert_close(np_(prog.Ht[t]), Ht_ref[t], FP32_TOL, f"Ht[{t}]")
    for t in prog.blocks:
        assert_close(np_(prog.dY[t]), dY_ref[t], FP32_TOL, f"dY[{t}]")
        dX, dW, _ = oracle.project_bwd(mag["h"][t], np_(prog.W[t]), np_(prog.dY[t]), want_db=False)
        assert_close(np_(prog.dH[t]), dX, FP32_TOL, f"dH[{t}]")
        assert_close(np_(prog.dW[t]), dW, FP32_TOL, f"dW[{t}]")


def test_dense_groups_index(P):
    """RNN_IDX_DENSE_GROUPS: every T row is a group in key order; empty groups aggregate to 0."""
    from paper_2605_24207_b200 import rnn
    rng = np.random.default_rng(2)
    db = synth.random_db(rng, 50, 80, 400, d_s=16)
    cu = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
    gi = rnn.build_join_index(cu(db["e_src"]), cu(db["e_dst"]), cu(db["s_key"]), cu(db["t_key"]),
                              dense_groups=True, rows_per_item=8)
    oi = oracle.build_join_index(db["e_src"], db["e_dst"], db["s_key"], db["t_key"])
    assert gi.n_groups == 80
    np.testing.assert_array_equal(np_(gi.group_key), np.sort(db["t_key"]))
    np.testing.assert_array_equal(np_(gi.src_row), oi["src_row"])
    z = db["z_s"]
    for agg in ("sum", "mean"):
        out = np_(rnn.join_aggregate_fwd(gi, rnn.make_query("src", agg, src=cu(z))))
        ref, _ = oracle.lja_fwd(oi, "src", agg, src=z)
        rows = np.searchsorted(np.sort(db["t_key"]), oi["group_key"])
        assert_close(out[rows], ref, FP32_TOL, agg)
        empty = np.setdiff1d(np.arange(80), rows)
        assert np.all(out[empty] == 0.0)
        dO = rng.standard_normal((80, 16)).astype(np.float32)
        g = rnn.join_aggregate_bwd(gi, rnn.make_query("src", agg, src=cu(z)), cu(dO))["src"]
        gr = oracle.lja_bwd(oi, dO[rows], "src", agg, src=z)["src"]
        assert_close(np_(g), gr, FP32_TOL, "d_src " + agg)
