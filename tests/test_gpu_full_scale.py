"""Full-size parity of configs 3 (MAG-shaped HGT) and 4 (hypergraph) in the launch
configuration bench.py times (one step of the whole program), against the oracle on the
inputs the GPU consumed -- the same scheme as the arxiv test in test_gpu_programs.py:
join indices bit-exact, projections on sampled rows, forward outputs on sampled groups
(including the largest hubs), backward gradients on every row of selected relations, and the
weight gradients on the GPU's own upstream gradient."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.util import FP32_TOL, assert_close, np_

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def P():
    from paper_2605_24207_b200 import programs
    return programs


def sample_groups(rng, o, n=2000, hubs=20):
    sizes = np.diff(o["group_ptr"])
    k = min(n, o["n_groups"])
    return np.unique(np.concatenate([rng.choice(o["n_groups"], k, replace=False),
                                     np.argsort(sizes)[-hubs:]]))


def test_hgt_mag_full_size_sampled(P):
    mag = synth.mag_like(42)
    prog = P.HGTProgram(mag)
    prog.step()
    torch.cuda.synchronize()
    assert prog.join_rows_per_step == 21_111_007
    d, h = prog.d, prog.h
    rng = np.random.default_rng(3)
    Y = {t: np_(prog.Y[t]) for t in prog.blocks}
    dY = {t: np_(prog.dY[t]) for t in prog.blocks}
    blk = lambda a, t, kind, key: a[t][:, prog.col[(kind, key)][1] * d:(prog.col[(kind, key)][1] + 1) * d]
    # projections (tcgen05 3xTF32) on sampled rows of every node type
    for t in prog.blocks:
        rows = rng.choice(prog.n[t], min(1500, prog.n[t]), replace=False)
        assert_close(Y[t][rows], oracle.project(mag["h"][t][rows], np_(prog.W[t])), FP32_TOL, f"Y[{t}]")
    dQ_sum = {t: np.zeros((prog.n[t], d)) for t in prog.targets}
    for name, r in mag["rels"].items():
        ts, tt = r["src_type"], r["dst_type"]
        o = oracle.build_join_index(r["src"], r["dst"], mag["key"][ts], mag["key"][tt])
        gi = prog.idx[name]
        # dense-group index: T rows in key order; the compact oracle groups sit at their rank
        rows = np.searchsorted(np.sort(mag["key"][tt]), o["group_key"])
        np.testing.assert_array_equal(np_(gi.group_key)[rows], o["group_key"])
        np.testing.assert_array_equal(np_(gi.src_row), o["src_row"], err_msg=name)
        np.testing.assert_array_equal(np_(gi.group_ptr)[np.append(rows, gi.n_groups)],
                                      np.append(o["group_ptr"][:-1], o["n_join_rows"]))
        K, M, Q = blk(Y, ts, "k", name), blk(Y, ts, "m", name), blk(Y, tt, "q", tt)
        sel = sample_groups(rng, o)
        ref, rlse = oracle.lja_fwd(o, agg="softmax", src=M, src_key=K, dst=Q, heads=h, scale=1.0,
                                   sel=sel)
        assert_close(np_(prog.O[name])[rows[sel]], ref, FP32_TOL, f"O[{name}] sampled")
        assert_close(np_(prog.lse[name])[rows[sel]], rlse, FP32_TOL, f"lse[{name}] sampled")
        if name in ("has_topic", "affiliated_with"):     # the hub-heaviest relations
            dO = np_(prog.d_out[tt])[rows]
            g = oracle.lja_bwd(o, dO, agg="softmax", src=M, src_key=K, dst=Q, heads=h, scale=1.0)
            assert_close(blk(dY, ts, "k", name), g["src_key"], FP32_TOL, f"dK'[{name}] all rows")
            assert_close(blk(dY, ts, "m", name), g["src"], FP32_TOL, f"dM'[{name}] all rows")
            dQ_sum[tt] += g["dst"]
    # the field / institution query gradients come from one relation each
    for t in ("field", "institution"):
        assert_close(blk(dY, t, "q", t), dQ_sum[t], FP32_TOL, f"dQ[{t}]")
    # dW / dH of the query-only types on the GPU's own dY (the oracle GEMM is a plain loop)
    for t in ("field", "institution"):
        dX, dW, _ = oracle.project_bwd(mag["h"][t], np_(prog.W[t]), dY[t], want_db=False)
        assert_close(np_(prog.dW[t]), dW, FP32_TOL, f"dW[{t}]")
        assert_close(np_(prog.dH[t]), dX, FP32_TOL, f"dH[{t}]")


def test_hypergraph_full_size_sampled(P):
    hg = synth.hypergraph_like(42)
    prog = P.HypergraphProgram(hg)
    prog.step()
    torch.cuda.synchronize()
    nk, hk = hg["nodes"]["key"], hg["hyperedges"]["key"]
    iv, ih = hg["inc"]["node"], hg["inc"]["hyper"]
    o1 = oracle.build_join_index(iv, ih, nk, hk)
    o2 = oracle.build_join_index(ih, iv, o1["group_key"], nk)
    for k in ("group_ptr", "group_key", "group_dst_row", "src_row", "edge_row", "src_ptr", "src_pos"):
        np.testing.assert_array_equal(np_(getattr(prog.idx1, k)), o1[k], err_msg=k)
        np.testing.assert_array_equal(np_(getattr(prog.idx2, k)), o2[k], err_msg=k)
    rng = np.random.default_rng(4)
    Z = np_(prog.Z)
    rows = rng.choice(len(nk), 2000, replace=False)
    assert_close(Z[rows], oracle.project(hg["nodes"]["x"][rows], hg["theta"]), FP32_TOL, "Z rows")
    sel1 = sample_groups(rng, o1)
    ref1, _ = oracle.lja_fwd(o1, "src", "sum", src=Z, sel=sel1)
    assert_close(np_(prog.Eh)[sel1], ref1, FP32_TOL, "hop 1 sampled")
    Eh = np_(prog.Eh)
    sel2 = sample_groups(rng, o2)
    ref2, _ = oracle.lja_fwd(o2, "src", "mean", src=Eh, sel=sel2)
    assert_close(np_(prog.Xo)[sel2], ref2, FP32_TOL, "hop 2 sampled")
    # backward, every row: hop 2 (MEAN) into dEh, hop 1 (SUM) into dZ on the GPU's dEh
    dEh = oracle.lja_bwd(o2, np_(prog.d_out), "src", "mean", src=Eh, want=("src",))["src"]
    assert_close(np_(prog.dEh), dEh, FP32_TOL, "dEh all rows")
    dZ = oracle.lja_bwd(o1, np_(prog.dEh), "src", "sum", src=Z, want=("src",))["src"]
    assert_close(np_(prog.dZ), dZ, FP32_TOL, "dZ all rows")
    dX, dTheta, _ = oracle.project_bwd(hg["nodes"]["x"], hg["theta"], np_(prog.dZ), want_db=False)
    assert_close(np_(prog.dTheta), dTheta, FP32_TOL, "dTheta")
    assert_close(np_(prog.dX), dX, FP32_TOL, "dX")
