"""GPU parity of A6 (DHN closed-walk aggregates C2/C3/C4, rnn_dhn_fwd / rnn_dhn_bwd) against
the fp64 oracle (ora_dhn_fwd / ora_dhn_bwd, pinned in test_oracle_dhn.py), element by element.

Graphs: directed and undirected, with duplicated Edge tuples (multiplicity), dangling nodes
(no out-edges) and isolated ones, and a power-law products-shaped instance (synth.products_like,
config 5 structure) at reduced scale; widths d = 32 (config 5), 7 and 100 (ragged lanes and
channel slices); both plain and RNN_IDX_DENSE_GROUPS indices."""
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


def random_graph(seed, n, m, directed, dup=0.05, dangling=0.1):
    rng = np.random.default_rng(seed)
    keys = (rng.permutation(n).astype(np.int64) * 7 - 1000)
    s = rng.integers(0, n, m)
    t = rng.integers(0, n, m)
    if dangling:   # some nodes get no out-edges
        dead = rng.random(n) < dangling
        keep = ~dead[t]
        s, t = s[keep], t[keep]
    ok = s != t
    s, t = s[ok], t[ok]
    if not directed:
        s, t = np.concatenate([s, t]), np.concatenate([t, s])
    nd = int(len(s) * dup)
    if nd:
        j = rng.integers(0, len(s), nd)
        s, t = np.concatenate([s, s[j]]), np.concatenate([t, t[j]])
    return keys, keys[t], keys[s]      # keys, e_root (n), e_nbr (v): Edge(n, v)


def feats(seed, n, d, k):
    rng = np.random.default_rng(seed + 1)
    return [rng.standard_normal((n, d)).astype(np.float32) for _ in range(k)]


def cu(a):
    return torch.as_tensor(np.ascontiguousarray(a)).cuda()


def build(rnn, keys, e_n, e_v, dense=False):
    gi = rnn.build_join_index(cu(e_v), cu(e_n), cu(keys), cu(keys), dense_groups=dense)
    oi = oracle.build_join_index(e_v, e_n, keys, keys, within_by_src_key=True)
    return gi, oi


def run_case(rnn, keys, e_n, e_v, k, d, seed, dense=False, f0_none=False, bwd=True):
    gi, oi = build(rnn, keys, e_n, e_v, dense)
    n = len(keys)
    f = feats(seed, n, d, k)
    if f0_none:
        f[0] = np.ones((n, d), np.float32)
    fg = [None if (i == 0 and f0_none) else cu(x) for i, x in enumerate(f)]
    out = np_(rnn.dhn_fwd(gi, k, fg))
    ref = oracle.dhn_fwd(k, oi, keys, f)
    rows = np.searchsorted(np_(gi.group_key), oi["group_key"])
    assert_close(out[rows], ref, FP32_TOL, f"C{k} fwd")
    if dense:    # roots without out-edges are dense groups with no walks -> 0
        empty = np.setdiff1d(np.arange(gi.n_groups), rows)
        assert np.all(out[empty] == 0.0)
    if not bwd:
        return
    rng = np.random.default_rng(seed + 2)
    d_out = rng.standard_normal((gi.n_groups, d)).astype(np.float32)
    grads = rnn.dhn_bwd(gi, k, fg, cu(d_out))
    ref_g = oracle.dhn_bwd(k, oi, keys, f, d_out[rows])
    for i in range(k):
        assert_close(np_(grads[i]), ref_g[i], FP32_TOL, f"C{k} d f{i}")
    # saved walk sum (rnn_dhn_fwd_save / rnn_dhn_bwd_saved): the sum is C_k with f0 = 1, and
    # d f0 = dOut (.) sum replaces the f0 walk
    ws = torch.full((max(gi.n_groups, 1), d + 5), float("nan"), device="cuda")[: gi.n_groups, :d]
    out2 = np_(rnn.dhn_fwd(gi, k, fg, walk_sum=ws))
    assert_close(out2[rows], ref, FP32_TOL, f"C{k} fwd (save)")
    ones = [np.ones((n, d), np.float32)] + f[1:]
    assert_close(np_(ws)[rows], oracle.dhn_fwd(k, oi, keys, ones), FP32_TOL, f"C{k} walk sum")
    grads2 = rnn.dhn_bwd(gi, k, fg, cu(d_out), walk_sum=ws)
    for i in range(k):
        assert_close(np_(grads2[i]), ref_g[i], FP32_TOL, f"C{k} d f{i} (saved)")
    if symmetric(e_n, e_v):   # RNN_DHN_SYMMETRIC_EDGE: d f1 | d f3 from one C4 walk
        grads3 = rnn.dhn_bwd(gi, k, fg, cu(d_out), walk_sum=ws, symmetric=True)
        for i in range(k):
            assert_close(np_(grads3[i]), ref_g[i], FP32_TOL, f"C{k} d f{i} (saved, symmetric)")


def symmetric(e_n, e_v):
    """Edge equals its reverse as a multiset."""
    a = np.stack([np.asarray(e_n), np.asarray(e_v)], 1)
    rec = [("x", a.dtype), ("y", a.dtype)]
    return np.array_equal(np.sort(np.ascontiguousarray(a).view(rec), axis=0),
                          np.sort(np.ascontiguousarray(a[:, ::-1]).view(rec), axis=0))


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("directed", [False, True])
def test_random_graph(rnn, k, directed):
    keys, e_n, e_v = random_graph(10 + k, 300, 2400, directed)
    run_case(rnn, keys, e_n, e_v, k, 32, seed=k)


@pytest.mark.parametrize("k", [3, 4])
def test_random_graph_symmetric(rnn, k):
    """Undirected without duplicates: the symmetric-Edge backward path runs (checked inside)."""
    keys, e_n, e_v = random_graph(30 + k, 300, 2400, directed=False, dup=0)
    assert symmetric(e_n, e_v)
    run_case(rnn, keys, e_n, e_v, k, 32, seed=k + 5)


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("d", [7, 100])
def test_ragged_width(rnn, k, d):
    keys, e_n, e_v = random_graph(20 + d, 200, 1500, directed=False)
    run_case(rnn, keys, e_n, e_v, k, d, seed=d)


@pytest.mark.parametrize("k", [2, 3, 4])
def test_dense_groups_and_no_f0(rnn, k):
    keys, e_n, e_v = random_graph(30 + k, 250, 1800, directed=True, dangling=0.3)
    run_case(rnn, keys, e_n, e_v, k, 32, seed=30 + k, dense=True, f0_none=True)


@pytest.mark.parametrize("k", [3, 4])
def test_products_shaped(rnn, k):
    """Power-law DC-SBM (config 5 structure), hubs and high clustering, d = 32."""
    g = synth.products_like(5, scale=0.0004 if k == 4 else 0.002)
    keys = g["nodes"]["key"]
    run_case(rnn, keys, g["edges"]["dst"], g["edges"]["src"], k, 32, seed=40 + k)


def test_triangle_counts_exact(rnn):
    """all-ones features, d = 1: C3(n) = (A^3)_nn exactly (integers in fp32)."""
    keys, e_n, e_v = random_graph(50, 120, 900, directed=True, dup=0.1)
    gi, oi = build(rnn, keys, e_n, e_v)
    ones = cu(np.ones((len(keys), 1), np.float32))
    for k in (2, 3, 4):
        out = np_(rnn.dhn_fwd(gi, k, [None] + [ones] * (k - 1)))[:, 0]
        ref = oracle.dhn_fwd(k, oi, keys, [np.ones((len(keys), 1))] * k)[:, 0]
        np.testing.assert_array_equal(out, ref)


def test_empty_and_errors(rnn):
    keys = np.arange(10, dtype=np.int64)
    gi = rnn.build_join_index(cu(np.zeros(0, np.int64)), cu(np.zeros(0, np.int64)), cu(keys), cu(keys))
    f = [cu(np.ones((10, 4), np.float32))] * 3
    out = rnn.dhn_fwd(gi, 3, f)
    assert out.shape[0] == 0
    gs = rnn.dhn_bwd(gi, 3, f, torch.zeros(1, 4, device="cuda"))
    assert all(float(x.abs().sum()) == 0.0 for x in gs)
    keys2, e_n, e_v = random_graph(1, 20, 60, directed=False)
    gi2, _ = build(rnn, keys2, e_n, e_v)
    with pytest.raises(rnn.RnnError, match="UNSUPPORTED"):
        rnn.dhn_fwd(gi2, 5, [None] + [cu(np.ones((20, 4), np.float32))] * 4)
    t = rnn.build_join_index(cu(e_v), cu(e_n), cu(keys2), cu(keys2), transpose=False)
    with pytest.raises(rnn.RnnError, match="transposed"):
        rnn.dhn_fwd(t, 3, [None] + [cu(np.ones((20, 4), np.float32))] * 2)


def test_dhn_program(rnn):
    """Config-5 layer (nine stacked 32x32 projections, C2/C3/C4, concat) vs oracle.dhn_step."""
    from oracle import programs as op
    from paper_2605_24207_b200 import programs
    g = synth.products_like(9, scale=0.0003)
    prog = programs.DHNProgram(g)
    prog.step()
    torch.cuda.synchronize()
    ref = op.dhn_step(g, np_(prog.W), np_(prog.d_out))
    assert_close(np_(prog.out), ref["out"], FP32_TOL, "out")
    assert_close(np_(prog.dY), ref["dY"], FP32_TOL, "dY")
    assert_close(np_(prog.dW), ref["dW"], FP32_TOL, "dW")
    assert_close(np_(prog.dH), ref["dH"], FP32_TOL, "dH")
    # join rows: Edge rows + closed 3- and 4-walks (homomorphism counts, exact integers)
    oi = oracle.build_join_index(g["edges"]["src"], g["edges"]["dst"], g["nodes"]["key"],
                                 g["nodes"]["key"], within_by_src_key=True)
    n = len(g["nodes"]["key"])
    cnt = sum(oracle.dhn_fwd(k, oi, g["nodes"]["key"], [np.ones((n, 1))] * k).sum() for k in (3, 4))
    ref_rows = oi["n_join_rows"] + int(cnt)
    assert abs(prog.join_rows_per_step - ref_rows) <= 1e-6 * ref_rows   # fp32 count sums


def test_symmetry_decided_on_index(rnn):
    """RNN_DHN_SYMMETRIC_EDGE is asserted only when the SURVIVING join rows are symmetric:
    Edge tuples whose endpoint keys are absent are dropped by the join and must not make a
    non-symmetric relation look symmetric."""
    from paper_2605_24207_b200.programs import edge_is_symmetric
    keys = np.array([1, 2, 3], np.int64)
    # Edge(n, v) as (n, v): (1,2), (2,1), (1,3) survive; (3,99) dangles -> not symmetric
    e_n, e_v = np.array([1, 2, 1, 3]), np.array([2, 1, 3, 99])
    gi = rnn.build_join_index(cu(e_v), cu(e_n), cu(keys), cu(keys), dense_groups=True)
    assert gi.n_join_rows == 3 and not edge_is_symmetric(gi)
    # (1,2), (2,1) survive; the dangling pair (3,99), (99,3) is dropped -> symmetric
    e_n, e_v = np.array([1, 2, 3, 99]), np.array([2, 1, 99, 3])
    gi = rnn.build_join_index(cu(e_v), cu(e_n), cu(keys), cu(keys), dense_groups=True)
    assert gi.n_join_rows == 2 and edge_is_symmetric(gi)
    # multiplicity counts: (1,2) twice, (2,1) once -> not symmetric
    e_n, e_v = np.array([1, 1, 2]), np.array([2, 2, 1])
    gi = rnn.build_join_index(cu(e_v), cu(e_n), cu(keys), cu(keys), dense_groups=True)
    assert not edge_is_symmetric(gi)


@pytest.mark.parametrize("k", [3, 4])
def test_root_subset(rnn, k):
    """rnn_dhn_fwd_roots / rnn_dhn_bwd_roots: only the listed roots are computed (repeats and
    out-of-range ids ignored; other output rows untouched); the backward gives the listed
    roots' nodes their complete gradient rows (walks rooted there, operands rotated) and 0
    elsewhere, from the FULL upstream gradient."""
    keys, e_n, e_v = random_graph(60 + k, 300, 2400, directed=False)
    gi, oi = build(rnn, keys, e_n, e_v)
    n, d = len(keys), 16
    f = feats(k, n, d, k)
    fg = [cu(x) for x in f]
    rng = np.random.default_rng(k)
    sel = np.sort(rng.choice(gi.n_groups, 60, replace=False)).astype(np.int32)
    roots = cu(np.concatenate([sel, sel[:5], [-3, gi.n_groups + 7]]).astype(np.int32))
    out = torch.full((gi.n_groups, d), float("nan"), device="cuda")
    ws = torch.full((gi.n_groups, d), float("nan"), device="cuda")
    rnn.dhn_fwd(gi, k, fg, out=out, walk_sum=ws, roots=roots)
    o = np_(out)
    full = np_(rnn.dhn_fwd(gi, k, fg))
    if k == 3:
        np.testing.assert_array_equal(o[sel], full[sel])       # deterministic walk
    else:
        assert_close(o[sel], full[sel], FP32_TOL, "C4 subset")  # fp32 atomics: order only
    others = np.setdiff1d(np.arange(gi.n_groups), sel)
    assert np.all(np.isnan(o[others]))
    d_out = rng.standard_normal((gi.n_groups, d)).astype(np.float32)
    grads = rnn.dhn_bwd(gi, k, fg, cu(d_out), walk_sum=ws, roots=roots)
    rows = np.searchsorted(np_(gi.group_key), oi["group_key"])
    ref = oracle.dhn_bwd(k, oi, keys, f, d_out[rows])
    node_rows = np_(gi.group_dst_row)[sel]
    other_rows = np.setdiff1d(np.arange(n), node_rows)
    for i in range(k):
        g = np_(grads[i])
        assert_close(g[node_rows], ref[i][node_rows], FP32_TOL, f"d f{i} listed")
        assert np.all(g[other_rows] == 0.0), i
