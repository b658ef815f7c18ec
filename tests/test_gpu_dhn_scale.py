"""A6 at config scale: the DHN code paths that only large roots take, exact int64 closed-walk
counts, and sampled-root parity on the full ogbn-products-shaped graph (config 5).

* Exact counts (rnn_dhn_count): C_k(n) with every operand 1 is the homomorphism count of the
  closed k-walk pattern rooted at n (Eq. 3 :1500) = (A^k)_nn of the Edge
  multigraph -- bit-exact against dense integer matrix powers and against the oracle.
* Big-root paths of the fp32 walk kernels, each forced by a constructed graph and proven to
  have run by the library's path counters (rnn_internal_dhn_stats):
    C3 global mark array (a root with in-degree > 6144),
    C4 hash-partitioned roots (> 8192 possible 2-hop keys), chunked neighbour passes and
    roots past the shared-memory cursor arrays (degree > 8192),
    C4 long-run queue overflow (> 512 runs longer than 96 entries in one pass).
  Forward and every backward operand are compared with the oracle element by element.
* Full scale (2,449,029 nodes, 123,718,280 Edge tuples): counts, fp32 C3 / C4 forward and the
  C4 backward at sampled roots.  The oracle runs on the subrelation induced by the sampled
  roots' 2-hop ball, which holds every closed 3- and 4-walk through them (the Edge relation
  is symmetric, so the closing node of a 4-walk is itself a neighbour of the root); the
  backward at node x is the walk aggregate rooted at x with rotated operands (rotation
  invariance of closed walks, SURVEY sec 8c O6 pin iv), evaluated by the oracle forward.
"""
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


def gpu_adj(rnn, keys, e_n, e_v):
    return rnn.build_join_index(cu(e_v), cu(e_n), cu(keys), cu(keys))


def ora_adj(keys, e_n, e_v):
    return oracle.build_join_index(e_v, e_n, keys, keys, within_by_src_key=True)


def dense_counts(keys, e_n, e_v, roots_key):
    """diag(A^k) for k = 2..4 by dense integer matrix powers, A[n, v] = multiplicity of
    Edge(n, v) (k = 2: the out-degree, the C2 rule's single Edge atom)."""
    order = np.argsort(keys)
    row = lambda k: order[np.searchsorted(keys[order], k)]
    n = len(keys)
    A = np.zeros((n, n), np.int64)
    np.add.at(A, (row(np.asarray(e_n)), row(np.asarray(e_v))), 1)
    r = row(np.asarray(roots_key))
    A2 = A @ A
    return {2: A.sum(1)[r], 3: np.einsum("ij,ji->i", A2, A)[r], 4: np.einsum("ij,ji->i", A2, A2)[r]}


def random_multigraph(seed, n, m, directed, dup):
    rng = np.random.default_rng(seed)
    keys = rng.permutation(n).astype(np.int64) * 3 - 77
    s, t = rng.integers(0, n, m), rng.integers(0, n, m)
    ok = s != t
    s, t = s[ok], t[ok]
    if not directed:
        s, t = np.concatenate([s, t]), np.concatenate([t, s])
    j = rng.integers(0, len(s), int(dup * len(s)))
    s, t = np.concatenate([s, s[j]]), np.concatenate([t, t[j]])
    return keys, keys[t], keys[s]


@pytest.mark.parametrize("directed,dup", [(False, 0.0), (True, 0.1), (False, 0.2)])
def test_counts_exact_small(rnn, directed, dup):
    keys, e_n, e_v = random_multigraph(7 + int(directed), 400, 5000, directed, dup)
    gi = gpu_adj(rnn, keys, e_n, e_v)
    oi = ora_adj(keys, e_n, e_v)
    ref = dense_counts(keys, e_n, e_v, oi["group_key"])
    for k in (2, 3, 4):
        got = np_(rnn.dhn_count(gi, k))
        np.testing.assert_array_equal(got, ref[k], err_msg=f"C{k}")
        o = oracle.dhn_fwd(k, oi, keys, [np.ones((len(keys), 1))] * k)[:, 0]
        np.testing.assert_array_equal(got, o.astype(np.int64), err_msg=f"C{k} oracle")
    # deterministic (integer arithmetic)
    assert torch.equal(rnn.dhn_count(gi, 4), rnn.dhn_count(gi, 4))


def test_counts_beyond_fp32(rnn):
    """A dense multigraph whose C4 counts exceed 2^24 (where fp32 stops being exact)."""
    rng = np.random.default_rng(3)
    n = 60
    keys = np.arange(n, dtype=np.int64) * 11
    s = rng.integers(0, n, 60_000)
    t = rng.integers(0, n, 60_000)
    ok = s != t
    e_n, e_v = keys[t[ok]], keys[s[ok]]
    gi = gpu_adj(rnn, keys, e_n, e_v)
    ref = dense_counts(keys, e_n, e_v, np_(gi.group_key))
    got = np_(rnn.dhn_count(gi, 4))
    assert got.max() > 2 ** 24
    np.testing.assert_array_equal(got, ref[4])
    np.testing.assert_array_equal(np_(rnn.dhn_count(gi, 3)), ref[3])


# ------------------------------------------------------------------------------------------
# big-root paths of the fp32 walk kernels
# ------------------------------------------------------------------------------------------
def check_walks(rnn, keys, e_n, e_v, k, d, seed, ks_count=True, dyadic=False, sym=False):
    """fp32 forward + every backward operand vs the oracle; exact counts vs the oracle.
    dyadic: features k/8 in [0.5, 1.5] -- for multigraphs whose walk sums run over 10^5
    terms through ONE key: every partial sum (< 2^21 in units of 1/8) is then exact in fp32
    whatever the accumulation order (random features put the order-dependent fp32
    rounding of 1.2e5-term atomic sums at ~1e-4, measured), so the comparison isolates the
    walk logic; a dropped or doubled run still shows as >= 1/600 relative error."""
    gi = gpu_adj(rnn, keys, e_n, e_v)
    oi = ora_adj(keys, e_n, e_v)
    n = len(keys)
    rng = np.random.default_rng(seed)
    if dyadic:
        f = [(rng.integers(4, 13, (n, d)) / 8.0).astype(np.float32) for _ in range(k)]
    else:
        f = [rng.standard_normal((n, d)).astype(np.float32) for _ in range(k)]
    fg = [cu(x) for x in f]
    rows = np.searchsorted(np_(gi.group_key), oi["group_key"])
    rnn.dhn_path_counters(reset=True)
    out = np_(rnn.dhn_fwd(gi, k, fg))
    paths = rnn.dhn_path_counters()
    assert paths["c4_value_overflow"] == 0, paths
    assert_close(out[rows], oracle.dhn_fwd(k, oi, keys, f), FP32_TOL, f"C{k} fwd")
    if dyadic:
        d_out = (rng.integers(-8, 9, (gi.n_groups, d)) / 8.0).astype(np.float32)
    else:
        d_out = rng.standard_normal((gi.n_groups, d)).astype(np.float32)
    grads = rnn.dhn_bwd(gi, k, fg, cu(d_out))
    ref_g = oracle.dhn_bwd(k, oi, keys, f, d_out[rows])
    for i in range(k):
        assert_close(np_(grads[i]), ref_g[i], FP32_TOL, f"C{k} d f{i}")
    if ks_count:
        got = np_(rnn.dhn_count(gi, k))
        ref = oracle.dhn_fwd(k, oi, keys, [np.ones((n, 1))] * k)[:, 0]
        np.testing.assert_array_equal(got[rows], ref.astype(np.int64))
    if sym:   # symmetric Edge: the dual-middle backward (d f1 | d f3 from one walk)
        ws_s = torch.empty((gi.n_groups, d), dtype=torch.float32, device="cuda")
        rnn.dhn_fwd(gi, k, fg, walk_sum=ws_s)
        rnn.dhn_path_counters(reset=True)
        grads_s = rnn.dhn_bwd(gi, k, fg, cu(d_out), walk_sum=ws_s, symmetric=True)
        paths_s = rnn.dhn_path_counters()
        for i in range(k):
            assert_close(np_(grads_s[i]), ref_g[i], FP32_TOL, f"C{k} d f{i} (sym)")
        return paths, paths_s
    return paths


def star_graph(seed, n_leaves, extra):
    """Undirected hub joined to every leaf, plus `extra` random leaf-leaf edges (triangles
    and 4-cycles through the hub)."""
    rng = np.random.default_rng(seed)
    n = n_leaves + 1
    keys = rng.permutation(n).astype(np.int64) + 1000
    hub = 0
    s = np.concatenate([np.full(n_leaves, hub), rng.integers(1, n, extra)])
    t = np.concatenate([np.arange(1, n), rng.integers(1, n, extra)])
    ok = s != t
    s, t = s[ok], t[ok]
    s, t = np.concatenate([s, t]), np.concatenate([t, s])
    return keys, keys[t], keys[s]


def test_c3_mark_array_path(rnn):
    """A root with in-degree 7,000 > H3_MAX_INDEG (3,072) keeps its in-neighbours in the
    per-CTA global mark array instead of the shared-memory hash set."""
    keys, e_n, e_v = star_graph(1, 7000, 3000)
    paths = check_walks(rnn, keys, e_n, e_v, 3, 8, seed=5)
    assert paths["c3_mark_roots"] >= 1, paths


@pytest.fixture(params=["slot", "compact_ids", "smem_s1"])
def c4_variant(request, monkeypatch):
    """Every C4 walk variant (switches read by the library at every launch): the
    slot-indexed L2 slab (default), the compact-id L2 slab it replaced (RNN_DHN_COMPACT_IDS)
    and shared-memory values (RNN_DHN_SMEM_S1)."""
    monkeypatch.delenv("RNN_DHN_SMEM_S1", raising=False)
    if request.param == "smem_s1":
        monkeypatch.setenv("RNN_DHN_SMEM_S1", "1")
    elif request.param == "compact_ids":
        monkeypatch.setenv("RNN_DHN_COMPACT_IDS", "1")
    else:
        monkeypatch.delenv("RNN_DHN_COMPACT_IDS", raising=False)
    return request.param


def test_c4_partitioned_chunked_path(rnn, c4_variant):
    """Leaves see 8,300 two-hop keys through the hub (> 8,192: hash partitions of w); the hub
    itself has 8,300 neighbours (> H4_DEG_CAP: no smem cursors, binary-searched partition
    starts) and walks its neighbours 32 at a time (chunked mode)."""
    keys, e_n, e_v = star_graph(2, 8300, 1000)
    paths, paths_s = check_walks(rnn, keys, e_n, e_v, 4, 4, seed=6, sym=True)
    for p in (paths, paths_s):   # the dual-middle symmetric walk takes the same big-root paths
        assert p["c4_partitioned_roots"] >= 1, p
        assert p["c4_chunked_passes"] >= 1, p
        assert p["c4_passes"] > p["c4_roots"], p


def test_c4_long_run_overflow(rnn, c4_variant):
    """Root n -> 600 neighbours v_i, each v_i -> w0 with multiplicity 200 (one long run per
    v_i in w0's partition; 600 > the 512-entry queue), w0 -> p0 -> n closes the walks.
    Directed multigraph plus random noise edges."""
    rng = np.random.default_rng(9)
    nv = 600
    n_nodes = nv + 3 + 400
    keys = rng.permutation(n_nodes).astype(np.int64) * 5
    root, w0, p0 = 0, 1, 2
    v = np.arange(3, 3 + nv)
    src = [np.full(nv, root), np.repeat(v, 200), [w0], [p0]]
    dst = [v, np.full(nv * 200, w0), [p0], [root]]
    a, b = rng.integers(0, n_nodes, 4000), rng.integers(0, n_nodes, 4000)
    ok = a != b
    src.append(a[ok]); dst.append(b[ok])
    s, t = np.concatenate(src), np.concatenate(dst)
    # Edge(n, v): root n = s side of the walk step n -> v
    paths = check_walks(rnn, keys, keys[s], keys[t], 4, 8, seed=7, dyadic=True)
    assert paths["c4_long_runs"] >= 512 and paths["c4_long_overflow"] >= 1, paths


# ------------------------------------------------------------------------------------------
# full ogbn-products-shaped graph (config 5), sampled roots
# ------------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def products():
    return synth.products_like(42, scale=1.0)


def ball_subrelation(keys, e_n, e_v, root_keys, hops):
    """Edge rows induced by the `hops`-hop out-ball of the roots (node keys are a permutation
    of [0, n), so a boolean array indexed by key is the membership test).  On a symmetric
    Edge relation a closed 3-walk n -> v -> w -> n stays in the 1-hop ball (w is a neighbour
    of n) and a closed 4-walk n -> v -> w -> p -> n in the 2-hop ball."""
    n = len(keys)
    inb = np.zeros(n, bool)
    inb[root_keys] = True
    for _ in range(hops):
        nb = e_v[inb[e_n]]
        inb[nb] = True
    m = inb[e_n] & inb[e_v]
    return e_n[m], e_v[m]


def test_products_full_scale_sampled(rnn, products):
    g = products
    keys = g["nodes"]["key"]
    e_n, e_v = g["edges"]["dst"], g["edges"]["src"]
    assert len(e_n) == 123_718_280 and len(keys) == 2_449_029
    gi = gpu_adj(rnn, keys, e_n, e_v)
    G, d = gi.n_groups, 32
    gk = np_(gi.group_key)
    deg = np.diff(np_(gi.group_ptr))
    # exact counts and fp32 walks for every root on the GPU
    counts = {k: np_(rnn.dhn_count(gi, k)) for k in (2, 3, 4)}
    x = g["nodes"]["x"]
    rng = np.random.default_rng(17)
    W = (rng.standard_normal((4, d, d)) / np.sqrt(d)).astype(np.float32)
    f = [(x @ W[i]).astype(np.float32) for i in range(4)]          # mu_{k,i}(h), given inputs
    fg = [cu(a) for a in f]
    rnn.dhn_path_counters(reset=True)
    c3 = np_(rnn.dhn_fwd(gi, 3, fg[:3]))
    c4 = np_(rnn.dhn_fwd(gi, 4, fg))
    paths = rnn.dhn_path_counters()
    d_out = rng.standard_normal((G, d)).astype(np.float32)
    g4 = rnn.dhn_bwd(gi, 4, fg, cu(d_out), want=[False, True, False, False])[1]
    g4 = np_(g4)
    # the symmetric Edge backward the bench runs (d f1 | d f3 from one dual-middle walk)
    ws4 = torch.empty((G, d), dtype=torch.float32, device="cuda")
    c4s = np_(rnn.dhn_fwd(gi, 4, fg, walk_sum=ws4))
    g4s = np_(rnn.dhn_bwd(gi, 4, fg, cu(d_out), want=[False, True, False, True], walk_sum=ws4,
                          symmetric=True)[1])
    assert paths["c4_roots"] == G and paths["c4_partitioned_roots"] > 0, paths
    assert paths["c4_value_overflow"] == 0, paths
    # sampled roots: 48 random + 8 of degree 200-600 (C3 also gets the 4 largest hubs)
    pick = rng.choice(G, 48, replace=False)
    mid = np.nonzero((deg >= 200) & (deg <= 600))[0]
    pick = np.unique(np.concatenate([pick, rng.choice(mid, min(8, len(mid)), replace=False)]))
    hubs = np.argsort(-deg)[:4]
    for k, sel in ((3, np.unique(np.concatenate([pick, hubs]))), (4, pick)):
        sub_n, sub_v = ball_subrelation(keys, e_n, e_v, gk[sel], hops=k - 2)
        oi = ora_adj(keys, sub_n, sub_v)
        # sampled roots are groups of the subrelation with their full out-lists
        og = np.searchsorted(oi["group_key"], gk[sel])
        assert np.array_equal(oi["group_key"][og], gk[sel])
        assert np.array_equal(np.diff(oi["group_ptr"])[og], deg[sel])
        ones = [np.ones((len(keys), 1))] * k
        ref_cnt = oracle.dhn_fwd(k, oi, keys, ones, sel=og)[:, 0]
        np.testing.assert_array_equal(counts[k][sel], ref_cnt.astype(np.int64), err_msg=f"C{k} counts")
        ref = oracle.dhn_fwd(k, oi, keys, f[:k], sel=og)
        assert_close((c3 if k == 3 else c4)[sel], ref, FP32_TOL, f"C{k} fwd (sampled roots)")
        if k == 4:
            assert_close(c4s[sel], ref, FP32_TOL, "C4 fwd, with walk sum (sampled roots)")
        if k == 4:
            # d f1(x) = sum over closed walks x -> w -> p -> n -> x of f2(w) f3(p) g(n),
            # g = f0 (.) dOut by node row: the walk aggregate rooted at x, operands rotated
            row_of = np_(gi.group_dst_row)
            gnode = np.zeros((len(keys), d))
            gnode[row_of] = f[0][row_of].astype(np.float64) * d_out
            rot = [np.ones((len(keys), d)), f[2], f[3], gnode]
            ref_d1 = oracle.dhn_fwd(4, oi, keys, rot, sel=og)
            assert_close(g4[row_of[sel]], ref_d1, FP32_TOL, "C4 d f1 (sampled nodes)")
            assert_close(g4s[row_of[sel]], ref_d1, FP32_TOL, "C4 d f1, symmetric (sampled nodes)")
    np.testing.assert_array_equal(counts[2], deg)
    assert counts[3].sum() > 0 and counts[4].sum() > counts[3].sum()
