"""Pins for the oracle's forward lifted join-aggregate (O2) -- CPU only.

Pinned against: the paper's worked examples (tests/golden/*.json, cited there), the GCN
closed form D^-1/2 (A+I) D^-1/2 X (textbook GCN, which the paper matches "by construction",
PAPER.md:865, :900), the hypergraph closed form D_v^-1 H H^T X, mass conservation,
one-shot MEAN and group sizes with all-ones d=1 embeddings.
"""
import json
import os

import numpy as np
import pytest

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_projected_union_worked_example(ora):
    g = load("projected_union_k1.json")
    L = g["letters"]
    x = [L[r[0]] for r in g["R"]]
    y = [L[r[1]] for r in g["R"]]
    z = np.array([r[2] for r in g["R"]])
    idx = ora.build_join_index(y, x)                 # E = R, no S/T, group by x
    out, _ = ora.lja_fwd(idx, "mul", "sum", edge=z)  # the only operand is R's own embedding
    got = {k: out[list(idx["group_key"]).index(v)].tolist() for k, v in L.items()
           if v in idx["group_key"]}
    assert got == g["expected"]


def test_join_worked_example_concat(ora):
    g = load("join_concat.json")
    L = g["letters"]
    # S = R1 keyed by its y value (unique here), E = R2(y, w), one output row per E row
    s_key = [L[r[1]] for r in g["R1"]]
    z1 = np.array([r[2] for r in g["R1"]])
    e_src = [L[r[0]] for r in g["R2"]]
    e_dst = list(range(len(g["R2"])))
    z2 = np.array([r[2] for r in g["R2"]])
    idx = ora.build_join_index(e_src, e_dst, s_key=s_key)
    out, _ = ora.lja_fwd(idx, "concat", "sum", src=z1, edge=z2)
    assert out.tolist() == [r[3] for r in g["expected"]]
    # content: (x, y, w) of every output row
    rows = [(g["R1"][idx["src_row"][p]][0], g["R2"][idx["edge_row"][p]][0], g["R2"][idx["edge_row"][p]][1])
            for p in range(idx["n_join_rows"])]
    assert rows == [tuple(r[:3]) for r in g["expected"]]


def gcn_dense(n, edges, X):
    A = np.zeros((n, n))
    for s, t in edges:
        A[t, s] += 1.0            # message s -> t
    A += np.eye(n)
    deg = A.sum(1)
    Dm = np.diag(deg ** -0.5)
    return Dm @ A @ Dm @ X


@pytest.mark.parametrize("seed", range(20))
def test_gcn_closed_form(ora, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 40))
    m = int(rng.integers(0, 3 * n))
    pairs = set()
    for _ in range(m):
        s, t = (int(v) for v in rng.integers(0, n, 2))
        if s != t:
            pairs.add((s, t))
    pairs = sorted(pairs)
    keys = rng.permutation(n).astype(np.int64) * 7 - 50      # key of node row i
    X = rng.standard_normal((n, 5))
    e_src = [keys[s] for s, _ in pairs] + list(keys)
    e_dst = [keys[t] for _, t in pairs] + list(keys)
    perm = rng.permutation(len(e_src))
    e_src, e_dst = np.array(e_src)[perm], np.array(e_dst)[perm]
    idx = ora.build_join_index(e_src, e_dst, s_key=keys, t_key=keys)
    w = ora.gcn_norm(idx, n)
    out, _ = ora.lja_fwd(idx, "src", "sum", src=X, edge=w, edge_mode=1)
    ref = gcn_dense(n, pairs, X)
    np.testing.assert_allclose(out, ref[idx["group_dst_row"]], rtol=1e-12, atol=1e-12)


def test_gcn_path_graph_fixture(ora):
    """path 10-20-30-40 stored in row order [30,10,40,20]; canonical index values."""
    keys = np.array([30, 10, 40, 20])
    e = [(20, 10), (10, 20), (30, 20), (20, 30), (40, 30), (30, 40), (30, 30), (10, 10), (40, 40), (20, 20)]
    idx = ora.build_join_index([s for s, _ in e], [t for _, t in e], s_key=keys, t_key=keys)
    # expected values derived by hand from the O1 definition
    assert idx["group_key"].tolist() == [10, 20, 30, 40]
    assert idx["group_ptr"].tolist() == [0, 2, 5, 8, 10]
    assert idx["src_row"].tolist() == [3, 1, 1, 0, 3, 3, 2, 0, 0, 2]
    assert idx["edge_row"].tolist() == [0, 7, 1, 2, 9, 3, 4, 6, 5, 8]
    assert idx["group_dst_row"].tolist() == [1, 3, 0, 2]
    assert idx["src_ptr"].tolist() == [0, 3, 5, 7, 10]
    assert idx["src_pos"].tolist() == [3, 7, 8, 1, 2, 6, 9, 0, 4, 5]
    X = np.array([[1, 1], [1, 0], [2, -1], [0, 1]], float)   # rows for keys 30,10,40,20
    w = ora.gcn_norm(idx, 4)
    out, _ = ora.lja_fwd(idx, "src", "sum", src=X, edge=w, edge_mode=1)
    ref = gcn_dense(4, [(3, 1), (1, 3), (0, 3), (3, 0), (2, 0), (0, 2)], X)
    np.testing.assert_allclose(out, ref[[1, 3, 0, 2]], rtol=1e-13)


@pytest.mark.parametrize("combine", ["src", "mul", "add", "concat"])
def test_mass_conservation(ora, combine):
    """sum_g out[g] = sum over join rows of c(.)  (scatter-sum then sum)."""
    rng = np.random.default_rng(11)
    db = synth.random_db(rng, 25, 15, 300, d_s=3, d_e=1 if combine == "src" else 3, d_t=3)
    idx = ora.build_join_index(db["e_src"], db["e_dst"], db["s_key"], db["t_key"])
    kw = dict(src=db["z_s"], edge=db["z_e"])
    if combine != "src":
        kw["dst"] = db["z_t"]
    out, _ = ora.lja_fwd(idx, combine, "sum", **kw)
    zs, ze, zt = (np.asarray(db[k], float) for k in ("z_s", "z_e", "z_t"))
    tot = 0.0
    for g in range(idx["n_groups"]):
        for p in range(idx["group_ptr"][g], idx["group_ptr"][g + 1]):
            a, b, c = zs[idx["src_row"][p]], ze[idx["edge_row"][p]], zt[idx["group_dst_row"][g]]
            tot = tot + {"src": lambda: b[0] * a, "mul": lambda: a * b * c,
                         "add": lambda: a + b + c, "concat": lambda: np.concatenate([a, b, c])}[combine]()
    np.testing.assert_allclose(out.sum(0), tot, rtol=1e-12, atol=1e-12)


def test_all_ones_sum_is_group_size(ora):
    rng = np.random.default_rng(5)
    db = synth.random_db(rng, 40, 30, 500)
    idx = ora.build_join_index(db["e_src"], db["e_dst"], db["s_key"], db["t_key"])
    out, _ = ora.lja_fwd(idx, "src", "sum", src=np.ones((40, 1)))
    assert out[:, 0].tolist() == np.diff(idx["group_ptr"]).astype(float).tolist()


def test_mean_is_one_shot(ora):
    """Union of two relations then MEAN over the stacked multiset, not mean-of-means."""
    # R1 contributes {1, 2} to key 7, R2 contributes {6} to key 7: mean = 3, mean-of-means = 3.75
    z = np.array([[1.0], [2.0], [6.0]])
    idx = ora.build_join_index([0, 1, 2], [7, 7, 7], s_key=[0, 1, 2])
    out, _ = ora.lja_fwd(idx, "src", "mean", src=z)
    assert out.tolist() == [[3.0]]


def test_hypergraph_two_hop_closed_form(ora):
    """SURVEY F4 and the closed form D_v^-1 H H^T X (hop 1 SUM by hyperedge, hop 2 MEAN by node)."""
    rng = np.random.default_rng(2)
    for trial in range(10):
        nv, ne = int(rng.integers(2, 20)), int(rng.integers(1, 10))
        inc = sorted({(int(rng.integers(0, nv)), int(rng.integers(0, ne))) for _ in range(3 * nv)})
        vkey = rng.permutation(nv).astype(np.int64) + 100
        hkey = rng.choice(2 ** 62, ne, replace=False).astype(np.int64)
        X = rng.standard_normal((nv, 3))
        H = np.zeros((nv, ne))
        for v, e in inc:
            H[v, e] = 1
        i1 = ora.build_join_index([vkey[v] for v, _ in inc], [hkey[e] for _, e in inc], vkey, hkey)
        Eh, _ = ora.lja_fwd(i1, "src", "sum", src=X)                 # [G1] rows = hyperedges present
        Eh_full = np.zeros((ne, 3)); Eh_full[i1["group_dst_row"]] = Eh
        i2 = ora.build_join_index([hkey[e] for _, e in inc], [vkey[v] for v, _ in inc], hkey, vkey)
        Xn, _ = ora.lja_fwd(i2, "src", "mean", src=Eh_full)
        deg = H.sum(1)
        ref = (H @ (H.T @ X))[i2["group_dst_row"]] / deg[i2["group_dst_row"], None]
        np.testing.assert_allclose(Xn, ref, rtol=1e-12, atol=1e-12)
    # F4: e1={v1,v2}, e2={v2,v3}, X=[1,2,4]
    i1 = ora.build_join_index([1, 2, 2, 3], [10, 10, 20, 20], [1, 2, 3], [10, 20])
    Eh, _ = ora.lja_fwd(i1, "src", "sum", src=np.array([[1.0], [2.0], [4.0]]))
    assert Eh.ravel().tolist() == [3.0, 6.0]
    i2 = ora.build_join_index([10, 10, 20, 20], [1, 2, 2, 3], [10, 20], [1, 2, 3])
    assert ora.lja_fwd(i2, "src", "mean", src=Eh)[0].ravel().tolist() == [3.0, 4.5, 6.0]
    assert ora.lja_fwd(i2, "src", "sum", src=Eh)[0].ravel().tolist() == [3.0, 9.0, 6.0]


def test_intro_attention_example(ora):
    """Attention(p; sum(a*v)) with a = q*k, via MUL combine.

    Attention(p) = sum_t q_p * k_t * v_t; k*v is the pushed-down per-t product relation.
    Numbers: q_p1=[1,2], q_p2=[0.5,-1], k_t1=[3,1], k_t2=[-1,2], v_t1=[1,1], v_t2=[2,0],
    Treat={(p1,t1),(p1,t2),(p2,t2)}.  By hand: p1 -> [1,2]*([3,1]+[-2,0]) = [1,2];
    p2 -> [0.5,-1]*[-2,0] = [-1,0].
    """
    q = np.array([[1, 2], [0.5, -1]]); k = np.array([[3, 1], [-1, 2]]); v = np.array([[1, 1], [2, 0]])
    idx = ora.build_join_index([1, 2, 2], [101, 101, 102], s_key=[1, 2], t_key=[101, 102])
    out, _ = ora.lja_fwd(idx, "mul", "sum", src=k * v, dst=q)
    assert out.tolist() == [[1.0, 2.0], [-1.0, 0.0]]
    # the same without pushdown: MUL of an edge operand (score a per row) and the value
    idx2 = ora.build_join_index([1, 2, 2], [101, 101, 102], s_key=[1, 2], t_key=[101, 102])
    a = np.array([q[0] * k[0], q[0] * k[1], q[1] * k[1]])     # Score(p,t; q*k), edge-row order
    out2, _ = ora.lja_fwd(idx2, "mul", "sum", src=v, edge=a)
    assert out2.tolist() == out.tolist()


def test_sampled_groups_equal_full(ora):
    rng = np.random.default_rng(9)
    db = synth.random_db(rng, 50, 40, 400, d_s=6)
    idx = ora.build_join_index(db["e_src"], db["e_dst"], db["s_key"], db["t_key"])
    full, _ = ora.lja_fwd(idx, "src", "mean", src=db["z_s"], edge=db["z_e"])
    sel = np.array([idx["n_groups"] - 1, 0, 3])
    part, _ = ora.lja_fwd(idx, "src", "mean", src=db["z_s"], edge=db["z_e"], sel=sel)
    np.testing.assert_array_equal(part, full[sel])
