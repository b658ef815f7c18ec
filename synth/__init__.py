"""Seeded synthetic relation generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic: it only draws keys, edge/incidence
tuples and fp32 embeddings with the shapes, sizes and degree distributions of the paper's
workloads (recipe: SURVEY.md sec 8(d), restated in DESIGN.md "Input recipe").  Degrees,
normalisations, joins and aggregates are computed separately by oracle/ and by the CUDA
path.  Everything is numpy on the host; PCG64(seed), consumed in a fixed order.

Relations are returned as plain dicts of numpy arrays:
  node relation : {"key": int64[n], "x": float32[n, d]}
  edge relation : {"src": int64[m], "dst": int64[m]}     (keys, not rows)
"""
from __future__ import annotations

import numpy as np

BETA = 2.5


def rng_for(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def powerlaw_weights(rng, n, beta=BETA, cap_ratio=1000.0):
    """w = (1-u)^(-1/(beta-1)), truncated at cap_ratio * mean(w)."""
    w = (1.0 - rng.random(n)) ** (-1.0 / (beta - 1.0))
    return np.minimum(w, cap_ratio * w.mean())


def _search_right(cdf, q):
    """np.searchsorted(cdf, q, side="right") for a large batch of random queries, in
    cache-friendly steps (identical result): a bucket table gives a lower bound of every
    answer, then a few vectorised forward steps finish it (random probes of a multi-MB CDF
    are ~20x slower than this)."""
    n = len(cdf)
    if n < 4096 or len(q) < 65536:
        return np.searchsorted(cdf, q, side="right")
    nb = 1 << max(10, int(np.ceil(np.log2(n))) + 1)
    width = cdf[-1] / nb
    # lower bound: entries <= bucket start (b - 1 guards the rounding of q / width)
    table = np.searchsorted(cdf, np.arange(nb + 1) * width, side="right")
    b = np.clip((q / width).astype(np.int64) - 1, 0, nb)
    idx = table[b]
    act = np.nonzero((idx < n) & (cdf[np.minimum(idx, n - 1)] <= q))[0]
    while len(act):
        idx[act] += 1
        i = idx[act]
        act = act[(i < n) & (cdf[np.minimum(i, n - 1)] <= q[act])]
    return idx


def _sorted_unique(x):
    """np.unique(x) (sorted distinct values) via one in-place sort."""
    x = np.sort(x)
    if len(x) == 0:
        return x
    keep = np.empty(len(x), bool)
    keep[0] = True
    np.not_equal(x[1:], x[:-1], out=keep[1:])
    return x[keep]


def _draw(rng, cdf, k):
    return _search_right(cdf, rng.random(k) * cdf[-1]).clip(0, len(cdf) - 1)


def chung_lu(rng, w_s, w_t, m, same_set, undirected, block=None, mu_intra=0.0):
    """Exactly m distinct (s, t) id pairs with endpoint probability proportional to weight.

    same_set: reject self-loops.  undirected: canonicalise to (min, max) before dedup.
    block/mu_intra: degree-corrected SBM -- with prob mu_intra the second endpoint is drawn
    within the first endpoint's contiguous block of `block` ids.
    """
    n_s, n_t = len(w_s), len(w_t)
    cs, ct = np.cumsum(w_s), np.cumsum(w_t)
    have = np.zeros(0, np.int64)
    while len(have) < m:
        k = int((m - len(have)) * 1.3) + 1024
        s = _draw(rng, cs, k)
        t = _draw(rng, ct, k)
        if block is not None:
            intra = rng.random(k) < mu_intra
            b0 = (s[intra] // block) * block
            b1 = np.minimum(b0 + block, n_t)
            lo = np.where(b0 > 0, ct[np.maximum(b0 - 1, 0)], 0.0)
            hi = ct[b1 - 1]
            u = lo + rng.random(int(intra.sum())) * (hi - lo)
            t[intra] = _search_right(ct, u).clip(b0, b1 - 1)
        if same_set:
            keep = s != t
            s, t = s[keep], t[keep]
        if undirected:
            s, t = np.minimum(s, t), np.maximum(s, t)
        code = s.astype(np.int64) * n_t + t
        have = _sorted_unique(np.concatenate([have, code]))
    pick = np.sort(rng.choice(len(have), size=m, replace=False))
    code = have[pick]
    return code // n_t, code % n_t


def _normal_f32(rng, shape, std):
    return (rng.standard_normal(shape) * std).astype(np.float32)


def gcn_graph(seed, n_nodes, n_edge_tuples, d_in, undirected, cap_ratio, with_loops=True):
    """Citation-like graph for a GCN lifted query.

    Returns nodes {"key","x"} and the edge relation AEdge = Edge U {(v,v)} as key columns
    (the union rule adding self-loops, SURVEY sec 8c ambiguity #1), rows shuffled.
    """
    rng = rng_for(seed)
    w_out = powerlaw_weights(rng, n_nodes, cap_ratio=cap_ratio)
    w_in = w_out if undirected else powerlaw_weights(rng, n_nodes, cap_ratio=cap_ratio)
    m = n_edge_tuples // 2 if undirected else n_edge_tuples
    s, t = chung_lu(rng, w_out, w_in, m, same_set=True, undirected=undirected)
    if undirected:
        s, t = np.concatenate([s, t]), np.concatenate([t, s])
    perm = rng.permutation(len(s))
    s, t = s[perm], t[perm]
    key_of_id = rng.permutation(n_nodes).astype(np.int64)
    x = _normal_f32(rng, (n_nodes, d_in), 1.0 / np.sqrt(d_in))
    src, dst = key_of_id[s], key_of_id[t]
    if with_loops:
        # self-loops appended in node-row order, then the whole relation shuffled
        src = np.concatenate([src, key_of_id])
        dst = np.concatenate([dst, key_of_id])
        p2 = rng.permutation(len(src))
        src, dst = src[p2], dst[p2]
    return {"nodes": {"key": key_of_id, "x": x}, "edges": {"src": src, "dst": dst}, "rng": rng}


def cora_like(seed=42):
    """Config 1: 2,708 nodes, 10,556 directed tuples (5,278 undirected pairs), 1,433 features."""
    g = gcn_graph(seed, 2708, 10556, 1433, undirected=True, cap_ratio=60.0)
    rng = g.pop("rng")
    g["W"] = [_normal_f32(rng, (16, 1433), 1.0 / np.sqrt(1433)),
              _normal_f32(rng, (7, 16), 1.0 / np.sqrt(16))]
    g["d_out"] = _normal_f32(rng, (2708, 7), 1.0)
    g["dims"] = [1433, 16, 7]
    _gcn_extras(g, rng)
    return g


def _gcn_extras(g, rng):
    """Drawn after everything else (the earlier draws are unchanged): per-layer biases of the
    O7 epilogue ~ N(0, 0.1^2), class labels uniform over the last width, and a training mask of
    the first 5% of node rows (Cora's public split labels 140 of 2,708 nodes)."""
    dims = g["dims"]
    g["b"] = [_normal_f32(rng, (dims[l + 1],), 0.1) for l in range(len(dims) - 1)]
    n = len(g["nodes"]["key"])
    lab = rng.integers(0, dims[-1], n).astype(np.int64)
    lab[max(1, n // 20):] = -1
    g["labels"] = lab


def arxiv_like(seed=42, n_nodes=169343, n_edges=1166243, d=128, layers=3):
    """Config 2: ogbn-arxiv-shaped directed citation graph, 3 GCN layers 128 -> 128."""
    g = gcn_graph(seed, n_nodes, n_edges, d, undirected=False, cap_ratio=1500.0)
    rng = g.pop("rng")
    g["W"] = [_normal_f32(rng, (d, d), 1.0 / np.sqrt(d)) for _ in range(layers)]
    g["d_out"] = _normal_f32(rng, (n_nodes, d), 1.0)
    g["dims"] = [d] * (layers + 1)
    _gcn_extras(g, rng)
    return g


def hypergraph_like(seed=42, n_nodes=1_000_000, n_hyper=200_000, n_inc=5_000_000, d=128):
    """Config 4: incidence relation Inc(v, e) between nodes and hyperedges (sparse 63-bit keys)."""
    rng = rng_for(seed)
    w_v = powerlaw_weights(rng, n_nodes, cap_ratio=1000.0)
    w_e = powerlaw_weights(rng, n_hyper, cap_ratio=1000.0)
    v, e = chung_lu(rng, w_v, w_e, n_inc, same_set=False, undirected=False)
    # every hyperedge has >= 2 incidences: top up small ones with fresh nodes
    cnt = np.bincount(e, minlength=n_hyper)
    short = np.nonzero(cnt < 2)[0]
    if len(short):
        codes = set((v.astype(np.int64) * n_hyper + e).tolist()) if len(short) < 10000 else None
        add_v, add_e = [], []
        for h in short:
            need = 2 - cnt[h]
            while need > 0:
                cand = int(rng.integers(0, n_nodes))
                c = cand * n_hyper + int(h)
                if codes is not None and c in codes:
                    continue
                if codes is not None:
                    codes.add(c)
                add_v.append(cand); add_e.append(int(h)); need -= 1
        v = np.concatenate([v, np.array(add_v, np.int64)])
        e = np.concatenate([e, np.array(add_e, np.int64)])
    perm = rng.permutation(len(v))
    v, e = v[perm], e[perm]
    node_key = rng.permutation(n_nodes).astype(np.int64)
    hyper_key = np.unique(rng.integers(0, 2 ** 63 - 1, size=n_hyper + 1024, dtype=np.int64))
    hyper_key = rng.permutation(hyper_key)[:n_hyper]
    x = _normal_f32(rng, (n_nodes, d), 1.0 / np.sqrt(d))
    theta = _normal_f32(rng, (d, d), 1.0 / np.sqrt(d))
    d_out = _normal_f32(rng, (n_nodes, d), 1.0)
    # per-tuple hyperedge embeddings (HyGNN attention queries), drawn last
    hx = _normal_f32(rng, (n_hyper, d), 1.0 / np.sqrt(d))
    return {"nodes": {"key": node_key, "x": x}, "hyperedges": {"key": hyper_key},
            "inc": {"node": node_key[v], "hyper": hyper_key[e]}, "theta": theta, "d_out": d_out,
            "hx": hx}


MAG_NODES = {"paper": 736_389, "author": 1_134_649, "institution": 8_740, "field": 59_965}
MAG_EDGES = [("writes", "author", "paper", 7_145_660),
             ("cites", "paper", "paper", 5_416_271),
             ("has_topic", "paper", "field", 7_505_078),
             ("affiliated_with", "author", "institution", 1_043_998)]


def mag_like(seed=42, scale=1.0, d=128, heads=8):
    """Config 3: OGB-MAG-shaped heterogeneous schema (4 node relations, 4 edge relations)."""
    rng = rng_for(seed)
    n = {k: max(8, int(v * scale)) for k, v in MAG_NODES.items()}
    w = {k: powerlaw_weights(rng, n[k], cap_ratio=1000.0) for k in n}
    key = {k: rng.permutation(n[k]).astype(np.int64) + (i << 40) for i, k in enumerate(n)}
    rels = {}
    for name, a, b, m in MAG_EDGES:
        m = max(16, int(m * scale))
        wa = w[a]
        wb = powerlaw_weights(rng, n[b], cap_ratio=1000.0) if a == b else w[b]
        s, t = chung_lu(rng, wa, wb, m, same_set=(a == b), undirected=False)
        perm = rng.permutation(m)
        rels[name] = {"src_type": a, "dst_type": b,
                      "src": key[a][s[perm]], "dst": key[b][t[perm]]}
    h = {k: _normal_f32(rng, (n[k], d), 1.0 / np.sqrt(d)) for k in n}
    return {"n": n, "key": key, "h": h, "rels": rels, "d": d, "heads": heads, "rng": rng}


def products_like(seed=42, scale=1.0, d=32, block=1000, mu_intra=0.8):
    """Config 5: ogbn-products-shaped undirected DC-SBM graph (both directions stored)."""
    rng = rng_for(seed)
    n_nodes = max(64, int(2_449_029 * scale))
    m = max(64, int(61_859_140 * scale))
    w = powerlaw_weights(rng, n_nodes, cap_ratio=400.0)
    s, t = chung_lu(rng, w, w, m, same_set=True, undirected=True, block=block, mu_intra=mu_intra)
    s, t = np.concatenate([s, t]), np.concatenate([t, s])
    perm = rng.permutation(len(s))
    s, t = s[perm], t[perm]
    key_of_id = rng.permutation(n_nodes).astype(np.int64)
    h = _normal_f32(rng, (n_nodes, d), 1.0 / np.sqrt(d))
    return {"nodes": {"key": key_of_id, "x": h},
            "edges": {"src": key_of_id[s], "dst": key_of_id[t]}, "rng": rng}


def random_db(rng, n_s, n_t, n_e, key_space=None, dangling=0.2, d_s=4, d_e=1, d_t=4,
              neg_keys=True):
    """Tiny random relations for property tests: unique S/T keys, E may dangle / repeat."""
    ks = key_space or max(4 * (n_s + n_t + 1), 16)
    lo = -ks if neg_keys else 0
    s_key = rng.choice(np.arange(lo, ks, dtype=np.int64), size=n_s, replace=False)
    t_key = rng.choice(np.arange(lo, ks, dtype=np.int64), size=n_t, replace=False)

    def pick(keys, k):
        if len(keys) == 0:
            return rng.integers(lo, ks, size=k).astype(np.int64)
        out = keys[rng.integers(0, len(keys), size=k)]
        miss = rng.random(k) < dangling
        out[miss] = rng.integers(lo, ks, size=int(miss.sum()))
        return out.astype(np.int64)

    e_src = pick(s_key, n_e)
    e_dst = pick(t_key, n_e)
    return {"s_key": s_key, "t_key": t_key, "e_src": e_src, "e_dst": e_dst,
            "z_s": _normal_f32(rng, (n_s, d_s), 1.0),
            "z_e": _normal_f32(rng, (n_e, d_e), 1.0),
            "z_t": _normal_f32(rng, (n_t, d_t), 1.0)}


def rgcn_like(seed=42, n_nodes=8285, n_pairs=29043, n_rel=45, d=16):
    """AIFB-shaped multi-relational graph for R-GCN: power-law Chung-Lu
    pairs, each with a relation type (Zipf-like: a few types hold most edges), stored in both
    directions with the inverse as its own type (2 n_rel types, the R-GCN convention);
    dense node features ~ N(0, 1/d)."""
    rng = rng_for(seed)
    w = powerlaw_weights(rng, n_nodes, cap_ratio=200.0)
    s, t = chung_lu(rng, w, w, n_pairs, same_set=True, undirected=False)
    p = 1.0 / np.arange(1, n_rel + 1) ** 1.2
    rel = rng.choice(n_rel, size=n_pairs, p=p / p.sum())
    src = np.concatenate([s, t]); dst = np.concatenate([t, s])
    rel = np.concatenate([rel, rel + n_rel])
    perm = rng.permutation(len(src))
    key = rng.permutation(n_nodes).astype(np.int64)
    x = _normal_f32(rng, (n_nodes, d), 1.0 / np.sqrt(d))
    W = _normal_f32(rng, (2 * n_rel + 1, d, d), 1.0 / np.sqrt(d))
    d_out = _normal_f32(rng, (n_nodes, d), 1.0)
    return {"nodes": {"key": key, "x": x},
            "edges": {"src": key[src[perm]], "dst": key[dst[perm]], "rel": rel[perm].astype(np.int32)},
            "n_rel": 2 * n_rel, "W": W, "d_out": d_out}
