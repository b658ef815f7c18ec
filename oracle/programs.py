"""Oracle compositions of the paper's programs (TEST INFRASTRUCTURE, see oracle/__init__.py).

Only oracle functions are used; nothing here imports the product package.
"""
import numpy as np

import oracle
def gcn_fit(graph, labels, epochs, lr=0.01, weight_decay=5e-4):
    """fit: `epochs` full-batch steps of Loss = CrossEntropy(H^L, label)
    with Adam on every W and b; returns the per-epoch losses and the final parameters."""
    g = dict(graph)
    g["W"] = [np.asarray(w, np.float64).copy() for w in graph["W"]]
    g["b"] = [np.asarray(b, np.float64).copy() for b in graph["b"]]
    key = graph["nodes"]["key"]
    o1 = oracle.build_join_index(graph["edges"]["src"], graph["edges"]["dst"], key, key)
    lab = np.asarray(labels, np.int64)[o1["group_dst_row"]]     # logits rows: group order
    state = [(np.zeros_like(p), np.zeros_like(p)) for p in g["W"] + g["b"]]
    losses = []
    for t in range(1, epochs + 1):
        ex = {}
        g["d_out"] = None
        H, _, _ = gcn_step(g, out=ex, forward_only=True)
        loss, dl = oracle.softmax_xent(H[-1], lab)
        losses.append(loss)
        g["d_out"] = dl
        ex = {}
        _, dW, _ = gcn_step(g, out=ex)
        grads = dW + ex["db"]
        for p, gr, (m, v) in zip(g["W"] + g["b"], grads, state):
            oracle.adam(p.reshape(-1) if p.ndim == 1 else p, np.asarray(gr).reshape(p.shape),
                        m, v, lr, t, wd=weight_decay)
    return losses, g["W"], g["b"]


def gcn_step(graph, layers=None, out=None, forward_only=False):
    """O7: fp64 forward + backward of the L-layer GCN program (reading #1).

    Same rules as paper_2605_24207_b200.programs.GCNProgram, evaluated with the plain oracle
    functions: AEdge join index, w = deg^-1/2 deg^-1/2, A^l = sum_s w (H^l W_l^T)[s], and when
    the graph carries biases "b" the PyG GCNConv epilogue H^{l+1} = ReLU(A^l + b_l) on hidden
    layers, A^L + b_L on the last; else H^{l+1} = A^l.
    `layers` limits the evaluation to the first layers (bounded CPU-baseline samples).
    `out` (a dict) receives the bias gradients "db" and the activations "H"."""
    nodes, edges = graph["nodes"], graph["edges"]
    key = nodes["key"]
    L = len(graph["W"]) if layers is None else layers
    o1 = oracle.build_join_index(edges["src"], edges["dst"], key, key)
    w1 = oracle.gcn_norm(o1, len(key))
    if L > 1:
        o2 = oracle.build_join_index(edges["src"], edges["dst"], o1["group_key"], o1["group_key"])
        w2 = oracle.gcn_norm(o2, len(o1["group_key"]))
    bias = graph.get("b")
    act = lambda l: "relu" if l < len(graph["W"]) - 1 else "none"
    H = [np.asarray(nodes["x"], np.float64)]
    Z, A = [], []
    for l in range(L):
        Z.append(oracle.project(H[l], graph["W"][l]))
        o, w = (o1, w1) if l == 0 else (o2, w2)
        A.append(oracle.lja_fwd(o, "src", "sum", src=Z[l], edge=w, edge_mode=1)[0])
        H.append(A[l] if bias is None else oracle.epilogue_fwd(A[l], bias[l], act(l)))
    if forward_only:
        return H, None, None
    G = o1["n_groups"]
    dY = np.asarray(graph["d_out"][:G, : H[-1].shape[1]], np.float64)
    dW, dH0, db = [None] * L, None, [None] * L
    for l in reversed(range(L)):
        o, w = (o1, w1) if l == 0 else (o2, w2)
        if bias is not None:
            dY, db[l], _, _ = oracle.epilogue_bwd(dY, A[l], bias[l], act(l))
        dZ = oracle.lja_bwd(o, dY, "src", "sum", src=Z[l], edge=w, edge_mode=1, want=("src",))["src"]
        dX, dW[l], _ = oracle.project_bwd(H[l], graph["W"][l], dZ, want_db=False)
        dY = dX
    if out is not None:
        out.update(db=db, H=H)
    return H, dW, dY


def hypergraph_step(hg):
    """O8: two-hop node -> hyperedge -> node (hop 1 SUM by hyperedge, hop 2 MEAN by node),
    after the projection Z = X Theta^T; backward with dOut = hg['d_out'][:G2]."""
    nk, hk = hg["nodes"]["key"], hg["hyperedges"]["key"]
    iv, ih = hg["inc"]["node"], hg["inc"]["hyper"]
    o1 = oracle.build_join_index(iv, ih, nk, hk)
    o2 = oracle.build_join_index(ih, iv, o1["group_key"], nk)
    X = np.asarray(hg["nodes"]["x"], np.float64)
    Z = oracle.project(X, hg["theta"])
    Eh = oracle.lja_fwd(o1, "src", "sum", src=Z)[0]
    Xo = oracle.lja_fwd(o2, "src", "mean", src=Eh)[0]
    dXo = np.asarray(hg["d_out"][: o2["n_groups"]], np.float64)
    dEh = oracle.lja_bwd(o2, dXo, "src", "mean", src=Eh, want=("src",))["src"]
    dZ = oracle.lja_bwd(o1, dEh, "src", "sum", src=Z, want=("src",))["src"]
    dX, dTheta, _ = oracle.project_bwd(X, hg["theta"], dZ, want_db=False)
    return {"Xo": Xo, "dTheta": dTheta, "dX": dX, "o1": o1, "o2": o2}


def hgt_relation(H_src, H_dst, Wk, Wm, Wq, src_keys, dst_keys, e_src, e_dst, heads, d_out_dense):
    """One relation phi of the HGT layer (Fig. 4): K' = H_s Wk^T (scale folded),
    M' = H_s Wm^T, Q = H_t Wq^T, O = per-target per-head softmax-weighted sum.  Returns the
    compact oracle outputs, the key-sorted dense placement and the gradients."""
    K = oracle.project(H_src, Wk)
    M = oracle.project(H_src, Wm)
    Q = oracle.project(H_dst, Wq)
    o = oracle.build_join_index(e_src, e_dst, src_keys, dst_keys)
    out, lse = oracle.lja_fwd(o, agg="softmax", src=M, src_key=K, dst=Q, heads=heads, scale=1.0)
    # dense rows in T-key order: rank of every T key
    order = np.argsort(dst_keys, kind="stable")
    rank = np.empty(len(dst_keys), np.int64)
    rank[order] = np.arange(len(dst_keys))
    dense_rows = rank[o["group_dst_row"]]
    dO = np.asarray(d_out_dense, np.float64)[dense_rows]
    g = oracle.lja_bwd(o, dO, agg="softmax", src=M, src_key=K, dst=Q, heads=heads, scale=1.0)
    return {"index": o, "out": out, "lse": lse, "dense_rows": dense_rows,
            "dK": g["src_key"], "dM": g["src"], "dQ": g["dst"], "K": K, "M": M, "Q": Q}


def dhn_step(g, W, d_out_dense, ks=(2, 3, 4)):
    """O9: DHN layer: f_{k,i} = h W_{k,i}^T (positions stacked in W, C2 then
    C3 then C4), C_k closed-walk aggregates, out = C2 (+) C3 (+) C4 placed densely in node-key
    order (roots without out-edges: 0); backward with d_out_dense [n, 3d]."""
    keys = np.asarray(g["nodes"]["key"])
    h = np.asarray(g["nodes"]["x"], np.float64)
    n, d = h.shape
    adj = oracle.build_join_index(g["edges"]["src"], g["edges"]["dst"], keys, keys,
                                  within_by_src_key=True)
    Y = oracle.project(h, W)
    rank = np.argsort(np.argsort(keys, kind="stable"), kind="stable")
    rows = rank[adj["group_dst_row"]]              # dense position of every oracle group
    out = np.zeros((n, len(ks) * d))
    dY = np.zeros_like(Y)
    p = 0
    for j, k in enumerate(ks):
        f = [Y[:, (p + i) * d:(p + i + 1) * d] for i in range(k)]
        out[rows, j * d:(j + 1) * d] = oracle.dhn_fwd(k, adj, keys, f)
        dO = np.asarray(d_out_dense, np.float64)[rows, j * d:(j + 1) * d]
        grads = oracle.dhn_bwd(k, adj, keys, f, dO)
        for i in range(k):
            dY[:, (p + i) * d:(p + i + 1) * d] = grads[i]
        p += k
    dH, dW, _ = oracle.project_bwd(h, W, dY, want_db=False)
    return {"out": out, "dY": dY, "dW": dW, "dH": dH}


def hgt_joint_step(mag, par, heads):
    """Joint-softmax HGT layer (the original HGT's attention, normalised over the sources of
    every relation into a target type at once; SURVEY sec 8c reading 3): per target type one
    softmax join-aggregate over the union of the relations into it, the source relation being
    the stack of every relation's (K', M') rows keyed by (relation, source key)."""
    d = mag["d"]
    col, W = par["col"], par["W"]
    blk = lambda t, kind, key: W[t][col[(kind, key)][1] * d:(col[(kind, key)][1] + 1) * d]
    out, grads = {}, {"dWk": {}, "dWm": {}, "dWq": {}, "dH": {}}
    add = lambda t, x: grads["dH"].__setitem__(t, grads["dH"].get(t, 0) + x)
    for t in par["targets"]:
        names = [n for n, r in mag["rels"].items() if r["dst_type"] == t]
        K, M, skeys, es, ed = [], [], [], [], []
        for j, name in enumerate(names):
            r = mag["rels"][name]
            s = r["src_type"]
            K.append(oracle.project(mag["h"][s], blk(s, "k", name)))
            M.append(oracle.project(mag["h"][s], blk(s, "m", name)))
            skeys.append((np.int64(j) << np.int64(56)) | np.asarray(mag["key"][s], np.int64))
            es.append((np.int64(j) << np.int64(56)) | np.asarray(r["src"], np.int64))
            ed.append(np.asarray(r["dst"], np.int64))
        K, M = np.concatenate(K), np.concatenate(M)
        Q = oracle.project(mag["h"][t], blk(t, "q", t))
        o = oracle.build_join_index(np.concatenate(es), np.concatenate(ed), np.concatenate(skeys),
                                    mag["key"][t])
        o_out, _ = oracle.lja_fwd(o, agg="softmax", src=M, src_key=K, dst=Q, heads=heads, scale=1.0)
        rank = np.argsort(np.argsort(mag["key"][t], kind="stable"), kind="stable")
        rows = rank[o["group_dst_row"]]
        dense = np.zeros((mag["n"][t], d))
        dense[rows] = o_out
        out[t] = dense
        g = oracle.lja_bwd(o, np.asarray(par["d_out"][t], np.float64)[rows], agg="softmax", src=M,
                           src_key=K, dst=Q, heads=heads, scale=1.0)
        dX, grads["dWq"][t], _ = oracle.project_bwd(mag["h"][t], blk(t, "q", t), g["dst"], want_db=False)
        add(t, dX)
        off = 0
        for name in names:
            s = mag["rels"][name]["src_type"]
            n = mag["n"][s]
            dXk, grads["dWk"][name], _ = oracle.project_bwd(mag["h"][s], blk(s, "k", name),
                                                            g["src_key"][off:off + n], want_db=False)
            dXm, grads["dWm"][name], _ = oracle.project_bwd(mag["h"][s], blk(s, "m", name),
                                                            g["src"][off:off + n], want_db=False)
            add(s, dXk + dXm)
            off += n
    return out, grads


def hygnn_attention_step(hg, P, heads):
    """HyGNN double attention: node-level softmax attention grouped by hyperedge,
    then hyperedge-level grouped by node; P = the six maps (scale 1/sqrt(d/h) on the keys)."""
    d = hg["nodes"]["x"].shape[1]
    scale = 1.0 / np.sqrt(d / heads)
    nk, hk = hg["nodes"]["key"], hg["hyperedges"]["key"]
    iv, ih = hg["inc"]["node"], hg["inc"]["hyper"]
    X, E0 = np.asarray(hg["nodes"]["x"], np.float64), np.asarray(hg["hx"], np.float64)
    rank = lambda k: np.argsort(np.argsort(k, kind="stable"), kind="stable")
    o1 = oracle.build_join_index(iv, ih, nk, hk)
    K1, V1 = oracle.project(X, P["k1"] * scale), oracle.project(X, P["v1"])
    Q1 = oracle.project(E0, P["q1"])
    e_out, _ = oracle.lja_fwd(o1, agg="softmax", src=V1, src_key=K1, dst=Q1, heads=heads, scale=1.0)
    r1 = rank(hk)[o1["group_dst_row"]]
    Eh = np.zeros((len(hk), d)); Eh[r1] = e_out                 # dense, hyperedge-key order
    hks = np.sort(hk)
    o2 = oracle.build_join_index(ih, iv, hks, nk)
    K2, V2 = oracle.project(Eh, P["k2"] * scale), oracle.project(Eh, P["v2"])
    Q2 = oracle.project(X, P["q2"])
    x_out, _ = oracle.lja_fwd(o2, agg="softmax", src=V2, src_key=K2, dst=Q2, heads=heads, scale=1.0)
    r2 = rank(nk)[o2["group_dst_row"]]
    Xo = np.zeros((len(nk), d)); Xo[r2] = x_out
    dXo = np.asarray(hg["d_out"][: len(nk)], np.float64)
    g2 = oracle.lja_bwd(o2, dXo[r2], agg="softmax", src=V2, src_key=K2, dst=Q2, heads=heads, scale=1.0)
    dXq, dWq2, _ = oracle.project_bwd(X, P["q2"], g2["dst"], want_db=False)
    dEk, dWk2, _ = oracle.project_bwd(Eh, P["k2"] * scale, g2["src_key"], want_db=False)
    dEv, dWv2, _ = oracle.project_bwd(Eh, P["v2"], g2["src"], want_db=False)
    dEh = dEk + dEv
    g1 = oracle.lja_bwd(o1, dEh[r1], agg="softmax", src=V1, src_key=K1, dst=Q1, heads=heads, scale=1.0)
    dE0, dWq1, _ = oracle.project_bwd(E0, P["q1"], g1["dst"], want_db=False)
    dXk, dWk1, _ = oracle.project_bwd(X, P["k1"] * scale, g1["src_key"], want_db=False)
    dXv, dWv1, _ = oracle.project_bwd(X, P["v1"], g1["src"], want_db=False)
    return {"Eh": Eh, "Xo": Xo, "dX": dXq + dXk + dXv, "dE0": dE0, "dWk1": dWk1, "dWv1": dWv1,
            "dWq1": dWq1, "dWk2": dWk2, "dWv2": dWv2, "dWq2": dWq2}
