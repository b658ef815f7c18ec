"""Oracle compositions of the paper's programs (TEST INFRASTRUCTURE, see oracle/__init__.py).

Only oracle functions are used; nothing here imports the product package.
"""
import numpy as np

import oracle
def gcn_step(graph, layers=None):
    """O7: fp64 forward + backward of the L-layer GCN program (reading #1).

    Same rules as paper_2605_24207_b200.programs.GCNProgram, evaluated with the plain oracle
    functions: AEdge join index, w = deg^-1/2 deg^-1/2, H^{l+1} = sum_s w (H^l W_l^T)[s].
    `layers` limits the evaluation to the first layers (bounded CPU-baseline samples).
    """
    nodes, edges = graph["nodes"], graph["edges"]
    key = nodes["key"]
    L = len(graph["W"]) if layers is None else layers
    o1 = oracle.build_join_index(edges["src"], edges["dst"], key, key)
    w1 = oracle.gcn_norm(o1, len(key))
    if L > 1:
        o2 = oracle.build_join_index(edges["src"], edges["dst"], o1["group_key"], o1["group_key"])
        w2 = oracle.gcn_norm(o2, len(o1["group_key"]))
    H = [np.asarray(nodes["x"], np.float64)]
    Z = []
    for l in range(L):
        Z.append(oracle.project(H[l], graph["W"][l]))
        o, w = (o1, w1) if l == 0 else (o2, w2)
        H.append(oracle.lja_fwd(o, "src", "sum", src=Z[l], edge=w, edge_mode=1)[0])
    G = o1["n_groups"]
    dY = np.asarray(graph["d_out"][:G, : H[-1].shape[1]], np.float64)
    dW, dH0 = [None] * L, None
    for l in reversed(range(L)):
        o, w = (o1, w1) if l == 0 else (o2, w2)
        dZ = oracle.lja_bwd(o, dY, "src", "sum", src=Z[l], edge=w, edge_mode=1, want=("src",))["src"]
        dX, dW[l], _ = oracle.project_bwd(H[l], graph["W"][l], dZ, want_db=False)
        dY = dX
    return H, dW, dY
