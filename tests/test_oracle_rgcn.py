"""Pins for the R-GCN oracle (per-join-row W_rel x_s with no pushdown; PAPER.md:444 T_tau,
R-GCN PAPER.md:890, :897) -- CPU only: the dense matrix form of R-GCN
out = X W0^T + sum_r D_r^-1 A_r X W_r^T on small graphs, and finite differences of the
backward."""
import numpy as np

import synth


def small(seed, n=40, m=300, R=3, d=4, d_out=5):
    rng = np.random.default_rng(seed)
    keys = rng.permutation(n).astype(np.int64) * 5 + 2
    s, t = rng.integers(0, n, m), rng.integers(0, n, m)
    rel = rng.integers(0, R, m).astype(np.int32)
    x = rng.standard_normal((n, d))
    W = rng.standard_normal((R + 1, d_out, d))
    return keys, keys[s], keys[t], s, t, rel, x, W


def test_rgcn_dense_form(ora):
    for seed in range(5):
        keys, es, et, s, t, rel, x, W = small(seed)
        n, R = len(keys), W.shape[0] - 1
        idx = ora.build_join_index(es, et, keys, keys)
        out = ora.rgcn_fwd(idx, rel, x, W)
        ref = x @ W[0].T
        for r in range(R):
            A = np.zeros((n, n))
            np.add.at(A, (t[rel == r], s[rel == r]), 1.0)
            deg = A.sum(1, keepdims=True)
            ref += np.divide(A, deg, out=np.zeros_like(A), where=deg > 0) @ x @ W[r + 1].T
        rows = idx["group_dst_row"]
        np.testing.assert_allclose(out, ref[rows], rtol=1e-12, atol=1e-12)


def test_rgcn_bwd_fd(ora):
    keys, es, et, s, t, rel, x, W = small(7, n=15, m=60)
    idx = ora.build_join_index(es, et, keys, keys)
    rng = np.random.default_rng(1)
    dO = rng.standard_normal((idx["n_groups"], W.shape[1]))
    dx, dW = ora.rgcn_bwd(idx, rel, x, W, dO)
    f = lambda xx, WW: float(np.sum(ora.rgcn_fwd(idx, rel, xx, WW) * dO))
    eps = 1e-6
    for (i, j) in [(0, 0), (3, 2), (14, 3)]:
        xp, xm = x.copy(), x.copy()
        xp[i, j] += eps; xm[i, j] -= eps
        assert abs((f(xp, W) - f(xm, W)) / (2 * eps) - dx[i, j]) < 1e-6
    for (r, i, j) in [(0, 1, 2), (1, 0, 0), (3, 4, 3)]:
        Wp, Wm = W.copy(), W.copy()
        Wp[r, i, j] += eps; Wm[r, i, j] -= eps
        assert abs((f(x, Wp) - f(x, Wm)) / (2 * eps) - dW[r, i, j]) < 1e-6


def test_rgcn_generator_shape():
    g = synth.rgcn_like(3, n_nodes=500, n_pairs=2000, n_rel=5, d=8)
    assert g["n_rel"] == 10 and g["W"].shape == (11, 8, 8)
    assert g["edges"]["rel"].max() == 9 and len(g["edges"]["src"]) == 4000
