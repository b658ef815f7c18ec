"""Pins for grouped softmax and softmax-weighted aggregation (O3) -- CPU only.

HGT attention (Fig. 4): ATT = softmax_t(K W_ATT Q^T mu / sqrt(d/h)), the
softmax normalising over the sources s of each target t (SURVEY sec 8c reading #3), then
out[t] = sum_s ATT * MSG.  Pinned against a dense masked softmax in numpy, SPEC.md:133
(singleton group -> 1.0), SPEC.md:572 (groups sum to 1 within 1e-9) and shift invariance.
"""
import numpy as np
import pytest


def dense_attention(K, M, Q, edges, n_t, heads, scale):
    n_s = K.shape[0]
    dk, dv = K.shape[1] // heads, M.shape[1] // heads
    mask = np.zeros((n_t, n_s), bool)
    for s, t in edges:
        mask[t, s] = True
    out = np.zeros((n_t, M.shape[1]))
    lse = np.zeros((n_t, heads))
    for h in range(heads):
        S = scale * Q[:, h * dk:(h + 1) * dk] @ K[:, h * dk:(h + 1) * dk].T
        S = np.where(mask, S, -np.inf)
        mx = S.max(1, keepdims=True)
        E = np.exp(S - mx)
        A = E / E.sum(1, keepdims=True)
        out[:, h * dv:(h + 1) * dv] = A @ M[:, h * dv:(h + 1) * dv]
        lse[:, h] = (mx + np.log(E.sum(1, keepdims=True)))[:, 0]
    return out, lse


def test_hgt_toy(ora):
    """SURVEY F2 / SPEC.md:572 shape: 3 sources, 2 targets, h=1, d=2, scale 1."""
    K = np.array([[1, 0], [0, 1], [1, 1]], float)
    M = np.array([[1, 2], [3, 4], [5, 6]], float)
    Q = np.array([[1, 0], [0, 2]], float)
    edges = [(0, 0), (1, 0), (2, 0), (1, 1), (2, 1)]
    idx = ora.build_join_index([s for s, _ in edges], [t for _, t in edges], [0, 1, 2], [0, 1])
    out, lse = ora.lja_fwd(idx, agg="softmax", src=M, src_key=K, dst=Q, heads=1, scale=1.0)
    ref, rlse = dense_attention(K, M, Q, edges, 2, 1, 1.0)
    np.testing.assert_allclose(out, ref, rtol=1e-14)
    np.testing.assert_allclose(lse, rlse, rtol=1e-14)
    assert abs(lse[1, 0] - (2 + np.log(2))) < 1e-14          # two equal scores 2


@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("heads", [1, 2, 4])
def test_attention_matches_dense(ora, seed, heads):
    rng = np.random.default_rng(seed)
    n_s, n_t = int(rng.integers(1, 20)), int(rng.integers(1, 12))
    edges = sorted({(int(rng.integers(0, n_s)), int(rng.integers(0, n_t))) for _ in range(40)})
    d = 4 * heads
    K, M, Q = (rng.standard_normal((n, d)) for n in (n_s, n_s, n_t))
    s_key = rng.permutation(n_s) * 3
    t_key = rng.permutation(n_t) * 5 + 1
    idx = ora.build_join_index([s_key[s] for s, _ in edges], [t_key[t] for _, t in edges], s_key, t_key)
    out, lse = ora.lja_fwd(idx, agg="softmax", src=M, src_key=K, dst=Q, heads=heads, scale=0.5)
    ref, rlse = dense_attention(K, M, Q, edges, n_t, heads, 0.5)
    rows = idx["group_dst_row"]
    np.testing.assert_allclose(out, ref[rows], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(lse, rlse[rows], rtol=1e-12, atol=1e-12)


def test_group_softmax_properties(ora):
    rng = np.random.default_rng(1)
    sizes = [1, 3, 1, 7, 2]
    gp = np.concatenate([[0], np.cumsum(sizes)])
    idx = {"group_ptr": gp, "n_groups": len(sizes)}
    s = rng.standard_normal((gp[-1], 2)) * 10
    p = ora.group_softmax(idx, s, 2)
    for g in range(len(sizes)):
        blk = p[gp[g]:gp[g + 1]]
        np.testing.assert_allclose(blk.sum(0), 1.0, atol=1e-9)
        assert np.all(blk > 0)
        if sizes[g] == 1:
            assert blk.tolist() == [[1.0, 1.0]]
    shift = np.repeat(rng.standard_normal((len(sizes), 2)) * 100, sizes, axis=0)
    np.testing.assert_allclose(ora.group_softmax(idx, s + shift, 2), p, rtol=1e-12, atol=1e-15)
