"""Pins for the DHN closed-walk aggregates (O6) and hash partition -- CPU only.

C_k rules PAPER.md:1509-1518 (C3 in the body at :943-949), read as homomorphisms = closed
walks (Eq. 3 at :1500).  Pinned against dense integer matrix powers
diag(A^k) (all-ones d=1 features, identity mu), the golden counts (K3 -> 2),
a dense einsum closed form with random features, and finite differences for the backward.
"""
import json
import os

import numpy as np
import pytest

EPS = 1e-5


def adjacency(ora, n, arcs, keys):
    e_n = [keys[a] for a, _ in arcs]
    e_v = [keys[b] for _, b in arcs]
    # Edge(n, v) grouped by n; neighbours v sorted by key (DHN adjacency variant)
    return ora.build_join_index(e_v, e_n, s_key=keys, t_key=keys, within_by_src_key=True)


def both_dirs(edges):
    return sorted({(a, b) for a, b in edges} | {(b, a) for a, b in edges})


def test_golden_counts(ora):
    with open(os.path.join(os.path.dirname(__file__), "golden", "dhn_counts.json")) as f:
        gold = json.load(f)
    for name, g in gold["graphs"].items():
        n = g["n"]
        keys = np.arange(n, dtype=np.int64) * 10 + 3
        adj = adjacency(ora, n, both_dirs(g["edges"]), keys)
        ones = [np.ones((n, 1))] * 4
        for k in (2, 3, 4):
            out = ora.dhn_fwd(k, adj, keys, ones[:k])
            assert out[:, 0].tolist() == [float(g[f"C{k}"])] * n, (name, k)


@pytest.mark.parametrize("seed", range(50))
def test_counts_equal_matrix_powers(ora, seed):
    """SPEC.md:571 (50 random graphs <= 12 nodes) incl. directed ones: C_k(n) = (A^k)_nn."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 13))
    p = rng.uniform(0.1, 0.7)
    A = (rng.random((n, n)) < p).astype(np.int64)
    np.fill_diagonal(A, 0)
    if seed % 2 == 0:
        A = np.maximum(A, A.T)
    arcs = [(a, b) for a in range(n) for b in range(n) if A[a, b]]
    if not arcs:
        return
    keys = rng.permutation(n).astype(np.int64) - 5
    adj = adjacency(ora, n, arcs, keys)
    roots = adj["group_dst_row"]
    for k in (2, 3, 4):
        out = ora.dhn_fwd(k, adj, keys, [np.ones((n, 1))] * k)
        if k == 2:
            ref = A.sum(1)              # C2 = one Edge atom: out-degree
        else:
            ref = np.diag(np.linalg.matrix_power(A, k))
        assert out[:, 0].astype(np.int64).tolist() == ref[roots].tolist()


@pytest.mark.parametrize("seed", range(8))
def test_random_features_closed_form(ora, seed):
    rng = np.random.default_rng(seed)
    n, d = int(rng.integers(3, 10)), 3
    A = (rng.random((n, n)) < 0.5).astype(float)
    np.fill_diagonal(A, 0)
    arcs = [(a, b) for a in range(n) for b in range(n) if A[a, b]]
    keys = rng.permutation(n).astype(np.int64)
    adj = adjacency(ora, n, arcs, keys)
    f = [rng.standard_normal((n, d)) for _ in range(4)]
    r = adj["group_dst_row"]
    ref = {2: f[0] * np.einsum("nv,vc->nc", A, f[1]),
           3: f[0] * np.einsum("nv,vw,wn,vc,wc->nc", A, A, A, f[1], f[2]),
           4: f[0] * np.einsum("nv,vw,wp,pn,vc,wc,pc->nc", A, A, A, A, f[1], f[2], f[3])}
    for k in (2, 3, 4):
        np.testing.assert_allclose(ora.dhn_fwd(k, adj, keys, f[:k]), ref[k][r], rtol=1e-12, atol=1e-12)
    sel = np.array([len(r) - 1, 0])
    np.testing.assert_allclose(ora.dhn_fwd(4, adj, keys, f, sel=sel), ref[4][r][sel], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("k", [2, 3, 4])
def test_dhn_bwd_finite_differences(ora, k):
    rng = np.random.default_rng(k)
    n, d = 7, 2
    A = (rng.random((n, n)) < 0.6).astype(int)
    np.fill_diagonal(A, 0)
    A = np.maximum(A, A.T)
    arcs = [(a, b) for a in range(n) for b in range(n) if A[a, b]]
    keys = np.arange(n, dtype=np.int64)
    adj = adjacency(ora, n, arcs, keys)
    f = [rng.standard_normal((n, d)) for _ in range(k)]
    dO = rng.standard_normal((adj["n_groups"], d))
    grads = ora.dhn_bwd(k, adj, keys, f, dO)
    for j in range(k):
        flat = f[j].reshape(-1)
        for i in range(flat.size):
            old = flat[i]
            flat[i] = old + EPS; fp = float((ora.dhn_fwd(k, adj, keys, f) * dO).sum())
            flat[i] = old - EPS; fm = float((ora.dhn_fwd(k, adj, keys, f) * dO).sum())
            flat[i] = old
            num = (fp - fm) / (2 * EPS)
            assert abs(num - grads[j].reshape(-1)[i]) <= 1e-4 * max(1.0, abs(num))


def test_splitmix64_published_vectors(ora):
    """SplitMix64 (Steele, Lea & Flood 2014) seeded with 0 emits 0xe220a8397b1dcdaf,
    0x6e789e6aa1b965f4, 0x06c45d188009454f; ora_splitmix64(x) is the output for state x."""
    gamma = 0x9E3779B97F4A7C15
    assert ora.splitmix64(0) == 0xE220A8397B1DCDAF
    assert ora.splitmix64(gamma) == 0x6E789E6AA1B965F4
    assert ora.splitmix64((2 * gamma) % 2 ** 64) == 0x06C45D188009454F


def test_hash_partition_balance(ora):
    keys = np.arange(100000, dtype=np.int64)
    own = ora.hash_partition(keys, 8, 42)
    cnt = np.bincount(own, minlength=8)
    assert cnt.min() > 0.95 * 12500 and cnt.max() < 1.05 * 12500
