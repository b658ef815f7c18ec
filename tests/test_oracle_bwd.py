"""Pins for the oracle's backward passes (O4, O5 bwd, O6 bwd, softmax bwd) -- CPU only.

Gradients flow through embeddings only.  Pinned by central finite
differences in double (eps = 1e-5, rel. 1e-4: SPEC.md:135, :570), by the adjoint identity
<fwd(x), y> = <x, bwd(y)> for the linear SUM/MEAN paths, and by the SPEC.md:131 duplicate-
index example (tests/golden/index_select_dup.json).
"""
import json
import os

import numpy as np
import pytest

import synth

EPS = 1e-5


def fd_check(f, x, grad, n_probe=12, rng=None, rtol=1e-4):
    """Compare grad (analytic) with central differences of the scalar f at probed entries."""
    rng = rng or np.random.default_rng(0)
    flat = x.reshape(-1)
    idxs = rng.choice(flat.size, size=min(n_probe, flat.size), replace=False)
    for i in idxs:
        old = flat[i]
        flat[i] = old + EPS; fp = f()
        flat[i] = old - EPS; fm = f()
        flat[i] = old
        num = (fp - fm) / (2 * EPS)
        ana = grad.reshape(-1)[i]
        assert abs(num - ana) <= rtol * max(1.0, abs(num)), (i, num, ana)


CASES = [("src", "sum"), ("src", "mean"), ("mul", "sum"), ("mul", "mean"), ("add", "sum"),
         ("add", "mean"), ("concat", "sum"), ("concat", "mean"), ("mul_scalar_edge", "sum")]


@pytest.mark.parametrize("combine,agg", CASES)
@pytest.mark.parametrize("seed", range(3))
def test_lja_bwd_finite_differences(ora, combine, agg, seed):
    rng = np.random.default_rng(100 + seed)
    d_e = 1 if combine in ("src", "mul_scalar_edge") else 3
    db = synth.random_db(rng, 9, 7, 40, d_s=3, d_e=d_e, d_t=3)
    comb = "mul" if combine == "mul_scalar_edge" else combine
    idx = ora.build_join_index(db["e_src"], db["e_dst"], db["s_key"], db["t_key"])
    zs = db["z_s"].astype(float); ze = db["z_e"].astype(float); zt = db["z_t"].astype(float)
    kw = dict(src=zs, edge=ze)
    if comb != "src":
        kw["dst"] = zt
    out, _ = ora.lja_fwd(idx, comb, agg, **kw)
    dO = rng.standard_normal(out.shape)
    grads = ora.lja_bwd(idx, dO, comb, agg, **kw)

    def loss():
        return float((ora.lja_fwd(idx, comb, agg, **kw)[0] * dO).sum())

    fd_check(loss, zs, grads["src"], rng=rng)
    fd_check(loss, ze, grads["edge"], rng=rng)
    if comb != "src":
        fd_check(loss, zt, grads["dst"], rng=rng)


@pytest.mark.parametrize("heads", [1, 2])
def test_softmax_attention_bwd_finite_differences(ora, heads):
    rng = np.random.default_rng(5)
    n_s, n_t, d = 8, 5, 2 * heads
    edges = sorted({(int(rng.integers(0, n_s)), int(rng.integers(0, n_t))) for _ in range(25)})
    K, M, Q = (rng.standard_normal((n, d)) for n in (n_s, n_s, n_t))
    idx = ora.build_join_index([s for s, _ in edges], [t for _, t in edges], np.arange(n_s), np.arange(n_t))
    kw = dict(agg="softmax", src=M, src_key=K, dst=Q, heads=heads, scale=0.7)
    out, _ = ora.lja_fwd(idx, **kw)
    dO = rng.standard_normal(out.shape)
    g = ora.lja_bwd(idx, dO, **kw)

    def loss():
        return float((ora.lja_fwd(idx, **kw)[0] * dO).sum())

    for x, name in ((K, "src_key"), (M, "src"), (Q, "dst")):
        fd_check(loss, x, g[name], n_probe=x.size, rng=rng)


def test_hgt_toy_gradients(ora):
    """SURVEY F2 bwd: dOut = [[1,0],[0,1]] (also re-derived by finite differences above)."""
    K = np.array([[1, 0], [0, 1], [1, 1]], float)
    M = np.array([[1, 2], [3, 4], [5, 6]], float)
    Q = np.array([[1, 0], [0, 2]], float)
    edges = [(0, 0), (1, 0), (2, 0), (1, 1), (2, 1)]
    idx = ora.build_join_index([s for s, _ in edges], [t for _, t in edges], [0, 1, 2], [0, 1])
    g = ora.lja_bwd(idx, np.eye(2), agg="softmax", src=M, src_key=K, dst=Q, heads=1, scale=1.0)
    a = np.exp([1, 0, 1]) / np.exp([1, 0, 1]).sum()
    np.testing.assert_allclose(g["src"], [[a[0], 0], [a[1], 0.5], [a[2], 0.5]], rtol=1e-12)
    # t1 has equal scores: its score gradient is zero, so dQ[1] only sees t0's routing... dQ[0][0] = 0
    assert abs(g["dst"][0, 0]) < 1e-12 and abs(g["dst"][1, 1]) < 1e-12


def test_group_softmax_bwd_fd(ora):
    rng = np.random.default_rng(8)
    sizes = [1, 4, 3]
    gp = np.concatenate([[0], np.cumsum(sizes)])
    idx = {"group_ptr": gp, "n_groups": 3}
    s = rng.standard_normal((8, 2))
    w = rng.standard_normal((8, 2))
    p = ora.group_softmax(idx, s, 2)
    ds = ora.group_softmax_bwd(idx, p, w, 2)
    fd_check(lambda: float((ora.group_softmax(idx, s, 2) * w).sum()), s, ds, n_probe=16, rng=rng)


@pytest.mark.parametrize("agg", ["sum", "mean"])
def test_adjoint_identity(ora, agg):
    """<fwd(x), y> = <x, bwd(y)> for the linear SRC/SUM and SRC/MEAN maps, to 1e-12."""
    rng = np.random.default_rng(21)
    db = synth.random_db(rng, 60, 40, 700, d_s=5, d_e=1)
    idx = ora.build_join_index(db["e_src"], db["e_dst"], db["s_key"], db["t_key"])
    x = rng.standard_normal((60, 5))
    w = rng.standard_normal((700, 1))
    y = rng.standard_normal((idx["n_groups"], 5))
    fx, _ = ora.lja_fwd(idx, "src", agg, src=x, edge=w)
    bx = ora.lja_bwd(idx, y, "src", agg, src=x, edge=w)["src"]
    lhs, rhs = float((fx * y).sum()), float((x * bx).sum())
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


def test_index_select_duplicate_example(ora):
    with open(os.path.join(os.path.dirname(__file__), "golden", "index_select_dup.json")) as f:
        g = json.load(f)
    A = np.array(g["A"])
    # one output group per position of idx (E row j -> group j), source = row idx[j] of A
    idx = ora.build_join_index(g["idx"], list(range(len(g["idx"]))), s_key=[0, 1, 2])
    out, _ = ora.lja_fwd(idx, "src", "sum", src=A)
    assert out.tolist() == g["forward"]
    gr = ora.lja_bwd(idx, np.ones_like(out), "src", "sum", src=A)["src"]
    assert gr.tolist() == g["grad_in"]


def test_unreferenced_rows_get_zero_gradient(ora):
    idx = ora.build_join_index([0, 0], [5, 6], s_key=[0, 1, 2], t_key=[5, 6])
    g = ora.lja_bwd(idx, np.ones((2, 2)), "src", "sum", src=np.ones((3, 2)))["src"]
    assert g[1].tolist() == [0, 0] and g[2].tolist() == [0, 0] and g[0].tolist() == [2, 2]


def test_projection_numpy_and_fd(ora):
    rng = np.random.default_rng(4)
    X, W, b = rng.standard_normal((7, 5)), rng.standard_normal((3, 5)), rng.standard_normal(3)
    Y = ora.project(X, W, b)
    np.testing.assert_allclose(Y, np.matmul(X, W.T) + b, rtol=1e-13)   # library GEMM pin
    dY = rng.standard_normal(Y.shape)
    dX, dW, db = ora.project_bwd(X, W, dY)

    def loss():
        return float((ora.project(X, W, b) * dY).sum())

    fd_check(loss, X, dX, n_probe=35, rng=rng)
    fd_check(loss, W, dW, n_probe=15, rng=rng)
    fd_check(loss, b, db, n_probe=3, rng=rng)
