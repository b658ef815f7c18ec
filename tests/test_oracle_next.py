"""Pins for the oracle of the SURVEY sec 8f rows (oracle/oracle_next.c) -- CPU only.

epilogue : GELU at textbook values (x Phi(x)), ReLU, the gate's two ends, finite differences
MAX      : brute force per group / column with ties resolved to the lowest join position,
           empty groups 0, the adjoint identity (max is linear on a fixed arg-max pattern),
           finite differences away from ties
loss     : uniform logits give log C exactly, rows of d_logits sum to 0, unlabelled rows are
           ignored, finite differences
Adam     : closed forms -- a constant gradient moves every step by lr g / (|g| + eps) (the
           bias corrections cancel the moment decay), weight decay alone moves by lr sign(p)
           on the first step (Kingma & Ba 2015)
"""
import math

import numpy as np
import pytest

import synth

EPS = 1e-6


def fd(f, x, eps=EPS):
    g = np.zeros_like(x)
    it = np.nditer(x, flags=["multi_index"])
    for _ in it:
        i = it.multi_index
        x0 = x[i]
        x[i] = x0 + eps
        a = f(x)
        x[i] = x0 - eps
        b = f(x)
        x[i] = x0
        g[i] = (a - b) / (2 * eps)
    return g


# ---------------------------------------------------------------- epilogue
def test_gelu_relu_values(ora):
    x = np.array([[-2.0, -1.0, 0.0, 1.0, 2.0, 0.5]])
    gelu = [x * 0.5 * (1 + math.erf(x / math.sqrt(2))) for x in x[0]]
    # textbook values of x Phi(x)
    ref = [-0.04550026389635842, -0.15865525393145707, 0.0, 0.8413447460685429,
           1.9544997361036416, 0.34573123063700656]
    np.testing.assert_allclose(gelu, ref, rtol=1e-14)
    np.testing.assert_allclose(ora.epilogue_fwd(x, act="gelu")[0], ref, rtol=1e-14, atol=1e-16)
    np.testing.assert_array_equal(ora.epilogue_fwd(x, act="relu")[0], [0, 0, 0, 1, 2, 0.5])
    b = np.array([1.0, 1, 1, 1, 1, 1])
    np.testing.assert_array_equal(ora.epilogue_fwd(x, bias=b, act="relu")[0], [0, 0, 1, 2, 3, 1.5])


def test_gate_ends(ora):
    rng = np.random.default_rng(0)
    x, r, b = rng.standard_normal((5, 4)), rng.standard_normal((5, 4)), rng.standard_normal(4)
    np.testing.assert_array_equal(ora.epilogue_fwd(x, b, "relu", 1.0, r), ora.epilogue_fwd(x, b, "relu"))
    np.testing.assert_array_equal(ora.epilogue_fwd(x, b, "gelu", 0.0, r), r)


@pytest.mark.parametrize("act", ["none", "relu", "gelu"])
@pytest.mark.parametrize("gated", [False, True])
def test_epilogue_bwd_fd(ora, act, gated):
    rng = np.random.default_rng(1 + gated)
    x = rng.standard_normal((6, 5)) + 0.05          # keep ReLU kinks away from 0
    b = rng.standard_normal(5) * 0.3
    r = rng.standard_normal((6, 5)) if gated else None
    gate = 0.3 if gated else 1.0
    dy = rng.standard_normal((6, 5))
    loss = lambda: float(np.sum(ora.epilogue_fwd(x, b, act, gate, r) * dy))
    dx, db, dr, dg = ora.epilogue_bwd(dy, x, b, act, gate, r)
    np.testing.assert_allclose(dx, fd(lambda xx: loss(), x), rtol=1e-6, atol=1e-8)
    np.testing.assert_allclose(db, fd(lambda bb: loss(), b), rtol=1e-6, atol=1e-8)
    if gated:
        np.testing.assert_allclose(dr, fd(lambda rr: loss(), r), rtol=1e-6, atol=1e-8)
        g0 = gate
        num = (float(np.sum(ora.epilogue_fwd(x, b, act, g0 + EPS, r) * dy)) -
               float(np.sum(ora.epilogue_fwd(x, b, act, g0 - EPS, r) * dy))) / (2 * EPS)
        assert abs(dg - num) < 1e-6 * max(1, abs(num))


# ---------------------------------------------------------------- MAX aggregate
def _db(seed, n_e=400, hub=True):
    rng = np.random.default_rng(seed)
    db = synth.random_db(rng, 30, 25, n_e, d_s=6)
    if hub:
        db["e_dst"][: n_e // 4] = db["t_key"][0]
    return db, rng


def test_max_bruteforce_and_ties(ora):
    db, rng = _db(3)
    idx = ora.build_join_index(db["e_src"], db["e_dst"], db["s_key"], db["t_key"])
    z = rng.integers(-3, 4, (30, 6)).astype(np.float64)     # many exact ties
    w = rng.choice([0.5, 1.0, 2.0], idx["n_join_rows"])
    out, am = ora.lja_max_fwd(idx, z, w)
    gp = idx["group_ptr"]
    for g in range(idx["n_groups"]):
        rows = np.arange(gp[g], gp[g + 1])
        vals = w[rows, None] * z[idx["src_row"][rows]]
        np.testing.assert_array_equal(out[g], vals.max(0))
        # the arg-max is the FIRST position attaining the max
        np.testing.assert_array_equal(am[g], rows[np.argmax(vals == vals.max(0), axis=0)])


def test_max_empty_group_is_zero(ora):
    idx = {"group_ptr": np.array([0, 0, 2], np.int64), "n_groups": 2,
           "src_row": np.array([0, 1], np.int32), "edge_row": np.array([0, 1], np.int32)}
    z = np.array([[-5.0, 1.0], [-7.0, 3.0]])
    out, am = ora.lja_max_fwd(idx, z)
    np.testing.assert_array_equal(out, [[0, 0], [-5, 3]])
    np.testing.assert_array_equal(am, [[-1, -1], [0, 1]])


def test_max_adjoint_and_fd(ora):
    db, rng = _db(5)
    idx = ora.build_join_index(db["e_src"], db["e_dst"], db["s_key"], db["t_key"])
    z = rng.standard_normal((30, 6))
    w = rng.uniform(0.5, 1.5, idx["n_join_rows"])
    out, am = ora.lja_max_fwd(idx, z, w)
    dO = rng.standard_normal(out.shape)
    dz, dw = ora.lja_max_bwd(idx, z, am, dO, w)
    # max is linear in (z, w-scaled rows) on a fixed arg-max pattern: <out, dO> = <z, dz>
    assert abs(float(np.sum(out * dO)) - float(np.sum(z * dz))) < 1e-12 * max(1, abs(float(np.sum(out * dO))))
    loss_z = lambda zz: float(np.sum(ora.lja_max_fwd(idx, zz, w)[0] * dO))
    loss_w = lambda ww: float(np.sum(ora.lja_max_fwd(idx, z, ww)[0] * dO))
    np.testing.assert_allclose(dz, fd(loss_z, z), rtol=1e-6, atol=1e-8)
    np.testing.assert_allclose(dw, fd(loss_w, w), rtol=1e-6, atol=1e-8)


# ---------------------------------------------------------------- loss
def test_xent_closed_forms(ora):
    C = 7
    loss, d = ora.softmax_xent(np.zeros((4, C)), np.array([0, 3, 6, 2]))
    assert loss == pytest.approx(math.log(C), rel=1e-15)
    np.testing.assert_allclose(d.sum(1), 0, atol=1e-16)
    x = np.zeros((2, 3)); x[0, 1] = 50.0; x[1, 2] = 50.0
    loss, _ = ora.softmax_xent(x, np.array([1, -1]))      # unlabelled row ignored
    assert loss < 1e-20
    _, d2 = ora.softmax_xent(x, np.array([1, -1]))
    np.testing.assert_array_equal(d2[1], 0)


def test_xent_fd(ora):
    rng = np.random.default_rng(2)
    x = rng.standard_normal((6, 5))
    lab = np.array([0, 4, -1, 2, 2, 1])
    _, d = ora.softmax_xent(x, lab)
    np.testing.assert_allclose(d, fd(lambda xx: ora.softmax_xent(xx, lab)[0], x), rtol=1e-6, atol=1e-9)


# ---------------------------------------------------------------- Adam
def test_adam_constant_gradient_closed_form(ora):
    rng = np.random.default_rng(4)
    p0 = rng.standard_normal(9)
    g = rng.standard_normal(9)
    p, m, v = p0.copy(), np.zeros(9), np.zeros(9)
    lr, eps, T = 0.01, 1e-8, 25
    for t in range(1, T + 1):
        ora.adam(p, g, m, v, lr, t, eps=eps)
    np.testing.assert_allclose(p, p0 - T * lr * g / (np.abs(g) + eps), rtol=1e-12, atol=1e-14)


def test_adam_weight_decay_first_step(ora):
    p0 = np.array([2.0, -3.0, 0.5])
    p, m, v = p0.copy(), np.zeros(3), np.zeros(3)
    ora.adam(p, np.zeros(3), m, v, 0.1, 1, eps=0.0, wd=5e-4)
    np.testing.assert_allclose(p, p0 - 0.1 * np.sign(p0), rtol=1e-15)
