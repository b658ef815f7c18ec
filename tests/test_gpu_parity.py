"""GPU parity: librnn.so (through its C ABI) against the CPU oracle, element by element.

Integer outputs (join index, group ids, CSR, partition) must be bit-exact; fp32 outputs are
judged with the DESIGN.md metric (tests/util.py) at 1e-4 (fp32 paths) / 1e-2 (tf32 paths).
Inputs are seeded synthetic relations (synth/), sized to span several work items, hub
groups split across items, ragged tails, dangling keys, empty relations.
"""
import zlib

import numpy as np
import pytest
import torch

import synth
from tests.util import FP32_TOL, TF32_TOL, assert_close, assert_close_scale, np_

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    from paper_2605_24207_b200 import rnn
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    rnn.lib()
    return rnn


def cu(a, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def padded(x, ld=None):
    """fp32 device tensor with a padded leading dimension (ld % 4 == 0), returned as a view."""
    x = np.asarray(x, np.float32)
    if x.ndim == 1:
        x = x[:, None]
    n, d = x.shape
    ld = ld or (d + 3) // 4 * 4
    buf = torch.full((max(n, 1), ld), float("nan"), dtype=torch.float32, device="cuda")
    buf[:n, :d] = torch.from_numpy(x)
    return buf[:n, :d]


def check_index(gi, oi, transpose=True):
    assert gi.n_join_rows == oi["n_join_rows"] and gi.n_groups == oi["n_groups"]
    for k in ("group_ptr", "group_key", "group_dst_row", "src_row", "edge_row"):
        np.testing.assert_array_equal(np_(getattr(gi, k)), oi[k], err_msg=k)
    if transpose and oi["src_ptr"] is not None:
        np.testing.assert_array_equal(np_(gi.src_ptr), oi["src_ptr"])
        np.testing.assert_array_equal(np_(gi.src_pos), oi["src_pos"])
        gp = oi["group_ptr"]
        grp = np.searchsorted(gp, oi["src_pos"], side="right") - 1
        np.testing.assert_array_equal(np_(gi.src_group), grp)
    # schedule sanity: items partition [0, E'), long segments start/end at boundaries
    wp = np_(gi.work_ptr)
    assert wp[0] == 0 and wp[-1] == gi.n_join_rows and np.all(np.diff(wp) > 0)


@pytest.mark.parametrize("seed", range(40))
def test_index_random(R, ora, seed):
    rng = np.random.default_rng(seed)
    n_s, n_t = int(rng.integers(0, 60)), int(rng.integers(0, 60))
    n_e = int(rng.integers(0, 3000))
    db = synth.random_db(rng, n_s, n_t, n_e, key_space=int(rng.integers(40, 400)))
    if seed % 4 == 0 and n_e:  # hubs: a few groups hold most rows
        db["e_dst"][: n_e // 2] = db["e_dst"][0]
    use_s, use_t = seed % 5 != 1, seed % 3 != 2
    by_key = use_s and use_t and seed % 6 == 0
    s_key = db["s_key"] if use_s else None
    t_key = db["t_key"] if use_t else None
    rpi = [0, 4, 7, 64][seed % 4]
    gi = R.build_join_index(cu(db["e_src"]), cu(db["e_dst"]), None if s_key is None else cu(s_key),
                            None if t_key is None else cu(t_key), within_group_by_src_key=by_key,
                            rows_per_item=rpi)
    oi = ora.build_join_index(db["e_src"], db["e_dst"], s_key, t_key, within_by_src_key=by_key)
    check_index(gi, oi)


def test_index_duplicate_key(R):
    with pytest.raises(R.RnnError, match="DUPLICATE"):
        R.build_join_index(cu(np.array([1, 2])), cu(np.array([3, 3])), cu(np.array([1, 2, 1])),
                           cu(np.array([3])))
    with pytest.raises(R.RnnError, match="DUPLICATE"):   # INT64_MIN sentinel path
        m = np.iinfo(np.int64).min
        R.build_join_index(cu(np.array([1])), cu(np.array([3])), cu(np.array([m, 1, m])), None)


def test_index_deterministic(R):
    rng = np.random.default_rng(1)
    db = synth.random_db(rng, 500, 300, 20000)
    a = R.build_join_index(cu(db["e_src"]), cu(db["e_dst"]), cu(db["s_key"]), cu(db["t_key"]))
    b = R.build_join_index(cu(db["e_src"]), cu(db["e_dst"]), cu(db["s_key"]), cu(db["t_key"]))
    for k, v in a.arrays.items():
        assert torch.equal(v, b.arrays[k]), k


def make_case(rng, n_s=300, n_t=200, n_e=6000, d=16, d_e=1, d_t=16, hub=True):
    db = synth.random_db(rng, n_s, n_t, n_e, d_s=d, d_e=d_e, d_t=d_t)
    if hub:
        db["e_dst"][: n_e // 3] = db["t_key"][0]   # one group of ~n_e/3 rows -> split pieces
    return db


FWD_CASES = [
    # combine, agg, d_src, d_edge, d_dst, edge_mode
    ("src", "sum", 16, 1, None, 0), ("src", "mean", 16, 1, None, 1), ("src", "sum", 128, None, None, 0),
    ("src", "sum", 7, 1, None, 1), ("src", "mean", 3, None, None, 0), ("src", "sum", 200, 1, None, 0),
    ("src", "sum", 512, 1, None, 0), ("src", "sum", 32, 1, None, 0), ("src", "sum", 1, 1, None, 0),
    ("mul", "sum", 32, None, 32, 0), ("mul", "mean", 16, 16, 16, 0), ("mul", "sum", 16, 1, 16, 1),
    ("mul", "sum", 128, 128, None, 0), ("mul", "sum", 8, None, 1, 0), ("mul", "sum", None, 12, None, 0),
    ("add", "sum", 16, 16, 16, 0), ("add", "mean", 16, 1, 16, 0), ("add", "sum", 64, None, None, 0),
    ("concat", "sum", 5, 3, 2, 0), ("concat", "mean", 16, 1, None, 0),
]


def operands(db, d_s, d_e, d_t, edge_mode, idx_o, rng):
    src = rng.standard_normal((len(db["s_key"]), d_s)).astype(np.float32) if d_s else None
    n_e = len(db["e_src"]) if edge_mode == 0 else idx_o["n_join_rows"]
    edge = rng.standard_normal((n_e, d_e)).astype(np.float32) if d_e else None
    dst = rng.standard_normal((len(db["t_key"]), d_t)).astype(np.float32) if d_t else None
    return src, edge, dst


@pytest.mark.parametrize("case", FWD_CASES, ids=lambda c: "-".join(map(str, c)))
def test_fwd_bwd_parity(R, ora, case):
    combine, agg, d_s, d_e, d_t, emode = case
    rng = np.random.default_rng(zlib.crc32(repr(case).encode()))
    db = make_case(rng, n_e=5000, d=4)
    s_key = db["s_key"] if d_s else None
    gi = R.build_join_index(cu(db["e_src"]), cu(db["e_dst"]), None if s_key is None else cu(s_key),
                            cu(db["t_key"]), rows_per_item=16)
    oi = ora.build_join_index(db["e_src"], db["e_dst"], s_key, db["t_key"])
    src, edge, dst = operands(db, d_s, d_e, d_t, emode, oi, rng)
    q = R.make_query(combine, agg, src=None if src is None else padded(src),
                     edge=None if edge is None else padded(edge), dst=None if dst is None else padded(dst),
                     edge_mode=emode)
    out = R.join_aggregate_fwd(gi, q)
    ref, _ = ora.lja_fwd(oi, combine, agg, src=src, edge=edge, dst=dst, edge_mode=emode)
    assert_close(np_(out), ref, FP32_TOL, "fwd")
    # beta = 1 accumulation (union over relations) for SUM
    if agg == "sum":
        out2 = padded(np_(out))
        R.join_aggregate_fwd(gi, q, out=out2, beta=1.0)
        assert_close(np_(out2), 2 * ref, FP32_TOL, "beta")
    dO = rng.standard_normal(ref.shape).astype(np.float32)
    g = R.join_aggregate_bwd(gi, q, padded(dO))
    gr = ora.lja_bwd(oi, dO, combine, agg, src=src, edge=edge, dst=dst, edge_mode=emode)
    for k in ("src", "edge", "dst"):
        if gr[k] is not None:
            assert_close(np_(g[k]), gr[k], FP32_TOL, f"d_{k}")


@pytest.mark.parametrize("heads,D", [(8, 128), (1, 128), (2, 128), (4, 128), (16, 128), (32, 128),
                                     (1, 4), (2, 16), (4, 32), (2, 64)])
def test_softmax_attention_parity(R, ora, heads, D):
    rng = np.random.default_rng(D + heads)
    db = make_case(rng, n_s=400, n_t=150, n_e=8000)
    gi = R.build_join_index(cu(db["e_src"]), cu(db["e_dst"]), cu(db["s_key"]), cu(db["t_key"]),
                            rows_per_item=32)
    oi = ora.build_join_index(db["e_src"], db["e_dst"], db["s_key"], db["t_key"])
    K = (rng.standard_normal((400, D)) * 0.5).astype(np.float32)
    M = rng.standard_normal((400, D)).astype(np.float32)
    Q = (rng.standard_normal((150, D)) * 0.5).astype(np.float32)
    scale = 1.0 / np.sqrt(D / heads)
    q = R.make_query("src", "softmax", src=padded(M), src_key=padded(K), dst=padded(Q), heads=heads,
                     scale=scale)
    out, lse = R.join_aggregate_fwd(gi, q)
    ref, rlse = ora.lja_fwd(oi, agg="softmax", src=M, src_key=K, dst=Q, heads=heads, scale=scale)
    assert_close(np_(out), ref, FP32_TOL, "out")
    assert_close(np_(lse)[: oi["n_groups"]], rlse, FP32_TOL, "lse")
    dO = rng.standard_normal(ref.shape).astype(np.float32)
    g = R.join_aggregate_bwd(gi, q, padded(dO), out=out, lse=lse)
    gr = ora.lja_bwd(oi, dO, agg="softmax", src=M, src_key=K, dst=Q, heads=heads, scale=scale)
    for k in ("src", "src_key", "dst"):
        assert_close(np_(g[k]), gr[k], FP32_TOL, f"d_{k}")


@pytest.mark.parametrize("n_t,n_e,rpi", [(3000, 4000, 32), (900, 5000, 64), (2500, 2600, 0)])
def test_softmax_small_groups(R, ora, n_t, n_e, rpi):
    """Many groups of 1-3 rows next to a split hub: the group-cached walkers see batches that
    cross one or two group ends, groups that start mid-batch and pieces of the hub."""
    rng = np.random.default_rng(n_t + n_e)
    D, heads = 128, 8
    db = make_case(rng, n_s=500, n_t=n_t, n_e=n_e)
    gi = R.build_join_index(cu(db["e_src"]), cu(db["e_dst"]), cu(db["s_key"]), cu(db["t_key"]),
                            rows_per_item=rpi)
    oi = ora.build_join_index(db["e_src"], db["e_dst"], db["s_key"], db["t_key"])
    K = (rng.standard_normal((500, D)) * 0.5).astype(np.float32)
    M = rng.standard_normal((500, D)).astype(np.float32)
    Q = (rng.standard_normal((n_t, D)) * 0.5).astype(np.float32)
    scale = 1.0 / np.sqrt(D / heads)
    q = R.make_query("src", "softmax", src=padded(M), src_key=padded(K), dst=padded(Q), heads=heads,
                     scale=scale)
    out, lse = R.join_aggregate_fwd(gi, q)
    ref, rlse = ora.lja_fwd(oi, agg="softmax", src=M, src_key=K, dst=Q, heads=heads, scale=scale)
    assert_close(np_(out), ref, FP32_TOL, "out")
    assert_close(np_(lse)[: oi["n_groups"]], rlse, FP32_TOL, "lse")
    dO = rng.standard_normal(ref.shape).astype(np.float32)
    g = R.join_aggregate_bwd(gi, q, padded(dO), out=out, lse=lse)
    gr = ora.lja_bwd(oi, dO, agg="softmax", src=M, src_key=K, dst=Q, heads=heads, scale=scale)
    for k in ("src", "src_key", "dst"):
        assert_close(np_(g[k]), gr[k], FP32_TOL, f"d_{k}")


def test_softmax_dense_groups_beta(R, ora):
    """Row-split softmax (D = 128) over a dense-group index: T keys with no join row give
    out 0 / lse -inf / dQ 0; beta = 1 adds onto an existing union (A7); hub pieces merge."""
    rng = np.random.default_rng(77)
    db = make_case(rng, n_s=500, n_t=300, n_e=9000)
    db["e_dst"] = np.where(np.isin(db["e_dst"], db["t_key"][100:140]), db["t_key"][0], db["e_dst"])
    gi = R.build_join_index(cu(db["e_src"]), cu(db["e_dst"]), cu(db["s_key"]), cu(db["t_key"]),
                            dense_groups=True, rows_per_item=48)
    oi = ora.build_join_index(db["e_src"], db["e_dst"], db["s_key"], db["t_key"])
    D, h = 128, 8
    K = (rng.standard_normal((500, D)) * 0.5).astype(np.float32)
    M = rng.standard_normal((500, D)).astype(np.float32)
    Q = (rng.standard_normal((300, D)) * 0.5).astype(np.float32)
    q = R.make_query("src", "softmax", src=padded(M), src_key=padded(K), dst=padded(Q), heads=h,
                     scale=0.25)
    out, lse = R.join_aggregate_fwd(gi, q)
    ref, rlse = ora.lja_fwd(oi, agg="softmax", src=M, src_key=K, dst=Q, heads=h, scale=0.25)
    # dense groups are every T key in ascending key order; present groups sit at their key's rank
    rows = np.searchsorted(np.sort(db["t_key"]), oi["group_key"])
    assert gi.n_groups == 300
    full = np.zeros((300, D)); full[rows] = ref
    flse = np.full((300, h), -np.inf); flse[rows] = rlse
    absent = np.setdiff1d(np.arange(300), rows)
    assert len(absent) >= 40
    assert_close(np_(out), full, FP32_TOL, "out")
    got_lse = np_(lse)
    assert np.all(np.isneginf(got_lse[absent]))
    assert_close(got_lse[rows], rlse, FP32_TOL, "lse")
    base = rng.standard_normal((300, D)).astype(np.float32)
    acc = padded(base)
    R.join_aggregate_fwd(gi, q, out=acc, lse=torch.empty(300, h, device="cuda"), beta=1.0)
    assert_close(np_(acc), base + full, FP32_TOL, "beta")
    dO = rng.standard_normal((300, D)).astype(np.float32)
    g = R.join_aggregate_bwd(gi, q, padded(dO), out=out, lse=lse)
    gr = ora.lja_bwd(oi, dO[rows], agg="softmax", src=M, src_key=K, dst=Q, heads=h, scale=0.25)
    for k in ("src", "src_key", "dst"):
        assert_close(np_(g[k]), gr[k], FP32_TOL, f"d_{k}")


def test_group_softmax_parity(R, ora):
    rng = np.random.default_rng(3)
    db = make_case(rng, n_e=3000)
    gi = R.build_join_index(cu(db["e_src"]), cu(db["e_dst"]), cu(db["s_key"]), cu(db["t_key"]))
    oi = ora.build_join_index(db["e_src"], db["e_dst"], db["s_key"], db["t_key"])
    s = (rng.standard_normal((oi["n_join_rows"], 3)) * 3).astype(np.float32)
    p = R.group_softmax(gi, cu(s), 3)
    assert_close(np_(p), ora.group_softmax(oi, s, 3), FP32_TOL, "probs")
    dp = rng.standard_normal(s.shape).astype(np.float32)
    ds = R.group_softmax_bwd(gi, p, cu(dp), 3)
    assert_close(np_(ds), ora.group_softmax_bwd(oi, np_(p), dp, 3), FP32_TOL, "dscores")


@pytest.mark.parametrize("M,K,N", [(300, 128, 128), (2708, 1433, 16), (2708, 16, 7), (1000, 40, 200),
                                   (129, 32, 48), (5000, 128, 256), (77, 8, 3),
                                   # persistent resident-W kernel: many row tiles per CTA,
                                   # several column blocks, ragged K / N
                                   (100000, 128, 128), (60001, 128, 384), (40000, 64, 256),
                                   (3001, 200, 100)])
@pytest.mark.parametrize("prec", ["3xtf32", "tf32"])
def test_projection_parity(R, ora, M, K, N, prec):
    rng = np.random.default_rng(M + K + N)
    X = (rng.standard_normal((M, K)) / np.sqrt(K)).astype(np.float32)
    W = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    b = rng.standard_normal(N).astype(np.float32)
    tol = FP32_TOL if prec == "3xtf32" else TF32_TOL
    Xd, Wd = padded(X), padded(W)
    Y = R.project(Xd, Wd, cu(b), prec=prec)
    assert_close(np_(Y), ora.project(X, W, b), tol, "Y")
    dY = rng.standard_normal((M, N)).astype(np.float32)
    dX, dW, db = R.project_bwd(Xd, Wd, padded(dY), want_db=True, prec=prec)
    rdX, rdW, rdb = ora.project_bwd(X, W, dY)
    assert_close(np_(dX), rdX, tol, "dX")
    assert_close(np_(dW), rdW, tol, "dW")
    assert_close(np_(db), rdb, FP32_TOL, "db")


def bf16_rne(a):
    """fp32 -> nearest bf16 (ties to even), returned as fp32 (test-side input rounding, SURVEY
    O5: 'inputs rounded to tf32/bf16 first when checking the reduced-precision path')."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


@pytest.mark.parametrize("M,K,N", [(300, 128, 128), (60001, 128, 384), (5001, 200, 100),
                                   (2708, 1433, 16), (1000, 40, 200), (77, 8, 3)])
def test_projection_bf16(R, ora, M, K, N):
    """RNN_PREC_BF16 (north_star: 1e-2 for bf16 projections) on every kernel family (TMEM-resident
    W, resident-B, tile GEMM; dW split-K): within 1e-2 of the exact product, and within fp32
    tolerance of the oracle on bf16-rounded inputs -- which pins the rounding (RNE to bf16, not a
    tf32 truncation) and the exactness of the products."""
    rng = np.random.default_rng(11 * M + K + N)
    X = (rng.standard_normal((M, K)) / np.sqrt(K)).astype(np.float32)
    W = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    b = rng.standard_normal(N).astype(np.float32)
    dY = rng.standard_normal((M, N)).astype(np.float32)
    Y = np_(R.project(padded(X), padded(W), cu(b), prec="bf16"))
    assert_close_scale(Y, ora.project(X, W, b), TF32_TOL, "Y vs exact")
    assert_close(Y, ora.project(bf16_rne(X), bf16_rne(W), b), FP32_TOL, "Y vs rounded inputs")
    dX, dW, db = R.project_bwd(padded(X), padded(W), padded(dY), want_db=True, prec="bf16")
    rdX, rdW, rdb = ora.project_bwd(X, W, dY)
    assert_close_scale(np_(dX), rdX, TF32_TOL, "dX vs exact")
    assert_close_scale(np_(dW), rdW, TF32_TOL, "dW vs exact")
    qdX, qdW, _ = ora.project_bwd(bf16_rne(X), bf16_rne(W), bf16_rne(dY))
    assert_close(np_(dX), qdX, FP32_TOL, "dX vs rounded inputs")
    assert_close(np_(dW), qdW, FP32_TOL, "dW vs rounded inputs")
    assert_close(np_(db), rdb, FP32_TOL, "db (fp32 column sums)")


def test_bf16_rne_helper():
    x = np.array([1.0, 1 + 2 ** -8, 1 + 3 * 2 ** -8, 1 + 2 ** -7, -2.5, 3e-39], np.float32)
    # 1 + 2^-8 is a tie -> even (1.0); 1 + 3 * 2^-8 is a tie -> even (1 + 2^-6)
    np.testing.assert_array_equal(bf16_rne(x)[:5], np.array([1.0, 1.0, 1 + 2 ** -6, 1 + 2 ** -7, -2.5],
                                                            np.float32))


@pytest.mark.parametrize("M,K,N,ldx,lddy", [(5000, 40, 100, 64, 128), (70001, 128, 48, 128, 64),
                                             (3000, 96, 16, 96, 32)])
def test_projection_bwd_wide_ld(R, ora, M, K, N, ldx, lddy):
    """dW through the 3D-box TMA path with ragged MN widths: the last 32-wide chunk reads the
    NaN row padding, which may only reach accumulator rows / columns that are never stored."""
    rng = np.random.default_rng(M + N)
    X = (rng.standard_normal((M, K)) / np.sqrt(K)).astype(np.float32)
    W = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    dY = rng.standard_normal((M, N)).astype(np.float32)
    dX, dW, _ = R.project_bwd(padded(X, ldx), padded(W), padded(dY, lddy), prec="3xtf32")
    rdX, rdW, _ = ora.project_bwd(X, W, dY)
    assert_close(np_(dX), rdX, FP32_TOL, "dX")
    assert_close(np_(dW), rdW, FP32_TOL, "dW")


@pytest.mark.parametrize("M,K,N", [(300, 128, 40), (100000, 128, 40), (5001, 256, 7), (77, 8, 3),
                                   (60001, 384, 128), (2708, 16, 7),
                                   # N > 128: unfused path (mask + column-sum kernels)
                                   (3000, 64, 200)])
def test_projection_bwd_relu_parity(R, ora, M, K, N):
    """rnn_project_bwd_relu = rnn_project_bwd then the ReLU epilogue backward on dX (reading
     of the GCN hidden layer): dP = (dY W) * [X > 0], d_in_bias = colsum(dP).
    X is a ReLU output (about half exact zeros), so the mask is the same decision on both sides."""
    rng = np.random.default_rng(3 * M + K + N)
    X = np.maximum(rng.standard_normal((M, K)) / np.sqrt(K), 0).astype(np.float32)
    W = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    dY = rng.standard_normal((M, N)).astype(np.float32)
    dbi = torch.full((K,), float("nan"), device="cuda")
    dX, dW, db = R.project_bwd(padded(X), padded(W), padded(dY), want_db=True, relu_in=True,
                               d_in_bias=dbi)
    rdX, rdW, rdb = ora.project_bwd(X, W, dY)
    rdP, rdbi, _, _ = ora.epilogue_bwd(rdX, X, np.zeros(K), "relu")
    assert_close(np_(dX), rdP, FP32_TOL, "dP")
    assert (np_(dX)[X == 0] == 0).all()
    assert_close(np_(dbi), rdbi, FP32_TOL, "d_in_bias")
    assert_close(np_(dW), rdW, FP32_TOL, "dW")
    assert_close(np_(db), rdb, FP32_TOL, "db")
    # deterministic: the fused column sums are reduced in a fixed order
    dbi2 = torch.empty_like(dbi)
    R.project_bwd(padded(X), padded(W), padded(dY), relu_in=True, d_in_bias=dbi2)
    assert torch.equal(dbi, dbi2)


def test_gcn_norm_and_partition(R, ora):
    g = synth.cora_like(42)
    keys = g["nodes"]["key"]
    gi = R.build_join_index(cu(g["edges"]["src"]), cu(g["edges"]["dst"]), cu(keys), cu(keys))
    oi = ora.build_join_index(g["edges"]["src"], g["edges"]["dst"], keys, keys)
    check_index(gi, oi)
    assert_close(np_(R.gcn_norm(gi)), ora.gcn_norm(oi, len(keys)), FP32_TOL, "norm")
    for P in (1, 2, 8, 7):
        np.testing.assert_array_equal(np_(R.hash_partition(cu(keys), P, 42)),
                                      ora.hash_partition(keys, P, 42))


def test_fwd_deterministic(R):
    rng = np.random.default_rng(5)
    db = make_case(rng, n_e=20000)
    gi = R.build_join_index(cu(db["e_src"]), cu(db["e_dst"]), cu(db["s_key"]), cu(db["t_key"]),
                            rows_per_item=8)
    src = padded(rng.standard_normal((300, 128)).astype(np.float32))
    q = R.make_query("src", "sum", src=src)
    a = R.join_aggregate_fwd(gi, q)
    b = R.join_aggregate_fwd(gi, q)
    assert torch.equal(a, b)
    dO = padded(rng.standard_normal((gi.n_groups, 128)).astype(np.float32))
    ga = R.join_aggregate_bwd(gi, q, dO)["src"]
    gb = R.join_aggregate_bwd(gi, q, dO)["src"]
    assert torch.equal(ga, gb)


def test_empty_join(R):
    gi = R.build_join_index(cu(np.array([5, 6])), cu(np.array([7, 8])), cu(np.array([1, 2])),
                            cu(np.array([7, 8])))
    assert gi.n_join_rows == 0 and gi.n_groups == 0
    src = padded(np.ones((2, 4), np.float32))
    q = R.make_query("src", "sum", src=src)
    out = R.join_aggregate_fwd(gi, q)
    assert out.shape[0] == 0
    g = R.join_aggregate_bwd(gi, q, torch.zeros(1, 4, device="cuda"))
    assert torch.count_nonzero(g["src"]) == 0


@pytest.mark.parametrize("M,K,N", [(2708, 1433, 16), (1000, 40, 200), (100000, 128, 128)])
def test_projection_repeat_bitwise(R, M, K, N):
    """Repeated projection fwd / bwd calls give bit-identical results (catches races in the
    asynchronous TMA-store epilogue: a partial last row tile once lost a 32-row chunk)."""
    rng = np.random.default_rng(7 * M + K)
    Xd = padded((rng.standard_normal((M, K)) / np.sqrt(K)).astype(np.float32))
    Wd = padded((rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32))
    dYd = padded(rng.standard_normal((M, N)).astype(np.float32))
    Y0 = R.project(Xd, Wd).clone()
    dX0, dW0, _ = R.project_bwd(Xd, Wd, dYd)
    dX0, dW0 = dX0.clone(), dW0.clone()
    for _ in range(12):
        assert torch.equal(R.project(Xd, Wd), Y0)
        dX, dW, _ = R.project_bwd(Xd, Wd, dYd)
        assert torch.equal(dX, dX0) and torch.equal(dW, dW0)


@pytest.mark.parametrize("agg", ["sum", "softmax"])
def test_empty_join_dense_groups(R, agg):
    """Dense-group index over an empty join (no S key matches): every T row is a group with no
    rows, so out = 0 (beta = 0; beta = 1 leaves out unchanged), lse = -inf and every gradient
    is 0 -- even though there are no work items (rnn.h contract)."""
    gi = R.build_join_index(cu(np.array([5, 6, 5])), cu(np.array([7, 8, 8])), cu(np.array([1, 2])),
                            cu(np.array([7, 8, 9])), dense_groups=True)
    assert gi.n_join_rows == 0 and gi.n_groups == 3
    D, h = (8, 1) if agg == "sum" else (128, 8)
    src = padded(np.ones((2, D), np.float32))
    if agg == "sum":
        q = R.make_query("mul", "sum", src=src, dst=padded(np.ones((3, D), np.float32)))
    else:
        q = R.make_query("src", "softmax", src=src, src_key=src, dst=padded(np.ones((3, D), np.float32)),
                         heads=h, scale=0.25)
    out = padded(np.full((3, D), np.nan, np.float32))
    lse = torch.full((3, h), 7.0, device="cuda") if agg == "softmax" else None
    R.join_aggregate_fwd(gi, q, out=out, lse=lse)
    assert torch.count_nonzero(out) == 0
    if lse is not None:
        assert bool(torch.all(torch.isneginf(lse)))
    base = padded(np.full((3, D), 2.0, np.float32))
    R.join_aggregate_fwd(gi, q, out=base, lse=lse, beta=1.0)
    assert bool(torch.all(base == 2.0))
    dO = padded(np.ones((3, D), np.float32))
    kw = {"out": out, "lse": lse} if agg == "softmax" else {}
    g = R.join_aggregate_bwd(gi, q, dO, **kw)
    for k in ("src", "src_key", "dst"):
        if g.get(k) is not None:
            assert torch.count_nonzero(g[k]) == 0, k


@pytest.mark.parametrize("D", [128, 16, 256])
@pytest.mark.parametrize("act", ["none", "relu", "gelu"])
@pytest.mark.parametrize("gated", [False, True])
def test_epilogue_fused_parity(R, ora, D, act, gated):
    """rnn_join_aggregate_fwd_epi: y = gate act(LJA + b) + (1 - gate) r fused into the lean
    store (D = 128, 256) or applied after the aggregate (D = 16); rnn_epilogue_bwd: dx, d_bias,
    d_resid, d_gate -- against oracle.lja_fwd + oracle.epilogue_fwd / _bwd."""
    rng = np.random.default_rng(D + 7 * gated + len(act))
    db = make_case(rng, n_s=300, n_t=200, n_e=5000, d=4)
    gi = R.build_join_index(cu(db["e_src"]), cu(db["e_dst"]), cu(db["s_key"]), cu(db["t_key"]),
                            rows_per_item=16, dense_groups=True)
    oi = ora.build_join_index(db["e_src"], db["e_dst"], db["s_key"], db["t_key"])
    z = rng.standard_normal((300, D)).astype(np.float32)
    w = rng.uniform(0.5, 1.5, gi.n_join_rows).astype(np.float32)
    b = (rng.standard_normal(D) * 0.5).astype(np.float32)
    G = gi.n_groups
    r = rng.standard_normal((G, D)).astype(np.float32) if gated else None
    gate = 0.35 if gated else 1.0
    pre = padded(np.full((G, D), np.nan, np.float32))
    zg, bg, rg = padded(z), cu(b), (padded(r) if gated else None)
    epi = R.make_epilogue(bias=bg, act=act, gate=gate, resid=rg, pre=pre)
    q = R.make_query("src", "sum", src=zg, edge=cu(w), edge_mode=R.BY_POSITION)
    out = R.join_aggregate_fwd_epi(gi, q, epi)
    # oracle: compact groups sit at their key's rank among the dense groups; empty ones
    # aggregate to 0 before the epilogue
    rows = np.searchsorted(np.sort(db["t_key"]), oi["group_key"])
    agg = np.zeros((G, D))
    ow = np.zeros(oi["n_join_rows"])
    ow[:] = w[: oi["n_join_rows"]]
    agg[rows], _ = ora.lja_fwd(oi, "src", "sum", src=z, edge=ow, edge_mode=1)
    ref = ora.epilogue_fwd(agg, b, act, gate, r)
    assert_close(np_(out), ref, FP32_TOL, "y")
    assert_close(np_(pre), agg + b, FP32_TOL, "pre")
    dy = rng.standard_normal((G, D)).astype(np.float32)
    dx, dbias, dres, dgate = R.epilogue_bwd(padded(dy), out, epi, want_resid=gated, want_gate=gated)
    # the activation's kink is a floating-point decision: take it from the GPU's pre
    rdx, rdb, rdr, rdg = ora.epilogue_bwd(dy, np_(pre) - b, b, act, gate, r)
    assert_close(np_(dx), rdx, FP32_TOL, "dx")
    assert_close(np_(dbias), rdb, FP32_TOL, "d_bias")
    if gated:
        assert_close(np_(dres), rdr, FP32_TOL, "d_resid")
        assert abs(float(dgate.item()) - rdg) <= FP32_TOL * max(1.0, abs(rdg))
    if act == "none" and not gated:   # the bias-only path (no dx): column sums of dy alone
        _, dbias2, _, _ = R.epilogue_bwd(padded(dy), out, epi, want_dx=False)
        assert_close(np_(dbias2), rdb, FP32_TOL, "d_bias (bias only)")


@pytest.mark.parametrize("D,wmode,dense", [(16, 1, False), (128, 0, True), (7, 1, True),
                                           (200, None, False)])
def test_max_aggregate_parity(R, ora, D, wmode, dense):
    """RNN_AGG_MAX: out and the arg-max bit-exact against the oracle
    (integer-valued features and weights in {0.5, 1, 2}: every product is exact in fp32, so
    both sides take each max / tie decision on the same values; ties go to the lowest join
    position), empty dense groups 0 / -1, and the backward to the arg-max rows only."""
    rng = np.random.default_rng(D + 3 * (wmode or 0))
    db = make_case(rng, n_s=300, n_t=200, n_e=6000, d=4)
    # T keys 100..139 get no join row (empty dense groups)
    db["e_dst"] = np.where(np.isin(db["e_dst"], db["t_key"][100:140]), db["t_key"][0], db["e_dst"])
    gi = R.build_join_index(cu(db["e_src"]), cu(db["e_dst"]), cu(db["s_key"]), cu(db["t_key"]),
                            dense_groups=dense)
    oi = ora.build_join_index(db["e_src"], db["e_dst"], db["s_key"], db["t_key"])
    z = rng.integers(-6, 7, (300, D)).astype(np.float32)
    n_w = oi["n_join_rows"] if wmode == 1 else len(db["e_src"])
    w = rng.choice([0.5, 1.0, 2.0], n_w).astype(np.float32) if wmode is not None else None
    q = R.make_query("src", "max", src=padded(z), edge=None if w is None else cu(w),
                     edge_mode=wmode or 0)
    out, am = R.join_aggregate_max_fwd(gi, q)
    ro, ram = ora.lja_max_fwd(oi, z, w, w_by_pos=wmode == 1)
    rows = np.searchsorted(np.sort(db["t_key"]), oi["group_key"]) if dense else np.arange(oi["n_groups"])
    np.testing.assert_array_equal(np_(out)[rows], ro)
    np.testing.assert_array_equal(np_(am)[rows], ram)
    if dense:
        empty = np.setdiff1d(np.arange(gi.n_groups), rows)
        assert len(empty) and np.all(np_(out)[empty] == 0) and np.all(np_(am)[empty] == -1)
    dO = rng.standard_normal((gi.n_groups, D)).astype(np.float32)
    d_src, d_edge = R.join_aggregate_max_bwd(gi, q, am, padded(dO), want_edge=w is not None)
    rdz, rdw = ora.lja_max_bwd(oi, z, ram, dO[rows], w, w_by_pos=wmode == 1)
    assert_close(np_(d_src), rdz, FP32_TOL, "d_src")
    if w is not None:
        assert_close(np_(d_edge).reshape(-1), rdw, FP32_TOL, "d_edge")


@pytest.mark.parametrize("heads,D,split", [(8, 128, 32), (8, 128, 0), (2, 16, 32)])
def test_union_fwd_and_accumulating_bwd(R, ora, heads, D, split):
    """rnn_join_aggregate_fwd_union: out = the relation's own aggregate (what its backward
    needs) and acc = beta acc + out in the same pass (fused for D = 128, one extra pass
    otherwise); rnn_join_aggregate_bwd_acc: d_dst = d_dst + gradient of a query shared by two
    relations -- the union of two relations into one target type against the oracle's sum."""
    rng = np.random.default_rng(D + heads + split)
    n_s, n_t = 400, 150
    scale = 1.0 / np.sqrt(D / heads)
    Q = (rng.standard_normal((n_t, D)) * 0.5).astype(np.float32)
    t_key = rng.permutation(n_t).astype(np.int64) * 3 + 1
    rels = []
    for r in range(2):
        s_key = rng.permutation(n_s).astype(np.int64) * 7 + r
        # every target once (dense groups = the compact ones) plus Zipf-distributed hub rows
        e_dst = np.concatenate([t_key, t_key[np.minimum(rng.zipf(1.5, 6000) - 1, n_t - 1)]])
        e_src = s_key[rng.integers(0, n_s, len(e_dst))]
        gi = R.build_join_index(cu(e_src), cu(e_dst), cu(s_key), cu(t_key), dense_groups=True,
                                rows_per_item=split)
        oi = ora.build_join_index(e_src, e_dst, s_key, t_key)
        assert gi.n_groups == oi["n_groups"] == n_t
        K = (rng.standard_normal((n_s, D)) * 0.5).astype(np.float32)
        M = rng.standard_normal((n_s, D)).astype(np.float32)
        rels.append((gi, oi, K, M))
    Qd = padded(Q)
    acc = padded(np.full((n_t, D), 123.0, np.float32))
    dQ = padded(np.full((n_t, D), -7.0, np.float32))
    dO = rng.standard_normal((n_t, D)).astype(np.float32)
    ref_acc = np.zeros((n_t, D))
    ref_dq = np.zeros((n_t, D))
    for r, (gi, oi, K, M) in enumerate(rels):
        q = R.make_query("src", "softmax", src=padded(M), src_key=padded(K), dst=Qd, heads=heads,
                         scale=scale)
        out = padded(np.zeros((n_t, D), np.float32))
        out, lse = R.join_aggregate_fwd_union(gi, q, out, acc, beta_acc=float(r))
        ref, _ = ora.lja_fwd(oi, agg="softmax", src=M, src_key=K, dst=Q, heads=heads, scale=scale)
        assert_close(np_(out), ref, FP32_TOL, f"out[{r}]")
        ref_acc += ref
        if D != 128:
            continue   # beta_dst = 1 is a D = 128 (source-major walker) feature
        ws = R.Workspace(torch.device("cuda"))
        _, bb = R.lja_workspace_size(gi, q)
        w = ws.get(bb)
        import ctypes as C
        R._check(R.lib().rnn_join_aggregate_bwd_acc(
            C.byref(gi.c), C.byref(q), R._ptr(out), out.stride(0), R._ptr(lse), R._ptr(padded(dO)),
            padded(dO).stride(0), None, None, None, R._ptr(dQ), float(r), R._ptr(w), w.numel(),
            R._stream()))
        gr = ora.lja_bwd(oi, dO, agg="softmax", src=M, src_key=K, dst=Q, heads=heads, scale=scale)
        ref_dq += gr["dst"]
    assert_close(np_(acc), ref_acc, FP32_TOL, "acc = O_0 + O_1")
    if D == 128:
        assert_close(np_(dQ), ref_dq, FP32_TOL, "dQ = dQ_0 + dQ_1")


def test_union_errors_and_empty(R):
    """beta_dst = 1 outside the source-major softmax backward is refused; MEAN unions are
    refused; an empty dense-group join leaves acc + 0 and an accumulated dQ untouched."""
    import ctypes as C
    keys = cu(np.arange(10, dtype=np.int64))
    gi = R.build_join_index(cu(np.zeros(0, np.int64)), cu(np.zeros(0, np.int64)), keys, keys,
                            dense_groups=True)
    M = padded(np.ones((10, 128), np.float32))
    q = R.make_query("src", "softmax", src=M, src_key=M, dst=M, heads=8, scale=1.0)
    acc = padded(np.full((10, 128), 5.0, np.float32))
    out = padded(np.zeros((10, 128), np.float32))
    out, lse = R.join_aggregate_fwd_union(gi, q, out, acc, beta_acc=1.0)
    assert np.all(np_(acc) == 5.0) and np.all(np_(out) == 0.0)
    dQ = padded(np.full((10, 128), 3.0, np.float32))
    dO = padded(np.ones((10, 128), np.float32))
    w = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    R._check(R.lib().rnn_join_aggregate_bwd_acc(
        C.byref(gi.c), C.byref(q), R._ptr(out), out.stride(0), R._ptr(lse), R._ptr(dO),
        dO.stride(0), None, None, None, R._ptr(dQ), 1.0, R._ptr(w), w.numel(), R._stream()))
    torch.cuda.synchronize()
    assert np.all(np_(dQ) == 3.0)
    with pytest.raises(R.RnnError):
        R.join_aggregate_fwd_union(gi, R.make_query("src", "mean", src=M), out, acc)
    # a non-empty SUM join with a group-side operand: d_dst accumulation is refused there
    e = cu(np.arange(10, dtype=np.int64))
    gs = R.build_join_index(e, e, keys, keys)
    qs = R.make_query("mul", "sum", src=M, dst=M)
    st = R.lib().rnn_join_aggregate_bwd_acc(
        C.byref(gs.c), C.byref(qs), None, 0, None, R._ptr(dO), dO.stride(0), None, None, None,
        R._ptr(dQ), 1.0, R._ptr(w), w.numel(), R._stream())
    assert st != 0
