"""CPU oracle (IEEE double) for RelaNN's lifted join-aggregate -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2605_24207_b200``) never imports it and shares no code with it.

This module is argument marshalling only: numpy arrays are widened to float64 (exactly)
and handed to ``oracle.c``, which evaluates the paper's definitions with plain loops.
See ``oracle.h`` for the citations of every function.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SRC2 = os.path.join(_HERE, "oracle_next.c")
_HDR = os.path.join(_HERE, "oracle.h")
_LIB = os.path.join(_HERE, "_build", "liboracle.so")

COMBINE = {"src": 0, "mul": 1, "add": 2, "concat": 3}
AGG = {"sum": 0, "mean": 1, "softmax": 2}


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, no fast-math) into oracle/_build/liboracle.so."""
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    stale = (not os.path.exists(_LIB)) or any(
        os.path.getmtime(p) > os.path.getmtime(_LIB) for p in (_SRC, _SRC2, _HDR))
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-Wall", "-Werror",
                               "-fno-fast-math", "-o", tmp, _SRC, _SRC2, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Operand(C.Structure):
    _fields_ = [("data", C.POINTER(C.c_double)), ("ld", C.c_int64), ("dim", C.c_int32),
                ("mode", C.c_int32)]


_lib = None
P64 = C.POINTER(C.c_int64)
P32 = C.POINTER(C.c_int32)
PD = C.POINTER(C.c_double)
POP = C.POINTER(_Operand)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.ora_epilogue_fwd.argtypes = [PD, C.c_int64, C.c_int, C.c_int64, PD, C.c_int, C.c_double,
                                       PD, C.c_int64, PD, C.c_int64]
        L.ora_epilogue_bwd.argtypes = [PD, PD, C.c_int64, C.c_int, PD, C.c_int, C.c_double, PD, PD,
                                       PD, PD, PD]
        L.ora_lja_max_fwd.argtypes = [P64, C.c_int64, P32, P32, PD, C.c_int64, C.c_int, PD, C.c_int,
                                      PD, C.c_int64, P64]
        L.ora_lja_max_bwd.argtypes = [P64, C.c_int64, P32, P32, PD, C.c_int64, C.c_int, PD, C.c_int,
                                      P64, PD, C.c_int64, C.c_int64, C.c_int64, PD, PD]
        L.ora_softmax_xent.argtypes = [PD, C.c_int64, C.c_int, C.c_int64, P64, PD, PD]
        L.ora_adam.argtypes = [PD, PD, PD, PD, C.c_int64, C.c_double, C.c_double, C.c_double,
                               C.c_double, C.c_double, C.c_int64]
        L.ora_rgcn_fwd.argtypes = [P64, C.c_int64, P32, P32, P32, P32, C.c_int, PD, C.c_int64,
                                   C.c_int, PD, C.c_int, PD, C.c_int64]
        L.ora_rgcn_bwd.argtypes = [P64, C.c_int64, P32, P32, P32, P32, C.c_int, PD, C.c_int64,
                                   C.c_int64, C.c_int, PD, C.c_int, PD, C.c_int64, PD, PD]
        L.ora_build_join_index.argtypes = [P64, P64, C.c_int64, P64, C.c_int64, P64, C.c_int64,
                                           C.c_int, P64, P64, P64, P64, P32, P32, P32, P64, P32]
        L.ora_lja_fwd.argtypes = [P64, C.c_int64, P32, P32, P32, C.c_int, C.c_int, C.c_int,
                                  C.c_double, POP, POP, POP, POP, P64, C.c_int64, PD, C.c_int64, PD]
        L.ora_lja_bwd.argtypes = [P64, C.c_int64, P32, P32, P32, C.c_int, C.c_int, C.c_int,
                                  C.c_double, POP, POP, POP, POP, PD, C.c_int64, C.c_int64,
                                  C.c_int64, C.c_int64, PD, PD, PD, PD]
        L.ora_group_softmax.argtypes = [P64, C.c_int64, C.c_int, PD, PD]
        L.ora_group_softmax_bwd.argtypes = [P64, C.c_int64, C.c_int, PD, PD, PD]
        L.ora_project.argtypes = [PD, C.c_int64, C.c_int64, C.c_int64, PD, C.c_int64, C.c_int64,
                                  PD, PD, C.c_int64]
        L.ora_project_bwd.argtypes = [PD, C.c_int64, C.c_int64, C.c_int64, PD, C.c_int64,
                                      C.c_int64, PD, C.c_int64, PD, PD, PD]
        L.ora_gcn_norm.argtypes = [P64, C.c_int64, P32, P32, C.c_int64, PD]
        L.ora_dhn_fwd.argtypes = [C.c_int, P64, C.c_int64, P32, P32, P64, C.c_int64,
                                  C.POINTER(PD), C.c_int64, C.c_int, P64, C.c_int64, PD, C.c_int64]
        L.ora_dhn_bwd.argtypes = [C.c_int, P64, C.c_int64, P32, P32, P64, C.c_int64,
                                  C.POINTER(PD), C.c_int64, C.c_int, PD, C.c_int64, C.POINTER(PD)]
        L.ora_hash_partition.argtypes = [P64, C.c_int64, C.c_int32, C.c_uint64, P32]
        L.ora_splitmix64.argtypes = [C.c_uint64]
        L.ora_splitmix64.restype = C.c_uint64
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


_ERR = {1: "duplicate key", 2: "bad argument", 3: "out of memory"}


def _check(rc: int) -> None:
    if rc != 0:
        raise OracleError(_ERR.get(rc, f"error {rc}"))


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _i64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int64)


def _i32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(-1, 1) if a.ndim == 1 else a


def build_join_index(e_src_key, e_dst_key, s_key=None, t_key=None, within_by_src_key=False):
    """O1: canonical join index of E(s,t) |><| S(s) |><| T(t), grouped by t.  Returns a dict."""
    e_dst_key = _i64(e_dst_key)
    e_src_key = _i64(e_src_key)
    s_key, t_key = _i64(s_key), _i64(t_key)
    n_e = len(e_dst_key)
    n_s = 0 if s_key is None else len(s_key)
    n_t = 0 if t_key is None else len(t_key)
    ub = max(n_e, 1)
    gp = np.zeros(ub + 1, np.int64); gk = np.zeros(ub, np.int64); gd = np.zeros(ub, np.int32)
    sr = np.zeros(ub, np.int32); er = np.zeros(ub, np.int32)
    sp = np.zeros(n_s + 1, np.int64); spos = np.zeros(ub, np.int32)
    nj, ng = C.c_int64(), C.c_int64()
    _check(lib().ora_build_join_index(_p(e_src_key, P64), _p(e_dst_key, P64), n_e,
                                      _p(s_key, P64), n_s, _p(t_key, P64), n_t,
                                      int(bool(within_by_src_key)), C.byref(nj), C.byref(ng),
                                      _p(gp, P64), _p(gk, P64), _p(gd, P32), _p(sr, P32),
                                      _p(er, P32), _p(sp, P64), _p(spos, P32)))
    nj, ng = nj.value, ng.value
    return {"n_join_rows": nj, "n_groups": ng, "n_src_rows": n_s, "n_dst_rows": n_t,
            "n_edge_rows": n_e,
            "group_ptr": gp[:ng + 1].copy(), "group_key": gk[:ng].copy(),
            "group_dst_row": gd[:ng].copy(), "src_row": sr[:nj].copy(), "edge_row": er[:nj].copy(),
            "src_ptr": sp.copy() if s_key is not None else None,
            "src_pos": spos[:nj].copy() if s_key is not None else None}


def _operand(a, mode=0):
    if a is None:
        return None, None
    a = _f64(a)
    op = _Operand(a.ctypes.data_as(PD), a.shape[1], a.shape[1], mode)
    return op, a


def _out_dim(combine, agg, src, key, edge, dst):
    if agg == "softmax" or combine == "src":
        return src.shape[1]
    if combine == "concat":
        return sum(x.shape[1] for x in (src, edge, dst) if x is not None)
    return max(x.shape[1] for x in (src, edge, dst) if x is not None)


def lja_fwd(idx, combine="src", agg="sum", src=None, src_key=None, edge=None, dst=None,
            heads=1, scale=1.0, edge_mode=0, dst_mode=0, src_mode=0, sel=None):
    """O2/O3: forward lifted join-aggregate in double.  Returns (out, lse or None)."""
    ops = [_operand(src, src_mode), _operand(src_key, src_mode), _operand(edge, edge_mode),
           _operand(dst, dst_mode)]
    arrs = [o[1] for o in ops]
    D = _out_dim(combine, agg, *arrs)
    sel = _i64(sel)
    n = idx["n_groups"] if sel is None else len(sel)
    out = np.zeros((max(n, 1), D), np.float64)
    lse = np.zeros((max(n, 1), heads), np.float64) if agg == "softmax" else None
    _check(lib().ora_lja_fwd(_p(idx["group_ptr"], P64), idx["n_groups"], _p(_i32(idx["src_row"]), P32),
                             _p(_i32(idx["edge_row"]), P32), _p(_i32(idx["group_dst_row"]), P32),
                             COMBINE[combine], AGG[agg], heads, scale,
                             *[C.byref(o[0]) if o[0] is not None else None for o in ops],
                             _p(sel, P64), 0 if sel is None else len(sel),
                             _p(out, PD), D, _p(lse, PD)))
    return out[:n], (lse[:n] if lse is not None else None)


def lja_bwd(idx, d_out, combine="src", agg="sum", src=None, src_key=None, edge=None, dst=None,
            heads=1, scale=1.0, edge_mode=0, dst_mode=0, src_mode=0, want=("src", "src_key", "edge", "dst")):
    """O4: backward.  Returns dict of full-size gradients (rows never referenced are 0)."""
    ops = [_operand(src, src_mode), _operand(src_key, src_mode), _operand(edge, edge_mode),
           _operand(dst, dst_mode)]
    arrs = [o[1] for o in ops]
    d_out = _f64(d_out)
    rows = [arrs[0].shape[0] if arrs[0] is not None else 0,
            arrs[1].shape[0] if arrs[1] is not None else 0,
            arrs[2].shape[0] if arrs[2] is not None else 0,
            arrs[3].shape[0] if arrs[3] is not None else 0]
    names = ["src", "src_key", "edge", "dst"]
    grads = [np.zeros((max(rows[i], 1), arrs[i].shape[1]), np.float64)
             if arrs[i] is not None and names[i] in want else None for i in range(4)]
    n_src_rows = rows[0] if arrs[0] is not None else rows[1]
    _check(lib().ora_lja_bwd(_p(idx["group_ptr"], P64), idx["n_groups"], _p(_i32(idx["src_row"]), P32),
                             _p(_i32(idx["edge_row"]), P32), _p(_i32(idx["group_dst_row"]), P32),
                             COMBINE[combine], AGG[agg], heads, scale,
                             *[C.byref(o[0]) if o[0] is not None else None for o in ops],
                             _p(d_out, PD), d_out.shape[1], n_src_rows, rows[2], rows[3],
                             *[_p(g, PD) for g in grads]))
    return {names[i]: (grads[i][:rows[i]] if grads[i] is not None else None) for i in range(4)}


def group_softmax(idx, scores, heads):
    s = np.ascontiguousarray(scores, np.float64).reshape(-1, heads)
    out = np.zeros_like(s)
    _check(lib().ora_group_softmax(_p(idx["group_ptr"], P64), idx["n_groups"], heads, _p(s, PD), _p(out, PD)))
    return out


def group_softmax_bwd(idx, probs, d_probs, heads):
    p = np.ascontiguousarray(probs, np.float64).reshape(-1, heads)
    dp = np.ascontiguousarray(d_probs, np.float64).reshape(-1, heads)
    out = np.zeros_like(p)
    _check(lib().ora_group_softmax_bwd(_p(idx["group_ptr"], P64), idx["n_groups"], heads,
                                       _p(p, PD), _p(dp, PD), _p(out, PD)))
    return out


def project(X, W, bias=None):
    """O5: Y = X W^T + b with W laid out [N, K] (torch.nn.Linear.weight)."""
    X, W = _f64(X), _f64(W)
    b = None if bias is None else np.ascontiguousarray(bias, np.float64)
    M, K = X.shape
    N = W.shape[0]
    Y = np.zeros((M, N), np.float64)
    _check(lib().ora_project(_p(X, PD), M, K, K, _p(W, PD), N, W.shape[1], _p(b, PD), _p(Y, PD), N))
    return Y


def project_bwd(X, W, dY, want_dx=True, want_db=True):
    X, W, dY = _f64(X), _f64(W), _f64(dY)
    M, K = X.shape
    N = W.shape[0]
    dX = np.zeros((M, K), np.float64) if want_dx else None
    dW = np.zeros((N, K), np.float64)
    db = np.zeros(N, np.float64) if want_db else None
    _check(lib().ora_project_bwd(_p(X, PD), M, K, K, _p(W, PD), N, W.shape[1], _p(dY, PD), N,
                                 _p(dX, PD), _p(dW, PD), _p(db, PD)))
    return dX, dW, db


def gcn_norm(idx, n_nodes):
    w = np.zeros(max(idx["n_join_rows"], 1), np.float64)
    _check(lib().ora_gcn_norm(_p(idx["group_ptr"], P64), idx["n_groups"], _p(_i32(idx["src_row"]), P32),
                              _p(_i32(idx["group_dst_row"]), P32), n_nodes, _p(w, PD)))
    return w[:idx["n_join_rows"]]


def _fptrs(f):
    arrs = [_f64(x) for x in f]
    ld = arrs[0].shape[1]
    assert all(a.shape == arrs[0].shape for a in arrs)
    ptrs = (PD * len(arrs))(*[a.ctypes.data_as(PD) for a in arrs])
    return arrs, ptrs, ld


def dhn_fwd(k, adj, node_key, f, sel=None):
    """O6: C_k(n) = f0(n) (.) sum over closed walks of prod f_i."""
    arrs, ptrs, d = _fptrs(f)
    nk = _i64(node_key)
    sel = _i64(sel)
    n = adj["n_groups"] if sel is None else len(sel)
    out = np.zeros((max(n, 1), d), np.float64)
    _check(lib().ora_dhn_fwd(k, _p(adj["group_ptr"], P64), adj["n_groups"], _p(_i32(adj["src_row"]), P32),
                             _p(_i32(adj["group_dst_row"]), P32), _p(nk, P64), len(nk), ptrs, d, d,
                             _p(sel, P64), 0 if sel is None else len(sel), _p(out, PD), d))
    return out[:n]


def dhn_bwd(k, adj, node_key, f, d_out):
    arrs, ptrs, d = _fptrs(f)
    nk = _i64(node_key)
    d_out = _f64(d_out)
    grads = [np.zeros((len(nk), d), np.float64) for _ in range(k)]
    gptrs = (PD * k)(*[g.ctypes.data_as(PD) for g in grads])
    _check(lib().ora_dhn_bwd(k, _p(adj["group_ptr"], P64), adj["n_groups"], _p(_i32(adj["src_row"]), P32),
                             _p(_i32(adj["group_dst_row"]), P32), _p(nk, P64), len(nk), ptrs, d, d,
                             _p(d_out, PD), d_out.shape[1], gptrs))
    return grads


def hash_partition(keys, P, seed):
    keys = _i64(keys)
    owner = np.zeros(max(len(keys), 1), np.int32)
    _check(lib().ora_hash_partition(_p(keys, P64), len(keys), P, seed, _p(owner, P32)))
    return owner[:len(keys)]


def splitmix64(x: int) -> int:
    return int(lib().ora_splitmix64(x))


# ---- SURVEY sec 8f rows (oracle_next.c) ----
ACT = {"none": 0, "relu": 1, "gelu": 2}


def epilogue_fwd(x, bias=None, act="none", gate=1.0, resid=None):
    """y = gate * act(x + b) + (1 - gate) * resid (resid None: act(x + b))."""
    x = _f64(x)
    rows, dim = x.shape
    y = np.zeros((max(rows, 1), dim))
    b = None if bias is None else _f64(np.asarray(bias).reshape(-1))
    r = None if resid is None else _f64(resid)
    _check(lib().ora_epilogue_fwd(_p(x, PD), rows, dim, dim, _p(b, PD), ACT[act], float(gate),
                                  _p(r, PD), dim, _p(y, PD), dim))
    return y[:rows]


def epilogue_bwd(dy, x, bias=None, act="none", gate=1.0, resid=None):
    """(dx, d_bias, d_resid, d_gate) of epilogue_fwd at x."""
    dy, x = _f64(dy), _f64(x)
    rows, dim = x.shape
    dx = np.zeros((max(rows, 1), dim))
    db = np.zeros(dim)
    b = None if bias is None else _f64(np.asarray(bias).reshape(-1))
    r = None if resid is None else _f64(resid)
    dr = np.zeros((max(rows, 1), dim)) if r is not None else None
    dg = np.zeros(1)
    _check(lib().ora_epilogue_bwd(_p(dy, PD), _p(x, PD), rows, dim, _p(b, PD), ACT[act],
                                  float(gate), _p(r, PD), _p(dx, PD), _p(db, PD), _p(dr, PD),
                                  _p(dg, PD) if r is not None else None))
    return dx[:rows], db, (None if dr is None else dr[:rows]), (float(dg[0]) if r is not None else None)


def lja_max_fwd(idx, z, w=None, w_by_pos=True):
    """MAX aggregate of w * z_s per group and column; returns (out [G, d], argmax [G, d])."""
    z = _f64(z)
    d = z.shape[1]
    G = idx["n_groups"]
    out = np.zeros((max(G, 1), d))
    am = np.zeros((max(G, 1), d), np.int64)
    wv = None if w is None else _f64(np.asarray(w).reshape(-1))
    _check(lib().ora_lja_max_fwd(_p(idx["group_ptr"], P64), G, _p(_i32(idx["src_row"]), P32),
                                 _p(_i32(idx["edge_row"]), P32), _p(z, PD), d, d, _p(wv, PD),
                                 1 if w_by_pos else 0, _p(out, PD), d, _p(am, P64)))
    return out[:G], am[:G]


def lja_max_bwd(idx, z, argmax, d_out, w=None, w_by_pos=True):
    """(d_z [n_src, d], d_w or None) of lja_max_fwd."""
    z, d_out = _f64(z), _f64(d_out)
    n_s, d = z.shape
    G = idx["n_groups"]
    wv = None if w is None else _f64(np.asarray(w).reshape(-1))
    dz = np.zeros((max(n_s, 1), d))
    n_w = 0 if wv is None else len(wv)
    dw = np.zeros(max(n_w, 1))
    am = np.ascontiguousarray(argmax, np.int64)
    _check(lib().ora_lja_max_bwd(_p(idx["group_ptr"], P64), G, _p(_i32(idx["src_row"]), P32),
                                 _p(_i32(idx["edge_row"]), P32), _p(z, PD), d, d, _p(wv, PD),
                                 1 if w_by_pos else 0, _p(am, P64), _p(d_out, PD), d, n_s, n_w,
                                 _p(dz, PD), _p(dw, PD) if wv is not None else None))
    return dz[:n_s], (dw[:n_w] if wv is not None else None)


def softmax_xent(logits, label):
    """(mean cross-entropy over rows with label >= 0, d_logits)."""
    x = _f64(logits)
    n, Cn = x.shape
    lab = np.ascontiguousarray(label, np.int64)
    loss = np.zeros(1)
    dl = np.zeros((max(n, 1), Cn))
    _check(lib().ora_softmax_xent(_p(x, PD), n, Cn, Cn, _p(lab, P64), _p(loss, PD), _p(dl, PD)))
    return float(loss[0]), dl[:n]


def adam(p, g, m, v, lr, t, b1=0.9, b2=0.999, eps=1e-8, wd=0.0):
    """One Adam step in place on float64 arrays p, m, v (returns them)."""
    for a in (p, m, v):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    gg = _f64(g)
    _check(lib().ora_adam(_p(p, PD), _p(gg, PD), _p(m, PD), _p(v, PD), p.size, lr, b1, b2, eps,
                          wd, t))
    return p, m, v


def rgcn_fwd(idx, rel, x, W):
    """R-GCN layer with per-join-row W_rel x_s (no pushdown): W [n_rel + 1, d_out, d_in]
    (W[0] self-loop); rel int per E row.  Returns out [G, d_out]."""
    x, W = _f64(x), np.ascontiguousarray(W, np.float64)
    n_rel = W.shape[0] - 1
    d_out, d_in = W.shape[1], W.shape[2]
    G = idx["n_groups"]
    out = np.zeros((max(G, 1), d_out))
    _check(lib().ora_rgcn_fwd(_p(idx["group_ptr"], P64), G, _p(_i32(idx["src_row"]), P32),
                              _p(_i32(idx["edge_row"]), P32), _p(_i32(idx["group_dst_row"]), P32),
                              _p(_i32(rel), P32), n_rel, _p(x, PD), x.shape[1], d_in, _p(W, PD),
                              d_out, _p(out, PD), d_out))
    return out[:G]


def rgcn_bwd(idx, rel, x, W, d_out):
    """(d_x [n, d_in], d_W [n_rel + 1, d_out, d_in]) of rgcn_fwd."""
    x, W, d_out = _f64(x), np.ascontiguousarray(W, np.float64), _f64(d_out)
    n_rel = W.shape[0] - 1
    do, di = W.shape[1], W.shape[2]
    dx = np.zeros((max(x.shape[0], 1), di))
    dW = np.zeros(W.shape)
    _check(lib().ora_rgcn_bwd(_p(idx["group_ptr"], P64), idx["n_groups"],
                              _p(_i32(idx["src_row"]), P32), _p(_i32(idx["edge_row"]), P32),
                              _p(_i32(idx["group_dst_row"]), P32), _p(_i32(rel), P32), n_rel,
                              _p(x, PD), x.shape[1], x.shape[0], di, _p(W, PD), do, _p(d_out, PD),
                              d_out.shape[1], _p(dx, PD), _p(dW, PD)))
    return dx[: x.shape[0]], dW
