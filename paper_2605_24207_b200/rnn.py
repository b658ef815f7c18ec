"""Thin Python binding of librnn.so (include/rnn.h): argument marshalling only.

Every step of the path runs in librnn.so's CUDA kernels; this module only turns torch CUDA
tensors into (pointer, size, stride) arguments, allocates caller-owned outputs/workspaces
with torch (PyTorch is device memory + streams here) and raises on a non-OK status.
There is no CPU fallback: if the extension or a GPU is missing, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# RNN_LIB: an alternative in-tree build of the same library (measurement variants built by
# profiles/build_variant.py); default the package's librnn.so
LIB_PATH = os.environ.get("RNN_LIB") or os.path.join(_HERE, "librnn.so")

# enums (include/rnn.h)
RNN_OK = 0
AGG = {"sum": 0, "mean": 1, "softmax": 2, "max": 3}
COMBINE = {"src": 0, "mul": 1, "add": 2, "concat": 3}
BY_ROW, BY_POSITION = 0, 1
IDX_VALIDATE, IDX_WITHIN_GROUP_BY_SRC_KEY, IDX_NO_TRANSPOSE, IDX_DENSE_GROUPS = 1, 2, 4, 8
PREC = {"tf32": 0, "3xtf32": 1, "bf16": 2}


class RnnError(RuntimeError):
    def __init__(self, status: int, name: str, detail: str):
        super().__init__(f"{name}: {detail}")
        self.status = status
        self.name = name


class JoinIndexC(C.Structure):
    _fields_ = [("n_edge_rows", C.c_int64), ("n_join_rows", C.c_int64), ("n_groups", C.c_int64),
                ("n_src_rows", C.c_int64), ("n_dst_rows", C.c_int64),
                ("group_ptr", C.c_void_p), ("group_key", C.c_void_p),
                ("group_dst_row", C.c_void_p), ("src_row", C.c_void_p), ("edge_row", C.c_void_p),
                ("pos_group", C.c_void_p),
                ("src_ptr", C.c_void_p), ("src_pos", C.c_void_p), ("src_group", C.c_void_p),
                ("src_seg", C.c_void_p),
                ("n_work", C.c_int64), ("work_ptr", C.c_void_p), ("work_seg", C.c_void_p),
                ("n_src_work", C.c_int64), ("src_work_ptr", C.c_void_p),
                ("src_work_seg", C.c_void_p)]


class OperandC(C.Structure):
    _fields_ = [("data", C.c_void_p), ("ld", C.c_int64), ("dim", C.c_int32), ("mode", C.c_int32)]


class QueryC(C.Structure):
    _fields_ = [("combine", C.c_int), ("agg", C.c_int), ("heads", C.c_int32), ("scale", C.c_float),
                ("src", OperandC), ("src_key", OperandC), ("edge", OperandC), ("dst", OperandC)]


class AdamC(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float)]


class EpilogueC(C.Structure):
    """rnn_epilogue: y = gate * act(x + bias) + (1 - gate) * resid."""
    _fields_ = [("bias", C.c_void_p), ("act", C.c_int32), ("gate", C.c_float),
                ("resid", C.c_void_p), ("ld_resid", C.c_int64), ("pre", C.c_void_p),
                ("ld_pre", C.c_int64)]


ACT = {"none": 0, "relu": 1, "gelu": 2}


def make_epilogue(bias=None, act="none", gate=1.0, resid=None, pre=None) -> EpilogueC:
    e = EpilogueC(None if bias is None else bias.data_ptr(), ACT[act], float(gate),
                  None if resid is None else resid.data_ptr(),
                  0 if resid is None else resid.stride(0),
                  None if pre is None else pre.data_ptr(), 0 if pre is None else pre.stride(0))
    e.keep = (bias, resid, pre)
    return e


_lib = None


def lib():
    """Load librnn.so (never builds implicitly; run __graft_entry__.build() first)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, sz = C.c_void_p, C.c_int64, C.c_int32, C.c_size_t
        L.rnn_status_string.restype = C.c_char_p
        L.rnn_status_string.argtypes = [C.c_int]
        L.rnn_last_error.restype = C.c_char_p
        L.rnn_abi_version.restype = C.c_int
        L.rnn_build_join_index.argtypes = [vp, vp, i64, vp, i64, vp, i64, C.c_int, i64,
                                           C.POINTER(JoinIndexC), vp, C.POINTER(sz), vp]
        L.rnn_lja_workspace_size.argtypes = [C.POINTER(JoinIndexC), C.POINTER(QueryC),
                                             C.POINTER(sz), C.POINTER(sz)]
        L.rnn_join_aggregate_fwd.argtypes = [C.POINTER(JoinIndexC), C.POINTER(QueryC), vp, i64,
                                             C.c_float, vp, vp, sz, vp]
        L.rnn_join_aggregate_bwd.argtypes = [C.POINTER(JoinIndexC), C.POINTER(QueryC), vp, i64, vp,
                                             vp, i64, vp, vp, vp, vp, vp, sz, vp]
        L.rnn_join_aggregate_fwd_union.argtypes = [C.POINTER(JoinIndexC), C.POINTER(QueryC), vp,
                                                   i64, vp, vp, i64, C.c_float, vp, sz, vp]
        L.rnn_join_aggregate_bwd_acc.argtypes = [C.POINTER(JoinIndexC), C.POINTER(QueryC), vp, i64,
                                                 vp, vp, i64, vp, vp, vp, vp, C.c_float, vp, sz, vp]
        L.rnn_group_softmax.argtypes = [C.POINTER(JoinIndexC), vp, i32, vp, vp]
        L.rnn_group_softmax_bwd.argtypes = [C.POINTER(JoinIndexC), vp, vp, i32, vp, vp]
        L.rnn_project.argtypes = [vp, i64, i32, i64, vp, i32, i64, vp, vp, i64, C.c_int, vp]
        L.rnn_project_bwd_workspace_size.argtypes = [i64, i32, i32, C.POINTER(sz)]
        L.rnn_project_bwd.argtypes = [vp, i64, i32, i64, vp, i32, i64, vp, i64, vp, i64, vp, vp,
                                      C.c_int, vp, sz, vp]
        L.rnn_project_bwd_relu.argtypes = [vp, i64, i32, i64, vp, i32, i64, vp, i64, vp, i64, vp,
                                           vp, vp, C.c_int, vp, sz, vp]
        L.rnn_stream_l2_window.argtypes = [vp, vp, sz, C.c_float]
        L.rnn_stream_l2_window.restype = C.c_int
        L.rnn_gcn_norm.argtypes = [C.POINTER(JoinIndexC), vp, vp, sz, vp]
        L.rnn_hash_partition.argtypes = [vp, i64, i32, C.c_uint64, vp, vp]
        L.rnn_accumulate.argtypes = [vp, i64, vp, i64, i64, i32, C.c_float, vp]
        L.rnn_accumulate.restype = C.c_int
        L.rnn_gather_rows.argtypes = [vp, i64, vp, i64, vp, i64, i32, vp]
        L.rnn_build_join_index_sel.argtypes = [vp, vp, vp, i64, vp, i64, vp, i64, C.c_int, i64,
                                               C.POINTER(JoinIndexC), vp, C.POINTER(sz), vp]
        L.rnn_select_mask.argtypes = [vp, i32, i64, i32, C.c_double, i32, vp, vp]
        L.rnn_build_join_index_sel.restype = C.c_int
        L.rnn_select_mask.restype = C.c_int
        L.rnn_scatter_add_rows.argtypes = [vp, i64, vp, i64, vp, i64, i32, vp]
        L.rnn_scatter_add_rows.restype = C.c_int
        L.rnn_softmax_xent_workspace_size.argtypes = [i64, C.POINTER(sz)]
        L.rnn_softmax_xent.argtypes = [vp, i64, i32, i64, vp, vp, vp, i64, vp, sz, vp]
        L.rnn_adam_tick.argtypes = [vp, vp]
        L.rnn_adam.argtypes = [vp, i64, i32, i64, vp, i64, vp, vp, C.POINTER(AdamC), vp, vp]
        for f in ("rnn_softmax_xent_workspace_size", "rnn_softmax_xent", "rnn_adam_tick", "rnn_adam"):
            getattr(L, f).restype = C.c_int
        L.rnn_join_aggregate_max_fwd.argtypes = [C.POINTER(JoinIndexC), C.POINTER(QueryC), vp, i64,
                                                 vp, i64, vp]
        L.rnn_join_aggregate_max_bwd.argtypes = [C.POINTER(JoinIndexC), C.POINTER(QueryC), vp, i64,
                                                 vp, i64, vp, vp, vp]
        L.rnn_join_aggregate_max_fwd.restype = C.c_int
        L.rnn_join_aggregate_max_bwd.restype = C.c_int
        L.rnn_join_aggregate_fwd_epi.argtypes = [C.POINTER(JoinIndexC), C.POINTER(QueryC),
                                                 C.POINTER(EpilogueC), vp, i64, vp, sz, vp]
        L.rnn_epilogue_fwd.argtypes = [vp, i64, i64, i32, C.POINTER(EpilogueC), vp, i64, vp]
        L.rnn_epilogue_bwd_workspace_size.argtypes = [i64, i32, C.POINTER(sz)]
        L.rnn_epilogue_bwd.argtypes = [vp, i64, vp, i64, i64, i32, C.POINTER(EpilogueC), vp, i64,
                                       vp, vp, i64, vp, vp, sz, vp]
        for f in ("rnn_join_aggregate_fwd_epi", "rnn_epilogue_fwd",
                  "rnn_epilogue_bwd_workspace_size", "rnn_epilogue_bwd"):
            getattr(L, f).restype = C.c_int
        L.rnn_gather_rows.restype = C.c_int
        L.rnn_dhn_workspace_size.argtypes = [C.POINTER(JoinIndexC), i32, i32, C.POINTER(sz)]
        L.rnn_dhn_fwd.argtypes = [C.POINTER(JoinIndexC), i32, C.POINTER(OperandC), vp, i64, vp, sz, vp]
        L.rnn_dhn_fwd_save.argtypes = [C.POINTER(JoinIndexC), i32, C.POINTER(OperandC), vp, i64,
                                       vp, i64, vp, sz, vp]
        L.rnn_dhn_bwd_saved.argtypes = [C.POINTER(JoinIndexC), i32, C.POINTER(OperandC), vp, i64,
                                        vp, i64, C.POINTER(vp), i64, C.c_uint32, vp, sz, vp]
        L.rnn_dhn_bwd.argtypes = [C.POINTER(JoinIndexC), i32, C.POINTER(OperandC), vp, i64,
                                  C.POINTER(vp), i64, vp, sz, vp]
        L.rnn_dhn_fwd_roots.argtypes = [C.POINTER(JoinIndexC), i32, C.POINTER(OperandC), vp, i64,
                                        vp, i64, vp, i64, vp, sz, vp]
        L.rnn_dhn_bwd_roots.argtypes = [C.POINTER(JoinIndexC), i32, C.POINTER(OperandC), vp, i64,
                                        vp, i64, vp, i64, C.POINTER(vp), i64, C.c_uint32, vp, sz, vp]
        L.rnn_dhn_count_workspace_size.argtypes = [C.POINTER(JoinIndexC), i32, C.POINTER(sz)]
        L.rnn_dhn_count.argtypes = [C.POINTER(JoinIndexC), i32, vp, vp, sz, vp]
        L.rnn_internal_dhn_stats.argtypes = [C.POINTER(C.c_ulonglong), C.c_int, C.c_int]
        L.rnn_gcn_norm_src_deg.argtypes = [C.POINTER(JoinIndexC), vp, vp, vp]
        L.rnn_group_sizes.argtypes = [C.POINTER(JoinIndexC), vp, vp]
        for f in ("rnn_dhn_workspace_size", "rnn_dhn_fwd", "rnn_dhn_bwd", "rnn_dhn_fwd_save",
                  "rnn_dhn_bwd_saved", "rnn_gcn_norm_src_deg", "rnn_dhn_count_workspace_size",
                  "rnn_dhn_count", "rnn_internal_dhn_stats", "rnn_dhn_fwd_roots",
                  "rnn_dhn_bwd_roots",
                  "rnn_group_sizes"):
            getattr(L, f).restype = C.c_int
        for f in ("rnn_build_join_index", "rnn_lja_workspace_size", "rnn_join_aggregate_fwd",
                  "rnn_join_aggregate_bwd", "rnn_group_softmax", "rnn_group_softmax_bwd",
                  "rnn_join_aggregate_fwd_union", "rnn_join_aggregate_bwd_acc",
                  "rnn_project", "rnn_project_bwd_workspace_size", "rnn_project_bwd",
                  "rnn_project_bwd_relu", "rnn_gcn_norm", "rnn_hash_partition"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _check(st: int):
    if st != RNN_OK:
        L = lib()
        raise RnnError(st, L.rnn_status_string(st).decode(), L.rnn_last_error().decode())


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _cuda(t, dtype, name):
    if t is None:
        return None
    if not (t.is_cuda and t.dtype == dtype):
        raise TypeError(f"{name} must be a CUDA {dtype} tensor")
    return t


def _ws(nbytes, device):
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


# ------------------------------------------------------------------------------------------
# A1 join index
# ------------------------------------------------------------------------------------------
class JoinIndex:
    """Key-grouped CSR of the join rows of E(s,t) |><| S(s) |><| T(t), grouped by t.

    Immutable once built (content caching): reuse it for every iteration.  Arrays are torch
    tensors owned by this object; ``c`` is the POD handed to the C ABI.
    """

    def __init__(self, c: JoinIndexC, arrays: dict):
        self.c = c
        self.arrays = arrays
        for k, v in arrays.items():
            setattr(self, k, v)

    @property
    def n_join_rows(self):
        return self.c.n_join_rows

    @property
    def n_groups(self):
        return self.c.n_groups

    @property
    def n_src_rows(self):
        return self.c.n_src_rows

    @property
    def n_dst_rows(self):
        return self.c.n_dst_rows


def build_join_index(e_src_key, e_dst_key, src_key=None, dst_key=None, *, validate=False,
                     within_group_by_src_key=False, transpose=True, dense_groups=False,
                     rows_per_item=0, stream=None, e_mask=None) -> JoinIndex:
    """rnn_build_join_index: phase 1 (sizes, SYNC), allocate, phase 2 (fill).  e_mask (uint8
    per E row, device): the selection sigma(E) pushed into the probe (rnn_build_join_index_sel)."""
    L = lib()
    e_dst_key = _cuda(e_dst_key, torch.int64, "e_dst_key").contiguous()
    dev = e_dst_key.device
    e_src_key = None if e_src_key is None else _cuda(e_src_key, torch.int64, "e_src_key").contiguous()
    src_key = None if src_key is None else _cuda(src_key, torch.int64, "src_key").contiguous()
    dst_key = None if dst_key is None else _cuda(dst_key, torch.int64, "dst_key").contiguous()
    flags = (IDX_VALIDATE if validate else 0) | (IDX_WITHIN_GROUP_BY_SRC_KEY if within_group_by_src_key else 0) \
        | (0 if transpose else IDX_NO_TRANSPOSE) | (IDX_DENSE_GROUPS if dense_groups else 0)
    n_e = e_dst_key.numel()
    n_s = 0 if src_key is None else src_key.numel()
    n_t = 0 if dst_key is None else dst_key.numel()
    # an EMPTY relation is not an ABSENT one: hand the C ABI a non-NULL pointer for it
    if src_key is not None and n_s == 0:
        src_key = torch.zeros(1, dtype=torch.int64, device=dev)
    if dst_key is not None and n_t == 0:
        dst_key = torch.zeros(1, dtype=torch.int64, device=dev)
    if e_src_key is not None and n_e == 0:
        e_src_key = torch.zeros(1, dtype=torch.int64, device=dev)
    if n_e == 0:
        e_dst_key = torch.zeros(1, dtype=torch.int64, device=dev)
    idx = JoinIndexC()
    wsb = C.c_size_t(0)
    if e_mask is not None:
        e_mask = _cuda(e_mask, torch.uint8, "e_mask").contiguous()
        if n_e == 0:
            e_mask = torch.zeros(1, dtype=torch.uint8, device=dev)
        args = (_ptr(e_src_key), _ptr(e_dst_key), _ptr(e_mask), n_e, _ptr(src_key), n_s,
                _ptr(dst_key), n_t, flags, rows_per_item)
        fn = L.rnn_build_join_index_sel
    else:
        args = (_ptr(e_src_key), _ptr(e_dst_key), n_e, _ptr(src_key), n_s, _ptr(dst_key), n_t,
                flags, rows_per_item)
        fn = L.rnn_build_join_index
    _check(fn(*args, C.byref(idx), None, C.byref(wsb), _stream(stream)))
    ws = _ws(wsb.value, dev)
    _check(fn(*args, C.byref(idx), _ptr(ws), C.byref(wsb), _stream(stream)))
    nj, ng = idx.n_join_rows, idx.n_groups
    i64 = dict(dtype=torch.int64, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    has_t = src_key is not None and transpose
    arrays = {
        "group_ptr": torch.empty(ng + 1, **i64), "group_key": torch.empty(max(ng, 1), **i64),
        "group_dst_row": torch.empty(max(ng, 1), **i32), "src_row": torch.empty(max(nj, 1), **i32),
        "edge_row": torch.empty(max(nj, 1), **i32), "pos_group": torch.empty(max(nj, 1), **i32),
        "work_ptr": torch.empty(idx.n_work + 1, **i64),
        "work_seg": torch.empty(max(idx.n_work, 1), **i32),
    }
    if has_t:
        arrays.update({"src_ptr": torch.empty(n_s + 1, **i64), "src_pos": torch.empty(max(nj, 1), **i32),
                       "src_group": torch.empty(max(nj, 1), **i32),
                       "src_seg": torch.empty(max(nj, 1), **i32),
                       "src_work_ptr": torch.empty(idx.n_src_work + 1, **i64),
                       "src_work_seg": torch.empty(max(idx.n_src_work, 1), **i32)})
    for k, v in arrays.items():
        setattr(idx, k, v.data_ptr())
    _check(fn(*args, C.byref(idx), _ptr(ws), C.byref(wsb), _stream(stream)))
    arrays["group_key"] = arrays["group_key"][:ng]
    arrays["group_dst_row"] = arrays["group_dst_row"][:ng]
    for k in ("src_row", "edge_row", "pos_group", "src_pos", "src_group", "src_seg"):
        if k in arrays:
            arrays[k] = arrays[k][:nj]
    return JoinIndex(idx, arrays)


# ------------------------------------------------------------------------------------------
# A3/A4/A5 lifted join-aggregate
# ------------------------------------------------------------------------------------------
def _operand(t, mode=BY_ROW):
    if t is None:
        return OperandC(None, 0, 0, 0)
    t = _cuda(t, torch.float32, "operand")
    if t.dim() == 1:
        t = t.view(-1, 1)
    if t.stride(1) != 1:
        raise ValueError("operands must be row-major (stride(1) == 1)")
    return OperandC(t.data_ptr(), t.stride(0), t.shape[1], mode)


def make_query(combine="src", agg="sum", src=None, src_key=None, edge=None, dst=None, heads=1,
               scale=1.0, edge_mode=BY_ROW, dst_mode=BY_ROW) -> QueryC:
    q = QueryC(COMBINE[combine], AGG[agg], heads, scale, _operand(src), _operand(src_key),
               _operand(edge, edge_mode), _operand(dst, dst_mode))
    # the struct holds raw pointers: keep the operand tensors alive as long as the query
    q.keep = (src, src_key, edge, dst)
    return q


def out_width(q: QueryC) -> int:
    if q.agg == AGG["softmax"] or q.combine == COMBINE["src"]:
        return q.src.dim
    dims = [o.dim for o in (q.src, q.edge, q.dst) if o.data]
    return sum(dims) if q.combine == COMBINE["concat"] else max(dims)


class Workspace:
    """Grow-only device scratch buffer (reused across calls; never shared by concurrent calls)."""

    def __init__(self, device="cuda"):
        self.buf = None
        self.device = device

    def get(self, nbytes):
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=self.device)
        return self.buf


def lja_workspace_size(idx: JoinIndex, q: QueryC):
    f, b = C.c_size_t(0), C.c_size_t(0)
    _check(lib().rnn_lja_workspace_size(C.byref(idx.c), C.byref(q), C.byref(f), C.byref(b)))
    return f.value, b.value


def join_aggregate_fwd(idx: JoinIndex, q: QueryC, out=None, beta=0.0, lse=None, ws=None,
                       stream=None, ld_out=None):
    dev = idx.group_ptr.device
    D = out_width(q)
    if out is None:
        ldo = ld_out or (D + 3) // 4 * 4
        out = torch.empty(idx.n_groups, ldo, dtype=torch.float32, device=dev)[:, :D]
    if q.agg == AGG["softmax"] and lse is None:
        lse = torch.empty(max(idx.n_groups, 1), q.heads, dtype=torch.float32, device=dev)
    fb, _ = lja_workspace_size(idx, q)
    w = ws.get(fb) if ws is not None else _ws(fb, dev)
    _check(lib().rnn_join_aggregate_fwd(C.byref(idx.c), C.byref(q), _ptr(out), out.stride(0),
                                        float(beta), _ptr(lse), _ptr(w), w.numel(), _stream(stream)))
    return (out, lse) if q.agg == AGG["softmax"] else out


def join_aggregate_fwd_union(idx: JoinIndex, q: QueryC, out, acc, beta_acc=0.0, lse=None,
                             ws=None, stream=None):
    """out = the aggregate (as join_aggregate_fwd, beta 0) and, in the same pass,
    acc = beta_acc * acc + out (rnn_join_aggregate_fwd_union: HGT's union over relations that
    keeps each relation's own output for its backward)."""
    dev = idx.group_ptr.device
    if q.agg == AGG["softmax"] and lse is None:
        lse = torch.empty(max(idx.n_groups, 1), q.heads, dtype=torch.float32, device=dev)
    fb, _ = lja_workspace_size(idx, q)
    w = ws.get(fb) if ws is not None else _ws(fb, dev)
    _check(lib().rnn_join_aggregate_fwd_union(C.byref(idx.c), C.byref(q), _ptr(out), out.stride(0),
                                              _ptr(lse), _ptr(acc), acc.stride(0), float(beta_acc),
                                              _ptr(w), w.numel(), _stream(stream)))
    return (out, lse) if q.agg == AGG["softmax"] else out


def _grad_like(op: OperandC, rows, dev):
    if not op.data:
        return None
    return torch.empty(max(rows, 1), op.ld, dtype=torch.float32, device=dev)[:rows, :op.dim]


def join_aggregate_bwd(idx: JoinIndex, q: QueryC, d_out, *, out=None, lse=None, want_src=True,
                       want_src_key=True, want_edge=True, want_dst=True, n_src_rows=None,
                       n_edge_rows=None, n_dst_rows=None, ws=None, stream=None):
    """Returns dict of gradient tensors (same ld as the operands; rows never referenced = 0)."""
    dev = idx.group_ptr.device
    ns = idx.n_src_rows if n_src_rows is None else n_src_rows
    ne = (idx.c.n_edge_rows if q.edge.mode == BY_ROW else idx.n_join_rows) if n_edge_rows is None else n_edge_rows
    nt = (idx.n_dst_rows if q.dst.mode == BY_ROW else idx.n_groups) if n_dst_rows is None else n_dst_rows
    g = {"src": _grad_like(q.src, ns, dev) if want_src else None,
         "src_key": _grad_like(q.src_key, ns, dev) if want_src_key else None,
         "edge": _grad_like(q.edge, ne, dev) if want_edge else None,
         "dst": _grad_like(q.dst, nt, dev) if want_dst else None}
    _, bb = lja_workspace_size(idx, q)
    w = ws.get(bb) if ws is not None else _ws(bb, dev)
    _check(lib().rnn_join_aggregate_bwd(C.byref(idx.c), C.byref(q), _ptr(out),
                                        0 if out is None else out.stride(0), _ptr(lse), _ptr(d_out),
                                        d_out.stride(0), _ptr(g["src"]), _ptr(g["src_key"]),
                                        _ptr(g["edge"]), _ptr(g["dst"]), _ptr(w), w.numel(),
                                        _stream(stream)))
    return g


def group_softmax(idx: JoinIndex, scores, heads, stream=None):
    scores = _cuda(scores, torch.float32, "scores").contiguous()
    probs = torch.empty_like(scores)
    _check(lib().rnn_group_softmax(C.byref(idx.c), _ptr(scores), heads, _ptr(probs), _stream(stream)))
    return probs


def group_softmax_bwd(idx: JoinIndex, probs, d_probs, heads, stream=None):
    ds = torch.empty_like(probs)
    _check(lib().rnn_group_softmax_bwd(C.byref(idx.c), _ptr(probs.contiguous()),
                                       _ptr(d_probs.contiguous()), heads, _ptr(ds), _stream(stream)))
    return ds


# ------------------------------------------------------------------------------------------
# A2 projection
# ------------------------------------------------------------------------------------------
# tensor-core work of the projections, counted when a dict is installed here (bench.py's
# projection roofline): {"proj_fwd": flops, "proj_bwd": flops}, MMA flops as issued (3xTF32
# issues three tf32 products per term)
FLOP_COUNTER = None
_MMAS = {"tf32": 1, "3xtf32": 3, "bf16": 1}


def _count(kind, flops):
    if FLOP_COUNTER is not None:
        FLOP_COUNTER[kind] = FLOP_COUNTER.get(kind, 0) + flops


def project(X, W, bias=None, out=None, prec="3xtf32", stream=None):
    """Y = X W^T + b on tcgen05 (W is [N, K] like nn.Linear.weight)."""
    M, K = X.shape
    N = W.shape[0]
    _count("proj_fwd", 2 * M * K * N * _MMAS[prec])
    if out is None:
        out = torch.empty(M, (N + 3) // 4 * 4, dtype=torch.float32, device=X.device)[:, :N]
    _check(lib().rnn_project(_ptr(X), M, K, X.stride(0), _ptr(W), N, W.stride(0), _ptr(bias),
                             _ptr(out), out.stride(0), PREC[prec], _stream(stream)))
    return out


def project_bwd(X, W, dY, want_dx=True, want_db=False, prec="3xtf32", ws=None, stream=None,
                dx_out=None, dw_out=None, relu_in=False, d_in_bias=None):
    """dX = dY W, dW = dY^T X, db = colsum(dY).  relu_in: X is a ReLU epilogue's output, dX
    becomes the gradient at that epilogue's input (dY W) * [X > 0] and d_in_bias (a [K]
    tensor, optional) its bias gradient (rnn_project_bwd_relu)."""
    M, K = X.shape
    N = W.shape[0]
    dev = X.device
    _count("proj_bwd", 2 * M * K * N * _MMAS[prec] * (2 if want_dx else 1))
    dX = None
    if want_dx:
        dX = dx_out if dx_out is not None else torch.empty(M, (K + 3) // 4 * 4, dtype=torch.float32, device=dev)[:, :K]
    dW = dw_out if dw_out is not None else torch.empty(N, K, dtype=torch.float32, device=dev)
    db = torch.empty(N, dtype=torch.float32, device=dev) if want_db else None
    nb = C.c_size_t(0)
    _check(lib().rnn_project_bwd_workspace_size(M, K, N, C.byref(nb)))
    w = ws.get(nb.value) if ws is not None else _ws(nb.value, dev)
    if relu_in:
        if dX is None:
            raise ValueError("relu_in needs dX (want_dx=True)")
        _check(lib().rnn_project_bwd_relu(
            _ptr(X), M, K, X.stride(0), _ptr(W), N, W.stride(0), _ptr(dY), dY.stride(0), _ptr(dX),
            dX.stride(0), _ptr(dW), _ptr(db), _ptr(d_in_bias), PREC[prec], _ptr(w), w.numel(),
            _stream(stream)))
        return dX, dW, db
    _check(lib().rnn_project_bwd(_ptr(X), M, K, X.stride(0), _ptr(W), N, W.stride(0), _ptr(dY),
                                 dY.stride(0), _ptr(dX), 0 if dX is None else dX.stride(0), _ptr(dW),
                                 _ptr(db), PREC[prec], _ptr(w), w.numel(), _stream(stream)))
    return dX, dW, db


# ------------------------------------------------------------------------------------------
# helpers
# ------------------------------------------------------------------------------------------
def stream_l2_window(t=None, hit_ratio=1.0, stream=None):
    """Persisting-L2 window over tensor t on the stream (rnn_stream_l2_window); t=None clears."""
    if t is None:
        _check(lib().rnn_stream_l2_window(_stream(stream), None, 0, 0.0))
    else:
        span = (1 + sum((n - 1) * st for n, st in zip(t.shape, t.stride()))) * t.element_size()
        _check(lib().rnn_stream_l2_window(_stream(stream), _ptr(t), span, float(hit_ratio)))


def gcn_norm(idx: JoinIndex, stream=None):
    dev = idx.group_ptr.device
    w = torch.empty(max(idx.n_join_rows, 1), dtype=torch.float32, device=dev)
    nb = 4 * idx.n_dst_rows + 256
    ws = _ws(nb, dev)
    _check(lib().rnn_gcn_norm(C.byref(idx.c), _ptr(w), _ptr(ws), ws.numel(), _stream(stream)))
    return w[:idx.n_join_rows]


def gcn_norm_src_deg(idx: JoinIndex, src_deg, stream=None):
    """w[p] = src_deg[src_row[p]]^-1/2 |g|^-1/2 (sharded GCN: src_deg all-gathered)."""
    src_deg = _cuda(src_deg, torch.int32, "src_deg").contiguous()
    w = torch.empty(max(idx.n_join_rows, 1), dtype=torch.float32, device=src_deg.device)
    _check(lib().rnn_gcn_norm_src_deg(C.byref(idx.c), _ptr(src_deg), _ptr(w), _stream(stream)))
    return w[:idx.n_join_rows]


def group_sizes(idx: JoinIndex, out=None, stream=None):
    dev = idx.group_ptr.device
    out = out if out is not None else torch.empty(max(idx.n_groups, 1), dtype=torch.int32, device=dev)
    _check(lib().rnn_group_sizes(C.byref(idx.c), _ptr(out), _stream(stream)))
    return out


def hash_partition(keys, P, seed, stream=None):
    keys = _cuda(keys, torch.int64, "keys").contiguous()
    owner = torch.empty(keys.numel(), dtype=torch.int32, device=keys.device)
    _check(lib().rnn_hash_partition(_ptr(keys), keys.numel(), P, seed, _ptr(owner), _stream(stream)))
    return owner


def accumulate(y, x, beta=1.0, stream=None):
    """y = beta * y + x (union over relations of per-relation results)."""
    rows, cols = x.shape
    _check(lib().rnn_accumulate(_ptr(y), y.stride(0), _ptr(x), x.stride(0), rows, cols,
                                float(beta), _stream(stream)))
    return y


def gather_rows(y, x, idx, stream=None):
    """y[i] = x[idx[i]] (0 where idx[i] < 0), idx int32 on the device (rnn_gather_rows)."""
    n, cols = y.shape
    _check(lib().rnn_gather_rows(_ptr(y), y.stride(0), _ptr(x), x.stride(0), _ptr(idx), n, cols,
                                 _stream(stream)))
    return y


# ------------------------------------------------------------------------------------------
# A6 DHN closed-walk aggregates
# ------------------------------------------------------------------------------------------
def dhn_workspace_size(adj: JoinIndex, k, d):
    b = C.c_size_t(0)
    _check(lib().rnn_dhn_workspace_size(C.byref(adj.c), k, d, C.byref(b)))
    return b.value


def _dhn_ops(f):
    ops = (OperandC * len(f))(*[_operand(t) for t in f])
    return ops


def dhn_fwd(adj: JoinIndex, k, f, out=None, ws=None, stream=None, walk_sum=None, roots=None):
    """C_k per root (group order) of the closed-walk rule; f = [f0 (or None), f1, ..., f_{k-1}]
    by node row (rnn_dhn_fwd).  walk_sum [n_groups, >= d]: also save the walk sum before the
    root factor for dhn_bwd (rnn_dhn_fwd_save).  roots: int32 device tensor of group ids --
    only those roots are computed (rnn_dhn_fwd_roots)."""
    assert len(f) == k
    dev = adj.group_ptr.device
    d = f[1].shape[1]
    if out is None:
        out = torch.empty(max(adj.n_groups, 1), (d + 3) // 4 * 4, dtype=torch.float32, device=dev)[:adj.n_groups, :d]
    nb = dhn_workspace_size(adj, k, d)
    w = ws.get(nb) if ws is not None else _ws(nb, dev)
    if roots is not None:
        _check(lib().rnn_dhn_fwd_roots(C.byref(adj.c), k, _dhn_ops(f), _ptr(roots), roots.numel(),
                                       _ptr(out), out.stride(0), _ptr(walk_sum),
                                       0 if walk_sum is None else walk_sum.stride(0), _ptr(w),
                                       w.numel(), _stream(stream)))
        return out
    if walk_sum is not None:
        _check(lib().rnn_dhn_fwd_save(C.byref(adj.c), k, _dhn_ops(f), _ptr(out), out.stride(0),
                                      _ptr(walk_sum), walk_sum.stride(0), _ptr(w), w.numel(),
                                      _stream(stream)))
        return out
    _check(lib().rnn_dhn_fwd(C.byref(adj.c), k, _dhn_ops(f), _ptr(out), out.stride(0), _ptr(w),
                             w.numel(), _stream(stream)))
    return out


DHN_SYMMETRIC_EDGE = 1


def dhn_bwd(adj: JoinIndex, k, f, d_out, want=None, d_f=None, ws=None, stream=None,
            walk_sum=None, symmetric=False, roots=None):
    """[d f0, ..., d f_{k-1}] by node row (rnn_dhn_bwd); want[i] False -> None.  walk_sum: the
    forward's saved walk sum (d f0 without a walk launch, rnn_dhn_bwd_saved)."""
    dev = adj.group_ptr.device
    d = f[1].shape[1]
    n = adj.n_src_rows
    want = want or [True] * k
    if d_f is None:
        d_f = [torch.empty(max(n, 1), (d + 3) // 4 * 4, dtype=torch.float32, device=dev)[:n, :d]
               if want[i] else None for i in range(k)]
    lds = {t.stride(0) for t in d_f if t is not None}
    if len(lds) > 1:
        raise ValueError("all d_f tensors must share one ld")
    ld = lds.pop() if lds else d
    ptrs = (C.c_void_p * k)(*[None if t is None else t.data_ptr() for t in d_f])
    nb = dhn_workspace_size(adj, k, d)
    w = ws.get(nb) if ws is not None else _ws(nb, dev)
    if roots is not None:
        _check(lib().rnn_dhn_bwd_roots(C.byref(adj.c), k, _dhn_ops(f), _ptr(roots), roots.numel(),
                                       _ptr(d_out), d_out.stride(0), _ptr(walk_sum),
                                       0 if walk_sum is None else walk_sum.stride(0), ptrs, ld,
                                       DHN_SYMMETRIC_EDGE if symmetric else 0, _ptr(w), w.numel(),
                                       _stream(stream)))
        return d_f
    if walk_sum is not None:
        _check(lib().rnn_dhn_bwd_saved(C.byref(adj.c), k, _dhn_ops(f), _ptr(d_out),
                                       d_out.stride(0), _ptr(walk_sum), walk_sum.stride(0), ptrs,
                                       ld, DHN_SYMMETRIC_EDGE if symmetric else 0, _ptr(w),
                                       w.numel(), _stream(stream)))
        return d_f
    if symmetric:
        raise ValueError("symmetric=True needs walk_sum or roots (rnn_dhn_bwd takes no flags)")
    _check(lib().rnn_dhn_bwd(C.byref(adj.c), k, _dhn_ops(f), _ptr(d_out), d_out.stride(0), ptrs,
                             ld, _ptr(w), w.numel(), _stream(stream)))
    return d_f


def dhn_count(adj: JoinIndex, k, out=None, stream=None):
    """Exact closed-walk counts C_k(n) (all operands 1) per root in group order, int64
    (rnn_dhn_count): (A^k)_nn of the Edge relation, with multiplicity."""
    dev = adj.group_ptr.device
    if out is None:
        out = torch.empty(max(adj.n_groups, 1), dtype=torch.int64, device=dev)[:adj.n_groups]
    b = C.c_size_t(0)
    _check(lib().rnn_dhn_count_workspace_size(C.byref(adj.c), k, C.byref(b)))
    w = _ws(b.value, dev)
    _check(lib().rnn_dhn_count(C.byref(adj.c), k, _ptr(out), _ptr(w), w.numel(), _stream(stream)))
    return out


DHN_PATHS = ("c3_roots", "c3_mark_roots", "c4_roots", "c4_passes", "c4_chunked_passes",
             "c4_long_runs", "c4_long_overflow", "c4_partitioned_roots", "c4_value_overflow")


def dhn_path_counters(reset=False):
    """Internal: which code paths the DHN walk kernels took since the last reset (SYNC)."""
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 16)()
    if lib().rnn_internal_dhn_stats(buf, 1 if reset else 0, 0) != 0:
        raise RuntimeError("rnn_internal_dhn_stats failed")
    return dict(zip(DHN_PATHS, [int(x) for x in buf[:len(DHN_PATHS)]]))


# ------------------------------------------------------------------------------------------
# node epilogues
# ------------------------------------------------------------------------------------------
def join_aggregate_fwd_epi(idx: JoinIndex, q: QueryC, epi: EpilogueC, out=None, ws=None,
                           stream=None):
    """The SUM/MEAN LJA with the epilogue fused into its store (rnn_join_aggregate_fwd_epi)."""
    dev = idx.group_ptr.device
    D = out_width(q)
    if out is None:
        out = torch.empty(max(idx.n_groups, 1), (D + 3) // 4 * 4, dtype=torch.float32, device=dev)[: idx.n_groups, :D]
    fb, _ = lja_workspace_size(idx, q)
    w = ws.get(fb) if ws is not None else _ws(fb, dev)
    _check(lib().rnn_join_aggregate_fwd_epi(C.byref(idx.c), C.byref(q), C.byref(epi), _ptr(out),
                                            out.stride(0), _ptr(w), w.numel(), _stream(stream)))
    return out


def epilogue_fwd(x, epi: EpilogueC, out=None, stream=None):
    rows, dim = x.shape
    y = out if out is not None else torch.empty_like(x)
    _check(lib().rnn_epilogue_fwd(_ptr(x), x.stride(0), rows, dim, C.byref(epi), _ptr(y),
                                  y.stride(0), _stream(stream)))
    return y


def epilogue_bwd(dy, y, epi: EpilogueC, dx=None, want_bias=True, want_resid=False,
                 want_gate=False, ws=None, stream=None, db_out=None, want_dx=True):
    """(dx, d_bias, d_resid, d_gate) of the epilogue (rnn_epilogue_bwd); y = the forward output.
    want_dx=False skips dx (e.g. the bias-only epilogue, where dx would be a copy of dy)."""
    rows, dim = dy.shape
    dev = dy.device
    dx = dx if dx is not None else (torch.empty_like(dy) if want_dx else None)
    db = db_out if db_out is not None else (
        torch.empty(dim, dtype=torch.float32, device=dev) if want_bias else None)
    dr = torch.empty_like(dy) if want_resid else None
    dg = torch.empty(1, dtype=torch.float32, device=dev) if want_gate else None
    nb = C.c_size_t(0)
    _check(lib().rnn_epilogue_bwd_workspace_size(rows, dim, C.byref(nb)))
    w = ws.get(nb.value) if ws is not None else _ws(nb.value, dev)
    _check(lib().rnn_epilogue_bwd(_ptr(dy), dy.stride(0), _ptr(y), 0 if y is None else y.stride(0),
                                  rows, dim, C.byref(epi), _ptr(dx),
                                  dim if dx is None else dx.stride(0), _ptr(db),
                                  _ptr(dr), 0 if dr is None else dr.stride(0), _ptr(dg), _ptr(w),
                                  w.numel(), _stream(stream)))
    return dx, db, dr, dg


def join_aggregate_max_fwd(idx: JoinIndex, q: QueryC, out=None, argmax=None, stream=None):
    """MAX aggregate (rnn_join_aggregate_max_fwd): (out [G, D], argmax int32 [G, D])."""
    dev = idx.group_ptr.device
    D = q.src.dim
    G = idx.n_groups
    if out is None:
        out = torch.empty(max(G, 1), (D + 3) // 4 * 4, dtype=torch.float32, device=dev)[:G, :D]
    if argmax is None:
        argmax = torch.empty(max(G, 1), D, dtype=torch.int32, device=dev)[:G]
    _check(lib().rnn_join_aggregate_max_fwd(C.byref(idx.c), C.byref(q), _ptr(out), out.stride(0),
                                            _ptr(argmax), argmax.stride(0), _stream(stream)))
    return out, argmax


def join_aggregate_max_bwd(idx: JoinIndex, q: QueryC, argmax, d_out, want_edge=False,
                           stream=None):
    """(d_src, d_edge) of the MAX aggregate (rnn_join_aggregate_max_bwd)."""
    dev = idx.group_ptr.device
    d_src = _grad_like(q.src, idx.n_src_rows, dev)
    ne = idx.c.n_edge_rows if q.edge.mode == BY_ROW else idx.n_join_rows
    d_edge = _grad_like(q.edge, ne, dev) if want_edge else None
    _check(lib().rnn_join_aggregate_max_bwd(C.byref(idx.c), C.byref(q), _ptr(argmax),
                                            argmax.stride(0), _ptr(d_out), d_out.stride(0),
                                            _ptr(d_src), _ptr(d_edge), _stream(stream)))
    return d_src, d_edge


# ------------------------------------------------------------------------------------------
# training step
# ------------------------------------------------------------------------------------------
def softmax_xent(logits, label, loss=None, d_logits=None, ws=None, stream=None):
    """(loss device scalar, d_logits) of the mean cross-entropy over labelled rows."""
    n, Cn = logits.shape
    dev = logits.device
    loss = loss if loss is not None else torch.empty(1, dtype=torch.float32, device=dev)
    d_logits = d_logits if d_logits is not None else torch.empty_like(logits)
    nb = C.c_size_t(0)
    _check(lib().rnn_softmax_xent_workspace_size(n, C.byref(nb)))
    w = ws.get(nb.value) if ws is not None else _ws(nb.value, dev)
    _check(lib().rnn_softmax_xent(_ptr(logits), n, Cn, logits.stride(0), _ptr(label), _ptr(loss),
                                  _ptr(d_logits), d_logits.stride(0), _ptr(w), w.numel(),
                                  _stream(stream)))
    return loss, d_logits


class Adam:
    """rnn_adam over a list of parameter tensors (2-D views or 1-D vectors), with the step
    counter on the device (rnn_adam_tick), so a training step is graph-capturable."""

    def __init__(self, params, lr=0.01, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.0):
        self.params = [p if p.dim() == 2 else p.view(1, -1) for p in params]
        dev = self.params[0].device
        self.m = [torch.zeros(p.shape, dtype=torch.float32, device=dev) for p in self.params]
        self.v = [torch.zeros(p.shape, dtype=torch.float32, device=dev) for p in self.params]
        self.t = torch.zeros(1, dtype=torch.int64, device=dev)
        self.cfg = AdamC(lr, betas[0], betas[1], eps, weight_decay)

    def step(self, grads, stream=None):
        _check(lib().rnn_adam_tick(_ptr(self.t), _stream(stream)))
        for p, g, m, v in zip(self.params, grads, self.m, self.v):
            g = g if g.dim() == 2 else g.view(1, -1)
            _check(lib().rnn_adam(_ptr(p), p.shape[0], p.shape[1], p.stride(0), _ptr(g),
                                  g.stride(0), _ptr(m), _ptr(v), C.byref(self.cfg), _ptr(self.t),
                                  _stream(stream)))


# ------------------------------------------------------------------------------------------
# selection sigma pushdown
# ------------------------------------------------------------------------------------------
SELECT_OPS = {"==": 0, "!=": 1, "<": 2, "<=": 3, ">": 4, ">=": 5}


def select_mask(attr, op, value, mask=None, combine="set", stream=None):
    """mask[j] (uint8) = attr[j] <op> value, or AND / OR-ed into an existing mask
    (rnn_select_mask); attr int64 or float32 per E row (device)."""
    n = attr.numel()
    dtype = 0 if attr.dtype == torch.int64 else 1 if attr.dtype == torch.float32 else None
    if dtype is None:
        raise TypeError("attr must be int64 or float32")
    if mask is None:
        mask = torch.empty(max(n, 1), dtype=torch.uint8, device=attr.device)[:n]
    _check(lib().rnn_select_mask(_ptr(attr.contiguous()), dtype, n, SELECT_OPS[op], float(value),
                                 {"set": 0, "and": 1, "or": 2}[combine], _ptr(mask),
                                 _stream(stream)))
    return mask


def scatter_add_rows(y, x, idx, stream=None):
    """y[idx[i]] += x[i] (distinct idx within the call; rnn_scatter_add_rows)."""
    n, cols = x.shape
    _check(lib().rnn_scatter_add_rows(_ptr(y), y.stride(0), _ptr(x), x.stride(0), _ptr(idx), n,
                                      cols, _stream(stream)))
    return y
