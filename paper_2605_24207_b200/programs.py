"""Neuro-relational programs of the paper's workloads, run through librnn.so.

Each program is the set of join rules the paper compiles (sec 3.1) with
the transformation pushed below the join: per layer a dense projection
(A2, tcgen05) followed by one lifted join-aggregate (A3/A4) and, backward, the LJA
backward (A5) and the projection backward.  Join indices are built once (A1, content
caching) and reused by every step.  All arithmetic runs in librnn.so; torch only owns the
buffers and the stream.

GCN (configs 1-2; PyG GCNConv reading):
    AEdge = Edge U {(v,v)};  w(s,t) = deg(s)^-1/2 deg(t)^-1/2
    H^{l+1}(t; sum(w * z)) :- AEdge(s,t), Z^l(s; z),   Z^l = H^l W_l^T
The layer-1 source relation is the node relation (rows in storage order); the output of a
layer is keyed by the group keys (ascending), so layers >= 2 use a second index whose S and
T are that key-ordered relation.
"""
from __future__ import annotations

import numpy as np
import torch

from . import rnn


def _dev_f32(a, device, ld=None):
    """fp32 device tensor with ld % 4 == 0 (a padded, 16-byte aligned row-major view)."""
    a = np.asarray(a, np.float32)
    n, d = a.shape
    ld = ld or (d + 3) // 4 * 4
    buf = torch.zeros((max(n, 1), ld), dtype=torch.float32, device=device)
    buf[:n, :d] = torch.from_numpy(a).to(device)
    return buf[:n, :d]


def _empty(n, d, device):
    ld = (d + 3) // 4 * 4
    return torch.empty((max(n, 1), ld), dtype=torch.float32, device=device)[:n, :d]


class GCNProgram:
    """L-layer GCN as lifted queries; step() = forward + backward of every layer."""

    def __init__(self, graph: dict, device="cuda", prec="3xtf32", rows_per_item=0):
        self.device = torch.device(device)
        self.prec = prec
        dev = self.device
        nodes, edges = graph["nodes"], graph["edges"]
        self.dims = list(graph["dims"])
        self.L = len(self.dims) - 1
        key = torch.as_tensor(nodes["key"]).to(dev)
        e_src = torch.as_tensor(edges["src"]).to(dev)
        e_dst = torch.as_tensor(edges["dst"]).to(dev)
        # A1 (content caching): index 1 joins AEdge with the node relation in storage order
        self.idx1 = rnn.build_join_index(e_src, e_dst, key, key, rows_per_item=rows_per_item)
        self.w1 = rnn.gcn_norm(self.idx1)
        if self.L > 1:
            gk = self.idx1.group_key.clone()
            self.idx2 = rnn.build_join_index(e_src, e_dst, gk, gk, rows_per_item=rows_per_item)
            self.w2 = rnn.gcn_norm(self.idx2)
        self.n_nodes = len(nodes["key"])
        self.G = self.idx1.n_groups
        self.X0 = _dev_f32(nodes["x"], dev)
        self.W = [_dev_f32(w, dev) for w in graph["W"]]
        # activations and gradients (preallocated so the step can be graph-captured)
        self.H = [self.X0] + [_empty(self.G, self.dims[l + 1], dev) for l in range(self.L)]
        self.Z = [_empty(self.n_nodes if l == 0 else self.G, self.dims[l + 1], dev) for l in range(self.L)]
        self.dZ = [_empty(self.n_nodes if l == 0 else self.G, self.dims[l + 1], dev) for l in range(self.L)]
        self.dH = [_empty(self.n_nodes if l == 0 else self.G, self.dims[l], dev) for l in range(self.L)]
        self.dW = [torch.empty(self.dims[l + 1], self.dims[l], dtype=torch.float32, device=dev) for l in range(self.L)]
        self.d_out = _dev_f32(graph["d_out"][: self.G, : self.dims[-1]], dev)
        self.ws = rnn.Workspace(dev)
        self.ws_p = rnn.Workspace(dev)
        self.q = []
        for l in range(self.L):
            idx, w = (self.idx1, self.w1) if l == 0 else (self.idx2, self.w2)
            self.q.append((idx, rnn.make_query("src", "sum", src=self.Z[l], edge=w,
                                               edge_mode=rnn.BY_POSITION)))
        self.timers = None  # optional {"lja_fwd": [...], ...} event lists

    @property
    def join_rows_per_step(self):
        return self.idx1.n_join_rows + (self.L - 1) * (self.idx2.n_join_rows if self.L > 1 else 0)

    def _t(self, name):
        if self.timers is None:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.timers.setdefault(name, []).append(e)
        return e

    def forward(self):
        for l in range(self.L):
            self._t("proj_fwd")
            rnn.project(self.H[l], self.W[l], out=self.Z[l], prec=self.prec)
            self._t("proj_fwd_end")
            idx, q = self.q[l]
            self._t("lja_fwd")
            rnn.join_aggregate_fwd(idx, q, out=self.H[l + 1], ws=self.ws)
            self._t("lja_fwd_end")
        return self.H[-1]

    def backward(self, d_out=None):
        dY = self.d_out if d_out is None else d_out
        for l in reversed(range(self.L)):
            idx, q = self.q[l]
            self._t("lja_bwd")
            g = self._lja_bwd_into(idx, q, dY, self.dZ[l])
            self._t("lja_bwd_end")
            self._t("proj_bwd")
            rnn.project_bwd(self.H[l], self.W[l], g, want_dx=True, prec=self.prec, ws=self.ws_p,
                            dx_out=self.dH[l], dw_out=self.dW[l])
            self._t("proj_bwd_end")
            dY = self.dH[l]
        return self.dW, self.dH[0]

    def _lja_bwd_into(self, idx, q, d_out, d_src):
        import ctypes as C
        _, bb = rnn.lja_workspace_size(idx, q)
        w = self.ws.get(bb)
        rnn._check(rnn.lib().rnn_join_aggregate_bwd(
            C.byref(idx.c), C.byref(q), None, 0, None, rnn._ptr(d_out), d_out.stride(0),
            rnn._ptr(d_src), None, None, None, rnn._ptr(w), w.numel(), rnn._stream()))
        return d_src

    def step(self):
        self.forward()
        return self.backward()

