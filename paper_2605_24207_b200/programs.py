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


class _Program:
    """Shared plumbing: optional per-kernel CUDA-event timers (bench.py), the algorithmic
    byte model of the LJA launches and the step's host I/O."""
    timers = None  # optional {"lja_fwd": [...], "lja_fwd_end": [...], ...} event lists

    def _t(self, name):
        if self.timers is None:
            return None
        # inside a CUDA-graph capture the event becomes a record node of the graph, re-recorded
        # by every replay (cudaEventRecordExternal)
        e = torch.cuda.Event(enable_timing=True,
                             external=torch.cuda.is_current_stream_capturing())
        e.record()
        self.timers.setdefault(name, []).append(e)
        return e

    def step(self):
        self.forward()
        return self.backward()

    def roof_model(self):
        """{kernel timer name: {"bound": "hbm", "amount": algorithmic bytes per launch,
        "compulsory": compulsory bytes per launch}}"""
        comp = self.compulsory_bytes() if hasattr(self, "compulsory_bytes") else {}
        return {k: {"bound": "hbm", "amount": v, "compulsory": comp.get(k)}
                for k, v in self.lja_bytes().items()}

    def build_indices(self):
        """(Re)build every join index of the program (A1; content caching: done once)."""
        raise NotImplementedError


def _sum_bytes(idx, d, weighted=False, mean=False):
    """Gather-model bytes of one SUM/MEAN LJA forward launch: per join row the source row id
    (4), the edge weight (4, if any), the gathered d-vector (4d), the group's extent for MEAN
    (8); per group the output row (4d) and its CSR pointer (8)."""
    return idx.n_join_rows * (4 + 4 * d + (4 if weighted else 0) + (8 if mean else 0)) + \
        idx.n_groups * (4 * d + 8)


def _sum_bwd_bytes(idx, d, weighted=False, mean=False):
    """... backward launch over the transposed CSR: per join row src_pos (4) + group id (4)
    + weight (4, if any) + gathered upstream d-vector (4d) (+8 MEAN); per source row the
    gradient row (4d) + pointer (8)."""
    return idx.n_join_rows * (8 + 4 * d + (4 if weighted else 0) + (8 if mean else 0)) + \
        idx.n_src_rows * (4 * d + 8)


def _n_referenced(idx):
    """U = distinct source rows the join rows reference (cached on the index object)."""
    u = getattr(idx, "_n_ref", None)
    if u is None:
        u = int((idx.src_ptr[1:] > idx.src_ptr[:-1]).sum().item()) if idx.n_join_rows else 0
        idx._n_ref = u
    return u


def _comp_fwd(idx, d, weighted=False):
    """Compulsory bytes of one SUM/MEAN forward launch: every index entry,
    every REFERENCED input row and every output row crosses HBM once -- src_row (4) and the
    weight (4) per join row, the CSR pointers, U source rows and G output rows of 4d."""
    return idx.n_join_rows * (4 + (4 if weighted else 0)) + 8 * (idx.n_groups + 1) + \
        4 * d * (_n_referenced(idx) + idx.n_groups)


def _comp_bwd(idx, d, weighted=False):
    """... of one backward launch over the transposed CSR: src_pos + group id (8) and the
    weight (4) per join row, the source CSR pointers, G upstream rows read and every source
    gradient row written (4d each)."""
    return idx.n_join_rows * (8 + (4 if weighted else 0)) + 8 * (idx.n_src_rows + 1) + \
        4 * d * (idx.n_groups + idx.n_src_rows)


class GCNProgram(_Program):
    """L-layer GCN as lifted queries; step() = forward + backward of every layer."""
    # experiment knob (profiles/r02/l2window): a persisting-L2 window over each LJA's gathered
    # matrix (eager steps only: the limit change is not capturable)
    l2_window = False

    def __init__(self, graph: dict, device="cuda", prec="3xtf32", rows_per_item=0):
        self.device = torch.device(device)
        self.prec = prec
        dev = self.device
        nodes, edges = graph["nodes"], graph["edges"]
        self.dims = list(graph["dims"])
        self.L = len(self.dims) - 1
        self._key = torch.as_tensor(nodes["key"]).to(dev)
        self._e = (torch.as_tensor(edges["src"]).to(dev), torch.as_tensor(edges["dst"]).to(dev))
        self._rpi = rows_per_item
        self.build_indices()
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
        self.ws_e = rnn.Workspace(dev)
        # O7 node epilogue (PyG GCNConv): bias then ReLU on hidden layers, bias
        # only on the last, fused into the LJA's store; graphs without "b" run the bare LJA
        self.b = [torch.as_tensor(np.asarray(b, np.float32)).to(dev) for b in graph["b"]] \
            if graph.get("b") is not None else None
        self.epi, self.dP, self.db = [], [], []
        if self.b is not None:
            for l in range(self.L):
                act = "relu" if l < self.L - 1 else "none"
                self.epi.append(rnn.make_epilogue(bias=self.b[l], act=act))
                self.dP.append(_empty(self.G, self.dims[l + 1], dev))
                self.db.append(torch.empty(self.dims[l + 1], dtype=torch.float32, device=dev))
        self.q = []
        for l in range(self.L):
            idx, w = (self.idx1, self.w1) if l == 0 else (self.idx2, self.w2)
            self.q.append((idx, rnn.make_query("src", "sum", src=self.Z[l], edge=w,
                                               edge_mode=rnn.BY_POSITION)))

    def build_indices(self):
        """A1 (content caching, built once): index 1 joins AEdge with the node relation in
        storage order, index 2 with the key-ordered layer output; plus the GCN weights."""
        e_src, e_dst = self._e
        self.idx1 = rnn.build_join_index(e_src, e_dst, self._key, self._key, rows_per_item=self._rpi)
        self.w1 = rnn.gcn_norm(self.idx1)
        if self.L > 1:
            gk = self.idx1.group_key.clone()
            self.idx2 = rnn.build_join_index(e_src, e_dst, gk, gk, rows_per_item=self._rpi)
            self.w2 = rnn.gcn_norm(self.idx2)

    @property
    def join_rows_per_step(self):
        return self.idx1.n_join_rows + (self.L - 1) * (self.idx2.n_join_rows if self.L > 1 else 0)

    def _layer_idx(self):
        return [self.idx1] + [self.idx2] * (self.L - 1)

    def lja_bytes(self):
        """Average algorithmic bytes per LJA launch {kernel: bytes} (fwd, bwd over layers)."""
        ix = self._layer_idx()
        d = self.dims[1:]
        return {"lja_fwd": float(np.mean([_sum_bytes(i, dd, True) for i, dd in zip(ix, d)])),
                "lja_bwd": float(np.mean([_sum_bwd_bytes(i, dd, True) for i, dd in zip(ix, d)]))}

    def compulsory_bytes(self):
        ix = self._layer_idx()
        d = self.dims[1:]
        return {"lja_fwd": float(np.mean([_comp_fwd(i, dd, True) for i, dd in zip(ix, d)])),
                "lja_bwd": float(np.mean([_comp_bwd(i, dd, True) for i, dd in zip(ix, d)]))}

    def host_io(self):
        """(inputs, outputs) a user's step moves across PCIe: features + upstream gradient in,
        parameter gradients out."""
        return [self.X0, self.d_out], list(self.dW)

    def forward(self):
        for l in range(self.L):
            self._t("proj_fwd")
            rnn.project(self.H[l], self.W[l], out=self.Z[l], prec=self.prec)
            self._t("proj_fwd_end")
            idx, q = self.q[l]
            if self.l2_window:
                rnn.stream_l2_window(self.Z[l])      # the gathered matrix of this layer
            self._t("lja_fwd")
            if self.b is not None:
                rnn.join_aggregate_fwd_epi(idx, q, self.epi[l], out=self.H[l + 1], ws=self.ws)
            else:
                rnn.join_aggregate_fwd(idx, q, out=self.H[l + 1], ws=self.ws)
            self._t("lja_fwd_end")
        return self.H[-1]

    def backward(self, d_out=None):
        """With the O7 epilogue: the last layer's (bias only) backward is d bias = colsum(dY)
        and dY passes through unchanged; every hidden layer's ReLU backward is fused into the
        next layer's projection backward (rnn_project_bwd_relu: its input H^l is the ReLU
        output, so dX comes out as d(pre-activation) and the bias gradient as its column sums).
        Without it, dH^l = dZ^l W^l as in the bare lifted query."""
        dY = self.d_out if d_out is None else d_out
        for l in reversed(range(self.L)):
            idx, q = self.q[l]
            if self.b is not None and l == self.L - 1:
                self._t("epi_bwd")
                rnn.epilogue_bwd(dY, self.H[l + 1], self.epi[l], ws=self.ws_e, db_out=self.db[l],
                                 want_dx=False)
                self._t("epi_bwd_end")
            if self.l2_window:
                rnn.stream_l2_window(dY)              # gathered by the source-major backward
            self._t("lja_bwd")
            g = self._lja_bwd_into(idx, q, dY, self.dZ[l])
            self._t("lja_bwd_end")
            self._t("proj_bwd")
            if self.b is not None and l > 0:
                rnn.project_bwd(self.H[l], self.W[l], g, want_dx=True, prec=self.prec,
                                ws=self.ws_p, dx_out=self.dP[l - 1], dw_out=self.dW[l],
                                relu_in=True, d_in_bias=self.db[l - 1])
                dY = self.dP[l - 1]
            else:
                rnn.project_bwd(self.H[l], self.W[l], g, want_dx=True, prec=self.prec,
                                ws=self.ws_p, dx_out=self.dH[l], dw_out=self.dW[l])
                dY = self.dH[l]
            self._t("proj_bwd_end")
        if self.l2_window:
            rnn.stream_l2_window(None)
        return self.dW, self.dH[0]

    # ---- fit (SURVEY sec 8f item 3; PAPER.md:549 Loss, :554 ?fit) ----
    def setup_training(self, labels, lr=0.01, weight_decay=5e-4, learn_embeddings=False):
        """Loss(; CrossEntropyLoss()(H^L, label)) over the labelled nodes and an Adam fit of
        every W and b (and, with learn_embeddings, of the per-tuple input embeddings X0 --
        PAPER.md:568).  labels: int64 per node row (-1 = unlabelled); the logits are H^L in
        group (key) order, so the labels are permuted to that order once here."""
        dev = self.device
        lab = np.asarray(labels, np.int64)
        row = self.idx1.group_dst_row.cpu().numpy()
        self.labels_g = torch.as_tensor(lab[row]).to(dev)
        self.loss = torch.zeros(1, dtype=torch.float32, device=dev)
        self.d_logits = _empty(self.G, self.dims[-1], dev)
        self.ws_x = rnn.Workspace(dev)
        params, self._grads = list(self.W), list(self.dW)
        if self.b is not None:
            params += self.b
            self._grads += self.db
        if learn_embeddings:
            params.append(self.X0)
            self._grads.append(self.dH[0])
        self.opt = rnn.Adam(params, lr=lr, weight_decay=weight_decay)

    def train_step(self):
        """One epoch of full-batch training: forward, loss, backward, Adam (all on device)."""
        self.forward()
        self._t("loss")
        rnn.softmax_xent(self.H[-1], self.labels_g, loss=self.loss, d_logits=self.d_logits,
                         ws=self.ws_x)
        self._t("loss_end")
        self.backward(d_out=self.d_logits)
        self._t("adam")
        self.opt.step(self._grads)
        self._t("adam_end")
        return self.loss

    def _lja_bwd_into(self, idx, q, d_out, d_src):
        import ctypes as C
        _, bb = rnn.lja_workspace_size(idx, q)
        w = self.ws.get(bb)
        rnn._check(rnn.lib().rnn_join_aggregate_bwd(
            C.byref(idx.c), C.byref(q), None, 0, None, rnn._ptr(d_out), d_out.stride(0),
            rnn._ptr(d_src), None, None, None, rnn._ptr(w), w.numel(), rnn._stream()))
        return d_src


class HypergraphProgram(_Program):
    """HyGNN-style two-hop incidence join (config 4, reading 13):

        Z = X Theta^T                                          (A2)
        E_h(e; sum(z))  :- Inc(v, e), Z(v; z)                  hop 1, grouped by hyperedge
        X'(v; mean(z))  :- Inc(v, e), E_h(e; z)                hop 2, grouped by node
    """

    def __init__(self, hg: dict, device="cuda", prec="3xtf32", rows_per_item=0):
        dev = self.device = torch.device(device)
        self.prec = prec
        self._in = tuple(torch.as_tensor(a).to(dev) for a in (
            hg["nodes"]["key"], hg["hyperedges"]["key"], hg["inc"]["node"], hg["inc"]["hyper"]))
        self._rpi = rows_per_item
        self.build_indices()
        d = hg["nodes"]["x"].shape[1]
        self.d = d
        self.X = _dev_f32(hg["nodes"]["x"], dev)
        self.theta = _dev_f32(hg["theta"], dev)
        n = len(hg["nodes"]["key"])
        self.Z = _empty(n, d, dev)
        self.Eh = _empty(self.idx1.n_groups, d, dev)
        self.Xo = _empty(self.idx2.n_groups, d, dev)
        self.dEh = _empty(self.idx1.n_groups, d, dev)
        self.dZ = _empty(n, d, dev)
        self.dX = _empty(n, d, dev)
        self.dTheta = torch.empty(d, d, dtype=torch.float32, device=dev)
        self.d_out = _dev_f32(hg["d_out"][: self.idx2.n_groups], dev)
        self.q1 = rnn.make_query("src", "sum", src=self.Z)
        self.q2 = rnn.make_query("src", "mean", src=self.Eh)
        self.ws = rnn.Workspace(dev)
        self.ws_p = rnn.Workspace(dev)

    def build_indices(self):
        nk, hk, iv, ih = self._in
        self.idx1 = rnn.build_join_index(iv, ih, nk, hk, rows_per_item=self._rpi)
        self.idx2 = rnn.build_join_index(ih, iv, self.idx1.group_key.clone(), nk,
                                         rows_per_item=self._rpi)

    @property
    def join_rows_per_step(self):
        return self.idx1.n_join_rows + self.idx2.n_join_rows

    def lja_bytes(self):
        d = self.d
        return {"lja_fwd": (_sum_bytes(self.idx1, d) + _sum_bytes(self.idx2, d, mean=True)) / 2,
                "lja_bwd": (_sum_bwd_bytes(self.idx1, d) + _sum_bwd_bytes(self.idx2, d, mean=True)) / 2}

    def compulsory_bytes(self):
        d = self.d
        return {"lja_fwd": (_comp_fwd(self.idx1, d) + _comp_fwd(self.idx2, d)) / 2,
                "lja_bwd": (_comp_bwd(self.idx1, d) + _comp_bwd(self.idx2, d)) / 2}

    def host_io(self):
        return [self.X, self.d_out], [self.dTheta]

    def forward(self):
        self._t("proj_fwd")
        rnn.project(self.X, self.theta, out=self.Z, prec=self.prec)
        self._t("proj_fwd_end")
        for idx, q, out in ((self.idx1, self.q1, self.Eh), (self.idx2, self.q2, self.Xo)):
            self._t("lja_fwd")
            rnn.join_aggregate_fwd(idx, q, out=out, ws=self.ws)
            self._t("lja_fwd_end")
        return self.Xo

    def backward(self):
        for idx, q, dout, dsrc in ((self.idx2, self.q2, self.d_out, self.dEh),
                                   (self.idx1, self.q1, self.dEh, self.dZ)):
            self._t("lja_bwd")
            _lja_src_grad(idx, q, dout, dsrc, self.ws)
            self._t("lja_bwd_end")
        self._t("proj_bwd")
        rnn.project_bwd(self.X, self.theta, self.dZ, want_dx=True, prec=self.prec, ws=self.ws_p,
                        dx_out=self.dX, dw_out=self.dTheta)
        self._t("proj_bwd_end")
        return self.dTheta, self.dX


def _lja_src_grad(idx, q, d_out, d_src, ws):
    """rnn_join_aggregate_bwd writing only the source-embedding gradient into d_src."""
    import ctypes as C
    _, bb = rnn.lja_workspace_size(idx, q)
    w = ws.get(bb)
    rnn._check(rnn.lib().rnn_join_aggregate_bwd(
        C.byref(idx.c), C.byref(q), None, 0, None, rnn._ptr(d_out), d_out.stride(0),
        rnn._ptr(d_src), None, None, None, rnn._ptr(w), w.numel(), rnn._stream()))
    return d_src


def hgt_parameters(mag: dict, seed=7):
    """Weights and upstream gradient of the HGT layer (host, numpy), shared by HGTProgram and
    the sharded program: per node type the stacked projection W [nb * d, d] whose column
    blocks are (K'_phi, M'_phi) for every relation phi leaving the type and ONE query block
    ("q", type) for the relations entering it (QLin<L, tau_t> is per target type, PAPER.md
    Fig. 4, so every relation into t reads the same Q and dQ is the sum over them; K'
    carries mu / sqrt(d / h), reading 12); d_out [n_t, d] per target type in T-key order."""
    d, h = mag["d"], mag["heads"]
    rng = np.random.default_rng(seed)
    types = list(mag["n"].keys())
    blocks = {t: [] for t in types}
    for name, r in mag["rels"].items():
        blocks[r["src_type"]] += [("k", name), ("m", name)]
    # the query block last: the K'/M' blocks of a type are one contiguous column range (the
    # only columns the sharded program exchanges)
    for r in mag["rels"].values():
        if ("q", r["dst_type"]) not in blocks[r["dst_type"]]:
            blocks[r["dst_type"]] += [("q", r["dst_type"])]
    blocks = {t: b for t, b in blocks.items() if b}
    scale = 1.0 / np.sqrt(d / h)
    wq = {t: rng.standard_normal((d, d)) / np.sqrt(d) for t in types}
    W = {}
    for t, b in blocks.items():
        ws = []
        for kind, name in b:
            w = rng.standard_normal((d, d)) / np.sqrt(d)
            if kind == "k":
                w = w * scale            # mu / sqrt(d/h) folded into K'
            if kind == "q":
                w = wq[t]                # the target type's query map
            ws.append(w)
        W[t] = np.concatenate(ws, 0).astype(np.float32)
    col = {(kind, name): (t, i) for t, b in blocks.items() for i, (kind, name) in enumerate(b)}
    targets = sorted({r["dst_type"] for r in mag["rels"].values()})
    d_out = {t: rng.standard_normal((mag["n"][t], d)).astype(np.float32) for t in targets}
    return {"blocks": blocks, "W": W, "col": col, "targets": targets, "d_out": d_out}


class HGTProgram(_Program):
    """One HGT attention layer over a heterogeneous schema (config 3; Fig. 4, PAPER.md:905-936,
    appendix :1343-1409; SURVEY sec 8c reading 3/12).

    Per relation phi = (tau_s -> tau_t), with the transformations pushed below the join:
        K'_phi = H_{tau_s} Wk_phi^T      (KLin . W_ATT . mu / sqrt(d/h) folded)
        M'_phi = H_{tau_s} Wm_phi^T      (MLin . W_MSG folded)
        Q_phi  = H_{tau_t} Wq_{tau_t}^T
        O_phi(t; softmax-weighted sum) :- phi(s, t), K'(s), M'(s), Q(t)     (A4, per head)
        H_tilda_{tau_t} = sum_phi O_phi                                      (A7 union)
    All projections of one node type are ONE tcgen05 GEMM (weights stacked); every relation's
    index has dense groups over its target type, so outputs share the target's key order.
    """

    def __init__(self, mag: dict, device="cuda", prec="3xtf32", rows_per_item=0, seed=7):
        dev = self.device = torch.device(device)
        self.prec = prec
        self.d, self.h = mag["d"], mag["heads"]
        d = self.d
        types = list(mag["n"].keys())
        self.keys = {t: torch.as_tensor(mag["key"][t]).to(dev) for t in types}
        self.H = {t: _dev_f32(mag["h"][t], dev) for t in types}
        self.n = dict(mag["n"])
        rels = mag["rels"]
        par = hgt_parameters(mag, seed)
        self.blocks, self.col, self.targets = par["blocks"], par["col"], par["targets"]
        self.W, self.Y, self.dY, self.dW, self.dH = {}, {}, {}, {}, {}
        for t, b in self.blocks.items():
            self.W[t] = _dev_f32(par["W"][t], dev)
            nb = len(b)
            self.Y[t] = _empty(self.n[t], nb * d, dev)
            self.dY[t] = _empty(self.n[t], nb * d, dev)
            self.dW[t] = torch.empty(nb * d, d, dtype=torch.float32, device=dev)
            self.dH[t] = _empty(self.n[t], d, dev)
        self.idx, self.q, self.O, self.lse, self.dO = {}, {}, {}, {}, {}
        self.targets = sorted({r["dst_type"] for r in rels.values()})
        self.Ht = {t: _empty(self.n[t], d, dev) for t in self.targets}
        self.d_out = {t: _dev_f32(par["d_out"][t], dev) for t in self.targets}
        self._rel_keys = {name: (torch.as_tensor(r["src"]).to(dev), torch.as_tensor(r["dst"]).to(dev))
                          for name, r in rels.items()}
        self._rpi = rows_per_item
        self.rels = rels
        self.build_indices()
        for name, r in rels.items():
            ts, tt = r["src_type"], r["dst_type"]
            self.q[name] = rnn.make_query("src", "softmax", src=self._blk("m", name),
                                          src_key=self._blk("k", name), dst=self._blk("q", tt),
                                          heads=self.h, scale=1.0)
            # a target type reached by ONE relation: H_tilda is that relation's output itself
            n_into = sum(x["dst_type"] == tt for x in rels.values())
            self.O[name] = self.Ht[tt] if n_into == 1 else _empty(self.n[tt], d, dev)
            self.lse[name] = torch.empty(max(self.n[tt], 1), self.h, dtype=torch.float32, device=dev)
        self.ws = rnn.Workspace(dev)
        self.ws_p = rnn.Workspace(dev)

    def _blk(self, kind, name, grad=False):
        t, i = self.col[(kind, name)]
        buf = self.dY[t] if grad else self.Y[t]
        return buf[:, i * self.d:(i + 1) * self.d]

    def build_indices(self):
        """One dense-group index per relation phi (A1, built once)."""
        for name, r in self.rels.items():
            e_src, e_dst = self._rel_keys[name]
            self.idx[name] = rnn.build_join_index(
                e_src, e_dst, self.keys[r["src_type"]], self.keys[r["dst_type"]],
                dense_groups=True, rows_per_item=self._rpi)

    @property
    def join_rows_per_step(self):
        return sum(ix.n_join_rows for ix in self.idx.values())

    def compulsory_bytes(self):
        """Every index entry, referenced input row and output row once.  fwd: src_row (4) per
        join row, CSR pointers, U referenced sources' K' and M' rows (8d), per group the Q
        row, the output row and lse (8d + 4h).  bwd: src_row + src_group + src_pos (12) per
        join row, both CSRs' pointers, K' and M' of the U sources (8d), per group Q, O and dO
        (12d) and lse (4h) read and dQ written (4d), every source's dK' and dM' written (8d)."""
        d, h = self.d, self.h
        f, b = [], []
        for ix in self.idx.values():
            U = _n_referenced(ix)
            G, E, ns = ix.n_groups, ix.n_join_rows, ix.n_src_rows
            f.append(E * 4 + 8 * (G + 1) + 8 * d * U + G * (8 * d + 4 * h))
            b.append(E * 12 + 8 * (G + 1) + 8 * (ns + 1) + 8 * d * U + G * (16 * d + 4 * h) +
                     ns * 8 * d)
        return {"lja_fwd": float(np.mean(f)), "lja_bwd": float(np.mean(b))}

    def lja_bytes(self):
        """Softmax LJA gather model (h heads), for the algorithm the library
        runs.  fwd, per join row: src id 4 + K' and M' rows 8d; per group: Q row 4d, out 4d,
        lse 4h, pointer 8.  bwd (source-major): D = <dO, O> per group reads
        8d and writes 4h; pass A per join row: group id + position 8 + Q[t] and dO[g] rows 8d +
        lse and D 8h + DE written 4h, per source row: K', M' read 8d + dK', dM' written 8d +
        pointer 8; pass B per join row: src id 4 + K' row 4d + DE 4h, per group dQ written 4d +
        pointer 8.  (The two-pass (a, de) scheme, RNN_SM_TWOPASS, moved 16d + 16h per row.)"""
        d, h = self.d, self.h
        f, b = [], []
        for ix in self.idx.values():
            f.append(ix.n_join_rows * (4 + 8 * d) + ix.n_groups * (8 * d + 4 * h + 8))
            b.append(ix.n_join_rows * ((8 + 8 * d + 12 * h) + (4 + 4 * d + 4 * h)) +
                     ix.n_groups * (8 * d + 4 * h + 4 * d + 8) + ix.n_src_rows * (16 * d + 8))
        return {"lja_fwd": float(np.mean(f)), "lja_bwd": float(np.mean(b))}

    def host_io(self):
        return list(self.H.values()) + list(self.d_out.values()), list(self.dW.values())

    def forward(self):
        self._t("proj_fwd")
        for t in self.blocks:
            rnn.project(self.H[t], self.W[t], out=self.Y[t], prec=self.prec)
        self._t("proj_fwd_end")
        first = {t: True for t in self.targets}
        for name, r in self.rels.items():
            tt = r["dst_type"]
            self._t("lja_fwd")
            if self.O[name] is self.Ht[tt]:
                rnn.join_aggregate_fwd(self.idx[name], self.q[name], out=self.O[name],
                                       lse=self.lse[name], ws=self.ws)
            else:   # union over the relations into tt, fused into the walker's store
                rnn.join_aggregate_fwd_union(self.idx[name], self.q[name], self.O[name],
                                             self.Ht[tt], beta_acc=0.0 if first[tt] else 1.0,
                                             lse=self.lse[name], ws=self.ws)
            self._t("lja_fwd_end")
            first[tt] = False
        return self.Ht

    def backward(self):
        import ctypes as C
        first = {t: True for t in self.targets}
        for name, r in self.rels.items():
            tt = r["dst_type"]
            idx, q = self.idx[name], self.q[name]
            dO = self.d_out[tt]
            _, bb = rnn.lja_workspace_size(idx, q)
            w = self.ws.get(bb)
            dm, dk = self._blk("m", name, True), self._blk("k", name, True)
            dq = self._blk("q", tt, True)
            self._t("lja_bwd")
            # the shared query's gradient is the sum over the relations into tt: the first
            # writes it, the others accumulate in place (rnn_join_aggregate_bwd_acc)
            rnn._check(rnn.lib().rnn_join_aggregate_bwd_acc(
                C.byref(idx.c), C.byref(q), rnn._ptr(self.O[name]), self.O[name].stride(0),
                rnn._ptr(self.lse[name]), rnn._ptr(dO), dO.stride(0), rnn._ptr(dm), rnn._ptr(dk),
                None, rnn._ptr(dq), 0.0 if first[tt] else 1.0, rnn._ptr(w), w.numel(),
                rnn._stream()))
            self._t("lja_bwd_end")
            first[tt] = False
        self._t("proj_bwd")
        for t in self.blocks:
            rnn.project_bwd(self.H[t], self.W[t], self.dY[t], want_dx=True, prec=self.prec,
                            ws=self.ws_p, dx_out=self.dH[t], dw_out=self.dW[t])
        self._t("proj_bwd_end")
        return self.dW, self.dH


def edge_is_symmetric(idx) -> bool:
    """True iff the Edge join rows of a DHN adjacency index (root row, neighbour row) equal
    their reverse as a multiset -- decided on the index itself, so Edge tuples dropped by the
    join (absent keys) cannot make a non-symmetric relation look symmetric."""
    if idx.n_join_rows == 0:
        return True
    r = idx.group_dst_row.long()[idx.pos_group.long()]
    v = idx.src_row.long()
    n = max(int(idx.n_src_rows), 1)
    return bool(torch.equal(torch.sort(r * n + v).values, torch.sort(v * n + r).values))


class DHNProgram(_Program):
    """Deep homomorphism network layer on one node relation (config 5; PAPER.md:938-950,
    SURVEY sec 8a A6 and sec 8c readings 9 / 14):

        f_{k,i} = mu_{k,i}(h) = h W_{k,i}^T             (A2: all nine 32x32 maps in ONE GEMM)
        C_k(n)  = f_{k,0}(n) (.) sum_{closed k-walks} prod_i f_{k,i}(v_i)    k = 2, 3, 4   (A6)
        out     = C_2 (+) C_3 (+) C_4                    (concat; rho and the readout are OUT)

    The adjacency index has dense groups, so root n of every C_k is node n in key order and
    out is [n_nodes, 3d] in key order.  Backward: rnn_dhn_bwd per pattern (rotation) into the
    column blocks of dY, then the projection backward."""

    KS = (2, 3, 4)

    def __init__(self, g: dict, device="cuda", prec="3xtf32", seed=11, ks=KS):
        dev = self.device = torch.device(device)
        self.prec = prec
        self.ks = tuple(ks)
        self._in = tuple(torch.as_tensor(a).to(dev) for a in (
            g["nodes"]["key"], g["edges"]["src"], g["edges"]["dst"]))
        self.build_indices()
        self.n = len(g["nodes"]["key"])
        self.d = d = g["nodes"]["x"].shape[1]
        self.H = _dev_f32(g["nodes"]["x"], dev)
        rng = np.random.default_rng(seed)
        self.npos = sum(self.ks)
        W = rng.standard_normal((self.npos * d, d)) / np.sqrt(d)
        self.W = _dev_f32(W.astype(np.float32), dev)
        self.Y = _empty(self.n, self.npos * d, dev)
        self.dY = _empty(self.n, self.npos * d, dev)
        self.dW = torch.empty(self.npos * d, d, dtype=torch.float32, device=dev)
        self.dH = _empty(self.n, d, dev)
        G = self.idx.n_groups
        self.out = _empty(G, len(self.ks) * d, dev)
        self.d_out = _dev_f32(rng.standard_normal((G, len(self.ks) * d)).astype(np.float32), dev)
        # each pattern's walk sum before the root factor, saved by the forward so the backward
        # forms d f0 = dOut (.) sum without a walk (rnn_dhn_fwd_save / rnn_dhn_bwd_saved)
        self.walk_sum = {k: _empty(G, d, dev) for k in self.ks}
        # RNN_DHN_SYMMETRIC_EDGE: verified once at setup on the built index (the join rows
        # that survived, as (root row, neighbour row) pairs, equal their reverse as a multiset)
        self.symmetric = edge_is_symmetric(self.idx)
        self.ws = rnn.Workspace(dev)
        self.ws_p = rnn.Workspace(dev)
        self.pos0 = {}
        p = 0
        for k in self.ks:
            self.pos0[k] = p
            p += k
        self._rows = None

    def build_indices(self):
        """Edge(n, v): root n = dst column, neighbour v = src column; dense groups."""
        keys, e_src, e_dst = self._in
        self.idx = rnn.build_join_index(e_src, e_dst, keys, keys, dense_groups=True)

    def _f(self, k, buf):
        p = self.pos0[k]
        return [buf[:, (p + i) * self.d:(p + i + 1) * self.d] for i in range(k)]

    @property
    def join_rows_per_step(self):
        """Rows of the lifted joins: Edge rows for C2, closed 3- / 4-walks for C3 / C4 (the
        homomorphism counts, measured once with all-ones operands)."""
        if self._rows is None:
            tot = 0
            for k in self.ks:
                tot += self.idx.n_join_rows if k == 2 else int(self._walks(k))
            self._rows = tot
        return self._rows

    def host_io(self):
        return [self.H, self.d_out], [self.dW]

    def roof_model(self):
        """The walk kernels are bound by the FP32 pipe and on-chip (L2 / L1) traffic, not HBM:
        algorithmic flops per launch of the factorised plans:
          C2: E' d adds;  C3: per closed 3-walk (hit) 2d (scale + multiply-add);
          C4: per 2-path into the root d adds (S3 scatter) + per 2-path out of the root 2d
              (f2 * S3 fma) + per root neighbour d (f1 scaling)."""
        if getattr(self, "_flops", None) is None:
            deg = np.zeros(self.n)
            deg[self.idx.group_dst_row.cpu().numpy()] = np.diff(self.idx.group_ptr.cpu().numpy())
            # Edge is symmetric here (both directions stored): in-degree = out-degree
            two_paths = float(deg[self.idx.src_row.cpu().numpy()].sum())
            d = self.d
            E = float(self.idx.n_join_rows)
            walks3 = self._walks(3)
            self._flops = {"dhn2_fwd": E * d, "dhn3_fwd": 2 * d * walks3,
                           "dhn4_fwd": d * (3 * two_paths + E)}
            # backward: one walk per rotated operand f1 .. f_{k-1}; d f0 = dOut (.) the saved
            # walk sum (elementwise, not counted)
            self._flops["dhn2_bwd"] = self._flops["dhn2_fwd"]
            self._flops["dhn3_bwd"] = (1.5 if self.symmetric else 2) * self._flops["dhn3_fwd"]
            # (symmetric Edge: d f1 and d f3 share one walk with two middle operands, which
            # adds 2d per in-wedge to that walk)
            self._flops["dhn4_bwd"] = (2 * self._flops["dhn4_fwd"] + 2 * d * two_paths
                                       if self.symmetric else 3 * self._flops["dhn4_fwd"])
        return {k: {"bound": "alu", "amount": v} for k, v in self._flops.items()
                if int(k[3]) in self.ks}

    def _walks(self, k):
        """Closed k-walks over all roots: the exact int64 homomorphism counts (rnn_dhn_count)."""
        return int(rnn.dhn_count(self.idx, k).sum().item())

    def forward(self):
        self._t("proj_fwd")
        rnn.project(self.H, self.W, out=self.Y, prec=self.prec)
        self._t("proj_fwd_end")
        for j, k in enumerate(self.ks):
            self._t(f"dhn{k}_fwd")
            rnn.dhn_fwd(self.idx, k, self._f(k, self.Y), out=self.out[:, j * self.d:(j + 1) * self.d],
                        ws=self.ws, walk_sum=self.walk_sum[k])
            self._t(f"dhn{k}_fwd_end")
        return self.out

    def backward(self):
        for j, k in enumerate(self.ks):
            self._t(f"dhn{k}_bwd")
            rnn.dhn_bwd(self.idx, k, self._f(k, self.Y), self.d_out[:, j * self.d:(j + 1) * self.d],
                        d_f=self._f(k, self.dY), ws=self.ws, walk_sum=self.walk_sum[k],
                        symmetric=self.symmetric)
            self._t(f"dhn{k}_bwd_end")
        self._t("proj_bwd")
        rnn.project_bwd(self.H, self.W, self.dY, want_dx=True, prec=self.prec, ws=self.ws_p,
                        dx_out=self.dH, dw_out=self.dW)
        self._t("proj_bwd_end")
        return self.dW, self.dH


class CapturedStep:
    """One program step captured once as a CUDA graph and replayed (the step is launch-bound
    at small sizes: Cora's 14 kernels take ~10 us of GPU time each).  Every buffer the step
    touches is preallocated by the program, so replays read the current contents of its
    input tensors (copy new features / upstream gradients into them, then replay).

    timed=True also captures CUDA-event record nodes around the step and around each kernel
    the program brackets (prog.timers), so per-step and per-kernel device times can be read
    after every replay (`times()`)."""

    def __init__(self, prog, timed=False, warmup=2, step_fn=None):
        self.prog = prog
        step = step_fn or prog.step
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(warmup):       # workspaces reach their final size before capture
                step()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        saved = prog.timers
        prog.timers = {} if timed else None
        self.t0 = self.t1 = None
        with torch.cuda.graph(self.graph):
            if timed:
                self.t0 = torch.cuda.Event(enable_timing=True, external=True)
                self.t0.record()
            step()
            if timed:
                self.t1 = torch.cuda.Event(enable_timing=True, external=True)
                self.t1.record()
        self.events = prog.timers
        prog.timers = saved

    def replay(self):
        self.graph.replay()

    def times(self):
        """(step ms, {kernel: ms summed over its launches in the step}) of the LAST replay
        (call after it completed)."""
        step = self.t0.elapsed_time(self.t1)
        per = {}
        for k, ev in self.events.items():
            if k.endswith("_end"):
                continue
            ends = self.events.get(k + "_end", [])
            per[k] = [a.elapsed_time(b) for a, b in zip(ev, ends)]
        return step, per


class HostStreamedSteps:
    """Run program steps whose inputs arrive from (pinned) HOST memory and whose parameter
    gradients go back to it, with the host->device copy of step i+1's inputs overlapped with
    step i's compute: a copy stream fills a device staging buffer while the compute stream
    runs; each step then moves staging -> the program's input tensors on the device (a D2D
    copy, ~10 us per 100 MB) and launches the step (`run`, e.g. CapturedStep.replay).

        pipe = HostStreamedSteps(prog, run)
        for batch in host_batches:           # lists of pinned CPU tensors, prog.host_io() shapes
            grads = pipe.step(batch)         # pinned CPU tensors, valid after synchronize()
    """

    def __init__(self, prog, run=None):
        self.prog = prog
        self.run = run or prog.step
        self.ins, self.outs = prog.host_io()
        self.stage = [torch.empty(x.shape, dtype=x.dtype, device=x.device) for x in self.ins]
        self.out_host = [torch.empty(w.shape, dtype=w.dtype).pin_memory() for w in self.outs]
        self.copy_stream = torch.cuda.Stream()
        self.filled = torch.cuda.Event()
        self.freed = torch.cuda.Event()
        self.freed.record()
        self.pending = False

    def prefetch(self, host_inputs):
        """Start the host->device copy of the next step's inputs on the copy stream."""
        cs = self.copy_stream
        cs.wait_event(self.freed)                 # staging consumed by the previous step
        with torch.cuda.stream(cs):
            for d, h in zip(self.stage, host_inputs):
                d.copy_(h, non_blocking=True)
            self.filled.record(cs)
        self.pending = True

    def step(self, host_inputs=None, next_inputs=None):
        """One step on the inputs prefetched before (or `host_inputs`, copied now); starts the
        prefetch of `next_inputs` so it overlaps this step's compute."""
        if host_inputs is not None and not self.pending:
            self.prefetch(host_inputs)
        cur = torch.cuda.current_stream()
        cur.wait_event(self.filled)
        for a, s in zip(self.ins, self.stage):
            a.copy_(s)
        self.freed.record(cur)
        self.pending = False
        if next_inputs is not None:
            self.prefetch(next_inputs)
        self.run()
        for h, w in zip(self.out_host, self.outs):
            h.copy_(w, non_blocking=True)
        return self.out_host


class MiniBatchLJA:
    """Mini-batch streaming of one SUM/MEAN lifted join-aggregate whose source embeddings live
    in (pinned) HOST memory -- the paper's future-work "scaling for memory" (PAPER.md:1028-1031:
    relations beyond GPU memory, sampled / streamed in mini-batches).

    The group keys (T) are split into batches of `batch_groups` keys.  Per batch, built once
    (content caching): the E rows grouped into the batch, the source rows they reference S_b,
    and a device join index over S_b x T_b (dense groups).  A step streams, batch by batch:
        H2D   S_b's embedding rows (gathered into pinned staging on the host, copy stream)
        LJA   out_b = agg over the batch's join rows                       (A3, librnn)
        D2H   out_b into the host output
    with batch b+1's copy in flight during batch b's compute, so the device holds two batches
    of source rows, never the whole relation.  The backward streams dOut_b the same way and
    adds each batch's source-gradient rows into a device (or host) gradient with
    rnn_scatter_add_rows (rows of one batch are distinct; batches apply in order, so the
    result is deterministic and equals the single-shot LJA's up to summation order)."""

    def __init__(self, e_src, e_dst, s_key, t_key, z_host, agg="sum", batch_groups=65536,
                 device="cuda", e_weight=None):
        dev = self.device = torch.device(device)
        self.agg = agg
        e_src, e_dst = np.asarray(e_src, np.int64), np.asarray(e_dst, np.int64)
        s_key, t_key = np.asarray(s_key, np.int64), np.asarray(t_key, np.int64)
        self.z_host = z_host if isinstance(z_host, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(z_host, np.float32))
        if not self.z_host.is_pinned():
            self.z_host = self.z_host.pin_memory()
        self.d = d = self.z_host.shape[1]
        self.n_s = len(s_key)
        t_sorted = np.sort(t_key)
        s_order = np.argsort(s_key, kind="stable")
        self.batches = []
        max_rows = 1
        for b0 in range(0, len(t_sorted), batch_groups):
            tb = t_sorted[b0:b0 + batch_groups]
            rows = np.isin(e_dst, tb)
            es, ed = e_src[rows], e_dst[rows]
            # the batch's source relation: referenced S keys (present in S), ascending
            sk = np.unique(es)
            pos = np.searchsorted(s_key[s_order], sk)
            ok = (pos < len(s_key)) & (s_key[s_order][np.minimum(pos, len(s_key) - 1)] == sk)
            sk = sk[ok]
            srows = s_order[pos[ok]].astype(np.int64)          # rows of S in the host matrix
            cu = lambda a: torch.as_tensor(a).to(dev)
            idx = rnn.build_join_index(cu(es), cu(ed), cu(sk), cu(tb), dense_groups=True)
            w = None
            if e_weight is not None:
                w = cu(np.asarray(e_weight, np.float32)[rows])
            self.batches.append({"t_lo": b0, "n_t": len(tb), "idx": idx, "srows": srows,
                                 "srows_dev": cu(srows.astype(np.int32)), "w": w})
            max_rows = max(max_rows, len(srows))
        self.n_t = len(t_sorted)
        self.stage_h = [torch.empty(max_rows, d, dtype=torch.float32).pin_memory() for _ in range(2)]
        self.stage_d = [torch.empty(max_rows, d, dtype=torch.float32, device=dev) for _ in range(2)]
        self.out_d = [torch.empty(batch_groups, (d + 3) // 4 * 4, dtype=torch.float32,
                                  device=dev)[:, :d] for _ in range(2)]
        self.copy = torch.cuda.Stream(device=dev)
        self.ws = rnn.Workspace(dev)

    def _query(self, b, z):
        w = b["w"]
        return rnn.make_query("src", self.agg, src=z, edge=w, edge_mode=rnn.BY_ROW)

    def _stage(self, i, b):
        """Gather batch b's source rows on the host and start their H2D copy (copy stream)."""
        n = len(b["srows"])
        torch.index_select(self.z_host, 0, torch.from_numpy(b["srows"]), out=self.stage_h[i][:n])
        ev = torch.cuda.Event()
        with torch.cuda.stream(self.copy):
            self.copy.wait_stream(torch.cuda.current_stream())
            self.stage_d[i][:n].copy_(self.stage_h[i][:n], non_blocking=True)
            ev.record(self.copy)
        return ev

    def forward(self, out_host=None):
        """Streamed forward: returns the [n_t, d] output (host, T-key order)."""
        out = out_host if out_host is not None else torch.empty(self.n_t, self.d).pin_memory()
        cur = torch.cuda.current_stream()
        nxt = self._stage(0, self.batches[0]) if self.batches else None
        for k, b in enumerate(self.batches):
            i = k & 1
            cur.wait_event(nxt)
            if k + 1 < len(self.batches):
                nxt = self._stage(1 - i, self.batches[k + 1])
            n = len(b["srows"])
            z = self.stage_d[i][:n]
            o = self.out_d[i][: b["n_t"]]
            rnn.join_aggregate_fwd(b["idx"], self._query(b, z), out=o, ws=self.ws)
            out[b["t_lo"]:b["t_lo"] + b["n_t"]].copy_(o, non_blocking=True)
        torch.cuda.synchronize()
        return out

    def backward(self, d_out_host, d_src=None):
        """Streamed source gradient: d_src [n_s, d] (device) = sum over batches of each batch's
        LJA backward, scattered onto the batch's source rows."""
        dev = self.device
        d = self.d
        if d_src is None:
            d_src = torch.zeros(self.n_s, d, dtype=torch.float32, device=dev)
        dout_d = torch.empty(max(b["n_t"] for b in self.batches), d, dtype=torch.float32, device=dev)
        for k, b in enumerate(self.batches):
            n = len(b["srows"])
            ev = self._stage(0, b)
            dout_d[: b["n_t"]].copy_(d_out_host[b["t_lo"]:b["t_lo"] + b["n_t"]], non_blocking=True)
            torch.cuda.current_stream().wait_event(ev)
            q = self._query(b, self.stage_d[0][:n])
            g = rnn.join_aggregate_bwd(b["idx"], q, dout_d[: b["n_t"]], want_edge=False,
                                       want_dst=False, ws=self.ws)["src"]
            rnn.scatter_add_rows(d_src, g[:n], b["srows_dev"])
            torch.cuda.synchronize()
        return d_src


def _joint_keys(rel_idx, keys):
    """Composite S keys (relation index j, source key) of a union over relations: j << 56 | key
    (keys must lie in [0, 2^56))."""
    keys = np.asarray(keys, np.int64)
    if len(keys) and (keys.min() < 0 or keys.max() >= (1 << 56)):
        raise ValueError("joint softmax: keys must lie in [0, 2^56)")
    return (np.int64(rel_idx) << np.int64(56)) | keys


class HGTJointProgram(_Program):
    """HGT layer with the ORIGINAL HGT's joint softmax: the attention of target t normalises over
    the sources of EVERY relation phi into t's type at once (SURVEY sec 8c reading 3 / sec 8f
    item 2), instead of per relation then summing (HGTProgram, the paper's templated rule,
    PAPER.md:1351-1358, :1409).  It is one SOFTMAX LJA per target type over the UNION of the
    relations into it: the source relation is the stack of every relation's (K'_phi, M'_phi)
    rows, keyed by (phi, source key) -- the union of PAPER.md:451-460 with a relation tag --
    so no new kernel: per relation one projection writes its rows of the stack, one index per
    target type joins the union."""

    def __init__(self, mag: dict, device="cuda", prec="3xtf32", seed=7):
        dev = self.device = torch.device(device)
        self.prec = prec
        self.d, self.h = d, h = mag["d"], mag["heads"]
        types = list(mag["n"].keys())
        self.n = dict(mag["n"])
        self.rels = mag["rels"]
        par = hgt_parameters(mag, seed)
        self.col = par["col"]
        self.targets = par["targets"]
        self.H = {t: _dev_f32(mag["h"][t], dev) for t in types}
        Wt = par["W"]
        blk = lambda t, kind, key: Wt[t][self.col[(kind, key)][1] * d:(self.col[(kind, key)][1] + 1) * d]
        # per relation: W_km = [Wk; Wm] ([2d, d]); per target type: Wq
        self.Wkm = {name: _dev_f32(np.concatenate([blk(r["src_type"], "k", name),
                                                   blk(r["src_type"], "m", name)], 0), dev)
                    for name, r in self.rels.items()}
        self.Wq = {t: _dev_f32(blk(t, "q", t), dev) for t in self.targets}
        self.into = {t: [name for name, r in self.rels.items() if r["dst_type"] == t]
                     for t in self.targets}
        self.off = {}
        self.KM, self.dKM, self.Q, self.dQ, self.idx, self.q, self.lse = {}, {}, {}, {}, {}, {}, {}
        self.Ht = {t: _empty(self.n[t], d, dev) for t in self.targets}
        self.d_out = {t: _dev_f32(par["d_out"][t], dev) for t in self.targets}
        for t in self.targets:
            off, skeys, es, ed = 0, [], [], []
            for j, name in enumerate(self.into[t]):
                r = self.rels[name]
                self.off[name] = off
                off += self.n[r["src_type"]]
                skeys.append(_joint_keys(j, mag["key"][r["src_type"]]))
                es.append(_joint_keys(j, r["src"]))
                ed.append(np.asarray(r["dst"], np.int64))
            cu = lambda a: torch.as_tensor(np.concatenate(a)).to(dev)
            self.idx[t] = rnn.build_join_index(cu(es), cu(ed), cu(skeys),
                                               torch.as_tensor(mag["key"][t]).to(dev),
                                               dense_groups=True)
            self.KM[t] = _empty(off, 2 * d, dev)
            self.dKM[t] = _empty(off, 2 * d, dev)
            self.Q[t] = _empty(self.n[t], d, dev)
            self.dQ[t] = _empty(self.n[t], d, dev)
            self.lse[t] = torch.empty(max(self.n[t], 1), h, dtype=torch.float32, device=dev)
            self.q[t] = rnn.make_query("src", "softmax", src=self.KM[t][:, d:], src_key=self.KM[t][:, :d],
                                       dst=self.Q[t], heads=h, scale=1.0)
        self.dWkm = {name: torch.empty(2 * d, d, dtype=torch.float32, device=dev) for name in self.rels}
        self.dWq = {t: torch.empty(d, d, dtype=torch.float32, device=dev) for t in self.targets}
        self.dH = {t: _empty(self.n[t], d, dev) for t in types}
        self.dH_tmp = _empty(max(self.n.values()), d, dev)
        self.ws = rnn.Workspace(dev)
        self.ws_p = rnn.Workspace(dev)

    @property
    def join_rows_per_step(self):
        return sum(ix.n_join_rows for ix in self.idx.values())

    def lja_bytes(self):
        return {}

    def forward(self):
        d = self.d
        for name, r in self.rels.items():
            t, s = r["dst_type"], r["src_type"]
            o = self.off[name]
            rnn.project(self.H[s], self.Wkm[name], out=self.KM[t][o:o + self.n[s]], prec=self.prec)
        for t in self.targets:
            rnn.project(self.H[t], self.Wq[t], out=self.Q[t], prec=self.prec)
            rnn.join_aggregate_fwd(self.idx[t], self.q[t], out=self.Ht[t], lse=self.lse[t],
                                   ws=self.ws)
        return self.Ht

    def _add_dh(self, t, first):
        if first[t]:
            first[t] = False
        else:
            rnn.accumulate(self.dH[t], self.dH_tmp[: self.n[t]], beta=1.0)

    def backward(self):
        import ctypes as C
        d = self.d
        first = {t: True for t in self.dH}
        for t in self.targets:
            idx, q = self.idx[t], self.q[t]
            _, bb = rnn.lja_workspace_size(idx, q)
            w = self.ws.get(bb)
            dO = self.d_out[t]
            rnn._check(rnn.lib().rnn_join_aggregate_bwd(
                C.byref(idx.c), C.byref(q), rnn._ptr(self.Ht[t]), self.Ht[t].stride(0),
                rnn._ptr(self.lse[t]), rnn._ptr(dO), dO.stride(0),
                rnn._ptr(self.dKM[t][:, d:]), rnn._ptr(self.dKM[t][:, :d]), None,
                rnn._ptr(self.dQ[t]), rnn._ptr(w), w.numel(), rnn._stream()))
            dst = self.dH[t] if first[t] else self.dH_tmp[: self.n[t]]
            rnn.project_bwd(self.H[t], self.Wq[t], self.dQ[t], want_dx=True, prec=self.prec,
                            ws=self.ws_p, dx_out=dst, dw_out=self.dWq[t])
            self._add_dh(t, first)
        for name, r in self.rels.items():
            t, s = r["dst_type"], r["src_type"]
            o = self.off[name]
            dst = self.dH[s] if first[s] else self.dH_tmp[: self.n[s]]
            rnn.project_bwd(self.H[s], self.Wkm[name], self.dKM[t][o:o + self.n[s]], want_dx=True,
                            prec=self.prec, ws=self.ws_p, dx_out=dst, dw_out=self.dWkm[name])
            self._add_dh(s, first)
        return self.dWkm, self.dWq, self.dH


def hygnn_attention_parameters(d, seed=13):
    """Six d x d maps of the two attention hops (K, V, Q per hop), N(0, 1/d); the score scale
    1/sqrt(d/h) is folded into the key maps (reading 12)."""
    rng = np.random.default_rng(seed)
    return {k: (rng.standard_normal((d, d)) / np.sqrt(d)).astype(np.float32)
            for k in ("k1", "v1", "q1", "k2", "v2", "q2")}


class HypergraphAttentionProgram(_Program):
    """HyGNN's double attention (node-level then hyperedge-level attention;
    SURVEY sec 8f item 2) as two SOFTMAX lifted join-aggregates over the incidence relation:

        hop 1 (group by hyperedge e):  Eh(e) = sum_{v in e} softmax_v(<K1 x_v, Q1 h_e>) V1 x_v
        hop 2 (group by node v):       Xo(v) = sum_{e ∋ v} softmax_e(<K2 Eh_e, Q2 x_v>) V2 Eh_e

    with h_e the hyperedges' per-tuple (learnable) embeddings; K/V of a hop are one stacked
    tcgen05 projection.  Outputs are dense in key order (nodes / hyperedges without incidences
    aggregate to 0); the backward returns every weight gradient and d x, d h."""

    def __init__(self, hg: dict, device="cuda", prec="3xtf32", heads=8, seed=13):
        dev = self.device = torch.device(device)
        self.prec, self.h = prec, heads
        d = self.d = hg["nodes"]["x"].shape[1]
        nk = torch.as_tensor(hg["nodes"]["key"]).to(dev)
        hk = torch.as_tensor(hg["hyperedges"]["key"]).to(dev)
        iv = torch.as_tensor(hg["inc"]["node"]).to(dev)
        ih = torch.as_tensor(hg["inc"]["hyper"]).to(dev)
        self.idx1 = rnn.build_join_index(iv, ih, nk, hk, dense_groups=True)
        hk_sorted = torch.sort(hk).values
        self.idx2 = rnn.build_join_index(ih, iv, hk_sorted, nk, dense_groups=True)
        self.nv, self.ne = len(hg["nodes"]["key"]), len(hg["hyperedges"]["key"])
        self.X = _dev_f32(hg["nodes"]["x"], dev)
        self.E0 = _dev_f32(hg["hx"], dev)
        P = hygnn_attention_parameters(d, seed)
        scale = 1.0 / np.sqrt(d / heads)
        self.W = {k: _dev_f32(v * (scale if k[0] == "k" else 1.0), dev) for k, v in P.items()}
        self.Wkv1 = _dev_f32(np.concatenate([P["k1"] * scale, P["v1"]]), dev)
        self.Wkv2 = _dev_f32(np.concatenate([P["k2"] * scale, P["v2"]]), dev)
        self.KV1, self.KV2 = _empty(self.nv, 2 * d, dev), _empty(self.ne, 2 * d, dev)
        self.dKV1, self.dKV2 = _empty(self.nv, 2 * d, dev), _empty(self.ne, 2 * d, dev)
        self.Q1, self.Q2 = _empty(self.ne, d, dev), _empty(self.nv, d, dev)
        self.dQ1, self.dQ2 = _empty(self.ne, d, dev), _empty(self.nv, d, dev)
        self.Eh, self.Xo = _empty(self.ne, d, dev), _empty(self.nv, d, dev)
        self.dEh = _empty(self.ne, d, dev)
        self.lse1 = torch.empty(self.ne, heads, dtype=torch.float32, device=dev)
        self.lse2 = torch.empty(self.nv, heads, dtype=torch.float32, device=dev)
        self.q1 = rnn.make_query("src", "softmax", src=self.KV1[:, d:], src_key=self.KV1[:, :d],
                                 dst=self.Q1, heads=heads, scale=1.0)
        self.q2 = rnn.make_query("src", "softmax", src=self.KV2[:, d:], src_key=self.KV2[:, :d],
                                 dst=self.Q2, heads=heads, scale=1.0)
        self.d_out = _dev_f32(hg["d_out"][: self.nv], dev)
        self.dWkv1 = torch.empty(2 * d, d, dtype=torch.float32, device=dev)
        self.dWkv2 = torch.empty(2 * d, d, dtype=torch.float32, device=dev)
        self.dWq1 = torch.empty(d, d, dtype=torch.float32, device=dev)
        self.dWq2 = torch.empty(d, d, dtype=torch.float32, device=dev)
        self.dX, self.dX2 = _empty(self.nv, d, dev), _empty(self.nv, d, dev)
        self.dE0 = _empty(self.ne, d, dev)
        self.dEh_in = _empty(self.ne, d, dev)
        self.ws = rnn.Workspace(dev)
        self.ws_p = rnn.Workspace(dev)

    @property
    def join_rows_per_step(self):
        return self.idx1.n_join_rows + self.idx2.n_join_rows

    def lja_bytes(self):
        return {}

    def forward(self):
        rnn.project(self.X, self.Wkv1, out=self.KV1, prec=self.prec)
        rnn.project(self.E0, self.W["q1"], out=self.Q1, prec=self.prec)
        rnn.join_aggregate_fwd(self.idx1, self.q1, out=self.Eh, lse=self.lse1, ws=self.ws)
        rnn.project(self.Eh, self.Wkv2, out=self.KV2, prec=self.prec)
        rnn.project(self.X, self.W["q2"], out=self.Q2, prec=self.prec)
        rnn.join_aggregate_fwd(self.idx2, self.q2, out=self.Xo, lse=self.lse2, ws=self.ws)
        return self.Xo

    def _sm_bwd(self, idx, q, out, lse, d_out, dKV, dQ):
        import ctypes as C
        d = self.d
        _, bb = rnn.lja_workspace_size(idx, q)
        w = self.ws.get(bb)
        rnn._check(rnn.lib().rnn_join_aggregate_bwd(
            C.byref(idx.c), C.byref(q), rnn._ptr(out), out.stride(0), rnn._ptr(lse),
            rnn._ptr(d_out), d_out.stride(0), rnn._ptr(dKV[:, d:]), rnn._ptr(dKV[:, :d]), None,
            rnn._ptr(dQ), rnn._ptr(w), w.numel(), rnn._stream()))

    def backward(self):
        p = dict(want_dx=True, prec=self.prec, ws=self.ws_p)
        self._sm_bwd(self.idx2, self.q2, self.Xo, self.lse2, self.d_out, self.dKV2, self.dQ2)
        rnn.project_bwd(self.X, self.W["q2"], self.dQ2, dx_out=self.dX, dw_out=self.dWq2, **p)
        rnn.project_bwd(self.Eh, self.Wkv2, self.dKV2, dx_out=self.dEh, dw_out=self.dWkv2, **p)
        self._sm_bwd(self.idx1, self.q1, self.Eh, self.lse1, self.dEh, self.dKV1, self.dQ1)
        rnn.project_bwd(self.E0, self.W["q1"], self.dQ1, dx_out=self.dE0, dw_out=self.dWq1, **p)
        rnn.project_bwd(self.X, self.Wkv1, self.dKV1, dx_out=self.dX2, dw_out=self.dWkv1, **p)
        rnn.accumulate(self.dX, self.dX2, beta=1.0)
        return self.dX, self.dE0


class RGCNProgram(_Program):
    """R-GCN layer: a per-join-row transformation
    with one weight matrix per relation type,

        out(t) = W0 x_t + sum_r sum_{(s, t) in E_r} W_r x_s / |N_r(t)|.

    The paper applies W_r to every join row (no pushdown) and reports R-GCN ~30x slower than
    torch-rgcn.  By linearity W_r distributes over the per-relation mean, so
    here the transformation is moved ABOVE the aggregation instead: per relation one MEAN LJA
    of the raw features over sigma_{rel = r}(E) (the selection pushed into the index build)
    writes its column block of A = [x | mean_1 | ... | mean_R], and ONE tcgen05 GEMM
    out = A [W0 | W_1 | ... | W_R]^T applies every relation's map -- R d_in^2 d_out FLOPs per
    node instead of per join row, with the same result (oracle: the per-row definition)."""

    def __init__(self, g: dict, device="cuda", prec="3xtf32"):
        dev = self.device = torch.device(device)
        self.prec = prec
        keys = torch.as_tensor(g["nodes"]["key"]).to(dev)
        es = torch.as_tensor(g["edges"]["src"]).to(dev)
        ed = torch.as_tensor(g["edges"]["dst"]).to(dev)
        rel = torch.as_tensor(g["edges"]["rel"].astype(np.int64)).to(dev)
        self.R = R = g["n_rel"]
        self.n, self.d = g["nodes"]["x"].shape
        d, n = self.d, self.n
        self.X = _dev_f32(g["nodes"]["x"], dev)
        W = np.asarray(g["W"], np.float32)                     # [R + 1, d_out, d_in]
        self.d_out_w = W.shape[1]
        self.Wst = _dev_f32(np.concatenate(list(W), axis=1), dev)   # [d_out, (R + 1) d_in]
        self.idx = []
        for r in range(R):
            m = rnn.select_mask(rel, "==", r)
            self.idx.append(rnn.build_join_index(es, ed, keys, keys, dense_groups=True, e_mask=m))
        self.A = _empty(n, (R + 1) * d, dev)
        self.dA = _empty(n, (R + 1) * d, dev)
        self.out = _empty(n, self.d_out_w, dev)
        self.dWst = torch.empty(self.d_out_w, (R + 1) * d, dtype=torch.float32, device=dev)
        self.dX = _empty(n, d, dev)
        self.dX_r = _empty(n, d, dev)
        self.d_out = _dev_f32(g["d_out"], dev)
        # the self-loop block: row i of A holds x of the node whose key has rank i
        order = np.argsort(np.asarray(g["nodes"]["key"]), kind="stable").astype(np.int32)
        self.key_order = torch.as_tensor(order).to(dev)
        self.q = [rnn.make_query("src", "mean", src=self.X) for _ in range(R)]
        self.ws, self.ws_p = rnn.Workspace(dev), rnn.Workspace(dev)

    @property
    def join_rows_per_step(self):
        return sum(ix.n_join_rows for ix in self.idx)

    def lja_bytes(self):
        return {}

    def forward(self):
        d = self.d
        rnn.gather_rows(self.A[:, :d], self.X, self.key_order)          # x in key order
        for r in range(self.R):
            rnn.join_aggregate_fwd(self.idx[r], self.q[r], out=self.A[:, (r + 1) * d:(r + 2) * d],
                                   ws=self.ws)
        rnn.project(self.A, self.Wst, out=self.out, prec=self.prec)
        return self.out

    def backward(self):
        import ctypes as C
        d = self.d
        rnn.project_bwd(self.A, self.Wst, self.d_out, want_dx=True, prec=self.prec, ws=self.ws_p,
                        dx_out=self.dA, dw_out=self.dWst)
        # self-loop block: dA[:, :d] row i belongs to the node of key rank i
        self.dX.zero_()
        rnn.scatter_add_rows(self.dX, self.dA[:, :d], self.key_order)
        for r in range(self.R):
            idx, q = self.idx[r], self.q[r]
            _, bb = rnn.lja_workspace_size(idx, q)
            w = self.ws.get(bb)
            blk = self.dA[:, (r + 1) * d:(r + 2) * d]
            rnn._check(rnn.lib().rnn_join_aggregate_bwd(
                C.byref(idx.c), C.byref(q), None, 0, None, rnn._ptr(blk), blk.stride(0),
                rnn._ptr(self.dX_r), None, None, None, rnn._ptr(w), w.numel(), rnn._stream()))
            rnn.accumulate(self.dX, self.dX_r, beta=1.0)
        return self.dX, self.dWst
