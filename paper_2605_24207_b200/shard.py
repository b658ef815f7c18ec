"""Multi-GPU sharding of the lifted join-aggregate (BASELINE.json north_star).

The join relation is hash-partitioned by the GROUP BY key: owner(t) = splitmix64(t ^ seed) % P
(rnn_hash_partition).  Every group is reduced entirely on its owner, in the same within-group
order as on one GPU.  Per layer of a GCN:

    Z_own  = H_own W^T                                   (A2, owned rows only)
    Z_all  = all_gather(Z_own)                           (NCCL over NVLink; rank-major blocks)
    H'_own = LJA_fwd(index_r, src = Z_all, w)            (A3 over the rank's join rows)
  backward
    dZ_all = LJA_bwd(index_r, dH'_own)                   (A5: partial over referenced sources)
    dZ_own = reduce_scatter(dZ_all)                      (sum to the owners)
    dW     = all_reduce(H_own^T dZ_own),  dH_own = dZ_own W

Layout: rank r's block of the gathered source relation holds its owned node keys in
ascending order, padded to n_pad = max_r |owned_r| with sentinel keys that match no edge.
Because a layer's output rows are the owned keys in ascending order (every node has a
self-loop, so every owned node is a group), the SAME S-key layout serves every layer: one
join index per rank, built once (content caching).

This module holds the host-side partition plan (numpy, setup time) and the program; the
collectives are torch.distributed calls on the rank's process group (NCCL on the GPU box;
gloo works too, which the world-size-2 CPU tests use).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


class ShardPlan:
    """Which node keys and which edge rows rank `rank` of `P` owns (host, numpy).

    owner[i] = owning rank of node i (from rnn_hash_partition over the node keys)."""

    def __init__(self, node_keys, e_src, e_dst, owner, P, rank):
        keys = np.asarray(node_keys, np.int64)
        owner = np.asarray(owner, np.int64)
        self.P, self.rank = int(P), int(rank)
        self.owned_keys = [np.sort(keys[owner == r]) for r in range(self.P)]
        self.counts = np.array([len(k) for k in self.owned_keys], np.int64)
        self.n_pad = int(max(1, self.counts.max())) if len(keys) else 1
        lo = int(keys.min()) if len(keys) else 0
        n_all = self.P * self.n_pad
        if lo - n_all - 1 < np.iinfo(np.int64).min + 1:
            raise ValueError("node keys too close to INT64_MIN for sentinel padding")
        # sentinel keys (unique, below every real key) pad each rank's block
        s = np.empty(n_all, np.int64)
        for r in range(self.P):
            blk = s[r * self.n_pad:(r + 1) * self.n_pad]
            c = self.counts[r]
            blk[:c] = self.owned_keys[r]
            blk[c:] = lo - 1 - (r * self.n_pad + np.arange(self.n_pad - c))
        self.s_keys = s                                   # S relation of every layer (all ranks)
        self.my_keys = self.owned_keys[self.rank]         # T relation (= this rank's groups)
        # storage rows of this rank's nodes, in key order (to lay out the layer-1 features)
        order = np.argsort(keys, kind="stable")
        pos = np.searchsorted(keys[order], self.my_keys)
        self.my_rows = order[pos]
        # join rows owned here: the edge's group key (dst) is owned by this rank
        e_dst = np.asarray(e_dst, np.int64)
        ks = keys[order]
        j = np.searchsorted(ks, e_dst)
        j = np.clip(j, 0, max(len(ks) - 1, 0))
        present = (len(ks) > 0) & (ks[j] == e_dst) if len(ks) else np.zeros(len(e_dst), bool)
        e_owner = np.where(present, owner[order[j]] if len(ks) else 0, -1)
        mine = e_owner == self.rank
        self.e_src = np.asarray(e_src, np.int64)[mine]
        self.e_dst = e_dst[mine]


class HaloPlan:
    """Halo-only exchange of a hash-partitioned source relation (SURVEY sec 8e "Mitigations":
    every rank receives only the rows its join rows reference, not the whole relation;
    0.44x the all-gather rows at P = 8 on arxiv).  Built identically on every rank from the
    global relation (host, numpy, setup time).

    Rank r's source relation S_r = [its owned keys, padded to n_pad | halo keys it needs from
    rank q, q = 0..P-1, q != r, each ascending] -- its join index is built over S_r once.
      send_idx  int32 [sum_q send_counts[q]]: rows of r's owned block sent to q, q ascending
      send_counts[q] = |need(r <- ... q wants from r)|, recv_counts[q] = |need(q -> r)|"""

    def __init__(self, owned, n_pad, referenced, rank):
        P = len(owned)
        self.P, self.rank, self.n_pad = P, rank, n_pad
        pos = [{int(k): i for i, k in enumerate(o)} for o in owned]
        need = [[np.intersect1d(referenced[q], owned[o], assume_unique=True) if o != q
                 else np.zeros(0, np.int64) for o in range(P)] for q in range(P)]
        # need[q][o] = keys rank q needs from owner o
        self.recv_counts = [len(need[rank][o]) for o in range(P)]
        self.send_counts = [len(need[q][rank]) for q in range(P)]
        self.send_idx = np.concatenate([np.array([pos[rank][int(k)] for k in need[q][rank]],
                                                 np.int32) for q in range(P)]) \
            if sum(self.send_counts) else np.zeros(0, np.int32)
        self.halo_keys = np.concatenate([need[rank][o] for o in range(P)]) \
            if sum(self.recv_counts) else np.zeros(0, np.int64)
        self.n_halo = len(self.halo_keys)
        # bytes moved per exchanged row set, against the all-gather's (P - 1) n_pad rows
        self.rows_recv = int(sum(self.recv_counts))
        self.rows_allgather = (P - 1) * n_pad

    def s_keys(self, own_block_keys):
        return np.concatenate([own_block_keys, self.halo_keys])


def _all_to_all_rows(out, x, out_splits, in_splits, group=None):
    """all_to_all_single over rows; backends without it for device tensors (gloo + CUDA, the
    1-GPU functional tests) exchange through host copies."""
    try:
        dist.all_to_all_single(out, x, output_split_sizes=out_splits, input_split_sizes=in_splits,
                               group=group)
    except (RuntimeError, NotImplementedError):
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(o, x.cpu(), output_split_sizes=out_splits,
                               input_split_sizes=in_splits, group=group)
        out.copy_(o)


def halo_exchange_fwd(be, plan, Zs, send_buf, group=None):
    """Zs [n_pad + n_halo, d]: rows [:n_pad] are this rank's own (filled); the halo rows are
    received from their owners (all_to_all_single of the gathered send rows)."""
    n_pad = plan.n_pad
    if plan.P == 1 or not dist.is_initialized():
        return
    if len(plan.send_idx):
        be.gather_rows(send_buf, Zs[:n_pad], plan.send_idx_dev)
    _all_to_all_rows(Zs[n_pad:], send_buf, plan.recv_counts, plan.send_counts, group)


def halo_exchange_bwd(be, plan, dZs, back_buf, group=None):
    """dZs [n_pad + n_halo, d]: partial source gradients of own and halo rows; the halo rows'
    partials go back to their owners and are added onto the owned rows they came from (one
    scatter per destination: rows within one destination's list are distinct -> no collisions,
    fixed order -> deterministic).  Leaves the result in dZs[:n_pad]."""
    n_pad = plan.n_pad
    if plan.P == 1 or not dist.is_initialized():
        return
    _all_to_all_rows(back_buf, dZs[n_pad:], plan.send_counts, plan.recv_counts, group)
    off = 0
    for q, c in enumerate(plan.send_counts):
        if c:
            be.scatter_add_rows(dZs[:n_pad], back_buf[off:off + c], plan.send_idx_dev[off:off + c])
        off += c


def all_gather_rows(out, x, group=None):
    """out[P * n, d] <- concat over ranks of x[n, d] (contiguous tensors)."""
    if not dist.is_initialized():
        out.copy_(x)
        return
    try:
        dist.all_gather_into_tensor(out, x, group=group)
    except (RuntimeError, NotImplementedError):
        # backends without the fused variant (gloo + CUDA tensors): list all-gather
        n = x.shape[0]
        parts = [out[r * n:(r + 1) * n] for r in range(dist.get_world_size(group))]
        bufs = [torch.empty_like(x) for _ in parts]
        dist.all_gather(bufs, x.contiguous(), group=group)
        for p, b in zip(parts, bufs):
            p.copy_(b)


def reduce_scatter_rows(out, x, group=None):
    """out[n, d] <- sum over ranks of the rank-th block of x[P * n, d]."""
    if not dist.is_initialized():
        out.copy_(x)
        return
    try:
        dist.reduce_scatter_tensor(out, x, group=group)
    except (RuntimeError, NotImplementedError):
        # backends without reduce_scatter (gloo + CUDA tensors): all-reduce, keep own block
        y = x.clone()
        dist.all_reduce(y, group=group)
        r = dist.get_rank(group)
        out.copy_(y[r * out.shape[0]:(r + 1) * out.shape[0]])


class ShardedGCNProgram:
    """L-layer GCN step over P ranks (hash partition by group key, one process per GPU).

    backend: the compute primitives (``RnnBackend`` = librnn.so on this rank's GPU; the CPU
    tests plug in an fp64 backend built from the oracle to check the sharding logic)."""

    def __init__(self, graph: dict, backend=None, group=None, seed=0x5EED, prec="3xtf32",
                 halo=True):
        self.group = group
        self.P = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        be = self.be = backend if backend is not None else RnnBackend(prec=prec)
        nodes, edges = graph["nodes"], graph["edges"]
        keys = np.asarray(nodes["key"], np.int64)
        owner = be.hash_partition(keys, self.P, seed)
        plan = self.plan = ShardPlan(keys, edges["src"], edges["dst"], owner, self.P, self.rank)
        # halo exchange (default): only the referenced source rows cross the links
        self.halo = None
        if halo and self.P > 1:
            e_src, e_dst = np.asarray(edges["src"], np.int64), np.asarray(edges["dst"], np.int64)
            o_dst = _owner_of(keys, owner, e_dst)
            referenced = [np.intersect1d(np.unique(e_src[o_dst == q]), keys) for q in range(self.P)]
            self.halo = HaloPlan(plan.owned_keys, plan.n_pad, referenced, self.rank)
            self.halo.send_idx_dev = be.index_i32(self.halo.send_idx)
        # layer widths padded to a multiple of 4 (rnn_project / the LJA need ld % 4 == 0 and
        # the collectives contiguous rows): W, features and d_out are zero-padded, so padded
        # columns stay exactly 0 and the real columns are unchanged (Cora: 1,433 -> 16 -> 7)
        self.dims = list(graph["dims"])
        dp = self.dims_pad = [(x + 3) // 4 * 4 for x in self.dims]
        self.L = len(self.dims) - 1
        n_pad, P = plan.n_pad, self.P
        self.n_own = int(plan.counts[self.rank])
        r0 = self.rank * n_pad
        if self.halo is not None:
            s_keys = self.halo.s_keys(plan.s_keys[r0:r0 + n_pad])
        else:
            s_keys = plan.s_keys
        self.n_s = len(s_keys)
        self.idx = be.build_index(plan.e_src, plan.e_dst, s_keys, plan.my_keys)
        assert be.n_groups(self.idx) == self.n_own, "every owned node needs a self-loop"
        # normalisation: deg(s) from its owner (all-gathered group sizes, setup time)
        own_idx = be.build_index(plan.e_src, plan.e_dst, plan.s_keys, plan.my_keys) \
            if self.halo is not None else self.idx
        own_deg = be.zeros_i32(n_pad)
        be.group_sizes(own_idx, own_deg)
        all_deg = be.zeros_i32(P * n_pad)
        all_gather_rows(all_deg, own_deg, group)
        if self.halo is not None:
            # S-row degrees of the halo layout: own block, then every halo key's owner row
            pos = {int(k): i for i, k in enumerate(plan.s_keys)}
            rows = np.concatenate([np.arange(r0, r0 + n_pad),
                                   [pos[int(k)] for k in self.halo.halo_keys]]).astype(np.int64)
            all_deg = all_deg[torch.as_tensor(rows, device=all_deg.device)].contiguous()
        self.w = be.gcn_norm_src_deg(self.idx, all_deg)
        # activations (rows >= n_own stay zero: padding of the gathered blocks)
        x0 = np.zeros((n_pad, dp[0]), np.float32)
        x0[: self.n_own, : self.dims[0]] = np.asarray(nodes["x"], np.float32)[plan.my_rows]
        self.H = [be.tensor(x0)] + [be.zeros(n_pad, dp[l + 1]) for l in range(self.L)]
        Wp = []
        for l, w in enumerate(graph["W"]):
            wp = np.zeros((dp[l + 1], dp[l]), np.float32)
            wp[: self.dims[l + 1], : self.dims[l]] = np.asarray(w, np.float32)
            Wp.append(be.tensor(wp))
        self.W = Wp
        self.Z = [be.zeros(n_pad, dp[l + 1]) for l in range(self.L)]
        # the layer's source relation: all-gathered [P n_pad] or own + halo [n_pad + n_halo]
        self.Zall = [be.zeros(self.n_s, dp[l + 1]) for l in range(self.L)]
        self.dZall = [be.zeros(self.n_s, dp[l + 1]) for l in range(self.L)]
        if self.halo is not None:
            self.send = [be.zeros(max(len(self.halo.send_idx), 1), dp[l + 1]) for l in range(self.L)]
        self.dZ = [be.zeros(n_pad, dp[l + 1]) for l in range(self.L)]
        self.dH = [be.zeros(n_pad, dp[l]) for l in range(self.L)]
        self._dW = [be.zeros(dp[l + 1], dp[l]) for l in range(self.L)]
        self.dW = [w[: self.dims[l + 1], : self.dims[l]] for l, w in enumerate(self._dW)]
        # upstream gradient of the owned output rows (the oracle's d_out row of each group)
        G_all = np.sort(keys)
        rank_of = np.searchsorted(G_all, plan.my_keys)
        d_out = np.zeros((n_pad, dp[-1]), np.float32)
        d_out[: self.n_own, : self.dims[-1]] = np.asarray(graph["d_out"], np.float32)[rank_of, : self.dims[-1]]
        self.d_out = be.tensor(d_out)
        # O7 node epilogue (bias then ReLU on hidden layers, bias on the last), when the graph
        # carries biases: fused into the owned rows' LJA store; d bias all-reduced
        self.bias = None
        if graph.get("b") is not None:
            self.bias, self.dP, self.db = [], [], []
            for l in range(self.L):
                bp = np.zeros((1, dp[l + 1]), np.float32)
                bp[0, : self.dims[l + 1]] = np.asarray(graph["b"][l], np.float32)
                self.bias.append(be.tensor(bp)[0])
                self.dP.append(be.zeros(n_pad, dp[l + 1]))
                self.db.append(be.zeros(1, dp[l + 1])[0])
        self.timers = None

    def _act(self, l):
        return "relu" if l < self.L - 1 else "none"

    @property
    def join_rows_per_step(self):
        """Join rows this rank processes per step (all layers)."""
        return self.L * self.be.n_join_rows(self.idx)

    def roof_model(self):
        from .programs import _sum_bwd_bytes, _sum_bytes
        d = self.dims_pad[1:]
        return {"lja_fwd": {"bound": "hbm", "amount": float(np.mean([_sum_bytes(self.idx, x, True) for x in d]))},
                "lja_bwd": {"bound": "hbm", "amount": float(np.mean([_sum_bwd_bytes(self.idx, x, True) for x in d]))}}

    def host_io(self):
        return [self.H[0], self.d_out], list(self._dW)

    def _t(self, name):
        if self.timers is None:
            return
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.timers.setdefault(name, []).append(e)

    def forward(self):
        be, g = self.be, self.group
        for l in range(self.L):
            self._t("proj_fwd")
            be.project(self.H[l], self.W[l], self.Z[l])
            self._t("proj_fwd_end")
            self._t("allgather")
            if self.halo is not None:
                n_pad = self.plan.n_pad
                self.Zall[l][:n_pad].copy_(self.Z[l])
                halo_exchange_fwd(be, self.halo, self.Zall[l], self.send[l][: len(self.halo.send_idx)], g)
            else:
                all_gather_rows(self.Zall[l], self.Z[l], g)
            self._t("allgather_end")
            self._t("lja_fwd")
            if self.bias is not None:
                be.lja_fwd_epi(self.idx, self.Zall[l], self.w, self.H[l + 1], self.bias[l],
                               self._act(l))
            else:
                be.lja_fwd(self.idx, self.Zall[l], self.w, self.H[l + 1])
            self._t("lja_fwd_end")
        return self.H[-1]

    def backward(self):
        be, g = self.be, self.group
        dY = self.d_out
        for l in reversed(range(self.L)):
            if self.bias is not None:
                be.epilogue_bwd(dY, self.H[l + 1], self.bias[l], self._act(l), self.dP[l],
                                self.db[l], self.n_own)
                if self.P > 1:
                    dist.all_reduce(self.db[l], group=g)
                dY = self.dP[l]
            self._t("lja_bwd")
            be.lja_bwd_src(self.idx, self.Zall[l], self.w, dY, self.dZall[l])
            self._t("lja_bwd_end")
            self._t("reduce_scatter")
            if self.halo is not None:
                n_pad = self.plan.n_pad
                halo_exchange_bwd(be, self.halo, self.dZall[l], self.send[l][: len(self.halo.send_idx)], g)
                self.dZ[l].copy_(self.dZall[l][:n_pad])
            else:
                reduce_scatter_rows(self.dZ[l], self.dZall[l], g)
            self._t("reduce_scatter_end")
            self._t("proj_bwd")
            be.project_bwd(self.H[l], self.W[l], self.dZ[l], self.dH[l], self._dW[l])
            self._t("proj_bwd_end")
            if self.P > 1:
                dist.all_reduce(self._dW[l], group=g)
            dY = self.dH[l]
        return self.dW, self.dH[0]

    def step(self):
        self.forward()
        return self.backward()

    # ---- gathering results for checks (host) ----
    def owned_output(self):
        return self.be.numpy(self.H[-1])[: self.n_own, : self.dims[-1]]

    def owned_dx(self):
        return self.be.numpy(self.dH[0])[: self.n_own, : self.dims[0]]


class RnnBackend:
    """The product backend: every primitive is a librnn.so call on the current CUDA device."""

    def __init__(self, prec="3xtf32", device=None):
        from . import rnn
        self.rnn = rnn
        self.prec = prec
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.ws = rnn.Workspace(self.dev)
        self.ws_p = rnn.Workspace(self.dev)
        self._q = {}

    def tensor(self, a):
        a = np.asarray(a, np.float32)
        ld = (a.shape[1] + 3) // 4 * 4
        t = torch.zeros(a.shape[0], ld, dtype=torch.float32, device=self.dev)
        t[:, : a.shape[1]] = torch.from_numpy(a).to(self.dev)
        return t[:, : a.shape[1]] if ld != a.shape[1] else t

    def zeros(self, n, d):
        # collectives need contiguous buffers: keep d a multiple of 4 in the product configs
        return torch.zeros(n, d, dtype=torch.float32, device=self.dev)

    def zeros_i32(self, n):
        return torch.zeros(n, dtype=torch.int32, device=self.dev)

    def numpy(self, t):
        return t.detach().cpu().numpy()

    def hash_partition(self, keys, P, seed):
        k = torch.as_tensor(np.asarray(keys, np.int64), device=self.dev)
        return self.rnn.hash_partition(k, P, seed).cpu().numpy()

    def build_index(self, e_src, e_dst, s_keys, t_keys, dense=False):
        cu = lambda a: torch.as_tensor(np.asarray(a, np.int64), device=self.dev)
        return self.rnn.build_join_index(cu(e_src), cu(e_dst), cu(s_keys), cu(t_keys),
                                         dense_groups=dense)

    def n_groups(self, idx):
        return idx.n_groups

    def n_join_rows(self, idx):
        return idx.n_join_rows

    def group_sizes(self, idx, out):
        self.rnn.group_sizes(idx, out=out)

    def gcn_norm_src_deg(self, idx, deg):
        return self.rnn.gcn_norm_src_deg(idx, deg)

    def _query(self, idx, Z, w):
        key = (id(idx), Z.data_ptr(), w.data_ptr())
        q = self._q.get(key)
        if q is None:
            q = self._q[key] = self.rnn.make_query("src", "sum", src=Z, edge=w,
                                                   edge_mode=self.rnn.BY_POSITION)
        return q

    def _query_agg(self, idx, Z, agg):
        key = (id(idx), Z.data_ptr(), agg)
        q = self._q.get(key)
        if q is None:
            q = self._q[key] = self.rnn.make_query("src", agg, src=Z)
        return q

    def lja_fwd_agg(self, idx, Z, agg, out):
        self.rnn.join_aggregate_fwd(idx, self._query_agg(idx, Z, agg), out=out, ws=self.ws)

    def lja_bwd_src_agg(self, idx, Z, agg, d_out, d_src):
        from .programs import _lja_src_grad
        _lja_src_grad(idx, self._query_agg(idx, Z, agg), d_out, d_src, self.ws)

    def n_src_rows(self, idx):
        return idx.n_src_rows

    def fill_zero(self, t):
        t.zero_()

    def accumulate(self, out, x, beta):
        self.rnn.accumulate(out, x, beta=beta)

    # ---- DHN (A6) ----
    def build_dhn_index(self, e_src, e_dst, s_keys):
        """Replicated adjacency Edge(n, v) over the gathered node layout: S = T = s_keys
        (rank-major blocks), dense groups in key order."""
        cu = lambda a: torch.as_tensor(np.asarray(a, np.int64), device=self.dev)
        k = cu(s_keys)
        return self.rnn.build_join_index(cu(e_src), cu(e_dst), k, k, dense_groups=True)

    def dhn_groups(self, idx):
        """(group keys, T row of every group) on the host."""
        return self.numpy(idx.group_key), self.numpy(idx.group_dst_row)

    def dhn_symmetric(self, idx):
        from .programs import edge_is_symmetric
        return edge_is_symmetric(idx)

    def index_i32(self, a):
        return torch.as_tensor(np.asarray(a, np.int32), device=self.dev)

    def gather_rows(self, out, x, idx):
        self.rnn.gather_rows(out, x, idx)

    def scatter_add_rows(self, y, x, idx):
        self.rnn.scatter_add_rows(y, x, idx)

    def dhn_fwd(self, idx, k, f, roots, out, walk_sum):
        self.rnn.dhn_fwd(idx, k, f, out=out, ws=self.ws, walk_sum=walk_sum, roots=roots)

    def dhn_bwd(self, idx, k, f, roots, d_out, walk_sum, d_f, symmetric):
        self.rnn.dhn_bwd(idx, k, f, d_out, d_f=d_f, ws=self.ws, walk_sum=walk_sum,
                         symmetric=symmetric, roots=roots)

    def dhn_rows(self, idx, roots, ks):
        """Edge rows + exact closed-walk counts of the listed roots (rnn_dhn_count)."""
        tot = 0
        r = roots.long()
        for k in ks:
            tot += int(self.rnn.dhn_count(idx, k)[r].sum().item())
        return tot

    def lja_sm_fwd(self, idx, M, K, Q, heads, out, lse):
        q = self.rnn.make_query("src", "softmax", src=M, src_key=K, dst=Q, heads=heads, scale=1.0)
        self.rnn.join_aggregate_fwd(idx, q, out=out, lse=lse, ws=self.ws)

    def lja_sm_bwd(self, idx, M, K, Q, heads, out, lse, d_out, dM, dK, dQ):
        import ctypes as C
        rnn = self.rnn
        q = rnn.make_query("src", "softmax", src=M, src_key=K, dst=Q, heads=heads, scale=1.0)
        _, bb = rnn.lja_workspace_size(idx, q)
        w = self.ws.get(bb)
        rnn._check(rnn.lib().rnn_join_aggregate_bwd(
            C.byref(idx.c), C.byref(q), rnn._ptr(out), out.stride(0), rnn._ptr(lse),
            rnn._ptr(d_out), d_out.stride(0), rnn._ptr(dM), rnn._ptr(dK), None, rnn._ptr(dQ),
            rnn._ptr(w), w.numel(), rnn._stream()))

    def project(self, X, W, out):
        self.rnn.project(X, W, out=out, prec=self.prec)

    def lja_fwd(self, idx, Z, w, out):
        self.rnn.join_aggregate_fwd(idx, self._query(idx, Z, w), out=out, ws=self.ws)

    def lja_fwd_epi(self, idx, Z, w, out, bias, act):
        G = idx.n_groups
        epi = self.rnn.make_epilogue(bias=bias, act=act)
        self.rnn.join_aggregate_fwd_epi(idx, self._query(idx, Z, w), epi, out=out[:G], ws=self.ws)

    def epilogue_bwd(self, dy, y, bias, act, dx, db, rows):
        """dx / db over the first `rows` (owned) rows; padding rows of dx are left 0."""
        epi = self.rnn.make_epilogue(bias=bias, act=act)
        self.rnn.epilogue_bwd(dy[:rows], y[:rows], epi, dx=dx[:rows], ws=self.ws, db_out=db)

    def lja_bwd_src(self, idx, Z, w, d_out, d_src):
        from .programs import _lja_src_grad
        _lja_src_grad(idx, self._query(idx, Z, w), d_out, d_src, self.ws)

    def project_bwd(self, X, W, dY, dX, dW):
        self.rnn.project_bwd(X, W, dY, want_dx=True, prec=self.prec, ws=self.ws_p, dx_out=dX,
                             dw_out=dW)


def block_layout(keys, owner, P):
    """Rank-major padded layout of one relation over P ranks: rank r's block holds its owned
    keys ascending, padded to n_pad = max_r |owned_r| with unique sentinel keys below every
    real key (they match no join row).  Returns (owned keys per rank, n_pad, s_keys [P*n_pad])."""
    keys = np.asarray(keys, np.int64)
    owner = np.asarray(owner, np.int64)
    owned = [np.sort(keys[owner == r]) for r in range(P)]
    n_pad = int(max(1, max(len(k) for k in owned))) if len(keys) else 1
    lo = int(keys.min()) if len(keys) else 0
    if lo - P * n_pad - 1 < np.iinfo(np.int64).min + 1:
        raise ValueError("keys too close to INT64_MIN for sentinel padding")
    s = np.empty(P * n_pad, np.int64)
    for r in range(P):
        blk = s[r * n_pad:(r + 1) * n_pad]
        c = len(owned[r])
        blk[:c] = owned[r]
        blk[c:] = lo - 1 - (r * n_pad + np.arange(n_pad - c))
    return owned, n_pad, s


def _owner_of(rel_keys, owner, query):
    """Owning rank of each query key (-1 if the key is not in the relation: dangling)."""
    rel_keys = np.asarray(rel_keys, np.int64)
    o = np.argsort(rel_keys, kind="stable")
    ks = rel_keys[o]
    q = np.asarray(query, np.int64)
    if len(ks) == 0:
        return np.full(len(q), -1, np.int64)
    j = np.clip(np.searchsorted(ks, q), 0, len(ks) - 1)
    return np.where(ks[j] == q, np.asarray(owner, np.int64)[o[j]], -1)


class ShardedHypergraphProgram:
    """Two-hop hypergraph layer (config 4; O8) over P ranks, one exchange per hop:

        Z_own   = X_own Theta^T                                    (owned nodes)
        Z_all   = all_gather(Z_own)
        Eh_own  = LJA_sum(Inc rows of owned hyperedges, Z_all)      hop 1, group by hyperedge
        Eh_all  = all_gather(Eh_own)
        Xo_own  = LJA_mean(Inc rows of owned nodes, Eh_all)         hop 2, group by node
      backward: hop 2 source grads over all hyperedges -> reduce_scatter -> hop 1 source grads
      over all nodes -> reduce_scatter -> projection backward, all_reduce(dTheta).

    Both hops use dense groups over the rank's owned keys (key order), so a hop's output block
    is exactly the next hop's all-gather block; nodes without incidences output 0 (MEAN of an
    empty multiset, reading #4's dense mode)."""

    def __init__(self, hg: dict, backend=None, group=None, seed=0x5EED, prec="3xtf32"):
        self.group = group
        self.P = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        be = self.be = backend if backend is not None else RnnBackend(prec=prec)
        P, r = self.P, self.rank
        nk = np.asarray(hg["nodes"]["key"], np.int64)
        hk = np.asarray(hg["hyperedges"]["key"], np.int64)
        iv = np.asarray(hg["inc"]["node"], np.int64)
        ih = np.asarray(hg["inc"]["hyper"], np.int64)
        ov = be.hash_partition(nk, P, seed)
        oe = be.hash_partition(hk, P, seed)
        v_owned, self.nv_pad, v_s = block_layout(nk, ov, P)
        e_owned, self.ne_pad, e_s = block_layout(hk, oe, P)
        self.my_v, self.my_e = v_owned[r], e_owned[r]
        self.nv, self.ne = len(self.my_v), len(self.my_e)
        m1 = _owner_of(hk, oe, ih) == r          # hop 1: incidences of owned hyperedges
        m2 = _owner_of(nk, ov, iv) == r          # hop 2: incidences of owned nodes
        self.idx1 = be.build_index(iv[m1], ih[m1], v_s, self.my_e, dense=True)
        self.idx2 = be.build_index(ih[m2], iv[m2], e_s, self.my_v, dense=True)
        d = int(np.asarray(hg["nodes"]["x"]).shape[1])
        self.d = d
        order = np.argsort(nk, kind="stable")
        self.my_rows = order[np.searchsorted(nk[order], self.my_v)]
        x = np.zeros((self.nv_pad, d), np.float32)
        x[: self.nv] = np.asarray(hg["nodes"]["x"], np.float32)[self.my_rows]
        self.X = be.tensor(x)
        self.theta = be.tensor(np.asarray(hg["theta"], np.float32))
        self.Z = be.zeros(self.nv_pad, d)
        self.Zall = be.zeros(P * self.nv_pad, d)
        self.Eh = be.zeros(self.ne_pad, d)
        self.Ehall = be.zeros(P * self.ne_pad, d)
        self.Xo = be.zeros(self.nv_pad, d)
        self.dEhall = be.zeros(P * self.ne_pad, d)
        self.dEh = be.zeros(self.ne_pad, d)
        self.dZall = be.zeros(P * self.nv_pad, d)
        self.dZ = be.zeros(self.nv_pad, d)
        self.dX = be.zeros(self.nv_pad, d)
        self.dTheta = be.zeros(d, d)
        # upstream gradient: the single-process program's d_out row of each node group (groups
        # = nodes with >= 1 incidence, ascending key); nodes without incidences get 0
        present = np.unique(iv[np.isin(iv, nk) & np.isin(ih, hk)])
        g_pos = np.searchsorted(present, self.my_v)
        has = (g_pos < len(present)) & (present[np.minimum(g_pos, max(len(present) - 1, 0))] == self.my_v) \
            if len(present) else np.zeros(self.nv, bool)
        dout = np.zeros((self.nv_pad, d), np.float32)
        dout[: self.nv][has] = np.asarray(hg["d_out"], np.float32)[g_pos[has], :d]
        self.d_out = be.tensor(dout)
        self.timers = None

    @property
    def join_rows_per_step(self):
        return self.be.n_join_rows(self.idx1) + self.be.n_join_rows(self.idx2)

    def roof_model(self):
        from .programs import _sum_bwd_bytes, _sum_bytes
        i1, i2, d = self.idx1, self.idx2, self.d
        return {"lja_fwd": {"bound": "hbm", "amount": (_sum_bytes(i1, d) + _sum_bytes(i2, d, mean=True)) / 2},
                "lja_bwd": {"bound": "hbm", "amount": (_sum_bwd_bytes(i1, d) + _sum_bwd_bytes(i2, d, mean=True)) / 2}}

    def host_io(self):
        return [self.X, self.d_out], [self.dTheta]

    def _t(self, name):
        if self.timers is None:
            return
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.timers.setdefault(name, []).append(e)

    def forward(self):
        be, g = self.be, self.group
        self._t("proj_fwd")
        be.project(self.X, self.theta, self.Z)
        self._t("proj_fwd_end")
        all_gather_rows(self.Zall, self.Z, g)
        self._t("lja_fwd")
        be.lja_fwd_agg(self.idx1, self.Zall, "sum", self.Eh[: self.ne])
        self._t("lja_fwd_end")
        all_gather_rows(self.Ehall, self.Eh, g)
        self._t("lja_fwd")
        be.lja_fwd_agg(self.idx2, self.Ehall, "mean", self.Xo[: self.nv])
        self._t("lja_fwd_end")
        return self.Xo

    def backward(self):
        be, g = self.be, self.group
        self._t("lja_bwd")
        be.lja_bwd_src_agg(self.idx2, self.Ehall, "mean", self.d_out, self.dEhall)
        self._t("lja_bwd_end")
        reduce_scatter_rows(self.dEh, self.dEhall, g)
        self._t("lja_bwd")
        be.lja_bwd_src_agg(self.idx1, self.Zall, "sum", self.dEh, self.dZall)
        self._t("lja_bwd_end")
        reduce_scatter_rows(self.dZ, self.dZall, g)
        self._t("proj_bwd")
        be.project_bwd(self.X, self.theta, self.dZ, self.dX, self.dTheta)
        self._t("proj_bwd_end")
        if self.P > 1:
            dist.all_reduce(self.dTheta, group=g)
        return self.dTheta, self.dX

    def step(self):
        self.forward()
        return self.backward()

    def owned_output(self):
        return self.be.numpy(self.Xo)[: self.nv]

    def owned_dx(self):
        return self.be.numpy(self.dX)[: self.nv]


class ShardedHGTProgram:
    """One HGT layer (config 3) over P ranks.  Every node type is hash-partitioned by key;
    each relation's join rows live on the owner of their TARGET key (the GROUP BY key), with
    dense groups over the rank's owned target keys.  Per step:

        KM_own[t] = H_own[t] Wkm[t]^T               stacked K', M' blocks, owned rows
        Q_own[t]  = H_own[t] Wq[t]^T                 the target type's queries (stay local)
        KM_all[s] = all_gather(KM_own[s])            for every source type s: ONLY K'/M'
        O_phi     = softmax-LJA(K' = KM_all[s][k], M' = KM_all[s][m], Q = Q_own[t])
        Ht[t]     = sum_phi O_phi                    (rnn_accumulate)
      backward: per phi dK', dM' over all source rows into dKM_all[s] (disjoint column
      blocks) and dQ summed into dQ_own[t]; reduce_scatter(dKM_all[s]) added to dKM_own[s];
      both projection backwards on owned rows; all_reduce(dW[t])."""

    def __init__(self, mag: dict, backend=None, group=None, seed=0x5EED, prec="3xtf32",
                 param_seed=7, halo=True):
        from .programs import hgt_parameters
        self.group = group
        self.P = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        be = self.be = backend if backend is not None else RnnBackend(prec=prec)
        P, r = self.P, self.rank
        self.d, self.h = d, h = mag["d"], mag["heads"]
        par = hgt_parameters(mag, param_seed)
        self.blocks, self.col, self.targets = par["blocks"], par["col"], par["targets"]
        self.rels = mag["rels"]
        types = list(self.blocks)
        self.owner, self.n_pad, self.s_keys, self.my_keys, self.my_rows = {}, {}, {}, {}, {}
        for t in types:
            k = np.asarray(mag["key"][t], np.int64)
            o = be.hash_partition(k, P, seed)
            owned, self.n_pad[t], self.s_keys[t] = block_layout(k, o, P)
            self.owner[t] = o
            self.my_keys[t] = owned[r]
            order = np.argsort(k, kind="stable")
            self.my_rows[t] = order[np.searchsorted(k[order], owned[r])]
        self.n_own = {t: len(self.my_keys[t]) for t in types}
        self.sources = sorted({x["src_type"] for x in self.rels.values()})
        self.H, self.W, self.dW, self.dH, self.dH2 = {}, {}, {}, {}, {}
        self.Y, self.dY, self.Yq, self.dYq = {}, {}, {}, {}      # Y / dY: the K'/M' blocks
        self.Yall, self.dYall, self.R = {}, {}, {}
        self.nkm = {t: sum(k != "q" for k, _ in self.blocks[t]) for t in types}
        for t in types:
            nb, nkm = len(self.blocks[t]), self.nkm[t]
            x = np.zeros((self.n_pad[t], d), np.float32)
            x[: self.n_own[t]] = np.asarray(mag["h"][t], np.float32)[self.my_rows[t]]
            self.H[t] = be.tensor(x)
            self.W[t] = be.tensor(par["W"][t])
            self.dW[t] = be.zeros(nb * d, d)
            self.dH[t] = be.zeros(self.n_pad[t], d)
            self.dH2[t] = be.zeros(self.n_pad[t], d)
            if nkm:
                self.Y[t] = be.zeros(self.n_pad[t], nkm * d)
                self.dY[t] = be.zeros(self.n_pad[t], nkm * d)
            if nkm < nb:
                self.Yq[t] = be.zeros(self.n_pad[t], d)
                self.dYq[t] = be.zeros(self.n_pad[t], d)
        # halo exchange per source type (default at P > 1): rank r receives only the K'/M'
        # rows its join rows reference (union over the relations leaving the type)
        self.halo = {}
        if halo and P > 1:
            for t in self.sources:
                k = np.asarray(mag["key"][t], np.int64)
                owned_t = [np.sort(k[self.owner[t] == q]) for q in range(P)]
                refs = []
                for q in range(P):
                    srcs = []
                    for x in self.rels.values():
                        if x["src_type"] != t:
                            continue
                        tt = x["dst_type"]
                        mine = _owner_of(mag["key"][tt], self.owner[tt], x["dst"]) == q
                        srcs.append(np.asarray(x["src"], np.int64)[mine])
                    refs.append(np.intersect1d(np.unique(np.concatenate(srcs)), k))
                hp = HaloPlan(owned_t, self.n_pad[t], refs, r)
                hp.send_idx_dev = be.index_i32(hp.send_idx)
                self.halo[t] = hp
                r0 = r * self.n_pad[t]
                self.s_keys[t] = hp.s_keys(self.s_keys[t][r0:r0 + self.n_pad[t]])
        for t in types:
            nkm = self.nkm[t]
            if t in self.sources:
                n_s = len(self.s_keys[t])      # all-gathered P n_pad rows, or own + halo rows
                self.Yall[t] = be.zeros(n_s, nkm * d)
                self.dYall[t] = be.zeros(n_s, nkm * d)
                self.R[t] = be.zeros(self.n_pad[t], nkm * d)
                if t in self.halo:
                    self.R[t] = be.zeros(max(len(self.halo[t].send_idx), 1), nkm * d)
        self.idx, self.O, self.lse = {}, {}, {}
        for name, x in self.rels.items():
            ts, tt = x["src_type"], x["dst_type"]
            mine = _owner_of(mag["key"][tt], self.owner[tt], x["dst"]) == r
            self.idx[name] = be.build_index(np.asarray(x["src"])[mine], np.asarray(x["dst"])[mine],
                                            self.s_keys[ts], self.my_keys[tt], dense=True)
            self.O[name] = be.zeros(self.n_pad[tt], d)
            self.lse[name] = be.zeros(self.n_pad[tt], h)
        self.Ht = {t: be.zeros(self.n_pad[t], d) for t in self.targets}
        # per-relation dQ, summed into the target type's query gradient
        self.dQ = {t: be.zeros(self.n_pad[t], d) for t in self.targets}
        self.d_out = {}
        for t in self.targets:
            full = np.asarray(par["d_out"][t], np.float32)       # T-key order of all keys
            ks = np.sort(np.asarray(mag["key"][t], np.int64))
            dout = np.zeros((self.n_pad[t], d), np.float32)
            dout[: self.n_own[t]] = full[np.searchsorted(ks, self.my_keys[t])]
            self.d_out[t] = be.tensor(dout)
        self.timers = None

    def _blk(self, buf, t, kind, name):
        if kind == "q":
            return buf[t]
        i = self.col[(kind, name)][1]               # K'/M' blocks precede Q (hgt_parameters)
        return buf[t][:, i * self.d:(i + 1) * self.d]

    def _w(self, t, q):
        """W[t] rows of the K'/M' blocks (q False) or of the query block (q True); likewise dW."""
        k = self.nkm[t] * self.d
        return (self.W[t][k:], self.dW[t][k:]) if q else (self.W[t][:k], self.dW[t][:k])

    @property
    def join_rows_per_step(self):
        return sum(self.be.n_join_rows(i) for i in self.idx.values())

    def roof_model(self):
        d, h = self.d, self.h
        f, b = [], []
        for ix in self.idx.values():
            nj, ng, ns = self.be.n_join_rows(ix), self.be.n_groups(ix), self.be.n_src_rows(ix)
            f.append(nj * (4 + 8 * d) + ng * (8 * d + 4 * h + 8))
            b.append(nj * ((4 + 8 * d + 8 * h) + (8 + 8 * h + 8 * d)) + ng * (16 * d + 4 * h + 8)
                     + ns * (8 * d + 8))
        return {"lja_fwd": {"bound": "hbm", "amount": float(np.mean(f))},
                "lja_bwd": {"bound": "hbm", "amount": float(np.mean(b))}}

    def host_io(self):
        return list(self.H.values()) + list(self.d_out.values()), list(self.dW.values())

    def _t(self, name):
        if self.timers is None:
            return
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.timers.setdefault(name, []).append(e)

    def forward(self):
        be, g = self.be, self.group
        self._t("proj_fwd")
        for t in self.blocks:
            if t in self.Y:
                be.project(self.H[t], self._w(t, False)[0], self.Y[t])
            if t in self.Yq:
                be.project(self.H[t], self._w(t, True)[0], self.Yq[t])
        self._t("proj_fwd_end")
        for s in self.sources:
            if s in self.halo:                                   # K'/M' of referenced rows
                hp = self.halo[s]
                self.Yall[s][: hp.n_pad].copy_(self.Y[s])
                halo_exchange_fwd(be, hp, self.Yall[s], self.R[s][: len(hp.send_idx)], g)
            else:
                all_gather_rows(self.Yall[s], self.Y[s], g)      # K'/M' only
        first = {t: True for t in self.targets}
        for name, x in self.rels.items():
            ts, tt = x["src_type"], x["dst_type"]
            n = self.n_own[tt]
            self._t("lja_fwd")
            be.lja_sm_fwd(self.idx[name], self._blk(self.Yall, ts, "m", name),
                          self._blk(self.Yall, ts, "k", name), self._blk(self.Yq, tt, "q", tt),
                          self.h, self.O[name][:n], self.lse[name][:n])
            self._t("lja_fwd_end")
            be.accumulate(self.Ht[tt][:n], self.O[name][:n], 0.0 if first[tt] else 1.0)
            first[tt] = False
        return self.Ht

    def backward(self):
        be, g = self.be, self.group
        for t in self.blocks:
            if t in self.dY:
                be.fill_zero(self.dY[t])
            if t in self.dYq:
                be.fill_zero(self.dYq[t])
        for name, x in self.rels.items():
            ts, tt = x["src_type"], x["dst_type"]
            n = self.n_own[tt]
            self._t("lja_bwd")
            be.lja_sm_bwd(self.idx[name], self._blk(self.Yall, ts, "m", name),
                          self._blk(self.Yall, ts, "k", name), self._blk(self.Yq, tt, "q", tt),
                          self.h, self.O[name][:n], self.lse[name][:n], self.d_out[tt][:n],
                          self._blk(self.dYall, ts, "m", name), self._blk(self.dYall, ts, "k", name),
                          self.dQ[tt][:n])
            self._t("lja_bwd_end")
            be.accumulate(self.dYq[tt][:n], self.dQ[tt][:n], 1.0)
        for s in self.sources:
            if s in self.halo:
                hp = self.halo[s]
                halo_exchange_bwd(be, hp, self.dYall[s], self.R[s][: len(hp.send_idx)], g)
                be.accumulate(self.dY[s], self.dYall[s][: hp.n_pad], 1.0)
            else:
                reduce_scatter_rows(self.R[s], self.dYall[s], g)
                be.accumulate(self.dY[s], self.R[s], 1.0)
        self._t("proj_bwd")
        for t in self.blocks:
            first = True
            for q, dY in ((False, self.dY.get(t)), (True, self.dYq.get(t))):
                if dY is None:
                    continue
                W, dW = self._w(t, q)
                be.project_bwd(self.H[t], W, dY, self.dH[t] if first else self.dH2[t], dW)
                if not first:
                    be.accumulate(self.dH[t], self.dH2[t], 1.0)
                first = False
        self._t("proj_bwd_end")
        if self.P > 1:
            for t in self.blocks:
                dist.all_reduce(self.dW[t], group=g)
        return self.dW, self.dH

    def step(self):
        self.forward()
        return self.backward()


class ShardedDHNProgram:
    """One DHN layer (config 5) over P ranks (DHN bullet):
    roots hash-partitioned by node key, the Edge adjacency replicated on every rank (built
    once over the gathered node layout), the position features all-gathered once per layer.

        Y_own   = H_own W^T                            (A2, the nine position maps)
        Y_all   = all_gather(Y_own)                    (NCCL: f_{k,i} of every node)
        C_k(n)  = closed-walk aggregate, n in owned roots        (rnn_dhn_fwd_roots)
      backward: closed walks are rotation invariant, so d f_j(x) is the walk aggregate ROOTED
      at x with rotated operands (g = f0 (.) dOut in the walk): each rank computes the
      complete gradient rows of its OWN nodes from the all-gathered dOut -- no reduce-scatter
        dOut_all = all_gather(dOut_own)                (3d per node)
        d f_j(x), x owned                              (rnn_dhn_bwd_roots)
        dH_own, dW = projection backward;  all_reduce(dW)
    Owned rows sit at [rank * n_pad, rank * n_pad + n_own) of the gathered layout (ShardPlan),
    so d f of owned nodes is a contiguous slice; outputs come back in owned-key order through
    rnn_gather_rows (group order -> owned rows, dOut rows -> group order)."""

    KS = (2, 3, 4)

    def __init__(self, g: dict, backend=None, group=None, seed=0x5EED, prec="3xtf32",
                 param_seed=11, ks=KS):
        self.group = group
        self.P = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        be = self.be = backend if backend is not None else RnnBackend(prec=prec)
        P, r = self.P, self.rank
        self.ks = tuple(ks)
        keys = np.asarray(g["nodes"]["key"], np.int64)
        owner = be.hash_partition(keys, P, seed)
        e_src, e_dst = np.asarray(g["edges"]["src"]), np.asarray(g["edges"]["dst"])
        plan = self.plan = ShardPlan(keys, e_src, e_dst, owner, P, r)
        self.n_pad, self.n_own = plan.n_pad, int(plan.counts[r])
        self.d = d = g["nodes"]["x"].shape[1]
        self.npos = sum(self.ks)
        # replicated adjacency over ALL Edge rows, S = T = the gathered layout
        self.idx = be.build_dhn_index(e_src, e_dst, plan.s_keys)
        gkey, grow = be.dhn_groups(self.idx)
        self.G = len(gkey)
        self.symmetric = be.dhn_symmetric(self.idx)
        # owned roots: groups whose key this rank owns (owned nodes without a group -- no
        # out-edges -- aggregate to 0)
        pos = np.searchsorted(gkey, plan.my_keys)
        pos = np.clip(pos, 0, max(self.G - 1, 0))
        has = (self.G > 0) & (gkey[pos] == plan.my_keys) if self.G else np.zeros(len(plan.my_keys), bool)
        own_grp = np.where(has, pos, -1).astype(np.int32)
        self.roots = be.index_i32(own_grp[own_grp >= 0])
        og = np.full(self.n_pad, -1, np.int32)
        og[: self.n_own] = own_grp
        self.own_grp = be.index_i32(og)                   # owned row -> group (or -1)
        self.row_of_grp = be.index_i32(grow)              # group -> gathered row
        # parameters (DHNProgram's draws) and owned inputs
        rng = np.random.default_rng(param_seed)
        W = rng.standard_normal((self.npos * d, d)) / np.sqrt(d)
        d_out_full = rng.standard_normal((len(keys), len(self.ks) * d)).astype(np.float32)
        ks_sorted = np.sort(keys)
        x = np.zeros((self.n_pad, d), np.float32)
        x[: self.n_own] = np.asarray(g["nodes"]["x"], np.float32)[plan.my_rows]
        dO = np.zeros((self.n_pad, len(self.ks) * d), np.float32)
        dO[: self.n_own] = d_out_full[np.searchsorted(ks_sorted, plan.my_keys)]
        self.H = be.tensor(x)
        self.W = be.tensor(W.astype(np.float32))
        self.d_out = be.tensor(dO)
        nall = P * self.n_pad
        self.Y = be.zeros(self.n_pad, self.npos * d)
        self.Yall = be.zeros(nall, self.npos * d)
        self.dYall = be.zeros(nall, self.npos * d)
        self.out_grp = be.zeros(max(self.G, 1), len(self.ks) * d)[: self.G]
        self.out = be.zeros(self.n_pad, len(self.ks) * d)
        self.walk_sum = {k: be.zeros(max(self.G, 1), d)[: self.G] for k in self.ks}
        self.dOall = be.zeros(nall, len(self.ks) * d)
        self.dOgrp = be.zeros(max(self.G, 1), len(self.ks) * d)[: self.G]
        self.dW = be.zeros(self.npos * d, d)
        self.dH = be.zeros(self.n_pad, d)
        self.pos0 = {}
        p = 0
        for k in self.ks:
            self.pos0[k] = p
            p += k
        self.timers = None
        self._rows = None

    def _f(self, k, buf):
        p, d = self.pos0[k], self.d
        return [buf[:, (p + i) * d:(p + i + 1) * d] for i in range(k)]

    @property
    def join_rows_per_step(self):
        """This rank's rows: Edge rows of its roots (C2) + closed 3- and 4-walks rooted at
        them (exact counts over the replicated adjacency)."""
        if self._rows is None:
            self._rows = self.be.dhn_rows(self.idx, self.roots, self.ks)
        return self._rows

    def roof_model(self):
        return {"dhn4_fwd": {"bound": "alu", "amount": float("nan")}}

    def host_io(self):
        return [self.H, self.d_out], [self.dW]

    def _t(self, name):
        if self.timers is None:
            return
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.timers.setdefault(name, []).append(e)

    def forward(self):
        be, g, d = self.be, self.group, self.d
        self._t("proj_fwd")
        be.project(self.H, self.W, self.Y)
        self._t("proj_fwd_end")
        self._t("allgather")
        all_gather_rows(self.Yall, self.Y, g)
        self._t("allgather_end")
        for j, k in enumerate(self.ks):
            self._t(f"dhn{k}_fwd")
            be.dhn_fwd(self.idx, k, self._f(k, self.Yall), self.roots,
                       self.out_grp[:, j * d:(j + 1) * d], self.walk_sum[k])
            self._t(f"dhn{k}_fwd_end")
        be.gather_rows(self.out, self.out_grp, self.own_grp)
        return self.out

    def backward(self):
        be, g, d = self.be, self.group, self.d
        self._t("allgather")
        all_gather_rows(self.dOall, self.d_out, g)
        self._t("allgather_end")
        be.gather_rows(self.dOgrp, self.dOall, self.row_of_grp)
        for j, k in enumerate(self.ks):
            self._t(f"dhn{k}_bwd")
            be.dhn_bwd(self.idx, k, self._f(k, self.Yall), self.roots,
                       self.dOgrp[:, j * d:(j + 1) * d], self.walk_sum[k],
                       self._f(k, self.dYall), self.symmetric)
            self._t(f"dhn{k}_bwd_end")
        lo = self.rank * self.n_pad
        dY_own = self.dYall[lo:lo + self.n_pad]
        self._t("proj_bwd")
        be.project_bwd(self.H, self.W, dY_own, self.dH, self.dW)
        self._t("proj_bwd_end")
        if self.P > 1:
            dist.all_reduce(self.dW, group=g)
        return self.dW, self.dH

    def step(self):
        self.forward()
        return self.backward()

    def owned_output(self):
        return self.be.numpy(self.out)[: self.n_own]

    def owned_dx(self):
        return self.be.numpy(self.dH)[: self.n_own]
