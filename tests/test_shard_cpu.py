"""Multi-GPU sharding logic (paper_2605_24207_b200/shard.py) checked on CPU: world size 1 and 2
over gloo, with the compute primitives supplied by an fp64 backend built from the oracle (test
infrastructure), against the single-process oracle GCN step (oracle.programs.gcn_step).

What this pins: the hash partition by group key, the per-rank index over the
all-gathered source layout with sentinel padding, the degree exchange of the normalisation,
the all-gather / reduce-scatter / all-reduce sequence of the forward and backward."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from oracle import programs as op
from paper_2605_24207_b200.shard import ShardPlan, ShardedGCNProgram


class OracleBackend:
    """fp64 CPU primitives from oracle/ (tests only)."""

    def tensor(self, a):
        return torch.tensor(np.asarray(a, np.float64))

    def zeros(self, n, d):
        return torch.zeros(n, d, dtype=torch.float64)

    def zeros_i32(self, n):
        return torch.zeros(n, dtype=torch.int32)

    def numpy(self, t):
        return t.numpy()

    def hash_partition(self, keys, P, seed):
        return oracle.hash_partition(keys, P, seed)

    def build_index(self, e_src, e_dst, s_keys, t_keys):
        return oracle.build_join_index(e_src, e_dst, s_keys, t_keys)

    def n_groups(self, idx):
        return idx["n_groups"]

    def n_join_rows(self, idx):
        return idx["n_join_rows"]

    def group_sizes(self, idx, out):
        g = idx["n_groups"]
        out[:g] = torch.from_numpy(np.diff(idx["group_ptr"]).astype(np.int32))

    def gcn_norm_src_deg(self, idx, deg):
        deg = deg.numpy().astype(np.float64)
        sizes = np.diff(idx["group_ptr"]).astype(np.float64)
        grp = np.repeat(np.arange(idx["n_groups"]), np.diff(idx["group_ptr"]))
        ds = deg[idx["src_row"]]
        return np.where(ds > 0, 1.0 / np.sqrt(np.maximum(ds, 1)), 0.0) / np.sqrt(sizes[grp])

    def project(self, X, W, out):
        out[:] = torch.from_numpy(oracle.project(X.numpy(), W.numpy()))

    def lja_fwd(self, idx, Z, w, out):
        r, _ = oracle.lja_fwd(idx, "src", "sum", src=Z.numpy(), edge=w, edge_mode=1)
        out[: idx["n_groups"]] = torch.from_numpy(r)

    def lja_bwd_src(self, idx, Z, w, d_out, d_src):
        g = oracle.lja_bwd(idx, d_out.numpy()[: idx["n_groups"]], "src", "sum", src=Z.numpy(),
                           edge=w, edge_mode=1, want=("src",))["src"]
        d_src[:] = torch.from_numpy(g)

    def index_i32(self, a):
        return torch.as_tensor(np.asarray(a, np.int32))

    def gather_rows(self, out, x, idx):
        i = idx.numpy()
        out[:] = x[torch.as_tensor(i.astype(np.int64))]

    def scatter_add_rows(self, y, x, idx):
        y[torch.as_tensor(idx.numpy().astype(np.int64))] += x

    def lja_fwd_epi(self, idx, Z, w, out, bias, act):
        self.lja_fwd(idx, Z, w, out)
        G = idx["n_groups"]
        out[:G] = torch.from_numpy(oracle.epilogue_fwd(out[:G].numpy(), bias.numpy(), act))

    def epilogue_bwd(self, dy, y, bias, act, dx, db, rows):
        # the pre-activation from the output: y - b (ReLU: where y = 0 it gives -b, i.e. pre
        # = 0, whose derivative is 0 like any pre <= 0)
        b = bias.numpy()
        d, bb, _, _ = oracle.epilogue_bwd(dy[:rows].numpy(), y[:rows].numpy() - b, b, act)
        dx[:rows] = torch.from_numpy(d)
        db[:] = torch.from_numpy(bb)

    def project_bwd(self, X, W, dY, dX, dW):
        a, b, _ = oracle.project_bwd(X.numpy(), W.numpy(), dY.numpy(), want_db=False)
        dX[:] = torch.from_numpy(a)
        dW[:] = torch.from_numpy(b)


def graph_with_weights(dims=(12, 8, 4), bias=False):
    """Small GCN; dims (13, 6, 7) gives Cora-like widths that are not multiples of 4; bias:
    the O7 epilogue's per-layer biases."""
    g = synth.gcn_graph(7, n_nodes=400, n_edge_tuples=2400, d_in=dims[0], undirected=True,
                        cap_ratio=50.0)
    rng = np.random.default_rng(3)
    g["dims"] = list(dims)
    g["W"] = [(rng.standard_normal((dims[l + 1], dims[l])) / 3).astype(np.float32)
              for l in range(len(dims) - 1)]
    g["d_out"] = rng.standard_normal((400, dims[-1])).astype(np.float32)
    if bias:
        g["b"] = [(rng.standard_normal(dims[l + 1]) * 0.3).astype(np.float32)
                  for l in range(len(dims) - 1)]
    return g


def reference(g):
    H, dW, dH0 = op.gcn_step(g)
    keys = np.asarray(g["nodes"]["key"])
    return {"out_keys": np.sort(keys), "out": H[-1], "dW": dW, "dH0": dH0}


def _worker(rank, world, port, path, dims=(12, 8, 4), halo=True):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = graph_with_weights(dims)
        prog = ShardedGCNProgram(g, backend=OracleBackend(), halo=halo)
        if halo and world > 1:
            assert prog.halo is not None and prog.halo.rows_recv < prog.halo.rows_allgather
        prog.step()
        np.savez(os.path.join(path, f"r{rank}.npz"), keys=prog.plan.my_keys, rows=prog.plan.my_rows,
                 out=prog.owned_output(), dx=prog.owned_dx(),
                 **{f"dW{l}": prog.dW[l].numpy() for l in range(prog.L)})
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def check(results, ref, g):
    keys = np.concatenate([r["keys"] for r in results])
    assert sorted(keys.tolist()) == sorted(np.asarray(g["nodes"]["key"]).tolist())  # a partition
    out = np.concatenate([r["out"] for r in results])
    pos = np.searchsorted(ref["out_keys"], keys)
    np.testing.assert_allclose(out, ref["out"][pos], rtol=1e-10, atol=1e-12)
    rows = np.concatenate([r["rows"] for r in results])
    dx = np.concatenate([r["dx"] for r in results])
    np.testing.assert_allclose(dx, ref["dH0"][rows], rtol=1e-9, atol=1e-12)
    for l in range(len(ref["dW"])):
        for r in results:
            np.testing.assert_allclose(r[f"dW{l}"], ref["dW"][l], rtol=1e-9, atol=1e-12)


def test_plan_partitions_keys_and_edges():
    g = graph_with_weights()
    keys = g["nodes"]["key"]
    owner = oracle.hash_partition(keys, 3, 5)
    plans = [ShardPlan(keys, g["edges"]["src"], g["edges"]["dst"], owner, 3, r) for r in range(3)]
    assert sum(len(p.e_dst) for p in plans) == len(g["edges"]["dst"])     # every edge once
    for p in plans:
        assert len(set(p.s_keys.tolist())) == len(p.s_keys)               # S is a set
        assert np.all(owner[np.searchsorted(np.sort(keys), p.e_dst)] >= 0)
        assert np.array_equal(p.s_keys[p.rank * p.n_pad:][: len(p.my_keys)], p.my_keys)
        assert not np.isin(p.s_keys[p.s_keys < np.min(keys)], keys).any()   # sentinels


def test_world_size_1():
    g = graph_with_weights()
    prog = ShardedGCNProgram(g, backend=OracleBackend())
    prog.step()
    res = {"keys": prog.plan.my_keys, "rows": prog.plan.my_rows, "out": prog.owned_output(),
           "dx": prog.owned_dx(), **{f"dW{l}": prog.dW[l].numpy() for l in range(prog.L)}}
    check([res], reference(g), g)


def test_world_size_2_gloo():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(2)]
    g = graph_with_weights()
    check(res, reference(g), g)


def test_world_size_2_gloo_ragged_widths():
    """Layer widths 13 -> 6 -> 7 (Cora-like, not multiples of 4): the program pads them with
    zeros for the ld % 4 == 0 kernels and collectives; the real columns are unchanged."""
    dims = (13, 6, 7)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d, dims), nprocs=2, join=True)
        res = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(2)]
    g = graph_with_weights(dims)
    check(res, reference(g), g)


def test_world_size_2_gloo_with_epilogue():
    """O7 epilogue (bias + ReLU hidden, bias last) in the sharded step: fused on the owned
    rows, backward through the epilogue, d bias all-reduced (checked through dW / dX)."""
    dims = (12, 8, 4)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker_b, args=(2, _free_port(), d), nprocs=2, join=True)
        res = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(2)]
    g = graph_with_weights(dims, bias=True)
    check(res, reference(g), g)


def _worker_b(rank, world, port, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = graph_with_weights((12, 8, 4), bias=True)
        prog = ShardedGCNProgram(g, backend=OracleBackend())
        prog.step()
        np.savez(os.path.join(path, f"r{rank}.npz"), keys=prog.plan.my_keys, rows=prog.plan.my_rows,
                 out=prog.owned_output(), dx=prog.owned_dx(),
                 **{f"dW{l}": prog.dW[l].numpy() for l in range(prog.L)})
    finally:
        dist.destroy_process_group()


def test_world_size_2_gloo_allgather():
    """The all-gather exchange (halo=False) gives the same result as the halo exchange."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d, (12, 8, 4), False), nprocs=2, join=True)
        res = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(2)]
    g = graph_with_weights()
    check(res, reference(g), g)


def test_world_size_3_gloo_halo():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(3, _free_port(), d), nprocs=3, join=True)
        res = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(3)]
    g = graph_with_weights()
    check(res, reference(g), g)
