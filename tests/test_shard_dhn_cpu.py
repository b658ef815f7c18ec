"""Sharded DHN layer (paper_2605_24207_b200/shard.py ShardedDHNProgram, config 5 at P ranks)
checked on CPU: world size 1 and 2 over gloo, compute primitives from an fp64 backend built
on the oracle (test infrastructure), against the single-process oracle DHN step
(oracle.programs.dhn_step).

What this pins (DHN bullet): roots hash-partitioned by node key, the adjacency
replicated over the gathered node layout, one all-gather of the position features per layer,
and the rotation backward -- every rank computes the complete gradient rows of its OWN nodes
from the all-gathered upstream gradient, so no reduce-scatter is needed -- plus the dW
all-reduce."""
import os
import tempfile

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import programs as op
from paper_2605_24207_b200.shard import ShardedDHNProgram
from tests.test_shard_cpu import OracleBackend, _free_port


class OracleDHNBackend(OracleBackend):
    """fp64 DHN primitives from oracle/ with the product backend's contract (tests only)."""

    def build_dhn_index(self, e_src, e_dst, s_keys):
        self.keys = np.asarray(s_keys, np.int64)
        return oracle.build_join_index(e_src, e_dst, s_keys, s_keys, within_by_src_key=True)

    def dhn_groups(self, idx):
        return idx["group_key"], idx["group_dst_row"]

    def dhn_symmetric(self, idx):
        r = np.repeat(idx["group_dst_row"], np.diff(idx["group_ptr"])).astype(np.int64)
        v = idx["src_row"].astype(np.int64)
        n = len(self.keys)
        return np.array_equal(np.sort(r * n + v), np.sort(v * n + r))

    def index_i32(self, a):
        return torch.as_tensor(np.asarray(a, np.int32))

    def gather_rows(self, out, x, idx):
        i = idx.numpy()
        y = np.zeros(tuple(out.shape))
        ok = i >= 0
        y[ok] = x.numpy()[i[ok]]
        out[:] = torch.from_numpy(y)

    def dhn_fwd(self, idx, k, f, roots, out, walk_sum):
        sel = roots.numpy().astype(np.int64)
        fn = [t.numpy() for t in f]
        out[sel] = torch.from_numpy(oracle.dhn_fwd(k, idx, self.keys, fn, sel=sel))
        ones = [np.ones_like(fn[0])] + fn[1:]
        walk_sum[sel] = torch.from_numpy(oracle.dhn_fwd(k, idx, self.keys, ones, sel=sel))

    def dhn_bwd(self, idx, k, f, roots, d_out, walk_sum, d_f, symmetric):
        grads = oracle.dhn_bwd(k, idx, self.keys, [t.numpy() for t in f], d_out.numpy())
        rows = idx["group_dst_row"][roots.numpy()]
        for j in range(k):
            g = np.zeros_like(grads[j])
            g[rows] = grads[j][rows]          # listed roots get their full rows, others 0
            d_f[j][:] = torch.from_numpy(g)

    def dhn_rows(self, idx, roots, ks):
        sel = roots.numpy().astype(np.int64)
        ones = [np.ones((len(self.keys), 1))] * 4
        return int(sum(oracle.dhn_fwd(k, idx, self.keys, ones[:k], sel=sel).sum() for k in ks))


def graph():
    """Sparse undirected graph (both directions stored, reading 10) with a hub, 150
    nodes, d = 32: small enough for the oracle's closed-walk enumeration in seconds."""
    rng = np.random.default_rng(9)
    n, m = 150, 500
    s, t = rng.integers(0, n, m), rng.integers(0, n, m)
    s[:40] = 0                                        # a hub
    ok = s != t
    pairs = np.unique(np.stack([np.minimum(s[ok], t[ok]), np.maximum(s[ok], t[ok])], 1), axis=0)
    src = np.concatenate([pairs[:, 0], pairs[:, 1]])
    dst = np.concatenate([pairs[:, 1], pairs[:, 0]])
    key = rng.permutation(n).astype(np.int64) * 3 + 11
    x = (rng.standard_normal((n, 32)) / np.sqrt(32)).astype(np.float32)
    return {"nodes": {"key": key, "x": x}, "edges": {"src": key[src], "dst": key[dst]}}


def reference(g):
    n, d = g["nodes"]["x"].shape
    rng = np.random.default_rng(11)                   # the program's parameter draws
    W = (rng.standard_normal((9 * d, d)) / np.sqrt(d)).astype(np.float32)   # stored as fp32
    d_out = rng.standard_normal((n, 3 * d)).astype(np.float32)
    return op.dhn_step(g, W, d_out)


def _run(g):
    prog = ShardedDHNProgram(g, backend=OracleDHNBackend())
    prog.step()
    return {"keys": prog.plan.my_keys, "rows": prog.plan.my_rows, "out": prog.owned_output(),
            "dx": prog.owned_dx(), "dW": prog.dW.numpy(), "n_rows": prog.join_rows_per_step}


def _worker(rank, world, port, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        np.savez(os.path.join(path, f"r{rank}.npz"), **_run(graph()))
    finally:
        dist.destroy_process_group()


def check(res, g):
    ref = reference(g)
    keys = np.sort(np.asarray(g["nodes"]["key"]))
    got_keys = np.concatenate([r["keys"] for r in res])
    assert sorted(got_keys.tolist()) == keys.tolist()                     # roots partition
    out = np.concatenate([r["out"] for r in res])
    np.testing.assert_allclose(out, ref["out"][np.searchsorted(keys, got_keys)], rtol=1e-9,
                               atol=1e-11)
    rows = np.concatenate([r["rows"] for r in res])
    dx = np.concatenate([r["dx"] for r in res])
    np.testing.assert_allclose(dx, ref["dH"][rows], rtol=1e-9, atol=1e-11)
    for r in res:
        np.testing.assert_allclose(r["dW"], ref["dW"], rtol=1e-9, atol=1e-11)


def test_sharded_dhn_world_1():
    g = graph()
    check([_run(g)], g)


def test_sharded_dhn_world_2_gloo():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(2)]
    g = graph()
    check(res, g)
    # join rows: the ranks' roots partition the closed walks (Edge rows + 3- and 4-walks)
    n = len(g["nodes"]["key"])
    oi = oracle.build_join_index(g["edges"]["src"], g["edges"]["dst"], g["nodes"]["key"],
                                 g["nodes"]["key"], within_by_src_key=True)
    ones = [np.ones((n, 1))] * 4
    total = sum(oracle.dhn_fwd(k, oi, g["nodes"]["key"], ones[:k]).sum() for k in (2, 3, 4))
    assert sum(int(r["n_rows"]) for r in res) == int(total)
