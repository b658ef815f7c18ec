"""Sharded hypergraph layer (shard.ShardedHypergraphProgram, config 4) on CPU: world size 1
and 2 over gloo, fp64 oracle primitives (tests only), against the single-process oracle
hypergraph step (oracle.programs.hypergraph_step).  Pins the two hash partitions (nodes and
hyperedges), the dense per-rank blocks that chain hop 1's output into hop 2's all-gather, and
the all-gather / reduce-scatter / all-reduce sequence."""
import os
import tempfile

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from oracle import programs as op
from paper_2605_24207_b200.shard import ShardedHypergraphProgram, block_layout
from tests.test_shard_cpu import OracleBackend, _free_port


class DenseOracleBackend(OracleBackend):
    """Adds dense-group indices (rows = every T key in ascending order, empty groups 0) and
    SUM / MEAN aggregation without edge weights on top of the GCN test backend."""

    def build_index(self, e_src, e_dst, s_keys, t_keys, dense=False):
        idx = oracle.build_join_index(e_src, e_dst, s_keys, t_keys)
        if dense:
            idx = dict(idx)
            idx["dense_pos"] = np.searchsorted(np.sort(np.asarray(t_keys)), idx["group_key"])
        return idx

    def lja_fwd_agg(self, idx, Z, agg, out):
        r, _ = oracle.lja_fwd(idx, "src", agg, src=Z.numpy())
        out.zero_()
        out[torch.from_numpy(idx["dense_pos"])] = torch.from_numpy(r)

    def lja_bwd_src_agg(self, idx, Z, agg, d_out, d_src):
        dO = d_out.numpy()[idx["dense_pos"]]
        g = oracle.lja_bwd(idx, dO, "src", agg, src=Z.numpy(), want=("src",))["src"]
        d_src[:] = torch.from_numpy(g)


def small_hypergraph():
    return synth.hypergraph_like(5, n_nodes=300, n_hyper=60, n_inc=1200, d=8)


def reference(hg):
    ref = op.hypergraph_step(hg)
    return ref, np.asarray(ref["o2"]["group_key"])


def _run(hg, backend):
    prog = ShardedHypergraphProgram(hg, backend=backend)
    prog.step()
    return {"keys": prog.my_v, "rows": prog.my_rows, "out": prog.owned_output(),
            "dx": prog.owned_dx(), "dtheta": prog.be.numpy(prog.dTheta)}


def check(res, hg, rtol=1e-9):
    ref, gk = reference(hg)
    keys = np.concatenate([r["keys"] for r in res])
    assert sorted(keys.tolist()) == sorted(np.asarray(hg["nodes"]["key"]).tolist())
    out = np.concatenate([r["out"] for r in res])
    pos = np.searchsorted(gk, keys)
    has = (pos < len(gk)) & (gk[np.minimum(pos, len(gk) - 1)] == keys)
    np.testing.assert_allclose(out[has], ref["Xo"][pos[has]], rtol=rtol, atol=1e-12)
    assert np.all(out[~has] == 0)                       # no incidence: MEAN of nothing = 0
    rows = np.concatenate([r["rows"] for r in res])
    dx = np.concatenate([r["dx"] for r in res])
    np.testing.assert_allclose(dx, ref["dX"][rows], rtol=rtol, atol=1e-12)
    for r in res:
        np.testing.assert_allclose(r["dtheta"], ref["dTheta"], rtol=rtol, atol=1e-12)


def test_block_layout():
    keys = np.array([5, -3, 9, 100, 7], np.int64)
    owned, n_pad, s = block_layout(keys, np.array([0, 1, 0, 1, 1]), 2)
    assert n_pad == 3 and len(s) == 6
    assert list(s[:2]) == [5, 9] and list(s[3:]) == [-3, 7, 100]
    assert s[2] < -3 and len(set(s.tolist())) == 6


def test_world_size_1():
    hg = small_hypergraph()
    check([_run(hg, DenseOracleBackend())], hg)


def _worker(rank, world, port, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        np.savez(os.path.join(path, f"r{rank}.npz"), **_run(small_hypergraph(), DenseOracleBackend()))
    finally:
        dist.destroy_process_group()


def test_world_size_2_gloo():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(2)]
    check(res, small_hypergraph())
