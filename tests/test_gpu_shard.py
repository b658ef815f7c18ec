"""GPU parity of the sharded GCN step (paper_2605_24207_b200/shard.py with the librnn.so
backend) against the oracle GCN step: world size 1, and world size 2 as two processes sharing
cuda:0 over gloo (the GPU box has one GPU; NCCL needs one device per rank).  Checks the owned
outputs, the gathered input gradients and the all-reduced weight gradients."""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.test_shard_cpu import _free_port, graph_with_weights, reference
from tests.util import FP32_TOL, assert_close

pytestmark = pytest.mark.gpu


def arxiv_small():
    import synth
    g = synth.arxiv_like(3, n_nodes=6000, n_edges=40000, d=128, layers=2)
    return g


def _run(g):
    from paper_2605_24207_b200.shard import ShardedGCNProgram
    prog = ShardedGCNProgram(g)
    prog.step()
    torch.cuda.synchronize()
    return {"keys": prog.plan.my_keys, "rows": prog.plan.my_rows, "out": prog.owned_output(),
            "dx": prog.owned_dx(), **{f"dW{l}": prog.dW[l].cpu().numpy() for l in range(prog.L)}}


def _worker(rank, world, port, path, which):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = graph_with_weights() if which == "small" else arxiv_small()
        np.savez(os.path.join(path, f"r{rank}.npz"), **_run(g))
    finally:
        dist.destroy_process_group()


def check(res, g):
    ref = reference(g)
    keys = np.concatenate([r["keys"] for r in res])
    pos = np.searchsorted(ref["out_keys"], keys)
    assert_close(np.concatenate([r["out"] for r in res]), ref["out"][pos], FP32_TOL, "out")
    rows = np.concatenate([r["rows"] for r in res])
    assert_close(np.concatenate([r["dx"] for r in res]), ref["dH0"][rows], FP32_TOL, "dX")
    for l in range(len(ref["dW"])):
        for r in res:
            assert_close(r[f"dW{l}"], ref["dW"][l], FP32_TOL, f"dW{l}")


@pytest.mark.parametrize("which", ["small", "arxiv"])
def test_sharded_world_1(which):
    g = graph_with_weights() if which == "small" else arxiv_small()
    check([_run(g)], g)


@pytest.mark.parametrize("which", ["small", "arxiv"])
def test_sharded_world_2(which):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d, which), nprocs=2, join=True)
        res = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(2)]
    check(res, graph_with_weights() if which == "small" else arxiv_small())


def _run_hyper():
    from paper_2605_24207_b200.shard import ShardedHypergraphProgram
    from tests.test_shard_hyper_cpu import small_hypergraph
    import synth
    hg = synth.hypergraph_like(5, n_nodes=20000, n_hyper=4000, n_inc=100000, d=128)
    prog = ShardedHypergraphProgram(hg)
    prog.step()
    torch.cuda.synchronize()
    return hg, {"keys": prog.my_v, "rows": prog.my_rows, "out": prog.owned_output(),
                "dx": prog.owned_dx(), "dtheta": prog.dTheta.cpu().numpy()}


def _worker_hyper(rank, world, port, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        np.savez(os.path.join(path, f"r{rank}.npz"), **_run_hyper()[1])
    finally:
        dist.destroy_process_group()


def check_hyper(res, hg):
    from tests.test_shard_hyper_cpu import reference
    ref, gk = reference(hg)
    keys = np.concatenate([r["keys"] for r in res])
    out = np.concatenate([r["out"] for r in res])
    pos = np.searchsorted(gk, keys)
    has = (pos < len(gk)) & (gk[np.minimum(pos, len(gk) - 1)] == keys)
    assert_close(out[has], ref["Xo"][pos[has]], FP32_TOL, "out")
    assert np.all(out[~has] == 0)
    rows = np.concatenate([r["rows"] for r in res])
    assert_close(np.concatenate([r["dx"] for r in res]), ref["dX"][rows], FP32_TOL, "dX")
    for r in res:
        assert_close(r["dtheta"], ref["dTheta"], FP32_TOL, "dTheta")


def test_sharded_hyper_world_1():
    hg, r = _run_hyper()
    check_hyper([r], hg)


def test_sharded_hyper_world_2():
    import synth
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker_hyper, args=(2, _free_port(), d), nprocs=2, join=True)
        res = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(2)]
    check_hyper(res, synth.hypergraph_like(5, n_nodes=20000, n_hyper=4000, n_inc=100000, d=128))


def _mag_gpu():
    import synth
    m = synth.mag_like(9, scale=0.003, d=128, heads=8)
    m.pop("rng", None)
    return m


def _run_hgt():
    from paper_2605_24207_b200.shard import ShardedHGTProgram
    from tests.test_shard_hgt_cpu import _run
    from paper_2605_24207_b200.shard import RnnBackend
    r = _run(_mag_gpu(), RnnBackend())
    torch.cuda.synchronize()
    return r


def _worker_hgt(rank, world, port, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        np.savez(os.path.join(path, f"r{rank}.npz"), **_run_hgt())
    finally:
        dist.destroy_process_group()


def _check_hgt(res):
    from tests.test_shard_hgt_cpu import check
    check(res, _mag_gpu(), close=lambda a, b, what: assert_close(a, b, FP32_TOL, what))


def test_sharded_hgt_world_1():
    _check_hgt([_run_hgt()])


def test_sharded_hgt_world_2():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker_hgt, args=(2, _free_port(), d), nprocs=2, join=True)
        res = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(2)]
    _check_hgt(res)


def test_sharded_cora_widths_world_1():
    """Cora-shaped GCN (1,433 -> 16 -> 7) through the sharded program on the GPU: the
    ld-padded buffers let rnn_project / the LJA run at width 7."""
    import synth
    g = synth.cora_like(42)
    check([_run(g)], g)


def _run_dhn():
    from paper_2605_24207_b200.shard import ShardedDHNProgram
    from tests.test_shard_dhn_cpu import graph
    prog = ShardedDHNProgram(graph())
    prog.step()
    torch.cuda.synchronize()
    return {"keys": prog.plan.my_keys, "rows": prog.plan.my_rows, "out": prog.owned_output(),
            "dx": prog.owned_dx(), "dW": prog.dW.cpu().numpy(), "n_rows": prog.join_rows_per_step}


def _worker_dhn(rank, world, port, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        np.savez(os.path.join(path, f"r{rank}.npz"), **_run_dhn())
    finally:
        dist.destroy_process_group()


def _check_dhn(res):
    from tests.test_shard_dhn_cpu import graph, reference
    g = graph()
    ref = reference(g)
    keys = np.sort(np.asarray(g["nodes"]["key"]))
    got = np.concatenate([r["keys"] for r in res])
    assert sorted(got.tolist()) == keys.tolist()
    assert_close(np.concatenate([r["out"] for r in res]), ref["out"][np.searchsorted(keys, got)],
                 FP32_TOL, "out")
    rows = np.concatenate([r["rows"] for r in res])
    assert_close(np.concatenate([r["dx"] for r in res]), ref["dH"][rows], FP32_TOL, "dH")
    for r in res:
        assert_close(r["dW"], ref["dW"], FP32_TOL, "dW")


def test_sharded_dhn_world_1():
    """ShardedDHNProgram on librnn.so (rnn_dhn_fwd_roots / rnn_dhn_bwd_roots, rnn_gather_rows)."""
    _check_dhn([_run_dhn()])


def test_sharded_dhn_world_2():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker_dhn, args=(2, _free_port(), d), nprocs=2, join=True)
        res = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(2)]
    _check_dhn(res)
