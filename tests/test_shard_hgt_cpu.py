"""Sharded HGT layer (shard.ShardedHGTProgram, config 3) on CPU: world size 1 and 2 over gloo,
fp64 oracle primitives (tests only), against a single-process reference assembled from the
oracle's per-relation HGT (oracle.programs.hgt_relation) with the same parameters.  Pins the
per-type hash partitions, target-owned relation rows with dense groups, the all-gather of the
stacked source projections, the reduce-scatter of dK'/dM' and the all-reduce of dW."""
import os
import tempfile

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from oracle import programs as op
from paper_2605_24207_b200.programs import hgt_parameters
from paper_2605_24207_b200.shard import ShardedHGTProgram
from tests.test_shard_cpu import _free_port
from tests.test_shard_hyper_cpu import DenseOracleBackend


class HGTOracleBackend(DenseOracleBackend):
    def n_src_rows(self, idx):
        return idx["n_src_rows"] if "n_src_rows" in idx else len(idx["src_ptr"]) - 1

    def fill_zero(self, t):
        t.zero_()

    def accumulate(self, out, x, beta):
        out.mul_(beta).add_(x)

    def lja_sm_fwd(self, idx, M, K, Q, heads, out, lse):
        r, l = oracle.lja_fwd(idx, agg="softmax", src=M.numpy(), src_key=K.numpy(),
                              dst=Q.numpy(), heads=heads, scale=1.0)
        out.zero_()
        lse.fill_(-np.inf)
        pos = torch.from_numpy(idx["dense_pos"])
        out[pos] = torch.from_numpy(r)
        lse[pos] = torch.from_numpy(np.asarray(l))

    def lja_sm_bwd(self, idx, M, K, Q, heads, out, lse, d_out, dM, dK, dQ):
        dO = d_out.numpy()[idx["dense_pos"]]
        g = oracle.lja_bwd(idx, dO, agg="softmax", src=M.numpy(), src_key=K.numpy(),
                           dst=Q.numpy(), heads=heads, scale=1.0)
        dM[:] = torch.from_numpy(g["src"])
        dK[:] = torch.from_numpy(g["src_key"])
        dQ[:] = torch.from_numpy(g["dst"][: dQ.shape[0]])   # Q operand is the padded block


def small_mag():
    m = synth.mag_like(9, scale=0.0006, d=16, heads=2)
    m.pop("rng", None)
    return m


def reference(mag):
    par = hgt_parameters(mag)
    d = mag["d"]
    blocks, col = par["blocks"], par["col"]
    Ht = {t: np.zeros((mag["n"][t], d)) for t in par["targets"]}
    dY = {t: np.zeros((mag["n"][t], len(b) * d)) for t, b in blocks.items()}
    for name, r in mag["rels"].items():
        ts, tt = r["src_type"], r["dst_type"]
        ik, im, iq = col[("k", name)][1], col[("m", name)][1], col[("q", tt)][1]
        Ws, Wt = par["W"][ts], par["W"][tt]
        res = op.hgt_relation(mag["h"][ts], mag["h"][tt], Ws[ik * d:(ik + 1) * d],
                              Ws[im * d:(im + 1) * d], Wt[iq * d:(iq + 1) * d], mag["key"][ts],
                              mag["key"][tt], r["src"], r["dst"], mag["heads"], par["d_out"][tt])
        Ht[tt][res["dense_rows"]] += res["out"]
        dY[ts][:, ik * d:(ik + 1) * d] += res["dK"]
        dY[ts][:, im * d:(im + 1) * d] += res["dM"]
        dY[tt][:, iq * d:(iq + 1) * d] += res["dQ"]          # [n_t, d]: every T row
    dW, dH = {}, {}
    for t in blocks:
        dH[t], dW[t], _ = oracle.project_bwd(np.asarray(mag["h"][t], np.float64), par["W"][t], dY[t],
                                             want_db=False)
    return {"Ht": Ht, "dW": dW, "dH": dH}


def _run(mag, backend, halo=True):
    prog = ShardedHGTProgram(mag, backend=backend, halo=halo)
    if halo and prog.P > 1:      # the halo exchange moves fewer K'/M' rows than the all-gather
        assert all(h.rows_recv <= h.rows_allgather for h in prog.halo.values())
    prog.step()
    nm = prog.be.numpy
    out = {}
    for t in prog.blocks:
        out[f"keys_{t}"] = prog.my_keys[t]
        out[f"rows_{t}"] = prog.my_rows[t]
        out[f"dH_{t}"] = nm(prog.dH[t])[: prog.n_own[t]]
        out[f"dW_{t}"] = nm(prog.dW[t])
    for t in prog.targets:
        out[f"Ht_{t}"] = nm(prog.Ht[t])[: prog.n_own[t]]
    return out


def check(res, mag, rtol=1e-9, atol=1e-11, close=None):
    ref = reference(mag)
    close = close or (lambda a, b, what: np.testing.assert_allclose(a, b, rtol=rtol, atol=atol,
                                                                    err_msg=what))
    for t in ref["dW"]:
        keys = np.concatenate([r[f"keys_{t}"] for r in res])
        assert sorted(keys.tolist()) == sorted(np.asarray(mag["key"][t]).tolist())
        rows = np.concatenate([r[f"rows_{t}"] for r in res])
        close(np.concatenate([r[f"dH_{t}"] for r in res]), ref["dH"][t][rows], f"dH {t}")
        for r in res:
            close(r[f"dW_{t}"], ref["dW"][t], f"dW {t}")
        if t in ref["Ht"]:
            ks = np.sort(np.asarray(mag["key"][t]))
            close(np.concatenate([r[f"Ht_{t}"] for r in res]), ref["Ht"][t][np.searchsorted(ks, keys)],
                  f"Ht {t}")


def test_world_size_1():
    mag = small_mag()
    check([_run(mag, HGTOracleBackend())], mag)


def _worker(rank, world, port, path, halo=True):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        np.savez(os.path.join(path, f"r{rank}.npz"), **_run(small_mag(), HGTOracleBackend(), halo))
    finally:
        dist.destroy_process_group()


def test_world_size_2_gloo():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(2)]
    check(res, small_mag())


def test_world_size_2_gloo_allgather():
    """K'/M' all-gather (halo=False) gives the same result as the per-type halo exchange."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d, False), nprocs=2, join=True)
        res = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(2)]
    check(res, small_mag())
