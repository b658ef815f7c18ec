#!/usr/bin/env python
"""bench.py -- lifted join-aggregate join-rows/s (fwd+bwd) on B200 (BASELINE.json metric).

A step is one pass of the whole hot path over one batch of synthetic input: for every layer
of the program the tcgen05 projection, the fused gather-combine-reduce forward, the
transposed-CSR backward and the projection backward (the join index is built once before
timing -- content caching, PAPER.md comment :737).  Default workload: BASELINE.json
configs[1], the 3-layer GCN on synthetic ogbn-arxiv-shaped relations (169,343 nodes,
1,166,243 edges + self-loops, d = 128).

Contract: `python bench.py --gpus N --steps K --warmup W [--impl reference]` prints ONE JSON
line on rank 0.  Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA
events on the launching stream with L2 flushed (a 256 MiB write) between steps outside the
events; barrier + synchronize on both sides; the max over ranks.  `--impl reference` times
the fp64 CPU oracle (the reference arm of this tier) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "lifted join-aggregate join-rows/s (fwd+bwd)"
UNIT = "join-rows/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mag", choices=["arxiv", "cora", "hyper", "mag", "dhn"],
                    help="workload (default: MAG-shaped HGT, the largest single-GPU config)")
    ap.add_argument("--dhn-scale", type=float, default=1.0,
                    help="fraction of the ogbn-products-shaped graph for --config dhn")
    ap.add_argument("--prec", default="3xtf32", choices=["3xtf32", "tf32", "bf16"])
    ap.add_argument("--seeds", default=None,
                    help="comma-separated input seeds (default 42..46, PAPER.md:851; dhn: 42)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--eager", action="store_true",
                    help="launch the step kernel by kernel instead of replaying its CUDA graph")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--l2-window", action="store_true",
                    help="experiment (GCN configs, implies --eager): persisting-L2 window over "
                         "each LJA's gathered matrix")
    ap.add_argument("--profile-launches", action="store_true",
                    help="count kernel launches with torch.profiler (untimed pass)")
    a = ap.parse_args()
    if a.l2_window:
        a.eager = True
    if a.seeds is None:
        a.seeds = "42" if a.config == "dhn" else "42,43,44,45,46"
    return a


def make_graph(cfg, seed, sample=False):
    """Seeded synthetic input of a config; `sample` = the bounded
    same-structure instance the CPU oracle is timed on (hyper, mag: 1/20)."""
    import synth
    if cfg == "arxiv":
        return synth.arxiv_like(seed)
    if cfg == "hyper":
        if sample:
            return synth.hypergraph_like(seed, n_nodes=50_000, n_hyper=10_000, n_inc=250_000)
        return synth.hypergraph_like(seed)
    if cfg == "mag":
        return synth.mag_like(seed, scale=0.05 if sample else 1.0)
    if cfg == "dhn":
        return synth.products_like(seed, scale=0.0001 if sample else DHN_SCALE[0])
    return synth.cora_like(seed)


DHN_SCALE = [1.0]


def make_program(cfg, data, dev, prec):
    from paper_2605_24207_b200 import programs
    if cfg == "hyper":
        return programs.HypergraphProgram(data, device=dev, prec=prec)
    if cfg == "mag":
        return programs.HGTProgram(data, device=dev, prec=prec)
    if cfg == "dhn":
        return programs.DHNProgram(data, device=dev, prec=prec)
    return programs.GCNProgram(data, device=dev, prec=prec)


WORKLOAD = {
    "arxiv": "3-layer GCN as lifted query on synthetic ogbn-arxiv-shaped relations "
             "(169,343 node tuples, 1,166,243 edge tuples + self-loops, 128-dim)",
    "cora": "2-layer GCN as lifted query on synthetic Cora-shaped relations "
            "(2,708 node tuples, 10,556 edge tuples + self-loops, 1,433->16->7)",
    "hyper": "HyGNN two-hop incidence join (node->hyperedge SUM, hyperedge->node MEAN) on "
             "synthetic power-law hypergraph (1M nodes, 200K hyperedges, 5M incidences, 128-dim)",
    "dhn": "DHN layer (C2 + C3 triangle + C4 4-cycle closed-walk aggregates, nine 32x32 "
           "projections) on a synthetic ogbn-products-shaped DC-SBM graph",
    "mag": "HGT attention layer (4 relations, 8-head grouped softmax, dense target groups) on "
           "synthetic ogbn-mag-shaped schema (1.94M nodes, 21.1M edges, 128-dim)",
}


# ------------------------------------------------------------------------------------------
# clocks sampled DURING the timed region (B200_PROFILING.md recipe)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.stop = threading.Event()
        self.th = None

    def start(self):
        def run():
            while not self.stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self.stop.wait(0.2)
        self.th = threading.Thread(target=run, daemon=True)
        self.th.start()

    def finish(self):
        self.stop.set()
        if self.th:
            self.th.join(timeout=10)
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# fp32 FMA pipe: 148 SMs x 128 lanes x 2 flops x 1.965 GHz (B200_PROFILING.md unit counts and
# the max SM clock nvidia-smi reports on this pool) -- the ALU roof of the DHN walk kernels
FP32_ALU_TFLOPS = round(148 * 128 * 2 * 1.965e9 / 1e12, 2)
FP32_ALU_SRC = "derived: 148 SM x 128 FP32 lanes x 2 flop x 1965 MHz"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def _dist_setup():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # RNN_BENCH_DIST_BACKEND=gloo: exercise the N > 1 path with several ranks sharing the
    # visible GPUs (LOCAL_RANK mod device count; smoke-testing on a 1-GPU box only -- NCCL over
    # NVLink with one GPU per rank is the measured configuration)
    backend = os.environ.get("RNN_BENCH_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group(backend)
    return world, rank, local, torch.device("cuda", local)


def _build(args, seed, world, dev):
    """(program, job join rows per step, sharded?) for one seed's synthetic input."""
    import torch
    import torch.distributed as dist
    graph = make_graph(args.config, seed)
    sharded = world > 1 and args.config in SHARDED
    if sharded:
        # multi-GPU: the join relation hash-partitioned by group key, NCCL all-gather of the
        # source embeddings / reduce-scatter of their gradients per hop
        from paper_2605_24207_b200 import shard
        prog = SHARDED[args.config](shard)(graph, prec=args.prec)
        r = torch.tensor([prog.join_rows_per_step], dtype=torch.float64, device=dev)
        dist.all_reduce(r)
        rows = int(r.item())              # all ranks' join rows = the whole job
    else:
        # other configs at N > 1: independent replicas
        prog = make_program(args.config, graph, dev, args.prec)
        rows = world * prog.join_rows_per_step
    prog._labels = graph.get("labels")
    del graph
    return prog, rows, sharded


SHARDED = {
    "arxiv": lambda m: m.ShardedGCNProgram, "cora": lambda m: m.ShardedGCNProgram,
    "hyper": lambda m: m.ShardedHypergraphProgram, "mag": lambda m: m.ShardedHGTProgram,
    "dhn": lambda m: m.ShardedDHNProgram,
}


def _time_steps(prog, args, world, dev, graphed, flush):
    """W untimed warm-up steps, then K timed steps (barrier + synchronize on both sides; L2
    flushed between steps outside the events).  Returns (per-step ms, {kernel: [launch ms]},
    replay function)."""
    import torch
    import torch.distributed as dist

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    cs = None
    if graphed:
        # the step as ONE CUDA graph (programs.CapturedStep): event record nodes around the
        # step and around every kernel the program brackets give device times per replay
        from paper_2605_24207_b200.programs import CapturedStep
        cs = CapturedStep(prog, timed=True)
        run_step = cs.replay
    else:
        run_step = prog.step
    for _ in range(args.warmup):
        run_step()
    barrier()
    step_ms, launches_ms = [], {}
    if graphed:
        barrier()
        for _ in range(args.steps):
            flush.fill_(1.0)                  # L2 flush outside the step's events
            cs.replay()
            torch.cuda.synchronize()          # read this replay's event nodes
            t, per = cs.times()
            step_ms.append(t)
            for k, v in per.items():
                launches_ms.setdefault(k, []).extend(v)
        barrier()
    else:
        prog.timers = {}
        starts, ends = [], []
        barrier()
        for _ in range(args.steps):
            flush.fill_(1.0)                  # L2 flush outside the step's events
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record()
            prog.step()
            e.record()
            starts.append(s)
            ends.append(e)
        barrier()
        step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
        timers = prog.timers
        prog.timers = None
        for k, a in timers.items():
            if not k.endswith("_end"):
                launches_ms[k] = [x.elapsed_time(y) for x, y in zip(a, timers.get(k + "_end", []))]
    return step_ms, launches_ms, (cs.replay if cs is not None else None)


def _index_build_ms(prog, world):
    """One-time join-index build (A1, content caching -- excluded from the metric): the
    program's build_indices() again after warm-up, wall clock with a synchronize on both
    sides (its size-query phase is a host sync), max over ranks."""
    import torch
    if not hasattr(prog, "build_indices"):
        return float("nan")
    # the captured step graph and the queries hold the current index / weight pointers: build
    # a second copy, time it, then restore the program's own attributes
    saved = {k: (dict(v) if isinstance(v, dict) else v) for k, v in vars(prog).items()}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prog.build_indices()
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) * 1e3
    prog.__dict__.update(saved)
    return t


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local, dev = _dist_setup()
    seeds = [int(x) for x in str(args.seeds).split(",") if x != ""]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    sampler = ClockSampler(local)
    per_seed, launches_ms = [], {}
    first = None
    for si, seed in enumerate(seeds):
        prog, rows, sharded = _build(args, seed, world, dev)
        if args.l2_window:
            prog.l2_window = True
        graphed = not args.eager and (not sharded or args.config != "dhn")
        if si == 0:
            sampler.start()                   # clocks sampled during the timed regions
        step_ms, lm, replay = _time_steps(prog, args, world, dev, graphed, flush)
        t_seed = float(np.mean(step_ms))
        if world > 1:
            t = torch.tensor([t_seed], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_seed = float(t.item())
        per_seed.append({"seed": seed, "ms_per_step": t_seed, "value": rows / (t_seed * 1e-3),
                         "join_rows_per_step": rows})
        for k, v in lm.items():
            launches_ms.setdefault(k, []).extend(v)
        if si == 0:
            clocks = sampler.finish()
            first = {"prog": prog, "rows": rows, "sharded": sharded, "graphed": graphed,
                     "replay": replay}
            first["index_ms"] = _index_build_ms(prog, world)
            first["model"] = prog.roof_model()
            first["launches"] = count_launches(prog)
            first["proj_flops"] = count_proj_flops(prog)
            if not args.no_e2e:
                first["e2e"] = run_e2e(prog, args, world, dev, rows, replay)
            first["meta"] = {k: getattr(prog, k) for k in ("L", "dims") if hasattr(prog, k)}
            if (hasattr(prog, "setup_training") and prog._labels is not None and not sharded
                    and not args.l2_window):   # (the window is a stream attribute: no capture)
                first["train"] = run_train(prog, args)
            first["prog"] = None
        del prog, replay
        torch.cuda.empty_cache()
    vals = np.array([r["value"] for r in per_seed])
    msl = np.array([r["ms_per_step"] for r in per_seed])
    value = float(np.median(vals))
    t_step = float(np.median(msl))
    rows, sharded = first["rows"], first["sharded"]
    if world > 1:
        t = torch.tensor([first["index_ms"]], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        first["index_ms"] = float(t.item())

    def kernel_ms(name):
        v = launches_ms.get(name)
        return float(np.mean(v)) if v else None

    model = first["model"]
    per = {k: kernel_ms(k) for k in ["proj_fwd", "proj_bwd", "epi_bwd", "allgather", "reduce_scatter"]
           + list(model)}
    n_steps = args.steps * len(seeds)

    # ---- roofline of the dominant hot-path kernel (the fused LJA) ----
    peak, peak_src = peaks()
    # algorithmic bytes (or flops) per launch of each hot-path kernel (
    # programs._sum_bytes / _sum_bwd_bytes / HGTProgram.lja_bytes / DHNProgram.roof_model)
    dom = max(model, key=lambda k: per[k] or 0)
    ms, spec = per[dom], model[dom]
    if spec["bound"] == "hbm":
        achieved = spec["amount"] / (ms * 1e-3) / 1e9
        unit, pk, pk_src = "GB/s", peak, peak_src
    else:
        achieved = spec["amount"] / (ms * 1e-3) / 1e12
        unit, pk, pk_src = "TFLOP/s", FP32_ALU_TFLOPS, FP32_ALU_SRC
    roof = {"kernel": dom, "bound": spec["bound"], "achieved": round(achieved, 3), "peak": pk,
            "peak_source": pk_src, "unit": unit, "frac": round(achieved / pk, 4),
            "model": "gather (SURVEY sec 8d: every gathered row counted per join row)"
            if spec["bound"] == "hbm" else "factorised flop count (DESIGN.md sec 6)",
            "algorithmic_per_launch": int(spec["amount"]), "avg_launch_ms": round(ms, 5),
            "traffic": None}
    if spec.get("compulsory"):
        c = spec["compulsory"] / (ms * 1e-3) / 1e9
        roof["compulsory_per_launch"] = int(spec["compulsory"])
        roof["frac_compulsory"] = round(c / pk, 4)
    tr = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tr):
        with open(tr) as f:
            roof["traffic"] = json.load(f).get(dom)
        if roof["traffic"] and spec["bound"] == "hbm":
            # ncu DRAM bytes (one --set full capture, per launch) over the live launch time
            roof["frac_dram"] = round(roof["traffic"] / (ms * 1e-3) / 1e9 / pk, 4)
    # every bracketed kernel's mean launch time and its launches per step
    roof["kernel_ms"] = {k: (round(v, 5) if v else None) for k, v in per.items()}
    roof["launches_per_step"] = {k: len(v) // max(n_steps, 1) for k, v in launches_ms.items()}
    # the projections: bound by the tensor pipe under 3xTF32
    pf = first.get("proj_flops") or {}
    tpk, tpk_src = tf32_peak()
    proj = {}
    for k in ("proj_fwd", "proj_bwd"):
        n_l = roof["launches_per_step"].get(k, 0)
        if pf.get(k) and per.get(k) and n_l:
            t = per[k] * n_l * 1e-3
            proj[k] = {"flops_per_step": int(pf[k]), "ms_per_step": round(per[k] * n_l, 5),
                       "achieved": round(pf[k] / t / 1e12, 2),
                       "frac": round(pf[k] / t / 1e12 / tpk, 4)}
    if proj:
        roof["projection"] = {"bound": "tensor", "unit": "TFLOP/s", "peak": tpk,
                              "peak_source": tpk_src, "precision": args.prec, **proj}
    lja_ms = sum((per[k] or 0.0) * roof["launches_per_step"].get(k, 0) for k in model)
    result = None
    if rank == 0:
        cfg = {"workload": workload(args), "config": args.config,
               "join_rows_per_step": rows, **first["meta"],
               "projection_precision": args.prec, "l2": "flushed between timed steps",
               "step_launch": "one CUDA graph replay" if first["graphed"] else "eager launches",
               "seeds": seeds,
               **({"l2_window": "persisting window over each LJA's gathered matrix"}
                  if args.l2_window else {}),
               "parallelism": (f"hash-partition by group key x{world} ({SHARD_DESC[args.config]})"
                               if sharded else f"replica x{world}" if world > 1 else "single")}
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded; shapes of BASELINE.json configs, see DESIGN.md)",
            "config": cfg,
            "seed_stats": {"statistic": f"median over seeds {seeds} of the per-seed mean of "
                                        f"{args.steps} timed steps",
                           "value_median": value, "value_std": float(np.std(vals)),
                           "ms_median": t_step, "ms_std": float(np.std(msl)), "per_seed": per_seed},
            "lja_only": {"value": rows / (lja_ms * 1e-3) if lja_ms else None, "unit": UNIT,
                         "lja_ms_per_step": lja_ms,
                         "what": "join rows / summed LJA kernel time of a step (first seed's "
                                 "kernels bracketed by CUDA events)"},
            "index_build_ms": round(first["index_ms"], 3),
            "roofline": roof, "e2e": first.get("e2e"), "gpu_launches": first["launches"],
            **({"train": first["train"]} if first.get("train") else {}),
            "clocks": clocks,
        }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


SHARD_DESC = {
    "arxiv": "NCCL all-gather / reduce-scatter of the layer's source rows per layer",
    "cora": "NCCL all-gather / reduce-scatter of the layer's source rows per layer",
    "hyper": "NCCL all-gather / reduce-scatter per hop",
    "mag": "NCCL all-gather of K'/M' per source type, reduce-scatter of dK'/dM'",
    "dhn": "roots hash-partitioned, adjacency replicated, NCCL all-gather of f per layer and "
           "reduce-scatter of d f",
}


def workload(args):
    w = WORKLOAD[args.config]
    if args.config == "dhn":
        n = max(64, int(2_449_029 * args.dhn_scale))
        m = 2 * max(64, int(61_859_140 * args.dhn_scale))
        w += f" at scale {args.dhn_scale:g} ({n:,} nodes, {m:,} Edge tuples)"
    return w


def run_train(prog, args):
    """Full-batch training epochs of the GCN program (the paper's own
    Table 1 unit, ms/epoch -- PAPER.md:876 quotes 6.8 ms/epoch for GCN on Cora on an A40):
    forward + Loss(CrossEntropy) + backward + Adam(lr 0.01, weight decay 5e-4) on W, b, as one
    CUDA-graph replay per epoch (Adam's step counter on the device); device time per epoch
    with CUDA events, median of K epochs after W warm-up epochs."""
    import torch
    from paper_2605_24207_b200.programs import CapturedStep
    prog.setup_training(prog._labels)
    cs = CapturedStep(prog, timed=True, step_fn=prog.train_step)
    for _ in range(args.warmup):
        cs.replay()
    torch.cuda.synchronize()
    loss0 = float(prog.loss.item())
    ms = []
    for _ in range(args.steps):
        cs.replay()
        torch.cuda.synchronize()
        ms.append(cs.times()[0])
    return {"ms_per_epoch": float(np.median(ms)), "epochs_timed": args.steps,
            "loss_first_timed": loss0, "loss_last": float(prog.loss.item()),
            "what": "fit epoch: forward + CrossEntropy loss + backward + Adam (lr 0.01, "
                    "wd 5e-4) on W and b, one CUDA graph replay, L2 not flushed",
            "paper_context": "PAPER.md:876: RelaNN 6.8 +- 0.3 ms/epoch, PyG 4.9 +- 0.4 "
                             "(GCN on Cora, A40) -- other hardware and framework overheads"}


def count_proj_flops(prog):
    """Tensor-core flops of one step's projections as issued (rnn.FLOP_COUNTER; 3xTF32 = three
    tf32 products per term), from one untimed eager step."""
    import torch
    from paper_2605_24207_b200 import rnn
    rnn.FLOP_COUNTER = {}
    try:
        prog.step()
        torch.cuda.synchronize()
        return dict(rnn.FLOP_COUNTER)
    finally:
        rnn.FLOP_COUNTER = None


def tf32_peak():
    """Dense tf32 tensor peak: the measured bf16 matmul peak (MEASURED_PEAKS.json) x the
    guide's nominal tf32 / bf16 ratio (1.1 / 2.25 PFLOP/s, B200_PROFILING.md)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            bf16 = json.load(f)["bf16_tflops"]
        return round(bf16 * 1.1 / 2.25, 1), "derived: measured bf16 (MEASURED_PEAKS.json) x 1.1/2.25"
    except Exception:
        return 1100.0, "fallback: nominal dense tf32 (B200_PROFILING.md)"


def count_launches(prog):
    """Kernels launched by librnn.so in one step, counted by the CUDA profiler (CUPTI)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        prog.step()
        torch.cuda.synchronize()
    names = [e.name for e in p.events() if e.device_type.name == "CUDA"]
    ours = [n for n in names if "rnn::" in n or "seg_kernel" in n or "tc_gemm" in n]
    return len(ours)


def run_e2e(prog, args, world, dev, job_rows, replay=None):
    """Same metric through the public API with HOST buffers (programs.HostStreamedSteps):
    every step's inputs (node features and the upstream gradient, prog.host_io()) come from
    pinned host memory -- the H2D copy of step i+1 overlaps step i's compute on a copy stream
    -- and the parameter gradients are read back to pinned host memory; all of it inside the
    timed region (first copy to last read-back)."""
    import torch
    from paper_2605_24207_b200.programs import HostStreamedSteps
    ins, _ = prog.host_io()
    in_host = [x.cpu().pin_memory() for x in ins]
    pipe = HostStreamedSteps(prog, replay)
    h2d = sum(x.numel() * x.element_size() for x in in_host)
    d2h = sum(w.numel() * w.element_size() for w in pipe.out_host)
    steps = max(3, args.steps // 2)
    pipe.step(in_host)                 # warm-up
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    pipe.prefetch(in_host)
    for i in range(steps):
        pipe.step(next_inputs=in_host if i + 1 < steps else None)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / steps
    if world > 1:
        tt = torch.tensor([t], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t = float(tt.item())
    return {"value": job_rows / (t * 1e-3), "unit": UNIT, "ms_per_step": t,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "overlap": "H2D of step i+1 on a copy stream during step i"}


# ------------------------------------------------------------------------------------------
# the oracle (CPU, fp64): cpu_baseline and the --impl reference arm
# ------------------------------------------------------------------------------------------
def oracle_sample(cfg, seed):
    """The bounded sample of a config's step the oracle (fp64, single-threaded C, as it
    stands) is timed on (~5-30 s of one core): returns (run, join rows, description).
    arxiv -- the first of the three layers (fwd + bwd incl. projections); cora -- both
    layers; hyper / mag -- the whole step on a 1/20-scale instance of the same generator;
    dhn -- the whole layer on a 1/10,000-scale products-shaped graph (the oracle enumerates
    closed walks, so the full graph is out of reach)."""
    import oracle
    from oracle import programs as op
    oracle.build()
    if cfg == "hyper":
        data = make_graph(cfg, seed, sample=True)
        o1 = oracle.build_join_index(data["inc"]["node"], data["inc"]["hyper"],
                                     data["nodes"]["key"], data["hyperedges"]["key"])
        rows = 2 * o1["n_join_rows"]
        what = (f"whole step on a 1/20-scale hypergraph ({len(data['nodes']['key'])} nodes, "
                f"{len(data['inc']['node'])} incidences)")
        return (lambda: op.hypergraph_step(data)), rows, what
    if cfg == "mag":
        data = make_graph(cfg, seed, sample=True)
        rng = np.random.default_rng(1)
        d, h = data["d"], data["heads"]
        rows = sum(len(r["src"]) for r in data["rels"].values())
        Ws = {k: rng.standard_normal((d, d)) / np.sqrt(d) for k in ("k", "m", "q")}
        dO = {name: rng.standard_normal((data["n"][r["dst_type"]], d)) for name, r in data["rels"].items()}

        def run():
            for name, r in data["rels"].items():
                ts, tt = r["src_type"], r["dst_type"]
                op.hgt_relation(data["h"][ts], data["h"][tt], Ws["k"], Ws["m"], Ws["q"],
                                data["key"][ts], data["key"][tt], r["src"], r["dst"], h, dO[name])
        return run, rows, f"whole HGT layer on a 1/20-scale ogbn-mag-shaped schema ({rows} edges)"
    if cfg == "dhn":
        g = make_graph("dhn", seed, sample=True)
        keys = g["nodes"]["key"]
        n, d = g["nodes"]["x"].shape
        rng = np.random.default_rng(11)
        W = rng.standard_normal((9 * d, d)) / np.sqrt(d)
        dO = rng.standard_normal((n, 3 * d))
        oi = oracle.build_join_index(g["edges"]["src"], g["edges"]["dst"], keys, keys,
                                     within_by_src_key=True)
        ones = [np.ones((n, 1))]
        rows = int(oi["n_join_rows"]) + sum(int(round(oracle.dhn_fwd(k, oi, keys, ones * k).sum()))
                                            for k in (3, 4))
        return (lambda: op.dhn_step(g, W, dO)), rows, (
            f"whole layer (C2/C3/C4 fwd+bwd, projections) on a {n}-node products-shaped graph "
            f"({len(g['edges']['src'])} Edge rows, {rows} homomorphisms)")
    graph = make_graph(cfg, seed)
    L = len(graph["W"])
    layers = 1 if cfg == "arxiv" else L
    o = oracle.build_join_index(graph["edges"]["src"], graph["edges"]["dst"],
                                graph["nodes"]["key"], graph["nodes"]["key"])
    rows = o["n_join_rows"] * layers
    return (lambda: op.gcn_step(graph, layers=layers)), rows, (
        f"first {layers} of {L} layers (fwd+bwd incl. projections, {rows} join rows)")


def _oracle_worker(cfg, seed, reps, barrier, out):
    import time as _t
    run, rows, what = oracle_sample(cfg, seed)
    barrier.wait()
    t0 = _t.time()
    for _ in range(reps):
        run()
    out.put((t0, _t.time(), rows, what))


def host_info():
    info = {"nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["model"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        info["lscpu"] = {k.strip(): v.strip() for k, v in (
            l.split(":", 1) for l in subprocess.run(["lscpu"], capture_output=True, text=True,
                                                     timeout=10).stdout.splitlines() if ":" in l)
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core",
                             "NUMA node(s)", "L3 cache")}
    except Exception:
        pass
    return info


def oracle_timing(args, procs=None, reps=1):
    """The oracle timed on the host's cores: `procs` concurrent processes (default: every
    core), each running the bounded sample `reps` times; value = procs x reps x rows / wall
    (first start to last end).  The single-core figure is one process alone.  Returns
    (cpu_baseline dict, wall seconds of the all-core run, rows per sample)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")        # fresh interpreters: no CUDA state in the workers
    seed = int(str(args.seeds).split(",")[0])

    def run(p):
        barrier, q = ctx.Barrier(p), ctx.Queue()
        ws = [ctx.Process(target=_oracle_worker, args=(args.config, seed, reps, barrier, q))
              for _ in range(p)]
        for w in ws:
            w.start()
        res = [q.get() for _ in ws]
        for w in ws:
            w.join()
        wall = max(r[1] for r in res) - min(r[0] for r in res)
        return wall, res[0][2], res[0][3]

    P = procs or os.cpu_count() or 1
    t1, rows, what = run(1)
    tP, _, _ = run(P) if P > 1 else (t1, rows, what)
    single = rows * reps / t1
    value = P * rows * reps / tP
    return {"value": value, "unit": UNIT, "cores": P, "kind": "oracle",
            "sample": f"{args.config}: {what}; {P} concurrent processes (one per host core), "
                      f"each running the sample {reps}x; value = {P} x rows / wall "
                      f"({tP:.2f} s); fp64 single-threaded C per process",
            "single_core": {"value": single, "cores": 1, "seconds": t1 / reps},
            "host": host_info()}, tP, rows


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and rank != 0:
        return None
    reps = max(1, min(args.steps, 2))
    cb, t, rows = oracle_timing(args, reps=reps)
    return {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": reps, "warmup": 0, "ms_per_step": t * 1e3 / reps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(args), "config": args.config,
                       "join_rows_per_step": rows},
            "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    DHN_SCALE[0] = args.dhn_scale
    if args.impl == "reference":
        res = run_reference(args)
    else:
        res = run_ours(args)
        if res is not None and not args.no_cpu_baseline:
            res["cpu_baseline"] = oracle_timing(args)[0]
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
