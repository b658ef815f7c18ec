#!/usr/bin/env python
"""Summarise ncu output brought back by profiles/run_r01.sh into markdown.

  python profiles/summarize.py gpurun_out > profiles/rNN_ncu_summary.md

Launch lists (`launches_<cfg>.csv`, gpu__time_duration.sum per launch, cold-cache and
serialised) give each kernel's SHARE of the run; full captures (`prof_<cfg>_raw.csv`) give DRAM
bytes, throughput, occupancy and cache hit rates per captured launch."""
import collections
import csv
import io
import os
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def launches(path):
    txt = open(path).read()
    lines = [l for l in txt.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    if not rows:
        return None
    hdr = rows[0]
    k, u, v, m = (hdr.index(x) for x in ("Kernel Name", "Metric Unit", "Metric Value", "Metric Name"))
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[m] != "gpu__time_duration.sum":
            continue
        agg.setdefault(r[k], []).append(float(r[v].replace(",", "")) * SCALE.get(r[u], 1.0))
    return agg


def short(name, n=90):
    name = name.replace("rnn::<unnamed>::", "").replace("rnn::", "").replace("(anonymous namespace)::", "")
    return name[:n]


RAW = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM rd"),
       ("dram__bytes_write.sum", "DRAM wr"),
       ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
       ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
       ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
       ("launch__registers_per_thread", "regs"),
       ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
       ("sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active", "tensor %")]


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for d in data:
        rec = {"Kernel": short(d[hdr.index("Kernel Name")], 70)}
        for key, lab in RAW:
            if key in hdr:
                i = hdr.index(key)
                rec[lab] = f"{d[i]} {units[i]}".strip()
        out.append(rec)
    return out


def main(d):
    print(f"# ncu summary ({os.path.abspath(d)})\n")
    for cfg in ("arxiv", "cora", "hyper", "mag", "dhn"):
        p = os.path.join(d, f"launches_{cfg}.csv")
        if os.path.exists(p):
            agg = launches(p)
            if agg:
                tot = sum(sum(v) for v in agg.values())
                print(f"## {cfg}: launch list (whole process: index build + warm-up + 1 step)\n")
                print(f"{sum(len(v) for v in agg.values())} launches, {tot / 1e3:.2f} ms total\n")
                print("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
                for n, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:16]:
                    print(f"| `{short(n)}` | {len(v)} | {sum(v):.1f} | {sum(v) / len(v):.1f} | "
                          f"{sum(v) / tot * 100:.1f}% |")
                print()
        p = os.path.join(d, f"prof_{cfg}_raw.csv")
        if os.path.exists(p):
            recs = raw(p)
            if recs:
                cols = list(recs[0].keys())
                print(f"## {cfg}: full capture (`ncu --set full`), per launch\n")
                print("| " + " | ".join(cols) + " |\n|" + "---|" * len(cols))
                for r in recs:
                    print("| " + " | ".join(str(r.get(c, "")) for c in cols) + " |")
                print()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out")
