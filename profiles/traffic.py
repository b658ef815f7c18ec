#!/usr/bin/env python
"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum, ncu --set full) of the
kernel bench.py reports the roofline for, written to profiles/traffic_<cfg>.json (bench.py puts
it in roofline.traffic).  A "launch" is what bench.py times as one kernel: one LJA call, i.e.
for the HGT softmax backward both passes (SmBwd1Pol + SmBwd2Pol) of one relation.

  python profiles/traffic.py gpurun_out profiles/r01
"""
import csv
import json
import os
import shutil
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def captures(path):
    rows = list(csv.reader(open(path)))
    rows = [r for r in rows if r]
    h, u = rows[0], rows[1]
    k = h.index("Kernel Name")
    rd, wr = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    out = []
    for r in rows[2:]:
        try:
            b = float(r[rd]) * UNIT[u[rd]] + float(r[wr]) * UNIT[u[wr]]
        except (ValueError, KeyError):
            continue
        out.append((r[k], b))
    return out


def mean(xs):
    return sum(xs) / len(xs) if xs else None


def main(src, dst):
    res = {}
    for cfg in ("arxiv", "hyper", "mag"):
        raw = os.path.join(src, f"prof_{cfg}_raw.csv")
        if not os.path.exists(raw):
            continue
        cap = captures(raw)
        t = {"_source": f"{dst}/prof_{cfg}_raw.csv (ncu --set full, one eager step): "
                        "dram__bytes_read.sum + dram__bytes_write.sum per launch, mean"}
        if cfg == "mag":
            f = [b for n, b in cap if "SmFwdPol" in n]
            t["lja_fwd"] = mean(f)
            dk = [b for n, b in cap if "sm_d_kernel" in n]
            ba = [b for n, b in cap if "SmBwdAPol" in n]
            bb = [b for n, b in cap if "SmBwdBPol" in n]
            b1 = [b for n, b in cap if "SmBwd1Pol" in n]
            b2 = [b for n, b in cap if "SmBwd2Pol" in n]
            if ba and len(ba) == len(bb) == len(dk):      # source-major backward (default)
                t["lja_bwd"] = mean([x + y + z for x, y, z in zip(dk, ba, bb)])
                t["_source"] += "; lja_bwd = D kernel + pass A + pass B of one relation"
            elif b1 and len(b1) == len(b2):                # two-pass (a, de) backward
                t["lja_bwd"] = mean([x + y for x, y in zip(b1, b2)])
                t["_source"] += "; lja_bwd = pass 1 + pass 2 of one relation"
        else:
            t["lja_fwd"] = mean([b for n, b in cap if "LeanFwdMeta" in n])
            t["lja_bwd"] = mean([b for n, b in cap if "LeanBwdMeta" in n])
        t = {k: (int(v) if isinstance(v, float) else v) for k, v in t.items() if v is not None}
        with open(os.path.join("profiles", f"traffic_{cfg}.json"), "w") as fh:
            json.dump(t, fh, indent=1)
        res[cfg] = t
        shutil.copy(raw, os.path.join(dst, f"prof_{cfg}_raw.csv"))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out",
         sys.argv[2] if len(sys.argv) > 2 else "profiles/r01")
