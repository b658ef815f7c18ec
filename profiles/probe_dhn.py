"""Phase timing of the DHN C4 kernel (clock64 per phase, summed over CTAs; internal hook
rnn_internal_dhn_stats) on the bench's products-shaped graph.  python profiles/probe_dhn.py [scale]"""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_24207_b200 import programs, rnn  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
g = synth.products_like(42, scale=scale)
prog = programs.DHNProgram(g, device="cuda", ks=(4,))
L = rnn.lib()
st = (C.c_ulonglong * 16)()
f = prog._f(4, prog.Y)
rnn.project(prog.H, prog.W, out=prog.Y)
rnn.dhn_fwd(prog.idx, 4, f, out=prog.out[:, :prog.d], ws=prog.ws)
torch.cuda.synchronize()
L.rnn_internal_dhn_stats(st, 1, 1)
t = time.time()
rnn.dhn_fwd(prog.idx, 4, f, out=prog.out[:, :prog.d], ws=prog.ws)
torch.cuda.synchronize()
el = time.time() - t
L.rnn_internal_dhn_stats(st, 0, 1)
names = ["root setup", "out sweep", "finalize G", "in sweep", "clear", "reduce/store"]
tot = sum(st[i] for i in range(6))
print(f"scale {scale}: dhn4 fwd {el * 1e3:.1f} ms wall; roots {st[7]}, partitions {st[6]}, chunked {st[8]}")
for i, nme in enumerate(names):
    print(f"  {nme:14s} {st[i] / 1e9:10.3f} Gclk  {st[i] / max(tot, 1) * 100:5.1f}%")
