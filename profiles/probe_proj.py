"""Per-role wait cycles of tc_projt_kernel (internal hook rnn_internal_proj_stats): which stage
of the TMA -> (3xTF32 split) -> tcgen05.mma -> epilogue pipeline is the bottleneck.
python profiles/probe_proj.py"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24207_b200 import rnn  # noqa: E402

L = rnn.lib()
names = ["producer waits slot", "MMA waits W", "MMA waits accum", "MMA waits stage",
         "converter waits stage", "epilogue waits accum"]
for (M, K, N) in [(169343, 128, 128), (1000000, 128, 128), (1134649, 128, 512), (736389, 128, 768)]:
    X = torch.randn(M, K, device="cuda"); W = torch.randn(N, K, device="cuda")
    Y = torch.empty(M, N, device="cuda")
    for prec in ("3xtf32", "tf32"):
        for _ in range(3):
            rnn.project(X, W, out=Y, prec=prec)
        torch.cuda.synchronize()
        st = (C.c_ulonglong * 16)()
        L.rnn_internal_proj_stats(st, 1)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); rnn.project(X, W, out=Y, prec=prec); b.record(); torch.cuda.synchronize()
        L.rnn_internal_proj_stats(st, 0)
        ms = a.elapsed_time(b)
        ctas = 148 // ((N + 127) // 128) * ((N + 127) // 128)
        tot = [st[8 + i] / ctas for i in range(4)]
        print(f"M={M} K={K} N={N} {prec}: {ms * 1e3:.1f} us, role totals (kclk/CTA) "
              f"prod {tot[0] / 1e3:.1f} mma {tot[1] / 1e3:.1f} conv {tot[2] / 1e3:.1f} epi {tot[3] / 1e3:.1f}")
        for i, nme in enumerate(names):
            print(f"    {nme:22s} {st[i] / ctas / 1e3:9.1f} kclk/CTA")
    del X, W, Y
