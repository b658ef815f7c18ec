"""Per-role wait cycles and TMA issue->landed latency of tc_gemm_kernel running the dW = dY^T X
split-K GEMM of rnn_project_bwd (internal hook rnn_internal_gemm_stats).
python profiles/probe_gemm.py"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24207_b200 import rnn  # noqa: E402

L = rnn.lib()
for (M, K, N) in [(169343, 128, 128), (1000000, 128, 128), (736389, 128, 768)]:
    X = torch.randn(M, K, device="cuda"); W = torch.randn(N, K, device="cuda")
    dY = torch.randn(M, N, device="cuda")
    ws = rnn.Workspace("cuda")
    for prec in ("3xtf32", "tf32"):
        for _ in range(3):
            rnn.project_bwd(X, W, dY, want_dx=False, prec=prec, ws=ws)
        torch.cuda.synchronize()
        st = (C.c_ulonglong * 16)()
        L.rnn_internal_gemm_stats(st, 1)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); rnn.project_bwd(X, W, dY, want_dx=False, prec=prec, ws=ws); b.record()
        torch.cuda.synchronize()
        L.rnn_internal_gemm_stats(st, 0)
        ms = a.elapsed_time(b)
        ctas = 148
        print(f"M={M} K={K} N={N} {prec}: {ms * 1e3:.1f} us (dW incl. reduce); per CTA kclk: "
              f"prod total {st[8] / ctas / 1e3:.1f} waits {st[0] / ctas / 1e3:.1f} | "
              f"mma total {st[9] / ctas / 1e3:.1f} waits {st[1] / ctas / 1e3:.1f} | "
              f"conv total {st[10] / ctas / 1e3:.1f} waits {st[2] / ctas / 1e3:.1f} | "
              f"TMA latency {st[3] / max(st[4], 1):.0f} clk over {st[4]} stages", flush=True)
    del X, W, dY
