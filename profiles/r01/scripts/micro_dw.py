"""Split the projection backward into its parts (CUDA events, median of 20): dW only
(want_dx=False) vs dX + dW, for both precisions, at the hot-path shapes."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24207_b200 import rnn


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2] * 1e3


for (M, K, N) in [(169343, 128, 128), (1000000, 128, 128), (736389, 128, 768)]:
    X = torch.randn(M, K, device="cuda"); W = torch.randn(N, K, device="cuda")
    Y = torch.empty(M, N, device="cuda"); dY = torch.randn(M, N, device="cuda")
    ws = rnn.Workspace("cuda")
    for prec in ("3xtf32", "tf32"):
        f = t(lambda: rnn.project(X, W, out=Y, prec=prec))
        dw = t(lambda: rnn.project_bwd(X, W, dY, want_dx=False, prec=prec, ws=ws))
        b = t(lambda: rnn.project_bwd(X, W, dY, want_dx=True, prec=prec, ws=ws))
        print(json.dumps(dict(M=M, K=K, N=N, prec=prec, fwd_us=round(f, 1), dw_us=round(dw, 1),
                              bwd_us=round(b, 1), dx_us=round(b - dw, 1),
                              ideal_dw_us=round((M * K + M * N) * 4 / 6542e3, 1))), flush=True)
    del X, W, Y, dY
