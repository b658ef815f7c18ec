"""Projection-backward time vs the TMEM accumulation chunk (RNN_GEMM_CHUNK) at MAG shapes."""
import sys, torch, numpy as np, json
sys.path.insert(0, '.')
from paper_2605_24207_b200 import rnn
res = {}
for (M, K, N) in [(736389, 128, 640), (1134649, 128, 512), (169343, 128, 128), (1000000, 128, 128)]:
    X = torch.randn(M, K, device="cuda") / K ** 0.5
    W = torch.randn(N, K, device="cuda") / K ** 0.5
    dY = torch.randn(M, N, device="cuda")
    ws = rnn.Workspace("cuda")
    dX = torch.empty(M, K, device="cuda"); dW = torch.empty(N, K, device="cuda")
    for _ in range(3):
        rnn.project_bwd(X, W, dY, ws=ws, dx_out=dX, dw_out=dW)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); rnn.project_bwd(X, W, dY, ws=ws, dx_out=dX, dw_out=dW); e.record()
        torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    ref = (dY.double().T @ X.double())
    err = float(((dW.double() - ref).abs() / torch.maximum(ref.abs(), ref.pow(2).mean().sqrt())).max())
    res[f"{M}x{K}x{N}"] = {"ms": float(np.median(ts)), "dW_err": err}
    del X, W, dY, dX, dW
print(json.dumps(res))
