import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2605_24207_b200 import rnn
def err(a, ref):
    a = a.double(); rms = ref.pow(2).mean().sqrt()
    return float(((a - ref).abs() / torch.maximum(ref.abs(), rms)).max()), float((a - ref).pow(2).mean().sqrt() / rms)
torch.manual_seed(0)
for M in (100000, 1000000):
    X = torch.randn(M, 128, device="cuda") / 128 ** 0.5
    W = torch.randn(128, 128, device="cuda") / 128 ** 0.5
    dY = torch.randn(M, 128, device="cuda")
    Yr = X.double() @ W.double().T
    dXr = dY.double() @ W.double()
    dWr = dY.double().T @ X.double()
    for prec in ("3xtf32", "tf32"):
        Y = rnn.project(X, W, prec=prec)
        dX, dW, _ = rnn.project_bwd(X, W, dY, want_dx=True, prec=prec)
        _, dW2, _ = rnn.project_bwd(X, W, dY, want_dx=False, prec=prec)
        print(M, prec, "Y", err(Y, Yr), "dX", err(dX, dXr), "dW", err(dW, dWr), "dW(no dx)", err(dW2, dWr), "nan", bool(torch.isnan(dW2).any()), flush=True)
# internal gemm hook: C = A B with MN / K-major combos, small
import ctypes as C
L = rnn.lib()
L.rnn_internal_gemm.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
for amn in (0, 1):
    for bmn in (0, 1):
        Mm, N, Kr = 256, 128, 4096
        A = torch.randn(Kr, Mm, device="cuda") if amn else torch.randn(Mm, Kr, device="cuda")
        B = torch.randn(Kr, N, device="cuda") if bmn else torch.randn(N, Kr, device="cuda")
        Ad = A.double().T if amn else A.double()
        Bd = B.double() if bmn else B.double().T
        ref = Ad @ Bd
        for prec in (1, 0):
            Cc = torch.zeros(Mm, N, device="cuda")
            st = L.rnn_internal_gemm(amn, bmn, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), Mm, N, Kr, Cc.data_ptr(), N, prec, None)
            torch.cuda.synchronize()
            print("gemm a_mn", amn, "b_mn", bmn, "prec", prec, "st", st, err(Cc, ref), flush=True)
