"""Probe: rnn_project_bwd vs rnn_project_bwd_relu at the arxiv shape (169,343 x 128, N = 128),
CUDA-event timed; the relu variant fuses the mask + bias column sums into tc_projt's epilogue."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_2605_24207_b200 import rnn  # noqa: E402

M, K, N = 169_343, 128, 128
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
X = torch.randn(M, K, device=dev, generator=g).relu_()
W = torch.randn(N, K, device=dev, generator=g) / 11.3
dY = torch.randn(M, N, device=dev, generator=g)
dX = torch.empty(M, K, device=dev)
dW = torch.empty(N, K, device=dev)
db = torch.empty(K, device=dev)
ws = rnn.Workspace(dev)


def run(relu, reps=20):
    for _ in range(3):
        rnn.project_bwd(X, W, dY, want_dx=True, ws=ws, dx_out=dX, dw_out=dW, relu_in=relu,
                        d_in_bias=db if relu else None)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        rnn.project_bwd(X, W, dY, want_dx=True, ws=ws, dx_out=dX, dw_out=dW, relu_in=relu,
                        d_in_bias=db if relu else None)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


if os.environ.get("PROBE_ONE"):
    run(os.environ["PROBE_ONE"] == "relu", reps=1)
else:
    print(f"plain {run(False) * 1e3:.1f} us   relu {run(True) * 1e3:.1f} us")
