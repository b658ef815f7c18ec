"""Probe: how does tcgen05.mma kind::tf32 convert raw fp32 operands?  (truncate to 10 mantissa
bits, round to nearest, or use them unconverted).  Decides whether the 3xTF32 split must store
hi = tf32(x) explicitly or can feed raw x as its hi part.

x = 1 + 3*2^-12 (0.75 tf32 ulp above 1) times w = 1:  truncation -> 1, RN -> 1 + 2^-10,
unconverted -> 1 + 3*2^-12.  Run on a GPU box:  python profiles/probe_tf32.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24207_b200 import rnn  # noqa: E402

xs = np.array([1 + 3 * 2.0 ** -12, 1 + 2.0 ** -12, -(1 + 3 * 2.0 ** -12), 1 + 2.0 ** -11], np.float64)
X = torch.zeros(128, 32, dtype=torch.float32, device="cuda")
X[: len(xs), 0] = torch.tensor(xs, dtype=torch.float32)
W = torch.zeros(32, 32, dtype=torch.float32, device="cuda")
W[0, 0] = 1.0
Y = rnn.project(X, W, prec="tf32")[: len(xs), 0].double().cpu().numpy()
trunc = np.array([np.float32(x).view(np.uint32) & 0xFFFFE000 for x in xs], np.uint32).view(np.float32)
for x, y, t in zip(xs, Y, trunc):
    kind = "truncate" if y == t else ("unconverted" if y == np.float32(x) else "round")
    print(f"x={x!r:24} mma={y!r:24} trunc={float(t)!r:24} -> {kind}")
