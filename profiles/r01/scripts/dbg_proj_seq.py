import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2605_24207_b200 import rnn
def padded(x):
    n, d = x.shape; ld = (d + 3) // 4 * 4
    buf = torch.full((n, ld), float("nan"), device="cuda"); buf[:, :d] = torch.from_numpy(x); return buf[:, :d]
fails = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    for (M, K, N) in [(300, 128, 128), (2708, 1433, 16), (2708, 16, 7), (1000, 40, 200), (129, 32, 48), (100000, 128, 128)]:
        for prec in ["3xtf32", "tf32"]:
            rng = np.random.default_rng(M + K + N)
            X = (rng.standard_normal((M, K)) / np.sqrt(K)).astype(np.float32)
            W = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
            dY = rng.standard_normal((M, N)).astype(np.float32)
            Xd, Wd = padded(X), padded(W)
            Y = rnn.project(Xd, Wd, prec=prec)
            dX, dW, db = rnn.project_bwd(Xd, Wd, padded(dY), want_db=True, prec=prec)
            for name, g, r in (("Y", Y, X.astype(np.float64) @ W.T), ("dX", dX, dY.astype(np.float64) @ W), ("dW", dW, dY.T.astype(np.float64) @ X)):
                g = g.cpu().numpy()
                tolr = 2e-3 if prec == "3xtf32" else 5e-2
                bad = np.abs(g - r) > tolr * (np.abs(r) + np.abs(r).max() * 0.05)
                if bad.any():
                    fails += 1
                    rr, cc = np.nonzero(bad)
                    print(it, M, K, N, prec, name, "bad", bad.sum(), "zeros", int((g[bad] == 0).sum()), "rows", np.unique(rr)[:8], "cols", np.unique(cc)[:8], flush=True)
print("fails", fails)
