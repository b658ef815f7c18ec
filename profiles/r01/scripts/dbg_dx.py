import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2605_24207_b200 import rnn
M, K, N = 2708, 1433, 16
rng = np.random.default_rng(M + K + N)
X = (rng.standard_normal((M, K)) / np.sqrt(K)).astype(np.float32)
W = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
b = rng.standard_normal(N).astype(np.float32)
def padded(x):
    n, d = x.shape; ld = (d + 3) // 4 * 4
    buf = torch.full((n, ld), float("nan"), device="cuda"); buf[:, :d] = torch.from_numpy(x); return buf[:, :d]
dY = rng.standard_normal((M, N)).astype(np.float32)
for prec in ["3xtf32", "tf32"]:
    Xd, Wd = padded(X), padded(W)
    Y = rnn.project(Xd, Wd, torch.from_numpy(b).cuda(), prec=prec)
    torch.cuda.synchronize()
    print(prec, "W intact", bool(torch.equal(Wd.cpu(), torch.from_numpy(W))), "X intact", bool(torch.equal(Xd.cpu(), torch.from_numpy(X))),
          "Y err", float(np.abs(Y.cpu().numpy() - (X.astype(np.float64) @ W.T.astype(np.float64) + b)).max()))
    dX, dW, db = rnn.project_bwd(Xd, Wd, padded(dY), want_db=True, prec=prec)
    ref = dY.astype(np.float64) @ W.astype(np.float64)
    g = dX.cpu().numpy()
    bad = np.abs(g - ref) > 1e-2 * (np.abs(ref) + 0.1)
    print(prec, "bad", bad.sum(), "nan", np.isnan(g).sum())
    if bad.any():
        r, c = np.nonzero(bad); print(" rows", np.unique(r)[:20], len(np.unique(r)), " cols", np.unique(c)[:40], len(np.unique(c)))
