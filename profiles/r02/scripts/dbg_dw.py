import sys, numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle
from paper_2605_24207_b200 import programs, rnn
hg = synth.hypergraph_like(42)
prog = programs.HypergraphProgram(hg)
prog.step(); torch.cuda.synchronize()
X = prog.X; dZ = prog.dZ
ref = (dZ.double().T @ X.double()).cpu().numpy()
def err(a):
    rms = np.sqrt(np.mean(ref**2)); den = np.maximum(np.abs(ref), rms)
    e = np.abs(a - ref) / den
    i = np.unravel_index(np.argmax(e), e.shape)
    return e.max(), i, np.sqrt(np.mean((a-ref)**2))/rms
d0 = prog.dTheta.cpu().numpy()
print("prog dTheta vs fp64:", err(d0))
for prec in ("3xtf32", "tf32"):
    outs = []
    for rep in range(3):
        _, dW, _ = rnn.project_bwd(X, prog.theta, dZ, want_dx=False, prec=prec)
        outs.append(dW.cpu().numpy())
    print(prec, [err(o)[0] for o in outs], "bitwise repeat:", all(np.array_equal(outs[0], o) for o in outs))
# random data same shape
rng = np.random.default_rng(0)
Xr = torch.tensor(rng.standard_normal((1000000, 128)).astype(np.float32) / np.sqrt(128), device="cuda")
Dr = torch.tensor(rng.standard_normal((1000000, 128)).astype(np.float32), device="cuda")
ref = (Dr.double().T @ Xr.double()).cpu().numpy()
for prec in ("3xtf32", "tf32"):
    _, dW, _ = rnn.project_bwd(Xr, prog.theta, Dr, want_dx=False, prec=prec)
    print("random", prec, err(dW.cpu().numpy()))
# row-norm distribution of dZ
n = dZ.norm(dim=1).cpu().numpy(); print("dZ row norms: max", n.max(), "median", np.median(n), "top share", np.sort(n**2)[-100:].sum() / (n**2).sum())
