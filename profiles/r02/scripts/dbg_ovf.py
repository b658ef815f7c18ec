import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle
from paper_2605_24207_b200 import rnn
from tests.test_gpu_dhn_scale import gpu_adj, ora_adj, cu
rng = np.random.default_rng(9)
nv = 600
n_nodes = nv + 3 + 400
keys = rng.permutation(n_nodes).astype(np.int64) * 5
root, w0, p0 = 0, 1, 2
v = np.arange(3, 3 + nv)
src = [np.full(nv, root), np.repeat(v, 200), [w0], [p0]]
dst = [v, np.full(nv * 200, w0), [p0], [root]]
a, b = rng.integers(0, n_nodes, 4000), rng.integers(0, n_nodes, 4000)
ok = a != b
src.append(a[ok]); dst.append(b[ok])
s, t = np.concatenate(src), np.concatenate(dst)
e_n, e_v = keys[s], keys[t]
gi = gpu_adj(rnn, keys, e_n, e_v); oi = ora_adj(keys, e_n, e_v)
rows = np.searchsorted(gi.group_key.cpu().numpy(), oi["group_key"])
n = len(keys)
ones = cu(np.ones((n, 1), np.float32))
for k in (3, 4):
    c = rnn.dhn_count(gi, k).cpu().numpy()
    f = rnn.dhn_fwd(gi, k, [None] + [ones] * (k - 1)).cpu().numpy()[:, 0]
    o = oracle.dhn_fwd(k, oi, keys, [np.ones((n, 1))] * k)[:, 0]
    print(k, "count==oracle", np.array_equal(c[rows], o.astype(np.int64)), "fp32 ones==oracle", np.array_equal(f[rows], o))
    bad = np.nonzero(f[rows] != o)[0]
    print("  bad roots", len(bad), [(int(i), float(f[rows][i]), float(o[i]), int(c[rows][i])) for i in bad[:10]])
d = 8
for trial in range(3):
    fr = [rng.uniform(0.5, 1.5, (n, d)).astype(np.float32) for _ in range(4)]
    out = rnn.dhn_fwd(gi, 4, [cu(x) for x in fr]).cpu().numpy()[rows]
    ref = oracle.dhn_fwd(4, oi, keys, fr)
    err = np.abs(out - ref) / np.maximum(np.abs(ref), np.sqrt(np.mean(ref ** 2)))
    i = np.unravel_index(np.argmax(err), err.shape)
    print("trial", trial, "max err", err.max(), "at group", i, "key", oi["group_key"][i[0]], "val", out[i], ref[i], "rms", np.sqrt(np.mean(ref**2)))
    # which node is it
    kk = oi["group_key"][i[0]]
    node = np.nonzero(keys == kk)[0][0]
    print("   node id", node, "deg", np.diff(oi["group_ptr"])[i[0]])
