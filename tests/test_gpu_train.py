"""GPU parity of the training step: the loss relation
Loss(; CrossEntropyLoss()(logits, label)) and the ?fit optimiser (PAPER.md:554,
:567-568: Adam, lr 0.01, weight decay 5e-4) against the oracle, and full-batch GCN training on
the Cora-shaped config: the per-epoch losses follow the oracle's fit, one step's parameter
update equals the oracle's Adam on the same gradients, and 100 epochs converge."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import programs as op
from tests.util import FP32_TOL, assert_close, np_

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rnn():
    from paper_2605_24207_b200 import rnn
    return rnn


def cu(a):
    return torch.as_tensor(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n,C", [(1000, 7), (70000, 40), (3, 128)])
def test_xent_parity(rnn, n, C):
    rng = np.random.default_rng(n + C)
    x = (rng.standard_normal((n, C)) * 3).astype(np.float32)
    lab = rng.integers(0, C, n).astype(np.int64)
    lab[rng.random(n) < 0.3] = -1
    lab[0] = 1
    loss, d = rnn.softmax_xent(cu(x), cu(lab))
    rl, rd = oracle.softmax_xent(x, lab)
    assert abs(float(loss.item()) - rl) <= FP32_TOL * rl
    assert_close(np_(d), rd, FP32_TOL, "d_logits")


def test_adam_parity(rnn):
    rng = np.random.default_rng(5)
    shapes = [(300, 40), (128,), (7, 16)]
    ps = [rng.standard_normal(s).astype(np.float32) for s in shapes]
    dev = [cu(p) for p in ps]
    opt = rnn.Adam(dev, lr=0.01, weight_decay=5e-4)
    ref = [(p.astype(np.float64).reshape(-1).copy(), np.zeros(p.size), np.zeros(p.size)) for p in ps]
    for t in range(1, 4):
        gs = [(rng.standard_normal(s) * 0.1).astype(np.float32) for s in shapes]
        opt.step([cu(g) for g in gs])
        for (p, m, v), g in zip(ref, gs):
            oracle.adam(p, g.reshape(-1), m, v, 0.01, t, wd=5e-4)
    assert int(opt.t.item()) == 3
    for d, (p, _, _) in zip(dev, ref):
        assert_close(np_(d).reshape(-1), p, FP32_TOL, "param after 3 Adam steps")


def test_gcn_fit_cora(rnn):
    from paper_2605_24207_b200 import programs
    g = synth.cora_like(42)
    prog = programs.GCNProgram(g)
    prog.setup_training(g["labels"])
    # one step: the update is the oracle's Adam on the GPU's own gradients (the Adam update
    # normalises the gradient, so both sides take it from the same values)
    W0 = [np_(w).astype(np.float64) for w in prog.W]
    b0 = [np_(b).astype(np.float64) for b in prog.b]
    prog.train_step()
    torch.cuda.synchronize()
    for l in range(prog.L):
        for p0, gr, new in ((W0[l], np_(prog.dW[l]), np_(prog.W[l])), (b0[l], np_(prog.db[l]), np_(prog.b[l]))):
            p = p0.reshape(-1).copy()
            oracle.adam(p, gr.reshape(-1), np.zeros(p.size), np.zeros(p.size), 0.01, 1, wd=5e-4)
            assert_close(new.reshape(-1), p, FP32_TOL, f"layer {l} update")
    # five epochs: the loss trajectory follows the oracle's fit from the same start
    prog2 = programs.GCNProgram(g)
    prog2.setup_training(g["labels"])
    losses = []
    for _ in range(5):
        losses.append(float(prog2.train_step().item()))
    ref, _, _ = op.gcn_fit(g, g["labels"], 5)
    np.testing.assert_allclose(losses, ref, rtol=FP32_TOL)


def test_gcn_fit_converges_graph_replay(rnn):
    """100 epochs, the training step captured once as a CUDA graph (the Adam
    step counter lives on the device): the training loss falls well below its start."""
    from paper_2605_24207_b200 import programs
    g = synth.cora_like(42)
    prog = programs.GCNProgram(g)
    prog.setup_training(g["labels"], learn_embeddings=True)
    l0 = float(prog.train_step().item())
    cs = programs.CapturedStep(prog, step_fn=prog.train_step)
    for _ in range(99):
        cs.replay()
    torch.cuda.synchronize()
    assert int(prog.opt.t.item()) == 100 + 2          # + the capture's 2 warm-up steps
    l1 = float(prog.loss.item())
    assert l1 < 0.5 * l0, (l0, l1)
