import sys, torch, numpy as np
sys.path.insert(0, '.')
import synth
from paper_2605_24207_b200 import programs, rnn
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.004
mag = synth.mag_like(5, scale=scale)
prog = programs.HGTProgram(mag)
print({t: tuple(prog.W[t].shape) for t in prog.W}, flush=True)
prog.forward(); torch.cuda.synchronize(); print("fwd ok", flush=True)
prog.backward(); torch.cuda.synchronize(); print("bwd ok", flush=True)
