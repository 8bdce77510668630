"""Compare batch-path sums between two libraries (HP_LIB=a vs b) and across repeats."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, numpy as np, torch
sys.path.insert(0, "%s")
import paper_2005_07068_b200 as hp, workloads as W, oracle as O
ctx = hp.Context(640, 480, max_particles=4096)
obs = O.synthesize(W.H_A, O.camera(640, 480))
ctx.set_observation(obs.depth, obs.mask)
P = torch.tensor(W.swarm_c4().astype(np.float32), device="cuda")
outs = []
for r in range(3):
    s, c = ctx.eval_sums(P)
    outs.append(s.cpu().numpy())
for r in range(1, 3):
    print("repeat", r, "differs at", int((outs[r] != outs[0]).any(axis=1).sum()), "poses")
np.save(sys.argv[1], outs[0])
''' % ROOT
for lib in sys.argv[1:]:
    env = dict(os.environ, HP_LIB=lib) if lib != "default" else dict(os.environ)
    out = f"/tmp/sums_{os.path.basename(lib)}.npy"
    r = subprocess.run([sys.executable, "-c", CODE, out], env=env, capture_output=True, text=True)
    print(lib, r.stdout.strip(), r.stderr[-500:])
a = np.load("/tmp/sums_default.npy")
for lib in sys.argv[1:]:
    if lib == "default":
        continue
    b = np.load(f"/tmp/sums_{os.path.basename(lib)}.npy")
    d = (a != b).any(axis=1)
    print(lib, "vs default: differing poses", int(d.sum()), "first", np.nonzero(d)[0][:10])
    if d.any():
        i = np.nonzero(d)[0][0]
        print("  default", a[i], "\n  other  ", b[i])
