"""Small end-to-end run for compute-sanitizer: batch path (k_fk_batch + k_render_persist),
split path (k_eval), depth hook, fused PSO fit, sharded world-1."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2005_07068_b200 as hp  # noqa: E402
import workloads as W  # noqa: E402

ctx = hp.Context(160, 120, max_particles=1024)
d, m = ctx.render_observation(W.H_A)
ctx.set_observation(d, m)
P = torch.tensor(W.swarm_c4(1024).astype(np.float32), device="cuda")
c1 = ctx.eval_costs(P)                 # batch path (S = 1)
c2 = ctx.eval_costs(P[:8])             # split path
dep = ctx.debug_render(P[0])
c, r = W.local_init_box()
fit = ctx.pso_fit(seed=1, particles=16, generations=5, init_center=c, init_radius=r)
torch.cuda.synchronize()
assert torch.equal(c1[:8], c2)
print("ok", float(c1.sum()), fit.best_cost)
