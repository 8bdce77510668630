"""Per-particle work spread of the C4 swarm: sum over primitives of the screen-box area
(pixel x primitive tests before culling) and the union-box area, from k_fk_batch's boxes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_07068_b200 as hp  # noqa: E402
import workloads as W  # noqa: E402

n = 4096
ctx = hp.Context(640, 480, max_particles=n)
d, m = ctx.render_observation(W.H_A)
ctx.set_observation(d, m)
poses = torch.from_numpy(W.swarm_c4(n)).float().cuda()
ctx.eval_costs(poses)
torch.cuda.synchronize()
work = np.zeros(n)
ub = np.zeros(n)
for p in range(n):
    _, b = ctx.debug_batch_fk(p)
    ok = b[:, 0] <= b[:, 2]
    w = (b[:, 2] - b[:, 0] + 1) * (b[:, 3] - b[:, 1] + 1)
    work[p] = (w * ok).sum()
    if ok.any():
        ub[p] = (b[ok, 2].max() - b[ok, 0].min() + 1) * (b[ok, 3].max() - b[ok, 1].min() + 1)
q = [0, 1, 10, 50, 90, 99, 100]
print("sum of box areas (px):", [int(np.percentile(work, x)) for x in q])
print("union box area (px):  ", [int(np.percentile(ub, x)) for x in q])
print("mean %.0f; heaviest / mean %.2f; top-1%% share of work %.3f" % (
    work.mean(), work.max() / work.mean(), np.sort(work)[-n // 100:].sum() / work.sum()))
# the work of the last 1776 (3 x grid) claimed particles vs the rest
print("mean work of the last 1776 particles / all: %.3f" % (work[-1776:].mean() / work.mean()))
