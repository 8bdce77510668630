"""Split path (k_eval) sums and depth for a few poses, saved for comparison across builds."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2005_07068_b200 as hp  # noqa: E402
import workloads as W  # noqa: E402

ctx = hp.Context(640, 480, max_particles=4096)
obs = O.synthesize(W.H_A, O.camera(640, 480))
ctx.set_observation(obs.depth, obs.mask)
sw = W.swarm_c4().astype(np.float32)
res = []
for i in (0, 1, 777):
    s, c = ctx.eval_sums(torch.tensor(sw[i:i + 1], device="cuda"))
    d = ctx.debug_render(torch.tensor(sw[i], device="cuda"))
    res.append((s.cpu().numpy()[0], d.cpu().numpy()))
    print(i, "S", ctx.splits_for(1), "sums", s.cpu().numpy()[0], "hits", int((d > 0).sum().item()))
np.save(sys.argv[1], np.stack([r[1] for r in res]))
