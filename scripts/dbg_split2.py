import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import oracle as O, paper_2005_07068_b200 as hp, workloads as W
ctx = hp.Context(640, 480, max_particles=4096)
obs = O.synthesize(W.H_A, O.camera(640, 480))
ctx.set_observation(obs.depth, obs.mask)
sw = W.swarm_c4().astype(np.float32)
P = torch.tensor(sw, device="cuda")
sb, _ = ctx.eval_sums(P)
print("launches", ctx.last_launch_count())
sb = sb.cpu().numpy()
for i in (0, 1, 777):
    s1, _ = ctx.eval_sums(P[i:i + 1].contiguous())
    print(i, "batch", sb[i], "split", s1.cpu().numpy()[0])
co, so, _, _ = O.eval_batch(sw[[0]].astype(np.float64), obs, with_sums=True)
print("oracle", so[0].s_rm, so[0].s_and, so[0].num, so[0].n_both)
