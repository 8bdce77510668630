import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, oracle as O, workloads as W, paper_2005_07068_b200 as hp
ctx = hp.Context(160, 120, max_particles=64)
obs = O.synthesize(W.H_A, O.camera(160, 120))
ctx.set_observation(obs.depth, obs.mask)
P = torch.tensor(W.random_poses(1, 8).astype(np.float32), device="cuda")
c = ctx.eval_costs(P); torch.cuda.synchronize(); print(os.environ.get("HP_NO_TMA"), c.cpu().numpy())
print(O.eval_batch(W.random_poses(1, 8).astype(np.float32).astype(np.float64), obs))
