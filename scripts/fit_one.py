import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2005_07068_b200 as hp, workloads as W
ctx = hp.Context(640, 480, max_particles=64)
d, m = ctx.render_observation(W.H_A); ctx.set_observation(d, m)
c, r = W.local_init_box()
for s in range(2): ctx.pso_fit(seed=s, particles=64, generations=40, init_center=c, init_radius=r)
rec, boxes, J, kc = ctx.debug_fk(W.H_A)
torch.cuda.synchronize()
