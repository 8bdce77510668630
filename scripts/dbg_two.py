import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, workloads as W, paper_2005_07068_b200 as hp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 600
ctx = hp.Context(640, 480, max_particles=4096)
d, m = ctx.render_observation(W.H_A); ctx.set_observation(d, m)
P = torch.tensor(W.swarm_c4(n).astype(np.float32), device="cuda")
s, c = ctx.eval_sums(P); torch.cuda.synchronize()
ref = [ctx.eval_sums(P[i:i+1])[0].cpu().numpy()[0] for i in range(0, n, max(1, n // 8))]
got = s.cpu().numpy()[::max(1, n // 8)]
for r, g in zip(ref, got): print(r, g)
import time
torch.cuda.synchronize(); t=time.perf_counter(); ctx.eval_costs(P); torch.cuda.synchronize(); print('ms', 1e3*(time.perf_counter()-t))
