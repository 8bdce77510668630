"""Per-phase clock64 stamps of one FK warp (build with -DHP_FK_PROF=1 into HP_LIB)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2005_07068_b200 as hp  # noqa: E402
import workloads as W  # noqa: E402

ctx = hp.Context(640, 480, max_particles=4096)
d, m = ctx.render_observation(W.H_A)
ctx.set_observation(d, m)
P = torch.tensor(W.swarm_c4().astype(np.float32), device="cuda")
for _ in range(5):
    ctx.eval_costs(P)
torch.cuda.synchronize()
out = (C.c_ulonglong * 16)()
hp.hp.lib().hp_debug_fk_prof(out)
t = [out[i] for i in range(7)]
names = ["pose+sincos", "chains (B)", "records (C)", "ubox/kc", "fence+s2g", "tile list", "ntl+wait"]
for i in range(6):
    print(f"{names[i]:12s} {(t[i + 1] - t[i]) / 1965:.2f} us")
print(f"total        {(t[6] - t[0]) / 1965:.2f} us")
