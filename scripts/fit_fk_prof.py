"""Per-phase clock64 stamps of the FK team of one k_eval CTA in the last generation of a C3
fit (build with -DHP_FK_PROF=1 into HP_LIB)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2005_07068_b200 as hp  # noqa: E402
import workloads as W  # noqa: E402

ctx = hp.Context(640, 480, max_particles=4096)
d, m = ctx.render_observation(W.H_A)
ctx.set_observation(d, m)
c, r = W.local_init_box()
for s in range(3):
    ctx.pso_fit(seed=s, particles=64, generations=40, init_center=c, init_radius=r)
torch.cuda.synchronize()
out = (C.c_ulonglong * 16)()
hp.hp.lib().hp_debug_fk_prof(out)
t = [out[i] for i in range(5)]
t_all = [out[i] for i in range(16)]
names = ["pose+sincos", "chains (B)", "records (C)", "union box, kc"]
for i in range(4):
    print(f"{names[i]:12s} {(t[i + 1] - t[i]) / 1965:.2f} us")
for i, n in ((5, "finish: loads"), (6, "finish: shfl")):
    print(f"{n:14s} {(t_all[i] - t_all[3]) / 1965:.2f} us")
print(f"total        {(t[4] - t[0]) / 1965:.2f} us")
