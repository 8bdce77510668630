"""Per-CTA timeline of the persistent fit kernel k_fit (build with -DHP_GEN_PROF=1 into
HP_LIB): clock64 stamps of CTA 0 and the last CTA per generation, in us at 1965 MHz."""
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
c, r = W.local_init_box()
for s in range(3):
    ctx.pso_fit(seed=s, particles=64, generations=40, init_center=c, init_radius=r)
torch.cuda.synchronize()
out = (C.c_longlong * (64 * 2 * 8))()
hp.hp.lib().hp_debug_fit_clk(out)
t = np.array(out[:], dtype=np.float64).reshape(64, 2, 8) / 1965.0
# stamps: 0 start, 5 update done, 1 FK done, 2 tiles done, 3 barrier passed, 6 sums read,
# 7 argmin/marks done, 4 bookkeeping done
names = ["update", "fk", "tiles", "barrier", "loads+fin", "argmin", "tail"]
order = [0, 5, 1, 2, 3, 6, 7, 4]
for cta in (0, 1):
    print("CTA", "0" if cta == 0 else "last")
    for k in (10, 20, 30, 38):
        row = t[k][cta]
        parts = [row[order[i + 1]] - row[order[i]] for i in range(len(order) - 1)]
        nxt = t[k + 1][cta][0] - row[4]
        print(f"  gen {k}: " + "  ".join(f"{n} {v:5.2f}" for n, v in zip(names, parts)) +
              f"  ->next {nxt:5.2f}  total {t[k + 1][cta][0] - row[0]:6.2f} us")
