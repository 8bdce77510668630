"""Per-generation timeline of the fused PSO kernel (build with -DHP_GEN_PROF=1 into HP_LIB):
start (first CTA) -> FK done (last CTA) -> tiles done -> bookkeeping start/end, in us."""
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
ctx.pso_fit(seed=0, particles=64, generations=40, init_center=c, init_radius=r)
L = hp.hp.lib()
out = (C.c_ulonglong * (64 * 8))()
L.hp_debug_gen_prof(out, 1)
ctx.pso_fit(seed=1, particles=64, generations=40, init_center=c, init_radius=r)
torch.cuda.synchronize()
L.hp_debug_gen_prof(out, 0)
t = np.array(out[:], dtype=np.float64).reshape(64, 8)
prev_end = None
for k in range(1, 40):
    s0, fk, tiles, b0, b1 = t[k][:5]
    gap = (s0 - prev_end) / 1e3 if prev_end else float("nan")
    print(f"gen {k:2d}: gap {gap:5.2f}  update+fk {(fk - s0) / 1e3:5.2f}  tiles "
          f"{(tiles - fk) / 1e3:5.2f}  ->last CTA {(b0 - tiles) / 1e3:5.2f}  finalize+book "
          f"{(b1 - b0) / 1e3:5.2f}  total {(b1 - s0) / 1e3:6.2f} us")
    prev_end = b1
