"""Time hp_pso_fit on C1/C2/C3 (median over seeds): python scripts/fit_time.py"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2005_07068_b200 as hp  # noqa: E402
import workloads as W  # noqa: E402

for name, (w, h), N, K in (("C1", (160, 120), 16, 10), ("C2", (320, 240), 64, 40),
                           ("C3", (640, 480), 64, 40)):
    ctx = hp.Context(w, h, max_particles=max(N, 64))
    d, m = ctx.render_observation(W.H_A)
    ctx.set_observation(d, m)
    c, r = W.local_init_box()
    ctx.pso_fit(seed=0, particles=N, generations=K, init_center=c, init_radius=r)
    ms = []
    for s in range(1, 11):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = ctx.pso_fit(seed=s, particles=N, generations=K, init_center=c, init_radius=r)
        ms.append(1e3 * (time.perf_counter() - t0))
    print(f"{name} {w}x{h} {N}x{K}: median {statistics.median(ms):.3f} ms/frame, "
          f"min {min(ms):.3f}, launches {ctx.last_launch_count()}, best E {res.best_cost:.4f}")
    ctx.close()
