"""Renderer tail: per-warp loop-exit times of k_render_persist on the C4 step (build with
-DHP_TAIL_PROF=1 into HP_LIB).  Reports the warp-time the grid leaves idle after each warp's
last block, as a fraction of warps x kernel span."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_07068_b200 as hp  # noqa: E402
import workloads as W  # noqa: E402

n = 4096
ctx = hp.Context(640, 480, max_particles=n)
d, m = ctx.render_observation(W.H_A)
ctx.set_observation(d, m)
poses = torch.from_numpy(W.swarm_c4(n)).float().cuda()
for _ in range(5):
    ctx.eval_costs(poses)
torch.cuda.synchronize()
out = (C.c_ulonglong * (1024 * 17))()
hp.hp.lib().hp_debug_tail_prof(out)
a = np.frombuffer(out, dtype=np.uint64).reshape(1024, 17).astype(np.float64)
g = int(os.environ.get("HP_PERSIST_GRID", "592"))
a = a[:g]
t0 = a[:, 0].min()
st = a[:, 0] - t0
ex = a[:, 1:9] - t0
end = ex.max()
print(f"grid {g}: span {end / 1e3:.2f} us, CTA start spread {st.max() / 1e3:.2f} us")
print(f"warp exit: min {ex.min() / 1e3:.2f} median {np.median(ex) / 1e3:.2f} max {end / 1e3:.2f} us")
idle = (end - ex).sum() + (st[:, None] * np.ones((1, 8))).sum()
print(f"idle warp-time fraction (late start + early exit): {idle / (ex.size * end):.4f}")
cta_end = ex.max(axis=1)
print(f"CTA end: p10 {np.percentile(cta_end, 10) / 1e3:.2f} p50 {np.median(cta_end) / 1e3:.2f} us")
r = np.frombuffer(out, dtype=np.uint64).reshape(1024, 17)[:g]
order = np.argsort(cta_end)
print("latest CTAs: end_us sm particles blocks last_p last_nlist last_particle_us")
for i in order[-12:]:
    print(f"  {cta_end[i] / 1e3:7.2f} {int(r[i, 9]):4d} {int(r[i, 10]):3d} {int(r[i, 11]):6d} "
          f"{int(r[i, 14]):5d} {int(np.int32(np.uint32(r[i, 15] & 0xffffffff))):5d} "
          f"{(float(r[i, 13]) - float(r[i, 12])) / 1e3:7.2f}")
print("CTA end percentiles (us):", [round(float(np.percentile(cta_end, q)) / 1e3, 2) for q in (1, 10, 50, 90, 99, 100)])
print("particles per CTA: min %d max %d; blocks per CTA: min %d median %d max %d" % (
    r[:, 10].min(), r[:, 10].max(), r[:, 11].min(), np.median(r[:, 11]), r[:, 11].max()))
term = (r[:, 16].astype(np.float64) - t0)
print("first terminator claim (us): min %.2f median %.2f max %.2f" % (term.min() / 1e3, np.median(term) / 1e3, term.max() / 1e3))
rem = cta_end - term
print("CTA end - its first terminator (us): p10 %.2f p50 %.2f p90 %.2f max %.2f" % tuple(np.percentile(rem, q) / 1e3 for q in (10, 50, 90, 100)))
