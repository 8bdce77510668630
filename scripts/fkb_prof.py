"""Phase timeline of k_fk_batch (one CTA, thread 0's clock64 stamps) on the C4 batch (build
with -DHP_FKB_PROF=1 into HP_LIB; timing mode, so FK runs alone)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_07068_b200 as hp  # noqa: E402
import workloads as W  # noqa: E402

ctx = hp.Context(640, 480, max_particles=4096)
d, m = ctx.render_observation(W.H_A)
ctx.set_observation(d, m)
P = torch.tensor(W.swarm_c4().astype(np.float32), device="cuda")
ctx.set_timing(True)
for _ in range(5):
    ctx.eval_costs(P)
torch.cuda.synchronize()
z = (C.c_ulonglong * 2048)()
ctx.eval_costs(P)
torch.cuda.synchronize()
hp.hp.lib().hp_debug_fkb_cta(z)
a = np.frombuffer(z, dtype=np.uint64).reshape(1024, 2).astype(np.float64)
t0 = a[:, 0].min()
st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
dur = en - st
print("CTA start: max %.2f us; end: p10 %.2f p50 %.2f p90 %.2f max %.2f us" % (
    st.max(), *np.percentile(en, [10, 50, 90, 100])))
print("CTA duration: p10 %.2f p50 %.2f p90 %.2f max %.2f us" % tuple(np.percentile(dur, [10, 50, 90, 100])))
print("slowest CTAs (index, start, end):", [(int(i), round(st[i], 2), round(en[i], 2)) for i in np.argsort(en)[-6:]])
out = (C.c_longlong * 16)()
hp.hp.lib().hp_debug_fkb_prof(out)
t = [out[i] for i in range(8)]
names = ["A pose+sincos", "B chains", "C records+boxes", "C' exact", "D finish", "D block list",
         "D publish"]
for i, n in enumerate(names):
    print(f"{n:16s} {(t[i + 1] - t[i]) / 1965:.2f} us")
print(f"{'total':16s} {(t[7] - t[0]) / 1965:.2f} us  (FK launch {ctx.last_kernel_ms()[0] * 1e3:.1f} us)")
