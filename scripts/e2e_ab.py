"""End-to-end call time (hp_eval_costs_host, C4, pinned host buffers, L2 flushed between
calls as in bench.py's e2e leg): median host wall clock per call, in us.
    python scripts/e2e_ab.py   (HP_LIB / HP_NO_ZEROCOPY select the build / mode)"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2005_07068_b200 as hp  # noqa: E402
import workloads as W  # noqa: E402

ctx = hp.Context(640, 480, max_particles=4096)
d, m = ctx.render_observation(W.H_A)
ctx.set_observation(d, m)
pin_in = torch.from_numpy(W.swarm_c4().astype(np.float32)).pin_memory()
pin_out = torch.empty(4096, dtype=torch.float32).pin_memory()
hin, hout = pin_in.numpy(), pin_out.numpy()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for _ in range(30):
    ctx.eval_costs_host(hin, out=hout)
ts = []
for _ in range(300):
    flush.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.eval_costs_host(hin, out=hout)
    ts.append(time.perf_counter() - t0)
ts = np.array(ts) * 1e6
print(f"{os.environ.get('HP_LIB', 'default')} zc={os.environ.get('HP_NO_ZEROCOPY', '0') == '0'}: "
      f"median {np.median(ts):.1f} us  p10 {np.percentile(ts, 10):.1f}  mean {ts.mean():.1f}")
