"""Debug: GPU vs oracle depth for close-up poses (pixel-level mismatch report)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2005_07068_b200 as hp  # noqa: E402
import workloads as W  # noqa: E402

cam = O.camera(640, 480)
ctx = hp.Context(640, 480, max_particles=64)
for z in (250.0, 300.0, 350.0, 420.0):
    for dx in (-30.0, 0.0, 30.0):
        h = W.H_A.copy()
        h[0] += dx
        h[2] = z
        h32 = h.astype(np.float32)
        d = ctx.debug_render(torch.tensor(h32, device="cuda")).cpu().numpy()
        do = O.render(h32.astype(np.float64), cam)
        e = O.edge_mask(h32.astype(np.float64), cam)
        hg, ho = d > 0, do > 0
        bad = (hg != ho) & (e == 0)
        both = hg & ho
        dd = np.abs(d - do)[both]
        print(f"z={z} dx={dx}: hits gpu {hg.sum()} or {ho.sum()} sil-mismatch {int((hg != ho).sum())} "
              f"non-edge {int(bad.sum())} max|dd| {dd.max() if dd.size else 0:.2e}")
        if bad.sum():
            ys, xs = np.nonzero(bad)
            for y, x in list(zip(ys, xs))[:5]:
                print("   px", x, y, "gpu", d[y, x], "oracle", do[y, x])
