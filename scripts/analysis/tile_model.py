"""Design-space count for the renderer's tiling (analysis tool; oracle FK and boxes on the
C4 swarm): per hypothesis, (tile, primitive) pairs by kind for candidate warp-tile shapes,
box pixels by kind, union-box pixels and non-empty tiles.

    python scripts/analysis/tile_model.py [n_poses]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402

KIND = {0: "sph", 1: "ell", 2: "cone", 3: "cyl"}
SHAPES = [(16, 8), (16, 4), (8, 8), (8, 4), (32, 4), (16, 16), (32, 8)]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    cam = O.camera(640, 480)
    poses = np.asarray(np.asarray(W.swarm_c4(4096), np.float32), np.float64)[:: 4096 // n][:n]
    pairs = {s: {k: 0 for k in KIND.values()} for s in SHAPES}
    tiles = {s: 0 for s in SHAPES}
    boxpx = {k: 0 for k in KIND.values()}
    union = 0
    for h in poses:
        prims, _ = O.fk(h)
        bs = [(O.prim_box(p, cam, 0), KIND[p.kind]) for p in prims]
        bs = [(b, k) for b, k in bs if b]
        x0 = min(b[0] for b, _ in bs) & ~3
        y0 = min(b[1] for b, _ in bs)
        x1 = max(b[2] for b, _ in bs)
        y1 = max(b[3] for b, _ in bs)
        union += (x1 - x0 + 1) * (y1 - y0 + 1)
        for b, k in bs:
            boxpx[k] += (b[2] - b[0] + 1) * (b[3] - b[1] + 1)
        for (tw, th) in SHAPES:
            occ = set()
            for b, k in bs:
                qx0, qx1 = (b[0] - x0) // tw, (b[2] - x0) // tw
                qy0, qy1 = (b[1] - y0) // th, (b[3] - y0) // th
                pairs[(tw, th)][k] += (qx1 - qx0 + 1) * (qy1 - qy0 + 1)
                for qy in range(qy0, qy1 + 1):
                    for qx in range(qx0, qx1 + 1):
                        occ.add((qx, qy))
            tiles[(tw, th)] += len(occ)
    print(f"per hypothesis over {n} C4 poses: union-box px {union / n:.0f}, box px by kind",
          {k: round(v / n) for k, v in boxpx.items()}, "total", round(sum(boxpx.values()) / n))
    for s in SHAPES:
        px = s[0] * s[1]
        tot = sum(pairs[s].values())
        print(f"tile {s[0]:2d}x{s[1]:<2d}: tiles {tiles[s] / n:6.1f}  pairs {tot / n:6.1f}  px-tests "
              f"{tot * px / n:7.0f}  by kind", {k: round(v * px / n) for k, v in pairs[s].items()})


if __name__ == "__main__":
    main()
