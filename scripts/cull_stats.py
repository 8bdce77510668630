"""Tile-culling statistics for the C4 swarm (analysis tool, uses the oracle's FK / boxes /
single-primitive renders): per hypothesis, the (16x8 tile, primitive) pairs that the
renderer tests with box culling, with projected-circle / capsule culling, and the pairs
an exact per-tile cull would keep, weighted by the DESIGN §5 per-kind FLOP counts.

    python scripts/cull_stats.py [n_poses]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import workloads as W  # noqa: E402

TW, TH = int(os.environ.get("TW", "16")), int(os.environ.get("TH", "8"))
FLOPS = {0: 20, 1: 48, 2: 56, 3: 56}


def proj(c, cam):
    return np.array([cam.fx * c[0] / c[2] + cam.cx, cam.fy * c[1] / c[2] + cam.cy])


def rad(c, r, cam):
    # |p - c| <= r  =>  |proj(p) - proj(c)| <= f r |c| / (cz (cz - r))
    return max(cam.fx, cam.fy) * r * np.linalg.norm(c) / (c[2] * (c[2] - r))


def seg_rect_dist(p0, p1, ctr, hx, hy):
    """Distance between segment p0-p1 and the rectangle |x - ctr| <= (hx, hy)."""
    lo, hi = ctr - [hx, hy], ctr + [hx, hy]
    # segment / rectangle intersection (Liang-Barsky)
    d = p1 - p0
    t0, t1 = 0.0, 1.0
    inter = True
    for ax in range(2):
        if abs(d[ax]) < 1e-12:
            if p0[ax] < lo[ax] or p0[ax] > hi[ax]:
                inter = False
        else:
            a, b = (lo[ax] - p0[ax]) / d[ax], (hi[ax] - p0[ax]) / d[ax]
            t0, t1 = max(t0, min(a, b)), min(t1, max(a, b))
    if inter and t0 <= t1:
        return 0.0

    def pt_rect(p):
        q = np.maximum(np.abs(p - ctr) - [hx, hy], 0)
        return np.sqrt(q @ q)

    def pt_seg(q):
        L2 = d @ d
        t = 0.0 if L2 == 0 else min(max((q - p0) @ d / L2, 0.0), 1.0)
        r = p0 + t * d - q
        return np.sqrt(r @ r)

    corners = [np.array([x, y]) for x in (lo[0], hi[0]) for y in (lo[1], hi[1])]
    return min([pt_rect(p0), pt_rect(p1)] + [pt_seg(c) for c in corners])


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    cam = O.camera(640, 480)
    poses = np.asarray(np.asarray(W.swarm_c4(4096), np.float32), np.float64)[:: 4096 // n][:n]
    tot = {"box": 0.0, "cap": 0.0, "exact": 0.0}
    cnt = {"box": 0, "cap": 0, "exact": 0}
    ntiles = {"box": 0, "cap": 0, "exact": 0}
    culled = {}
    for h in poses:
        tiles = {"box": set(), "cap": set(), "exact": set()}
        prims, _ = O.fk(h)
        boxes = [O.prim_box(p, cam, int(os.environ.get("MARGIN", "1"))) for p in prims]
        ub = [b for b in boxes if b]
        x0 = min(b[0] for b in ub) & ~3
        y0 = min(b[1] for b in ub)
        x1 = max(b[2] for b in ub)
        y1 = max(b[3] for b in ub)
        tx = (x1 - x0 + TW) // TW
        ty = (y1 - y0 + TH) // TH
        for p, b in zip(prims, boxes):
            if not b:
                continue
            img = O.render_prims([p], cam, culled=False)
            hit = img > 0
            c = np.array(p.c)
            if p.kind == 0:
                circ = (proj(c, cam), None, rad(c, p.s[0], cam) + 0.02)
            elif p.kind == 2:
                a = np.array([p.R[i][1] for i in range(3)])
                c1 = c + p.s[2] * a
                circ = (proj(c, cam), proj(c1, cam),
                        max(rad(c, p.s[0], cam), rad(c1, p.s[1], cam)) + 0.02)
            else:
                circ = None
            for qy in range(ty):  # noqa: B007
                for qx in range(tx):
                    X0, Y0 = x0 + qx * TW, y0 + qy * TH
                    if b[0] > X0 + TW - 1 or b[2] < X0 or b[1] > Y0 + TH - 1 or b[3] < Y0:
                        continue
                    w = FLOPS[p.kind]
                    tot["box"] += w
                    cnt["box"] += 1
                    if hit[Y0:Y0 + TH, X0:X0 + TW].any():
                        tot["exact"] += w
                        cnt["exact"] += 1
                    keep = True
                    if circ is not None:
                        ctr = np.array([X0 + TW / 2, Y0 + TH / 2])
                        hx, hy = TW / 2 - 0.5, TH / 2 - 0.5
                        p0, p1, R = circ
                        if p1 is None:
                            d = np.maximum(np.abs(ctr - p0) - [hx, hy], 0)
                            keep = d @ d <= R * R
                        else:
                            e = p1 - p0
                            L = np.linalg.norm(e)
                            keep = seg_rect_dist(p0, p1, ctr, hx, hy) <= R
                    if not keep:
                        culled[p.kind] = culled.get(p.kind, 0) + w
                    if keep:
                        tot["cap"] += w
                        cnt["cap"] += 1
                        tiles["cap"].add((X0, Y0))
                    tiles["box"].add((X0, Y0))
                    if hit[Y0:Y0 + TH, X0:X0 + TW].any():
                        tiles["exact"].add((X0, Y0))
        for k in tiles:
            ntiles[k] += len(tiles[k])
    print("culled weight by kind:", {k: round(v / tot["box"], 4) for k, v in culled.items()})
    for k in tot:
        print(f"{k:6s} pairs/hyp {cnt[k] / n:8.1f}  weighted {tot[k] / tot['box']:.3f}"
              f"  non-empty tiles/hyp {ntiles[k] / n:6.1f}")


if __name__ == "__main__":
    main()
