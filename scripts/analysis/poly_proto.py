"""Prototype (analysis tool, numpy) of the renderer's polynomial ray-quadric formulation for
ellipsoids / cones / the palm cylinder, checked against the oracle's renders before it is
written in CUDA.  Spheres are rendered exactly (their formula is unchanged).

For a primitive with local coordinates l = M (p - c) and implicit F(l) = l'Ql + 2 g.l + h,
the ray p = t d, d = (x, y, 1) gives a t^2 - 2 b t + c0 = 0 with a = dl'Q dl, b = dl'Q cl -
g.dl, c0 = cl'Q cl - 2 g.cl + h (dl = M d, cl = M c); the entering root t = (b - sqrt(D))/a,
D = b^2 - a c0.  a and D are quadratic, b affine in (x, y); all three are expanded (fp64)
about the projected centre (xp, yp) and evaluated in fp32 by Horner in (x - xp, y - yp).

    python scripts/analysis/poly_proto.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402

f32 = np.float32


def fma(a, b, c):
    return f32(np.float64(a) * np.float64(b) + np.float64(c))


def record(p):
    """Fast record (fp64 math, fp32 storage) of an oracle primitive (not a sphere)."""
    c = np.array(p.c, float)
    R = np.array([[p.R[i][j] for j in range(3)] for i in range(3)])
    s = np.array(p.s, float)
    if p.kind == O.ELLIPSOID:
        M = (R / s[None, :]).T              # rows: local axes / semi-axes
        Q, g, h, cen = np.ones(3), np.zeros(3), -1.0, c
        ax = None
    elif p.kind == O.CONE:
        a = R[:, 1]  # the oracle stores only the axis column for cones: complete a frame
        e1 = np.cross(a, [1.0, 0, 0] if abs(a[0]) < 0.9 else [0, 1.0, 0])
        e1 /= np.linalg.norm(e1)
        e2 = np.cross(a, e1)
        r0, r1, L = s
        k = (r1 - r0) / L
        cen = c + 0.5 * L * a               # local origin: axis midpoint
        M = np.stack([e1, e2, a])
        rm = 0.5 * (r0 + r1)
        Q, g, h = np.array([1.0, 1.0, -k * k]), np.array([0, 0, -rm * k]), -rm * rm
        ax, hl = a, 0.5 * L
    else:  # cylinder: local (x/a, z/b), axial y in [-len, 0]
        a_, ln, b_ = s
        cx, cy, cz = R[:, 0], R[:, 1], R[:, 2]
        cen = c - 0.5 * ln * cy
        M = np.stack([cx / a_, cz / b_, cy])
        Q, g, h = np.array([1.0, 1.0, 0.0]), np.zeros(3), -1.0
        ax, hl = cy, 0.5 * ln
    cl = M @ cen
    xp, yp = f32(cen[0] / cen[2]), f32(cen[1] / cen[2])
    dp = np.array([float(xp), float(yp), 1.0])
    m0, m1 = M[:, 0], M[:, 1]
    dlp = M @ dp
    qx = lambda u, v: float(np.sum(Q * u * v))  # noqa: E731
    A = [qx(dlp, dlp), 2 * qx(m0, dlp), 2 * qx(m1, dlp), qx(m0, m0), 2 * qx(m0, m1), qx(m1, m1)]
    b0 = qx(dlp, cl) - g @ dlp
    bx = qx(m0, cl) - g @ m0
    by = qx(m1, cl) - g @ m1
    c0 = qx(cl, cl) - 2 * g @ cl + h
    D = [b0 * b0 - c0 * A[0], 2 * b0 * bx - c0 * A[1], 2 * b0 * by - c0 * A[2],
         bx * bx - c0 * A[3], 2 * bx * by - c0 * A[4], by * by - c0 * A[5]]
    rec = dict(xp=xp, yp=yp, D=[f32(v) for v in D], A=[f32(v) for v in A],
               B=[f32(b0), f32(bx), f32(by)], kind=p.kind)
    if ax is not None:
        rec.update(lz=[f32(M[2, 0]), f32(M[2, 1]), f32(M[2, 2])], clz=f32(cl[2]), hl=f32(hl))
    return rec


def poly_depth(rec, X, Y):
    """fp32 evaluation: X, Y ray slopes (fp32 arrays).  NaN = no hit."""
    xq = (X - rec["xp"]).astype(f32)
    yq = (Y - rec["yp"]).astype(f32)
    d, a, b = rec["D"], rec["A"], rec["B"]
    ed0 = fma(fma(d[3], xq, d[1]), xq, d[0])
    ed1 = fma(d[4], xq, d[2])
    ea0 = fma(fma(a[3], xq, a[1]), xq, a[0])
    ea1 = fma(a[4], xq, a[2])
    eb0 = fma(b[1], xq, b[0])
    Dv = fma(fma(d[5], yq, ed1), yq, ed0)
    Av = fma(fma(a[5], yq, ea1), yq, ea0)
    Bv = fma(b[2], yq, eb0)
    with np.errstate(invalid="ignore", divide="ignore"):
        t = ((Bv - np.sqrt(Dv).astype(f32)).astype(f32) * (f32(1) / Av).astype(f32)).astype(f32)
        if "lz" in rec:
            lz = fma(rec["lz"][1], Y, fma(rec["lz"][0], X, rec["lz"][2]))
            za = fma(t, lz, -rec["clz"])
            t = np.where(np.abs(za) <= rec["hl"], t, np.nan).astype(f32)
    return t


def render_fast(h, cam):
    prims, _ = O.fk(h)
    W_, H_ = cam.width, cam.height
    u = np.arange(W_, dtype=np.float64)
    v = np.arange(H_, dtype=np.float64)
    X = f32((u + 0.5 - cam.cx) / cam.fx)[None, :].repeat(H_, 0)
    Y = f32((v + 0.5 - cam.cy) / cam.fy)[:, None].repeat(W_, 1)
    z = np.full((H_, W_), np.inf)
    sph = [p for p in prims if p.kind == O.SPHERE]
    zs = O.render_prims(sph, cam).astype(np.float64)
    z = np.where(zs > 0, zs, z)
    for p in prims:
        if p.kind == O.SPHERE:
            continue
        t = poly_depth(record(p), X, Y).astype(np.float64)
        ok = np.isfinite(t) & (t >= cam.z_near) & (t <= cam.z_far)
        z = np.where(ok & (t < z), t, z)
    return np.where(np.isfinite(z), z, 0.0).astype(f32)


def main():
    for res in ("160x120", "640x480"):
        cam = O.camera(*W.RESOLUTIONS[res])
        worst, nbad, ntot = 0.0, 0, 0
        for h in list(W.NAMED.values()) + list(W.random_poses(7, 6)) + list(W.swarm_c4(8)):
            o = O.render(h, cam)
            g = render_fast(h, cam)
            edge = O.edge_mask(h, cam)
            sil = (g > 0) != (o > 0)
            nbad += int((sil & (edge == 0)).sum())
            ntot += int(((g > 0) | (o > 0)).sum())
            both = (g > 0) & (o > 0) & (edge == 0)
            if both.any():
                worst = max(worst, float(np.max(np.abs(g[both].astype(float) - o[both]))))
        print(f"{res}: max depth error {worst:.2e} mm, non-edge silhouette flips {nbad} of {ntot} px")


if __name__ == "__main__":
    main()
