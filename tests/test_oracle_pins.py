"""Pins for the CPU oracle (-m "not gpu").

Each test fixes part of the oracle against something other than itself: published
known-answer vectors, closed forms, worked examples, invariants, or an independent brute
force (ray marching) — chosen so that a dropped term, wrong sign/index or transposed
operand in oracle.c fails at least one of them.
"""
import math
import os

import numpy as np
import pytest

import oracle as O
import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


# ---------------------------------------------------------------- RNG
def test_philox_known_answers():
    for r in _rows("philox4x32_10_kat.txt"):
        v = [int(x, 16) for x in r]
        assert O.philox(v[:4], v[4:6]) == v[6:10]


def test_u01_range_and_resolution():
    assert O.u01(0, 0) == 0.0
    top = O.u01(0xFFFFFFFF, 0xFFFFFFFF)
    assert top < 1.0 and top == 1.0 - 2.0 ** -53
    assert O.u01(0, 1 << 6) == 2.0 ** -53


# ---------------------------------------------------------------- FK
FINGER = {"thumb": 0, "index": 1, "middle": 2, "ring": 3, "little": 4}


def test_fk_zero_pose_closed_form():
    h = np.zeros(26)
    h[2] = 800.0
    _, J = O.fk(h)
    for name, k, x, y, z in _rows("fk_zero_pose.txt"):
        np.testing.assert_allclose(J[FINGER[name], int(k)], [float(x), float(y), float(z)],
                                   atol=1e-7)


def test_fk_bounds_table_matches_paper():
    lo, hi = O.bounds()
    d = math.radians
    assert lo[:3].tolist() == [-900, -680, 500] and hi[:3].tolist() == [900, 680, 1500]
    assert lo[3] == d(-30) and hi[3] == d(120) and lo[4] == d(-70) and hi[4] == d(75)
    assert lo[5] == d(-35) and hi[5] == d(20)
    assert (lo[6], hi[6]) == (0.0, d(90))          # thumb MPx 0-90 (Table 1)
    assert (lo[7], hi[7]) == (d(-15), d(60))       # thumb MPz -15-60
    assert (lo[9], hi[9]) == (d(-15), d(70))       # thumb DIP -15-70
    assert (lo[6 + 4 * 4 + 1], hi[6 + 4 * 4 + 1]) == (d(-45), 0.0)  # little MPz -45-0


def _seg_dirs(J):
    return [J[k + 1] - J[k] for k in range(3)]


@pytest.mark.parametrize("seed", range(5))
def test_fk_segment_lengths_preserved(seed):
    dims = O.default_dims()
    for h in W.random_poses(seed, 20):
        _, J = O.fk(h)
        for f in range(5):
            for k, s in enumerate(_seg_dirs(J[f])):
                assert abs(np.linalg.norm(s) - dims.seg_len[f][k]) < 1e-9


def test_fk_translation_equivariance():
    h = W.NAMED["spread"].copy()
    prims0, J0 = O.fk(h)
    h2 = h.copy()
    h2[:3] += [13.0, -7.5, 101.0]
    prims1, J1 = O.fk(h2)
    np.testing.assert_allclose(J1 - J0, np.broadcast_to([13.0, -7.5, 101.0], J0.shape), atol=1e-9)
    for a, b in zip(prims0, prims1):
        np.testing.assert_allclose(np.array(b.c) - np.array(a.c), [13.0, -7.5, 101.0], atol=1e-9)


def test_fk_pip_90_perpendicular():
    h = np.zeros(26)
    h[2] = 900.0
    h[6 + 4 * 1 + 2] = math.pi / 2  # index PIP
    _, J = O.fk(h)
    s = _seg_dirs(J[1])
    u = [v / np.linalg.norm(v) for v in s]
    assert abs(np.dot(u[0], u[1])) < 1e-9
    assert abs(np.dot(u[1], u[2]) - 1.0) < 1e-9  # DIP = 0 keeps the last two aligned
    # positive flexion curls towards -z_H (the palm, which faces the camera)
    assert u[1][2] < -0.999


def test_fk_abduction_sign_towards_thumb():
    h = np.zeros(26)
    h[2] = 800.0
    h[6 + 4 * 1 + 1] = math.radians(10)  # index abduction +10 deg
    _, J = O.fk(h)
    d = J[1][1] - J[1][0]
    assert d[0] > 0  # towards +x_H (the thumb side)
    assert abs(math.degrees(math.atan2(d[0], -d[1])) - 10.0) < 1e-9


def test_fk_flat_hand_coplanar():
    h = np.zeros(26)
    h[2] = 1000.0
    _, J = O.fk(h)
    z = J[1:, :, 2]
    assert np.all(np.abs(z - 1000.0) < 1e-9)
    assert np.all(np.abs(J[0, :, 2] - 992.0) < 1e-9)


def test_fk_wrist_rotations_closed_form():
    """Non-zero wrist angles (AMB-10): at 90 degrees each rotation is a coordinate permutation
    written out by hand in the golden file; combined angles pin the order (x, then y, then
    z), the 30-degree cases the signs of Ry and Rx away from the permutations."""
    for case, ax, ay, az, name, k, x, y, z in _rows("fk_wrist_pins.txt"):
        h = np.zeros(26)
        h[2] = 800.0
        h[3:6] = [math.radians(float(ax)), math.radians(float(ay)), math.radians(float(az))]
        _, J = O.fk(h)
        np.testing.assert_allclose(J[FINGER[name], int(k)], [float(x), float(y), float(z)],
                                   atol=1e-7, err_msg=case)


def test_fk_thumb_and_finger_flexion_abduction_closed_form():
    """Thumb flexion sweeps it across the palm, thumb abduction lifts it palmarly, finger
    flexion curls towards the palm (hand derivations in the golden file)."""
    for case, dof, deg, name, k, x, y, z in _rows("fk_thumb_finger_pins.txt"):
        h = np.zeros(26)
        h[2] = 800.0
        h[int(dof)] = math.radians(float(deg))
        _, J = O.fk(h)
        np.testing.assert_allclose(J[FINGER[name], int(k)], [float(x), float(y), float(z)],
                                   atol=1e-7, err_msg=case)


def test_fk_primitive_structure():
    """38 primitives: 1 cylinder, 3 ellipsoids, 14 cones, 20 spheres."""
    h = W.random_poses(3, 1)[0]
    prims, J = O.fk(h)
    kinds = [p.kind for p in prims]
    assert len(prims) == 38
    assert kinds.count(O.SPHERE) == 20 and kinds.count(O.CONE) == 14
    assert kinds.count(O.ELLIPSOID) == 3 and kinds.count(O.CYLINDER) == 1
    dims = O.default_dims()
    for p in prims:
        if p.kind == O.CONE:  # axis is the unit segment direction, end radii = sphere radii
            a = np.array([p.R[0][1], p.R[1][1], p.R[2][1]])
            assert abs(np.linalg.norm(a) - 1) < 1e-12
    # thumb proximal ellipsoid: centred on the segment midpoint, long axis along it
    th = [p for p in prims if p.kind == O.ELLIPSOID and abs(p.s[1] - 22.5) < 1e-12]
    assert len(th) == 1
    mid = 0.5 * (J[0][0] + J[0][1])
    np.testing.assert_allclose(th[0].c, mid, atol=1e-9)
    ax = np.array([th[0].R[i][1] for i in range(3)])
    seg = (J[0][1] - J[0][0]) / dims.seg_len[0][0]
    assert abs(abs(np.dot(ax, seg)) - 1) < 1e-12


def test_kc_closed_forms():
    h = W.H_A.copy()
    assert O.kc(h) == 0.0
    h = np.zeros(26)
    assert O.kc(h) == 0.0
    # index swings 0.1 rad towards the middle finger: phi(index, middle) = -0.1
    h[6 + 4 * 1 + 1] = -0.1
    assert abs(O.kc(h) - 0.1) < 1e-15
    # additionally little swings away (negative) -> still only one violating pair
    h[6 + 4 * 4 + 1] = -0.3
    assert abs(O.kc(h) - 0.1) < 1e-15
    # ring towards little beyond it: phi(ring, little) = -0.5 - (-0.3) = -0.2
    h[6 + 4 * 3 + 1] = -0.5
    # now phi(middle, ring) = 0 - (-0.5) = 0.5 fine; pairs: 0.1 + 0.2
    assert abs(O.kc(h) - 0.3) < 1e-15
    assert abs(O.kc(np.zeros(26), rho=-0.25) - 0.75) < 1e-15  # rho shifts every pair


# ---------------------------------------------------------------- rendering
def _sphere(c, r):
    p = O.Prim()
    p.kind = O.SPHERE
    p.c[:] = c
    p.s[0] = r
    return p


def test_sphere_axis_depths():
    assert abs(O.first_hit(_sphere((0, 0, 1000), 50), (0, 0, 1)) - 950.0) < 1e-9
    cam = O.camera(640, 480)
    cam.cx, cam.cy = 320.5, 240.5  # pixel (320, 240)'s centre ray on the optical axis
    img = O.render_prims([_sphere((0, 0, 1000), 50), _sphere((0, 0, 900), 50)], cam)
    assert img[240, 320] == 850.0  # nearest surface wins
    img1 = O.render_prims([_sphere((0, 0, 1000), 50)], cam)
    assert img1[240, 320] == 950.0
    assert np.all(O.render_prims([], cam) == 0)


def test_sphere_disk_area_closed_form():
    cam = O.camera(640, 480)
    img = O.render_prims([_sphere((0, 0, 1000), 50)], cam)
    R = 525.0 * 50 / math.sqrt(1000 ** 2 - 50 ** 2)  # 26.283 px silhouette radius
    area = (img > 0).sum()
    assert abs(area - math.pi * R * R) < 2 * math.pi * R  # +- perimeter
    cam2 = O.camera(1280, 960)
    area2 = (O.render_prims([_sphere((0, 0, 1000), 50)], cam2) > 0).sum()
    assert abs(area2 / area - 4.0) < 0.2  # x2 intrinsics -> x4 area (+-5 %)


# --- independent brute force: ray marching against implicit inside-tests ---------------
def _inside(p, P):
    """Vectorised membership of points P (n,3) in primitive p (its definition in oracle.h)."""
    c = np.array(p.c)
    R = np.array([[p.R[i][j] for j in range(3)] for i in range(3)])
    q = (P - c) @ R  # local coordinates (columns of R are the local axes)
    s = np.array(p.s)
    if p.kind == O.SPHERE:
        return np.einsum("ij,ij->i", P - c, P - c) <= s[0] ** 2
    if p.kind == O.ELLIPSOID:
        return np.sum((q / s) ** 2, axis=1) <= 1.0
    if p.kind == O.CONE:
        a = R[:, 1]
        z = (P - c) @ a
        rad2 = np.einsum("ij,ij->i", P - c, P - c) - z * z
        rz = s[0] + (s[1] - s[0]) * z / s[2]
        return (z >= 0) & (z <= s[2]) & (rad2 <= rz * rz)
    if p.kind == O.CYLINDER:
        return ((q[:, 0] / s[0]) ** 2 + (q[:, 2] / s[2]) ** 2 <= 1.0) & (q[:, 1] <= 0) & (
            q[:, 1] >= -s[1])
    raise AssertionError


def _march(p, d, t_max=3000.0, step=0.02):
    t = np.arange(0.0, t_max, step)
    ins = _inside(p, t[:, None] * np.asarray(d)[None, :])
    if not ins.any():
        return math.inf
    k = int(np.argmax(ins))
    lo, hi = t[k] - step, t[k]
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if _inside(p, np.array([mid * np.asarray(d)]))[0]:
            hi = mid
        else:
            lo = mid
    return hi


def _rot(ax, ay, az):
    cx, sx, cy, sy, cz, sz = (math.cos(ax), math.sin(ax), math.cos(ay), math.sin(ay),
                              math.cos(az), math.sin(az))
    Rx = np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]])
    Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
    Rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]])
    return Rz @ Ry @ Rx


def _prim(kind, c, R, s):
    p = O.Prim()
    p.kind = kind
    p.c[:] = c
    for i in range(3):
        for j in range(3):
            p.R[i][j] = R[i][j]
    p.s[:] = s
    return p


def _cone(J0, J1, r0, r1):
    J0, J1 = np.array(J0, float), np.array(J1, float)
    L = np.linalg.norm(J1 - J0)
    R = np.zeros((3, 3))
    R[:, 1] = (J1 - J0) / L
    return _prim(O.CONE, J0, R, (r0, r1, L))


TINY_PRIMS = {
    "sphere": _sphere((3, -2, 400), 9),
    "ellipsoid": _prim(O.ELLIPSOID, (2, 1, 420), _rot(0.4, -0.7, 1.1), (12, 22.5, 10)),
    "cone_oblique": _cone((-10, 8, 410), (12, -10, 440), 9, 6),
    # axis pointing at the camera: exercises the far-nappe root of the double cone
    "cone_towards_camera": _cone((0.5, -0.3, 460), (0.2, 0.1, 420), 10, 5),
    "cylinder_oblique": _prim(O.CYLINDER, (0, 12, 430), _rot(0.3, 0.5, -0.2), (14, 24, 6)),
    "cylinder_end_on": _prim(O.CYLINDER, (1, -1, 450), _rot(math.pi / 2, 0, 0), (12, 30, 7)),
}


@pytest.mark.parametrize("name", sorted(TINY_PRIMS))
def test_first_hit_matches_ray_marching(name):
    """Brute force on a tiny 8x6 image: every pixel's first hit vs independent ray marching
    against the solid's implicit inequality (north star 'brute-force pixel checks
    on tiny images')."""
    p = TINY_PRIMS[name]
    cam = O.camera(8, 6)
    cam.fx = cam.fy = 180.0  # ~ 0.35 rad field of view: the primitive fills the image
    hits = 0
    for v in range(cam.height):
        for u in range(cam.width):
            d = np.array([(u + 0.5 - cam.cx) / cam.fx, (v + 0.5 - cam.cy) / cam.fy, 1.0])
            t_or = O.first_hit(p, d)
            t_bf = _march(p, d)
            if math.isinf(t_bf):
                assert math.isinf(t_or), (u, v, t_or)
            else:
                hits += 1
                assert abs(t_or - t_bf) < 1e-6, (u, v, t_or, t_bf)
    assert hits > 0


def test_edge_mask_on_axis_sphere_analytic():
    """or_edge_mask's three rules on a sphere on the optical axis, whose silhouette, depth
    and r_m boundaries have closed forms: ray d = (x, y, 1) hits the sphere |p - c| = r,
    c = (0, 0, Z), iff Z^2 - |d|^2 (Z^2 - r^2) >= 0, at depth t = (Z - sqrt(.)) / |d|^2.
    A pixel is an edge pixel iff moving its ray by +-delta px along u or v flips the hit
    status or moves the (fp32) depth by more than depth_tol, or | |o_d - z| - d_m | < rm_tol
    (DESIGN §6).  Decisions within 1e-6 of a threshold are not compared."""
    Z, r = 1000.0, 200.0
    cam = O.camera(160, 120)
    delta, dtol, rmtol, dm = 0.25, 0.5, 0.5, 10.0
    od = np.full((cam.height, cam.width), 820.0, np.float32)
    got = O.edge_mask_prims([_sphere((0.0, 0.0, Z), r)], cam, delta, dtol, od, dm, rmtol)

    def hit(u, v):
        x, y = (u - cam.cx) / cam.fx, (v - cam.cy) / cam.fy
        dd = 1.0 + x * x + y * y
        disc = Z * Z - dd * (Z * Z - r * r)
        if disc < 0:
            return None, abs(disc) / (Z * Z)
        return float(np.float32((Z - math.sqrt(disc)) / dd)), abs(disc) / (Z * Z)

    n_edge = n_amb = 0
    for v in range(cam.height):
        for u in range(cam.width):
            z, m0 = hit(u + 0.5, v + 0.5)
            amb = m0 < 1e-6
            e = False
            for du, dv in ((delta, 0), (-delta, 0), (0, delta), (0, -delta)):
                zk, mk = hit(u + 0.5 + du, v + 0.5 + dv)
                amb |= mk < 1e-6
                if (zk is None) != (z is None):
                    e = True
                elif z is not None:
                    amb |= abs(abs(zk - z) - dtol) < 1e-6
                    e |= abs(zk - z) > dtol
            if not e and z is not None:
                margin = abs(abs(820.0 - z) - dm) - rmtol
                amb |= abs(margin) < 1e-6
                e = margin < 0
            if amb:
                n_amb += 1
                continue
            assert bool(got[v, u]) == e, (u, v, z)
            n_edge += e
    assert n_amb < 10 and n_edge > 100  # the three rings are all populated
    # without an observation only the silhouette and depth-gradient rings remain
    got2 = O.edge_mask_prims([_sphere((0.0, 0.0, Z), r)], cam, delta, dtol, None, dm, rmtol)
    assert got2.sum() < got.sum() and np.all(got2 <= got)


def test_render_culled_equals_brute():
    for res in ("160x120", "640x480"):
        cam = O.camera(*W.RESOLUTIONS[res])
        for h in list(W.NAMED.values()) + list(W.random_poses(11, 3)):
            a = O.render(h, cam, culled=False)
            b = O.render(h, cam, culled=True)
            assert np.array_equal(a, b)


def test_render_depths_in_range_and_box_conservative():
    cam = O.camera(320, 240)
    for h in W.random_poses(12, 4):
        img = O.render(h, cam)
        nz = img[img > 0]
        assert np.all((nz >= cam.z_near) & (nz <= cam.z_far))
        prims, _ = O.fk(h)
        ys, xs = np.nonzero(img)
        boxes = [O.prim_box(p, cam, 0) for p in prims]
        for y, x in zip(ys, xs):
            assert any(b and b[0] <= x <= b[2] and b[1] <= y <= b[3] for b in boxes)


def test_synthetic_observation_flat_hand():
    cam = O.camera(160, 120)
    h = np.zeros(26)
    h[2] = 1000.0
    obs = O.synthesize(h, cam)
    nz = obs.depth[obs.depth > 0]
    assert nz.size > 0 and nz.min() >= 900 and nz.max() <= 1100
    h_behind = h.copy()
    h_behind[2] = 100.0  # inside the near plane: nothing within [z_near, z_far]
    assert np.all(O.render(h_behind, cam) == 0)


# ---------------------------------------------------------------- cost
def test_cost_worked_example():
    rows = {r[0]: r[1:] for r in _rows("cost_2x2_example.txt")}
    os_ = np.array(rows["o_s"], dtype=np.uint8)
    od = np.array(rows["o_d"], dtype=np.float32)
    rd = np.array(rows["r_d"], dtype=np.float32)
    s = O.score(od, os_, rd)
    assert s.s_or == int(rows["S_or"][0]) and s.s_and == int(rows["S_and"][0])
    assert s.num == float(rows["num_mm"][0])
    E, D = O.cost_from_sums(s)
    assert abs(E - float(rows["E"][0])) < 1e-12


def test_cost_disjoint_masks_area_term_is_lambda():
    od = np.array([0, 0, 0, 0], np.float32)
    os_ = np.array([1, 1, 0, 0], np.uint8)
    rd = np.array([0, 0, 1000, 1000], np.float32)
    E, D = O.cost_from_sums(O.score(od, os_, rd))
    assert E == 20.0


def test_cost_empty_is_zero_and_clamp_flag():
    z = np.zeros(4, np.float32)
    E, _ = O.cost_from_sums(O.score(z, np.zeros(4, np.uint8), z))
    assert E == 0.0  # AMB-6
    od = np.array([1000], np.float32)
    rd = np.array([1030], np.float32)
    s = O.score(od, np.ones(1, np.uint8), rd)
    assert s.num == 30.0 and s.s_rm == 0
    s2 = O.score(od, np.ones(1, np.uint8), rd, O.default_cost(clamp_at_dm=1))
    assert s2.num == 10.0
    s3 = O.score(od, np.ones(1, np.uint8), np.array([1100], np.float32))
    assert s3.num == 40.0  # clamped at d_M = 4 cm
    s4 = O.score(od, np.ones(1, np.uint8), np.array([1010], np.float32))
    assert s4.s_rm == 0  # |d| == d_m is not "smaller than" (AMB-5)


def test_cost_random_4x4_against_independent_pixel_loop():
    rng = np.random.default_rng(0)
    cp = O.default_cost()
    for _ in range(100):
        os_ = rng.integers(0, 2, 16).astype(np.uint8)
        od = np.where(rng.random(16) < 0.7, rng.uniform(950, 1050, 16), 0).astype(np.float32)
        rd = np.where(rng.random(16) < 0.7, rng.uniform(950, 1050, 16), 0).astype(np.float32)
        s = O.score(od, os_, rd, cp)
        rm = (rd > 0) & ((od == 0) | (np.abs(od.astype(float) - rd) < 10.0))
        both = (rd > 0) & (od > 0)
        s_or = int(((os_ == 1) | rm).sum())
        s_and = int(((os_ == 1) & rm).sum())
        num = math.fsum(min(abs(float(a) - float(b)), 40.0) for a, b in zip(od[both], rd[both]))
        assert (s.s_or, s.s_and) == (s_or, s_and)
        assert abs(s.num - num) <= 1e-9
        E, D = O.cost_from_sums(s, cp)
        if s_or:
            ref = 0.1 * num / s_or + 20 * (1 - 2 * s_and / (s_and + s_or))
        else:
            ref = 0.0
        assert abs(E - ref) < 1e-9
        assert 0 <= E and 0 <= 20 * (1 - 2 * s_and / max(s_and + s_or, 1)) <= 20


@pytest.mark.parametrize("res", ["160x120", "640x480"])
def test_self_match_is_exactly_zero(res):
    cam = O.camera(*W.RESOLUTIONS[res])
    for name, h in W.NAMED.items():
        obs = O.synthesize(h, cam)
        c = O.eval_batch(h[None], obs)
        assert c[0] == 0.0, name


def test_cost_monotone_along_perturbations():
    """E is non-decreasing along single-DOF perturbations away from h_true (north star):
    translations 0..8 mm in 1 mm steps, rotations 0..5 deg in 0.5 deg steps."""
    for res in ("160x120", "640x480"):
        cam = O.camera(*W.RESOLUTIONS[res])
        for name in ("h_A", "spread"):
            h0 = W.NAMED[name]
            obs = O.synthesize(h0, cam)
            for dof in (0, 1, 2, 3, 4, 5, 6 + 4, 6 + 8, 6 + 13):
                steps = np.arange(9.0) if dof < 3 else np.radians(np.arange(0, 5.01, 0.5))
                for sgn in (1, -1):
                    P = np.repeat(h0[None], len(steps), 0)
                    P[:, dof] += sgn * steps
                    c = O.eval_batch(P, obs)
                    assert np.all(np.diff(c) >= 0), (res, name, dof, sgn, c)
                    assert c[-1] > 0


def test_batch_invariances():
    cam = O.camera(160, 120)
    obs = O.synthesize(W.H_A, cam)
    P = W.random_poses(21, 12)
    c1 = O.eval_batch(P, obs, threads=1)
    c8 = O.eval_batch(P, obs, threads=8)
    assert np.array_equal(c1, c8)  # worker-count invariance
    perm = np.random.default_rng(1).permutation(12)
    assert np.array_equal(O.eval_batch(P[perm], obs), c1[perm])  # permutation equivariance
    assert np.array_equal(O.eval_batch(P[:1], obs), c1[:1])  # batch of 1
    same = O.eval_batch(np.repeat(P[:1], 5, 0), obs)
    assert np.all(same == same[0])


def test_walg_counts():
    cam = O.camera(640, 480)
    w, tests, upx = O.walg(W.H_A, cam)
    assert 5e3 < tests < 5e4 and 5e3 < upx < 3e4
    assert w == pytest.approx(w)  # finite
    w2, t2, u2 = O.walg(W.H_A, O.camera(160, 120))
    assert t2 < tests / 8  # ~1/16 of the pixels at quarter resolution


# ---------------------------------------------------------------- PSO
def test_constriction_closed_form():
    assert abs(O.constriction(2.8, 1.3) - 0.729843788128) < 1e-12
    assert abs(O.constriction(2.05, 2.05) - 0.729843788128) < 1e-12  # psi-only
    assert math.isnan(O.constriction(2.0, 2.0))


def _box(D, lo=-10.0, hi=10.0):
    return np.full(D, lo), np.full(D, hi)


def test_pso_sphere_convergence_and_invariants():
    """S:L414 (1-D x^2 on [-10, 10] -> < 1e-6) and S:L435 (6-D sphere -> < 1e-3; the box
    is unstated, [-1, 1]^6 here — the sphere value scales with the box squared)."""
    lo1, hi1 = _box(1)
    for seed in range(10):
        pp = O.default_pso(seed=seed, particles=64, generations=30, mutation_period=0)
        assert O.pso_sphere(1, lo1, hi1, lo1, hi1, 0, 0, np.zeros(1), pp).best_cost < 1e-6
    D = 6
    lo, hi = _box(D, -1.0, 1.0)
    for seed in range(10):
        pp = O.default_pso(seed=seed, particles=64, generations=30, mutation_period=0)
        r = O.pso_sphere(D, lo, hi, lo, hi, 0, 0, np.zeros(D), pp)
        assert r.best_cost < 1e-3
        assert np.all(np.diff(r.trace) <= 0)  # G monotone
        assert np.all((r.X >= lo) & (r.X <= hi))
        r2 = O.pso_sphere(D, lo, hi, lo, hi, 0, 0, np.zeros(D), pp)
        assert np.array_equal(r.best_x, r2.best_x) and np.array_equal(r.trace, r2.trace)


def test_pso_single_particle_never_moves():
    D = 4
    lo, hi = _box(D)
    pp = O.default_pso(seed=3, particles=1, generations=10, mutation_period=0)
    r = O.pso_sphere(D, lo, hi, lo, hi, 0, 0, np.full(D, 1.0), pp)
    r0 = O.pso_sphere(D, lo, hi, lo, hi, 0, 0, np.full(D, 1.0),
                      O.default_pso(seed=3, particles=1, generations=1, mutation_period=0))
    assert np.array_equal(r.X, r0.X) and np.all(r.V == 0)


def test_pso_degenerate_init_box_is_fixed_point():
    D = 3
    lo, hi = _box(D)
    c = np.array([1.0, -2.0, 3.0])
    pp = O.default_pso(seed=9, particles=8, generations=6, mutation_period=0)
    r = O.pso_sphere(D, lo, hi, c, c, 0, 0, np.zeros(D), pp)
    assert np.all(r.X == c) and np.all(r.V == 0)  # x = P = G, v = 0 is a fixed point


def test_pso_objective_scale_invariance():
    D = 5
    lo, hi = _box(D)
    pp = O.default_pso(seed=4, particles=16, generations=12)
    a = O.pso_sphere(D, lo, hi, lo, hi, 2, 5, np.zeros(D), pp)
    # scaling the objective by 4 (exact in binary) must not change any comparison
    b = O.pso_sphere(D, lo * 2, hi * 2, lo * 2, hi * 2, 2, 5, np.zeros(D), pp)
    np.testing.assert_array_equal(a.trace * 4, b.trace)
    np.testing.assert_array_equal(a.X * 2, b.X)


@pytest.mark.parametrize("N", [10, 11, 64])
def test_pso_mutation_marks_worst_half(N):
    """At k = 3 the worst floor(N/2) particles by Pcost at the end of generation 2 (ties:
    higher index worse) get their mutation dims re-drawn with zero velocity."""
    D = 8
    lo, hi = _box(D)
    big_lo, big_hi = lo * 1e6, hi * 1e6  # no clamping can zero a velocity
    r3 = O.pso_sphere(D, big_lo, big_hi, lo, hi, 2, D, np.zeros(D),
                      O.default_pso(seed=5, particles=N, generations=3, mutation_period=3))
    r4 = O.pso_sphere(D, big_lo, big_hi, lo, hi, 2, D, np.zeros(D),
                      O.default_pso(seed=5, particles=N, generations=4, mutation_period=3))
    order = sorted(range(N), key=lambda i: (r3.Pcost[i], i))
    expected = set(order[N - N // 2:])
    zero_v = set(np.nonzero(np.all(r4.V[:, 2:] == 0, axis=1))[0].tolist())
    assert zero_v == expected
    assert np.all(r4.V[:, :2] != 0)  # the 6 (here 2) non-finger dims keep moving
    # re-drawn uniformly in the search bounds (+-1e7 here), not in the +-10 init box
    marked = sorted(expected)
    assert np.all(np.abs(r4.X[marked][:, 2:]).max(axis=1) > 10.0)


def _golden_kv(name):
    out = {}
    for r in _rows(name):
        out[r[0]] = [float(x) for x in r[1:]]
    return out


def _scripted(costs_by_gen):
    """A batch objective returning fixed costs per generation (it ignores X)."""
    calls = []

    def f(X):
        calls.append(X.copy())
        return costs_by_gen[len(calls) - 1]
    return f, calls


def test_pso_eq6_hand_derived_two_particle_trajectory():
    """Eq. 6's coefficient and random-number assignment: c1 r1 multiplies
    (P - x), c2 r2 multiplies (G - x).  Scenario A of tests/golden/pso_eq6_hand.txt (hand
    derivation, scripts/gen_golden_pso.py): at k = 1 only c2 r2 acts on particle 1 (P = x),
    at k = 2 its c1 r1 term acts too.  A c1 <-> c2 or r1 <-> r2 swap changes every value."""
    g = _golden_kv("pso_eq6_hand.txt")
    assert abs(g["w"][0] - 0.729843788128) < 1e-12
    lo, hi = np.array([-100.0]), np.array([100.0])
    ilo, ihi = np.array([-10.0]), np.array([10.0])
    costs = [[1.0, 2.0], [1.0, 5.0], [0.5, 5.0]]
    for K in (2, 3):
        f, calls = _scripted(costs)
        pp = O.default_pso(seed=int(g["seed"][0]), particles=2, generations=K,
                           mutation_period=0)
        r = O.pso_run(1, lo, hi, ilo, ihi, 0, 0, pp, f)
        np.testing.assert_allclose(calls[0][:, 0], [g["A.x0_init"][0], g["A.x1_init"][0]],
                                   rtol=0, atol=1e-13)
        for key, arr in (("X", r.X[:, 0]), ("V", r.V[:, 0]), ("P", r.P[:, 0]),
                         ("Pcost", r.Pcost)):
            np.testing.assert_allclose(arr, g[f"A.K{K}.{key}"], rtol=1e-12, atol=1e-13,
                                       err_msg=f"K={K} {key}")
    np.testing.assert_array_equal(r.trace, g["A.K3.trace"])


def test_pso_mutation_orders_hand_derived():
    """Both mutation orders (AMB-17 reading 0; SPEC S:L447 order 1) on scenario B of the
    golden file: the worse particle's dim 1 re-drawn at k = 1 and evaluated as drawn
    (order 0), or re-drawn after k = 1's evaluation and moved by k = 2's update (order 1)."""
    g = _golden_kv("pso_eq6_hand.txt")
    lo, hi = np.full(2, -100.0), np.full(2, 100.0)
    ilo, ihi = np.full(2, -10.0), np.full(2, 10.0)
    costs = [[1.0, 2.0], [1.0, 5.0], [0.5, 5.0]]
    for order, K in ((0, 2), (1, 3)):
        f, calls = _scripted(costs)
        pp = O.default_pso(seed=int(g["seed"][0]), particles=2, generations=K,
                           mutation_period=1, mutation_fraction=0.5, mutation_after_eval=order)
        r = O.pso_run(2, lo, hi, ilo, ihi, 1, 2, pp, f)
        np.testing.assert_allclose(r.X.ravel(), g[f"B.order{order}.K{K}.X"], rtol=1e-12,
                                   atol=1e-13, err_msg=f"order {order}")
        np.testing.assert_allclose(r.V.ravel(), g[f"B.order{order}.K{K}.V"], rtol=1e-12,
                                   atol=1e-13, err_msg=f"order {order}")
    # order 0 evaluates the re-drawn coordinate at k = 1; order 1 first at k = 2, moved
    f, calls = _scripted(costs)
    O.pso_run(2, lo, hi, ilo, ihi, 1, 2,
              O.default_pso(seed=int(g["seed"][0]), particles=2, generations=3,
                            mutation_period=1, mutation_fraction=0.5), f)
    assert calls[1][1, 1] == g["B.order0.K2.X"][3]
    f, calls = _scripted(costs)
    O.pso_run(2, lo, hi, ilo, ihi, 1, 2,
              O.default_pso(seed=int(g["seed"][0]), particles=2, generations=3,
                            mutation_period=1, mutation_fraction=0.5, mutation_after_eval=1), f)
    assert calls[1][1, 1] != g["B.order0.K2.X"][3]
    assert calls[2][1, 1] == g["B.order1.K3.X"][3]


def test_pso_c2_zero_ignores_the_global_best_c1_zero_ignores_the_personal_best():
    """Eq. 6's two attractors in the limits: with c2 = 0 nothing pulls a particle
    towards G, and at generation 0 every P = x with v = 0, so no particle ever moves; with
    c1 = 0 (same psi = 4.1, so the same w) every particle but the best moves towards G."""
    D, N = 3, 12
    lo, hi = _box(D, -100.0, 100.0)
    ilo, ihi = _box(D)
    base = O.pso_sphere(D, lo, hi, ilo, ihi, 0, 0, np.full(D, 50.0),
                        O.default_pso(seed=7, particles=N, generations=1, mutation_period=0))
    a = O.pso_sphere(D, lo, hi, ilo, ihi, 0, 0, np.full(D, 50.0),
                     O.default_pso(seed=7, particles=N, generations=6, mutation_period=0,
                                   c1=4.1, c2=0.0))
    assert np.array_equal(a.X, base.X) and np.all(a.V == 0)
    b = O.pso_sphere(D, lo, hi, ilo, ihi, 0, 0, np.full(D, 50.0),
                     O.default_pso(seed=7, particles=N, generations=2, mutation_period=0,
                                   c1=0.0, c2=4.1))
    best = int(np.argmin(base.Pcost))
    moved = np.any(b.X != base.X, axis=1)
    assert not moved[best] and moved.sum() == N - 1
    # each moved particle stepped along G - x (c2 r2 (G - x), r2 >= 0, w > 0)
    G = base.X[best]
    for i in np.nonzero(moved)[0]:
        step, toward = b.X[i] - base.X[i], G - base.X[i]
        cos = step @ toward / (np.linalg.norm(step) * np.linalg.norm(toward))
        assert cos > 1 - 1e-12


def test_pso_hand_fit_recovers_from_local_init():
    cam = O.camera(160, 120)
    obs = O.synthesize(W.H_A, cam)
    c, rad = W.local_init_box()
    pp = O.default_pso(seed=1, particles=16, generations=10)
    r = O.pso_fit_hand(obs, pp, c, rad)
    assert np.all(np.diff(r.trace) <= 0)
    assert r.trace[-1] < r.trace[0]
    lo, hi = O.bounds()
    assert np.all((r.X >= lo) & (r.X <= hi))
    r2 = O.pso_fit_hand(obs, pp, c, rad, threads=3)
    assert np.array_equal(r.best_x, r2.best_x) and np.array_equal(r.trace, r2.trace)


# ------------------------------------------------------------------ observation front end
# Row f3: the depth-band segmentation is pinned by what it must recover, not by its
# own formula: a rendered hand in front of a background plane comes back exactly.
def _hand_scene(background=1500.0, **noise):
    cam = O.camera(160, 120)
    clean = O.render(W.H_A, cam)
    depth, skin = W.kinect_frame(clean, seed=3, background_mm=background, **noise)
    return cam, clean, depth, skin


@pytest.mark.parametrize("mode", [0, 1])
def test_segment_recovers_rendered_hand(mode):
    cam, clean, depth, _ = _hand_scene()
    hand = clean > 0
    obs, band = O.segment(depth, None, mode=mode, lo=500, hi=1100, width=250, cam=cam)
    assert np.array_equal(obs.mask, hand.astype(np.uint8))
    assert np.array_equal(obs.depth, np.where(hand, np.rint(clean), 0).astype(np.float32))
    if mode == 1:  # the nearest object is the hand: the band starts at its nearest depth
        assert band == (int(np.rint(clean[hand]).min()), int(np.rint(clean[hand]).min()) + 250)
    # the same scene without a background: identical result
    _, _, d2, _ = _hand_scene(background=None)
    obs2, _ = O.segment(d2, None, mode=mode, lo=500, hi=1100, width=250)
    assert np.array_equal(obs2.mask, obs.mask) and np.array_equal(obs2.depth, obs.depth)


def test_segment_keep_background_and_cost_ordering():
    cam, clean, depth, skin = _hand_scene()
    obs, _ = O.segment(depth, skin, mode=1, width=250, keep_background=True, cam=cam)
    assert np.array_equal(obs.depth, depth.astype(np.float32))   # every valid depth kept
    assert np.array_equal(obs.mask, (clean > 0).astype(np.uint8))
    # the truth still scores best against the segmented frame (background depth only
    # enters where the model renders: AMB-3/AMB-30)
    poses = np.stack([W.H_A] + list(W.random_poses(4, 6)))
    costs, _, _, _ = O.eval_batch(poses, obs, with_sums=True)
    assert costs[0] < 0.1 and np.all(costs[1:] > costs[0])


def test_segment_skin_dropout_and_flips():
    cam, clean, depth, skin = _hand_scene(dropout=0.2, mask_flip=0.05)
    hand = clean > 0
    obs, band = O.segment(depth, skin, mode=1, width=250)
    valid = depth > 0
    # skin pixels with no depth reading stay in O_s (missing depth is legal)
    assert np.all(obs.mask[(skin == 1) & ~valid] == 1)
    assert np.all(obs.depth[~valid] == 0)
    # skin flipped onto the far background (valid, outside the band) is rejected
    assert np.all(obs.mask[(skin == 1) & valid & ~hand] == 0)
    # non-skin pixels never enter O_s, and O_d is defined only inside the band
    assert np.all(obs.mask[skin == 0] == 0)
    assert np.all((obs.depth == 0) | ((obs.depth >= band[0]) & (obs.depth <= band[1])))


def test_segment_band_limits_inclusive_and_empty_frame():
    d = np.array([[699, 700, 850, 1000, 1001, 0]], np.uint16)
    obs, band = O.segment(d, None, mode=0, lo=700, hi=1000)
    assert obs.mask.tolist() == [[0, 1, 1, 1, 0, 0]] and band == (700, 1000)
    obs, band = O.segment(d, None, mode=1, width=301)
    assert obs.mask.tolist() == [[1, 1, 1, 1, 0, 0]] and band == (699, 1000)
    empty, band = O.segment(np.zeros((3, 4), np.uint16), None, mode=1, width=100)
    assert empty.mask.sum() == 0 and empty.depth.sum() == 0 and band == (1, 0)
