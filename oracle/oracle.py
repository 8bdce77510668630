"""ctypes binding of oracle/liboracle.so (TEST INFRASTRUCTURE ONLY; see oracle.h).

Argument marshalling only: every step of the oracle's arithmetic is in oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

NDOF = 26
NPRIM = 38
SPHERE, ELLIPSOID, CONE, CYLINDER = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (fp64, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
             "-Wall", "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _SO)
    return _SO


class Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("z_near", C.c_double), ("z_far", C.c_double)]


class Dims(C.Structure):
    _fields_ = [("palm_half_w", C.c_double), ("palm_half_t", C.c_double),
                ("palm_len", C.c_double), ("palm_cap_half_len", C.c_double),
                ("base", (C.c_double * 3) * 5), ("seg_len", (C.c_double * 3) * 5),
                ("radius", (C.c_double * 4) * 5), ("thumb_ell_x", C.c_double),
                ("thumb_ell_z", C.c_double), ("thumb_yaw_deg", C.c_double),
                ("thumb_pitch_deg", C.c_double)]


class CostParams(C.Structure):
    _fields_ = [("d_m", C.c_double), ("d_M", C.c_double), ("lam", C.c_double),
                ("lambda_k", C.c_double), ("depth_scale", C.c_double), ("kc_rest", C.c_double),
                ("clamp_at_dm", C.c_int32)]


class Prim(C.Structure):
    _fields_ = [("kind", C.c_int32), ("c", C.c_double * 3), ("R", (C.c_double * 3) * 3),
                ("s", C.c_double * 3)]


class Sums(C.Structure):
    _fields_ = [("s_o", C.c_int64), ("s_or", C.c_int64), ("s_and", C.c_int64),
                ("s_rm", C.c_int64), ("n_both", C.c_int64), ("num", C.c_double)]


class PsoParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("particles", C.c_int32), ("generations", C.c_int32),
                ("mutation_period", C.c_int32), ("per_dim_r", C.c_int32), ("c1", C.c_double),
                ("c2", C.c_double), ("mutation_fraction", C.c_double),
                ("stop_threshold", C.c_double), ("mutation_after_eval", C.c_int32)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
    return _lib


def _p(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


def default_dims() -> Dims:
    d = Dims()
    lib().or_default_dims(C.byref(d))
    return d


def default_cost(**kw) -> CostParams:
    p = CostParams()
    lib().or_default_cost(C.byref(p))
    for k, v in kw.items():
        setattr(p, "lam" if k == "lambda_" else k, v)
    return p


def default_pso(**kw) -> PsoParams:
    p = PsoParams()
    lib().or_default_pso(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def camera(width: int, height: int) -> Camera:
    c = Camera()
    lib().or_camera_for(width, height, C.byref(c))
    return c


def bounds():
    lo = np.zeros(NDOF)
    hi = np.zeros(NDOF)
    lib().or_bounds(_p(lo, C.c_double), _p(hi, C.c_double))
    return lo, hi


def philox(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().or_philox4x32_10(c, k, o)
    return list(o)


def u01(w0: int, w1: int) -> float:
    f = lib().or_u01
    f.restype = C.c_double
    return f(C.c_uint32(w0), C.c_uint32(w1))


def fk(h, dims: Dims | None = None):
    """Returns (list of Prim, joints[5,4,3])."""
    h = np.ascontiguousarray(h, dtype=np.float64)
    prims = (Prim * NPRIM)()
    joints = np.zeros((5, 4, 3))
    lib().or_fk(_p(h, C.c_double), C.byref(dims or default_dims()), prims, _p(joints, C.c_double))
    return list(prims), joints


def kc(h, rho: float = 0.0) -> float:
    f = lib().or_kc
    f.restype = C.c_double
    h = np.ascontiguousarray(h, dtype=np.float64)
    return f(_p(h, C.c_double), C.c_double(rho))


def first_hit(prim: Prim, direction) -> float:
    f = lib().or_first_hit
    f.restype = C.c_double
    d = np.ascontiguousarray(direction, dtype=np.float64)
    return f(C.byref(prim), _p(d, C.c_double))


def render_prims(prims, cam: Camera, culled: bool = False) -> np.ndarray:
    arr = (Prim * max(len(prims), 1))(*prims)
    out = np.zeros((cam.height, cam.width), dtype=np.float32)
    lib().or_render_prims(arr, len(prims), C.byref(cam), int(culled), _p(out, C.c_float))
    return out


def render(h, cam: Camera, dims: Dims | None = None, culled: bool = True) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.float64)
    out = np.zeros((cam.height, cam.width), dtype=np.float32)
    lib().or_render(_p(h, C.c_double), C.byref(dims or default_dims()), C.byref(cam), int(culled),
                    _p(out, C.c_float))
    return out


def edge_mask(h, cam: Camera, dims: Dims | None = None, delta: float = 1e-3,
              depth_tol: float = 1e-2, obs_depth=None, d_m: float = 10.0,
              rm_tol: float = 2e-3) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.float64)
    out = np.zeros((cam.height, cam.width), dtype=np.uint8)
    od = None if obs_depth is None else np.ascontiguousarray(obs_depth, dtype=np.float32)
    lib().or_edge_mask(_p(h, C.c_double), C.byref(dims or default_dims()), C.byref(cam),
                       C.c_double(delta), C.c_double(depth_tol), _p(od, C.c_float),
                       C.c_double(d_m), C.c_double(rm_tol), _p(out, C.c_uint8))
    return out


def edge_mask_prims(prims, cam: Camera, delta: float = 1e-3, depth_tol: float = 1e-2,
                    obs_depth=None, d_m: float = 10.0, rm_tol: float = 2e-3) -> np.ndarray:
    arr = (Prim * max(len(prims), 1))(*prims)
    out = np.zeros((cam.height, cam.width), dtype=np.uint8)
    od = None if obs_depth is None else np.ascontiguousarray(obs_depth, dtype=np.float32)
    lib().or_edge_mask_prims(arr, len(prims), C.byref(cam), C.c_double(delta),
                             C.c_double(depth_tol), _p(od, C.c_float), C.c_double(d_m),
                             C.c_double(rm_tol), _p(out, C.c_uint8))
    return out


def prim_box(prim: Prim, cam: Camera, margin: int = 0):
    b = (C.c_int32 * 4)()
    ok = lib().or_prim_box(C.byref(prim), C.byref(cam), margin, b)
    return tuple(b) if ok else None


def score(obs_depth, obs_mask, r_d, cp: CostParams | None = None) -> Sums:
    od = np.ascontiguousarray(obs_depth, dtype=np.float32).ravel()
    om = np.ascontiguousarray(obs_mask, dtype=np.uint8).ravel()
    rd = np.ascontiguousarray(r_d, dtype=np.float32).ravel()
    assert od.size == om.size == rd.size
    s = Sums()
    lib().or_score(_p(od, C.c_float), _p(om, C.c_uint8), _p(rd, C.c_float), C.c_int64(od.size),
                   C.byref(cp or default_cost()), C.byref(s))
    return s


def cost_from_sums(s: Sums, cp: CostParams | None = None, kc_value: float = 0.0):
    f = lib().or_cost_from_sums
    f.restype = C.c_double
    D = C.c_double()
    E = f(C.byref(s), C.byref(cp or default_cost()), C.c_double(kc_value), C.byref(D))
    return E, D.value


@dataclass
class Observation:
    depth: np.ndarray  # (H, W) float32 mm, 0 = undefined
    mask: np.ndarray   # (H, W) uint8 0/1
    cam: Camera


def synthesize(h_ref, cam: Camera, dims: Dims | None = None) -> Observation:
    """Simulation protocol: render h_ref; O_d = depth, O_s = silhouette."""
    d = render(h_ref, cam, dims)
    return Observation(d, (d > 0).astype(np.uint8), cam)


class SegmentParams(C.Structure):
    """or_segment_params (oracle.h): mode 0 fixed band [lo, hi], 1 nearest-object band."""
    _fields_ = [("mode", C.c_int32), ("lo", C.c_int32), ("hi", C.c_int32),
                ("width", C.c_int32), ("keep_background", C.c_int32)]


def segment(depth_u16, skin=None, mode: int = 1, lo: int = 0, hi: int = 0, width: int = 150,
            keep_background: bool = False, cam: Camera | None = None):
    """Row f3 front end: raw u16 depth (+ optional skin mask) -> Observation
    (O_d, O_s) and the band used."""
    d = np.ascontiguousarray(depth_u16, dtype=np.uint16)
    sk = None if skin is None else np.ascontiguousarray(skin, dtype=np.uint8)
    assert sk is None or sk.shape == d.shape
    od = np.zeros(d.shape, np.float32)
    os_ = np.zeros(d.shape, np.uint8)
    band = (C.c_int32 * 2)()
    sp = SegmentParams(mode, lo, hi, width, int(keep_background))
    lib().or_segment(_p(d, C.c_uint16), None if sk is None else _p(sk, C.c_uint8),
                     C.c_int64(d.size), C.byref(sp), _p(od, C.c_float), _p(os_, C.c_uint8), band)
    return Observation(od, os_, cam), (int(band[0]), int(band[1]))


def eval_batch(poses, obs: Observation, dims: Dims | None = None, cp: CostParams | None = None,
               culled: bool = True, threads: int = 0, with_sums: bool = False):
    poses = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, NDOF)
    n = poses.shape[0]
    costs = np.zeros(n)
    kcs = np.zeros(n)
    Ds = np.zeros(n)
    sums = (Sums * max(n, 1))()
    od = np.ascontiguousarray(obs.depth, dtype=np.float32)
    om = np.ascontiguousarray(obs.mask, dtype=np.uint8)
    lib().or_eval_batch(_p(poses, C.c_double), n, _p(od, C.c_float), _p(om, C.c_uint8),
                        C.byref(obs.cam), C.byref(dims or default_dims()),
                        C.byref(cp or default_cost()), int(culled), threads,
                        _p(costs, C.c_double), sums, _p(kcs, C.c_double), _p(Ds, C.c_double))
    if with_sums:
        return costs, [sums[i] for i in range(n)], kcs, Ds
    return costs


def walg(h, cam: Camera, dims: Dims | None = None):
    """(flops, primitive-pixel tests, union-box pixels) for one pose."""
    f = lib().or_walg
    f.restype = C.c_double
    h = np.ascontiguousarray(h, dtype=np.float64)
    t = C.c_int64()
    u = C.c_int64()
    w = f(_p(h, C.c_double), C.byref(dims or default_dims()), C.byref(cam), C.byref(t), C.byref(u))
    return w, t.value, u.value


def constriction(c1: float, c2: float) -> float:
    f = lib().or_constriction
    f.restype = C.c_double
    return f(C.c_double(c1), C.c_double(c2))


@dataclass
class PsoResult:
    best_x: np.ndarray
    best_cost: float
    trace: np.ndarray
    gens_run: int
    X: np.ndarray
    V: np.ndarray
    P: np.ndarray
    Pcost: np.ndarray


def _pso_outputs(N, D, K):
    return (np.zeros(D), C.c_double(), np.zeros(K), C.c_int32(), np.zeros((N, D)),
            np.zeros((N, D)), np.zeros((N, D)), np.zeros(N))


def pso_sphere(D, lo, hi, init_lo, init_hi, mut_lo, mut_hi, centre, pp: PsoParams) -> PsoResult:
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (lo, hi, init_lo, init_hi, centre)]
    bx, bc, tr, gr, X, V, P, Pc = _pso_outputs(pp.particles, D, pp.generations)
    rc = lib().or_pso_sphere(D, *[_p(a, C.c_double) for a in arrs[:4]], mut_lo, mut_hi,
                             _p(arrs[4], C.c_double), C.byref(pp), _p(bx, C.c_double),
                             C.byref(bc), _p(tr, C.c_double), C.byref(gr), _p(X, C.c_double),
                             _p(V, C.c_double), _p(P, C.c_double), _p(Pc, C.c_double))
    if rc != 0:
        raise ValueError("invalid PSO parameters")
    return PsoResult(bx, bc.value, tr, gr.value, X, V, P, Pc)


BATCH_FN = C.CFUNCTYPE(None, C.POINTER(C.c_double), C.c_int32, C.c_int32,
                       C.POINTER(C.c_double), C.c_void_p)


def pso_run(D, lo, hi, init_lo, init_hi, mut_lo, mut_hi, pp: PsoParams, objective) -> PsoResult:
    """or_pso_run with a Python batch objective: objective(X (n, D) array) -> n costs."""
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (lo, hi, init_lo, init_hi)]

    def cb(xp, n, d, costs, user):
        X = np.ctypeslib.as_array(xp, shape=(n, d)).copy()
        out = np.asarray(objective(X), dtype=np.float64)
        for i in range(n):
            costs[i] = float(out[i])

    fn = BATCH_FN(cb)
    bx, bc, tr, gr, X, V, P, Pc = _pso_outputs(pp.particles, D, pp.generations)
    rc = lib().or_pso_run(D, *[_p(a, C.c_double) for a in arrs], mut_lo, mut_hi, C.byref(pp),
                          fn, None, _p(bx, C.c_double), C.byref(bc), _p(tr, C.c_double),
                          C.byref(gr), _p(X, C.c_double), _p(V, C.c_double), _p(P, C.c_double),
                          _p(Pc, C.c_double))
    if rc != 0:
        raise ValueError("invalid PSO parameters")
    return PsoResult(bx, bc.value, tr, gr.value, X, V, P, Pc)


def pso_fit_hand(obs: Observation, pp: PsoParams, init_center=None, init_radius=None,
                 dims: Dims | None = None, cp: CostParams | None = None, culled: bool = True,
                 threads: int = 0) -> PsoResult:
    ic = None if init_center is None else np.ascontiguousarray(init_center, dtype=np.float64)
    ir = None if init_radius is None else np.ascontiguousarray(init_radius, dtype=np.float64)
    od = np.ascontiguousarray(obs.depth, dtype=np.float32)
    om = np.ascontiguousarray(obs.mask, dtype=np.uint8)
    bx, bc, tr, gr, X, V, P, Pc = _pso_outputs(pp.particles, NDOF, pp.generations)
    rc = lib().or_pso_fit_hand(_p(od, C.c_float), _p(om, C.c_uint8), C.byref(obs.cam),
                               C.byref(dims or default_dims()), C.byref(cp or default_cost()),
                               C.byref(pp), _p(ic, C.c_double), _p(ir, C.c_double), int(culled),
                               threads, _p(bx, C.c_double), C.byref(bc), _p(tr, C.c_double),
                               C.byref(gr), _p(X, C.c_double), _p(V, C.c_double),
                               _p(P, C.c_double), _p(Pc, C.c_double))
    if rc != 0:
        raise ValueError("invalid PSO parameters")
    return PsoResult(bx, bc.value, tr, gr.value, X, V, P, Pc)
