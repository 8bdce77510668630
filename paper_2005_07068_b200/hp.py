"""ctypes binding of libhp.so (include/hp.h) — argument marshalling only.

Every step of the path (FK, rendering, scoring, PSO) runs in the CUDA kernels behind the C
ABI; this module converts torch tensors to device pointers and the current CUDA stream to
a ``cudaStream_t``.  There is no CPU fallback: if ``libhp.so`` is missing or no sm_100
device is present, construction raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HP_LIB") or os.path.join(_HERE, "libhp.so")  # HP_LIB: A/B builds
NDOF = 26
NPRIM = 38
REC_FLOATS = 24

HP_OK, HP_ERR_INVALID_ARG, HP_ERR_CUDA, HP_ERR_OOM, HP_ERR_NCCL, HP_ERR_STATE, \
    HP_ERR_NO_DEVICE = range(7)


class HPError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"hp status {status}: {msg}")
        self.status = status


class Intrinsics(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("z_near_mm", C.c_float),
                ("z_far_mm", C.c_float)]


class HandDims(C.Structure):
    _fields_ = [("palm_half_w", C.c_float), ("palm_half_t", C.c_float), ("palm_len", C.c_float),
                ("palm_cap_half_len", C.c_float), ("base", (C.c_float * 3) * 5),
                ("seg_len", (C.c_float * 3) * 5), ("radius", (C.c_float * 4) * 5),
                ("thumb_ell_x", C.c_float), ("thumb_ell_z", C.c_float),
                ("thumb_yaw_deg", C.c_float), ("thumb_pitch_deg", C.c_float)]


class CostParams(C.Structure):
    _fields_ = [("d_m", C.c_double), ("d_M", C.c_double), ("lam", C.c_double),
                ("lambda_k", C.c_double), ("depth_scale", C.c_double), ("kc_rest", C.c_double),
                ("clamp_at_dm", C.c_int32)]


class PsoParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("particles", C.c_int32), ("generations", C.c_int32),
                ("mutation_period", C.c_int32), ("per_dim_r", C.c_int32), ("c1", C.c_double),
                ("c2", C.c_double), ("mutation_fraction", C.c_double),
                ("stop_threshold", C.c_double), ("init_center", C.POINTER(C.c_double)),
                ("init_radius", C.POINTER(C.c_double)), ("mutation_after_eval", C.c_int32)]


_libs = {}
_VP = C.c_void_p


class SegmentParams(C.Structure):
    """hp_segment_params (include/hp.h, row f3)."""
    _fields_ = [("mode", C.c_int32), ("lo_mm", C.c_int32), ("hi_mm", C.c_int32),
                ("width_mm", C.c_int32), ("keep_background", C.c_int32)]


def lib(path: str | None = None) -> C.CDLL:
    """Load libhp.so (raises if it was not built: run ``python -m paper_2005_07068_b200.build``).
    `path` selects another build of the same ABI (e.g. the debug loopback build)."""
    path = path or LIB_PATH
    if path not in _libs:
        if not os.path.exists(path):
            raise ImportError(f"{path} not found: build it with "
                              "`python -m paper_2005_07068_b200.build` (no CPU fallback)")
        L = C.CDLL(path)
        sig = {
            "hp_default_dims": [C.POINTER(HandDims)],
            "hp_default_cost": [C.POINTER(CostParams)],
            "hp_default_pso": [C.POINTER(PsoParams)],
            "hp_default_intrinsics": [C.c_int32, C.c_int32, C.POINTER(Intrinsics)],
            "hp_bounds": [_VP, _VP],
            "hp_create": [C.POINTER(Intrinsics), C.POINTER(HandDims), C.POINTER(CostParams),
                          C.c_int32, C.c_int32, C.POINTER(_VP)],
            "hp_set_observation": [_VP, _VP, _VP, C.c_int32, _VP],
            "hp_render_observation": [_VP, _VP, _VP, _VP, _VP],
            "hp_eval_costs": [_VP, _VP, C.c_int64, _VP, _VP],
            "hp_eval_costs_host": [_VP, _VP, C.c_int64, _VP, _VP],
            "hp_eval_sums": [_VP, _VP, C.c_int64, _VP, _VP, _VP],
            "hp_eval_sums_f64": [_VP, _VP, C.c_int64, _VP, _VP, _VP],
            "hp_pso_fit": [_VP, C.POINTER(PsoParams), _VP, _VP, _VP, _VP, _VP],
            "hp_pso_state": [_VP, C.c_int32, C.c_int32, _VP, _VP, _VP, _VP],
            "hp_debug_fk": [_VP, _VP, _VP, _VP, _VP, _VP],
            "hp_debug_batch_fk": [_VP, C.c_int64, _VP, _VP],
            "hp_debug_render": [_VP, _VP, _VP, _VP],
            "hp_debug_pso_sphere": [_VP, C.c_int32, _VP, _VP, _VP, _VP, C.c_int32, C.c_int32, _VP,
                                    C.POINTER(PsoParams), _VP, _VP, _VP, _VP, _VP],
            "hp_track": [_VP, _VP, _VP, C.c_int32, C.c_int32, C.POINTER(PsoParams), _VP, _VP,
                         _VP, _VP, _VP],
            "hp_shard_range": [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64),
                               C.POINTER(C.c_int64)],
            "hp_nccl_available": [C.POINTER(C.c_int32)],
            "hp_get_nccl_id": [_VP],
            "hp_shard": [_VP, _VP, C.c_int32, C.c_int32],
            "hp_set_timing": [_VP, C.c_int32],
            "hp_set_observations": [_VP, _VP, _VP, C.c_int32, C.c_int32, _VP],
            "hp_default_segment": [C.POINTER(SegmentParams)],
            "hp_set_observation_kinect": [_VP, _VP, _VP, C.c_int32, C.POINTER(SegmentParams),
                                          C.c_int32, _VP, _VP],
            "hp_get_observation": [_VP, C.c_int32, _VP, _VP, _VP],
            "hp_eval_costs_frames": [_VP, _VP, C.c_int32, C.c_int64, _VP, _VP],
            "hp_eval_sums_frames": [_VP, _VP, C.c_int32, C.c_int64, _VP, _VP, _VP],
            "hp_last_kernel_ms": [_VP, _VP],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        if hasattr(L, "hp_shard_loopback"):  # debug builds only (-DHP_LOOPBACK_TEST=1)
            L.hp_shard_loopback.argtypes = [_VP, C.c_char_p, C.c_int32, C.c_int32]
            L.hp_shard_loopback.restype = C.c_int
        L.hp_last_error.argtypes = [_VP]
        L.hp_last_error.restype = C.c_char_p
        L.hp_last_launch_count.argtypes = [_VP]
        L.hp_last_launch_count.restype = C.c_int64
        L.hp_splits_for.argtypes = [_VP, C.c_int64]
        L.hp_splits_for.restype = C.c_int32
        L.hp_destroy.argtypes = [_VP]
        L.hp_destroy.restype = None
        _libs[path] = L
    return _libs[path]


def exported_symbols():
    """Names of every function include/hp.h declares (used by the CPU load test)."""
    return ["hp_default_dims", "hp_default_cost", "hp_default_pso", "hp_default_intrinsics",
            "hp_bounds", "hp_create", "hp_set_observation", "hp_render_observation",
            "hp_eval_costs", "hp_eval_costs_host", "hp_eval_sums", "hp_eval_sums_f64", "hp_pso_fit",
            "hp_pso_state",
            "hp_debug_fk", "hp_debug_batch_fk", "hp_debug_render", "hp_debug_pso_sphere", "hp_last_launch_count",
            "hp_splits_for", "hp_last_error", "hp_destroy", "hp_shard_range",
            "hp_nccl_available", "hp_get_nccl_id", "hp_shard", "hp_track",
            "hp_set_timing", "hp_last_kernel_ms", "hp_set_observations",
            "hp_eval_costs_frames", "hp_eval_sums_frames", "hp_default_segment",
            "hp_set_observation_kinect", "hp_get_observation"]


def _check(status: int, ctx=None, L=None):
    if status != HP_OK:
        msg = (L or lib()).hp_last_error(ctx)
        raise HPError(status, msg.decode() if msg else "")


def default_dims() -> HandDims:
    d = HandDims()
    _check(lib().hp_default_dims(C.byref(d)))
    return d


def default_cost(**kw) -> CostParams:
    c = CostParams()
    _check(lib().hp_default_cost(C.byref(c)))
    for k, v in kw.items():
        setattr(c, "lam" if k == "lambda_" else k, v)
    return c


def default_intrinsics(width: int, height: int) -> Intrinsics:
    i = Intrinsics()
    _check(lib().hp_default_intrinsics(width, height, C.byref(i)))
    return i


def intrinsics_from(d: dict) -> Intrinsics:
    return Intrinsics(d["width"], d["height"], d["fx"], d["fy"], d["cx"], d["cy"], d["z_near"],
                      d["z_far"])


def bounds():
    lo = np.zeros(NDOF)
    hi = np.zeros(NDOF)
    _check(lib().hp_bounds(lo.ctypes.data, hi.ctypes.data))
    return lo, hi


def shard_range(n: int, rank: int, world: int):
    """[begin, end) of the poses rank `rank` of `world` scores (hp_shard_range)."""
    b, e = C.c_int64(), C.c_int64()
    _check(lib().hp_shard_range(n, rank, world, C.byref(b), C.byref(e)))
    return b.value, e.value


def nccl_available() -> bool:
    v = C.c_int32()
    _check(lib().hp_nccl_available(C.byref(v)))
    return bool(v.value)


def _nccl_lib_hint():
    """Point HP_NCCL_LIB at the NCCL torch ships (the same library torch.distributed uses)."""
    if os.environ.get("HP_NCCL_LIB"):
        return
    try:
        import nvidia.nccl  # noqa: F401

        cand = os.path.join(os.path.dirname(nvidia.nccl.__file__), "lib", "libnccl.so.2")
    except Exception:
        return
    if os.path.exists(cand):
        os.environ["HP_NCCL_LIB"] = cand


def nccl_unique_id() -> bytes:
    _nccl_lib_hint()
    buf = (C.c_uint8 * 128)()
    _check(lib().hp_get_nccl_id(buf))
    return bytes(buf)


def broadcast_bytes(payload: bytes | None, rank: int, nbytes: int = 128, group=None) -> bytes:
    """Broadcast `nbytes` from rank 0 over torch.distributed (any backend)."""
    import torch
    import torch.distributed as dist

    t = torch.zeros(nbytes, dtype=torch.uint8)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().numpy().tobytes())


def exchange_nccl_id(rank: int, group=None) -> bytes:
    """Rank 0 creates the NCCL unique id; torch.distributed broadcasts the 128 bytes."""
    return broadcast_bytes(nccl_unique_id() if rank == 0 else None, rank, 128, group)


def _dptr(t) -> int:
    """Device pointer of a contiguous CUDA tensor."""
    assert t.is_cuda and t.is_contiguous(), "expected a contiguous CUDA tensor"
    return t.data_ptr()


def _stream(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


@dataclass
class FitResult:
    best_pose: np.ndarray
    best_cost: float
    trace: np.ndarray
    gens_run: int


class Context:
    """One hp_ctx: a camera, a hand model, cost constants and a workspace for up to
    ``max_particles`` poses per call (include/hp.h hp_create)."""

    def __init__(self, width: int = 640, height: int = 480, max_particles: int = 4096,
                 intrinsics: Intrinsics | None = None, dims: HandDims | None = None,
                 cost: CostParams | None = None, device: int = -1, lib_path: str | None = None):
        self._L = lib(lib_path)
        self.cam = intrinsics or default_intrinsics(width, height)
        self.width, self.height = self.cam.width, self.cam.height
        self.max_particles = max_particles
        h = _VP()
        st = self._L.hp_create(C.byref(self.cam), C.byref(dims) if dims else None,
                               C.byref(cost) if cost else None, max_particles, device,
                               C.byref(h))
        _check(st, None, self._L)
        self._h = h

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None):
            self._L.hp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    # -- observation
    def set_observation(self, depth, mask, stream=None):
        """O = (O_s, O_d): depth fp32 [H][W] mm (0 = undefined), mask u8 [H][W]; numpy
        arrays (host) or CUDA tensors (device)."""
        if isinstance(depth, np.ndarray):
            d = np.ascontiguousarray(depth, dtype=np.float32)
            m = np.ascontiguousarray(mask, dtype=np.uint8)
            assert d.shape == (self.height, self.width) and m.shape == d.shape
            _check(self._L.hp_set_observation(self._h, d.ctypes.data, m.ctypes.data, 0,
                                              _stream(stream)), self._h, self._L)
        else:
            assert tuple(depth.shape) == (self.height, self.width)
            _check(self._L.hp_set_observation(self._h, _dptr(depth), _dptr(mask), 1,
                                              _stream(stream)), self._h, self._L)
        self.frames = 1

    def set_observations(self, depth, mask, stream=None):
        """Frame batch (row f2): depth fp32 [M][H][W], mask u8 [M][H][W]; host or device."""
        if isinstance(depth, np.ndarray):
            d = np.ascontiguousarray(depth, dtype=np.float32)
            m = np.ascontiguousarray(mask, dtype=np.uint8)
            assert d.ndim == 3 and d.shape[1:] == (self.height, self.width) and m.shape == d.shape
            _check(self._L.hp_set_observations(self._h, d.ctypes.data, m.ctypes.data, d.shape[0],
                                               0, _stream(stream)), self._h, self._L)
        else:
            assert depth.dim() == 3 and tuple(depth.shape[1:]) == (self.height, self.width)
            assert depth.is_contiguous() and mask.is_contiguous()
            _check(self._L.hp_set_observations(self._h, _dptr(depth), _dptr(mask),
                                               depth.shape[0], 1, _stream(stream)), self._h, self._L)
        self.frames = int(depth.shape[0])

    def set_observation_kinect(self, depth_u16, skin=None, mode: int = 1, lo_mm: int = 0,
                               hi_mm: int = 0, width_mm: int = 250,
                               keep_background: bool = False, stream=None):
        """Row f3 front end: Kinect u16 depth [H][W] or [M][H][W] (+ optional u8 skin image),
        numpy (host) or CUDA tensors (device) -> segmented observation frames.  Returns the
        band used per frame as an int array [M][2]."""
        seg = SegmentParams(mode, lo_mm, hi_mm, width_mm, int(keep_background))
        if isinstance(depth_u16, np.ndarray):
            d = np.ascontiguousarray(depth_u16, dtype=np.uint16)
            sk = None if skin is None else np.ascontiguousarray(skin, dtype=np.uint8)
            shape, dp, sp, dev = d.shape, d.ctypes.data, (None if sk is None else sk.ctypes.data), 0
        else:
            import torch

            assert depth_u16.dtype in (torch.uint16, torch.int16) and depth_u16.is_contiguous()
            shape, dp, dev = tuple(depth_u16.shape), _dptr(depth_u16), 1
            sp = None if skin is None else _dptr(skin)
        frames = 1 if len(shape) == 2 else shape[0]
        assert tuple(shape[-2:]) == (self.height, self.width)
        band = np.zeros((frames, 2), np.int32)
        _check(self._L.hp_set_observation_kinect(self._h, dp, sp, frames, C.byref(seg), dev,
                                                 band.ctypes.data, _stream(stream)), self._h, self._L)
        self.frames = frames
        return band

    def get_observation(self, frame: int = 0, stream=None):
        """(O_d fp32 [H][W], O_s u8 [H][W]) CUDA tensors of observation frame `frame`."""
        import torch

        d = torch.empty((self.height, self.width), dtype=torch.float32, device="cuda")
        m = torch.empty((self.height, self.width), dtype=torch.uint8, device="cuda")
        _check(self._L.hp_get_observation(self._h, frame, _dptr(d), _dptr(m), _stream(stream)),
               self._h, self._L)
        return d, m

    def render_observation(self, h_ref, stream=None):
        """Simulation protocol: render h_ref on the GPU -> (depth, mask) tensors."""
        import torch

        h = np.ascontiguousarray(h_ref, dtype=np.float64)
        depth = torch.empty((self.height, self.width), dtype=torch.float32, device="cuda")
        mask = torch.empty((self.height, self.width), dtype=torch.uint8, device="cuda")
        _check(self._L.hp_render_observation(self._h, h.ctypes.data, _dptr(depth), _dptr(mask),
                                             _stream(stream)), self._h, self._L)
        return depth, mask

    # -- evaluation
    def eval_costs(self, poses, out=None, stream=None):
        """E(h, O) for poses [N][26] fp32 CUDA tensor -> costs [N] fp32 (async)."""
        import torch

        assert poses.dtype == torch.float32 and poses.shape[-1] == NDOF
        n = poses.shape[0]
        if out is None:
            out = torch.empty(n, dtype=torch.float32, device=poses.device)
        _check(self._L.hp_eval_costs(self._h, _dptr(poses), n, _dptr(out), _stream(stream)),
               self._h, self._L)
        return out

    def eval_costs_frames(self, poses, out=None, stream=None):
        """Frame-batched E: poses [M][n][26] fp32 CUDA tensor (M = frames set) -> [M][n]."""
        import torch

        assert poses.dtype == torch.float32 and poses.dim() == 3 and poses.shape[-1] == NDOF
        assert poses.is_contiguous()
        m, n = poses.shape[0], poses.shape[1]
        if m != self.frames:
            raise ValueError(f"poses hold {m} frames, the observation {self.frames}")
        if out is None:
            out = torch.empty((m, n), dtype=torch.float32, device=poses.device)
        if out.dtype != torch.float32 or tuple(out.shape) != (m, n) or not out.is_contiguous():
            raise ValueError("out must be a contiguous float32 tensor of shape (frames, n)")
        _check(self._L.hp_eval_costs_frames(self._h, _dptr(poses), m, n, _dptr(out),
                                            _stream(stream)), self._h, self._L)
        return out

    def eval_sums_frames(self, poses, stream=None):
        """(sums [M][n][4] int64, costs fp64 [M][n]) of the frame-batched evaluation."""
        import torch

        assert poses.dtype == torch.float32 and poses.dim() == 3 and poses.shape[-1] == NDOF
        assert poses.is_contiguous()
        m, n = poses.shape[0], poses.shape[1]
        if m != self.frames:
            raise ValueError(f"poses hold {m} frames, the observation {self.frames}")
        sums = torch.zeros((m, n, 4), dtype=torch.int64, device=poses.device)
        costs = torch.empty((m, n), dtype=torch.float64, device=poses.device)
        _check(self._L.hp_eval_sums_frames(self._h, _dptr(poses), m, n, _dptr(sums),
                                           _dptr(costs), _stream(stream)), self._h, self._L)
        return sums, costs

    def eval_costs_host(self, poses: np.ndarray, out: np.ndarray | None = None,
                        stream=None) -> np.ndarray:
        """Host-buffer variant: copies in, scores, copies out, synchronises.  Page-locked
        arrays (e.g. numpy views of torch pin_memory tensors) are DMA'd directly."""
        p = np.ascontiguousarray(poses, dtype=np.float32).reshape(-1, NDOF)
        if out is None:
            out = np.empty(p.shape[0], dtype=np.float32)
        assert out.dtype == np.float32 and out.flags.c_contiguous and out.size >= p.shape[0]
        _check(self._L.hp_eval_costs_host(self._h, p.ctypes.data, p.shape[0], out.ctypes.data,
                                          _stream(stream)), self._h, self._L)
        return out

    def eval_sums(self, poses, stream=None):
        """(sums [N][4] u64 as int64 tensor, costs fp64 [N]) — test hook."""
        import torch

        n = poses.shape[0]
        sums = torch.zeros((n, 4), dtype=torch.int64, device=poses.device)
        costs = torch.empty(n, dtype=torch.float64, device=poses.device)
        _check(self._L.hp_eval_sums(self._h, _dptr(poses), n, _dptr(sums), _dptr(costs),
                                    _stream(stream)), self._h, self._L)
        return sums, costs

    def eval_sums_f64(self, poses, stream=None):
        """(sums [N][4], costs fp64 [N]) of fp64 poses [N][26] (CUDA tensor): the scoring a
        fit applies to its fp64 particles (hp_eval_sums_f64)."""
        import torch

        assert poses.dtype == torch.float64 and poses.dim() == 2 and poses.shape[1] == NDOF
        assert poses.is_contiguous()
        n = poses.shape[0]
        sums = torch.zeros((n, 4), dtype=torch.int64, device=poses.device)
        costs = torch.empty(n, dtype=torch.float64, device=poses.device)
        _check(self._L.hp_eval_sums_f64(self._h, _dptr(poses), n, _dptr(sums), _dptr(costs),
                                        _stream(stream)), self._h, self._L)
        return sums, costs

    def shard_loopback(self, group: str, rank: int, world: int):
        """Debug builds only: join an in-process loopback group (hp_shard_loopback)."""
        if not hasattr(self._L, "hp_shard_loopback"):
            raise RuntimeError("hp_shard_loopback exists only in -DHP_LOOPBACK_TEST builds")
        _check(self._L.hp_shard_loopback(self._h, group.encode(), rank, world), self._h, self._L)
        self.rank, self.world = rank, world

    def shard(self, rank: int, world: int, nccl_id: bytes | None = None, group=None):
        """Particle-sharded mode (hp_shard): collective over the `world` ranks."""
        _nccl_lib_hint()
        if nccl_id is None:
            nccl_id = exchange_nccl_id(rank, group)
        buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        _check(self._L.hp_shard(self._h, buf, rank, world), self._h, self._L)
        self.rank, self.world = rank, world

    def splits_for(self, n: int) -> int:
        return self._L.hp_splits_for(self._h, n)

    def last_launch_count(self) -> int:
        return self._L.hp_last_launch_count(self._h)

    def set_timing(self, on: bool = True):
        """Record per-launch CUDA events around every later evaluation (hp_set_timing)."""
        _check(self._L.hp_set_timing(self._h, 1 if on else 0), self._h, self._L)

    def last_kernel_ms(self) -> tuple[float, float, float]:
        """(first launch, renderer alone, near-plane pass) device ms of the last timed
        evaluation."""
        ms = (C.c_float * 3)()
        _check(self._L.hp_last_kernel_ms(self._h, ms), self._h, self._L)
        return float(ms[0]), float(ms[1]), float(ms[2])

    # -- PSO
    def pso_fit(self, seed: int = 0, particles: int = 64, generations: int = 30,
                mutation_period: int = 3, c1: float = 2.8, c2: float = 1.3,
                mutation_fraction: float = 0.5, per_dim_r: bool = False,
                stop_threshold: float = -math.inf, init_center=None, init_radius=None,
                mutation_after_eval: int = 0, stream=None) -> FitResult:
        """The paper's PSO fit on the GPU; synchronous."""
        p = PsoParams()
        _check(self._L.hp_default_pso(C.byref(p)), None, self._L)
        p.mutation_after_eval = int(mutation_after_eval)
        p.seed, p.particles, p.generations = seed, particles, generations
        p.mutation_period, p.c1, p.c2 = mutation_period, c1, c2
        p.mutation_fraction, p.per_dim_r, p.stop_threshold = mutation_fraction, int(per_dim_r), \
            stop_threshold
        keep = []
        if init_center is not None:
            ic = np.ascontiguousarray(init_center, dtype=np.float64)
            ir = np.ascontiguousarray(init_radius, dtype=np.float64)
            keep += [ic, ir]
            p.init_center = ic.ctypes.data_as(C.POINTER(C.c_double))
            p.init_radius = ir.ctypes.data_as(C.POINTER(C.c_double))
        best = np.zeros(NDOF)
        cost = C.c_double()
        trace = np.zeros(generations)
        gr = C.c_int32()
        _check(self._L.hp_pso_fit(self._h, C.byref(p), best.ctypes.data, C.byref(cost),
                                  trace.ctypes.data, C.byref(gr), _stream(stream)), self._h, self._L)
        return FitResult(best, cost.value, trace, gr.value)

    def track(self, depth_seq, mask_seq, track_radius, seed: int = 0, particles: int = 64,
              generations: int = 30, mutation_period: int = 3, init_center=None,
              init_radius=None, mutation_after_eval: int = 0, stream=None):
        """Temporal tracking (hp_track): per-frame fit warm-started at the previous best
        pose +- track_radius.  depth_seq / mask_seq: [F][H][W] numpy (host) or CUDA
        tensors.  Returns (poses [F][26], costs [F], traces [F][generations])."""
        p = PsoParams()
        _check(self._L.hp_default_pso(C.byref(p)), None, self._L)
        p.seed, p.particles, p.generations, p.mutation_period = (seed, particles, generations,
                                                                 mutation_period)
        p.mutation_after_eval = int(mutation_after_eval)
        keep = []
        if init_center is not None:
            ic = np.ascontiguousarray(init_center, dtype=np.float64)
            ir = np.ascontiguousarray(init_radius, dtype=np.float64)
            keep += [ic, ir]
            p.init_center = ic.ctypes.data_as(C.POINTER(C.c_double))
            p.init_radius = ir.ctypes.data_as(C.POINTER(C.c_double))
        tr = np.ascontiguousarray(track_radius, dtype=np.float64)
        if isinstance(depth_seq, np.ndarray):
            d = np.ascontiguousarray(depth_seq, dtype=np.float32)
            m = np.ascontiguousarray(mask_seq, dtype=np.uint8)
            F = d.shape[0]
            dp, mp_, dev = d.ctypes.data, m.ctypes.data, 0
        else:
            F = depth_seq.shape[0]
            dp, mp_, dev = _dptr(depth_seq), _dptr(mask_seq), 1
        poses = np.zeros((F, NDOF))
        costs = np.zeros(F)
        traces = np.zeros((F, generations))
        try:
            _check(self._L.hp_track(self._h, dp, mp_, F, dev, C.byref(p), tr.ctypes.data,
                                    poses.ctypes.data, costs.ctypes.data, traces.ctypes.data,
                                    _stream(stream)), self._h, self._L)
        finally:
            self.frames = 1  # hp_track sets one observation frame at a time
        return poses, costs, traces

    def pso_state(self, particles: int, D: int = NDOF):
        X = np.zeros((particles, D))
        V = np.zeros((particles, D))
        P = np.zeros((particles, D))
        Pc = np.zeros(particles)
        _check(self._L.hp_pso_state(self._h, particles, D, X.ctypes.data, V.ctypes.data,
                                    P.ctypes.data, Pc.ctypes.data), self._h, self._L)
        return X, V, P, Pc

    def debug_pso_sphere(self, D, lo, hi, init_lo, init_hi, mut_lo, mut_hi, centre, seed=0,
                         particles=64, generations=30, mutation_period=3, c1=2.8, c2=1.3,
                         mutation_fraction=0.5, per_dim_r=False, stop_threshold=-math.inf,
                         mutation_after_eval=0):
        p = PsoParams()
        _check(self._L.hp_default_pso(C.byref(p)), None, self._L)
        p.mutation_after_eval = int(mutation_after_eval)
        p.seed, p.particles, p.generations = seed, particles, generations
        p.mutation_period, p.c1, p.c2 = mutation_period, c1, c2
        p.mutation_fraction, p.per_dim_r, p.stop_threshold = mutation_fraction, int(per_dim_r), \
            stop_threshold
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (lo, hi, init_lo, init_hi,
                                                                     centre)]
        best = np.zeros(D)
        cost = C.c_double()
        trace = np.zeros(generations)
        gr = C.c_int32()
        _check(self._L.hp_debug_pso_sphere(self._h, D, *[a.ctypes.data for a in arrs[:4]],
                                           mut_lo, mut_hi, arrs[4].ctypes.data, C.byref(p),
                                           best.ctypes.data, C.byref(cost), trace.ctypes.data,
                                           C.byref(gr), None), self._h, self._L)
        return FitResult(best, cost.value, trace, gr.value)

    # -- test hooks
    def debug_fk(self, pose):
        h = np.ascontiguousarray(pose, dtype=np.float64)
        rec = np.zeros((NPRIM, REC_FLOATS), dtype=np.float32)
        boxes = np.zeros((NPRIM, 4), dtype=np.int32)
        joints = np.zeros((5, 4, 3))
        kc = C.c_double()
        _check(self._L.hp_debug_fk(self._h, h.ctypes.data, rec.ctypes.data, boxes.ctypes.data,
                                   joints.ctypes.data, C.byref(kc)), self._h, self._L)
        return rec, boxes, joints, kc.value

    def debug_batch_fk(self, p: int):
        """(records, boxes) k_fk_batch wrote for pose p of the last batch-path call."""
        rec = np.zeros((NPRIM, REC_FLOATS), dtype=np.float32)
        boxes = np.zeros((NPRIM, 4), dtype=np.int32)
        _check(self._L.hp_debug_batch_fk(self._h, p, rec.ctypes.data, boxes.ctypes.data),
               self._h, self._L)
        return rec, boxes

    def debug_render(self, pose_dev, stream=None):
        import torch

        depth = torch.empty((self.height, self.width), dtype=torch.float32, device="cuda")
        _check(self._L.hp_debug_render(self._h, _dptr(pose_dev), _dptr(depth), _stream(stream)),
               self._h, self._L)
        return depth
