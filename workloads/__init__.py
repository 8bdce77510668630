"""Seeded synthetic inputs shared by tests and bench (DESIGN.md §7 "input recipe").

This module holds NONE of the method's arithmetic: no kinematics, rendering, cost or PSO.
It only produces input data — camera intrinsics (AMB-12), named poses, seeded pose
batches with the shapes and distributions of the paper's workloads (P:L148, P:L193,
P:L201) — so that the oracle and the CUDA path can be fed identical inputs.  Both
``oracle/`` and ``paper_2005_07068_b200/`` are forbidden from importing each other; both
may be fed from here.

Pose layout: [x, y, z (mm), th_x, th_y, th_z, then thumb, index, middle, ring,
little each (MPx, MPz, PIP, DIP)], angles in radians.
"""
from __future__ import annotations

import math

import numpy as np

NDOF = 26

# Table 1-2 limits in degrees / mm, used only to keep generated inputs in range.
_WRIST_LO = (-900.0, -680.0, 500.0, -30.0, -70.0, -35.0)
_WRIST_HI = (900.0, 680.0, 1500.0, 120.0, 75.0, 20.0)
_FINGER_LO = ((0, -15, 0, -15), (0, -15, 0, 0), (0, -10, 0, 0), (0, -30, 0, 0), (0, -45, 0, 0))
_FINGER_HI = ((90, 60, 50, 70), (90, 15, 100, 60), (90, 10, 100, 60), (90, 0, 100, 60),
              (90, 0, 100, 60))

RESOLUTIONS = {"160x120": (160, 120), "320x240": (320, 240), "640x480": (640, 480)}


def input_bounds():
    """(lo, hi) 26-vectors in pose units, for clamping generated inputs."""
    lo = list(_WRIST_LO[:3]) + [math.radians(a) for a in _WRIST_LO[3:]]
    hi = list(_WRIST_HI[:3]) + [math.radians(a) for a in _WRIST_HI[3:]]
    for f in range(5):
        lo += [math.radians(a) for a in _FINGER_LO[f]]
        hi += [math.radians(a) for a in _FINGER_HI[f]]
    return np.array(lo), np.array(hi)


def intrinsics(width: int, height: int) -> dict:
    """AMB-12: Kinect-like fx = fy = 525 at 640x480, principal point at the centre,
    scaled with the resolution; z_near / z_far = 300 / 2000 mm."""
    s = width / 640.0
    return dict(width=width, height=height, fx=525.0 * s, fy=525.0 * s, cx=0.5 * width,
                cy=0.5 * height, z_near=300.0, z_far=2000.0)


def pose(wrist_mm, wrist_deg, fingers_deg) -> np.ndarray:
    """Build a 26-vector from mm / degree groups."""
    h = list(wrist_mm) + [math.radians(a) for a in wrist_deg]
    for f in fingers_deg:
        h += [math.radians(a) for a in f]
    return np.array(h, dtype=np.float64)


# Benchmark truth h_A: inside Tables 1-2, kc = 0.
H_A = pose((-20.0, 60.0, 800.0), (10.0, -10.0, 5.0),
           ((20, 30, 10, 10), (10, 5, 10, 5), (10, 0, 10, 5), (10, -5, 10, 5), (10, -10, 10, 5)))

NAMED = {
    "h_A": H_A,
    "flat": pose((0.0, 0.0, 800.0), (0, 0, 0), ((0, 0, 0, 0),) * 5),
    "fist": pose((-20.0, 60.0, 800.0), (10.0, -10.0, 5.0),
                 ((40, 20, 40, 40), (70, 0, 90, 50), (70, 0, 90, 50), (70, 0, 90, 50),
                  (70, 0, 90, 50))),
    "point": pose((10.0, 40.0, 750.0), (5.0, 10.0, -5.0),
                  ((50, 10, 40, 40), (0, 0, 0, 0), (80, 0, 90, 50), (80, 0, 90, 50),
                   (80, 0, 90, 50))),
    "spread": pose((-30.0, 50.0, 850.0), (-5.0, 5.0, 0.0),
                   ((10, 40, 10, 10), (5, 15, 5, 5), (5, 0, 5, 5), (5, -20, 5, 5),
                    (5, -35, 5, 5))),
    # fingers pointing (almost) straight at the camera: rays inside the cones' openings
    "toward_camera": pose((5.0, -3.0, 700.0), (90.0, 0.0, 0.0), ((0, 0, 0, 0),) * 5),
    "toward_camera_tilt": pose((-5.0, 8.0, 650.0), (88.5, 1.0, 0.5),
                               ((10, 0, 0, 0), (0, 3, 0, 0), (0, 0, 0, 0), (0, -3, 0, 0),
                                (0, -5, 0, 0))),
}


def random_poses(seed: int, n: int) -> np.ndarray:
    """Parity poses: finger DOFs uniform in Table 1, wrist angles uniform
    within +-20 deg of h_A (clipped to Table 2), x, y uniform +-100 mm around h_A,
    z uniform in [600, 1000] mm."""
    rng = np.random.default_rng(seed)
    lo, hi = input_bounds()
    out = np.empty((n, NDOF))
    for i in range(n):
        h = np.empty(NDOF)
        h[0] = H_A[0] + rng.uniform(-100.0, 100.0)
        h[1] = H_A[1] + rng.uniform(-100.0, 100.0)
        h[2] = rng.uniform(600.0, 1000.0)
        for k in range(3, 6):
            h[k] = np.clip(H_A[k] + rng.uniform(-math.radians(20), math.radians(20)), lo[k], hi[k])
        h[6:] = rng.uniform(lo[6:], hi[6:])
        out[i] = h
    return out


def swarm_c4(n: int = 4096, seed: int = 7068) -> np.ndarray:
    """C4 mid-fit swarm: clip(h_A + sigma * N(0,1)), sigma = 20 mm on position,
    10 deg on wrist angles, 15 deg on finger angles."""
    return swarm_around(H_A, n, seed)


def swarm_around(centre, n: int, seed: int) -> np.ndarray:
    """The C4 swarm recipe around an arbitrary pose (row f2: one swarm per frame)."""
    rng = np.random.default_rng(seed)
    sigma = np.array([20.0] * 3 + [math.radians(10.0)] * 3 + [math.radians(15.0)] * 20)
    lo, hi = input_bounds()
    c = np.asarray(centre, np.float64)
    return np.clip(c[None, :] + sigma[None, :] * rng.standard_normal((n, NDOF)), lo, hi)


def cold_box(n: int = 4096, seed: int = 7069) -> np.ndarray:
    """C4's cold-box variant: poses uniform in the full Tables 1-2 box —
    a first-generation swarm; most hands are small, partly or wholly off-screen."""
    rng = np.random.default_rng(seed)
    lo, hi = input_bounds()
    return rng.uniform(lo[None, :], hi[None, :], size=(n, NDOF))


def local_init_box():
    """C2/C3 local PSO init: centre h_A, +-50 mm, +-20 deg on the wrist angles,
    full Table 1 on the fingers (radius large enough to cover the whole range)."""
    radius = np.array([50.0] * 3 + [math.radians(20.0)] * 3 + [math.pi] * 20)
    return H_A.copy(), radius


def motion_sequence(frames: int = 100, seed: int = 5) -> np.ndarray:
    """C5: a smooth seeded hand motion (sum of low-frequency sinusoids per DOF around h_A),
    kept inside Tables 1-2; the next rank in DESIGN §8."""
    rng = np.random.default_rng(seed)
    lo, hi = input_bounds()
    amp = np.array([60.0, 40.0, 80.0] + [math.radians(15.0)] * 3 + [math.radians(25.0)] * 20)
    freq = rng.uniform(0.5, 2.0, NDOF) * 2 * math.pi / frames
    phase = rng.uniform(0, 2 * math.pi, NDOF)
    t = np.arange(frames)[:, None]
    centre = (lo + hi) / 2
    centre[:6] = H_A[:6]
    seq = centre[None, :] + amp[None, :] * np.sin(freq[None, :] * t + phase[None, :])
    return np.clip(seq, lo, hi)


def kinect_frame(clean_depth, seed: int, depth_sigma: float = 0.0, dropout: float = 0.0,
                 mask_flip: float = 0.0, background_mm: float | None = None,
                 background_slope=(0.0, 0.0)):
    """Row f3 input: a Kinect-like raw frame from a clean hand render (SPEC S:L219-244
    NoiseSpec; the paper's sensor is a Kinect).  Returns (depth u16 mm, skin u8).

    Scene: the hand render in front of an optional background plane whose depth is
    background_mm + sx (u - W/2) + sy (v - H/2).  Sensor: additive Gaussian noise of
    depth_sigma mm on every valid depth, rounding to integer mm, then each valid pixel
    drops to 0 with probability `dropout`.  Skin image (the colour detector's output): the
    hand silhouette with each pixel flipped with probability `mask_flip`.  Seeded numpy
    draws; no method arithmetic."""
    rng = np.random.default_rng(seed)
    clean = np.asarray(clean_depth, np.float64)
    H, W = clean.shape
    hand = clean > 0
    scene = clean.copy()
    if background_mm is not None:
        v, u = np.mgrid[0:H, 0:W]
        plane = background_mm + background_slope[0] * (u - W / 2) + background_slope[1] * (v - H / 2)
        scene = np.where(hand, clean, plane)
    valid = scene > 0
    noisy = scene + depth_sigma * rng.standard_normal(scene.shape)
    depth = np.where(valid, np.clip(np.rint(noisy), 1, 65535), 0)
    drop = rng.random(scene.shape) < dropout
    depth = np.where(drop, 0, depth).astype(np.uint16)
    flip = rng.random(scene.shape) < mask_flip
    skin = (hand ^ flip).astype(np.uint8)
    return depth, skin
