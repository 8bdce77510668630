"""The persistent fit kernel (k_fit): one cooperative launch per fit must return
bit for bit what the per-generation fused kernels return (same update order, FK, per-pixel
formulas and integer sums) — best pose, trace, generations run and the final swarm state
(hp_pso_state) — across the PSO flags, the stop rule and the C1 / C3 configurations.  Both
paths are themselves checked against the oracle (test_gpu_parity, test_gpu_next)."""
import math
import os

import numpy as np
import pytest

import oracle as O
import paper_2005_07068_b200 as hp
import workloads as W

pytestmark = pytest.mark.gpu


def _ctx(w, h, persist, cap=64):
    old = os.environ.pop("HP_NO_FIT_PERSIST", None)
    if not persist:
        os.environ["HP_NO_FIT_PERSIST"] = "1"
    try:
        return hp.Context(w, h, max_particles=cap)
    finally:
        os.environ.pop("HP_NO_FIT_PERSIST", None)
        if old is not None:
            os.environ["HP_NO_FIT_PERSIST"] = old


CASES = [
    ((160, 120), 16, 10, {}),
    ((160, 120), 16, 10, dict(per_dim_r=True, mutation_period=2, mutation_fraction=0.25)),
    ((160, 120), 16, 10, dict(mutation_after_eval=1)),
    ((160, 120), 16, 12, dict(stop_threshold="mid")),
    ((320, 240), 64, 40, {}),
    ((640, 480), 64, 40, {}),
    ((640, 480), 100, 8, dict(mutation_period=2)),
]


@pytest.mark.parametrize("res,N,K,kw", CASES)
def test_persistent_fit_equals_generation_kernels(res, N, K, kw):
    w, h = res
    obs = O.synthesize(W.H_A, O.camera(w, h))
    c, rad = W.local_init_box()
    out = []
    if kw.get("stop_threshold") == "mid":  # fires half way: just above the 5th trace value
        ctx = _ctx(w, h, False)
        ctx.set_observation(obs.depth, obs.mask)
        t = ctx.pso_fit(seed=1, particles=N, generations=K, init_center=c, init_radius=rad).trace
        ctx.close()
        assert t[4] < t[0]
        kw = dict(stop_threshold=float(t[4]) * (1 + 1e-12))
    for persist in (True, False):
        ctx = _ctx(w, h, persist, cap=max(N, 64))
        ctx.set_observation(obs.depth, obs.mask)
        for seed in (1, 2):
            r = ctx.pso_fit(seed=seed, particles=N, generations=K, init_center=c,
                            init_radius=rad, **kw)
            launches = ctx.last_launch_count()
            out.append((persist, seed, r, ctx.pso_state(N), launches))
        ctx.close()
    half = len(out) // 2
    for a, b in zip(out[:half], out[half:]):
        assert a[0] and not b[0] and a[1] == b[1]
        ra, rb = a[2], b[2]
        assert a[4] == 1 and b[4] == 1 + K  # one cooperative launch vs init + K kernels
        assert ra.gens_run == rb.gens_run
        assert np.array_equal(ra.best_pose, rb.best_pose)
        assert ra.best_cost == rb.best_cost
        assert np.array_equal(ra.trace, rb.trace)
        assert ra.gens_run == rb.gens_run
        for xa, xb in zip(a[3], b[3]):
            assert np.array_equal(xa, xb)
    if "stop_threshold" in kw:
        assert out[0][2].gens_run <= 6  # the stop rule fired (seed 1)


def test_persistent_fit_tracking_matches_generation_kernels():
    """hp_track (row f1) runs one fit per frame: the persistent kernel must reproduce the
    per-generation path frame by frame."""
    w, h, F = 160, 120, 4
    cam = O.camera(w, h)
    seq = W.motion_sequence(frames=100)[:F]
    obs = [O.synthesize(hf, cam) for hf in seq]
    depth = np.stack([o.depth for o in obs])
    mask = np.stack([o.mask for o in obs])
    radius = np.array([15.0] * 3 + [math.radians(8)] * 3 + [math.radians(20)] * 20)
    c0, r0 = seq[0], np.array([40.0] * 3 + [math.radians(15)] * 3 + [math.pi] * 20)
    res = []
    for persist in (True, False):
        ctx = _ctx(w, h, persist)
        res.append(ctx.track(depth, mask, radius, seed=21, particles=16, generations=6,
                             init_center=c0, init_radius=r0))
        ctx.close()
    for a, b in zip(res[0], res[1]):
        assert np.array_equal(a, b)
