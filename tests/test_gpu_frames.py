"""Next row f2: frame-batched scoring, M observation frames x n poses per call
(hp_set_observations + hp_eval_costs_frames), against the fp64 oracle frame by frame and
bitwise against single-frame scoring.  Observations are the oracle's renders."""
import numpy as np
import pytest

import oracle as O
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2005_07068_b200 as hp  # noqa: E402
from parity_check import check_sample  # noqa: E402

E_REL, E_ABS = 1e-5, 2.5e-5

TRUTHS = ["h_A", "fist", "spread"]


def _frames(w, h, names=TRUTHS):
    cam = O.camera(w, h)
    obs = [O.synthesize(W.NAMED[n], cam) for n in names]
    depth = np.stack([o.depth for o in obs]).astype(np.float32)
    mask = np.stack([o.mask for o in obs]).astype(np.uint8)
    return obs, depth, mask


def _poses(names, n, seed):
    """n poses per frame: the frame's truth, the next frame's truth, perturbed truths and
    random in-bounds poses."""
    rng = np.random.default_rng(seed)
    out = []
    for k, name in enumerate(names):
        t = np.asarray(W.NAMED[name], np.float64)
        blk = [t, np.asarray(W.NAMED[names[(k + 1) % len(names)]], np.float64)]
        while len(blk) < n // 2:
            d = rng.normal(size=26) * np.r_[[10.0] * 3, [np.radians(5)] * 3, [np.radians(8)] * 20]
            blk.append(t + d)
        blk += list(W.random_poses(seed + k, n - len(blk)))
        out.append(np.asarray(blk[:n], np.float32))
    return np.stack(out)


def _check_frame(obs, poses, sums, c64, w, h):
    p64 = np.asarray(poses, np.float64)
    co, so, _, _ = O.eval_batch(p64, obs, with_sums=True)
    check_sample(sums, c64, so, co, p64, range(len(co)), O.camera(w, h), obs,
                 max_edge=0.1 * len(co) + 1)


@pytest.mark.parametrize("n", [13, 160])  # split path (S > 1) and batch path (S = 1)
def test_frames_match_oracle_per_frame(n):
    w, h = 160, 120
    obs, depth, mask = _frames(w, h)
    ctx = hp.Context(w, h, max_particles=1024)
    ctx.set_observations(depth, mask)
    poses = _poses(TRUTHS, n, seed=11)
    P = torch.tensor(poses, device="cuda")
    sums, c64 = ctx.eval_sums_frames(P)
    c32 = ctx.eval_costs_frames(P)
    torch.cuda.synchronize()
    sums, c64, c32 = sums.cpu().numpy(), c64.cpu().numpy(), c32.cpu().numpy()
    for f in range(len(TRUTHS)):
        _check_frame(obs[f], poses[f], sums[f], c64[f], w, h)
        assert np.array_equal(c32[f], c64[f].astype(np.float32))
    # each frame's truth (pose 0) is near that frame's optimum; the next frame's truth
    # (pose 1) scored against this frame is not
    for f in range(len(TRUTHS)):
        assert c64[f, 0] < 1e-3  # fp32 copy of the fp64 truth
        assert c64[f, 1] > 1.0


def test_frames_bitwise_equal_single_frame_640():
    """Frame batching changes nothing but the observation each pose is scored against."""
    w, h = 640, 480
    names = ["h_A", "point", "flat", "toward_camera"]
    _, depth, mask = _frames(w, h, names)
    n = 600
    sw = W.swarm_c4(n * len(names)).astype(np.float32).reshape(len(names), n, 26)
    ctx = hp.Context(w, h, max_particles=4096)
    P = torch.tensor(sw, device="cuda")
    ctx.set_observations(depth, mask)
    batched = ctx.eval_costs_frames(P).cpu().numpy()
    batched_s, _ = ctx.eval_sums_frames(P)
    batched_s = batched_s.cpu().numpy()
    for f in range(len(names)):
        ctx.set_observation(depth[f], mask[f])
        single = ctx.eval_costs(P[f].contiguous()).cpu().numpy()
        s_single, _ = ctx.eval_sums(P[f].contiguous())
        assert np.array_equal(batched[f], single), f
        assert np.array_equal(batched_s[f], s_single.cpu().numpy()), f


def test_frames_device_upload_and_frame0_default():
    w, h = 160, 120
    obs, depth, mask = _frames(w, h)
    ctx = hp.Context(w, h, max_particles=256)
    ctx.set_observations(torch.tensor(depth, device="cuda"), torch.tensor(mask, device="cuda"))
    poses = _poses(TRUTHS, 20, seed=3)
    P = torch.tensor(poses, device="cuda")
    from_dev = ctx.eval_costs_frames(P).cpu().numpy()
    # plain hp_eval_costs scores frame 0
    c0 = ctx.eval_costs(P[1].contiguous()).cpu().numpy()
    ctx.set_observation(depth[0], mask[0])
    ref0 = ctx.eval_costs(P[1].contiguous()).cpu().numpy()
    assert np.array_equal(c0, ref0)
    ctx.set_observations(depth, mask)
    assert np.array_equal(ctx.eval_costs_frames(P).cpu().numpy(), from_dev)


def test_frames_edge_cases():
    w, h = 160, 120
    _, depth, mask = _frames(w, h)
    ctx = hp.Context(w, h, max_particles=64)
    ctx.set_observations(depth, mask)
    P = torch.zeros((3, 0, 26), dtype=torch.float32, device="cuda")
    assert ctx.eval_costs_frames(P).shape == (3, 0)  # n = 0: no-op
    P = torch.zeros((3, 22, 26), dtype=torch.float32, device="cuda")  # 66 > max_particles
    with pytest.raises(hp.HPError):
        ctx.eval_costs_frames(P)
    with pytest.raises(AssertionError):
        ctx.set_observations(depth[:, :10], mask[:, :10])
    # the poses' frame count must be the observation's (binding and C ABI both check)
    P2 = torch.zeros((2, 5, 26), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        ctx.eval_costs_frames(P2)
    out = torch.empty((3, 5), dtype=torch.float32, device="cuda")
    st = ctx._L.hp_eval_costs_frames(ctx.handle, P2.data_ptr(), 2, 5, out.data_ptr(), None)
    assert st == hp.hp.HP_ERR_INVALID_ARG
    with pytest.raises(ValueError):
        ctx.eval_costs_frames(torch.zeros((3, 5, 26), dtype=torch.float32, device="cuda"),
                              out=torch.empty((3, 4), dtype=torch.float32, device="cuda"))


def test_frames_growth_keeps_fit_graph_valid():
    """Growing the frame buffers re-encodes the tensor map; a fit captured before must not
    keep reading the freed buffer (the cached graph is rebuilt)."""
    w, h = 160, 120
    _, depth, mask = _frames(w, h)
    ctx = hp.Context(w, h, max_particles=64)
    ctx.set_observation(depth[0], mask[0])
    c, r = W.local_init_box()
    a = ctx.pso_fit(seed=5, particles=16, generations=6, init_center=c, init_radius=r)
    ctx.set_observations(depth, mask)   # frame 0 unchanged, buffers regrown
    b = ctx.pso_fit(seed=5, particles=16, generations=6, init_center=c, init_radius=r)
    assert a.best_cost == b.best_cost and np.array_equal(a.best_pose, b.best_pose)
