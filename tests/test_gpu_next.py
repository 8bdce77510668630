"""The next rows of SURVEY §8(f) on the GPU (-m gpu), to the same parity bar:
f4 — cost / PSO variants behind flags (literal Eq. 4 clamp at d_m, SPEC's 15-degree kc rest
separation, per-dimension r1/r2, other mutation schedules);
f1 — temporal tracking over a synthetic motion sequence (warm start from the previous
frame's best pose)."""
import math

import numpy as np
import pytest

import oracle as O
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2005_07068_b200 as hp  # noqa: E402

E_REL, E_ABS = 1e-5, 2.5e-5


@pytest.mark.parametrize("flags", [dict(clamp_at_dm=1), dict(kc_rest=math.radians(15)),
                                   dict(lambda_=10.0, lambda_k=3.0, depth_scale=1.0),
                                   dict(d_m=5.0, d_M=20.0)])
def test_cost_flag_variants_match_oracle(flags):
    w, h = 160, 120
    ctx = hp.Context(w, h, max_particles=64, cost=hp.default_cost(**flags))
    ocp = O.default_cost(**flags)
    obs = O.synthesize(W.H_A, O.camera(w, h))
    ctx.set_observation(obs.depth, obs.mask)
    poses = np.concatenate([W.random_poses(77, 30), np.stack(list(W.NAMED.values()))])
    poses = poses.astype(np.float32)
    sums, c64 = ctx.eval_sums(torch.tensor(poses, device="cuda"))
    sums, c64 = sums.cpu().numpy(), c64.cpu().numpy()
    co, so, kco, _ = O.eval_batch(poses.astype(np.float64), obs, cp=ocp, with_sums=True)
    n_clean = 0
    for i in range(len(co)):
        if int(sums[i, 0]) == so[i].s_rm and int(sums[i, 1]) == so[i].s_and and \
                int(sums[i, 3]) == so[i].n_both:
            n_clean += 1
            tol = E_REL * abs(co[i]) + E_ABS * max(1.0, ocp.depth_scale / 0.1)
            assert abs(c64[i] - co[i]) <= tol, (i, c64[i], co[i])
    assert n_clean >= 0.9 * len(co)


@pytest.mark.parametrize("kw", [dict(per_dim_r=1, mutation_period=2, mutation_fraction=0.25),
                                dict(per_dim_r=0, mutation_period=1, mutation_fraction=1.0),
                                dict(per_dim_r=1, mutation_period=5, mutation_fraction=0.0,
                                     c1=2.05, c2=2.05)])
def test_pso_flag_variants_bitwise(kw):
    ctx = hp.Context(160, 120, max_particles=64)
    D = 26
    lo, hi = O.bounds()
    centre = (lo + hi) / 2 + 0.1
    g = ctx.debug_pso_sphere(D, lo, hi, lo, hi, 6, 26, centre, seed=11, particles=24,
                             generations=8, **kw)
    r = O.pso_sphere(D, lo, hi, lo, hi, 6, 26, centre,
                     O.default_pso(seed=11, particles=24, generations=8, **kw))
    assert np.array_equal(g.best_pose, r.best_x) and np.array_equal(g.trace, r.trace)


def test_hand_fit_per_dim_r_matches_oracle():
    w, h = 160, 120
    ctx = hp.Context(w, h, max_particles=64)
    obs = O.synthesize(W.H_A, O.camera(w, h))
    ctx.set_observation(obs.depth, obs.mask)
    c, rad = W.local_init_box()
    g = ctx.pso_fit(seed=4, particles=16, generations=8, per_dim_r=True, init_center=c,
                    init_radius=rad)
    r = O.pso_fit_hand(obs, O.default_pso(seed=4, particles=16, generations=8, per_dim_r=1),
                       c, rad)
    assert np.max(np.abs(g.best_pose - r.best_x)) <= 1e-4
    np.testing.assert_allclose(g.trace, r.trace, rtol=E_REL, atol=E_ABS)


def test_tracking_sequence_matches_oracle():
    """f1 (C5 at desk scale): 4 frames of the seeded motion at 160x120, 16 x 6 per frame,
    warm start at the previous best +- (15 mm, 8 deg wrist, 20 deg fingers)."""
    w, h, F, N, K = 160, 120, 4, 16, 6
    cam = O.camera(w, h)
    seq = W.motion_sequence(frames=100)[:F]
    obs = [O.synthesize(hf, cam) for hf in seq]
    depth = np.stack([o.depth for o in obs])
    mask = np.stack([o.mask for o in obs])
    radius = np.array([15.0] * 3 + [math.radians(8)] * 3 + [math.radians(20)] * 20)
    c0, r0 = seq[0], np.array([40.0] * 3 + [math.radians(15)] * 3 + [math.pi] * 20)
    ctx = hp.Context(w, h, max_particles=64)
    poses, costs, traces = ctx.track(depth, mask, radius, seed=21, particles=N, generations=K,
                                     init_center=c0, init_radius=r0)
    centre, rad = c0, r0
    for f in range(F):
        r = O.pso_fit_hand(obs[f], O.default_pso(seed=21 + f, particles=N, generations=K),
                           centre, rad)
        assert np.max(np.abs(poses[f] - r.best_x)) <= 1e-4, f
        assert abs(costs[f] - r.best_cost) <= E_REL * abs(r.best_cost) + E_ABS
        np.testing.assert_allclose(traces[f], r.trace, rtol=E_REL, atol=E_ABS)
        centre, rad = r.best_x, radius
    # frame 0 starts from the motion truth's neighbourhood: the fit beats a cold start
    assert costs[0] < 25.0


def test_timing_hooks_and_two_contexts_on_two_streams():
    """hp_set_timing / hp_last_kernel_ms (bench's roofline leg) and the pipelined mode: two
    contexts driven on two streams concurrently give the single-context results."""
    import paper_2005_07068_b200 as hp

    ctx = hp.Context(320, 240, max_particles=2048)
    obs = O.synthesize(W.H_A, O.camera(320, 240))
    ctx.set_observation(obs.depth, obs.mask)
    P = torch.tensor(W.swarm_c4(1500).astype(np.float32), device="cuda")
    with pytest.raises(hp.HPError):
        ctx.last_kernel_ms()  # nothing timed yet
    ctx.set_timing(True)
    ref = ctx.eval_costs(P).cpu().numpy()
    fk_ms, render_ms = ctx.last_kernel_ms()
    assert ctx.last_launch_count() == 3 and fk_ms > 0 and render_ms > 0
    ctx.set_timing(False)
    ctx2 = hp.Context(320, 240, max_particles=2048)
    ctx2.set_observation(obs.depth, obs.mask)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    outs = [torch.empty(1500, device="cuda") for _ in range(6)]
    for k in range(6):
        (ctx if k % 2 == 0 else ctx2).eval_costs(P, out=outs[k], stream=sa if k % 2 == 0 else sb)
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(o.cpu().numpy(), ref)


def test_context_create_destroy_releases_device_memory():
    """hp_destroy frees everything hp_create and the calls allocated (frames, fit graphs)."""
    import paper_2005_07068_b200 as hp

    def cycle():
        ctx = hp.Context(320, 240, max_particles=1024)
        obs = O.synthesize(W.H_A, O.camera(320, 240))
        ctx.set_observations(np.stack([obs.depth] * 3), np.stack([obs.mask] * 3))
        ctx.eval_costs(torch.tensor(W.swarm_c4(600).astype(np.float32), device="cuda"))
        c, r = W.local_init_box()
        ctx.pso_fit(seed=1, particles=16, generations=3, init_center=c, init_radius=r)
        torch.cuda.synchronize()
        ctx.close()

    cycle()  # first use: lazy module / driver allocations
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(5):
        cycle()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < 16 << 20, (free0, free1)  # no per-context leak
