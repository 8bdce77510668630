"""Particle-sharded mode on the GPU (-m gpu): a world-1 NCCL communicator exercises the
whole sharded code path (slice, in-place allgather, replicated update + bookkeeping) and
must reproduce the unsharded results bit for bit (SURVEY §8(e) invariant)."""
import os

import numpy as np
import pytest

import oracle as O
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2005_07068_b200 as hp  # noqa: E402


def _ctx(w, h, n, shard):
    c = hp.Context(w, h, max_particles=n)
    obs = O.synthesize(W.H_A, O.camera(w, h))
    c.set_observation(obs.depth, obs.mask)
    if shard:
        assert hp.hp.nccl_available() or True
        c.shard(0, 1, nccl_id=hp.hp.nccl_unique_id())
    return c


def test_sharded_eval_equals_unsharded():
    a = _ctx(320, 240, 512, False)
    b = _ctx(320, 240, 512, True)
    P = torch.tensor(W.swarm_c4(300).astype(np.float32), device="cuda")
    ca = a.eval_costs(P).cpu().numpy()
    cb = b.eval_costs(P).cpu().numpy()
    assert np.array_equal(ca, cb)


def test_sharded_fit_equals_unsharded_fused_fit():
    a = _ctx(160, 120, 64, False)
    b = _ctx(160, 120, 64, True)
    c, r = W.local_init_box()
    fa = a.pso_fit(seed=3, particles=32, generations=9, init_center=c, init_radius=r)
    fb = b.pso_fit(seed=3, particles=32, generations=9, init_center=c, init_radius=r)
    assert np.array_equal(fa.best_pose, fb.best_pose)
    assert np.array_equal(fa.trace, fb.trace)
    Xa, Va, Pa, Pca = a.pso_state(32)
    Xb, Vb, Pb, Pcb = b.pso_state(32)
    assert np.array_equal(Xa, Xb) and np.array_equal(Va, Vb) and np.array_equal(Pca, Pcb)


# ---------------------------------------------------------------- loopback ranks (debug build)
def _loopback_ranks(world, w, h, max_particles, fn, group):
    """Run fn(ctx, rank) on `world` contexts of the debug loopback build (libhp_loopback.so,
    hp_shard_loopback), each on its own host thread and CUDA stream — the sharded code paths
    with rank > 0 on one GPU.  Returns the per-rank results."""
    import threading

    from paper_2005_07068_b200 import build as hpbuild

    path = hpbuild.LOOPBACK_LIB
    assert os.path.exists(path), "build it with __graft_entry__.build()"
    obs = O.synthesize(W.H_A, O.camera(w, h))
    ctxs = []
    for r in range(world):
        c = hp.Context(w, h, max_particles=max_particles, lib_path=path)
        c.set_observation(obs.depth, obs.mask)
        ctxs.append(c)
    out, errs = [None] * world, []

    def run(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                ctxs[r].shard_loopback(group, r, world)
                out[r] = fn(ctxs[r], r)
                torch.cuda.current_stream().synchronize()
        except Exception as e:  # pragma: no cover - reported below
            errs.append((r, repr(e)))

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    for c in ctxs:
        c.close()
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_loopback_sharded_eval_equals_world1(world):
    """Rank r scores poses [r ceil(N/W), ...) into its chunk and the allgather at NCCL's
    offsets returns all N costs on every rank — N = 301 leaves a padded last chunk; bitwise
    equal to the unsharded call, device and host paths."""
    n = 301
    P = W.swarm_c4(n).astype(np.float32)
    ref = _ctx(320, 240, 512, False).eval_costs(torch.tensor(P, device="cuda")).cpu().numpy()

    def fn(ctx, r):
        dev = ctx.eval_costs(torch.tensor(P, device="cuda")).cpu().numpy()
        host = ctx.eval_costs_host(P)
        return dev, host

    res = _loopback_ranks(world, 320, 240, 256, fn, f"eval{world}")
    for dev, host in res:
        assert np.array_equal(dev, ref) and np.array_equal(host, ref)


@pytest.mark.parametrize("world", [2, 3])
def test_loopback_sharded_fit_equals_unsharded_and_oracle(world):
    """The sharded fit (every rank updates all particles, scores its slice, allgathers the
    costs, runs the identical bookkeeping) on 2 / 3 loopback ranks: every rank returns the
    unsharded fused fit's bits, and the C1 fit matches the oracle (P:L162 particle
    parallelism)."""
    w, h = 160, 120
    c, r = W.local_init_box()
    a = _ctx(w, h, 64, False)
    fa = a.pso_fit(seed=7, particles=16, generations=10, init_center=c, init_radius=r)
    Xa, Va, Pa, Pca = a.pso_state(16)

    def fn(ctx, rank):
        f = ctx.pso_fit(seed=7, particles=16, generations=10, init_center=c, init_radius=r)
        return f, ctx.pso_state(16)

    res = _loopback_ranks(world, w, h, 64, fn, f"fit{world}")
    for f, (X, V, P, Pc) in res:
        assert np.array_equal(f.best_pose, fa.best_pose) and np.array_equal(f.trace, fa.trace)
        assert np.array_equal(X, Xa) and np.array_equal(V, Va) and np.array_equal(Pc, Pca)
    obs = O.synthesize(W.H_A, O.camera(w, h))
    o = O.pso_fit_hand(obs, O.default_pso(seed=7, particles=16, generations=10), c, r)
    assert np.max(np.abs(fa.best_pose - o.best_x)) <= 1e-4
