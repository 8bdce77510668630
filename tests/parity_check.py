"""Shared GPU-vs-oracle comparison of one scored pose (DESIGN §6 tolerances).

Pure test logic: the GPU's integer sums and cost against the oracle's for the same pose and
observation; nothing here computes the method (the oracle's own cost_from_sums and kc turn
sums into a cost)."""
import numpy as np

import oracle as O

E_REL, E_ABS = 1e-5, 2.5e-5


def check_pose(sums_g, c64_g, so, co, pose, cam, obs, cp=None, e_abs=E_ABS, pose_f32=True):
    """One pose, GPU vs oracle.  Returns True when the integer sums agree exactly (then the
    cost is within E_REL/E_ABS); otherwise the pose is an "edge" pose: every differing count
    must be explained by oracle-flagged edge pixels, the numerator may move by at
    most d_M per such pixel plus the fp32 depth bound per both-defined pixel, and the GPU
    cost must be Eq. 4-5 of the GPU's own sums (so the cost difference is bounded by those
    pixel flips and nothing else).  pose_f32: the GPU scored the fp32 rounding of `pose`
    (hp_eval_costs / hp_eval_sums); False for fp64 poses (hp_eval_sums_f64)."""
    cp = cp or O.default_cost()
    num_g = sums_g[2] / 2.0 ** 20
    exact = int(sums_g[0]) == so.s_rm and int(sums_g[1]) == so.s_and and int(sums_g[3]) == so.n_both
    if exact and abs(c64_g - co) <= E_REL * abs(co) + e_abs and \
            abs(num_g - so.num) <= 2.5e-4 * max(so.n_both, 1) + 1e-6:
        return True
    # counts differ, or the counts agree but a pixel on an INTERNAL occlusion edge (one
    # primitive's silhouette crossing another) took the other primitive's depth: both are
    # edge pixels by the oracle's definition, and the numerator may move by d_M at each
    p = np.asarray(np.asarray(pose, np.float32) if pose_f32 else pose, np.float64)
    ne = int(O.edge_mask(p, cam, obs_depth=obs.depth, d_m=cp.d_m).sum())
    assert ne > 0, "sums differ but the oracle flags no edge pixel"
    assert abs(int(sums_g[0]) - so.s_rm) <= ne
    assert abs(int(sums_g[1]) - so.s_and) <= ne
    assert abs(int(sums_g[3]) - so.n_both) <= ne
    clampv = cp.d_m if cp.clamp_at_dm else cp.d_M
    assert abs(num_g - so.num) <= ne * clampv + 2.5e-4 * max(so.n_both, 1) + 1e-6
    s = O.Sums(so.s_o, so.s_o + int(sums_g[0]) - int(sums_g[1]), int(sums_g[1]), int(sums_g[0]),
               int(sums_g[3]), num_g)
    e_own, _ = O.cost_from_sums(s, cp, O.kc(p, cp.kc_rest))
    assert abs(c64_g - e_own) <= E_REL * abs(e_own) + e_abs, (c64_g, e_own)
    return False


def check_sample(sums, c64, so, co, poses, idx, cam, obs, max_edge=None, cp=None, e_abs=E_ABS,
                 pose_f32=True):
    """Poses idx of a GPU batch against the oracle's results so[k], co[k] for idx[k]."""
    n_edge = 0
    for k, i in enumerate(idx):
        n_edge += not check_pose(sums[i], c64[i], so[k], co[k], poses[i], cam, obs, cp, e_abs,
                                 pose_f32)
    if max_edge is not None:
        assert n_edge <= max_edge, (n_edge, len(idx))
    return n_edge
