"""Write profiles/walg.json: the algorithmic work per hypothesis of each bench
workload, computed by the ORACLE's or_walg (FK + exact projected boxes x frozen per-kind
FLOP counts).  bench.py reads the stored figure; it never executes the oracle for this.

    python scripts/walg.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import workloads as W  # noqa: E402


def mean_walg(poses, cam):
    w = np.array([O.walg(p, cam) for p in poses])
    return {"flops_per_hyp": float(w[:, 0].mean()), "tests_per_hyp": float(w[:, 1].mean()),
            "union_px_per_hyp": float(w[:, 2].mean()), "poses": int(len(poses))}


def main():
    out = {"definition": "DESIGN.md §5: W_alg = sum_prims |box| F_kind + |union box| F_px; "
                         "F_sphere 20, F_ellipsoid 48, F_cone 56, F_px 15 (FMA = 2)"}
    cam = O.camera(640, 480)
    # C4: every rank's slice comes from swarm_c4(4096 * world); the union over 8 ranks
    sw = W.swarm_c4(4096 * 8)
    out["c4_640x480"] = mean_walg(np.asarray(np.asarray(sw, np.float32), np.float64), cam)
    out["c4_640x480_rank0_4096"] = mean_walg(
        np.asarray(np.asarray(W.swarm_c4(4096), np.float32), np.float64), cam)
    out["h_A_640x480"] = mean_walg(W.H_A[None], cam)
    for res in ("160x120", "320x240"):
        out[f"h_A_{res}"] = mean_walg(W.H_A[None], O.camera(*W.RESOLUTIONS[res]))
    # C3: every pose a 64 x 40 fit evaluates (the oracle's PSO on the oracle's costs, local
    # init box, seeds 1 and 2; bench.py's pso_fit leg divides it by the fit's time)
    obs = O.synthesize(W.H_A, cam)
    lo, hi = O.bounds()
    c, rad = W.local_init_box()
    ilo, ihi = np.maximum(lo, c - rad), np.minimum(hi, c + rad)
    seen = []

    def objective(X):
        seen.append(np.array(X))
        return O.eval_batch(X, obs)

    for seed in (1, 2):
        O.pso_run(26, lo, hi, ilo, ihi, 6, 26,
                  O.default_pso(seed=seed, particles=64, generations=40), objective)
    out["c3_fit_640x480"] = mean_walg(np.concatenate(seen), cam)
    path = os.path.join(ROOT, "profiles", "walg.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
