"""Write tests/golden/pso_eq6_hand.txt: hand-derived PSO trajectories that pin or_pso_run's
Eq. 6 coefficient / random-number assignment and both mutation orders (AMB-17).

Every step is written out for the specific scenario (straight-line arithmetic, no loop
over a generic PSO): the velocity update of Eq. 6, v = w (v + c1 r1 (P - x) + c2 r2 (G - x))
(Eq. 6), in DESIGN §4's operation order, then Eq. 7, x = x + v.
The random numbers come from the KAT-pinned Philox (oracle.philox / oracle.u01; layout
DESIGN §4: counter (particle, dim, generation, tag), r1 = u(w0, w1), r2 = u(w2, w3)) and w
from the closed-form-pinned oracle.constriction.  Only oracle/ is called.

    python scripts/gen_golden_pso.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

SEED = 20250
C1, C2 = 2.8, 1.3
KEY = [SEED & 0xFFFFFFFF, SEED >> 32]


def words(i, d, k, tag):
    return O.philox([i, d, k, tag], KEY)


def u(i, d, k, tag, pair=0):
    w = words(i, d, k, tag)
    return O.u01(w[2 * pair], w[2 * pair + 1])


def main():
    w = O.constriction(C1, C2)
    lines = [
        "# Hand-derived PSO trajectories (scripts/gen_golden_pso.py; only oracle.philox, u01 and",
        "# constriction are called).  Eq. 6 (P:L140/L144): v = w (v + c1 r1 (P - x) + c2 r2 (G - x)),",
        "# Eq. 7 (P:L142): x = x + v; c1 = 2.8, c2 = 1.3 (P:L150); w = 2/|2 - psi - sqrt(psi^2 - 4 psi)|.",
        "# RNG layout DESIGN §4: Philox4x32-10 key (seed_lo, seed_hi), counter (particle, dim,",
        "# generation, tag): tag 0 init (u(w0,w1)), tag 1 r1 = u(w0,w1) / r2 = u(w2,w3), tag 2 mutation.",
        f"seed {SEED}",
        f"w {w!r}",
    ]
    # ---------------- scenario A: D = 1, N = 2, no mutation, costs by generation
    # bounds [-100, 100], init box [-10, 10]; costs: gen 0 (1, 2), gen 1 (1, 5), gen 2 (0.5, 5)
    x0 = -10.0 + u(0, 0, 0, 0) * 20.0
    x1 = -10.0 + u(1, 0, 0, 0) * 20.0
    # gen 0: P = x, v = 0, G = particle 0 (cost 1 < 2)
    G = x0
    # k = 1.  particle 0: P = G = x -> every term is 0, it stays.
    r1_11, r2_11 = u(1, 0, 1, 1, 0), u(1, 0, 1, 1, 1)
    # particle 1: P - x = 0 (P = its initial position), so only c2 r2 (G - x) acts
    a = C1 * r1_11
    b = x1 - x1
    t1 = a * b
    t2 = 0.0 + t1
    c = C2 * r2_11
    e = G - x1
    t3 = c * e
    t4 = t2 + t3
    v1 = w * t4
    x1_1 = x1 + v1
    lines += [
        "# scenario A: D = 1, N = 2, bounds [-100, 100], init [-10, 10], mutation off;",
        "# objective returns (1, 2) at gen 0, (1, 5) at gen 1, (0.5, 5) at gen 2.",
        "# gen 0: G = particle 0.  k = 1: particle 0 has P = G = x (stays put); particle 1 has",
        "# P = x, so v = w c2 r2 (G - x) -- the c2/r2 pin.  Gen 1's costs improve nobody, so at",
        "# k = 2 particle 1's P - x = -v1 != 0 and the c1 r1 term acts -- the c1/r1 pin.",
        f"A.x0_init {x0!r}",
        f"A.x1_init {x1!r}",
        f"A.r1[1,1] {r1_11!r}",
        f"A.r2[1,1] {r2_11!r}",
        f"A.K2.X {x0!r} {x1_1!r}",
        f"A.K2.V 0.0 {v1!r}",
        f"A.K2.P {x0!r} {x1!r}",
        f"A.K2.Pcost 1.0 2.0",
    ]
    r1_12, r2_12 = u(1, 0, 2, 1, 0), u(1, 0, 2, 1, 1)
    a = C1 * r1_12
    b = x1 - x1_1          # P (not improved at gen 1) - x
    t1 = a * b
    t2 = v1 + t1
    c = C2 * r2_12
    e = G - x1_1
    t3 = c * e
    t4 = t2 + t3
    v2 = w * t4
    x1_2 = x1_1 + v2
    for x in (x0, x1, x1_1, x1_2):
        assert -100.0 < x < 100.0  # no clamping in this scenario
    lines += [
        f"A.r1[1,2] {r1_12!r}",
        f"A.r2[1,2] {r2_12!r}",
        # gen 2: particle 0 improves to 0.5 at the same position; particle 1 does not
        f"A.K3.X {x0!r} {x1_2!r}",
        f"A.K3.V 0.0 {v2!r}",
        f"A.K3.P {x0!r} {x1!r}",
        f"A.K3.Pcost 0.5 2.0",
        f"A.K3.trace 1.0 1.0 0.5",
    ]
    # ---------------- scenario B: D = 2, N = 2, mutation every generation of the worst half
    # (1 particle) in dim 1; bounds [-100, 100]^2, init [-10, 10]^2; costs (1, 2), (1, 5), (0.5, 5)
    xb0 = [-10.0 + u(0, d, 0, 0) * 20.0 for d in range(2)]
    xb1 = [-10.0 + u(1, d, 0, 0) * 20.0 for d in range(2)]
    # k = 1 update: particle 0 stays; particle 1 (P = x): v_d = w c2 r2 (G_d - x_d), r at dim 0
    r2b = u(1, 0, 1, 1, 1)
    vb = []
    xb1_1 = []
    for d in range(2):
        t1 = (C1 * u(1, 0, 1, 1, 0)) * (xb1[d] - xb1[d])
        t2 = 0.0 + t1
        t3 = (C2 * r2b) * (xb0[d] - xb1[d])
        vb.append(w * (t2 + t3))
        xb1_1.append(xb1[d] + vb[-1])
    mut = -100.0 + u(1, 1, 1, 2) * 200.0  # particle 1 is the worst (Pcost 2 > 1) at k = 1
    lines += [
        "# scenario B: D = 2, N = 2, bounds [-100, 100]^2, init [-10, 10]^2, mutation period 1,",
        "# fraction 0.5 (the worse particle), mutation dims [1, 2); costs as scenario A.",
        "# order 0 (AMB-17): at k = 1 particle 1 is updated, then dim 1 re-drawn (v = 0) and",
        "# evaluated as drawn.  order 1 (SPEC S:L447): at k = 1 it is updated and evaluated, then",
        "# re-drawn; at k = 2 the update moves the re-drawn particle before its evaluation.",
        f"B.u_mut[1,1,1] {u(1, 1, 1, 2)!r}",
        f"B.order0.K2.X {xb0[0]!r} {xb0[1]!r} {xb1_1[0]!r} {mut!r}",
        f"B.order0.K2.V 0.0 0.0 {vb[0]!r} 0.0",
    ]
    # order 1, K = 3: after k = 1's bookkeeping particle 1 (Pcost 2) is re-drawn in dim 1
    xm = [xb1_1[0], mut]
    vm = [vb[0], 0.0]
    r1c, r2c = u(1, 0, 2, 1, 0), u(1, 0, 2, 1, 1)
    xb1_2, vb2 = [], []
    for d in range(2):
        t1 = (C1 * r1c) * (xb1[d] - xm[d])   # P = initial position (never improved)
        t2 = vm[d] + t1
        t3 = (C2 * r2c) * (xb0[d] - xm[d])
        vb2.append(w * (t2 + t3))
        xb1_2.append(xm[d] + vb2[-1])
    for x in xb0 + xb1 + xb1_1 + xb1_2 + [mut]:
        assert -100.0 < x < 100.0
    lines += [
        f"B.order1.K3.X {xb0[0]!r} {xb0[1]!r} {xb1_2[0]!r} {xb1_2[1]!r}",
        f"B.order1.K3.V 0.0 0.0 {vb2[0]!r} {vb2[1]!r}",
    ]
    out = os.path.join(ROOT, "tests", "golden", "pso_eq6_hand.txt")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print(out)


if __name__ == "__main__":
    main()
