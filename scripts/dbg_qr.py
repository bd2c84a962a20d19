"""Debug aid: per-block QR factor check + iteration counts for small random SUR problems."""
import numpy as np
import oracle
from paper_2510_14471_b200 import api, synth

for p in (synth.random_sur(3, 200, [5, 7, 4], seed=21), synth.random_sur(4, 300, [3, 6, 8, 2], seed=22),
          synth.make_problem(0), synth.random_sur(2, 700, [5, 32], seed=3), synth.random_sur(2, 1500, [3, 17], seed=4)):
    sur = api.sur_from_problem(p)
    op = api.sur_preconditioner(sur)
    Q, R = op.factors()
    nb = np.asarray(p.nb); offs = np.concatenate([[0], np.cumsum(nb)])
    roff = np.concatenate([[0], np.cumsum(nb * nb)])
    errs = []
    for b in range(len(nb)):
        n = nb[b]
        Qb = Q[:, offs[b]:offs[b + 1]]
        Rb = R[roff[b]:roff[b + 1]].reshape(n, n, order="F")
        Xb = p.X[:, offs[b]:offs[b + 1]]
        errs.append((np.abs(Qb.T @ Qb - np.eye(n)).max(), np.abs(Qb @ Rb - Xb).max() / np.abs(Xb).max(),
                     np.abs(np.tril(Rb, -1)).max()))
    o = oracle.solve(p, "oracle", cfg=oracle.make_config(tol_rel=1e-6))
    g = api.pcg_aug(sur, op, config=api.PcgConfig(tol_rel=1e-6))
    print(p.G, p.M, list(nb), "orth/recon/tril", [tuple(f"{x:.1e}" for x in e) for e in errs],
          "iters gpu", g.solution.iterations, "oracle", o.iterations)
