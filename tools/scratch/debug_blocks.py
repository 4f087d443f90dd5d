import sys, numpy as np, torch, time
sys.path.insert(0, '.')
import workloads as W, paper_2204_05536_b200 as h2d
name = sys.argv[1] if len(sys.argv) > 1 else 'c3'
cfg = W.CONFIGS[name]
pts = W.config_points(cfg)
t = time.time()
op = h2d.Hodlr2d.build(torch.from_numpy(pts).cuda(), cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale, shift=cfg.shift, box_lo=cfg.box_lo, box_side=cfg.box_side)
torch.cuda.synchronize(); print('build', time.time() - t)
inf = op.info()
print({k: inf[k] for k in ('kappa', 'rank_max', 'u_values', 'v_values', 'tree_seconds', 'aca_seconds', 'pack_seconds', 'build_seconds', 'truncated')})
perm, ls = op.tree()
P = pts[perm]
kappa = inf['kappa']
rng = np.random.default_rng(0)
def K(A, B):
    d = A[:, None, :] - B[None, :, :]
    r2 = (d ** 2).sum(-1)
    if cfg.kernel == 0:
        return cfg.scale * np.where(r2 > 0, 0.5 * np.log(np.where(r2 > 0, r2, 1)), 0)
    return cfg.scale / np.sqrt(1 + r2 / cfg.c ** 2)
for l in range(1, kappa + 1):
    off, col = op.lists(l)
    ranks = op.ranks(l)
    sh = 2 * (kappa - l)
    errs = []
    nb = len(col)
    for e in rng.choice(nb, min(nb, 6), replace=False):
        X = np.searchsorted(off, e, side='right') - 1
        Y = col[e]
        r0, r1 = ls[X << sh], ls[(X + 1) << sh]
        c0, c1 = ls[Y << sh], ls[(Y + 1) << sh]
        rs = np.sort(rng.choice(r1 - r0, min(r1 - r0, 300), replace=False))
        cs = np.sort(rng.choice(c1 - c0, min(c1 - c0, 300), replace=False))
        U, V = op.block(l, int(e))
        A = K(P[r0 + rs], P[c0 + cs])
        Ap = U[rs] @ V[cs].T
        errs.append((int(e), int(ranks[e]), float(np.linalg.norm(A - Ap) / np.linalg.norm(A))))
    print(l, 'rmax', ranks.max(), 'mean', ranks.mean(), errs)
