"""CPU verification of the exact pruning plan (wt_prune_plan, host-only):
every config the plan drops from a (tile class, wave row, L bucket) cell is
strictly slower -- in the reference's own fp64 evaluation order -- than some
config the plan keeps, at the cell's corners and at random interior and far
points.  So a dropped config can never be the argmin nor tie with it."""
import numpy as np
import pytest

import wtutil as U


def f_ref(th, g, l):
    """BilinearCoeffs::predict (model.hpp:20-23) in binary64, no FMA."""
    t = th[..., 0] * g
    t = t * l
    t = t + th[..., 1] * g
    t = t + th[..., 2] * l
    return t + th[..., 3]


def rows_of(tables, C, W):
    th = tables["coeff_theta"].reshape(C, W, 4)
    te = tables["theta_ext"].reshape(C, 1, 4)
    return np.concatenate([th, te], 1)  # [C, R = W + 1, 4]


def check_plan(tables, cfg, n_sm=148, seed=0):
    from paper_2604_10187_b200 import capi

    plan = capi.prune_plan(tables, U.registry_arrays_of(cfg), n_sm)
    C, W, R = len(cfg["id"]), int(tables["W"][0]), plan["R"]
    assert R == W + 1
    rows = rows_of(tables, C, W)
    order = np.argsort(np.asarray(tables["macro_id"]), kind="stable")  # config index = ascending macro id
    rows = rows[order]
    tiles = np.stack([np.asarray(cfg[k])[order] for k in ("t_m", "t_n", "t_k")], 1)
    rng = np.random.default_rng(seed)
    dropped = total = 0
    cc, sp, sn, mk = plan["cls_cfg"], plan["seg_pos"], plan["seg_n"], plan["masks"]
    for s in range(len(sp)):
        cfgs = cc[sp[s]: sp[s] + sn[s]]
        cls = np.nonzero((tiles == tiles[cfgs[0]]).all(1))[0]  # every config of the tile class
        for r in range(R):
            G0 = r * n_sm + 1
            Gs = [G0, (r + 1) * n_sm] if r < R - 1 else [G0, G0 * 7, 2.0 ** 40]
            if r < R - 1:
                Gs += list(rng.integers(G0, (r + 1) * n_sm + 1, 4))
            for lb in range(16):
                L0 = 2 ** lb
                Ls = [L0, 2 ** (lb + 1) - 1] if lb < 15 else [L0, 2.0 ** 20, 2.0 ** 31 - 1]
                if lb < 15:
                    Ls += list(rng.integers(L0, 2 ** (lb + 1), 3))
                g, l = np.meshgrid(np.asarray(Gs, np.float64), np.asarray(Ls, np.float64))
                g, l = g.ravel(), l.ravel()
                m = int(mk[s, r, lb])
                keep = [c for c in cls if not (c in cfgs and not (m >> int(np.nonzero(cfgs == c)[0][0])) & 1)]
                vals_keep = f_ref(rows[keep, r][:, None, :], g[None, :], l[None, :]).min(0)
                for i, c in enumerate(cfgs):
                    total += 1
                    if (m >> i) & 1:
                        continue
                    dropped += 1
                    v = f_ref(rows[c, r][None, :], g, l)
                    assert (vals_keep < v).all(), (s, r, lb, int(c))
    return dropped, total


def test_prune_plan_is_exact_on_synthetic_tables():
    from paper_2604_10187_b200 import synthetic as S

    cfg = S.config_space(False)
    dropped, total = check_plan(S.synthetic_tables(cfg), cfg)
    assert dropped > total // 2  # the plan does prune (most pairs at config 1)


def test_prune_plan_is_exact_on_adversarial_tables():
    cfg, t = U.adversarial_tables()
    check_plan(t, cfg, seed=1)


def test_prune_plan_is_exact_on_odd_tiles():
    from paper_2604_10187_b200 import synthetic as S

    rows = [(tm, tn, tk, st, 4, 1, 1) for tm in (48, 112) for tn in (24, 200) for tk in (32, 96) for st in (2, 3, 4)]
    a = np.array(rows, np.int64)
    cfg = dict(id=(np.arange(len(a)) * 3 + 5).astype(np.int32), t_m=a[:, 0], t_n=a[:, 1], t_k=a[:, 2],
               stages=a[:, 3], warps=a[:, 4], cluster=a[:, 5], swizzle=a[:, 6])
    check_plan(S.synthetic_tables(cfg, seed=3), cfg, seed=2)
