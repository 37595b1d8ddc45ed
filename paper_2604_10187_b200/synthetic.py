"""Synthetic workloads for the BASELINE.json configs.

Everything here is deterministic input data (shape lists, config spaces,
sampled-latency records, coefficient tables); no decision logic lives here.
The (N, K) pairs come from public model configs; the reference ships none.
"""
from __future__ import annotations

import math

import numpy as np

# (N, K) per linear layer: QKV, O, gate+up, down.
LLAMA3_8B = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]
LLAMA3_70B = [(10240, 8192), (8192, 8192), (57344, 8192), (8192, 28672)]
QWEN2_72B = [(10240, 8192), (8192, 8192), (59136, 8192), (8192, 29568)]


def unique_pairs(*models):
    seen, out = set(), []
    for m in models:
        for p in m:
            if p not in seen:
                seen.add(p)
                out.append(p)
    return out


LOOP_ANCHORS = [16, 32, 48, 64, 80]


def config_space(full: bool):
    """Decomposed tile-config space, every full config its own macro id.

    full=False: config 1 (256) = BM{64,128} x BN{32..256 step 32} x BK{64,128}
                x stages{2,3,4,6} x cluster{1,2}
    full=True : config 3 (4608) = BM{64,128,256} x BN{8} x BK{64,128}
                x stages{2..7} x warps{4,8} x cluster{1,2} x swizzle{1,2,4,8}
    """
    BN = [32, 64, 96, 128, 160, 192, 224, 256]
    rows = []
    if not full:
        for bm in (64, 128):
            for bn in BN:
                for bk in (64, 128):
                    for st in (2, 3, 4, 6):
                        for cl in (1, 2):
                            rows.append((bm, bn, bk, st, 4, cl, 1))
    else:
        for bm in (64, 128, 256):
            for bn in BN:
                for bk in (64, 128):
                    for st in range(2, 8):
                        for wp in (4, 8):
                            for cl in (1, 2):
                                for sw in (1, 2, 4, 8):
                                    rows.append((bm, bn, bk, st, wp, cl, sw))
    a = np.array(rows, np.int64)
    return dict(id=np.arange(len(a), dtype=np.int32), t_m=a[:, 0], t_n=a[:, 1], t_k=a[:, 2], stages=a[:, 3],
                warps=a[:, 4], cluster=a[:, 5], swizzle=a[:, 6])


def _hash01(*xs):
    """Deterministic pseudo-random in [0, 1) from integers (splitmix64)."""
    z = np.uint64(0x9E3779B97F4A7C15)
    acc = np.zeros(np.broadcast(*xs).shape, np.uint64)
    with np.errstate(over="ignore"):
        for x in xs:
            acc = acc ^ np.asarray(x, np.uint64)
            acc = acc + z
            acc = (acc ^ (acc >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            acc = (acc ^ (acc >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            acc = acc ^ (acc >> np.uint64(31))
    return (acc >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def ground_truth(cfg):
    """Per-config block cost (two_regime_ground-style, helpers.hpp:40-56,
    extended with stages / warps / cluster / swizzle effects)."""
    area = cfg["t_m"] * cfg["t_n"] / 4096.0
    kf = cfg["t_k"] / 64.0
    st = cfg["stages"].astype(np.float64)
    base = 20.0 * area * (1.0 + 0.04 * (st - 2)) * (1.0 + 0.03 * (cfg["cluster"] - 1))
    per_iter = 2.0 * area ** 0.85 * kf * (1.0 - 0.05 * np.minimum(st - 2, 3)) * (1.0 - 0.04 * (cfg["cluster"] - 1))
    per_iter = per_iter * (1.0 + 0.02 * (cfg["warps"] == 8)) * (1.0 + 0.01 * np.log2(cfg["swizzle"]))
    j = _hash01(cfg["id"], 7)
    return base * (1.0 + 0.02 * j), per_iter * (1.0 + 0.02 * (1.0 - j))


def synthetic_tables(cfg, W=40, slots=148, anchors=LOOP_ANCHORS, n_micros=4, seed=11):
    """Dual tables as produced by a wave-structured fit of ground_truth:
    per wave w, T ~ alpha*g*l + beta*g + gamma*l + delta with the within-wave
    desynchronisation slope, plus deterministic jitter (ties are rare)."""
    C = len(cfg["id"])
    base, per = ground_truth(cfg)
    w = np.arange(1, W + 1, dtype=np.float64)[None, :]
    e1 = 0.15 + 0.1 * _hash01(cfg["id"][:, None], w.astype(np.int64), seed)
    e2 = 0.10 + 0.1 * _hash01(cfg["id"][:, None], w.astype(np.int64), seed + 1)
    alpha = e1 * per[:, None] / slots
    beta = e2 * base[:, None] / slots
    gamma = per[:, None] * (w - e1 * (w - 0.5))
    delta = base[:, None] * (w - e2 * (w - 0.5))
    theta = np.stack([alpha, beta, gamma, delta], axis=-1)  # [C, W, 4]
    theta_ext = np.stack([per / slots, base / slots, 0.02 * per, 0.5 * base], axis=-1)
    # anchors: micro variant per (wave, l) -- deeper pipelines win at long l
    A = len(anchors)
    micro = (np.arange(A)[None, None, :] * n_micros // A + (_hash01(cfg["id"][:, None, None],
             w.astype(np.int64)[:, :, None], np.arange(A)[None, None, :]) < 0.2)) % n_micros
    return dict(
        macro_id=cfg["id"].astype(np.int32),
        W=np.full(C, W, np.int32),
        theta_ext=theta_ext.reshape(-1),
        coeff_off=(np.arange(C + 1) * W).astype(np.int32),
        coeff_w=np.tile(np.arange(1, W + 1, dtype=np.int32), C),
        coeff_theta=theta.reshape(-1),
        awave_off=(np.arange(C + 1) * W).astype(np.int32),
        awave_w=np.tile(np.arange(1, W + 1, dtype=np.int32), C),
        awave_aoff=(np.arange(C * W + 1) * A).astype(np.int32),
        anchor_l=np.tile(np.array(anchors, np.int64), C * W),
        anchor_micro=(micro.reshape(-1) + cfg["id"].repeat(W * A) * n_micros).astype(np.int32),
        ext_aoff=(np.arange(C + 1) * A).astype(np.int32),
        ext_l=np.tile(np.array(anchors, np.int64), C),
        ext_micro=(np.arange(C * A) % A * n_micros // A + np.repeat(cfg["id"], A) * n_micros).astype(np.int32),
    )


def registry_arrays(cfg, family=0):
    return dict(family=family, id=cfg["id"].astype(np.int32), t_m=cfg["t_m"], t_n=cfg["t_n"], t_k=cfg["t_k"])


def query_stream(n, pairs, seed=21, off_grid_frac=0.01, m_max=8192):
    """Config 2: pair uniform over `pairs`; M 50% decode U[1,256], 50% prefill
    U[257, m_max]; an off-grid slice with random N, K in [256, 32768]."""
    rng = np.random.default_rng(seed)
    P = np.array(pairs, np.int64)
    pid = rng.integers(0, len(P), n)
    N = P[pid, 0].astype(np.int32)
    K = P[pid, 1].astype(np.int32)
    dec = rng.random(n) < 0.5
    M = np.where(dec, rng.integers(1, 257, n), rng.integers(257, m_max + 1, n)).astype(np.int32)
    off = rng.random(n) < off_grid_frac
    n_off = int(off.sum())
    N[off] = rng.integers(256, 32769, n_off)
    K[off] = rng.integers(256, 32769, n_off)
    return M, N, K


# ---- sampling plan (profiler.cpp:19-95) for the synthetic record generator
def _grid_point(a, b, tau):
    for g in range(b, a - 1, -1):
        root = int(math.isqrt(g))
        for m in range(root, 0, -1):
            if g % m:
                continue
            n = g // m
            if n < m:
                continue
            if n <= tau * m:
                return g, m, n
            break
    return None


def plan_points(slots=148, W=40, I=4, tau=1.1):
    width, rem = divmod(slots, I)
    pts = []
    for w in range(1, W + 1):
        a = (w - 1) * slots + 1
        for i in range(1, I + 1):
            ln = width + (1 if i <= rem else 0)
            b = a + ln - 1
            p = _grid_point(a, b, tau)
            if p:
                pts.append((w, p[0]))
            a = b + 1
    return pts


def synthetic_records(cfg, slots=148, W=40, I=4, tau=1.1, anchors=LOOP_ANCHORS, micros_per_macro=1,
                      noise=0.01, seed=5):
    """Config 4: records (g, l, w, macro, micro, latency) over the wave plan,
    latency = step law (base + per_iter*l)*w with a within-wave slope and
    deterministic multiplicative noise.  Record order follows run_profile
    (grid point, anchor, macro ascending, micro ascending)."""
    pts = plan_points(slots, W, I, tau)
    base, per = ground_truth(cfg)
    C = len(cfg["id"])
    P, A, U = len(pts), len(anchors), micros_per_macro
    pw = np.array([p[0] for p in pts], np.int64)
    pg = np.array([p[1] for p in pts], np.int64)
    g = np.broadcast_to(pg[:, None, None, None], (P, A, C, U)).reshape(-1)
    w = np.broadcast_to(pw[:, None, None, None], (P, A, C, U)).reshape(-1)
    l = np.broadcast_to(np.array(anchors, np.int64)[None, :, None, None], (P, A, C, U)).reshape(-1)
    mac = np.broadcast_to(cfg["id"].astype(np.int64)[None, None, :, None], (P, A, C, U)).reshape(-1)
    mic = np.broadcast_to(np.arange(U)[None, None, None, :], (P, A, C, U)).reshape(-1)
    b = base[mac] * (1.0 + 0.06 * mic)
    q = per[mac] * (1.0 - 0.04 * mic)
    frac = (g - (w - 1) * slots) / slots
    lat = (b + q * l) * (w - 0.3 + 0.3 * frac)
    lat = lat * (1.0 + noise * (_hash01(g, l, mac, mic, seed) - 0.5))
    return dict(g=g.copy(), l=l.copy(), w=w.astype(np.int32), macro=mac.astype(np.int32),
                micro=(mac * U + mic).astype(np.int32), lat=lat)
