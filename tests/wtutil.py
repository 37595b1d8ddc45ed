"""Test helpers: convert between the C-ABI table arrays, the reference's JSON
artefacts and the oracle's table objects; build reference fixtures."""
from __future__ import annotations

import json
import os

import numpy as np

import pyoracle as po


def pytables_from_arrays(t):
    out = []
    n = len(t["macro_id"])
    th = np.asarray(t["coeff_theta"]).reshape(-1, 4)
    te = np.asarray(t["theta_ext"]).reshape(-1, 4)
    for i in range(n):
        co = {int(t["coeff_w"][j]): tuple(float(x) for x in th[j]) for j in range(t["coeff_off"][i], t["coeff_off"][i + 1])}
        an = {}
        for j in range(t["awave_off"][i], t["awave_off"][i + 1]):
            an[int(t["awave_w"][j])] = {int(t["anchor_l"][q]): int(t["anchor_micro"][q])
                                        for q in range(t["awave_aoff"][j], t["awave_aoff"][j + 1])}
        ex = {int(t["ext_l"][q]): int(t["ext_micro"][q]) for q in range(t["ext_aoff"][i], t["ext_aoff"][i + 1])}
        out.append(po.PyTable(int(t["macro_id"][i]), int(t["W"][i]), 10, "b200", co, tuple(float(x) for x in te[i]),
                              an, ex))
    return out


def arrays_from_pytables(tabs):
    n = len(tabs)
    d = {k: [] for k in ("coeff_w", "coeff_theta", "awave_w", "anchor_l", "anchor_micro", "ext_l", "ext_micro")}
    co_off, aw_off, aw_aoff, ex_off = [0], [0], [0], [0]
    for t in tabs:
        for w in sorted(t.coeffs):
            d["coeff_w"].append(w)
            d["coeff_theta"].extend(t.coeffs[w])
        co_off.append(len(d["coeff_w"]))
        for w in sorted(t.anchors):
            d["awave_w"].append(w)
            for l in sorted(t.anchors[w]):
                d["anchor_l"].append(l)
                d["anchor_micro"].append(t.anchors[w][l])
            aw_aoff.append(len(d["anchor_l"]))
        aw_off.append(len(d["awave_w"]))
        for l in sorted(t.ext_anchors):
            d["ext_l"].append(l)
            d["ext_micro"].append(t.ext_anchors[l])
        ex_off.append(len(d["ext_l"]))
    return dict(
        macro_id=np.array([t.macro_id for t in tabs], np.int32), W=np.array([t.W for t in tabs], np.int32),
        theta_ext=np.array([t.theta_ext for t in tabs], np.float64).reshape(-1),
        coeff_off=np.array(co_off, np.int32), coeff_w=np.array(d["coeff_w"], np.int32),
        coeff_theta=np.array(d["coeff_theta"], np.float64), awave_off=np.array(aw_off, np.int32),
        awave_w=np.array(d["awave_w"], np.int32), awave_aoff=np.array(aw_aoff, np.int32),
        anchor_l=np.array(d["anchor_l"], np.int64), anchor_micro=np.array(d["anchor_micro"], np.int32),
        ext_aoff=np.array(ex_off, np.int32), ext_l=np.array(d["ext_l"], np.int64),
        ext_micro=np.array(d["ext_micro"], np.int32))


def write_tables_json(tabs, path, family="dense_gemm"):
    j = {"schema_version": 1, "kernel_family": family, "tables": []}
    for t in tabs:
        j["tables"].append({
            "macro_id": t.macro_id, "hardware": t.hardware, "W": t.W, "p": t.p,
            "coeffs": {str(w): [float(x).hex() for x in c] for w, c in t.coeffs.items()},
            "theta_ext": [float(x).hex() for x in t.theta_ext],
            "anchors": {str(w): {str(l): m for l, m in d.items()} for w, d in t.anchors.items()},
            "ext_anchors": {str(l): m for l, m in t.ext_anchors.items()},
            "diagnostics": {}, "ext_flags": [],
        })
    with open(path, "w") as f:
        json.dump(j, f)


def write_registry_json(reg, path, n_micros=4, family="dense_gemm"):
    ids = [int(x) for x in reg["id"]]
    j = {"version": 1, "family": family, "macros": [], "micros": [], "feasible": []}
    for i, mid in enumerate(ids):
        if family == "flash_attention":
            j["macros"].append({"id": mid, "t_q": int(reg["t_m"][i]), "t_kv": int(reg["t_k"][i])})
        else:
            j["macros"].append({"id": mid, "t_m": int(reg["t_m"][i]), "t_n": int(reg["t_n"][i]),
                                "t_k": int(reg["t_k"][i])})
    micro_ids = sorted({mid * n_micros + k for mid in ids for k in range(n_micros)})
    for u in micro_ids:
        j["micros"].append({"id": u, "n_stages": 2 + u % 4, "n_warps": 4})
    for mid in ids:
        for k in range(n_micros):
            j["feasible"].append([mid, mid * n_micros + k])
    with open(path, "w") as f:
        json.dump(j, f)


def registry_from_json(path):
    with open(path) as f:
        j = json.load(f)
    fam = {"dense_gemm": 0, "gemm": 0, "grouped_gemm": 1, "moe": 1, "flash_attention": 2, "attention": 2}[j["family"]]
    ids, tm, tn, tk = [], [], [], []
    for m in j["macros"]:
        ids.append(m["id"])
        if "t_q" in m:
            tm.append(m["t_q"]); tn.append(1); tk.append(m["t_kv"])
        else:
            tm.append(m["t_m"]); tn.append(m["t_n"]); tk.append(m["t_k"])
    return dict(family=fam, id=np.array(ids, np.int32), t_m=np.array(tm, np.int64), t_n=np.array(tn, np.int64),
                t_k=np.array(tk, np.int64))


def reference_fixture(ref, tmp, n_sm=132, n_macros=6, n_micros=8, W=10, I=4, tau=1.5,
                      anchors=(8, 16, 32, 48, 64), sigma=5.0, seed=7, p=10):
    """The reference's own acceptance landscape (acceptance.cpp:228-244),
    profiled with its simulator and fitted by its build_dual_table."""
    tmp = str(tmp)
    reg = os.path.join(tmp, f"reg_{n_macros}_{n_micros}_{W}_{seed}.json")
    rec = os.path.join(tmp, f"rec_{n_macros}_{n_micros}_{W}_{seed}.csv")
    tab = os.path.join(tmp, f"tab_{n_macros}_{n_micros}_{W}_{seed}.json")
    if not os.path.exists(tab):
        ref.fixture(n_sm, n_macros, n_micros, W, I, tau, list(anchors), sigma, seed, reg, rec)
        ref.build(rec, reg, "sim", n_sm, W, p, tab)
    return reg, rec, tab


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)


def adversarial_tables():
    """Config-1 tables with near-tie clones inside every tile class: exact
    duplicate, 1 ulp, 1e-12 relative, a clearly dominated copy, and a config
    whose advantage flips with L (tests of the exact pruning)."""
    from paper_2604_10187_b200 import synthetic as S

    cfg = S.config_space(False)
    t = S.synthetic_tables(cfg)
    C, W = len(cfg["id"]), int(t["W"][0])
    th = t["coeff_theta"].reshape(C, W, 4).copy()
    te = t["theta_ext"].reshape(C, 4).copy()
    key = list(zip(cfg["t_m"], cfg["t_n"], cfg["t_k"]))
    classes = {}
    for c, k in enumerate(key):
        classes.setdefault(k, []).append(c)
    rng = np.random.default_rng(7)
    for cs in classes.values():
        c0, c1, c2, c3, c4, c5 = cs[:6]
        th[c1] = th[c0]                                   # exact tie: c0 (smaller id) must win
        te[c1] = te[c0]
        th[c2] = np.nextafter(th[c0], np.inf)             # 1 ulp worse: within margin, kept
        th[c3] = th[c0] * (1 + 1e-12)                     # 1e-12 relative: kept
        th[c4] = th[c0] * 1.5 + np.abs(th[c0]) * 0.1      # clearly dominated: pruned
        te[c4] = te[c0] * 1.5 + np.abs(te[c0]) * 0.1
        # c5: cheaper fixed cost, steeper per-iteration slope -> wins only at short L
        th[c5, :, 1] = th[c0, :, 1] * 0.5
        th[c5, :, 3] = th[c0, :, 3] * 0.5
        th[c5, :, 0] = th[c0, :, 0] * (1.5 + rng.random())
        th[c5, :, 2] = th[c0, :, 2] * (1.5 + rng.random())
    t["coeff_theta"] = th.reshape(-1)
    t["theta_ext"] = te.reshape(-1)
    return cfg, t


def registry_arrays_of(cfg):
    from paper_2604_10187_b200 import synthetic as S

    return S.registry_arrays(cfg)


def oracle_tune_mt(orc, flat, n_sm, bps, M, N, K, threads=None, chunk=4096):
    """Oracle.tune over host threads (the ctypes call releases the GIL);
    results concatenated in query order."""
    from concurrent.futures import ThreadPoolExecutor

    n = len(M)
    threads = threads or max(1, min(32, len(os.sched_getaffinity(0))))
    parts = [(i, min(n, i + chunk)) for i in range(0, n, chunk)]
    with ThreadPoolExecutor(threads) as ex:
        outs = list(ex.map(lambda p: orc.tune(flat, n_sm, bps, M[p[0]:p[1]], N[p[0]:p[1]], K[p[0]:p[1]]), parts))
    return {k: np.concatenate([o[k] for o in outs]) for k in outs[0]}


def tiles_of(cfg):
    return {int(i): (int(a), int(b), int(c)) for i, a, b, c in zip(cfg["id"], cfg["t_m"], cfg["t_n"], cfg["t_k"])}
