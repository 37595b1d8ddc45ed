"""End-to-end WaveTune validation on real B200 kernels (SURVEY.md 8(f) row 2,
BASELINE.json configs[5]).

profile (run_profile over the sparse plan, B200GemmBackend = the tcgen05 GEMM
family behind the reference's MeasurementBackend) -> fit (build_tables on
the GPU) -> tune (the decision path) on Llama-3-8B prefill linear shapes, and
compare each pick with the exhaustive optimum measured the same way, with
static defaults and with cuBLAS (torch.matmul) for context.

Usage: python tools/validate_gemm.py [--out gpurun_out/gemm_validation.json]
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# Llama-3-8B linear layers: (N, K) of qkv, o, gate_up, down (weights [N, K])
LLAMA3_8B_LINEARS = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
PREFILL_M = [128, 512, 1000, 2048, 3000, 4096, 8192, 16384]


def geomean(x):
    x = np.asarray(x, dtype=np.float64)
    return float(np.exp(np.log(x).mean()))


def cublas_us(M, N, K, warmup, reps):
    import torch

    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    for _ in range(warmup):
        a @ b.T
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        a @ b.T
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000.0 / reps


def cutlass_xcheck_lib():
    """tools/bin/libwtgemm_cutlass.so (make -C tools cutlass): the same C-ABI
    over CUTLASS 4.5 sm100 collectives -- a cross-check of the hand-written
    family's speed, never the product."""
    import ctypes as C

    p = os.path.join(ROOT, "tools", "bin", "libwtgemm_cutlass.so")
    if not os.path.exists(p):
        return None
    L = C.CDLL(p)
    i32p = C.POINTER(C.c_int32)
    L.wt_gemm_family_size.restype = C.c_int
    L.wt_gemm_config.argtypes = [C.c_int] + [C.POINTER(C.c_int)] * 4
    L.wt_gemm_measure_batch.argtypes = [C.c_int] + [i32p] * 5 + [C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_double)]
    return L


def xcheck_best_us(L, M, N, K, warmup, reps):
    """Fastest CUTLASS instantiation x swizzle on one shape (us) and its label."""
    import ctypes as C

    n = L.wt_gemm_family_size()
    cfgs, labels = [], []
    for c in range(n):
        v = [C.c_int() for _ in range(4)]
        L.wt_gemm_config(c, *[C.byref(x) for x in v])
        for s in (1, 2, 4, 8):
            cfgs.append((c, s))
            labels.append(f"{v[0].value}x{v[1].value}x{v[2].value}/s{v[3].value}/w{s}")
    arr = [np.ascontiguousarray(x, dtype=np.int32) for x in
           ([c for c, _ in cfgs], [s for _, s in cfgs], [M] * len(cfgs), [N] * len(cfgs), [K] * len(cfgs))]
    out = np.empty(len(cfgs), dtype=np.float64)
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))
    rc = L.wt_gemm_measure_batch(len(cfgs), *[p(a) for a in arr], warmup, reps, 3,
                                 out.ctypes.data_as(C.POINTER(C.c_double)))
    if rc != 0:
        return None, None
    out[out <= 0] = np.inf
    i = int(np.argmin(out))
    return float(out[i]), labels[i]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--W", type=int, default=24)
    ap.add_argument("--I", type=int, default=4)
    ap.add_argument("--tau", type=float, default=1.1)
    ap.add_argument("--anchors", default="16,64,128,224")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--no-xcheck", action="store_true", help="skip the CUTLASS cross-check timings")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "gemm_validation.json"))
    args = ap.parse_args()

    import torch
    from paper_2604_10187_b200 import _core as wt

    xlib = cutlass_xcheck_lib() if not args.no_xcheck else None
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    hw = wt.HardwareSpec(n_sm, 1, "b200")
    reg = wt.gemm_registry()
    feasible = sorted(reg.feasible)
    backend = wt.B200GemmBackend(warmup=args.warmup, measured=args.reps, seed=1)
    anchors = [int(x) for x in args.anchors.split(",")]
    plan = wt.build_plan(hw, "dense_gemm", W=args.W, I=args.I, tau=args.tau, loop_anchors=anchors)

    t0 = time.perf_counter()
    records = backend.profile(plan, reg)
    t_profile = time.perf_counter() - t0
    t0 = time.perf_counter()
    art = wt.build_tables(records, reg, hw, W=args.W)
    t_fit = time.perf_counter() - t0
    # ablation baselines from the same records (tuner.cpp:191-220)
    step_bp = wt.fit_step_baseline(records)
    linear_bp = wt.fit_linear_baseline(records)
    # eval.cpp:48-52: the default heuristic = smallest macro id, its smallest feasible micro
    d_macro = min(m.id for m in reg.macros)
    d_micro = min(reg.feasible_micros(d_macro))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    wt.write_records(records, os.path.splitext(args.out)[0] + "_records.csv")
    wt.save_tables(art, os.path.splitext(args.out)[0] + "_tables.json")
    print(f"profiled {len(records)} measurements over {len(plan.grid_points)} grid points in {t_profile:.1f} s; "
          f"fit {len(art.tables)} dual tables in {t_fit * 1e3:.1f} ms", flush=True)

    def label(ma, mi):
        t, u = reg.macro(ma).tiles, reg.micro(mi)
        return f"{t.t_m}x{t.t_n}x{t.t_k}/s{u.n_stages}/w{dict(u.extra)['swizzle']}"

    rows = []
    for layer, (N, K) in LLAMA3_8B_LINEARS.items():
        for M in PREFILL_M:
            x = wt.DenseGemm(M, N, K)
            t_all = {}
            for ma, mi in feasible:
                t_all[(ma, mi)] = backend.measure(x, reg.macro(ma), reg.micro(mi))
            best = min(t_all, key=t_all.get)
            q0 = time.perf_counter()
            d = wt.tune(x, art, reg, hw)
            t_decide = (time.perf_counter() - q0) * 1e6
            pick = (d.macro_id, d.micro_id)
            sd = wt.baseline_tune(x, step_bp, art, reg, hw)
            ld = wt.baseline_tune(x, linear_bp, art, reg, hw)
            methods = {
                "wavetune": (pick, d.predicted_latency_us),
                "step": ((sd.macro_id, sd.micro_id), sd.predicted_latency_us),
                "linear": ((ld.macro_id, ld.micro_id), ld.predicted_latency_us),
                "oracle": (best, None),
                "default": ((d_macro, d_micro), None),
            }
            xc_us, xc_cfg = xcheck_best_us(xlib, M, N, K, args.warmup, args.reps) if xlib else (None, None)
            rows.append({
                "methods": {k: {"config": label(*c), "measured_us": t_all[c], "predicted_us": pr}
                            for k, (c, pr) in methods.items()},
                "layer": layer, "M": M, "N": N, "K": K,
                "oracle": label(*best), "oracle_us": t_all[best],
                "wavetune": label(*pick), "wavetune_us": t_all[pick], "predicted_us": d.predicted_latency_us,
                "extrapolated": bool(d.regime.extrapolated), "decide_us_host": t_decide,
                "all_us": {label(*k): v for k, v in t_all.items()},
                "cublas_us": cublas_us(M, N, K, args.warmup, args.reps),
                "cutlass_best_us": xc_us, "cutlass_best": xc_cfg,
            })
            r = rows[-1]
            print(f"{layer:8s} M={M:6d}: oracle {r['oracle']:22s} {r['oracle_us']:9.1f} us | wavetune "
                  f"{r['wavetune']:22s} {r['wavetune_us']:9.1f} us (pred {r['predicted_us']:9.1f}) | "
                  f"cuBLAS {r['cublas_us']:9.1f} us" + (f" | CUTLASS best {xc_us:9.1f} us" if xc_us else ""),
                  flush=True)

    # eval.cpp:106-116: geomean speedup over the default heuristic, MAPE of
    # each method's predicted latency against the measured one
    eval_report = {"geomean_speedup_vs_default": {}, "mape": {}}
    for meth in rows[0]["methods"]:
        eval_report["geomean_speedup_vs_default"][meth] = geomean(
            [r["methods"]["default"]["measured_us"] / r["methods"][meth]["measured_us"] for r in rows])
        pr = [r["methods"][meth] for r in rows if r["methods"][meth]["predicted_us"] is not None]
        if pr:
            eval_report["mape"][meth] = float(np.mean([abs(p["predicted_us"] - p["measured_us"]) / p["measured_us"]
                                                       for p in pr]))
    eval_report["default_config"] = label(d_macro, d_micro)
    sub = [r for r in rows if 512 <= r["M"] <= 8192]
    eval_report["geomean_speedup_vs_default_M512_8192"] = {
        meth: geomean([r["methods"]["default"]["measured_us"] / r["methods"][meth]["measured_us"] for r in sub])
        for meth in rows[0]["methods"]}
    # decision overhead on this registry: Engine (one launch) and resident server
    eng = wt.Engine(art, reg, hw)
    xq = wt.DenseGemm(3000, 6144, 4096)

    def p50_us(fn, n=3000):
        for _ in range(100):
            fn()
        ts = []
        for _ in range(n):
            q0 = time.perf_counter_ns()
            fn()
            ts.append((time.perf_counter_ns() - q0) / 1e3)
        return float(np.median(ts))

    overhead = {"tune_cached_engine": p50_us(lambda: wt.tune(xq, art, reg, hw)),
                "engine_tune_one": p50_us(lambda: eng.tune(xq))}
    eng.set_resident(20000)
    overhead["engine_tune_one_resident"] = p50_us(lambda: eng.tune(xq))
    eng.set_resident(0)
    labels = list(rows[0]["all_us"])
    # the best single static config in hindsight (a strong default) and a
    # common hand-picked default
    static_gm = {c: geomean([r["all_us"][c] / r["oracle_us"] for r in rows]) for c in labels}
    best_static = min(static_gm, key=static_gm.get)
    fixed_default = "128x256x64/s3/w1"
    wt_ratio = [r["wavetune_us"] / r["oracle_us"] for r in rows]
    summary = {
        "plan": {"W": args.W, "I": args.I, "tau": args.tau, "anchors": anchors, "grid_points": len(plan.grid_points),
                 "measurements": len(records), "profile_s": t_profile, "fit_ms": t_fit * 1e3},
        "family": {"configs": len(feasible), "macros": len(reg.macros)},
        "shapes": len(rows),
        "wavetune_vs_oracle_geomean": geomean(wt_ratio),
        "wavetune_vs_oracle_worst": max(wt_ratio),
        "wavetune_exact_oracle_frac": float(np.mean([r["wavetune"] == r["oracle"] for r in rows])),
        "wavetune_within_5pct_frac": float(np.mean([x <= 1.05 for x in wt_ratio])),
        "speedup_vs_fixed_default": geomean([r["all_us"][fixed_default] / r["wavetune_us"] for r in rows]),
        "fixed_default": fixed_default,
        "speedup_vs_best_static": geomean([r["all_us"][best_static] / r["wavetune_us"] for r in rows]),
        "best_static": best_static,
        "wavetune_vs_cublas_geomean": geomean([r["cublas_us"] / r["wavetune_us"] for r in rows]),
        "oracle_vs_cublas_geomean": geomean([r["cublas_us"] / r["oracle_us"] for r in rows]),
        "family_best_vs_cutlass_best_geomean": (geomean([r["cutlass_best_us"] / r["oracle_us"] for r in rows])
                                                if all(r["cutlass_best_us"] for r in rows) else None),
        "wavetune_vs_cutlass_best_geomean": (geomean([r["cutlass_best_us"] / r["wavetune_us"] for r in rows])
                                             if all(r["cutlass_best_us"] for r in rows) else None),
        "family_best_ge_cutlass_best_shapes": (int(sum(r["oracle_us"] <= r["cutlass_best_us"] * 1.0 for r in rows))
                                               if all(r["cutlass_best_us"] for r in rows) else None),
        "decide_us_host_median": float(np.median([r["decide_us_host"] for r in rows])),
        "prediction_mape": float(np.mean([abs(r["predicted_us"] - r["wavetune_us"]) / r["wavetune_us"]
                                          for r in rows])),
        "eval": eval_report,
        "decision_overhead_us_p50_python": overhead,
    }
    with open(args.out, "w") as f:
        json.dump({"summary": summary, "rows": rows}, f, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
