"""Single-query decision latency through the drop-in surfaces (host wall
clock, steady state), and a WT_FIT_TRACE stage breakdown of the config-4 fit.
Usage (GPU box): python tools/probe_latency.py"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def lat_us(fn, n=2000):
    for _ in range(50):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter_ns()
        fn()
        ts.append((time.perf_counter_ns() - t0) / 1e3)
    ts.sort()
    return {"p50": ts[n // 2], "p10": ts[n // 10], "p90": ts[9 * n // 10]}


def main():
    from paper_2604_10187_b200 import _core as wt

    reg = wt.gemm_registry()
    hw = wt.HardwareSpec(148, 1, "b200")
    g = wt.SyntheticKernelGround()
    for ma, mi in sorted(reg.feasible):
        t = reg.macro(ma).tiles
        g.set_entry(ma, mi, wt.GroundEntry(5.0 + 0.001 * t.t_m * t.t_n / 64, 0.02 * t.t_m * t.t_n / 16384 + 0.001 * mi))
    plan = wt.build_plan(hw, "dense_gemm", W=24, I=4, tau=1.1, loop_anchors=[16, 64, 128, 224])
    recs = wt.run_profile_sim(plan, reg, g, sigma=0.5, seed=3)
    art = wt.build_tables(recs, reg, hw, W=24)
    x = wt.DenseGemm(3000, 6144, 4096)
    eng = wt.Engine(art, reg, hw)
    print("tune() [fingerprint + engine]:", lat_us(lambda: wt.tune(x, art, reg, hw)))
    print("Engine.tune()               :", lat_us(lambda: eng.tune(x)))
    import numpy as np

    M, N, K = (np.array([v], np.int32) for v in (3000, 6144, 4096))
    print("Engine.tune_batch(1)        :", lat_us(lambda: eng.tune_batch(M, N, K)))
    from paper_2604_10187_b200 import capi, synthetic as S

    cfg = S.config_space(full=False)
    ce = capi.Engine(S.synthetic_tables(cfg), S.registry_arrays(cfg), n_sm=148)
    print("ctypes wt_tune_one (C=256)  :", lat_us(lambda: ce.tune_one(3000, 6144, 4096)))
    ce.set_resident(20000)
    print("ctypes resident (C=256)     :", lat_us(lambda: ce.tune_one(3000, 6144, 4096)))
    ce.set_resident(0)
    eng.set_resident(20000)
    print("Engine.tune() resident      :", lat_us(lambda: eng.tune(x)))
    eng.set_resident(0)
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    wt.save_tables(art, os.path.join(out, "lat_tables.json"))
    reg.save(os.path.join(out, "lat_registry.json"))
    import subprocess

    subprocess.run([os.path.join(ROOT, "tools", "bin", "lat_tune"), os.path.join(out, "lat_tables.json"),
                    os.path.join(out, "lat_registry.json"), "148", "3000", "6144", "4096"], check=False)

    cfg3 = S.config_space(full=True)
    rec4 = S.synthetic_records(cfg3, micros_per_macro=1)
    for _ in range(2):
        t0 = time.perf_counter()
        fit = capi.fit_build(rec4, cfg3["id"], 40, 10, device=0)
        print(f"fit_build: device_ms {fit['device_ms']:.2f}, wall {1e3 * (time.perf_counter() - t0):.1f} ms",
              flush=True)


if __name__ == "__main__":
    main()
