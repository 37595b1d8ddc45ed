"""Quick check of the hand-written tcgen05 GEMM family on the GPU: numerics of
every instantiation against torch fp32 on a few shapes, then device time vs
cuBLAS (torch.matmul) on square and Llama-3-8B shapes.  Prints as it goes so
a hang names its config (run it under `timeout`)."""
import math
import sys
import os

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2604_10187_b200 import gemm  # noqa: E402


def check(out, a, b):
    ref = a.float() @ b.float().T
    err = (out.float() - ref).abs()
    tol = ref.abs() * (2.0 ** -7) + 1e-3 * math.sqrt(a.shape[1])
    return int((err > tol).sum().item()), float(err.max().item())


def main():
    fam = gemm.family()
    shapes = [(256, 256, 128), (512, 1024, 512), (333, 264, 200), (1, 8, 64), (1000, 4104, 1096)]
    cfgs = range(len(fam)) if len(sys.argv) < 2 else [int(x) for x in sys.argv[1].split(",")]
    bad_total = 0
    for c in cfgs:
        for (M, N, K) in shapes:
            g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
            a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
            b = torch.randn(N, K, device="cuda", generator=g).bfloat16()
            print(f"cfg {c} {fam[c]} shape {M}x{N}x{K} ...", end=" ", flush=True)
            out = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
            gemm.matmul(a, b, c, 2, out=out)
            torch.cuda.synchronize()
            bad, mx = check(out, a, b)
            bad_total += bad
            print(f"bad={bad} maxerr={mx:.3g}", flush=True)
    print("TOTAL BAD", bad_total, flush=True)
    perf = [(4096, 4096, 4096), (8192, 8192, 8192), (4096, 14336, 4096), (4096, 4096, 14336), (128, 4096, 4096),
            (128, 14336, 4096), (16, 4096, 4096), (2048, 6144, 4096)]
    for (M, N, K) in perf:
        a = torch.randn(M, K, device="cuda").bfloat16()
        b = torch.randn(N, K, device="cuda").bfloat16()
        for _ in range(3):
            torch.matmul(a, b.T)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            torch.matmul(a, b.T)
        e1.record()
        torch.cuda.synchronize()
        cub = e0.elapsed_time(e1) / 20 * 1e3
        best = None
        row = []
        for c in cfgs:
            try:
                t = min(gemm.time_us(a, b, c, s, warmup=3, reps=20) for s in (1, 4))
            except Exception:
                t = float("nan")
            row.append(t)
            if t == t and (best is None or t < best[0]):
                best = (t, c)
        fl = 2.0 * M * N * K
        print(f"{M}x{N}x{K}: cublas {cub:.1f} us ({fl / cub / 1e6:.0f} TF/s)  best cfg {best[1]} {fam[best[1]]} "
              f"{best[0]:.1f} us ({fl / best[0] / 1e6:.0f} TF/s)  all: " + " ".join(f"{x:.0f}" for x in row),
              flush=True)


if __name__ == "__main__":
    main()
