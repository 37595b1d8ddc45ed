"""Small end-to-end drive of every decision kernel for compute-sanitizer
(memcheck / racecheck / synccheck): representative grid sweep (k_sweep_w +
k_expand) + run index (hand-written scan), a partial sweep, the every-M sweep
(k_sweep2, WT_SWEEP_DEDUP=0 run), hashed gather with off-grid queries (keys,
scan, scatter, k_eval4), tune_batch, the single-query kernel, a small host
fit, the device-resident build (records in HBM: sorted-key group / select /
sample kernels, quad + octet fits) -> device image -> async grid, and the
multi-GPU exchange kernels (pack / merge).  Sizes are tiny: the sanitizer
is ~100x."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_10187_b200 import capi, synthetic as S  # noqa: E402

cfg = S.config_space(False)
t = S.synthetic_tables(cfg)
eng = capi.Engine(t, S.registry_arrays(cfg), n_sm=148)
pairs = S.LLAMA3_8B
grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 3, 700)
grid.sweep()
M, N, K = S.query_stream(6001, pairs, seed=5, off_grid_frac=0.2, m_max=800)
o = [torch.empty(len(M), dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
grid.gather(*(torch.from_numpy(x).cuda() for x in (M, N, K)), capi.Engine.decisions(*o))
o2 = [torch.empty(len(M), dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
eng.tune_batch(*(torch.from_numpy(x).cuda() for x in (M, N, K)), capi.Engine.decisions(*o2))
torch.cuda.synchronize()
assert torch.equal(o[0], o2[0]) and torch.equal(o[2].view(torch.int64), o2[2].view(torch.int64))
d = eng.tune_one(3000, 6144, 4096)
rec = S.synthetic_records(cfg)
keep = np.isin(rec["macro"], cfg["id"][:16])
small = {k: v[keep] for k, v in rec.items()}
fit = capi.fit_build(small, cfg["id"][:16], 40, 10)
# partial sweep (representative path, ranges off the interval boundaries)
g2 = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 3, 700)
g2.sweep(100, 1500)
g2.sweep(1500, g2.n_entries)
g2.finalize()
# device-resident build -> image -> async grid -> sweep; pack / merge of two shards
cv = {"g": torch.int64, "l": torch.int64, "w": torch.int32, "macro": torch.int32, "micro": torch.int32,
      "lat": torch.float64}
dev = lambda r: {k: torch.as_tensor(np.ascontiguousarray(r[k])).to(dtype=cv[k], device="cuda") for k in cv}
ids = cfg["id"][:16]
b = capi.Build(dev(small), ids, 40, 10)
reg = S.registry_arrays(cfg)
e2 = capi.Engine.from_build(b, reg, n_sm=148)
st = torch.cuda.current_stream()
g3 = capi.Grid(e2, [p[0] for p in pairs], [p[1] for p in pairs], 1, 900, stream=st)
g3.sweep(stream=st)
parts, counts, sizes = [], [], []
for half in (ids[:8], ids[8:]):
    keep2 = np.isin(small["macro"], half)
    bp = capi.Build(dev({k: v[keep2] for k, v in small.items()}), half, 40, 10)
    c, nb = bp.pack_info()
    parts.append(bp)
    counts.append(c)
    sizes.append(nb)
stride = -(-max(sizes) // 256) * 256
buf = torch.empty(2 * stride, dtype=torch.uint8, device="cuda")
for i, bp in enumerate(parts):
    bp.pack(buf[i * stride:(i + 1) * stride])
mb = capi.Build.merge(buf, stride, np.array(counts))
torch.cuda.synchronize()
assert mb.result()["n_tables"] == b.result()["n_tables"]
print("sanitize drive ok", int(d.macro_id), fit["n_tables"])
