"""Artifact and record formats for the B200 decision path.

The reference stores dual tables as JSON with `%a` hex-float coefficients
(model.cpp:255-372, schema_version 1) and profile records as CSV
(profiler.cpp:155-188).  Both round-trip exactly but parse slowly at
config-3/4 scale.  This module adds:

* the reference formats, read into / written from the CSR arrays the C-ABI
  consumes (`wt_tables_desc` layout: per-table arrays + offsets), with the
  reference's error texts (schema "expected 1, found N", bad CSV header /
  rows, non-positive latency);
* a binary SoA image of the same arrays (`.wtt` tables, `.wtr` records):
  little-endian, 64-byte aligned raw arrays behind a small header, loaded as
  read-only `numpy.memmap` views -- zero-copy: the views' pointers go
  straight to `wt_engine_create` / `wt_fit_build`.  Bit-exact by
  construction (raw IEEE binary64 / integers).

Pure host code: no CUDA needed to convert or inspect artifacts.
"""
from __future__ import annotations

import json
import struct

import numpy as np

# wt_tables_desc arrays (include/wavetune_c.h), CSR layout
TABLE_FIELDS = {
    "macro_id": np.int32, "W": np.int32, "theta_ext": np.float64, "coeff_off": np.int32, "coeff_w": np.int32,
    "coeff_theta": np.float64, "awave_off": np.int32, "awave_w": np.int32, "awave_aoff": np.int32,
    "anchor_l": np.int64, "anchor_micro": np.int32, "ext_aoff": np.int32, "ext_l": np.int64,
    "ext_micro": np.int32,
}
# ProfileRecord (profiler.hpp:56-63) as SoA
RECORD_FIELDS = {"g": np.int64, "l": np.int64, "w": np.int32, "macro": np.int32, "micro": np.int32,
                 "lat": np.float64}

_MAGIC = {"tables": b"WTTBLS01", "records": b"WTRECS01"}
_DT = {np.dtype(np.int32): 1, np.dtype(np.int64): 2, np.dtype(np.float64): 3}
_DT_INV = {v: k for k, v in _DT.items()}
_ALIGN = 64
_CSV_HEADER = "g,l,w,macro_id,micro_id,latency_us"


# ------------------------------------------------------------ binary images
def _save_bin(path: str, kind: str, arrays: dict, fields: dict, meta: dict):
    names = list(fields)
    head = json.dumps({"meta": meta, "arrays": names}).encode()
    entries = []
    off = 16 + 4 + len(head)
    off += 24 * len(names)
    off = (off + _ALIGN - 1) // _ALIGN * _ALIGN
    data = []
    for k in names:
        a = np.ascontiguousarray(arrays[k], dtype=fields[k])
        entries.append(struct.pack("<QQQ", _DT[a.dtype], a.size, off))
        data.append((off, a))
        off = (off + a.nbytes + _ALIGN - 1) // _ALIGN * _ALIGN
    with open(path, "wb") as f:
        f.write(_MAGIC[kind] + struct.pack("<Q", len(names)))
        f.write(struct.pack("<I", len(head)) + head)
        f.write(b"".join(entries))
        for o, a in data:
            f.seek(o)
            f.write(a.tobytes())
        f.truncate(off)


def _load_bin(path: str, kind: str, fields: dict, mmap: bool):
    with open(path, "rb") as f:
        magic = f.read(8)
        if magic != _MAGIC[kind]:
            raise RuntimeError(f"not a wavetune {kind} image: {path}")
        (n,) = struct.unpack("<Q", f.read(8))
        (hl,) = struct.unpack("<I", f.read(4))
        head = json.loads(f.read(hl))
        entries = [struct.unpack("<QQQ", f.read(24)) for _ in range(n)]
    out = {}
    for name, (code, size, off) in zip(head["arrays"], entries):
        dt = _DT_INV[code]
        if name in fields and np.dtype(fields[name]) != dt:
            raise RuntimeError(f"{path}: array {name} has dtype {dt}, expected {np.dtype(fields[name])}")
        if mmap:
            out[name] = np.memmap(path, dtype=dt, mode="r", offset=off, shape=(size,)) if size else np.zeros(0, dt)
        else:
            out[name] = np.fromfile(path, dtype=dt, count=size, offset=off)
    out.update(head["meta"])
    return out


def save_tables_bin(path: str, tables: dict, family: str = "dense_gemm", hardware: str = "b200", p: int = 10):
    """Binary SoA image of a CSR table set (bit-exact)."""
    _save_bin(path, "tables", tables, TABLE_FIELDS,
              {"schema_version": 1, "kernel_family": family, "hardware": hardware, "p": int(p)})


def load_tables_bin(path: str, mmap: bool = True) -> dict:
    """CSR table set from a `.wtt` image; read-only memmap views by default."""
    return _load_bin(path, "tables", TABLE_FIELDS, mmap)


def save_records_bin(path: str, records: dict):
    _save_bin(path, "records", records, RECORD_FIELDS, {"n": int(len(records["g"]))})


def load_records_bin(path: str, mmap: bool = True) -> dict:
    """Records from a `.wtr` image; memmap views (zero-copy into wt_fit_build)."""
    r = _load_bin(path, "records", RECORD_FIELDS, mmap)
    r.pop("n", None)
    return r


# ------------------------------------------------------- reference formats
def load_tables_json(path: str) -> dict:
    """The reference's tables JSON (model.cpp:255-302) as CSR arrays; maps
    are key-sorted exactly as std::map iterates them."""
    with open(path) as f:
        j = json.load(f)
    v = j.get("schema_version")
    if v != 1:
        raise RuntimeError(f"table artifact schema mismatch: expected 1, found {v}")
    d = {k: [] for k in TABLE_FIELDS}
    co_off, aw_off, aw_aoff, ex_off = [0], [0], [0], [0]
    for t in j["tables"]:
        d["macro_id"].append(int(t["macro_id"]))
        d["W"].append(int(t["W"]))
        d["theta_ext"].extend(float.fromhex(x) for x in t["theta_ext"])
        for w in sorted(t["coeffs"], key=int):
            d["coeff_w"].append(int(w))
            d["coeff_theta"].extend(float.fromhex(x) for x in t["coeffs"][w])
        co_off.append(len(d["coeff_w"]))
        for w in sorted(t["anchors"], key=int):
            d["awave_w"].append(int(w))
            amap = t["anchors"][w]
            for l in sorted(amap, key=int):
                d["anchor_l"].append(int(l))
                d["anchor_micro"].append(int(amap[l]))
            aw_aoff.append(len(d["anchor_l"]))
        aw_off.append(len(d["awave_w"]))
        for l in sorted(t["ext_anchors"], key=int):
            d["ext_l"].append(int(l))
            d["ext_micro"].append(int(t["ext_anchors"][l]))
        ex_off.append(len(d["ext_l"]))
    d["coeff_off"], d["awave_off"], d["awave_aoff"], d["ext_aoff"] = co_off, aw_off, aw_aoff, ex_off
    out = {k: np.asarray(v, dtype=TABLE_FIELDS[k]) for k, v in d.items()}
    out["kernel_family"] = j.get("kernel_family", "dense_gemm")
    return out


def save_tables_json(path: str, tables: dict, family: str = "dense_gemm", hardware: str = "b200", p: int = 10):
    """CSR arrays to the reference's JSON (hex-float coefficients; diagnostics
    and ext_flags, which the CSR set does not carry, are written empty)."""
    t = tables
    th = np.asarray(t["coeff_theta"]).reshape(-1, 4)
    te = np.asarray(t["theta_ext"]).reshape(-1, 4)
    art = {"schema_version": 1, "kernel_family": family, "tables": []}
    for i in range(len(t["macro_id"])):
        co = {str(int(t["coeff_w"][q])): [float(x).hex() for x in th[q]]
              for q in range(t["coeff_off"][i], t["coeff_off"][i + 1])}
        an = {}
        for q in range(t["awave_off"][i], t["awave_off"][i + 1]):
            an[str(int(t["awave_w"][q]))] = {str(int(t["anchor_l"][a])): int(t["anchor_micro"][a])
                                             for a in range(t["awave_aoff"][q], t["awave_aoff"][q + 1])}
        ex = {str(int(t["ext_l"][q])): int(t["ext_micro"][q]) for q in range(t["ext_aoff"][i], t["ext_aoff"][i + 1])}
        art["tables"].append({"macro_id": int(t["macro_id"][i]), "hardware": hardware, "W": int(t["W"][i]), "p": p,
                              "coeffs": co, "theta_ext": [float(x).hex() for x in te[i]], "anchors": an,
                              "ext_anchors": ex, "diagnostics": {}, "ext_flags": []})
    with open(path, "w") as f:
        json.dump(art, f)


def load_records_csv(path: str) -> dict:
    """The reference's dataset CSV (profiler.cpp:168-188) as SoA arrays, with
    its checks: exact header, well-formed rows, positive latency."""
    with open(path) as f:
        header = f.readline().rstrip("\n")
        if header != _CSV_HEADER:
            raise RuntimeError("bad dataset header in " + path)
        lines = [ln for ln in f.read().split("\n") if ln]
    if not lines:
        return {k: np.zeros(0, dt) for k, dt in RECORD_FIELDS.items()}
    rows = [ln.split(",") for ln in lines]
    for ln, r in zip(lines, rows):
        if len(r) != 6:
            raise RuntimeError("malformed dataset row: " + ln)
    try:
        cols = np.array(rows)
        out = {"g": cols[:, 0].astype(np.int64), "l": cols[:, 1].astype(np.int64), "w": cols[:, 2].astype(np.int32),
               "macro": cols[:, 3].astype(np.int32), "micro": cols[:, 4].astype(np.int32),
               "lat": np.array([float(x) for x in cols[:, 5]], np.float64)}
    except ValueError as e:
        raise RuntimeError(f"malformed dataset row in {path}: {e}") from None
    bad = np.nonzero(~(out["lat"] > 0))[0]
    if len(bad):
        raise RuntimeError("non-positive latency in dataset row: " + lines[int(bad[0])])
    return out


def save_records_csv(path: str, records: dict):
    """The reference's CSV writer (latency as %.17g: exact round trip)."""
    with open(path, "w") as f:
        f.write(_CSV_HEADER + "\n")
        for g, l, w, m, u, t in zip(records["g"], records["l"], records["w"], records["macro"], records["micro"],
                                    records["lat"]):
            f.write(f"{int(g)},{int(l)},{int(w)},{int(m)},{int(u)},{float(t):.17g}\n")
