"""ctypes front-end to the oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module.  It exposes two independent CPU checkers:

* ``Oracle``  -- the plain-C restatement (oracle/wt_oracle.c), built into
  oracle/_build/libwtoracle.so;
* ``Reference`` -- the reference's own C++ sources compiled verbatim
  (oracle/Makefile -> oracle/_ref/libwtref.so) behind oracle/ref_capi.cpp.

Table artefacts are parsed here with an independent JSON reader (hex floats
via ``float.fromhex``, the inverse of the reference's ``%a`` writer,
model.cpp:261-290) so the restatement never consumes product-side code.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libwtoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libwtref.so")

I32, I64, F64 = np.int32, np.int64, np.float64


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


# ---------------------------------------------------------------- artefacts
@dataclass
class PyTable:
    macro_id: int
    W: int
    p: int
    hardware: str
    coeffs: dict  # w -> (a, b, c, d)
    theta_ext: tuple
    anchors: dict  # w -> {l: micro}
    ext_anchors: dict  # l -> micro
    diagnostics: dict = field(default_factory=dict)
    ext_flags: list = field(default_factory=list)


def parse_tables_json(path):
    with open(path) as f:
        j = json.load(f)
    if j.get("schema_version") != 1:
        raise RuntimeError("schema mismatch")
    out = []
    for jt in j["tables"]:
        co = {int(w): tuple(float.fromhex(x) for x in v) for w, v in jt["coeffs"].items()}
        an = {int(w): {int(l): int(m) for l, m in d.items()} for w, d in jt["anchors"].items()}
        ex = {int(l): int(m) for l, m in jt["ext_anchors"].items()}
        dg = {
            int(w): (float.fromhex(d["r2"]), float.fromhex(d["mape"]), int(d["samples"]), list(d["flags"]))
            for w, d in jt["diagnostics"].items()
        }
        out.append(
            PyTable(int(jt["macro_id"]), int(jt["W"]), int(jt["p"]), jt["hardware"], co,
                    tuple(float.fromhex(x) for x in jt["theta_ext"]), an, ex, dg, list(jt["ext_flags"]))
        )
    return j["kernel_family"], out


def parse_registry_json(path):
    with open(path) as f:
        j = json.load(f)
    tiles = {}
    for m in j["macros"]:
        tiles[int(m["id"])] = (int(m["t_m"]), int(m["t_n"]), int(m["t_k"]))
    order = [int(m["id"]) for m in j["macros"]]
    return tiles, order


class wto_tables(C.Structure):
    _fields_ = [("n_tables", C.c_int32)] + [
        (n, C.c_void_p)
        for n in ("macro_id W t_m t_n t_k theta_ext coeff_off coeff_w coeff_theta awave_off awave_w "
                  "awave_aoff anchor_l anchor_micro ext_aoff ext_l ext_micro").split()
    ]


class FlatTables:
    """DualTable maps flattened to key-sorted CSR arrays (artefact order kept)."""

    def __init__(self, tables, tiles):
        n = len(tables)
        self.macro_id = np.array([t.macro_id for t in tables], I32)
        self.W = np.array([t.W for t in tables], I32)
        self.t_m = np.array([tiles[t.macro_id][0] for t in tables], I64)
        self.t_n = np.array([tiles[t.macro_id][1] for t in tables], I64)
        self.t_k = np.array([tiles[t.macro_id][2] for t in tables], I64)
        self.theta_ext = np.array([t.theta_ext for t in tables], F64).reshape(n * 4)
        co_off, co_w, co_th = [0], [], []
        aw_off, aw_w, aw_aoff, al, am = [0], [], [0], [], []
        ex_off, el, em = [0], [], []
        for t in tables:
            for w in sorted(t.coeffs):
                co_w.append(w)
                co_th.extend(t.coeffs[w])
            co_off.append(len(co_w))
            for w in sorted(t.anchors):
                aw_w.append(w)
                for l in sorted(t.anchors[w]):
                    al.append(l)
                    am.append(t.anchors[w][l])
                aw_aoff.append(len(al))
            aw_off.append(len(aw_w))
            for l in sorted(t.ext_anchors):
                el.append(l)
                em.append(t.ext_anchors[l])
            ex_off.append(len(el))
        self.coeff_off = np.array(co_off, I32)
        self.coeff_w = np.array(co_w + [0], I32)
        self.coeff_theta = np.array(co_th + [0.0] * 4, F64)
        self.awave_off = np.array(aw_off, I32)
        self.awave_w = np.array(aw_w + [0], I32)
        self.awave_aoff = np.array(aw_aoff, I32)
        self.anchor_l = np.array(al + [0], I64)
        self.anchor_micro = np.array(am + [0], I32)
        self.ext_aoff = np.array(ex_off, I32)
        self.ext_l = np.array(el + [0], I64)
        self.ext_micro = np.array(em + [0], I32)
        s = wto_tables()
        s.n_tables = n
        for name, _ in wto_tables._fields_[1:]:
            setattr(s, name, getattr(self, name).ctypes.data)
        self.struct = s


# ---------------------------------------------------------------- restatement
class Oracle:
    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        self.lib = C.CDLL(path)

    def tune(self, flat: FlatTables, n_sm, bps, M, N, K):
        M, N, K = (np.ascontiguousarray(x, I64) for x in (M, N, K))
        n = len(M)
        o = {k: np.zeros(n, I32) for k in ("macro", "micro", "w", "extrap", "comps", "n_missing", "anchor_fb", "status")}
        o["lat"] = np.zeros(n, F64)
        o["g"] = np.zeros(n, I64)
        o["l"] = np.zeros(n, I64)
        self.lib.wto_tune(
            C.byref(flat.struct), C.c_int32(n_sm), C.c_int32(bps), _p(M, C.c_int64), _p(N, C.c_int64),
            _p(K, C.c_int64), C.c_int64(n), _p(o["macro"], C.c_int32), _p(o["micro"], C.c_int32),
            _p(o["lat"], C.c_double), _p(o["g"], C.c_int64), _p(o["l"], C.c_int64), _p(o["w"], C.c_int32),
            _p(o["extrap"], C.c_int32), _p(o["comps"], C.c_int32), _p(o["n_missing"], C.c_int32),
            _p(o["anchor_fb"], C.c_int32), _p(o["status"], C.c_int32))
        return o

    def topk(self, flat, n_sm, bps, M, N, K, k):
        mac = np.zeros(k, I32)
        lat = np.zeros(k, F64)
        st = self.lib.wto_topk(C.byref(flat.struct), C.c_int32(n_sm), C.c_int32(bps), C.c_int64(M),
                               C.c_int64(N), C.c_int64(K), C.c_int32(k), _p(mac, C.c_int32), _p(lat, C.c_double))
        return st, mac, lat

    def predict(self, flat, t, g, l, n_sm, bps):
        lat = C.c_double()
        ex, w, used = C.c_int32(), C.c_int32(), C.c_int32()
        st = self.lib.wto_predict(C.byref(flat.struct), C.c_int32(t), C.c_int64(g), C.c_int64(l),
                                  C.c_int32(n_sm), C.c_int32(bps), C.byref(lat), C.byref(ex), C.byref(w),
                                  C.byref(used))
        return st, lat.value, ex.value, w.value, used.value

    def nearest_anchor(self, anchors, l):
        a = np.ascontiguousarray(anchors, I64)
        out, comps = C.c_int64(), C.c_int32()
        st = self.lib.wto_nearest_anchor(_p(a, C.c_int64), C.c_int32(len(a)), C.c_int64(l), C.byref(out),
                                         C.byref(comps))
        return st, out.value, comps.value

    def fit_bucket(self, g, l, t):
        g, l, t = (np.ascontiguousarray(x, F64) for x in (g, l, t))
        co = np.zeros(4, F64)
        r2, mape, dg = C.c_double(), C.c_double(), C.c_int32()
        st = self.lib.wto_fit_bucket(_p(g, C.c_double), _p(l, C.c_double), _p(t, C.c_double),
                                     C.c_int32(len(g)), _p(co, C.c_double), C.byref(r2), C.byref(mape),
                                     C.byref(dg))
        return st, co, r2.value, mape.value, dg.value

    def select_shared_micro(self, g, micro, t):
        g = np.ascontiguousarray(g, I64)
        micro = np.ascontiguousarray(micro, I32)
        t = np.ascontiguousarray(t, F64)
        n = len(g)
        mo, part, no = C.c_int32(), C.c_int32(), C.c_int32()
        go, to = np.zeros(max(n, 1), I64), np.zeros(max(n, 1), F64)
        st = self.lib.wto_select_shared_micro(_p(g, C.c_int64), _p(micro, C.c_int32), _p(t, C.c_double),
                                              C.c_int32(n), C.byref(mo), C.byref(part), _p(go, C.c_int64),
                                              _p(to, C.c_double), C.byref(no))
        return st, mo.value, part.value, go[: no.value], to[: no.value]

    def build(self, rec, registry_ids, W, p):
        """rec: dict of numpy arrays g,l,w,macro,micro,lat."""
        n = len(rec["g"])
        cap = n + 2
        o = dict(
            macro_id=np.zeros(cap, I32), theta_ext=np.zeros(4 * cap, F64), ext_flags=np.zeros(cap, I32),
            coeff_off=np.zeros(cap + 1, I32), coeff_w=np.zeros(cap, I32), coeff_theta=np.zeros(4 * cap, F64),
            diag_r2=np.zeros(cap, F64), diag_mape=np.zeros(cap, F64), diag_samples=np.zeros(cap, I32),
            diag_flags=np.zeros(cap, I32), awave_off=np.zeros(cap + 1, I32), awave_w=np.zeros(cap, I32),
            awave_aoff=np.zeros(cap + 1, I32), anchor_l=np.zeros(cap, I64), anchor_micro=np.zeros(cap, I32),
            anchor_partial=np.zeros(cap, I32), ext_aoff=np.zeros(cap + 1, I32), ext_l=np.zeros(cap, I64),
            ext_micro=np.zeros(cap, I32))

        class Out(C.Structure):
            _fields_ = [("n_tables", C.c_int32), ("W", C.c_int32), ("p", C.c_int32)] + [
                (k, C.c_void_p) for k in o]

        s = Out()
        for k, v in o.items():
            setattr(s, k, v.ctypes.data)
        cols = [np.ascontiguousarray(rec[k], dt) for k, dt in
                (("g", I64), ("l", I64), ("w", I32), ("macro", I32), ("micro", I32), ("lat", F64))]
        ids = np.ascontiguousarray(registry_ids, I32)
        st = self.lib.wto_build(*[C.c_void_p(c.ctypes.data) for c in cols], C.c_int64(n),
                                C.c_void_p(ids.ctypes.data), C.c_int32(len(ids)), C.c_int32(W), C.c_int32(p),
                                C.byref(s))
        o["n_tables"], o["W"], o["p"] = s.n_tables, s.W, s.p
        return st, o


# ---------------------------------------------------------------- reference
class Reference:
    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` (needs /root/reference)")
        self.lib = C.CDLL(path)
        self.lib.wtref_open.restype = C.c_void_p
        self.lib.wtref_last_error.restype = C.c_char_p
        self.lib.wtref_nearest_anchor.restype = C.c_int64

    def err(self):
        return self.lib.wtref_last_error().decode()

    def open(self, tables_json, registry_json, n_sm, bps=1):
        h = self.lib.wtref_open(tables_json.encode(), registry_json.encode(), C.c_int(n_sm), C.c_int(bps))
        if not h:
            raise RuntimeError(self.err())
        return h

    def close(self, h):
        self.lib.wtref_close(C.c_void_p(h))

    def tune(self, h, M, N, K, nthreads=1):
        M, N, K = (np.ascontiguousarray(x, I64) for x in (M, N, K))
        n = len(M)
        o = {k: np.zeros(n, I32) for k in ("macro", "micro", "w", "extrap", "evals", "comps", "flag_count", "status")}
        o["lat"] = np.zeros(n, F64)
        o["g"] = np.zeros(n, I64)
        o["l"] = np.zeros(n, I64)
        self.lib.wtref_tune(
            C.c_void_p(h), _p(M, C.c_int64), _p(N, C.c_int64), _p(K, C.c_int64), C.c_int64(n),
            _p(o["macro"], C.c_int32), _p(o["micro"], C.c_int32), _p(o["lat"], C.c_double),
            _p(o["g"], C.c_int64), _p(o["l"], C.c_int64), _p(o["w"], C.c_int32), _p(o["extrap"], C.c_int32),
            _p(o["evals"], C.c_int32), _p(o["comps"], C.c_int32), _p(o["flag_count"], C.c_int32),
            _p(o["status"], C.c_int32), C.c_int(nthreads))
        return o

    def tune_flags(self, h, M, N, K):
        buf = C.create_string_buffer(1 << 16)
        st = self.lib.wtref_tune_flags(C.c_void_p(h), C.c_int64(M), C.c_int64(N), C.c_int64(K), buf, len(buf))
        return st, [s for s in buf.value.decode().split("\n") if s]

    def predict(self, h, t, g, l):
        lat = C.c_double()
        ex, w = C.c_int32(), C.c_int32()
        buf = C.create_string_buffer(4096)
        st = self.lib.wtref_predict(C.c_void_p(h), C.c_int(t), C.c_int64(g), C.c_int64(l), C.byref(lat),
                                    C.byref(ex), C.byref(w), buf, len(buf))
        return st, lat.value, ex.value, w.value, [s for s in buf.value.decode().split("\n") if s]

    def nearest_anchor(self, anchors, l):
        a = np.ascontiguousarray(anchors, I64)
        comps = C.c_int32()
        r = self.lib.wtref_nearest_anchor(_p(a, C.c_int64), C.c_int(len(a)), C.c_int64(l), C.byref(comps))
        return r, comps.value

    def fit_bucket(self, g, l, t):
        g, l, t = (np.ascontiguousarray(x, F64) for x in (g, l, t))
        co = np.zeros(4, F64)
        r2, mape, dg = C.c_double(), C.c_double(), C.c_int32()
        st = self.lib.wtref_fit_bucket(_p(g, C.c_double), _p(l, C.c_double), _p(t, C.c_double), C.c_int(len(g)),
                                       _p(co, C.c_double), C.byref(r2), C.byref(mape), C.byref(dg))
        return st, co, r2.value, mape.value, dg.value

    def select_shared_micro(self, g, micro, t):
        g = np.ascontiguousarray(g, I64)
        micro = np.ascontiguousarray(micro, I32)
        t = np.ascontiguousarray(t, F64)
        n = len(g)
        l = np.ones(n, I64)
        mo, part, no = C.c_int32(), C.c_int32(), C.c_int32()
        go, to = np.zeros(max(n, 1), I64), np.zeros(max(n, 1), F64)
        st = self.lib.wtref_select_shared_micro(_p(g, C.c_int64), _p(l, C.c_int64), _p(micro, C.c_int32),
                                                _p(t, C.c_double), C.c_int(n), C.byref(mo), C.byref(part),
                                                _p(go, C.c_int64), _p(to, C.c_double), C.c_int(n), C.byref(no))
        return st, mo.value, part.value, go[: no.value], to[: no.value]

    def build(self, records_csv, registry_json, hw_name, n_sm, W, p, out_json):
        st = self.lib.wtref_build(records_csv.encode(), registry_json.encode(), hw_name.encode(), C.c_int(n_sm),
                                  C.c_int(W), C.c_int(p), out_json.encode())
        if st:
            raise RuntimeError(self.err())

    def resave_tables(self, src, dst):
        return self.lib.wtref_resave_tables(src.encode(), dst.encode())

    def fixture(self, n_sm, n_macros, n_micros, W, I, tau, anchors, sigma, seed, registry_out, records_out):
        a = np.ascontiguousarray(anchors, I64)
        st = self.lib.wtref_fixture(C.c_int(n_sm), C.c_int(n_macros), C.c_int(n_micros), C.c_int(W), C.c_int(I),
                                    C.c_double(tau), _p(a, C.c_int64), C.c_int(len(a)), C.c_double(sigma),
                                    C.c_uint64(seed), registry_out.encode(), records_out.encode())
        if st:
            raise RuntimeError(self.err())

    def build_timed(self, rec, sample_ids, t_m, t_n, t_k, W, p, n_sm, nthreads):
        """Wall seconds of the reference's build_dual_table over ALL records
        for the sample macros, parallel across macros."""
        self.lib.wtref_build_timed.restype = C.c_double
        cols = [np.ascontiguousarray(rec[k], dt) for k, dt in
                (("g", I64), ("l", I64), ("w", I32), ("macro", I32), ("micro", I32), ("lat", F64))]
        ids = np.ascontiguousarray(sample_ids, I32)
        tm, tn, tk = (np.ascontiguousarray(x, I64) for x in (t_m, t_n, t_k))
        nt = C.c_int32()
        sec = self.lib.wtref_build_timed(*[C.c_void_p(c.ctypes.data) for c in cols], C.c_int64(len(cols[0])),
                                         C.c_void_p(ids.ctypes.data), C.c_void_p(tm.ctypes.data),
                                         C.c_void_p(tn.ctypes.data), C.c_void_p(tk.ctypes.data), C.c_int(len(ids)),
                                         C.c_int(W), C.c_int(p), C.c_int(n_sm), C.c_int(nthreads), C.byref(nt))
        if sec < 0:
            raise RuntimeError(self.err())
        return sec, nt.value

    def build_plan(self, n_sm, bps, W, I, tau, anchors, out_json):
        a = np.ascontiguousarray(anchors, I64)
        return self.lib.wtref_build_plan(C.c_int(n_sm), C.c_int(bps), C.c_int(W), C.c_int(I), C.c_double(tau),
                                         _p(a, C.c_int64), C.c_int(len(a)), out_json.encode())


def read_records_csv(path):
    d = np.loadtxt(path, delimiter=",", skiprows=1, dtype=np.float64, ndmin=2)
    # latency column must round-trip exactly: re-read it as text
    with open(path) as f:
        next(f)
        lat = np.array([float(line.rsplit(",", 1)[1]) for line in f if line.strip()], F64)
    return dict(g=d[:, 0].astype(I64), l=d[:, 1].astype(I64), w=d[:, 2].astype(I32),
                macro=d[:, 3].astype(I32), micro=d[:, 4].astype(I32), lat=lat)


def _ref_extra(ref):
    L = ref.lib
    return L


def ref_ground(ref, n_macros, n_micros, out):
    if ref.lib.wtref_ground(C.c_int(n_macros), C.c_int(n_micros), out.encode()):
        raise RuntimeError(ref.err())


def ref_simulate(ref, n_sm, g, l, mu, sigma=0.0, seed=0):
    out = C.c_double()
    st = ref.lib.wtref_simulate(C.c_int(n_sm), C.c_int64(g), C.c_int64(l), C.c_double(mu), C.c_double(sigma),
                                C.c_uint64(seed), C.byref(out))
    if st:
        raise RuntimeError(ref.err())
    return out.value


def ref_oracle_best(ref, registry_json, ground_json, n_sm, seed, M, N, K, sigma, reps):
    ma, mi, lat = C.c_int32(), C.c_int32(), C.c_double()
    st = ref.lib.wtref_oracle_best(registry_json.encode(), ground_json.encode(), C.c_int(n_sm), C.c_uint64(seed),
                                   C.c_int64(M), C.c_int64(N), C.c_int64(K), C.c_double(sigma), C.c_int(reps),
                                   C.byref(ma), C.byref(mi), C.byref(lat))
    if st:
        raise RuntimeError(ref.err())
    return ma.value, mi.value, lat.value


# ---- ablation baselines through the reference (tuner.cpp:168-250) ----------
def ref_fit_baselines(ref, records_csv, cap=1 << 20):
    sm, sl, st = np.zeros(cap, I32), np.zeros(cap, I64), np.zeros(cap, F64)
    lm, lt = np.zeros(cap, I32), np.zeros(4 * cap, F64)
    ns, nl = C.c_int64(), C.c_int64()
    if ref.lib.wtref_fit_baselines(records_csv.encode(), C.c_int64(cap), _p(sm, C.c_int32), _p(sl, C.c_int64),
                                   _p(st, C.c_double), C.byref(ns), _p(lm, C.c_int32), _p(lt, C.c_double),
                                   C.byref(nl)):
        raise RuntimeError(ref.err())
    k, j = ns.value, nl.value
    return dict(step_macro=sm[:k], step_l=sl[:k], step_t=st[:k], lin_macro=lm[:j], lin_theta=lt[:4 * j])


def _bp_arrays(kind, bp):
    if kind == 0:
        return (np.ascontiguousarray(bp["step_macro"], I32), np.ascontiguousarray(bp["step_l"], I64),
                np.ascontiguousarray(bp["step_t"], F64), len(bp["step_macro"]))
    m = np.ascontiguousarray(bp["lin_macro"], I32)
    return m, np.zeros(len(m), I64), np.ascontiguousarray(bp["lin_theta"], F64), len(m)


def ref_baseline_predict(ref, kind, bp, n_sm, bps, macro, g, l):
    m, ls, t, n = _bp_arrays(kind, bp)
    out = C.c_double()
    st = ref.lib.wtref_baseline_predict(C.c_int(kind), _p(m, C.c_int32), _p(ls, C.c_int64), _p(t, C.c_double),
                                        C.c_int64(n), C.c_int(n_sm), C.c_int(bps), C.c_int32(macro),
                                        C.c_int64(g), C.c_int64(l), C.byref(out))
    return st, out.value


def ref_baseline_tune(ref, h, kind, bp, M, N, K, nthreads=8):
    m, ls, t, nb = _bp_arrays(kind, bp)
    M, N, K = (np.ascontiguousarray(x, I64) for x in (M, N, K))
    n = len(M)
    o = {k: np.zeros(n, I32) for k in ("macro", "micro", "w", "extrap", "comps", "flag_count", "status")}
    o["lat"] = np.zeros(n, F64)
    ref.lib.wtref_baseline_tune(
        C.c_void_p(h), C.c_int(kind), _p(m, C.c_int32), _p(ls, C.c_int64), _p(t, C.c_double), C.c_int64(nb),
        _p(M, C.c_int64), _p(N, C.c_int64), _p(K, C.c_int64), C.c_int64(n), _p(o["macro"], C.c_int32),
        _p(o["micro"], C.c_int32), _p(o["lat"], C.c_double), _p(o["w"], C.c_int32), _p(o["extrap"], C.c_int32),
        _p(o["comps"], C.c_int32), _p(o["flag_count"], C.c_int32), _p(o["status"], C.c_int32), C.c_int(nthreads))
    return o
