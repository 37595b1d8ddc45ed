"""ctypes binding of the C-ABI in include/wavetune_c.h.

This is the exact binding a Python caller of the boundary would write (see
INTEGRATION.md).  Device buffers are torch tensors (plumbing only); every
computation happens in lib/libwtb200.so's sm_100a kernels.  Importing this
module fails loudly if the library is missing -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libwtb200.so")

WT_OK, WT_INVALID_ARGUMENT, WT_RUNTIME_ERROR, WT_OUT_OF_RANGE, WT_CUDA_ERROR, WT_UNSUPPORTED = range(6)
WT_FAMILY_DENSE_GEMM, WT_FAMILY_GROUPED_GEMM, WT_FAMILY_FLASH_ATTENTION = range(3)
WT_FLAG_EXTRAPOLATED, WT_FLAG_MISSING_WAVE, WT_FLAG_ANCHOR_FALLBACK = 1, 2, 4

STATUS_NAMES = {0: "ok", 1: "invalid_argument", 2: "runtime_error", 3: "out_of_range", 4: "cuda_error",
                5: "unsupported"}

vp = C.c_void_p


class WtError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.msg = msg


class wt_hw(C.Structure):
    _fields_ = [("n_sm", C.c_int32), ("blocks_per_sm", C.c_int32)]


class wt_registry_desc(C.Structure):
    _fields_ = [("family", C.c_int32), ("n_macros", C.c_int32), ("id", vp), ("t_m", vp), ("t_n", vp),
                ("t_k", vp)]


_TABLE_FIELDS = ("macro_id W theta_ext coeff_off coeff_w coeff_theta awave_off awave_w awave_aoff "
                 "anchor_l anchor_micro ext_aoff ext_l ext_micro").split()


class wt_tables_desc(C.Structure):
    _fields_ = [("n_tables", C.c_int32)] + [(n, vp) for n in _TABLE_FIELDS]


class wt_engine_info(C.Structure):
    _fields_ = [("n_configs", C.c_int32), ("n_rows", C.c_int32), ("slots", C.c_int32), ("family", C.c_int32),
                ("has_fallback_rows", C.c_int32), ("device", C.c_int32), ("device_bytes", C.c_size_t)]


class wt_decisions(C.Structure):
    _fields_ = [("macro_id", vp), ("micro_id", vp), ("latency_us", vp), ("g", vp), ("l", vp), ("wave", vp),
                ("flags", vp), ("comparisons", vp), ("tail_frac", vp), ("topk", C.c_int32),
                ("topk_macro", vp), ("topk_latency", vp)]


class wt_decision_one(C.Structure):
    _fields_ = [("latency_us", C.c_double), ("g", C.c_int64), ("l", C.c_int64), ("tail_frac", C.c_double),
                ("macro_id", C.c_int32), ("micro_id", C.c_int32), ("wave", C.c_int32), ("flags", C.c_uint32),
                ("comparisons", C.c_int32)]


class wt_grid_desc(C.Structure):
    _fields_ = [("n_pairs", C.c_int32), ("N", vp), ("K", vp), ("m_lo", C.c_int32), ("m_hi", C.c_int32),
                ("topk", C.c_int32)]


class wt_records_desc(C.Structure):
    _fields_ = [("n", C.c_int64), ("g", vp), ("l", vp), ("w", vp), ("macro_id", vp), ("micro_id", vp),
                ("latency_us", vp)]


_BUILD_FIELDS = ("macro_id theta_ext ext_flags coeff_off coeff_w coeff_theta diag_r2 diag_mape diag_samples "
                 "diag_flags awave_off awave_w awave_aoff anchor_l anchor_micro anchor_partial ext_aoff ext_l "
                 "ext_micro").split()


_BASELINE_FIELDS = "step_off step_l step_t lin_theta lin_r2 lin_mape lin_degenerate".split()


class wt_build_result(C.Structure):
    _fields_ = [("n_tables", C.c_int32), ("W", C.c_int32), ("p", C.c_int32)] + [(n, vp) for n in _BUILD_FIELDS] + [
        ("device_ms", C.c_double)] + [(n, vp) for n in _BASELINE_FIELDS]


# entry points declared in include/wavetune_c.h (tests check they all exist)
EXPORTS = (
    "wt_last_error wt_version wt_abi_version wt_engine_create wt_engine_destroy wt_engine_info_get "
    "wt_engine_config_index wt_engine_set_prune wt_engine_count_evals wt_engine_prune_masks wt_tune_batch wt_tune_batch_i64 wt_gather_batch_i64 wt_tune_grouped_batch wt_predict_batch wt_explain "
    "wt_engine_anchor_map wt_nearest_anchor_batch wt_grid_create wt_grid_create_async wt_grid_destroy wt_grid_representatives wt_grid_storage wt_sweep wt_grid_finalize "
    "wt_fit_build_device wt_build_result_get wt_build_pack_info wt_build_pack wt_build_merge wt_engine_create_from_build wt_gather_batch wt_decide_host_sync wt_decide_host_stream_sync wt_launch_count wt_fit_build wt_build_free wt_fit_bucket_batch "
    "wt_simulate_batch wt_profile_sim wt_tune_one wt_engine_set_resident wt_baseline_create "
    "wt_baseline_destroy wt_baseline_tune_batch wt_baseline_predict_batch wt_set_kernel_timing wt_kernel_time_ms "
    "wt_prune_plan wt_sweep_to wt_grid_ipc_handle wt_ipc_open wt_ipc_close").split()

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        L.wt_last_error.restype = C.c_char_p
        L.wt_version.restype = C.c_char_p
        L.wt_launch_count.restype = C.c_int64
        L.wt_engine_config_index.restype = C.c_int32
        L.wt_engine_anchor_map.restype = C.c_int32
        L.wt_grid_representatives.restype = C.c_int64
        _lib = L
    return _lib


def check(st):
    if st != WT_OK:
        raise WtError(st, lib().wt_last_error().decode())


def set_kernel_timing(on: bool):
    """Record CUDA events around the gather kernel / off-grid evaluation of
    every wt_gather_batch call (benchmarking)."""
    check(lib().wt_set_kernel_timing(1 if on else 0))


def kernel_time_ms(which: int) -> float:
    """Elapsed ms of the last timed call: 0 = gather kernel, 1 = off-grid evaluation."""
    ms = C.c_float()
    check(lib().wt_kernel_time_ms(which, C.byref(ms)))
    return ms.value


def launch_count():
    return int(lib().wt_launch_count())


def _ptr(t):
    """Raw pointer of a numpy array or torch tensor (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream_ptr(stream):
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _descs(tables: dict, registry: dict, keep: list):
    """ctypes descriptors of a table set + registry (arrays kept alive in `keep`)."""

    def arr(x, dt):
        a = np.ascontiguousarray(x, dtype=dt)
        if a.size == 0:
            a = np.zeros(1, dt)
        keep.append(a)
        return a.ctypes.data

    td = None
    if tables is not None:
        td = wt_tables_desc()
        td.n_tables = len(tables["macro_id"])
    dts = dict(macro_id=np.int32, W=np.int32, theta_ext=np.float64, coeff_off=np.int32, coeff_w=np.int32,
               coeff_theta=np.float64, awave_off=np.int32, awave_w=np.int32, awave_aoff=np.int32,
               anchor_l=np.int64, anchor_micro=np.int32, ext_aoff=np.int32, ext_l=np.int64,
               ext_micro=np.int32)
    for k in _TABLE_FIELDS if tables is not None else ():
        setattr(td, k, arr(tables[k], dts[k]))
    rd = wt_registry_desc()
    rd.family = registry.get("family", WT_FAMILY_DENSE_GEMM)
    rd.n_macros = len(registry["id"])
    rd.id = arr(registry["id"], np.int32)
    rd.t_m = arr(registry["t_m"], np.int64)
    rd.t_n = arr(registry["t_n"], np.int64)
    rd.t_k = arr(registry["t_k"], np.int64)
    return td, rd


def prune_plan(tables: dict, registry: dict, n_sm: int, blocks_per_sm: int = 1):
    """Host-only: the engine's exact pruning plan (wt_prune_plan) as numpy
    arrays: cls_cfg [C], seg_pos / seg_n [n_seg], masks [n_seg, R, 16]."""
    keep = []
    td, rd = _descs(tables, registry, keep)
    hw = wt_hw(n_sm, blocks_per_sm)
    ns, R, Cn = C.c_int32(), C.c_int32(), C.c_int32()
    check(lib().wt_prune_plan(C.byref(td), C.byref(rd), C.byref(hw), C.byref(ns), C.byref(R), C.byref(Cn),
                              None, None, None, None))
    cc = np.zeros(Cn.value, np.int32)
    sp = np.zeros(ns.value, np.int32)
    sn = np.zeros(ns.value, np.int32)
    mk = np.zeros(ns.value * R.value * 16, np.uint32)
    check(lib().wt_prune_plan(C.byref(td), C.byref(rd), C.byref(hw), C.byref(ns), C.byref(R), C.byref(Cn),
                              C.c_void_p(cc.ctypes.data), C.c_void_p(sp.ctypes.data), C.c_void_p(sn.ctypes.data),
                              C.c_void_p(mk.ctypes.data)))
    return dict(cls_cfg=cc, seg_pos=sp, seg_n=sn, masks=mk.reshape(ns.value, R.value, 16), R=R.value)


class Engine:
    """Owns a wt_engine (device image of tables + registry + hardware)."""

    def __init__(self, tables: dict, registry: dict, n_sm: int, blocks_per_sm: int = 1, device: int = 0):
        L = lib()
        self._keep = []
        td, rd = _descs(tables, registry, self._keep)
        hw = wt_hw(n_sm, blocks_per_sm)
        h = C.c_void_p()
        check(L.wt_engine_create(C.byref(td), C.byref(rd), C.byref(hw), C.c_int(device), C.byref(h)))
        self.handle = h
        self.device = device
        self._keep = []
        self._info = None

    @classmethod
    def from_build(cls, build: "Build", registry: dict, n_sm: int, blocks_per_sm: int = 1, stream=None):
        """Engine from a device-resident build (wt_engine_create_from_build)."""
        self = cls.__new__(cls)
        keep = []
        _, rd = _descs(None, registry, keep)
        hw = wt_hw(n_sm, blocks_per_sm)
        h = C.c_void_p()
        check(lib().wt_engine_create_from_build(build.handle, C.byref(rd), C.byref(hw), vp(_stream_ptr(stream)),
                                                C.byref(h)))
        self.handle = h
        self.device = build.device
        self._keep = []
        self._info = None
        return self

    @property
    def info(self):
        """wt_engine_info, read on first access: it resolves the special-row
        flag, which waits for the device image -- creation itself stays
        asynchronous, so a Grid built next overlaps the image kernels."""
        if self._info is None:
            info = wt_engine_info()
            check(lib().wt_engine_info_get(self.handle, C.byref(info)))
            self._info = info
        return self._info

    def close(self):
        if getattr(self, "handle", None):
            lib().wt_engine_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n_configs(self):
        return self.info.n_configs

    def prune_masks(self, n_seg):
        """The engine's device-built pruning masks [n_seg, R, 16] (inspection;
        n_seg from prune_plan of the same tables)."""
        R = self.info.n_rows
        m = np.zeros(n_seg * R * 16, np.uint32)
        check(lib().wt_engine_prune_masks(self.handle, C.c_void_p(m.ctypes.data), C.c_int64(m.size)))
        return m.reshape(n_seg, R, 16)

    def count_evals(self, counter):
        """Instrumentation: `counter` = a 1-element int64 CUDA tensor that the
        sweep / list evaluation add their physically executed evaluations to
        (None turns it off)."""
        check(lib().wt_engine_count_evals(self.handle, vp(_ptr(counter) if counter is not None else None)))

    def set_prune(self, enable: bool):
        """Extension: False evaluates every config (pruning masks ignored)."""
        check(lib().wt_engine_set_prune(self.handle, C.c_int32(1 if enable else 0)))

    def config_index(self, macro_id):
        return int(lib().wt_engine_config_index(self.handle, C.c_int32(macro_id)))

    def anchor_map(self, config, wave, extrapolated):
        a = np.zeros(64, np.int64)
        m = np.zeros(64, np.int32)
        fb = np.zeros(1, np.int32)
        n = lib().wt_engine_anchor_map(self.handle, C.c_int32(config), C.c_int32(wave), C.c_int32(extrapolated),
                                       C.c_void_p(a.ctypes.data), C.c_void_p(m.ctypes.data), C.c_int32(64),
                                       C.c_void_p(fb.ctypes.data))
        return (a[:n], m[:n], int(fb[0])) if n >= 0 else None

    @staticmethod
    def decisions(macro, micro, lat, g=None, l=None, wave=None, flags=None, comps=None, tail=None,
                  topk=0, topk_macro=None, topk_lat=None):
        d = wt_decisions()
        for name, t in (("macro_id", macro), ("micro_id", micro), ("latency_us", lat), ("g", g), ("l", l),
                        ("wave", wave), ("flags", flags), ("comparisons", comps), ("tail_frac", tail),
                        ("topk_macro", topk_macro), ("topk_latency", topk_lat)):
            setattr(d, name, _ptr(t))
        d.topk = topk
        return d

    def tune_batch(self, M, N, K, out: wt_decisions, stream=None):
        check(lib().wt_tune_batch(self.handle, vp(_ptr(M)), vp(_ptr(N)), vp(_ptr(K)), C.c_int64(M.numel()),
                                  C.byref(out), vp(_stream_ptr(stream))))

    def tune_batch_i64(self, M, N, K, out: wt_decisions, stream=None):
        """Queries with int64 dims (DenseGemm{i64 m, n, k}); dims >= 2^31 are
        evaluated in 64-bit arithmetic (wt_tune_batch_i64)."""
        check(lib().wt_tune_batch_i64(self.handle, vp(_ptr(M)), vp(_ptr(N)), vp(_ptr(K)), C.c_int64(M.numel()),
                                      C.byref(out), vp(_stream_ptr(stream))))

    def tune_one(self, M, N, K) -> wt_decision_one:
        """One query, synchronously, at minimum latency (wt_tune_one)."""
        o = wt_decision_one()
        check(lib().wt_tune_one(self.handle, C.c_int32(M), C.c_int32(N), C.c_int32(K), C.byref(o)))
        return o

    def set_resident(self, idle_us: int):
        """idle_us > 0: answer tune_one() from a resident polling CTA."""
        check(lib().wt_engine_set_resident(self.handle, C.c_int32(idle_us)))

    def tune_grouped_batch(self, row_off, rows, N, K, out, stream=None):
        check(lib().wt_tune_grouped_batch(self.handle, vp(_ptr(row_off)), vp(_ptr(rows)), vp(_ptr(N)),
                                          vp(_ptr(K)), C.c_int64(N.numel()), C.byref(out),
                                          vp(_stream_ptr(stream))))

    def predict_batch(self, config, g, l, lat, wave=None, extrap=None, used_w=None, status=None, stream=None):
        check(lib().wt_predict_batch(self.handle, vp(_ptr(config)), vp(_ptr(g)), vp(_ptr(l)),
                                     C.c_int64(config.numel()), vp(_ptr(lat)), vp(_ptr(wave)), vp(_ptr(extrap)),
                                     vp(_ptr(used_w)), vp(_ptr(status)), vp(_stream_ptr(stream))))

    def explain(self, M, N, K, g, l, wave, used_w, lat, status, stream=None):
        check(lib().wt_explain(self.handle, C.c_int64(M), C.c_int64(N), C.c_int64(K), vp(_ptr(g)), vp(_ptr(l)),
                               vp(_ptr(wave)), vp(_ptr(used_w)), vp(_ptr(lat)), vp(_ptr(status)),
                               vp(_stream_ptr(stream))))


class Baseline:
    """A device baseline predictor (wt_baseline): kind 0 = step, 1 = linear.
    Step entries sorted by (macro, l); linear: one theta row per macro."""

    def __init__(self, engine, kind, macro_id, anchor_l, values, device=0):
        self.engine = engine
        self._keep = [np.ascontiguousarray(macro_id, np.int32), np.ascontiguousarray(anchor_l, np.int64),
                      np.ascontiguousarray(values, np.float64)]
        h = C.c_void_p()
        m, l, v = self._keep
        check(lib().wt_baseline_create(engine.handle if engine is not None else None, C.c_int(device),
                                       C.c_int32(kind), vp(m.ctypes.data), vp(l.ctypes.data), vp(v.ctypes.data),
                                       C.c_int64(len(m)), C.byref(h)))
        self.handle = h.value

    def close(self):
        if self.handle:
            lib().wt_baseline_destroy(vp(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def tune_batch(self, M, N, K, out: wt_decisions, stream=None):
        check(lib().wt_baseline_tune_batch(self.engine.handle, vp(self.handle), vp(_ptr(M)), vp(_ptr(N)),
                                           vp(_ptr(K)), C.c_int64(M.numel()), C.byref(out),
                                           vp(_stream_ptr(stream))))

    def predict_batch(self, macro, g, l, n_sm, bps, lat, status, stream=None):
        hw = wt_hw(n_sm, bps)
        check(lib().wt_baseline_predict_batch(vp(self.handle), vp(_ptr(macro)), vp(_ptr(g)), vp(_ptr(l)),
                                              C.c_int64(macro.numel()), C.byref(hw), vp(_ptr(lat)),
                                              vp(_ptr(status)), vp(_stream_ptr(stream))))


class Grid:
    """A decision grid: tune() over n_pairs (N, K) x M in [m_lo, m_hi]."""

    def __init__(self, engine: Engine, N, K, m_lo, m_hi, topk=0, stream=None):
        """stream=None: synchronous create (IPC-exportable storage); a stream:
        wt_grid_create_async (pool storage, uploads queued on the stream)."""
        self.engine = engine
        self._N = np.ascontiguousarray(N, np.int32)
        self._K = np.ascontiguousarray(K, np.int32)
        d = wt_grid_desc(len(self._N), self._N.ctypes.data, self._K.ctypes.data, m_lo, m_hi, topk)
        h = C.c_void_p()
        if stream is None:
            check(lib().wt_grid_create(engine.handle, C.byref(d), C.byref(h)))
        else:
            check(lib().wt_grid_create_async(engine.handle, C.byref(d), vp(_stream_ptr(stream)), C.byref(h)))
        self.handle = h
        self.m_lo, self.m_hi, self.topk = m_lo, m_hi, topk
        ent, n = C.c_void_p(), C.c_int64()
        tkm, tkl = C.c_void_p(), C.c_void_p()
        check(lib().wt_grid_storage(h, C.byref(ent), C.byref(n), C.byref(tkm), C.byref(tkl)))
        self.entries_ptr, self.n_entries = ent.value, n.value
        self.n_representatives = int(lib().wt_grid_representatives(h))
        self.topk_macro_ptr, self.topk_lat_ptr = tkm.value, tkl.value

    def close(self):
        if getattr(self, "handle", None):
            lib().wt_grid_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sweep(self, begin=0, end=None, stream=None):
        end = self.n_entries if end is None else end
        check(lib().wt_sweep(self.engine.handle, self.handle, C.c_int64(begin), C.c_int64(end),
                             vp(_stream_ptr(stream))))

    def sweep_to(self, dest_ptrs, begin=0, end=None, stream=None):
        """Fused sweep: entries [begin, end) stored into every grid storage in
        `dest_ptrs` (device addresses: this grid's, peers' via ipc_open)."""
        end = self.n_entries if end is None else end
        arr = (C.c_void_p * len(dest_ptrs))(*[C.c_void_p(int(p)) for p in dest_ptrs])
        check(lib().wt_sweep_to(self.engine.handle, self.handle, C.c_int64(begin), C.c_int64(end), arr,
                                C.c_int(len(dest_ptrs)), vp(_stream_ptr(stream))))

    def ipc_handle(self):
        """(64-byte CUDA IPC handle of the storage, byte offset of the entries)."""
        h = (C.c_char * 64)()
        off = C.c_int64()
        check(lib().wt_grid_ipc_handle(self.handle, h, C.byref(off)))
        return bytes(h), off.value

    def finalize(self, stream=None):
        """Rebuild the run index after entries were written directly (e.g. the
        all-gather of a sharded sweep); a full sweep() does it itself."""
        check(lib().wt_grid_finalize(self.engine.handle, self.handle, vp(_stream_ptr(stream))))

    def gather(self, M, N, K, out: wt_decisions, stream=None):
        check(lib().wt_gather_batch(self.engine.handle, self.handle, vp(_ptr(M)), vp(_ptr(N)), vp(_ptr(K)),
                                    C.c_int64(M.numel()), C.byref(out), vp(_stream_ptr(stream))))

    def gather_i64(self, M, N, K, out: wt_decisions, stream=None):
        check(lib().wt_gather_batch_i64(self.engine.handle, self.handle, vp(_ptr(M)), vp(_ptr(N)), vp(_ptr(K)),
                                        C.c_int64(M.numel()), C.byref(out), vp(_stream_ptr(stream))))

    def decide_host(self, M, N, K, macro, micro, lat, chunk=1 << 22, stream=None):
        """End-to-end over host (pinned) buffers: H2D, gather, D2H, pipelined;
        ordered after the work queued on `stream` (default: torch's current
        stream of the engine's device)."""
        if stream is None:
            try:
                import torch

                stream = torch.cuda.current_stream(self.engine.device)
            except Exception:
                stream = None
        check(lib().wt_decide_host_stream_sync(self.engine.handle, self.handle, vp(_ptr(M)), vp(_ptr(N)),
                                               vp(_ptr(K)), C.c_int64(M.numel()), vp(_ptr(macro)), vp(_ptr(micro)),
                                               vp(_ptr(lat)), C.c_int64(chunk), vp(_stream_ptr(stream))))

    def entries_tensor(self):
        """The grid's device storage viewed as an int32 [n_entries, 8] torch tensor (no copy).
        Taking it invalidates the run index (gathers fall back to reading the
        entries) until finalize() or a full sweep() rebuilds it."""
        ent, n = C.c_void_p(), C.c_int64()
        check(lib().wt_grid_storage(self.handle, C.byref(ent), C.byref(n), None, None))
        import torch

        class _Cuda:
            pass

        holder = _Cuda()
        holder.__cuda_array_interface__ = {
            "shape": (self.n_entries, 8), "typestr": "<i4", "data": (self.entries_ptr, False), "version": 3,
            "strides": None,
        }
        return torch.as_tensor(holder, device=f"cuda:{self.engine.device}")


def _np_from(ptr, n, dt):
    if n == 0 or not ptr:
        return np.zeros(0, dt)
    ct = {np.int32: C.c_int32, np.int64: C.c_int64, np.float64: C.c_double}[dt]
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(n,)).copy()


def ipc_open(handle: bytes, offset: int, device: int = 0):
    """Map a peer's grid storage (wt_ipc_open): returns (entries address, base)."""
    h = (C.c_char * 64).from_buffer_copy(handle)
    ent, base = C.c_void_p(), C.c_void_p()
    check(lib().wt_ipc_open(h, C.c_int64(offset), C.c_int(device), C.byref(ent), C.byref(base)))
    return ent.value, base.value


def ipc_close(base):
    check(lib().wt_ipc_close(C.c_void_p(base)))


def fit_build(records: dict, registry_ids, W: int = 0, p: int = 10, device: int = 0):
    """build_dual_table on the GPU (K2).  records: dict of numpy arrays
    g, l (int64), w, macro, micro (int32), lat (float64).  Returns the built
    tables as CSR numpy arrays (same layout as the engine's input) plus
    diagnostics and the device time."""
    keep = []

    def arr(x, dt):
        a = np.ascontiguousarray(x, dtype=dt)
        keep.append(a)
        return a.ctypes.data

    rd = wt_records_desc()
    rd.n = len(records["g"])
    rd.g, rd.l = arr(records["g"], np.int64), arr(records["l"], np.int64)
    rd.w = arr(records["w"], np.int32)
    rd.macro_id, rd.micro_id = arr(records["macro"], np.int32), arr(records["micro"], np.int32)
    rd.latency_us = arr(records["lat"], np.float64)
    ids = np.ascontiguousarray(registry_ids, np.int32)
    h = C.c_void_p()
    res = wt_build_result()
    check(lib().wt_fit_build(C.byref(rd), C.c_void_p(ids.ctypes.data), C.c_int32(len(ids)), C.c_int32(W),
                             C.c_int32(p), C.c_int(device), C.byref(h), C.byref(res)))
    out = _result_dict(res)
    lib().wt_build_free(h)
    return out


def _result_dict(res):
    nt = res.n_tables
    co_off = _np_from(res.coeff_off, nt + 1, np.int32)
    aw_off = _np_from(res.awave_off, nt + 1, np.int32)
    ex_off = _np_from(res.ext_aoff, nt + 1, np.int32)
    ncoef, naw, next_ = int(co_off[-1]), int(aw_off[-1]), int(ex_off[-1])
    aw_aoff = _np_from(res.awave_aoff, naw + 1, np.int32)
    nan = int(aw_aoff[-1])
    out = dict(
        n_tables=nt, W=res.W, p=res.p, device_ms=res.device_ms,
        macro_id=_np_from(res.macro_id, nt, np.int32), theta_ext=_np_from(res.theta_ext, 4 * nt, np.float64),
        ext_flags=_np_from(res.ext_flags, nt, np.int32), coeff_off=co_off,
        coeff_w=_np_from(res.coeff_w, ncoef, np.int32), coeff_theta=_np_from(res.coeff_theta, 4 * ncoef, np.float64),
        diag_r2=_np_from(res.diag_r2, ncoef, np.float64), diag_mape=_np_from(res.diag_mape, ncoef, np.float64),
        diag_samples=_np_from(res.diag_samples, ncoef, np.int32),
        diag_flags=_np_from(res.diag_flags, ncoef, np.int32), awave_off=aw_off,
        awave_w=_np_from(res.awave_w, naw, np.int32), awave_aoff=aw_aoff,
        anchor_l=_np_from(res.anchor_l, nan, np.int64), anchor_micro=_np_from(res.anchor_micro, nan, np.int32),
        anchor_partial=_np_from(res.anchor_partial, nan, np.int32), ext_aoff=ex_off,
        ext_l=_np_from(res.ext_l, next_, np.int64), ext_micro=_np_from(res.ext_micro, next_, np.int32))
    out["W_arr"] = np.full(nt, res.W, np.int32)
    if res.step_off:  # ablation baselines from the same selected samples (tuner.cpp:191-220)
        s_off = _np_from(res.step_off, nt + 1, np.int32)
        out.update(step_off=s_off, step_l=_np_from(res.step_l, int(s_off[-1]), np.int64),
                   step_t=_np_from(res.step_t, int(s_off[-1]), np.float64),
                   lin_theta=_np_from(res.lin_theta, 4 * nt, np.float64),
                   lin_r2=_np_from(res.lin_r2, nt, np.float64), lin_mape=_np_from(res.lin_mape, nt, np.float64),
                   lin_degenerate=_np_from(res.lin_degenerate, nt, np.int32))
    return out


TABLE_KEYS = ("macro_id", "theta_ext", "coeff_off", "coeff_w", "coeff_theta", "awave_off", "awave_w", "awave_aoff",
              "anchor_l", "anchor_micro", "ext_aoff", "ext_l", "ext_micro")


def engine_tables(fit: dict) -> dict:
    """The tables of a fit result in wt_engine_create's input layout."""
    t = {k: fit[k] for k in TABLE_KEYS}
    t["W"] = fit["W_arr"]
    return t


class Build:
    """A K2 build whose tables stay on the device (wt_fit_build_device):
    records are device tensors, work is stream-ordered, and the engine is
    made from the device tables (Engine.from_build) without a host copy."""

    FIT_BASELINES = 1

    def __init__(self, records: dict, registry_ids, W: int = 0, p: int = 10, flags: int = 0, device: int = 0,
                 stream=None):
        rd = wt_records_desc()
        rd.n = int(records["g"].numel())
        rd.g, rd.l, rd.w = _ptr(records["g"]), _ptr(records["l"]), _ptr(records["w"])
        rd.macro_id, rd.micro_id = _ptr(records["macro"]), _ptr(records["micro"])
        rd.latency_us = _ptr(records["lat"])
        self._ids = np.ascontiguousarray(registry_ids, np.int32)
        h = C.c_void_p()
        check(lib().wt_fit_build_device(C.byref(rd), C.c_void_p(self._ids.ctypes.data), C.c_int32(len(self._ids)),
                                        C.c_int32(W), C.c_int32(p), C.c_int32(flags), C.c_int(device),
                                        vp(_stream_ptr(stream)), C.byref(h)))
        self.handle = h
        self.device = device

    @classmethod
    def _wrap(cls, handle, device):
        b = cls.__new__(cls)
        b.handle, b.device, b._ids = handle, device, None
        return b

    def pack_info(self):
        """(counts [n_tables, n_buckets, n_groups, W, p] int64, packed bytes)."""
        counts = np.zeros(5, np.int64)
        nbytes = C.c_size_t()
        check(lib().wt_build_pack_info(self.handle, vp(counts.ctypes.data), C.byref(nbytes)))
        return counts, nbytes.value

    def pack(self, dst, stream=None):
        """Pack the device tables into `dst` (a uint8 device tensor)."""
        check(lib().wt_build_pack(self.handle, vp(dst.data_ptr()), C.c_size_t(dst.numel()),
                                  vp(_stream_ptr(stream))))

    @classmethod
    def merge(cls, packed, stride: int, counts, device: int = 0, stream=None):
        """One build from n packed parts (packed: uint8 device tensor of
        n * stride bytes, counts: [n, 5] as pack_info reported them)."""
        counts = np.ascontiguousarray(counts, np.int64).reshape(-1, 5)
        h = C.c_void_p()
        check(lib().wt_build_merge(vp(packed.data_ptr()), C.c_size_t(stride), C.c_int32(len(counts)),
                                   vp(counts.ctypes.data), C.c_int(device), vp(_stream_ptr(stream)), C.byref(h)))
        return cls._wrap(h, device)

    def result(self) -> dict:
        """Host copies of the tables + diagnostics (wt_build_result_get)."""
        res = wt_build_result()
        check(lib().wt_build_result_get(self.handle, C.byref(res)))
        return _result_dict(res)

    def close(self):
        if getattr(self, "handle", None):
            lib().wt_build_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fit_bucket_batch(g, l, t, off, device: int = 0):
    """fit_bucket for many buckets at once: bucket b = samples [off[b], off[b+1])."""
    g, l, t = (np.ascontiguousarray(x, np.float64) for x in (g, l, t))
    off = np.ascontiguousarray(off, np.int64)
    nb = len(off) - 1
    co = np.zeros(4 * nb, np.float64)
    r2 = np.zeros(nb, np.float64)
    mape = np.zeros(nb, np.float64)
    dg = np.zeros(nb, np.int32)
    check(lib().wt_fit_bucket_batch(vp(g.ctypes.data), vp(l.ctypes.data), vp(t.ctypes.data), vp(off.ctypes.data),
                                    C.c_int64(nb), vp(co.ctypes.data), vp(r2.ctypes.data), vp(mape.ctypes.data),
                                    vp(dg.ctypes.data), C.c_int(device)))
    return co.reshape(nb, 4), r2, mape, dg


# ---------------------------------------------------------------- simulator
class wt_sim_profile_desc(C.Structure):
    _fields_ = [("n_points", C.c_int64), ("point_g", vp), ("n_anchors", C.c_int64), ("anchor_l", vp),
                ("n_pairs", C.c_int64), ("pair_macro", vp), ("pair_micro", vp), ("pair_base", vp),
                ("pair_per_iter", vp), ("pair_gap", vp), ("sigma", C.c_double), ("floor_frac", C.c_double),
                ("seed", C.c_uint64), ("warmup", C.c_int32), ("measured", C.c_int32), ("slots", C.c_int32)]


def simulate_batch(g, mean, sigma, eps, gap, seed, slots, device=0):
    """Makespans of independent wave simulations (wave_sim.cpp:80-117)."""
    g = np.ascontiguousarray(g, np.int64)
    arrs = [np.ascontiguousarray(np.broadcast_to(x, g.shape), np.float64) for x in (mean, sigma, eps, gap)]
    seed = np.ascontiguousarray(np.broadcast_to(seed, g.shape), np.uint64)
    out = np.zeros(len(g), np.float64)
    check(lib().wt_simulate_batch(vp(g.ctypes.data), *[vp(a.ctypes.data) for a in arrs], vp(seed.ctypes.data),
                                  C.c_int64(len(g)), C.c_int32(slots), vp(out.ctypes.data), C.c_int(device)))
    return out


def profile_sim(point_g, anchors, pair_macro, pair_micro, base, per_iter, gap, sigma, seed, slots, warmup=3,
                measured=5, floor_frac=0.01, device=0):
    """SimulatorBackend sweep: latencies for (point, anchor, pair) in run_profile order."""
    keep = []

    def arr(x, dt):
        a = np.ascontiguousarray(x, dtype=dt)
        keep.append(a)
        return a.ctypes.data

    d = wt_sim_profile_desc()
    d.n_points, d.point_g = len(point_g), arr(point_g, np.int64)
    d.n_anchors, d.anchor_l = len(anchors), arr(anchors, np.int64)
    d.n_pairs = len(pair_macro)
    d.pair_macro, d.pair_micro = arr(pair_macro, np.int32), arr(pair_micro, np.int32)
    d.pair_base, d.pair_per_iter, d.pair_gap = arr(base, np.float64), arr(per_iter, np.float64), arr(gap, np.float64)
    d.sigma, d.floor_frac, d.seed = sigma, floor_frac, seed
    d.warmup, d.measured, d.slots = warmup, measured, slots
    total = d.n_points * d.n_anchors * d.n_pairs
    lat = np.zeros(total, np.float64)
    st = np.zeros(total, np.int32)
    ms = C.c_double()
    check(lib().wt_profile_sim(C.byref(d), vp(lat.ctypes.data), vp(st.ctypes.data), C.c_int(device), C.byref(ms)))
    return lat, st, ms.value
