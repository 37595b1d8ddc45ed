"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every entry point include/wavetune_c.h declares; validation errors
surface with the reference's exception kind and message before any device
work; the C++ drop-in's host plumbing (mapping, plans, artefact formats)
matches the reference byte for byte."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import pyoracle as po
import wtutil as U
from conftest import ROOT, have_reference_build

HEADER = os.path.join(ROOT, "include", "wavetune_c.h")


@pytest.fixture(scope="module")
def capi():
    from paper_2604_10187_b200 import capi as c

    c.lib()
    return c


@pytest.fixture(scope="module")
def core():
    from paper_2604_10187_b200 import _core

    return _core


def test_header_symbols_exported(capi):
    text = open(HEADER).read()
    decl = set(re.findall(r"^\s*(?:const char\*|int64_t|int32_t|int|wt_status)\s+(wt_\w+)\(", text, re.M))
    assert len(decl) >= 20
    lib = capi.lib()
    missing = [s for s in decl if not hasattr(lib, s)]
    assert not missing, missing
    assert set(capi.EXPORTS) == decl
    assert lib.wt_abi_version() == 1
    assert b"sm_100a" in lib.wt_version()


def _engine_status(capi, tables, registry, n_sm=148, bps=1):
    try:
        capi.Engine(tables, registry, n_sm=n_sm, blocks_per_sm=bps)
    except capi.WtError as e:
        return e.status, e.msg
    return 0, ""


def test_engine_validation_matches_reference_errors(capi):
    from paper_2604_10187_b200 import synthetic as S

    cfg = S.config_space(False)
    t = S.synthetic_tables(cfg)
    reg = S.registry_arrays(cfg)
    # duplicate macro ids: std::sort leaves their order unspecified -> rejected
    t2 = dict(t)
    t2["macro_id"] = t["macro_id"].copy()
    t2["macro_id"][5] = t2["macro_id"][4]
    st, msg = _engine_status(capi, t2, reg)
    assert st == capi.WT_INVALID_ARGUMENT and "duplicate macro_id" in msg
    # table id absent from the registry: registry.macro(id) -> out_of_range
    r2 = dict(reg)
    r2["id"] = reg["id"].copy()
    r2["id"][7] = 100000
    st, msg = _engine_status(capi, t, r2)
    assert st == capi.WT_OUT_OF_RANGE and msg == "no macro config with id 7"
    # hardware capacity (kernel_map.cpp:268-269)
    st, msg = _engine_status(capi, t, reg, n_sm=0)
    assert st == capi.WT_INVALID_ARGUMENT and msg == "hardware spec must have positive capacities"
    # no tables (tuner.cpp:120)
    empty = {k: (v[:1] if k.endswith("off") else v[:0]) for k, v in t.items()}
    st, msg = _engine_status(capi, empty, reg)
    assert st == capi.WT_INVALID_ARGUMENT and msg == "no dual tables provided"


def test_core_mapping_golden(core):
    wt = core
    hw = wt.HardwareSpec(132)
    macro = wt.MacroConfig(0, wt.GemmTiles(128, 256, 64))
    assert wt.map_workload(wt.DenseGemm(4096, 4096, 4096), macro) == (512, 64)  # test_smoke.py:36-45
    assert wt.wave_count(512, hw) == 4
    assert wt.map_workload(wt.DenseGemm(128, 64, 4096), wt.MacroConfig(0, wt.GemmTiles(128, 64, 64))) == (1, 64)
    assert wt.map_workload(wt.GroupedGemm([100, 0, 50], 128, 64), wt.MacroConfig(0, wt.GemmTiles(128, 64, 64))) == (4, 1)
    assert wt.map_workload(wt.FlashAttention(16, 512, 2048), wt.MacroConfig(0, wt.AttnTiles(64, 64))) == (128, 32)
    with pytest.raises(ValueError):
        wt.map_workload(wt.GroupedGemm([0, 0], 128, 64), wt.MacroConfig(0, wt.GemmTiles(128, 64, 64)))
    with pytest.raises(ValueError):
        wt.map_workload(wt.DenseGemm(1, 1, 1), wt.MacroConfig(0, wt.AttnTiles(64, 64)))
    for gg, sm, bps, want in ((10, 4, 1, 3), (132, 132, 1, 1), (133, 132, 1, 2), (264, 132, 2, 1)):
        assert wt.wave_count(gg, wt.HardwareSpec(sm, bps)) == want
    for text in ("dense_gemm,4096,4096,2048", "flash_attention,16,512,2048", "grouped_gemm,768,2048,100;0;50"):
        assert wt.workload_to_string(wt.parse_workload(text)) == text
    with pytest.raises(ValueError):
        wt.parse_workload("dense_gemm,1,2")
    x = wt.instantiate_workload(11, 12, 64, wt.MacroConfig(0, wt.GemmTiles(128, 64, 64)))
    assert (x.m, x.n, x.k) == (1408, 768, 4096)


@pytest.mark.skipif(not have_reference_build(), reason="oracle/_ref not built")
def test_plan_bytes_match_reference(core, tmp_path):
    ref = po.Reference()
    for (sm, W, I, tau, anchors) in ((148, 40, 4, 1.1, [16, 32, 48, 64, 80]), (132, 3, 4, 1.2, [16, 32, 64]),
                                     (10, 2, 3, 4.0, [8])):
        a, b = str(tmp_path / "ref.json"), str(tmp_path / "ours.json")
        assert ref.build_plan(sm, 1, W, I, tau, anchors, a) == 0
        core.build_plan(core.HardwareSpec(sm, 1, "ref"), "dense_gemm", W=W, I=I, tau=tau, loop_anchors=anchors).save(b)
        assert open(a, "rb").read() == open(b, "rb").read()


@pytest.mark.skipif(not have_reference_build(), reason="oracle/_ref not built")
def test_artefacts_round_trip_byte_identical(core, tmpdir_session, tmp_path):
    """Registry JSON, records CSV and tables JSON written by the reference are
    read and re-written by the drop-in byte for byte (A8's identity)."""
    ref = po.Reference()
    reg, rec, tab = U.reference_fixture(ref, tmpdir_session)
    r = core.ConfigRegistry.load(reg)
    r.save(str(tmp_path / "reg.json"))
    assert open(reg, "rb").read() == open(tmp_path / "reg.json", "rb").read()
    recs = core.read_records(rec)
    core.write_records(recs, str(tmp_path / "rec.csv"))
    assert open(rec, "rb").read() == open(tmp_path / "rec.csv", "rb").read()
    art = core.load_tables(tab)
    core.save_tables(art, str(tmp_path / "tab.json"))
    assert open(tab, "rb").read() == open(tmp_path / "tab.json", "rb").read()
    # and the reference reads ours back identically
    assert ref.resave_tables(str(tmp_path / "tab.json"), str(tmp_path / "tab2.json")) == 0
    assert open(tab, "rb").read() == open(tmp_path / "tab2.json", "rb").read()
    bad = tmp_path / "bad.json"
    bad.write_text('{"schema_version": 99, "kernel_family": "dense_gemm", "tables": []}')
    with pytest.raises(RuntimeError, match="expected 1, found 99"):
        core.load_tables(str(bad))


def test_records_replay_profile(core, tmp_path):
    """run_profile through the CsvReplayBackend plugin: replayed latencies are
    exact and a miss is an error (test_profiler.cpp:163-178)."""
    wt = core
    hw = wt.HardwareSpec(132)
    reg = wt.ConfigRegistry()
    reg.family = "dense_gemm"
    reg.macros = [wt.MacroConfig(0, wt.GemmTiles(64, 64, 64)), wt.MacroConfig(1, wt.GemmTiles(128, 128, 64))]
    reg.micros = [wt.MicroConfig(0, 2, 4), wt.MicroConfig(1, 3, 4)]
    for a in (0, 1):
        for b in (0, 1):
            reg.add_feasible(a, b)
    reg.validate()
    plan = wt.build_plan(hw, "dense_gemm", W=2, I=2, tau=1.5, loop_anchors=[8, 16])
    recs = []
    for p in plan.grid_points:
        for l in (8, 16):
            for a in (0, 1):
                for b in (0, 1):
                    recs.append(wt.ProfileRecord(p.g, l, wt.wave_count(p.g, hw), a, b, 10.0 + p.g * 0.1 + l + a + 0.5 * b))
    out = wt.run_profile_replay(plan, reg, recs)
    assert [r.latency_us for r in out] == [r.latency_us for r in recs]
    # a miss is skipped with a log line (profiler.cpp:309-319) ...
    assert len(wt.run_profile_replay(plan, reg, recs[:-1])) == len(recs) - 1
    # ... and more than 10% misses abort the run (:324-327)
    with pytest.raises(RuntimeError, match="profiling aborted"):
        wt.run_profile_replay(plan, reg, recs[: len(recs) // 2])


def test_gemm_family_symbols_and_registry(core):
    """lib/libwtgemm.so exports every entry point include/wavetune_gemm.h
    declares; the family registry is valid and maps back onto instantiations."""
    from paper_2604_10187_b200 import gemm

    text = open(os.path.join(ROOT, "include", "wavetune_gemm.h")).read()
    decl = set(re.findall(r"^\s*int\s+(wt_gemm_\w+)\(", text, re.M))
    assert len(decl) == 6
    lib = gemm.lib()
    assert not [s for s in decl if not hasattr(lib, s)]
    fam = gemm.family()
    assert len(fam) == lib.wt_gemm_family_size() >= 10
    # swap-AB small-M tiles (BM 32 / 64), 1-SM (128) and CTA-pair (256) tiles; whole 64-element swizzle atoms
    assert all(bk in (64, 128) and bm in (32, 64, 128, 256) for bm, bn, bk, st in fam)
    assert {bm for bm, *_ in fam} == {32, 64, 128, 256} and {bk for _, _, bk, _ in fam} == {64, 128}
    reg = core.gemm_registry()
    assert len(reg.feasible) == 4 * len(fam)
    for ma, mi in reg.feasible:
        cfg = core.B200GemmBackend.family_config(reg.macro(ma), reg.micro(mi))
        bm, bn, bk, st = fam[cfg]
        t = reg.macro(ma).tiles
        assert (t.t_m, t.t_n, t.t_k, reg.micro(mi).n_stages) == (bm, bn, bk, st)
    # argument validation happens before any device work
    assert lib.wt_gemm_config(len(fam), None, None, None, None) == 3
    assert lib.wt_gemm_run(0, 3, 128, 128, 64, 1, 1, 1, None) == 1
    assert lib.wt_gemm_run(0, 1, 0, 128, 64, 1, 1, 1, None) == 1
