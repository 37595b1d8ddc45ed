"""Artifact / record formats (paper_2604_10187_b200.artifact) on CPU:
binary SoA images round-trip bit-exactly (memmap views), the reference's
tables JSON and dataset CSV -- produced by the reference itself
(oracle/_ref) -- parse to exactly the arrays the oracle's parser gives, the
CSV writer reproduces the reference's bytes, and the reference's error
texts are kept."""
import os

import numpy as np
import pytest

import pyoracle as po
import wtutil as U
from paper_2604_10187_b200 import artifact as A, synthetic as S


def _same(a, b):
    for k in b:
        x, y = np.asarray(a[k]), np.asarray(b[k])
        assert x.dtype == y.dtype, k
        if x.dtype == np.float64:
            np.testing.assert_array_equal(x.view(np.int64), y.view(np.int64), err_msg=k)
        else:
            np.testing.assert_array_equal(x, y, err_msg=k)


def test_tables_bin_roundtrip_is_bit_exact(tmp_path):
    cfg = S.config_space(False)
    t = S.synthetic_tables(cfg)
    t = {k: np.asarray(v, A.TABLE_FIELDS[k]) for k, v in t.items() if k in A.TABLE_FIELDS}
    t["theta_ext"][3] = -0.0
    t["coeff_theta"][5] = np.nextafter(1.0, 2.0)
    p = str(tmp_path / "t.wtt")
    A.save_tables_bin(p, t, p=7)
    got = A.load_tables_bin(p)
    assert isinstance(got["coeff_theta"], np.memmap) and got["p"] == 7 and got["schema_version"] == 1
    _same(got, t)
    _same(A.load_tables_bin(p, mmap=False), t)


def test_records_bin_roundtrip_and_csv_bytes(tmp_path):
    cfg = S.config_space(False)
    rec = S.synthetic_records(cfg)
    rec = {k: np.asarray(v, A.RECORD_FIELDS[k]) for k, v in rec.items()}
    p = str(tmp_path / "r.wtr")
    A.save_records_bin(p, rec)
    _same(A.load_records_bin(p), rec)
    sub = {k: v[:2000] for k, v in rec.items()}
    c = str(tmp_path / "r.csv")
    A.save_records_csv(c, sub)
    _same(A.load_records_csv(c), sub)


@pytest.fixture(scope="module")
def ref_fixture(tmp_path_factory):
    ref = po.Reference()
    return U.reference_fixture(ref, tmp_path_factory.mktemp("ref"))


def test_reference_tables_json_parses_exactly(ref_fixture):
    reg, rec, tab = ref_fixture
    got = A.load_tables_json(tab)
    want = U.arrays_from_pytables(po.parse_tables_json(tab)[1])
    _same(got, want)


def test_reference_csv_parses_and_rewrites_byte_identical(ref_fixture, tmp_path):
    reg, rec, tab = ref_fixture
    got = A.load_records_csv(rec)
    _same(got, po.read_records_csv(rec))
    out = str(tmp_path / "again.csv")
    A.save_records_csv(out, got)
    with open(rec, "rb") as f1, open(out, "rb") as f2:
        assert f1.read() == f2.read()


def test_reference_error_texts(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text('{"schema_version": 2, "kernel_family": "dense_gemm", "tables": []}')
    with pytest.raises(RuntimeError, match="expected 1, found 2"):
        A.load_tables_json(str(bad))
    c = tmp_path / "bad.csv"
    c.write_text("g,l,w,macro,micro,lat\n")
    with pytest.raises(RuntimeError, match="bad dataset header"):
        A.load_records_csv(str(c))
    c.write_text("g,l,w,macro_id,micro_id,latency_us\n1,2,3,4,5,-1\n")
    with pytest.raises(RuntimeError, match="non-positive latency in dataset row: 1,2,3,4,5,-1"):
        A.load_records_csv(str(c))
    c.write_text("g,l,w,macro_id,micro_id,latency_us\n1,2,3\n")
    with pytest.raises(RuntimeError, match="malformed dataset row"):
        A.load_records_csv(str(c))
