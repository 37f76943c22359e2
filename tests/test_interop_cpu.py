"""On-disk formats and trace reporting against files and values written by
the reference itself (tests/golden/make_golden.py `interop`): the CTKV dump
(ck/workload.py:247-287) and summarize_trace / TraceRow.as_record
(ck/session.py:67-100, ck/retrieval.py:76-108).  CPU only; the QIVF index
half is in tests/test_parity_gpu.py (the index lives on the device)."""

import json
import os

import numpy as np
import pytest

import paper_2512_15550_b200 as P
from paper_2512_15550_b200.retrieval import TraceRow

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _doc():
    with open(os.path.join(HERE, "interop.json")) as fh:
        return json.load(fh)


def test_read_dump_of_a_reference_file_and_byte_identical_rewrite(tmp_path):
    src = os.path.join(HERE, "interop_dump.ctkv")
    q, k, v, lay = P.read_dump(src)
    assert (lay.batch, lay.query_heads, lay.kv_heads, lay.seq_len, lay.head_dim) == (1, 4, 2, 96, 16)
    assert q.dtype == np.float32 and q.shape == (1, 4, 96, 16) and k.shape == v.shape == (1, 2, 96, 16)
    out = tmp_path / "again.ctkv"
    P.write_dump(out, q, k, v)
    assert out.read_bytes() == open(src, "rb").read()


def test_dump_errors(tmp_path):
    src = open(os.path.join(HERE, "interop_dump.ctkv"), "rb").read()
    for name, blob in (("short", src[:20]), ("magic", b"XXXX" + src[4:]),
                       ("trunc", src[:-4]), ("version", src[:4] + b"\x02" + src[5:])):
        p = tmp_path / name
        p.write_bytes(blob)
        with pytest.raises(P.FormatError):
            P.read_dump(p)
    with pytest.raises(P.ConfigError):
        P.write_dump(tmp_path / "x", np.zeros((1, 2, 3)), np.zeros((1, 1, 3, 2)), np.zeros((1, 1, 3, 2)))


def test_summarize_trace_matches_reference():
    doc = _doc()
    rows = [TraceRow(**r) for r in doc["rows"]]
    got = P.summarize_trace(rows)
    want = doc["summary"]
    assert set(got) == set(want)
    for key, val in want.items():
        if isinstance(val, float):
            assert got[key] == pytest.approx(val, rel=1e-12), key
        else:
            assert got[key] == val, key
    assert [r.as_record() for r in rows] == doc["records"]
    assert P.summarize_trace([]) == {"steps": 0}
