"""Pin the CPU oracle to the reference's own outputs (golden fixtures).

These run without a GPU.  They prove oracle/ctkv_oracle.py reproduces
centroidkv 0.1.0 bit-for-bit on: the generator, prefill lists, each decode
step's selected slots / recalled sets / sparse ids / merged output, and the
post-DCU index state.  The GPU parity tests then compare the CUDA path to
this pinned oracle (and to the same fixtures directly).
"""

import json
import os

import numpy as np
import pytest

from oracle import ctkv_oracle as O
from tests import golden_cases as G


def _run_oracle(name, steps=None):
    meta, p, flags = G.params(name)
    q, k, v = G.inputs(name)
    s = meta["drift"]["s"]
    store, index = O.prefill(np.ascontiguousarray(q[:, :, :s]), np.ascontiguousarray(k[:, :, :s]),
                             np.ascontiguousarray(v[:, :, :s]), p["init_len"], p["local_len"],
                             p["capacity"], p["rho"])
    lists0 = index.lists.copy()
    recs = []
    for t in range(steps or meta["steps"]):
        store.append(k[:, :, s + t], v[:, :, s + t])
        recs.append(O.decode_step(store, index, q[:, :, s + t], p["c_prime"], p["rho_prime"],
                                  **flags))
    return lists0, recs, index


def _pad(per_head, width):
    b, g = len(per_head), len(per_head[0])
    out = np.full((b, g, width), -1, dtype=np.int64)
    for bi in range(b):
        for gi in range(g):
            out[bi, gi, :len(per_head[bi][gi])] = per_head[bi][gi]
    return out


@pytest.mark.parametrize("name", G.SMALL)
def test_oracle_matches_reference_small(name):
    meta, arr = G.load(name)
    lists0, recs, index = _run_oracle(name)
    np.testing.assert_array_equal(lists0, arr["lists0"])
    for t, r in enumerate(recs):
        np.testing.assert_array_equal(r.selected, arr["step_selected"][t])
        np.testing.assert_array_equal(np.array([[len(x) for x in row] for row in r.recalled]),
                                      arr["step_recall_len"][t])
        width = arr["step_recalled"].shape[-1]
        np.testing.assert_array_equal(_pad(r.recalled, width), arr["step_recalled"][t])
        np.testing.assert_array_equal(_pad(r.sparse, arr["step_sparse"].shape[-1]), arr["step_sparse"][t])
        np.testing.assert_array_equal(r.out, arr["step_out"][t])
        np.testing.assert_array_equal(r.merged.row_max, arr["step_row_max"][t])
        np.testing.assert_allclose(r.merged.denom, arr["step_denom"][t], rtol=1e-12)
        assert r.digest == meta["digests"][t]
        g_ref = arr["step_grouped"][t]
        for bi in range(g_ref.shape[0]):
            for gi in range(g_ref.shape[1]):
                n = len(r.recalled[bi][gi])
                np.testing.assert_allclose(r.grouped[bi][gi], g_ref[bi, gi, :n], rtol=1e-13, atol=0)
    np.testing.assert_array_equal(index.lists, arr["lists_final"])
    np.testing.assert_array_equal(index.centroids, arr["centroids_final"])


@pytest.mark.parametrize("name", G.CFG1)
def test_oracle_matches_reference_cfg1(name):
    meta, arr = G.load(name)
    lists0, recs, index = _run_oracle(name)
    b, g = lists0.shape[:2]
    for bi in range(b):
        for gi in range(g):
            assert G.sha(lists0[bi, gi]) == meta["lists0_sha"][bi][gi]
    np.testing.assert_array_equal(lists0[:, :, ::32], arr["lists0_rows"])
    for t, r in enumerate(recs):
        np.testing.assert_array_equal(r.selected, arr["step_selected"][t])
        np.testing.assert_array_equal(_pad(r.sparse, 512), arr["step_sparse"][t])
        np.testing.assert_array_equal(r.out, arr["step_out"][t])
        assert r.digest == meta["digests"][t]
    assert G.sha(index.lists) == meta["lists_final_sha"]
    assert G.sha(index.centroids) == meta["centroids_final_sha"]


def test_oracle_kats():
    with open(os.path.join(G.GOLDEN, "kats.json")) as fh:
        kat = json.load(fh)
    e0 = np.zeros((1, 1, 1, 4), np.float32)
    e0[..., 0] = 1
    assert O.scaled_logits(e0, e0)[0, 0, 0, 0] == kat["dot_e0"] == 0.5
    np.testing.assert_allclose(O.softmax_rows(np.array([[1, 2, 3]], np.float32)), kat["softmax_123"], rtol=1e-6)
    np.testing.assert_allclose(O.softmax_rows(np.array([[1000, 0]], np.float32)), kat["softmax_1000_0"])
    gm = np.array([1, 3, 2, 0], np.float32).reshape(1, 4, 1, 1)
    assert O.head_group_max(gm, 2).ravel().tolist() == kat["group_max"] == [3.0, 2.0]
    assert O.topk_desc(np.array([5, 5, 1.0]), 1).tolist() == kat["top_k_tie"] == [0]
    c, _ = O.cos_rows(np.array([1.0, 1.0]), np.array([[1.0, 0.0]]))
    assert abs(c[0] - kat["cosine_11_10"]) < 1e-15
    st = O.partition(np.zeros((1, 1, 10, 2), np.float32), np.zeros((1, 1, 10, 2), np.float32), 2, 3)
    assert st.offloaded().tolist() == kat["partition_offloaded"] == [2, 3, 4, 5, 6]
    assert O.acceleration_factor(10000, 1000) == kat["accel_10000_1000"] == 0.6
    assert O.topk_desc(np.array(kat["top_k_ties_row"]), 37).tolist() == kat["top_k_ties_k37"]
    rows = np.array(kat["top_k_rows_in"], np.float32)
    assert O.topk_rows_desc(rows, 50).tolist() == kat["top_k_rows_k50"]
