"""Shared loader for the golden fixtures written by tests/golden/make_golden.py."""

from __future__ import annotations

import functools
import hashlib
import json
import os

import numpy as np

from oracle import ctkv_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

SMALL = ["small_a", "small_turns_gs1", "small_norerank", "small_nodcu", "small_bf16", "small_wrap"]
CFG1 = ["cfg1", "cfg1_bf16"]


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@functools.lru_cache(maxsize=None)
def load(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        meta = json.load(fh)
    arrs = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    return meta, arrs


@functools.lru_cache(maxsize=4)
def inputs(name):
    """Regenerate the case's Q/K/V with the oracle generator (pinned by the
    reference's sha256) and apply the bf16 rounding of bf16 variants."""
    meta, _ = load(name)
    b, h, g, d = meta["dims"]
    q, k, v = O.generate(O.Drift(**meta["drift"]), b, h, g, d)
    if sha(q, k, v) != meta["gen_sha"]:
        raise AssertionError(f"{name}: oracle generator diverged from the reference")
    if meta["variant"] == "bf16":
        q, k, v = O.bf16_round(q), O.bf16_round(k), O.bf16_round(v)
    return q, k, v


def params(name):
    meta, _ = load(name)
    p = dict(meta["params"])
    flags = dict(use_dcu=meta["flags"].get("use_dcu", True),
                 use_rerank=meta["flags"].get("use_rerank", True))
    return meta, p, flags
