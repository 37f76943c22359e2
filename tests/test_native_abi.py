"""CPU-only checks of the C-ABI library: it loads, exports exactly what
include/ctkv.h declares, the ctypes structs match the C layout, and the
pure-host sizing entry points answer (no kernel launches here)."""

import ctypes
import os
import re

import pytest

from paper_2512_15550_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ctkv.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ctkv_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(N.LIB_PATH):
        pytest.fail("libctkv.so not built (run __graft_entry__.build())")
    return N.load_library(require_device=False)


def test_header_and_binding_agree():
    assert _declared() == sorted(N.SIGNATURES), "ctypes SIGNATURES must mirror include/ctkv.h"


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.ctkv_abi_version() == 1
    assert lib.ctkv_status_string(2).decode().startswith("config error")


def test_struct_layouts():
    # offsets of the C structs (x86-64 SysV): see include/ctkv.h
    assert ctypes.sizeof(N.Layout) == 40 and N.Layout.capacity.offset == 16
    assert ctypes.sizeof(N.StoreDesc) == 24
    assert ctypes.sizeof(N.IndexDesc) == 48
    assert N.StepArgs.out.offset == 40 and ctypes.sizeof(N.StepArgs) == 112


def test_workspace_queries_host_only(lib):
    # cfg2 geometry: b=8, 32q/8kv, d=128, cap=98304+64, C=2048, rho=1280
    lay = N.Layout(8, 32, 8, 128, 98368, N.BF16, 128, 1024, 0)
    ws = lib.ctkv_decode_workspace_bytes(lay, 2048, 1280, 4, 512)
    # gcos U*C f64 + static partials + logits U*gs*C'rho f64
    assert ws >= 64 * 2048 * 8 + 64 * 4 * 5120 * 8
    assert lib.ctkv_build_workspace_bytes(lay, 2048, 1280, 97152, N.BUILD_FAST) > 0
    bad = N.Layout(8, 30, 8, 128, 98368, N.BF16, 128, 1024, 0)   # h % g != 0
    assert lib.ctkv_decode_workspace_bytes(bad, 2048, 1280, 4, 512) == 0


def test_errors_map_to_reference_types(lib):
    from paper_2512_15550_b200.errors import ConfigError, ShapeError
    with pytest.raises(ShapeError):
        N.check(N.ESHAPE, "x")
    with pytest.raises(ConfigError):
        N.check(N.ECONFIG, "x")
    with pytest.raises(IndexError):
        N.check(N.EINDEX, "x")
    with pytest.raises(ConfigError):
        N.raise_flags(N.FLAG_EMPTY_RECALL | N.FLAG_NONEMPTY_RECALL, "step")


def test_device_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        N.load_library(require_device=True)


def test_padded_digest_equals_reference_digest():
    """retrieval.digest_padded (one sha256 over the padded id array) equals
    the per-head digest of ck/retrieval.py:295-301 that trace rows carry."""
    import numpy as np
    from paper_2512_15550_b200.retrieval import _split_per_head, digest, digest_padded
    rng = np.random.default_rng(5)
    pad = rng.integers(0, 1 << 20, size=(3, 4, 64), dtype=np.int32)
    lens = rng.integers(0, 65, size=(3, 4)).astype(np.int32)
    lens[0, 0] = 0
    assert digest_padded(pad, lens) == digest(_split_per_head(pad, lens))
