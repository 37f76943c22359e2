"""Decode-time retrieval API (ck/retrieval.py), backed by the sm_100a kernels.

`decode_step` is the hot path: one call = two kernels (scan + unit, see
csrc/ctkv_decode.cu) that run recall -> rerank -> sparse/static attention
-> merge -> FIFO DCU entirely on the device.  The staged functions
(`recall`, `rerank`, `sparse_attention`, `merge`) expose each stage on its
own through the same kernels so every stage is parity-testable, and they
return the reference's host types (numpy, PerHead nested lists).
"""

from __future__ import annotations

import hashlib
import dataclasses
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, ShapeError
from .index import QueryCentroidIndex
from .store import KvStore
from .tensor_ops import is_host, like_input, to_device

PerHead = list  # [batch][kv_head] -> 1-D id / score arrays


@dataclass
class RecallResult:
    """ck/retrieval.py:30-41 (+ the device copies the next stage reuses)."""

    selected: np.ndarray
    recalled: PerHead
    recall_len: np.ndarray
    alpha: np.ndarray
    _dev: tuple | None = field(default=None, repr=False, compare=False)


@dataclass
class RerankResult:
    sparse_ids: PerHead
    rerank_len: np.ndarray


@dataclass
class AttentionPartial:
    out: np.ndarray        # [b,h,d] float32
    row_max: np.ndarray    # [b,h] float64
    denom: np.ndarray      # [b,h] float64


@dataclass
class DecodeConfig:
    c_prime: int
    rho_prime: int
    use_dcu: bool = True
    use_rerank: bool = True
    keep_sets: bool = False

    def __post_init__(self):
        if self.c_prime < 1:
            raise ConfigError(f"c_prime must be >= 1, got {self.c_prime}")
        if self.rho_prime < 1:
            raise ConfigError(f"rho_prime must be >= 1, got {self.rho_prime}")


@dataclass
class TraceRow:
    """ck/retrieval.py:76-108."""

    step: int
    recall_len: int
    alpha: float
    rerank_len: int
    sparse_digest: str
    macs_rerank_qk: int = 0
    macs_sparse_qk: int = 0
    macs_sparse_wv: int = 0
    recall_at_k: float | None = None
    round_index: int | None = None
    recalled: PerHead | None = None
    sparse: PerHead | None = None

    def as_record(self) -> dict:
        rec = {
            "step": self.step,
            "recall_len": self.recall_len,
            "alpha": round(self.alpha, 6),
            "rerank_len": self.rerank_len,
            "sparse_digest": self.sparse_digest,
            "macs_rerank_qk": self.macs_rerank_qk,
            "macs_sparse_qk": self.macs_sparse_qk,
            "macs_sparse_wv": self.macs_sparse_wv,
        }
        if self.recall_at_k is not None:
            rec["recall_at_k"] = round(self.recall_at_k, 6)
        if self.round_index is not None:
            rec["round"] = self.round_index
        return rec


@dataclass
class DecodeState:
    store: KvStore
    index: QueryCentroidIndex
    config: DecodeConfig
    oracle: object | None = None
    step: int = 0
    trace: list = field(default_factory=list)
    # device step buffers and pinned host mirrors, reused across decode_step
    # calls (rebuilt when the workspace size or the config changes)
    _cache: tuple | None = field(default=None, repr=False, compare=False)


# ---------------------------------------------------------------------------

def _as_query(query, b, h, d, dtype) -> torch.Tensor:
    """ck/retrieval.py:121-129 -> contiguous device [b,h,d]."""
    q = to_device(query, dtype)
    if q.dim() == 4:
        if tuple(q.shape) != (b, h, 1, d):
            raise ShapeError(f"query shape {tuple(q.shape)} != {(b, h, 1, d)}")
        q = q[:, :, 0, :]
    if tuple(q.shape) != (b, h, d):
        raise ShapeError(f"query shape {tuple(q.shape)} != {(b, h, d)}")
    return q.contiguous()


def _flags_check(flags: torch.Tensor, what: str, **kw) -> int:
    f = int(flags.item())
    N.raise_flags(f, what, **kw)
    return f


def _ws(nbytes: int, device) -> torch.Tensor:
    # zero-filled: the decode kernels' completion counters start at 0 and
    # are left at 0 by the CTA that consumes them (include/ctkv.h)
    return torch.zeros(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def _pad_per_head(per_head, b, g):
    lens = np.zeros((b, g), dtype=np.int32)
    for bi in range(b):
        for gi in range(g):
            lens[bi, gi] = len(per_head[bi][gi])
    lmax = max(int(lens.max()) if lens.size else 0, 1)
    pad = np.full((b, g, lmax), -1, dtype=np.int32)
    for bi in range(b):
        for gi in range(g):
            a = per_head[bi][gi]
            a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
            pad[bi, gi, :a.size] = a
    return pad, lens, lmax


def _split_per_head(pad: np.ndarray, lens: np.ndarray, dtype=np.int64) -> PerHead:
    b, g = lens.shape
    return [[pad[bi, gi, :lens[bi, gi]].astype(dtype) for gi in range(g)] for bi in range(b)]


# ---------------------------------------------------------------------------
# staged API
# ---------------------------------------------------------------------------

def recall(index: QueryCentroidIndex, query, c_prime: int) -> RecallResult:
    """Alg. 2 L1-4 (ck/retrieval.py:132-168) on the device."""
    if index.capacity == 0:
        raise ConfigError("recall: empty index")
    if c_prime < 1 or c_prime > index.capacity:
        raise ConfigError(f"recall: c_prime {c_prime} outside [1, {index.capacity}]")
    lay = index.layout
    b, h, g, d = lay.batch, lay.query_heads, lay.kv_heads, lay.head_dim
    q = _as_query(query, b, h, d, index.dtype)
    lib = N.lib()
    lmax = max(c_prime * index.rho, 1)
    dev = q.device
    sel = torch.empty((b, g, c_prime), dtype=torch.int32, device=dev)
    rec = torch.empty((b, g, lmax), dtype=torch.int32, device=dev)
    lens = torch.empty((b, g), dtype=torch.int32, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    clay = index.ctkv_layout()
    ws = _ws(lib.ctkv_decode_workspace_bytes(clay, index.capacity, index.rho, c_prime, 1), dev)
    N.check(lib.ctkv_recall(clay, index.desc(), index.id_bound, N.ptr(q), c_prime, N.ptr(sel),
                            N.ptr(rec), N.ptr(lens), N.ptr(flags), N.ptr(ws), ws.numel(),
                            N.stream_ptr()), "recall")
    _flags_check(flags, "recall", recall_mixed_is_error=False)
    lens_np = lens.cpu().numpy().astype(np.int64)
    rec_np = rec.cpu().numpy()
    denom = c_prime * index.rho
    alpha = lens_np / denom if denom else np.zeros((b, g), dtype=np.float64)
    return RecallResult(sel.cpu().numpy().astype(np.int64), _split_per_head(rec_np, lens_np),
                        lens_np, alpha.astype(np.float64), _dev=(rec, lens, lmax))


def _recall_dev(rec: RecallResult, b, g):
    if rec._dev is not None:
        return rec._dev
    pad, lens, lmax = _pad_per_head(rec.recalled, b, g)
    return to_device(pad), to_device(lens), lmax


def rerank(store: KvStore, query, recall_result: RecallResult, rho_prime: int):
    """Alg. 2 L5-6 (ck/retrieval.py:196-218): (RerankResult, grouped scores)."""
    lay = store.layout
    if int(np.asarray(recall_result.recall_len).sum()) == 0:
        raise ConfigError("rerank: empty recall set")
    b, h, g, d = lay.batch, lay.query_heads, lay.kv_heads, lay.head_dim
    q = _as_query(query, b, h, d, store.dtype)
    rec_d, len_d, lmax = _recall_dev(recall_result, b, g)
    dev = q.device
    grouped = torch.empty((b, g, lmax), dtype=torch.float64, device=dev)
    order = torch.empty((b, g, lmax), dtype=torch.int32, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = N.lib()
    clay = store.ctkv_layout()
    ws = _ws(lib.ctkv_decode_workspace_bytes(clay, 1, lmax, 1, 1), dev)
    N.check(lib.ctkv_rerank(clay, store.desc(), N.ptr(q), N.ptr(rec_d), N.ptr(len_d), lmax,
                            N.ptr(grouped), N.ptr(order), N.ptr(flags), N.ptr(ws), ws.numel(),
                            N.stream_ptr()), "rerank")
    _flags_check(flags, "rerank", recall_mixed_is_error=False)
    lens = len_d.cpu().numpy()
    order_np = order.cpu().numpy()
    grouped_np = grouped.cpu().numpy()
    sparse, gr = [], []
    rlen = np.zeros((b, g), dtype=np.int64)
    for bi in range(b):
        srow, grow = [], []
        for gi in range(g):
            L = int(lens[bi, gi])
            ids = np.asarray(recall_result.recalled[bi][gi], dtype=np.int64)
            keep = order_np[bi, gi, :min(rho_prime, L)]
            srow.append(ids[keep])
            grow.append(grouped_np[bi, gi, :L].copy())
            rlen[bi, gi] = keep.size
        sparse.append(srow)
        gr.append(grow)
    return RerankResult(sparse, rlen), gr


def _normalize_ids(store: KvStore, ids) -> tuple[bool, object]:
    """ck/retrieval.py:267-272: shared id sequence or [b][g] nested lists."""
    if isinstance(ids, (np.ndarray, torch.Tensor)) or ids == [] or (
            isinstance(ids, (list, tuple)) and ids and np.isscalar(ids[0])):
        arr = ids.detach().cpu().numpy() if isinstance(ids, torch.Tensor) else np.asarray(ids)
        return True, arr.astype(np.int64).reshape(-1)
    return False, [[np.asarray(a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a,
                                dtype=np.int64) for a in row] for row in ids]


def _attend(store: KvStore, q: torch.Tensor, shared: bool, ids, with_static: bool):
    lay = store.layout
    b, h, g, d = lay.batch, lay.query_heads, lay.kv_heads, lay.head_dim
    dev = q.device
    if shared:
        lmax = int(ids.size)
        ids_d = to_device(ids.astype(np.int32)) if lmax else None
        len_d = to_device(np.array([lmax], dtype=np.int32))
    else:
        pad, lens, lmax = _pad_per_head(ids, b, g)
        ids_d, len_d = to_device(pad), to_device(lens)
    out = torch.empty((b, h, d), dtype=torch.float32, device=dev)
    mx = torch.empty((b, h), dtype=torch.float64, device=dev)
    den = torch.empty((b, h), dtype=torch.float64, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = N.lib()
    clay = store.ctkv_layout()
    ws = _ws(lib.ctkv_attend_workspace_bytes(clay, lmax, int(with_static)), dev)
    N.check(lib.ctkv_attend(clay, store.desc(), N.ptr(q), N.ptr(ids_d), N.ptr(len_d), lmax,
                            int(shared), int(with_static), N.ptr(out), N.ptr(mx), N.ptr(den),
                            N.ptr(flags), N.ptr(ws), ws.numel(), N.stream_ptr()), "attention")
    _flags_check(flags, "attention", recall_mixed_is_error=False)
    return out, mx, den


def sparse_attention(store: KvStore, query, ids) -> AttentionPartial:
    """ck/retrieval.py:249-264: attention restricted to `ids` with the
    online-softmax statistics; every head's set nonempty and duplicate-free."""
    lay = store.layout
    q = _as_query(query, lay.batch, lay.query_heads, lay.head_dim, store.dtype)
    shared, ids_n = _normalize_ids(store, ids)
    sets = [ids_n] if shared else [a for row in ids_n for a in row]
    for arr in sets:
        if arr.size == 0:
            raise ConfigError("sparse_attention: empty id set")
        if np.unique(arr).size != arr.size:
            raise ConfigError("sparse_attention: duplicate ids")
        if arr.min() < 0 or arr.max() >= store.total_tokens:
            raise IndexError(f"gather: token id out of range [0, {store.total_tokens})")
    out, mx, den = _attend(store, q, shared, ids_n, False)
    return AttentionPartial(like_input(out, query), like_input(mx, query), like_input(den, query))


def merge(a: AttentionPartial, b: AttentionPartial) -> AttentionPartial:
    """ck/retrieval.py:275-284 on the device."""
    host = is_host(a.out)
    oa, ma, la = to_device(a.out, torch.float32), to_device(a.row_max, torch.float64), to_device(a.denom, torch.float64)
    ob, mb, lb = to_device(b.out, torch.float32), to_device(b.row_max, torch.float64), to_device(b.denom, torch.float64)
    if oa.shape != ob.shape:
        raise ShapeError(f"merge: {tuple(oa.shape)} vs {tuple(ob.shape)}")
    d = oa.shape[-1]
    rows = oa.numel() // d
    out = torch.empty_like(oa)
    m = torch.empty_like(ma)
    den = torch.empty_like(la)
    N.check(N.lib().ctkv_merge(rows, d, N.ptr(oa), N.ptr(ma), N.ptr(la), N.ptr(ob), N.ptr(mb),
                               N.ptr(lb), N.ptr(out), N.ptr(m), N.ptr(den), N.stream_ptr()), "merge")
    if host:
        return AttentionPartial(out.cpu().numpy(), m.cpu().numpy(), den.cpu().numpy())
    return AttentionPartial(out, m, den)


def acceleration_factor(l_recall: int, l_rerank: int) -> float:
    """ck/retrieval.py:287-292."""
    if l_recall <= 0:
        raise ConfigError(f"acceleration_factor: L_recall must be positive, got {l_recall}")
    return (l_recall + 2.0 * l_rerank) / (2.0 * l_recall)


def digest(ids_bg) -> str:
    """ck/retrieval.py:295-301."""
    hsh = hashlib.sha256()
    for per_g in ids_bg:
        for arr in per_g:
            hsh.update(np.asarray(arr, dtype=np.int64).tobytes())
            hsh.update(b"|")
    return hsh.hexdigest()[:16]


def digest_padded(pad: np.ndarray, lens: np.ndarray) -> str:
    """digest() of the per-(b, g) prefixes pad[b, g, :lens[b, g]] without
    building the per-head lists: one int64 conversion and one sha256 call
    over the same byte stream (sha256 releases the GIL, so run_decode hashes
    its steps on a thread pool)."""
    p64 = pad.astype(np.int64, copy=False)
    b, g = lens.shape
    parts = []
    for bi in range(b):
        for gi in range(g):
            parts.append(p64[bi, gi, :lens[bi, gi]].tobytes())
            parts.append(b"|")
    return hashlib.sha256(b"".join(parts)).hexdigest()[:16]


# ---------------------------------------------------------------------------
# fused step
# ---------------------------------------------------------------------------

@dataclass
class StepBuffers:
    """Device outputs of one fused step (reusable across steps)."""
    out: torch.Tensor
    row_max: torch.Tensor
    denom: torch.Tensor
    selected: torch.Tensor
    recall_len: torch.Tensor
    sparse_ids: torch.Tensor
    sparse_len: torch.Tensor
    flags: torch.Tensor
    ws: torch.Tensor
    sparse_cap: int

    @classmethod
    def allocate(cls, store: KvStore, index: QueryCentroidIndex, cfg: DecodeConfig):
        lay = store.layout
        b, h, g, d = lay.batch, lay.query_heads, lay.kv_heads, lay.head_dim
        dev = store.keys.device
        cap = cfg.rho_prime if cfg.use_rerank else max(cfg.c_prime * index.rho, 1)
        ws_bytes = N.lib().ctkv_decode_workspace_bytes(store.ctkv_layout(), index.capacity,
                                                      index.rho, cfg.c_prime, cfg.rho_prime)
        return cls(torch.empty((b, h, d), dtype=torch.float32, device=dev),
                   torch.empty((b, h), dtype=torch.float64, device=dev),
                   torch.empty((b, h), dtype=torch.float64, device=dev),
                   torch.empty((b, g, cfg.c_prime), dtype=torch.int32, device=dev),
                   torch.empty((b, g), dtype=torch.int32, device=dev),
                   torch.empty((b, g, cap), dtype=torch.int32, device=dev),
                   torch.empty((b, g), dtype=torch.int32, device=dev),
                   torch.zeros(1, dtype=torch.int32, device=dev),
                   _ws(ws_bytes, dev), cap)


def launch_step(store: KvStore, index: QueryCentroidIndex, cfg: DecodeConfig, q: torch.Tensor,
                bufs: StepBuffers, k_new: torch.Tensor | None = None,
                v_new: torch.Tensor | None = None, stream=None, phase: int = 3) -> None:
    """Enqueue one fused decode step (append when k_new is given) -- no
    host synchronisation; safe to capture in a CUDA graph."""
    if cfg.c_prime > index.capacity:
        raise ConfigError(f"recall: c_prime {cfg.c_prime} outside [1, {index.capacity}]")
    args = N.StepArgs(q.data_ptr(), N.ptr(k_new), N.ptr(v_new), cfg.c_prime, cfg.rho_prime,
                      int(cfg.use_dcu), int(cfg.use_rerank), bufs.out.data_ptr(),
                      bufs.row_max.data_ptr(), bufs.denom.data_ptr(), bufs.selected.data_ptr(),
                      bufs.recall_len.data_ptr(), bufs.sparse_ids.data_ptr(),
                      bufs.sparse_len.data_ptr(), bufs.sparse_cap, bufs.flags.data_ptr())
    N.check(N.lib().ctkv_decode_step_phase(store.ctkv_layout(), store.desc(), index.desc(), args,
                                           phase, bufs.ws.data_ptr(), bufs.ws.numel(),
                                           N.stream_ptr(stream)), "decode_step")


def trace_row(step: int, cfg: DecodeConfig, store: KvStore, index: QueryCentroidIndex,
              recall_len: np.ndarray, sparse_ids: np.ndarray, sparse_len: np.ndarray) -> TraceRow:
    lay = store.layout
    total = int(recall_len.sum())
    denom = cfg.c_prime * index.rho
    alpha = float((recall_len / denom).mean()) if denom else 0.0
    row = TraceRow(step=step, recall_len=total, alpha=alpha, rerank_len=0, sparse_digest="")
    if total > 0:
        n_sparse = int(sparse_len.sum())
        row.rerank_len = n_sparse
        if cfg.use_rerank:
            row.macs_rerank_qk = lay.group_size * lay.head_dim * total
        row.macs_sparse_qk = lay.group_size * lay.head_dim * n_sparse
        row.macs_sparse_wv = lay.group_size * lay.head_dim * n_sparse
        row.sparse_digest = digest_padded(sparse_ids, sparse_len)
        if cfg.keep_sets:
            row.sparse = _split_per_head(sparse_ids, sparse_len)
    return row


def decode_step(state: DecodeState, query):
    """ck/retrieval.py:304-378: one fused device step; returns (out, TraceRow)."""
    store, index, cfg = state.store, state.index, state.config
    lay = store.layout
    q = _as_query(query, lay.batch, lay.query_heads, lay.head_dim, store.dtype)
    ws_bytes = N.lib().ctkv_decode_workspace_bytes(store.ctkv_layout(), index.capacity, index.rho,
                                                  cfg.c_prime, cfg.rho_prime)
    key = (ws_bytes, dataclasses.astuple(cfg), index.capacity, index.rho, store.keys.device)
    if state._cache is None or state._cache[0] != key:
        bufs = StepBuffers.allocate(store, index, cfg)
        host = tuple(torch.empty(t.shape, dtype=t.dtype).pin_memory()
                     for t in (bufs.flags, bufs.recall_len, bufs.sparse_ids, bufs.sparse_len))
        state._cache = (key, bufs, host)
    _, bufs, host = state._cache
    bufs.flags.zero_()
    launch_step(store, index, cfg, q, bufs)
    # one device->host round trip for everything the trace row needs
    for h_, d_ in zip(host, (bufs.flags, bufs.recall_len, bufs.sparse_ids, bufs.sparse_len)):
        h_.copy_(d_, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    N.raise_flags(int(host[0].item()), "decode_step")
    row = trace_row(state.step, cfg, store, index, host[1].numpy().astype(np.int64),
                    host[2].numpy().copy(), host[3].numpy().copy())
    if state.oracle is not None and row.recall_len > 0:
        row.recall_at_k = state.oracle.recall_at_k(q, bufs.sparse_ids, bufs.sparse_len,
                                                   min(cfg.rho_prime, store.offloaded_ids().size))
    state.trace.append(row)
    state.step += 1
    return like_input(bufs.out.clone(), query), row
