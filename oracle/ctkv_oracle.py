"""CPU oracle for the CTkvr hot path -- TEST INFRASTRUCTURE ONLY.

This module is a from-scratch numpy restatement of the reference package
`centroidkv` 0.1.0 (/root/reference/pkg/src/centroidkv, abbreviated `ck/`)
for exactly the hot path BASELINE.json names: prefill index build, per-step
recall + rerank, partitioned sparse/static attention with the exact merge,
and the FIFO dynamic centroid update.  It is the CHECKER, never the product:
only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it.  The product package
(`paper_2512_15550_b200`) never imports anything from here and fails loudly
when its CUDA library is missing.

Pinning: `tests/test_oracle_golden.py` checks every function here against
golden vectors written by `tests/golden/make_golden.py`, which imports the
real reference from /root/reference (only possible in the build container).

Conventions kept from the reference (ck/tensor_ops.py:3-11): arithmetic in
float64, stored results float32, selection on logits, ties -> smaller index.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

EMPTY = -1  # ck/index.py:32


# ---------------------------------------------------------------------------
# L0 arithmetic (ck/tensor_ops.py)
# ---------------------------------------------------------------------------

def topk_desc(values: np.ndarray, k: int) -> np.ndarray:
    """Indices of the k largest entries of a 1-D row ordered (value desc,
    index asc); k clamps to [0, n].  Same contract as ck/tensor_ops.py:121-141
    (exact tie handling at the k-th value)."""
    v = np.asarray(values)
    n = v.shape[0]
    k = max(0, min(int(k), n))
    if k == 0:
        return np.zeros(0, dtype=np.int64)
    if k < n:
        kth = np.partition(v, n - k)[n - k]
        cand = np.flatnonzero(v >= kth)          # ascending index order
    else:
        cand = np.arange(n)
    order = np.argsort(-v[cand], kind="stable")   # stable => ties keep index order
    return cand[order[:k]].astype(np.int64)


def topk_rows_desc(values: np.ndarray, k: int) -> np.ndarray:
    """Row-wise `topk_desc` of a 2-D array -> int64 [rows, k]
    (ck/tensor_ops.py:144-169)."""
    rows, n = values.shape
    k = max(0, min(int(k), n))
    out = np.empty((rows, k), dtype=np.int64)
    if k == 0:
        return out
    if k < n:
        kth = np.partition(values, n - k, axis=1)[:, n - k:n - k + 1]
    for r in range(rows):
        row = values[r]
        cand = np.flatnonzero(row >= kth[r, 0]) if k < n else np.arange(n)
        order = np.argsort(-row[cand], kind="stable")
        out[r] = cand[order[:k]]
    return out


def scaled_logits(q: np.ndarray, k: np.ndarray) -> np.ndarray:
    """(q . k) / sqrt(d) accumulated in f64, returned f32 (ck/tensor_ops.py:72-92).
    q [b,h,m,d], k [b,g,n,d]; query head i reads kv head i // (h/g)."""
    b, h, m, d = q.shape
    g = k.shape[1]
    gs = h // g
    qq = q.astype(np.float64).reshape(b, g, gs * m, d)
    s = qq @ np.swapaxes(k.astype(np.float64), 2, 3)
    s *= 1.0 / math.sqrt(d)
    return s.reshape(b, h, m, -1).astype(np.float32)


def head_group_max(scores: np.ndarray, g: int) -> np.ndarray:
    """Max over each GQA group of query heads: [b,h,...] -> [b,g,...]
    (ck/tensor_ops.py:111-118)."""
    b, h = scores.shape[:2]
    return scores.reshape((b, g, h // g) + scores.shape[2:]).max(axis=2)


def cos_rows(q: np.ndarray, rows: np.ndarray) -> tuple[np.ndarray, bool]:
    """f64 cosine of q [...,d] against rows [...,C,d], clipped to [-1,1];
    zero norms give 0 and a degenerate flag (ck/tensor_ops.py:190-207)."""
    q64 = q.astype(np.float64)
    r64 = rows.astype(np.float64)
    dots = np.einsum("...d,...cd->...c", q64, r64)
    den = np.linalg.norm(q64, axis=-1)[..., None] * np.linalg.norm(r64, axis=-1)
    bad = den == 0.0
    degenerate = bool(bad.any())
    if degenerate:
        dots = np.where(bad, 0.0, dots)
        den = np.where(bad, 1.0, den)
    return np.clip(dots / den, -1.0, 1.0), degenerate


def softmax_rows(scores: np.ndarray) -> np.ndarray:
    """ck/tensor_ops.py:95-108."""
    s = scores.astype(np.float64)
    s = np.exp(s - s.max(axis=-1, keepdims=True))
    return (s / s.sum(axis=-1, keepdims=True)).astype(np.float32)


# ---------------------------------------------------------------------------
# L1 storage bookkeeping (ck/store.py)
# ---------------------------------------------------------------------------

@dataclass
class Store:
    """Token-major K/V [b,g,cap,d] f32 plus the partition counters
    (ck/store.py:23-44).  `keys`/`values` are grown on demand."""
    keys: np.ndarray
    values: np.ndarray
    init_len: int
    local_len: int
    total: int
    query_heads: int

    @property
    def ring_start(self) -> int:            # ck/store.py:78-81
        return max(self.init_len, self.total - self.local_len)

    def offloaded(self) -> np.ndarray:      # ck/store.py:91-92
        return np.arange(min(self.init_len, self.total), self.ring_start, dtype=np.int64)

    def static(self) -> np.ndarray:         # ck/store.py:83-96
        first = np.arange(min(self.init_len, self.total), dtype=np.int64)
        ring = np.arange(self.ring_start, self.total, dtype=np.int64)
        return np.concatenate([first, ring])

    def append(self, k_new: np.ndarray, v_new: np.ndarray) -> int:   # ck/store.py:114-138
        cap = self.keys.shape[2]
        if self.total == cap:
            grow = cap + max(1024, cap // 2)
            for name in ("keys", "values"):
                old = getattr(self, name)
                new = np.zeros(old.shape[:2] + (grow, old.shape[3]), dtype=np.float32)
                new[:, :, :cap] = old
                setattr(self, name, new)
        t = self.total
        self.keys[:, :, t] = k_new
        self.values[:, :, t] = v_new
        self.total += 1
        return t


def partition(keys: np.ndarray, values: np.ndarray, init_len: int, local_len: int,
              query_heads: int | None = None) -> Store:
    """ck/store.py:48-70: copy into [b,g,max(1024,s),d] storage."""
    b, g, s, d = keys.shape
    if init_len + local_len > s:
        raise ValueError("init_len + local_len exceeds seq_len")
    cap = max(1024, s)
    kk = np.zeros((b, g, cap, d), dtype=np.float32)
    vv = np.zeros((b, g, cap, d), dtype=np.float32)
    kk[:, :, :s] = keys
    vv[:, :, :s] = values
    return Store(kk, vv, init_len, local_len, s, g if query_heads is None else query_heads)


# ---------------------------------------------------------------------------
# L2 index (ck/index.py)
# ---------------------------------------------------------------------------

@dataclass
class Index:
    centroids: np.ndarray          # [b,h,C,d] f32
    lists: np.ndarray              # [b,g,C,rho] int32, -1 = empty
    fifo_head: np.ndarray          # [b] int64

    @property
    def capacity(self) -> int:
        return self.centroids.shape[2]

    @property
    def rho(self) -> int:
        return self.lists.shape[3]


def build_index(queries: np.ndarray, store: Store, capacity: int, rho: int,
                block_rows: int | None = None) -> Index:
    """Alg. 1 (ck/index.py:59-99): centroids are the last `capacity` queries;
    each centroid's list is the top-rho offloaded tokens by GQA group-max
    scaled logit (f64 accumulate, f32 rounding, ties -> smaller token id)."""
    b, h, s, d = queries.shape
    g = store.keys.shape[1]
    off = store.offloaded()
    if capacity < 1 or capacity > s:
        raise ValueError("capacity out of range")
    if rho < 0 or rho > off.size:
        raise ValueError("rho exceeds offloaded count")
    cent = np.ascontiguousarray(queries[:, :, s - capacity:, :])
    lists = np.full((b, g, capacity, rho), EMPTY, dtype=np.int32)
    if rho > 0:
        k_off = store.keys[:, :, off[0]:off[-1] + 1]
        n = off.size
        step = block_rows or max(1, min(capacity, (256 << 20) // max(1, 8 * h * n)))
        for c0 in range(0, capacity, step):
            c1 = min(capacity, c0 + step)
            grouped = head_group_max(scaled_logits(cent[:, :, c0:c1], k_off), g)
            for bi in range(b):
                for gi in range(g):
                    pos = topk_rows_desc(grouped[bi, gi], rho)
                    lists[bi, gi, c0:c1] = (off[pos]).astype(np.int32)
    return Index(cent, lists, np.zeros(b, dtype=np.int64))


def fifo_update(index: Index, q: np.ndarray, grouped: list, recalled: list) -> None:
    """DCU (ck/index.py:103-133): overwrite slot fifo_head[b] % C with the
    query and, per kv head, the top-min(rho, L) recalled ids by rerank score."""
    b, h, d = q.shape
    g = index.lists.shape[1]
    for bi in range(b):
        slot = int(index.fifo_head[bi] % index.capacity)
        index.centroids[bi, :, slot, :] = q[bi]
        for gi in range(g):
            ids = np.asarray(recalled[bi][gi], dtype=np.int64)
            keep = topk_desc(np.asarray(grouped[bi][gi]), min(index.rho, ids.size))
            row = np.full(index.rho, EMPTY, dtype=np.int32)
            row[:keep.size] = ids[keep]
            index.lists[bi, gi, slot] = row
        index.fifo_head[bi] = slot + 1


# ---------------------------------------------------------------------------
# L3 retrieval (ck/retrieval.py)
# ---------------------------------------------------------------------------

@dataclass
class Recall:
    selected: np.ndarray           # [b,g,C'] int64
    recalled: list                 # [b][g] int64 ids, first-occurrence order
    recall_len: np.ndarray         # [b,g]
    alpha: np.ndarray              # [b,g]
    degenerate: bool = False
    cosines: np.ndarray | None = None   # [b,g,C] f64 group-max cosines


def recall(index: Index, q: np.ndarray, c_prime: int, force_selected=None) -> Recall:
    """Alg. 2 lines 1-4 (ck/retrieval.py:132-168).  `force_selected[b, g]`
    (parity checkers only) replaces the top-C' slots of a unit whose
    selection differs from the device's inside the tie window, so the rest
    of the step is compared from equal state."""
    C = index.capacity
    if C == 0:
        raise ValueError("empty index")
    if c_prime < 1 or c_prime > C:
        raise ValueError("c_prime out of range")
    b, h, d = q.shape
    g = index.lists.shape[1]
    cosv, degenerate = cos_rows(q, index.centroids)               # [b,h,C]
    grouped = head_group_max(cosv, g)                              # [b,g,C]
    selected = np.zeros((b, g, c_prime), dtype=np.int64)
    recalled, rlen = [], np.zeros((b, g), dtype=np.int64)
    alpha = np.zeros((b, g), dtype=np.float64)
    for bi in range(b):
        row = []
        for gi in range(g):
            slots = topk_desc(grouped[bi, gi], c_prime)
            if force_selected is not None and force_selected[bi][gi] is not None:
                slots = np.asarray(force_selected[bi][gi], dtype=np.int64)
            selected[bi, gi] = slots
            flat = index.lists[bi, gi, slots].reshape(-1)
            flat = flat[flat != EMPTY].astype(np.int64)
            if flat.size:
                _, first = np.unique(flat, return_index=True)
                ids = flat[np.sort(first)]
            else:
                ids = flat
            row.append(ids)
            rlen[bi, gi] = ids.size
            denom = c_prime * index.rho
            alpha[bi, gi] = ids.size / denom if denom else 0.0
        recalled.append(row)
    return Recall(selected, recalled, rlen, alpha, degenerate, grouped)


def head_logits(store: Store, q: np.ndarray, ids_bg: list):
    """Per-(b,g) f64 logits [gs, L] of the current query against `ids`,
    plus the group-max row [L] (ck/retrieval.py:171-193)."""
    b, h, d = q.shape
    g = store.keys.shape[1]
    gs = h // g
    scale = 1.0 / math.sqrt(d)
    logits, grouped = [], []
    for bi in range(b):
        lrow, grow = [], []
        for gi in range(g):
            ids = np.asarray(ids_bg[bi][gi], dtype=np.int64)
            if ids.size and (ids.min() < 0 or ids.max() >= store.total):
                raise IndexError("token id out of range")
            kk = store.keys[bi, gi, ids].astype(np.float64)
            sc = (q[bi, gi * gs:(gi + 1) * gs].astype(np.float64) @ kk.T) * scale
            lrow.append(sc)
            grow.append(sc.max(axis=0) if ids.size else sc.reshape(0))
        logits.append(lrow)
        grouped.append(grow)
    return logits, grouped


def rerank(store: Store, q: np.ndarray, rec: Recall, rho_prime: int):
    """Alg. 2 lines 5-6 (ck/retrieval.py:196-218): returns (sparse ids per
    head, rerank_len, grouped f64 scores over the recalled ids)."""
    if int(rec.recall_len.sum()) == 0:
        raise ValueError("rerank: empty recall set")
    _, grouped = head_logits(store, q, rec.recalled)
    b, g = rec.recall_len.shape
    sparse, rlen = [], np.zeros((b, g), dtype=np.int64)
    for bi in range(b):
        row = []
        for gi in range(g):
            ids = rec.recalled[bi][gi]
            keep = topk_desc(grouped[bi][gi], min(rho_prime, ids.size))
            row.append(ids[keep])
            rlen[bi, gi] = keep.size
        sparse.append(row)
    return sparse, rlen, grouped


@dataclass
class Partial:
    out: np.ndarray       # [b,h,d] f32
    row_max: np.ndarray   # [b,h] f64
    denom: np.ndarray     # [b,h] f64


def attend(store: Store, q: np.ndarray, ids_bg: list):
    """Softmax partial over per-(b,g) id sets (ck/retrieval.py:221-246).
    Returns (Partial, grouped logits)."""
    b, h, d = q.shape
    g = store.keys.shape[1]
    gs = h // g
    out = np.zeros((b, h, d), dtype=np.float32)
    m_all = np.full((b, h), -np.inf)
    l_all = np.zeros((b, h))
    logits, grouped = head_logits(store, q, ids_bg)
    for bi in range(b):
        for gi in range(g):
            ids = np.asarray(ids_bg[bi][gi], dtype=np.int64)
            if ids.size == 0:
                raise ValueError("attention over an empty id set")
            vv = store.values[bi, gi, ids].astype(np.float64)
            sc = logits[bi][gi]
            m = sc.max(axis=1)
            e = np.exp(sc - m[:, None])
            l = e.sum(axis=1)
            hs = slice(gi * gs, (gi + 1) * gs)
            out[bi, hs] = ((e @ vv) / l[:, None]).astype(np.float32)
            m_all[bi, hs] = m
            l_all[bi, hs] = l
    return Partial(out, m_all, l_all), grouped


def merge(a: Partial, c: Partial) -> Partial:
    """Exact two-partial combination (ck/retrieval.py:275-284)."""
    m = np.maximum(a.row_max, c.row_max)
    wa = np.exp(a.row_max - m) * a.denom
    wc = np.exp(c.row_max - m) * c.denom
    den = wa + wc
    o = (a.out.astype(np.float64) * wa[..., None] + c.out.astype(np.float64) * wc[..., None])
    return Partial((o / den[..., None]).astype(np.float32), m, den)


def digest(ids_bg: list) -> str:
    """16-hex sha256 of per-head int64 ids in order (ck/retrieval.py:295-301)."""
    hsh = hashlib.sha256()
    for row in ids_bg:
        for ids in row:
            hsh.update(np.asarray(ids, dtype=np.int64).tobytes())
            hsh.update(b"|")
    return hsh.hexdigest()[:16]


@dataclass
class StepRecord:
    """What one decode step exposes for parity checks (subset of
    ck/retrieval.py:76-108 TraceRow plus the intermediate sets)."""
    out: np.ndarray
    selected: np.ndarray | None
    recalled: list | None
    sparse: list | None
    grouped: list | None
    recall_len: int
    alpha: float
    rerank_len: int
    digest: str
    merged: Partial | None = None
    cosines: np.ndarray | None = None


def decode_step(store: Store, index: Index, q: np.ndarray, c_prime: int, rho_prime: int,
                use_dcu: bool = True, use_rerank: bool = True,
                force_selected=None) -> StepRecord:
    """One decode step (ck/retrieval.py:304-378) without the flat oracle."""
    q = np.asarray(q, dtype=np.float32)
    if q.ndim == 4:
        q = q[:, :, 0, :]
    rec = recall(index, q, c_prime, force_selected)
    total = int(rec.recall_len.sum())
    sparse_p, grouped, sparse, rr_len, dig = None, None, None, 0, ""
    if total > 0:
        if rec.recall_len.min() == 0:
            raise ValueError("decode_step: mixed empty/nonempty recall sets")
        if use_rerank:
            sparse, rl, grouped = rerank(store, q, rec, rho_prime)
            rr_len = int(rl.sum())
            sparse_p, _ = attend(store, q, sparse)
        else:
            sparse = [[ids for ids in row] for row in rec.recalled]
            rr_len = total
            sparse_p, grouped = attend(store, q, sparse)
        dig = digest(sparse)
    st = store.static()
    b, g = store.keys.shape[:2]
    static_p = attend(store, q, [[st] * g for _ in range(b)])[0] if st.size else None
    if sparse_p is not None and static_p is not None:
        merged = merge(sparse_p, static_p)
    elif static_p is not None:
        merged = static_p
    elif sparse_p is not None:
        merged = sparse_p
    else:
        raise ValueError("decode_step: no attendable tokens")
    if use_dcu and total > 0:
        fifo_update(index, q, grouped, rec.recalled)
    return StepRecord(merged.out, rec.selected, rec.recalled, sparse, grouped, total,
                      float(rec.alpha.mean()), rr_len, dig, merged, rec.cosines)


# ---------------------------------------------------------------------------
# L4 session (ck/session.py)
# ---------------------------------------------------------------------------

def prefill(queries, keys, values, init_len, local_len, capacity, rho):
    """ck/session.py:32-39: partition, clamp rho to the offloaded count, build."""
    store = partition(keys, values, init_len, local_len, query_heads=queries.shape[1])
    rho = min(rho, store.offloaded().size)
    return store, build_index(queries, store, capacity, rho)


def run_decode(store, index, dec_q, dec_k, dec_v, c_prime, rho_prime,
               use_dcu=True, use_rerank=True):
    """ck/session.py:42-64: per step append THEN decode."""
    T = dec_q.shape[2]
    outs = np.empty(dec_q.shape, dtype=np.float32)
    recs = []
    for t in range(T):
        store.append(dec_k[:, :, t], dec_v[:, :, t])
        r = decode_step(store, index, dec_q[:, :, t], c_prime, rho_prime, use_dcu, use_rerank)
        outs[:, :, t] = r.out
        recs.append(r)
    return outs, recs


def acceleration_factor(l_recall: int, l_rerank: int) -> float:
    """ck/retrieval.py:287-292."""
    return (l_recall + 2.0 * l_rerank) / (2.0 * l_recall)


# ---------------------------------------------------------------------------
# Synthetic drift workload (ck/workload.py:95-242), needed to reproduce the
# reference's inputs bit-for-bit on hosts without /root/reference.
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Drift:
    seed: int = 42
    s: int = 32768
    decode_steps: int = 256
    drift_rate: float = 1e-4
    noise_sigma: float = 0.05
    turns: int = 1

    @property
    def total(self) -> int:
        return self.s + self.decode_steps


def _rope(x: np.ndarray, pos: np.ndarray) -> np.ndarray:
    """Rotate coordinate pairs (ck/workload.py:89-110); f64 out."""
    dim = x.shape[-1]
    inv = 10000.0 ** (-np.arange(0, dim, 2, dtype=np.float64) / dim)
    ang = np.asarray(pos, dtype=np.float64)[..., None] * inv
    c, s = np.cos(ang), np.sin(ang)
    a, bb = x[..., 0::2], x[..., 1::2]
    y = np.empty_like(x, dtype=np.float64)
    y[..., 0::2] = a * c - bb * s
    y[..., 1::2] = a * s + bb * c
    return y


def _spectral(d: int) -> np.ndarray:
    """ck/workload.py:113-123 (decay 0.8 toward the fast rotary pairs)."""
    w = np.repeat(0.8 ** np.arange(d // 2 - 1, -1, -1, dtype=np.float64), 2)
    return w / np.linalg.norm(w) * math.sqrt(d)


def _normalize(v):
    return v / np.linalg.norm(v)


def _segments(cfg: Drift):
    """ck/workload.py:134-146."""
    if cfg.decode_steps == 0 or cfg.turns == 1:
        return [(0, cfg.total, 0)]
    edges = np.linspace(cfg.s, cfg.total, cfg.turns + 1).astype(int)
    return [(0, int(edges[1]), 0)] + [(int(edges[r]), int(edges[r + 1]), r)
                                      for r in range(1, cfg.turns)]


def generate(cfg: Drift, b: int, h: int, g: int, d: int):
    """Drift-regime Q/K/V (ck/workload.py:156-242), bit-identical RNG stream.
    Returns (q [b,h,T,d], k [b,g,T,d], v [b,g,T,d]) float32, T = s+steps."""
    T = cfg.total
    rng = np.random.default_rng(cfg.seed)
    segs = _segments(cfg)
    w = _spectral(d)
    pos = np.arange(T, dtype=np.float64)
    q = np.empty((b, h, T, d), dtype=np.float32)
    for bi in range(b):
        for hi in range(h):
            raw = np.empty((T, d), dtype=np.float64)
            base = None
            for start, end, _ in segs:
                a = _normalize(w * rng.standard_normal(d))
                o = w * rng.standard_normal(d)
                o = _normalize(o - (o @ a) * a)
                if base is None:
                    base = a
                else:
                    a = _normalize(a - (a @ base) * base)
                    base = 0.75 * base + math.sqrt(1.0 - 0.75 ** 2) * a
                    o = _normalize(o - (o @ base) * base)
                phi = cfg.drift_rate * np.arange(end - start, dtype=np.float64)
                raw[start:end] = np.cos(phi)[:, None] * base + np.sin(phi)[:, None] * o
            if cfg.noise_sigma > 0:
                raw += cfg.noise_sigma * (w * rng.standard_normal((T, d))) / math.sqrt(d)
            q[bi, hi] = _rope(raw, pos).astype(np.float32)
    keys = _rope(w * rng.standard_normal((b, g, T, d)) / math.sqrt(d), pos).astype(np.float32)
    vals = rng.standard_normal((b, g, T, d)).astype(np.float32)
    lo, hi_pos = int(0.1 * cfg.s), int(0.75 * cfg.s)
    if hi_pos > lo:
        want = len(segs) * 2 * b * g
        spots = iter(rng.choice(np.arange(lo, hi_pos), size=min(want, hi_pos - lo),
                                replace=False).tolist())
        gs = h // g
        plan = []
        exhausted = False
        for start, end, turn in segs:
            if turn == 0:
                first = cfg.s if cfg.decode_steps > 0 else cfg.s - 1
            else:
                first = start
            for bi in range(b):
                for gi in range(g):
                    for j in range(2):
                        p = next(spots, None)
                        if p is None:
                            break
                        plan.append((bi, gi, p, turn, min(first + 3 * j, end - 1, T - 1)))
        best = {}
        for bi, gi, p, turn, des in plan:
            sc = (q[bi, gi * gs:(gi + 1) * gs, des].astype(np.float64)
                  @ keys[bi, gi].astype(np.float64).T).max(axis=0)
            val = float(sc.max() + 3.0 * sc.std())
            best[(bi, gi, turn)] = max(best.get((bi, gi, turn), 0.0), val)
        for bi, gi, p, turn, des in plan:
            dq = q[bi, gi * gs, des].astype(np.float64)
            keys[bi, gi, p] = (best[(bi, gi, turn)] * _normalize(dq)).astype(np.float32)
        del exhausted
    return q, keys, vals


def default_capacity(s: int) -> int:
    """ck/cli.py:83-86."""
    return max(1, min(2048, s // 16))


def default_rho(rho_prime: int) -> int:
    """ck/cli.py:88-91."""
    return int(round(2.5 * rho_prime))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round f32 to the nearest bf16 (ties to even) and widen back to f32 --
    how the bf16 parity configs feed the f32-only reference
    ('bf16 configs')."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)
