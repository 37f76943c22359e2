"""Exact flat-scan baseline on the device (ck/oracle.py:24-85 FlatOracle).

The paper's "Flat" baseline and the ground truth behind recall@k.  Scores
come from the build's exact scores kernel (f64 accumulate, f32 round, GQA
group max) and selection from the radix top-k kernel, so on identical
inputs this returns exactly the reference FlatOracle's ids.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError
from .store import KvStore
from .tensor_ops import like_input, to_device


class FlatOracle:
    def __init__(self, store: KvStore):
        self.store = store

    def _scope(self, scope: str) -> tuple[int, int]:
        if scope == "all":
            return 0, self.store.total_tokens
        if scope == "offloaded":
            off = self.store.offloaded_ids()
            return (int(off[0]), int(off[-1]) + 1) if off.size else (0, 0)
        raise ConfigError(f"unknown scope {scope!r}")

    def topk_device(self, q: torch.Tensor, k: int, scope: str = "all") -> torch.Tensor:
        """[b,g,k] int64 device ids, (score desc, id asc)."""
        st = self.store
        lay = st.layout
        lo, hi = self._scope(scope)
        n = hi - lo
        if n == 0:
            raise ConfigError(f"flat_topk: empty scope {scope!r}")
        if k > n:
            raise ConfigError(f"flat_topk: k={k} exceeds scope size {n}")
        b, h, g, d = lay.batch, lay.query_heads, lay.kv_heads, lay.head_dim
        if q.dim() == 4:
            q = q[:, :, 0, :]
        q4 = q.contiguous().view(b, h, 1, d)
        scores = torch.empty((b, g, 1, n), dtype=torch.float32, device=q.device)
        lib = N.lib()
        lay_c = st.ctkv_layout()
        keys = st.keys[:, :, lo:]
        N.check(lib.ctkv_scores(lay_c, N.ptr(q4), 1, keys.data_ptr(), n, st.capacity * d, 1,
                                N.ptr(scores), N.stream_ptr()), "flat scores")
        idx = torch.empty((b * g, k), dtype=torch.int32, device=q.device)
        N.check(lib.ctkv_topk_rows(N.ptr(scores), b * g, n, k, N.ptr(idx), None, 0,
                                   N.stream_ptr()), "flat topk")
        return (idx.long() + lo).view(b, g, k)

    def topk(self, query, k: int, scope: str = "all"):
        """ck/oracle.py:37-60: PerHead lists of int64 ids."""
        q = to_device(query, self.store.dtype)
        ids = self.topk_device(q, k, scope).cpu().numpy()
        return [[ids[bi, gi] for gi in range(ids.shape[1])] for bi in range(ids.shape[0])]

    def recall_at_k(self, q: torch.Tensor, sparse_ids: torch.Tensor, sparse_len: torch.Tensor,
                    k: int) -> float:
        """|sparse intersect flat top-k| / |flat top-k| summed over heads
        (ck/retrieval.py:360-370)."""
        truth = self.topk_device(q, k, "offloaded")
        b, g, _ = truth.shape
        sp = sparse_ids.long()
        valid = torch.arange(sp.shape[-1], device=sp.device)[None, None, :] < sparse_len[..., None]
        sp = torch.where(valid, sp, torch.full_like(sp, -1))
        hits = (truth[..., :, None] == sp[..., None, :]).any(-1).sum()
        return float(hits) / float(b * g * k)

    def full_attention(self, query, scope: str = "all"):
        """ck/oracle.py:62-85: exact attention over the scope."""
        from .retrieval import _as_query, _attend
        st = self.store
        lay = st.layout
        lo, hi = self._scope(scope)
        if hi <= lo:
            raise ConfigError(f"full_attention: empty scope {scope!r}")
        q = _as_query(query, lay.batch, lay.query_heads, lay.head_dim, st.dtype)
        out, _, _ = _attend(st, q, True, np.arange(lo, hi, dtype=np.int64), False)
        return like_input(out, query)
