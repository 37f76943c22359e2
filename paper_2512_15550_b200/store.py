"""Device KvStore (ck/store.py:23-171).

K/V live in HBM as [b, g, capacity, d] (float32 or bfloat16), token-major
per (b, kv_head) exactly like the reference, so a token's key is one
contiguous d-element row (256 B at d=128 bf16) -- the unit every gather
kernel moves.  The token counter exists twice: a host mirror (partition
bookkeeping, ids) and a device scalar that the fused decode kernels read
and advance, so a captured CUDA graph can replay steps without host sync.

Capacity is planned up front (`reserve=`): the reference grows by
max(1024, cap/2) with a full copy (ck/store.py:131-138); on a 180 GB part
we preallocate s+T and only fall back to the same growth rule when an
append would overflow.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, ShapeError
from .tensor_ops import HeadLayout, is_host, like_input, to_device, validate_tensor4


class KvStore:
    GROW = 1024

    def __init__(self, layout: HeadLayout, init_len: int, local_len: int, *,
                 dtype: torch.dtype = torch.float32, capacity: int | None = None,
                 host_api: bool = True):
        if init_len < 0 or local_len < 0:
            raise ConfigError(f"init_len/local_len must be non-negative: {init_len}, {local_len}")
        self.layout = layout
        self.init_len = init_len
        self.local_len = local_len
        self.dtype = dtype
        self.host_api = host_api
        cap = max(self.GROW, layout.seq_len) if capacity is None else max(capacity, layout.seq_len)
        dev = torch.device("cuda", torch.cuda.current_device())
        N.lib()
        shape = (layout.batch, layout.kv_heads, cap, layout.head_dim)
        self.keys = torch.zeros(shape, dtype=dtype, device=dev)
        self.values = torch.zeros(shape, dtype=dtype, device=dev)
        self.total_dev = torch.zeros(1, dtype=torch.int64, device=dev)
        self._total = 0

    # -- construction ------------------------------------------------------

    @classmethod
    def partition(cls, keys, values, init_len: int, local_len: int,
                  query_heads: int | None = None, *, dtype: torch.dtype | None = None,
                  reserve: int = 0) -> "KvStore":
        """ck/store.py:48-70.  `reserve` extra token rows are preallocated
        for the decode appends; `dtype` overrides the storage type (bf16)."""
        validate_tensor4(keys, "keys")
        validate_tensor4(values, "values")
        if tuple(keys.shape) != tuple(values.shape):
            raise ShapeError(f"keys {tuple(keys.shape)} vs values {tuple(values.shape)}")
        b, g, s, d = keys.shape
        if init_len + local_len > s:
            raise ConfigError(f"init_len + local_len = {init_len + local_len} exceeds seq_len {s}")
        h = g if query_heads is None else query_heads
        layout = HeadLayout(batch=b, query_heads=h, kv_heads=g, seq_len=s, head_dim=d)
        if dtype is None:
            dtype = keys.dtype if isinstance(keys, torch.Tensor) else torch.float32
        cap = max(cls.GROW, s + int(reserve))
        store = cls(layout, init_len, local_len, dtype=dtype, capacity=cap,
                    host_api=is_host(keys))
        store.keys[:, :, :s].copy_(to_device(keys, dtype))
        store.values[:, :, :s].copy_(to_device(values, dtype))
        store._set_total(s)
        return store

    def batch_view(self, b0: int, b1: int) -> "KvStore":
        """Sequences [b0, b1) as a store sharing this one's K/V memory, with
        its own token counter (a decode lane of DecodeEngine).  Every lane
        appends once per step, so the counters stay equal; `adopt_total`
        copies one back."""
        lay = self.layout
        if not 0 <= b0 < b1 <= lay.batch:
            raise ConfigError(f"batch_view: [{b0}, {b1}) outside [0, {lay.batch})")
        v = KvStore.__new__(KvStore)
        v.layout = HeadLayout(b1 - b0, lay.query_heads, lay.kv_heads, lay.seq_len, lay.head_dim)
        v.init_len, v.local_len, v.dtype, v.host_api = (self.init_len, self.local_len, self.dtype,
                                                        self.host_api)
        v.keys = self.keys[b0:b1]
        v.values = self.values[b0:b1]
        v.total_dev = self.total_dev.clone()
        v._total = self._total
        return v

    def adopt_total(self, other: "KvStore") -> None:
        """Take over the token counter of a batch view (device and host)."""
        self._total = other._total
        self.total_dev.copy_(other.total_dev)

    def _set_total(self, t: int) -> None:
        self._total = int(t)
        self.total_dev.fill_(int(t))

    # -- partition views (ck/store.py:74-110) -------------------------------

    @property
    def capacity(self) -> int:
        return self.keys.shape[2]

    @property
    def total_tokens(self) -> int:
        return self._total

    @property
    def ring_start(self) -> int:
        return max(self.init_len, self._total - self.local_len)

    def initial_ids(self) -> np.ndarray:
        return np.arange(min(self.init_len, self._total), dtype=np.int64)

    def local_ids(self) -> np.ndarray:
        return np.arange(self.ring_start, self._total, dtype=np.int64)

    def offloaded_ids(self) -> np.ndarray:
        return np.arange(min(self.init_len, self._total), self.ring_start, dtype=np.int64)

    def static_ids(self) -> np.ndarray:
        return np.concatenate([self.initial_ids(), self.local_ids()])

    def is_offloaded(self, ids) -> np.ndarray:
        ids = np.asarray(ids)
        return (ids >= self.init_len) & (ids < self.ring_start)

    def check_partition(self) -> None:
        parts = [self.initial_ids(), self.offloaded_ids(), self.local_ids()]
        merged = np.concatenate(parts)
        if merged.size != self._total or not np.array_equal(np.sort(merged), np.arange(self._total)):
            raise AssertionError(f"partition broken: sizes {[p.size for p in parts]} vs total {self._total}")
        ring = self.local_ids()
        if ring.size != min(self.local_len, max(self._total - self.init_len, 0)):
            raise AssertionError(f"ring size {ring.size} off for total={self._total}")
        dev_total = int(self.total_dev.item())
        if dev_total != self._total:
            raise AssertionError(f"device token counter {dev_total} != host {self._total}")

    @property
    def static_fraction(self) -> float:
        if self._total == 0:
            return 0.0
        return self.static_ids().size / self._total

    # -- mutation ------------------------------------------------------------

    def ctkv_layout(self) -> N.Layout:
        lay = self.layout
        return N.Layout(lay.batch, lay.query_heads, lay.kv_heads, lay.head_dim, self.capacity,
                        N.dtype_code(self.dtype), self.init_len, self.local_len, 0)

    def desc(self) -> N.StoreDesc:
        return N.StoreDesc(self.keys.data_ptr(), self.values.data_ptr(), self.total_dev.data_ptr())

    def ensure_room(self, extra: int = 1) -> None:
        """Grow like ck/store.py:131-138 when an append would overflow."""
        cap = self.capacity
        if self._total + extra <= cap:
            return
        new_cap = cap
        while self._total + extra > new_cap:
            new_cap = new_cap + max(self.GROW, new_cap // 2)
        for name in ("keys", "values"):
            old = getattr(self, name)
            grown = torch.zeros(old.shape[:2] + (new_cap, old.shape[3]), dtype=old.dtype,
                                device=old.device)
            grown[:, :, :cap].copy_(old)
            setattr(self, name, grown)

    def append(self, new_keys, new_values) -> int:
        """ck/store.py:114-129 (device append kernel)."""
        b, g, d = self.layout.batch, self.layout.kv_heads, self.layout.head_dim
        kn = to_device(new_keys, self.dtype)
        vn = to_device(new_values, self.dtype)
        if tuple(kn.shape) != (b, g, d) or tuple(vn.shape) != (b, g, d):
            raise ShapeError(f"append: expected [b, g, d] = {(b, g, d)}, got {tuple(kn.shape)}")
        self.ensure_room(1)
        N.check(N.lib().ctkv_append(self.ctkv_layout(), self.desc(), N.ptr(kn), N.ptr(vn),
                                    N.stream_ptr()), "append")
        tid = self._total
        self._total += 1
        return tid

    def note_device_append(self) -> int:
        """Host mirror of an append done inside a fused decode kernel."""
        tid = self._total
        self._total += 1
        return tid

    # -- access (ck/store.py:142-164) -----------------------------------------

    def _ids(self, ids) -> torch.Tensor:
        t = to_device(ids if not isinstance(ids, list) else np.asarray(ids, dtype=np.int64),
                      torch.int64)
        if t.numel() and (int(t.min()) < 0 or int(t.max()) >= self._total):
            raise IndexError(f"gather: token id out of range [0, {self._total})")
        return t

    def _out(self, t):
        return like_input(t, np.empty(0)) if self.host_api else t

    def gather(self, batch: int, kv_head: int, ids, which: str = "keys"):
        if which not in ("keys", "values"):
            raise ConfigError(f"gather: which must be 'keys' or 'values', got {which!r}")
        src = self.keys if which == "keys" else self.values
        return self._out(src[batch, kv_head, self._ids(ids)])

    def keys_view(self, ids):
        return self._out(self.keys[:, :, self._ids(ids)])

    def values_view(self, ids):
        return self._out(self.values[:, :, self._ids(ids)])
