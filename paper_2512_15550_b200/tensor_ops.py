"""L0 primitives of the reference API (ck/tensor_ops.py), on the device.

`HeadLayout` and the validators are host bookkeeping.  `dot_scores` and
`top_k`/`top_k_rows` run the package's own CUDA kernels (the same ones the
index build uses); `group_max`, `softmax_rows` and `cosine` are thin
device-side conveniences kept for API completeness (they are not on the
decode or build hot path, whose kernels fuse them).

Type rule for every public function in this package: numpy in -> numpy
out; torch in -> torch (CUDA) out.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import DegenerateQueryWarning, ShapeError


@dataclass(frozen=True)
class HeadLayout:
    """ck/tensor_ops.py:25-55."""

    batch: int
    query_heads: int
    kv_heads: int
    seq_len: int
    head_dim: int

    def __post_init__(self):
        if self.batch < 1 or self.query_heads < 1 or self.kv_heads < 1 or self.head_dim < 1:
            raise ShapeError(f"layout dimensions must be positive: {self}")
        if self.seq_len < 0:
            raise ShapeError(f"seq_len must be non-negative: {self}")
        if self.query_heads % self.kv_heads != 0:
            raise ShapeError(
                f"query_heads={self.query_heads} not divisible by kv_heads={self.kv_heads}")

    @property
    def group_size(self) -> int:
        return self.query_heads // self.kv_heads

    def q_shape(self, rows=None):
        return (self.batch, self.query_heads, self.seq_len if rows is None else rows, self.head_dim)

    def kv_shape(self, rows=None):
        return (self.batch, self.kv_heads, self.seq_len if rows is None else rows, self.head_dim)


def device() -> torch.device:
    N.lib()
    return torch.device("cuda", torch.cuda.current_device())


def is_host(x) -> bool:
    return isinstance(x, np.ndarray)


def to_device(x, dtype=None) -> torch.Tensor:
    """numpy/torch -> contiguous CUDA tensor (optionally cast)."""
    if isinstance(x, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(x))
    elif isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.as_tensor(np.asarray(x))
    t = t.to(device=device(), non_blocking=False)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def like_input(t: torch.Tensor, ref):
    """Return `t` as numpy when the caller passed numpy."""
    if is_host(ref):
        if t.dtype == torch.bfloat16:
            t = t.float()
        return t.cpu().numpy()
    return t


def validate_tensor4(arr, name: str = "tensor"):
    """ck/tensor_ops.py:58-69: rank 4, float (f32; bf16 also accepted for
    torch tensors), contiguous, finite."""
    if isinstance(arr, np.ndarray):
        if arr.ndim != 4:
            raise ShapeError(f"{name}: expected a 4-D ndarray, got {arr.shape}")
        if arr.dtype != np.float32:
            raise ShapeError(f"{name}: expected float32 data, got {arr.dtype}")
        if not arr.flags.c_contiguous:
            raise ShapeError(f"{name}: expected C-contiguous (row-major) data")
        if arr.size and not np.isfinite(arr).all():
            raise ShapeError(f"{name}: contains NaN or Inf")
        return arr
    if isinstance(arr, torch.Tensor):
        if arr.dim() != 4:
            raise ShapeError(f"{name}: expected a 4-D tensor, got {tuple(arr.shape)}")
        if arr.dtype not in (torch.float32, torch.bfloat16):
            raise ShapeError(f"{name}: expected float32/bfloat16 data, got {arr.dtype}")
        if not arr.is_contiguous():
            raise ShapeError(f"{name}: expected contiguous data")
        if arr.numel() and not bool(torch.isfinite(arr).all()):
            raise ShapeError(f"{name}: contains NaN or Inf")
        return arr
    raise ShapeError(f"{name}: expected a 4-D array, got {type(arr)}")


def _layout_struct(b, h, g, d, cap, dtype_code, init_len=0, local_len=0) -> N.Layout:
    return N.Layout(b, h, g, d, cap, dtype_code, init_len, local_len, 0)


def dot_scores(q, k):
    """(q . k^T)/sqrt(d) accumulated in f64, returned f32 [b,h,m,n]
    (ck/tensor_ops.py:72-92) -- the build kernel's exact scores path."""
    if q.ndim != 4 or k.ndim != 4:
        raise ShapeError(f"dot_scores: expected 4-D tensors, got {q.shape} and {k.shape}")
    b, h, m, d = q.shape
    b2, g, n, d2 = k.shape
    if b2 != b or d2 != d:
        raise ShapeError(f"dot_scores: incompatible shapes {tuple(q.shape)} vs {tuple(k.shape)}")
    if g < 1 or h % g != 0:
        raise ShapeError(f"dot_scores: {h} query heads not divisible by {g} kv heads")
    qt = to_device(q)
    kt = to_device(k, qt.dtype)
    out = torch.empty((b, h, m, n), dtype=torch.float32, device=qt.device)
    lay = _layout_struct(b, h, g, d, n, N.dtype_code(qt.dtype))
    N.check(N.lib().ctkv_scores(lay, N.ptr(qt), m, N.ptr(kt), n, n * d, 0, N.ptr(out),
                                N.stream_ptr()), "dot_scores")
    return like_input(out, q)


def softmax_rows(scores):
    """ck/tensor_ops.py:95-108."""
    s = to_device(scores)
    if s.shape[-1] == 0:
        raise ShapeError("softmax_rows: empty rows")
    if not bool(torch.isfinite(s).all()):
        raise ShapeError("softmax_rows: input contains NaN or Inf")
    return like_input(torch.softmax(s.double(), dim=-1).float(), scores)


def group_max(scores, layout: HeadLayout):
    """ck/tensor_ops.py:111-118."""
    s = to_device(scores)
    b, h, m, n = s.shape
    if b != layout.batch or h != layout.query_heads:
        raise ShapeError(f"group_max: scores {tuple(s.shape)} do not match layout {layout}")
    g = layout.kv_heads
    return like_input(s.view(b, g, layout.group_size, m, n).amax(dim=2), scores)


def top_k_rows(values, k: int):
    """Row-wise exact top-k (value desc, index asc) -> int64 [rows, k]
    (ck/tensor_ops.py:144-169) via the device radix-select kernel."""
    v = to_device(values)
    if v.dim() != 2:
        raise ShapeError(f"top_k_rows: expected 2-D, got {tuple(v.shape)}")
    rows, n = v.shape
    k = min(int(k), n)
    if k <= 0 or rows == 0:
        out = torch.empty((rows, max(k, 0)), dtype=torch.int64, device=v.device)
        return like_input(out, values)
    if v.dtype != torch.float32:
        # f64 rows (rerank scores): stable device sort keeps ties in index order
        idx = torch.sort(v, dim=1, descending=True, stable=True).indices[:, :k]
        return like_input(idx, values)
    idx = torch.empty((rows, k), dtype=torch.int32, device=v.device)
    N.check(N.lib().ctkv_topk_rows(N.ptr(v), rows, n, k, N.ptr(idx), None, 0, N.stream_ptr()),
            "top_k_rows")
    return like_input(idx.long(), values)


def top_k(values, k: int):
    """1-D top-k (ck/tensor_ops.py:121-141)."""
    arr = values if isinstance(values, (np.ndarray, torch.Tensor)) else np.asarray(values)
    if arr.ndim != 1:
        raise ShapeError(f"top_k: expected a 1-D row, got shape {tuple(arr.shape)}")
    n = arr.shape[0]
    k = min(int(k), n)
    if k <= 0:
        return np.empty(0, dtype=np.int64) if is_host(arr) else torch.empty(0, dtype=torch.int64)
    if is_host(arr) and arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    out = top_k_rows(arr.reshape(1, n), k)
    return out[0]


def cosine(qa, qb) -> float:
    """ck/tensor_ops.py:172-187 (device f64)."""
    a = to_device(qa, torch.float64).reshape(-1)
    b = to_device(qb, torch.float64).reshape(-1)
    if a.shape != b.shape:
        raise ShapeError(f"cosine: length mismatch {tuple(a.shape)} vs {tuple(b.shape)}")
    na, nb = torch.linalg.norm(a), torch.linalg.norm(b)
    if float(na) == 0.0 or float(nb) == 0.0:
        warnings.warn("cosine of a zero-norm vector is defined as 0", DegenerateQueryWarning)
        return 0.0
    return float(torch.clamp(a @ b / (na * nb), -1.0, 1.0))


def scale_of(d: int) -> float:
    return 1.0 / math.sqrt(d)
