"""Device QueryCentroidIndex (ck/index.py:35-190).

State in HBM: centroids [b,h,C,d] (store dtype, raw -- never pre-normalised,
see SURVEY.md section 7 hard part 2), lists [b,g,C,rho] int32 (-1 = empty),
fifo_head [b] int64, plus a tiny int32 sync word array the decode kernel's
last CTA uses to advance the FIFO cursor without a host round trip.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, FormatError, ShapeError
from .store import KvStore
from .tensor_ops import HeadLayout, is_host, to_device

MAGIC = b"QIVF"
VERSION = 1
EMPTY_SLOT = -1

# build precision per store dtype: f32 stores use the f64-exact scores
# kernel (the fp32 parity config); bf16 stores the fast path.
DEFAULT_BUILD_MODE = {torch.float32: N.BUILD_EXACT, torch.bfloat16: N.BUILD_FAST}


class QueryCentroidIndex:
    def __init__(self, layout: HeadLayout, capacity: int, rho: int, centroid_queries, lists,
                 fifo_head=None, *, dtype: torch.dtype | None = None, id_bound: int | None = None):
        b, h, g, d = layout.batch, layout.query_heads, layout.kv_heads, layout.head_dim
        if tuple(centroid_queries.shape) != (b, h, capacity, d):
            raise ShapeError(f"centroid_queries {tuple(centroid_queries.shape)} != {(b, h, capacity, d)}")
        if tuple(lists.shape) != (b, g, capacity, rho):
            raise ShapeError(f"lists {tuple(lists.shape)} != {(b, g, capacity, rho)}")
        ldt = lists.dtype
        if ldt not in (np.int32, torch.int32):
            raise ShapeError(f"lists must be int32, got {ldt}")
        self.layout = layout
        self.capacity = capacity
        self.rho = rho
        self.host_api = is_host(centroid_queries)
        if dtype is None:
            dtype = centroid_queries.dtype if isinstance(centroid_queries, torch.Tensor) else torch.float32
        self.dtype = dtype
        self.cent = to_device(centroid_queries, dtype).clone()
        self.lists_dev = to_device(lists, torch.int32).clone()
        fh = np.zeros(b, dtype=np.int64) if fifo_head is None else fifo_head
        self.fifo_dev = to_device(fh, torch.int64).clone()
        self.sync = torch.zeros(1 + b, dtype=torch.int32, device=self.cent.device)
        if id_bound is None:
            id_bound = int(self.lists_dev.max().item()) + 1 if self.lists_dev.numel() else 0
        self.id_bound = max(int(id_bound), 0)
        self._compute_norms()

    # -- views -----------------------------------------------------------------

    @property
    def centroid_queries(self):
        """Snapshot of the centroids (numpy f32 for host callers)."""
        if self.host_api:
            return self.cent.float().cpu().numpy()
        return self.cent

    @property
    def lists(self):
        return self.lists_dev.cpu().numpy() if self.host_api else self.lists_dev

    @property
    def fifo_head(self):
        return self.fifo_dev.cpu().numpy() if self.host_api else self.fifo_dev

    def desc(self) -> N.IndexDesc:
        return N.IndexDesc(self.cent.data_ptr(), self.lists_dev.data_ptr(),
                           self.fifo_dev.data_ptr(), self.sync.data_ptr(), self.cnorm.data_ptr(),
                           self.capacity, self.rho)

    def batch_view(self, b0: int, b1: int) -> "QueryCentroidIndex":
        """Sequences [b0, b1) sharing this index's centroids, lists, norms and
        FIFO cursors (all updated in place by the DCU), with a private
        completion word array (a decode lane of DecodeEngine)."""
        lay = self.layout
        if not 0 <= b0 < b1 <= lay.batch:
            raise ConfigError(f"batch_view: [{b0}, {b1}) outside [0, {lay.batch})")
        v = QueryCentroidIndex.__new__(QueryCentroidIndex)
        v.layout = HeadLayout(b1 - b0, lay.query_heads, lay.kv_heads, lay.seq_len, lay.head_dim)
        v.capacity, v.rho, v.host_api, v.dtype, v.id_bound = (self.capacity, self.rho, self.host_api,
                                                              self.dtype, self.id_bound)
        v.cent = self.cent[b0:b1]
        v.lists_dev = self.lists_dev[b0:b1]
        v.fifo_dev = self.fifo_dev[b0:b1]
        v.cnorm = self.cnorm[b0:b1]
        v.sync = torch.zeros(1 + b1 - b0, dtype=torch.int32, device=self.cent.device)
        return v

    def _compute_norms(self) -> None:
        """|c| per centroid row (f64-exact, stored f32); kept current by the DCU."""
        lay = self.layout
        self.cnorm = torch.empty((lay.batch, lay.query_heads, self.capacity), dtype=torch.float32,
                                 device=self.cent.device)
        N.check(N.lib().ctkv_centroid_norms(self.ctkv_layout(), self.cent.data_ptr(), self.capacity,
                                            self.cnorm.data_ptr(), N.stream_ptr()), "centroid norms")

    def ctkv_layout(self, store_capacity: int = 0, init_len: int = 0, local_len: int = 0):
        lay = self.layout
        return N.Layout(lay.batch, lay.query_heads, lay.kv_heads, lay.head_dim, store_capacity,
                        N.dtype_code(self.dtype), init_len, local_len, 0)

    # -- construction (ck/index.py:59-99) ----------------------------------------

    @classmethod
    def build(cls, queries, store: KvStore, capacity: int, rho: int, *,
              mode: int | None = None, workspace: torch.Tensor | None = None) -> "QueryCentroidIndex":
        if queries.ndim != 4:
            raise ShapeError(f"build: queries must be 4-D, got {tuple(queries.shape)}")
        b, h, s, d = queries.shape
        layout = HeadLayout(batch=b, query_heads=h, kv_heads=store.layout.kv_heads,
                            seq_len=store.layout.seq_len, head_dim=d)
        if store.layout.head_dim != d or store.layout.batch != b:
            raise ShapeError(f"build: queries {tuple(queries.shape)} do not match store layout")
        if capacity < 1 or capacity > s:
            raise ConfigError(f"build: capacity {capacity} outside [1, {s}]")
        off = store.offloaded_ids()
        if rho < 0 or rho > off.size:
            raise ConfigError(f"build: rho {rho} exceeds offloaded token count {off.size}")
        g = layout.kv_heads
        if isinstance(queries, torch.Tensor) and queries.is_cuda:
            cent = queries[:, :, s - capacity:, :].to(store.dtype).contiguous()
        else:
            cent = to_device(np.ascontiguousarray(np.asarray(queries)[:, :, s - capacity:, :]),
                             store.dtype)
        lists = torch.full((b, g, capacity, rho), EMPTY_SLOT, dtype=torch.int32, device=cent.device)
        if rho > 0:
            mode = DEFAULT_BUILD_MODE[store.dtype] if mode is None else mode
            lay = store.ctkv_layout()
            lib = N.lib()
            ws_bytes = lib.ctkv_build_workspace_bytes(lay, capacity, rho, off.size, mode)
            if workspace is not None and workspace.is_cuda and workspace.numel() >= ws_bytes:
                ws = workspace   # caller-owned scratch, reused across layers
            else:
                ws = torch.empty(max(int(ws_bytes), 1), dtype=torch.uint8, device=cent.device)
            flags = torch.zeros(1, dtype=torch.int32, device=cent.device)
            N.check(lib.ctkv_build_lists(lay, N.ptr(cent), N.ptr(store.keys), int(off[0]),
                                         off.size, capacity, rho, mode, N.ptr(lists), N.ptr(flags),
                                         N.ptr(ws), ws.numel(), N.stream_ptr()), "build")
        idx = cls.__new__(cls)
        idx.layout = layout
        idx.capacity = capacity
        idx.rho = rho
        idx.host_api = is_host(queries)
        idx.dtype = store.dtype
        idx.cent = cent
        idx.lists_dev = lists
        idx.fifo_dev = torch.zeros(b, dtype=torch.int64, device=cent.device)
        idx.sync = torch.zeros(1 + b, dtype=torch.int32, device=cent.device)
        idx.id_bound = store.total_tokens
        idx._compute_norms()
        return idx

    # -- DCU (ck/index.py:103-133) -------------------------------------------------

    def fifo_update(self, query, rerank_scores, recalled_ids) -> None:
        b, h, g, d = (self.layout.batch, self.layout.query_heads, self.layout.kv_heads,
                      self.layout.head_dim)
        q = to_device(query, self.dtype)
        if q.dim() == 4:
            q = q[:, :, 0, :].contiguous()
        if tuple(q.shape) != (b, h, d):
            raise ShapeError(f"fifo_update: query shape {tuple(q.shape)} != {(b, h, d)}")
        lens = np.zeros((b, g), dtype=np.int32)
        for bi in range(b):
            for gi in range(g):
                ids = np.asarray(_host(recalled_ids[bi][gi]))
                sc = np.asarray(_host(rerank_scores[bi][gi]))
                if ids.shape != sc.shape:
                    raise ShapeError(f"fifo_update: {ids.size} ids vs {sc.size} scores at ({bi},{gi})")
                lens[bi, gi] = ids.size
        lmax = max(int(lens.max()), 1)
        rec = np.full((b, g, lmax), -1, dtype=np.int32)
        grp = np.zeros((b, g, lmax), dtype=np.float64)
        for bi in range(b):
            for gi in range(g):
                n = lens[bi, gi]
                rec[bi, gi, :n] = np.asarray(_host(recalled_ids[bi][gi]))
                grp[bi, gi, :n] = np.asarray(_host(rerank_scores[bi][gi]), dtype=np.float64)
        rec_d, len_d, grp_d = to_device(rec), to_device(lens), to_device(grp)
        lib = N.lib()
        lay = self.ctkv_layout()
        ws = torch.empty(_decode_ws(lib, lay, 1, lmax, 1), dtype=torch.uint8, device=q.device)
        N.check(lib.ctkv_fifo_update(lay, self.desc(), N.ptr(q), N.ptr(rec_d), N.ptr(len_d), lmax,
                                     N.ptr(grp_d), N.ptr(ws), ws.numel(), N.stream_ptr()),
                "fifo_update")

    # -- accounting / invariants ---------------------------------------------------

    def size_bytes(self) -> int:
        """ck/index.py:137-139."""
        return self.layout.batch * self.layout.kv_heads * self.capacity * self.rho * 4

    def check_lists(self, store: KvStore) -> None:
        """ck/index.py:141-153, evaluated on the device."""
        if self.rho == 0:
            return
        L = self.lists_dev.long()
        valid = L != EMPTY_SLOT
        srt = torch.sort(torch.where(valid, L, torch.full_like(L, -(2 ** 40))), dim=-1).values
        dup = (srt[..., 1:] == srt[..., :-1]) & (srt[..., 1:] >= 0)
        if bool(dup.any()):
            bi, gi, ci, _ = [int(x) for x in dup.nonzero()[0]]
            raise AssertionError(f"duplicate ids in list ({bi},{gi},{ci})")
        off_ok = (L >= store.init_len) & (L < store.ring_start)
        bad = valid & ~off_ok
        if bool(bad.any()):
            bi, gi, ci, _ = [int(x) for x in bad.nonzero()[0]]
            raise AssertionError(f"non-offloaded id in list ({bi},{gi},{ci})")

    # -- QIVF serialization (ck/index.py:157-190), byte-compatible ------------
    # 32-byte little-endian header: b"QIVF", then u32 version, b, h, g, C,
    # rho, d; then the centroids [b,h,C,d] f32 and the lists [b,g,C,rho] i32.
    # The FIFO cursor is not part of the format (it restarts at 0 on load).

    _HDR = np.dtype([("magic", "S4"), ("version", "<u4"), ("b", "<u4"), ("h", "<u4"),
                     ("g", "<u4"), ("C", "<u4"), ("rho", "<u4"), ("d", "<u4")])

    def save(self, path) -> None:
        lay = self.layout
        hdr = np.array([(MAGIC, VERSION, lay.batch, lay.query_heads, lay.kv_heads,
                         self.capacity, self.rho, lay.head_dim)], dtype=self._HDR)
        with open(path, "wb") as fh:
            fh.write(hdr.tobytes())
            fh.write(self.cent.float().cpu().numpy().astype("<f4", copy=False).tobytes())
            fh.write(self.lists_dev.cpu().numpy().astype("<i4", copy=False).tobytes())

    @classmethod
    def load(cls, path, seq_len: int | None = None, *, dtype: torch.dtype = torch.float32,
             host_api: bool = True) -> "QueryCentroidIndex":
        blob = np.fromfile(path, dtype=np.uint8)
        n_hdr = cls._HDR.itemsize
        if blob.size < n_hdr or bytes(blob[:4]) != MAGIC:
            raise FormatError(f"{path}: not a QIVF index (missing {MAGIC!r} header)")
        hdr = blob[:n_hdr].view(cls._HDR)[0]
        if int(hdr["version"]) != VERSION:
            raise FormatError(f"{path}: QIVF version {int(hdr['version'])} is not supported")
        b, h, g, cap, rho, d = (int(hdr[f]) for f in ("b", "h", "g", "C", "rho", "d"))
        n_cent, n_list = b * h * cap * d, b * g * cap * rho
        need = n_hdr + 4 * (n_cent + n_list)
        if blob.size != need:
            raise FormatError(f"{path}: QIVF payload size mismatch: file has {blob.size} bytes, "
                              f"the header implies {need}")
        body = blob[n_hdr:]
        cq = body[:4 * n_cent].view("<f4").reshape(b, h, cap, d).astype(np.float32)
        li = body[4 * n_cent:].view("<i4").reshape(b, g, cap, rho).astype(np.int32)
        layout = HeadLayout(batch=b, query_heads=h, kv_heads=g,
                            seq_len=cap if seq_len is None else seq_len, head_dim=d)
        idx = cls(layout, cap, rho, cq, li, dtype=dtype)
        idx.host_api = host_api
        return idx


def _host(x):
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return x


def _decode_ws(lib, lay, capacity, lmax, c_prime) -> int:
    # workspace for the staged unit-kernel calls: logits [U, gs, lmax]
    rho = max(1, (lmax + c_prime - 1) // c_prime)
    return max(int(lib.ctkv_decode_workspace_bytes(lay, capacity, rho, c_prime, 1)), 1)
