"""Synthetic drift workload on the GPU + the CTKV dump format.

`generate` reproduces the *distribution* of the reference generator
(ck/workload.py:156-242): per-(b, head, turn) base direction with spectral
decay 0.8 (:42, :117-123), slow drift of drift_rate rad/token (:189-192),
spectrally weighted noise, RoPE base 1e4 (:95-110), keys w*N(0,1)/sqrt(d)
post-RoPE, values N(0,1), and two needles per turn per (b, kv head) planted
3 sigma above their designated query's background maximum (:211-241).  It
runs as batched torch ops on the device so a 96K x 32-layer x b=8 input
set takes seconds instead of the reference's ~54 s per (b=1, layer); the
random stream differs from numpy's, which is why bit-exact parity cases use
the reference-pinned CPU generator under oracle/ instead.

`q_rows` lets a caller materialise only the query positions it needs (the
last C prefill positions become the centroids, the decode tail drives the
steps), which keeps the bench's Q footprint at a few MB per layer.
"""

from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass

import numpy as np
import torch

from .errors import ConfigError, FormatError
from .tensor_ops import HeadLayout

MAGIC = b"CTKV"
VERSION = 1
ROPE_BASE = 10000.0
NEEDLES_PER_TURN = 2
SPECTRAL_DECAY = 0.8
TURN_CARRYOVER = 0.75


@dataclass(frozen=True)
class DriftConfig:
    """ck/workload.py:50-74."""

    seed: int = 42
    s: int = 32768
    decode_steps: int = 256
    drift_rate: float = 1e-4
    noise_sigma: float = 0.05
    turns: int = 1

    def __post_init__(self):
        if self.drift_rate < 0 or self.noise_sigma < 0:
            raise ConfigError("drift_rate and noise_sigma must be non-negative")
        if self.turns < 1:
            raise ConfigError("turns must be >= 1")
        if self.s < 1 or self.decode_steps < 0:
            raise ConfigError("s must be positive and decode_steps non-negative")

    @property
    def total_len(self) -> int:
        return self.s + self.decode_steps


def spectral_weights(d: int, device=None) -> torch.Tensor:
    w = SPECTRAL_DECAY ** torch.arange(d // 2 - 1, -1, -1, dtype=torch.float64, device=device)
    w = w.repeat_interleave(2)
    return w / torch.linalg.norm(w) * math.sqrt(d)


def apply_rope(x, position, base: float = ROPE_BASE):
    """Rotate coordinate pairs by position-scaled angles (f64 angles)."""
    host = isinstance(x, np.ndarray)
    t = torch.as_tensor(x)
    d = t.shape[-1]
    if d % 2:
        raise ConfigError(f"rotary embedding requires an even head_dim, got {d}")
    freqs = base ** (-torch.arange(0, d, 2, dtype=torch.float64, device=t.device) / d)
    pos = torch.as_tensor(position, dtype=torch.float64, device=t.device)
    ang = pos[..., None] * freqs
    c, s = torch.cos(ang), torch.sin(ang)
    tt = t.double()
    ev, od = tt[..., 0::2], tt[..., 1::2]
    out = torch.empty_like(tt)
    out[..., 0::2] = ev * c - od * s
    out[..., 1::2] = ev * s + od * c
    out = out.to(t.dtype) if t.dtype in (torch.float32, torch.bfloat16) else out
    return out.numpy() if host else out


def _segments(cfg: DriftConfig):
    if cfg.decode_steps == 0 or cfg.turns == 1:
        return [(0, cfg.total_len, 0)]
    edges = np.linspace(cfg.s, cfg.total_len, cfg.turns + 1).astype(int)
    return [(0, int(edges[1]), 0)] + [(int(edges[r]), int(edges[r + 1]), r)
                                      for r in range(1, cfg.turns)]


def _unit(v: torch.Tensor) -> torch.Tensor:
    return v / torch.linalg.norm(v, dim=-1, keepdim=True)


def _rope_rows(x: torch.Tensor, pos: torch.Tensor, freqs: torch.Tensor) -> torch.Tensor:
    """x [..., T, d] f64/f32, pos [T] f64 -> rotated, same dtype as x."""
    ang = pos[:, None] * freqs[None, :]
    c, s = torch.cos(ang).to(x.dtype), torch.sin(ang).to(x.dtype)
    ev, od = x[..., 0::2], x[..., 1::2]
    out = torch.empty_like(x)
    out[..., 0::2] = ev * c - od * s
    out[..., 1::2] = ev * s + od * c
    return out


def generate(cfg: DriftConfig, layout: HeadLayout, *, device=None, dtype=torch.float32,
             q_rows: tuple[int, int] | None = None, needles: bool = True):
    """Drift-regime (Q, K, V, needles) on the device.

    Q is [b, h, T_q, d] for positions q_rows=(lo, hi) (default: all),
    K/V are [b, g, T, d]; all `dtype`, post-RoPE.  `needles` lists
    (batch, kv_head, token_id, turn, designated_pos, scale) tuples.
    """
    if layout.head_dim % 2:
        raise ConfigError("generate: head_dim must be even for rotary embedding")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    b, h, g, d = layout.batch, layout.query_heads, layout.kv_heads, layout.head_dim
    gs = h // g
    T = cfg.total_len
    lo, hi = (0, T) if q_rows is None else q_rows
    gen = torch.Generator(device=dev)
    gen.manual_seed(cfg.seed)
    w = spectral_weights(d, dev)
    freqs = ROPE_BASE ** (-torch.arange(0, d, 2, dtype=torch.float64, device=dev) / d)
    segs = _segments(cfg)

    # per (b, h, segment) base / ortho directions (f64)
    def pair(n):
        a = _unit(w * torch.randn((n, d), generator=gen, device=dev, dtype=torch.float64))
        o = w * torch.randn((n, d), generator=gen, device=dev, dtype=torch.float64)
        o = _unit(o - (o * a).sum(-1, keepdim=True) * a)
        return a, o

    bases, orthos = [], []
    base = None
    for _ in segs:
        a, o = pair(b * h)
        if base is None:
            base = a
        else:
            a = _unit(a - (a * base).sum(-1, keepdim=True) * base)
            base = TURN_CARRYOVER * base + math.sqrt(1.0 - TURN_CARRYOVER ** 2) * a
            o = _unit(o - (o * base).sum(-1, keepdim=True) * base)
        bases.append(base)
        orthos.append(o)

    def queries(p0: int, p1: int) -> torch.Tensor:
        """f64 post-RoPE queries [b*h, p1-p0, d] for positions [p0, p1)."""
        out = torch.empty((b * h, p1 - p0, d), dtype=torch.float64, device=dev)
        for (s0, s1, _), bs, orr in zip(segs, bases, orthos):
            a0, a1 = max(s0, p0), min(s1, p1)
            if a1 <= a0:
                continue
            phi = cfg.drift_rate * torch.arange(a0 - s0, a1 - s0, dtype=torch.float64, device=dev)
            out[:, a0 - p0:a1 - p0] = (torch.cos(phi)[None, :, None] * bs[:, None, :]
                                       + torch.sin(phi)[None, :, None] * orr[:, None, :])
        if cfg.noise_sigma > 0:
            # noise is keyed by position so any row window sees the same draw
            g2 = torch.Generator(device=dev)
            g2.manual_seed(cfg.seed * 1000003 + p0)
            noise = torch.randn((b * h, p1 - p0, d), generator=g2, device=dev, dtype=torch.float64)
            out += cfg.noise_sigma * (w * noise) / math.sqrt(d)
        pos = torch.arange(p0, p1, dtype=torch.float64, device=dev)
        return _rope_rows(out, pos, freqs)

    q = queries(lo, hi).view(b, h, hi - lo, d).to(dtype)

    # keys / values, generated in position chunks to bound f32 temporaries
    keys = torch.empty((b, g, T, d), dtype=dtype, device=dev)
    values = torch.empty((b, g, T, d), dtype=dtype, device=dev)
    wf = (w / math.sqrt(d)).float()
    step = max(1, (1 << 26) // max(1, b * g * d))
    for p0 in range(0, T, step):
        p1 = min(T, p0 + step)
        kk = torch.randn((b, g, p1 - p0, d), generator=gen, device=dev, dtype=torch.float32) * wf
        pos = torch.arange(p0, p1, dtype=torch.float64, device=dev)
        keys[:, :, p0:p1] = _rope_rows(kk, pos, freqs).to(dtype)
        values[:, :, p0:p1] = torch.randn((b, g, p1 - p0, d), generator=gen, device=dev,
                                          dtype=torch.float32).to(dtype)

    planted = []
    n_lo, n_hi = int(0.1 * cfg.s), int(0.75 * cfg.s)
    if needles and n_hi > n_lo:
        want = len(segs) * NEEDLES_PER_TURN * b * g
        count = min(want, n_hi - n_lo)
        spots = (torch.randperm(n_hi - n_lo, generator=gen, device=dev)[:count] + n_lo).tolist()
        plan = []
        it = iter(spots)
        for s0, s1, turn in segs:
            first = (cfg.s if cfg.decode_steps > 0 else cfg.s - 1) if turn == 0 else s0
            for bi in range(b):
                for gi in range(g):
                    for j in range(NEEDLES_PER_TURN):
                        p = next(it, None)
                        if p is None:
                            break
                        plan.append((bi, gi, p, turn, min(first + 3 * j, s1 - 1, T - 1)))
        best = {}
        qdes = {}
        for bi, gi, p, turn, des in plan:
            if des not in qdes:
                qdes[des] = queries(des, des + 1)[:, 0].view(b, h, d)
            heads = qdes[des][bi, gi * gs:(gi + 1) * gs].float()
            bg = (heads @ keys[bi, gi].float().T).max(dim=0).values
            val = float(bg.max() + 3.0 * bg.std())
            best[(bi, gi, turn)] = max(best.get((bi, gi, turn), 0.0), val)
        for bi, gi, p, turn, des in plan:
            scale = best[(bi, gi, turn)]
            dq = qdes[des][bi, gi * gs]
            keys[bi, gi, p] = (scale * _unit(dq)).to(dtype)
            planted.append((bi, gi, p, turn, des, scale))
    return q, keys, values, planted


# -- CTKV dump format (ck/workload.py:247-287), byte-compatible -------------
# 28-byte little-endian header: b"CTKV", then u32 version, b, h, g, s, d;
# then Q [b,h,s,d], K [b,g,s,d], V [b,g,s,d] as little-endian f32, row-major.

_DUMP_HDR = np.dtype([("magic", "S4"), ("version", "<u4"), ("b", "<u4"), ("h", "<u4"),
                      ("g", "<u4"), ("s", "<u4"), ("d", "<u4")])


def _host_f32(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        x = x.detach().float().cpu().numpy()
    return np.asarray(x)


def write_dump(path, q, k, v) -> None:
    """Write Q/K/V as a CTKV dump (device tensors are copied to the host)."""
    q, k, v = _host_f32(q), _host_f32(k), _host_f32(v)
    if min(q.ndim, k.ndim, v.ndim) != 4 or max(q.ndim, k.ndim, v.ndim) != 4:
        raise ConfigError("write_dump: Q, K and V must all be rank-4 arrays")
    b, h, s, d = q.shape
    kv = (b, k.shape[1], s, d)
    if k.shape != kv or v.shape != kv:
        raise ConfigError(f"write_dump: K {k.shape} / V {v.shape} do not pair with Q {q.shape}")
    hdr = np.array([(MAGIC, VERSION, b, h, kv[1], s, d)], dtype=_DUMP_HDR)
    with open(path, "wb") as fh:
        fh.write(hdr.tobytes())
        for arr in (q, k, v):
            fh.write(np.ascontiguousarray(arr, dtype="<f4").tobytes())


def read_dump(path):
    """Read a CTKV dump -> (q, k, v, HeadLayout); FormatError on a bad or
    truncated file."""
    blob = np.fromfile(path, dtype=np.uint8)
    if blob.size < _DUMP_HDR.itemsize:
        raise FormatError(f"{path}: {blob.size} bytes is shorter than the "
                          f"{_DUMP_HDR.itemsize}-byte CTKV header")
    hdr = blob[:_DUMP_HDR.itemsize].view(_DUMP_HDR)[0]
    if bytes(hdr["magic"]) != MAGIC:
        raise FormatError(f"{path}: not a CTKV dump (magic {bytes(hdr['magic'])!r})")
    if int(hdr["version"]) != VERSION:
        raise FormatError(f"{path}: CTKV version {int(hdr['version'])} is not supported")
    b, h, g, s, d = (int(hdr[f]) for f in ("b", "h", "g", "s", "d"))
    shapes = ((b, h, s, d), (b, g, s, d), (b, g, s, d))
    need = _DUMP_HDR.itemsize + 4 * sum(int(np.prod(sh)) for sh in shapes)
    if blob.size != need:
        raise FormatError(f"{path}: CTKV payload size mismatch: file has {blob.size} bytes, "
                          f"the header implies {need}")
    body = blob[_DUMP_HDR.itemsize:].view("<f4")
    out, at = [], 0
    for sh in shapes:
        n = int(np.prod(sh))
        out.append(body[at:at + n].reshape(sh).astype(np.float32))
        at += n
    return out[0], out[1], out[2], HeadLayout(batch=b, query_heads=h, kv_heads=g, seq_len=s,
                                              head_dim=d)


def write_sidecar(path, cfg: DriftConfig, layout: HeadLayout, needles) -> None:
    doc = {"config": asdict(cfg), "layout": asdict(layout),
           "needles": [dict(zip(("batch", "kv_head", "token_id", "turn", "designated_pos", "scale"), n))
                       for n in needles]}
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=2, sort_keys=True)
        fh.write("\n")
