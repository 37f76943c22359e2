"""Per-CTA task timeline of the persistent scan kernel (scan4) on one
cfg2-sized layer (lanes=1): start/end per CTA and task ready times."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15550_b200 as P  # noqa: E402
from paper_2512_15550_b200 import _native as N  # noqa: E402
from paper_2512_15550_b200.engine import DecodeEngine  # noqa: E402
from paper_2512_15550_b200.index import QueryCentroidIndex  # noqa: E402
from paper_2512_15550_b200.store import KvStore  # noqa: E402

b, h, g, d, s, C, T = 8, 32, 8, 128, 98304, 2048, 16
lay = P.HeadLayout(b, h, g, s + T, d)
q, k, v, _ = P.generate(P.DriftConfig(seed=42, s=s, decode_steps=T), lay, dtype=torch.bfloat16,
                        q_rows=(s - C, s + T))
st = KvStore(P.HeadLayout(b, h, g, s, d), 128, 1024, dtype=torch.bfloat16, capacity=s + T, host_api=False)
st.keys[:, :, :s].copy_(k[:, :, :s])
st.values[:, :, :s].copy_(v[:, :, :s])
st._set_total(s)
ix = QueryCentroidIndex.build(q[:, :, :C].contiguous(), st, C, 1280)
eng = DecodeEngine([(st, ix)], P.DecodeConfig(4, 512), lanes=1)
lib = N.lib()
for t in range(4):
    eng.q[0].copy_(q[:, :, C + t])
    eng.k[0].copy_(k[:, :, s + t])
    eng.v[0].copy_(v[:, :, s + t])
    if t == 3:
        torch.cuda.synchronize()
        lib.ctkv_debug_scan_timeline(1, None, 0)
        eng._launch(eng.lane_layers[0][0], 1)
        torch.cuda.synchronize()
        n = 160 * 64
        buf = (ctypes.c_uint64 * n)()
        lib.ctkv_debug_scan_timeline(0, buf, n)
        a = np.frombuffer(buf, dtype=np.uint64).reshape(160, 64).astype(np.int64)[:148]
        t0 = a[:, 0].min()
        st_ = (a[:, 0] - t0) / 1e3
        en = (a[:, 1] - t0) / 1e3
        print(f"CTA start: min {st_.min():.2f} median {np.median(st_):.2f} max {st_.max():.2f} us")
        print(f"CTA end:   min {en.min():.2f} median {np.median(en):.2f} max {en.max():.2f} us")
        for cta in (0, 1, 74, 147):
            row = a[cta, 2:]
            row = row[row > 0]
            print(f"cta {cta}: task ready times (us):", np.round((row - t0) / 1e3, 2).tolist())
        gaps = []
        for cta in range(148):
            row = a[cta, 2:]
            row = row[row > 0]
            gaps += list(np.diff(row) / 1e3)
        gaps = np.array(gaps)
        print(f"inter-task gap: median {np.median(gaps):.2f} p90 {np.percentile(gaps, 90):.2f} max {gaps.max():.2f} us")
    else:
        eng.step()
    torch.cuda.synchronize()
