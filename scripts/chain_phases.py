"""Phase breakdown of the v6 chain kernel (4-CTA cluster per unit) on a
cfg2-sized layer (or B x G units: chain_phases.py LANES B G): one eager step with device phase timestamps on, printed
as per-phase medians over the units' CTAs."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15550_b200 as P  # noqa: E402
from paper_2512_15550_b200 import _native as N  # noqa: E402
N.use_profile_library()   # the timestamp marks exist only in the profiling build
from paper_2512_15550_b200.engine import DecodeEngine  # noqa: E402
from paper_2512_15550_b200.index import QueryCentroidIndex  # noqa: E402
from paper_2512_15550_b200.store import KvStore  # noqa: E402

lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 4
b = int(sys.argv[2]) if len(sys.argv) > 2 else 8     # cfg3 geometry: LANES 16 4
g = int(sys.argv[3]) if len(sys.argv) > 3 else 8
h, d, s, C, T = 32, 128, 98304, 2048, 16
lay = P.HeadLayout(b, h, g, s + T, d)
q, k, v, _ = P.generate(P.DriftConfig(seed=42, s=s, decode_steps=T), lay, dtype=torch.bfloat16,
                        q_rows=(s - C, s + T))
st = KvStore(P.HeadLayout(b, h, g, s, d), 128, 1024, dtype=torch.bfloat16, capacity=s + T,
             host_api=False)
st.keys[:, :, :s].copy_(k[:, :, :s])
st.values[:, :, :s].copy_(v[:, :, :s])
st._set_total(s)
ix = QueryCentroidIndex.build(q[:, :, :C].contiguous(), st, C, 1280)
eng = DecodeEngine([(st, ix)], P.DecodeConfig(4, 512), lanes=lanes)
lib = N.lib()
names = ["start", "q + slots", "lists+survivors", "sync2", "pull ids", "logits",
         "sync3", "pull keys", "threshold", "compaction", "attention", "sync4+merge"]
for t in range(4):
    eng.q[0].copy_(q[:, :, C + t])
    eng.k[0].copy_(k[:, :, s + t])
    eng.v[0].copy_(v[:, :, s + t])
    if t == 3:
        torch.cuda.synchronize()
        lib.ctkv_debug_phase_timing(1, None, 0)
        L0 = eng.lane_layers[0][0]
        eng._launch(L0, 1)
        torch.cuda.synchronize()
        eng._launch(L0, 2 | 8)
        torch.cuda.synchronize()
        n = 512 * 16
        buf = (ctypes.c_uint64 * n)()
        lib.ctkv_debug_phase_timing(0, buf, n)
        a = np.frombuffer(buf, dtype=np.uint64).reshape(512, 16).astype(np.int64)
        nct = eng.bl * g * 4
        a = a[:nct]
        t0 = a[:, 0].min()
        print(f"lanes={lanes}: {nct} CTAs; start spread {(a[:, 0].max() - t0) / 1e3:.2f} us")
        for kk in range(1, 12):
            rows = a[:, kk] > 0
            dd = (a[rows, kk] - a[rows, kk - 1]) / 1e3
            if len(dd):
                print(f"  {kk:2d} {names[kk]:18s} median {np.median(dd):7.2f} us  max {dd.max():7.2f}")
        print("  per rank (median us):", "  ".join(names[kk][:10] for kk in range(1, 12)))
        for rk in range(4):
            rr = a[rk::4]
            print(f"   rank {rk}:", "  ".join(f"{np.median(rr[:, kk] - rr[:, kk - 1]) / 1e3:10.2f}" for kk in range(1, 12)))
        sub = [(4, 12, "K round 1 issued"), (12, 13, "first K row done"), (13, 14, "rest of round 1"),
               (14, 5, "later rounds")]
        for a0, a1, nm in sub:
            dd = (a[:, a1] - a[:, a0]) / 1e3
            print(f"     logits: {nm:18s} median {np.median(dd):7.2f} us")
        r0 = a[0::4]
        print(f"  end-to-end (rank 0, mark 11 - mark 0): median {np.median(r0[:, 11] - r0[:, 0]) / 1e3:.2f} us")
        print(f"  kernel span: {(a[:, 11].max() - t0) / 1e3:.2f} us")
    else:
        eng.step()
    torch.cuda.synchronize()
