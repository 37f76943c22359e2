"""Per-CTA timeline of one scan2 launch at lane size (1 sequence = 8 units)
and at full-layer size: CTA start / first rows landed / compute done / end."""
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

b = int(sys.argv[1]) if len(sys.argv) > 1 else 8     # cfg3 geometry: 16 4
g = int(sys.argv[2]) if len(sys.argv) > 2 else 8
h, d, s, C, T = 32, 128, 98304, 2048, 16
CPU = C // (256 // (h // g))   # cosine chunks per unit
NS = 9                         # static splits per unit (1152 tokens / 128)
lay = P.HeadLayout(b, h, g, s + T, d)
q, k, v, _ = P.generate(P.DriftConfig(seed=42, s=s, decode_steps=T), lay, dtype=torch.bfloat16,
                        q_rows=(s - C, s + T))
st = KvStore(P.HeadLayout(b, h, g, s, d), 128, 1024, dtype=torch.bfloat16, capacity=s + T, host_api=False)
st.keys[:, :, :s].copy_(k[:, :, :s])
st.values[:, :, :s].copy_(v[:, :, :s])
st._set_total(s)
ix = QueryCentroidIndex.build(q[:, :, :C].contiguous(), st, C, 1280)
lib = N.lib()
for lanes in (4, 1):
    eng = DecodeEngine([(st, ix)], P.DecodeConfig(4, 512), lanes=lanes)
    for t in range(3):
        eng.q[0].copy_(q[:, :, C + t])
        eng.k[0].copy_(k[:, :, s + t])
        eng.v[0].copy_(v[:, :, s + t])
        if t == 2:
            torch.cuda.synchronize()
            lib.ctkv_debug_scan_timeline(1, None, 0)
            eng._launch(eng.lane_layers[0][0], 1)
            torch.cuda.synchronize()
            n = 4096 * 8
            buf = (ctypes.c_uint64 * n)()
            lib.ctkv_debug_scan_timeline(0, buf, n)
            nct = eng.bl * g * (CPU + NS)
            a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8).astype(np.int64)[:nct]
            t0 = a[:, 0].min()
            r = (a - t0) / 1e3
            print(f"lanes={lanes}: {nct} CTAs; span {r[:, 3].max():.1f} us")
            for nm, col in (("start", 0), ("rows landed", 1), ("compute done", 2), ("end", 3)):
                x = r[:, col][a[:, col] > 0]
                print(f"  {nm:13s} min {x.min():6.1f} median {np.median(x):6.1f} p90 {np.percentile(x, 90):6.1f} max {x.max():6.1f}")
            ncos = eng.bl * g * CPU
            lat = (a[:ncos, 1] - a[:ncos, 0]) / 1e3
            print(f"  cos CTA: start->rows median {np.median(lat):.1f} us; rows->done median {np.median((a[:ncos,2]-a[:ncos,1])/1e3):.1f}; done->end median {np.median((a[:ncos,3]-a[:ncos,2])/1e3):.1f}")
            stl = (a[ncos:, 2] - a[ncos:, 0]) / 1e3
            print(f"  static CTA: start->done median {np.median(stl):.1f} us")
            sa = a[ncos:]
            for nm, c0_, c1_ in (("start->K landed", 0, 1), ("logits", 1, 4), ("softmax", 4, 5),
                                 ("V wait", 5, 6), ("P.V + store", 6, 2)):
                print(f"    static {nm:16s} median {np.median((sa[:, c1_] - sa[:, c0_]) / 1e3):.2f} us")
            last = [i for i in range(ncos) if a[i, 7] > 0]
            for i in last[:8]:
                print(f"    last cos CTA {i}: rows {r[i,1]:.1f} dots+gcos {r[i,4]:.1f} atomic {r[i,5]:.1f} fence {r[i,6]:.1f} select done {r[i,7]:.1f}")
            order = np.argsort(-a[:, 3])[:10]
            for i in order:
                kind = f"cos u{i // CPU} c{i % CPU}" if i < ncos else f"static u{(i - ncos) // NS} s{(i - ncos) % NS}"
                print(f"    slow CTA {i:4d} {kind:16s} start {r[i,0]:5.1f} rows {r[i,1]:5.1f} done {r[i,2]:5.1f} end {r[i,3]:5.1f}")
        else:
            eng.step()
        torch.cuda.synchronize()
    eng.check()
    del eng
