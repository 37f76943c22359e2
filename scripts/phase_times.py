"""Phase breakdown of the fused unit kernel on a cfg2-sized layer set.

Runs bench-like setup for a few layers, then one eager step with the device
phase timestamps on, and prints per-phase durations (median over units).
"""
import ctypes
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15550_b200 as P  # noqa: E402
from paper_2512_15550_b200 import _native as N  # noqa: E402
from paper_2512_15550_b200.engine import DecodeEngine  # noqa: E402
from paper_2512_15550_b200.index import QueryCentroidIndex  # noqa: E402
from paper_2512_15550_b200.store import KvStore  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
b, h, g, d, s, C, T = 8, 32, 8, 128, 98304, 2048, 16
lay = P.HeadLayout(b, h, g, s + T, d)
built = []
tails = []
for li in range(layers):
    q, k, v, _ = P.generate(P.DriftConfig(seed=42 + li, s=s, decode_steps=T), lay,
                            dtype=torch.bfloat16, q_rows=(s - C, s + T))
    st = KvStore(P.HeadLayout(b, h, g, s, d), 128, 1024, dtype=torch.bfloat16, capacity=s + T,
                 host_api=False)
    st.keys[:, :, :s].copy_(k[:, :, :s])
    st.values[:, :, :s].copy_(v[:, :, :s])
    st._set_total(s)
    ix = QueryCentroidIndex.build(q[:, :, :C].contiguous(), st, C, 1280)
    built.append((st, ix))
    tails.append((q[:, :, C:].contiguous(), k[:, :, s:].contiguous(), v[:, :, s:].contiguous()))
eng = DecodeEngine(built, P.DecodeConfig(4, 512))
lib = N.lib()
for t in range(3):
    for li in range(layers):
        eng.q[li].copy_(tails[li][0][:, :, t])
        eng.k[li].copy_(tails[li][1][:, :, t])
        eng.v[li].copy_(tails[li][2][:, :, t])
    if t == 2:
        torch.cuda.synchronize()
        lib.ctkv_debug_phase_timing(1, None, 0)
        # only the first layer's unit kernel: run phase 1 + 2 of layer 0 alone
        eng._launch(eng.layers[0], 1)
        eng._launch(eng.layers[0], 2)
        torch.cuda.synchronize()
        buf = (ctypes.c_uint64 * (256 * 12))()
        lib.ctkv_debug_phase_timing(0, buf, 256 * 12)
        a = np.frombuffer(buf, dtype=np.uint64).reshape(256, 12).astype(np.int64)
        t0 = a[:128, 0].min()
        names = {0: "start", 1: "topC'", 2: "union", 3: "logits", 4: "cluster.sync",
                 5: "select|sort", 6: "attn-max|dcu+ids", 7: "attn-accum", 8: "merge"}
        for rank in (0, 1):
            rows = a[rank:128:2]
            print(f"rank {rank}: start offset median {statistics.median(rows[:, 0] - t0)/1e3:.2f} us")
            for k in range(1, 9):
                if (rows[:, k] == 0).all():
                    continue
                dd = rows[:, k] - rows[:, k - 1 if k != 5 or rank == 0 else 4]
                dd = dd[(rows[:, k] > 0) & (rows[:, k - 1] > 0)]
                if len(dd):
                    print(f"   {k} {names.get(k)}: median {np.median(dd)/1e3:7.2f} us  max {dd.max()/1e3:7.2f}")
            print(f"   end-to-end (last mark - start): median {np.median(rows.max(1) - rows[:, 0])/1e3:.2f} us")
    else:
        eng.step()
    torch.cuda.synchronize()
