"""Index build timing at cfg2 geometry (b=8, 32q/8kv, d=128, 96K, C=2048,
rho=1280): QueryCentroidIndex.build per layer, CUDA events, median of runs
after a warm-up (the workspace and list allocations are cached by then)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15550_b200 as P  # noqa: E402
from paper_2512_15550_b200.index import QueryCentroidIndex  # noqa: E402
from paper_2512_15550_b200.store import KvStore  # noqa: E402

b, h, g, d, s, C, rho = 8, 32, 8, 128, 98304, int(sys.argv[1]) if len(sys.argv) > 1 else 2048, 1280
lay = P.HeadLayout(b, h, g, s, d)
q, k, v, _ = P.generate(P.DriftConfig(seed=42, s=s, decode_steps=0), lay, dtype=torch.bfloat16,
                        q_rows=(s - C, s))
st = KvStore(lay, 128, 1024, dtype=torch.bfloat16, capacity=s, host_api=False)
st.keys.copy_(k)
st.values.copy_(v)
st._set_total(s)
cq = q.contiguous()
times = []
for r in range(4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ix = QueryCentroidIndex.build(cq, st, C, rho)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
    del ix
flop = 2 * h * C * (s - 128 - 1024) * d * b
ms = statistics.median(times[1:])
print(f"build C={C} rho={rho} b={b}: {ms:.2f} ms/layer ({ms / b:.2f} ms per layer-seq), "
      f"{flop / (ms * 1e-3) / 1e12:.0f} TFLOP/s; runs {[round(t, 2) for t in times]}")
