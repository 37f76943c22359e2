"""Per-call cost of the drop-in Python API (the reference's own entry
points, ck/session.py:42-64 and ck/retrieval.py:304-378) at the cfg2
single-layer geometry (b = 8, 32q/8kv, d = 128, 96K, C = 2048, rho = 1280,
C' = 4, rho' = 512, bf16), against the serving engine's per-layer time.

  * run_decode(T)                 -- T steps, one host transfer at the end
  * append + decode_step per step  -- the reference's per-step call pattern,
                                      one host round trip per step (the
                                      TraceRow needs the sparse ids)
  * DecodeEngine (1 layer, graph)  -- the same step replayed as a graph

One JSON line per leg.  usage: python scripts/api_bench.py [T]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15550_b200 as P  # noqa: E402
from paper_2512_15550_b200.engine import DecodeEngine  # noqa: E402
from paper_2512_15550_b200.index import QueryCentroidIndex  # noqa: E402
from paper_2512_15550_b200.store import KvStore  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 16
b, h, g, d, s, C = 8, 32, 8, 128, 98304, 2048
cfg = P.DecodeConfig(4, 512)


def layer(extra):
    lay = P.HeadLayout(b, h, g, s + extra, d)
    q, k, v, _ = P.generate(P.DriftConfig(seed=7, s=s, decode_steps=extra), lay, dtype=torch.bfloat16,
                            q_rows=(s - C, s + extra))
    st = KvStore(P.HeadLayout(b, h, g, s, d), 128, 1024, dtype=torch.bfloat16, capacity=s + extra,
                 host_api=False)
    st.keys[:, :, :s].copy_(k[:, :, :s])
    st.values[:, :, :s].copy_(v[:, :, :s])
    st._set_total(s)
    ix = QueryCentroidIndex.build(q[:, :, :C].contiguous(), st, C, 1280)
    return st, ix, q[:, :, C:].contiguous(), k[:, :, s:].contiguous(), v[:, :, s:].contiguous()


def line(leg, ms, n):
    print(json.dumps({"leg": leg, "ms_per_step": ms / n, "steps": n,
                      "tok_s_one_layer": b / (ms / n / 1e3)}))


st, ix, dq, dk, dv = layer(4 * T + 8)
# warm-up
P.run_decode(st, ix, cfg, dq[:, :, :2], dk[:, :, :2], dv[:, :, :2])
torch.cuda.synchronize()
t0 = time.perf_counter()
P.run_decode(st, ix, cfg, dq[:, :, 2:2 + T], dk[:, :, 2:2 + T], dv[:, :, 2:2 + T])
torch.cuda.synchronize()
line("run_decode", (time.perf_counter() - t0) * 1e3, T)

state = P.DecodeState(st, ix, cfg)
o = 2 + T
st.append(dk[:, :, o], dv[:, :, o])
P.decode_step(state, dq[:, :, o])
torch.cuda.synchronize()
t0 = time.perf_counter()
for t in range(o + 1, o + 1 + T):
    st.append(dk[:, :, t], dv[:, :, t])
    P.decode_step(state, dq[:, :, t])
torch.cuda.synchronize()
line("append+decode_step", (time.perf_counter() - t0) * 1e3, T)

o = o + 1 + T
eng = DecodeEngine([(st, ix)], cfg, lanes=1)
eng.q[0].copy_(dq[:, :, o])
eng.k[0].copy_(dk[:, :, o])
eng.v[0].copy_(dv[:, :, o])
eng.step()
eng.capture()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for t in range(o + 1, o + 1 + T):
    eng.q[0].copy_(dq[:, :, t])
    eng.k[0].copy_(dk[:, :, t])
    eng.v[0].copy_(dv[:, :, t])
    eng.replay()
e1.record()
torch.cuda.synchronize()
eng.check()
line("engine 1 layer, graph replay", e0.elapsed_time(e1), T)
