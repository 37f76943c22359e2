"""Where the e2e step time goes (cfg2, 32 layers, lanes=4): back-to-back
graph replays (device), replay + host sync per step, the bench's host-I/O
step (pinned inputs in, outputs out, sync), and the host-side cost of the
graph launch call itself."""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15550_b200 as P  # noqa: E402
from paper_2512_15550_b200.engine import DecodeEngine  # noqa: E402
from paper_2512_15550_b200.index import QueryCentroidIndex  # noqa: E402
from paper_2512_15550_b200.store import KvStore  # noqa: E402

NL = int(sys.argv[1]) if len(sys.argv) > 1 else 32
b, h, g, d, s, C, T = 8, 32, 8, 128, 98304, 2048, 64
built = []
for li in range(NL):
    lay = P.HeadLayout(b, h, g, s + T, d)
    q, k, v, _ = P.generate(P.DriftConfig(seed=42 + li, s=s, decode_steps=T), lay, dtype=torch.bfloat16,
                            q_rows=(s - C, s + T))
    st = KvStore(P.HeadLayout(b, h, g, s, d), 128, 1024, dtype=torch.bfloat16, capacity=s + T,
                 host_api=False)
    st.keys[:, :, :s].copy_(k[:, :, :s])
    st.values[:, :, :s].copy_(v[:, :, :s])
    st._set_total(s)
    built.append((st, QueryCentroidIndex.build(q[:, :, :C].contiguous(), st, C, 1280)))
    del q, k, v
eng = DecodeEngine(built, P.DecodeConfig(4, 512), lanes=4)
eng.q.normal_()
eng.k.normal_()
eng.v.normal_()
for _ in range(2):
    eng.step()
torch.cuda.synchronize()
eng.capture()
hb = eng.capture_host_io(2)
for x in hb:
    x[0].normal_(); x[1].normal_(); x[2].normal_()
n = 12
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(n):
    eng.replay()
e1.record()
torch.cuda.synchronize()
print(f"A back-to-back replay: {e0.elapsed_time(e1) / n * 1e3:.0f} us/step")
launch, tot = [], []
for _ in range(n):
    t0 = time.perf_counter()
    eng.replay()
    t1 = time.perf_counter()
    torch.cuda.current_stream().synchronize()
    t2 = time.perf_counter()
    launch.append((t1 - t0) * 1e6)
    tot.append((t2 - t0) * 1e6)
print(f"B replay + sync: {statistics.median(tot):.0f} us/step (launch call {statistics.median(launch):.0f} us)")
launch, tot = [], []
for i in range(n):
    t0 = time.perf_counter()
    eng.replay_host(i % 2)
    t1 = time.perf_counter()
    torch.cuda.current_stream().synchronize()
    t2 = time.perf_counter()
    launch.append((t1 - t0) * 1e6)
    tot.append((t2 - t0) * 1e6)
print(f"C host-I/O replay + sync: {statistics.median(tot):.0f} us/step (launch call {statistics.median(launch):.0f} us)")
# graph node counts
for nm, gr in (("device", eng.graph), ("host-io", eng._hgraphs[0])):
    try:
        from cuda import cudart
        err, cnt = cudart.cudaGraphGetNodes(gr.raw_cuda_graph() if hasattr(gr, "raw_cuda_graph") else None)
        print(nm, "nodes", cnt)
    except Exception as exc:   # informational only
        print(nm, "nodes: n/a", type(exc).__name__)
