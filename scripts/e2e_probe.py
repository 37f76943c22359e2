"""Where the e2e step time goes (cfg2 geometry, 32 layers, lanes=4, drift
inputs): per step, the device span of the host-I/O graph (CUDA events
recorded on the launching stream just before / after the replay) and the
host turnaround between one step's end and the next step's start (host
sync wake-up, Python, the graph launch call), against back-to-back device
replays."""
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
built, tails = [], []
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
    tails.append((q[:, :, C:].cpu(), k[:, :, s:].cpu(), v[:, :, s:].cpu()))
    del q, k, v
eng = DecodeEngine(built, P.DecodeConfig(4, 512), lanes=4)


def host_inputs(t):
    return (torch.stack([tl[0][:, :, t] for tl in tails]), torch.stack([tl[1][:, :, t] for tl in tails]),
            torch.stack([tl[2][:, :, t] for tl in tails]))


step = [0]


def load_dev():
    hq, hk, hv = host_inputs(step[0])
    eng.q.copy_(hq)
    eng.k.copy_(hk)
    eng.v.copy_(hv)
    step[0] += 1


for _ in range(2):
    load_dev()
    eng.step()
torch.cuda.synchronize()
eng.capture()
n = 10
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    load_dev()
    eng.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(n):
    eng.replay()
e1.record()
torch.cuda.synchronize()
print(f"A back-to-back replays (device inputs fixed): {e0.elapsed_time(e1) / n * 1e3:.0f} us/step")
hb = eng.capture_host_io(2)


def fill(slot):
    hq, hk, hv = host_inputs(step[0])
    hb[slot][0].copy_(hq)
    hb[slot][1].copy_(hk)
    hb[slot][2].copy_(hv)
    step[0] += 1


fill(0)
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
launch, wall = [], []
torch.cuda.synchronize()
w0 = time.perf_counter()
for t in range(n):
    cs = torch.cuda.current_stream()
    evs[t][0].record(cs)
    t0 = time.perf_counter()
    eng.replay_host(t % 2)
    launch.append((time.perf_counter() - t0) * 1e6)
    evs[t][1].record(cs)
    if t + 1 < n:
        fill((t + 1) % 2)
    cs.synchronize()
wall_us = (time.perf_counter() - w0) / n * 1e6
span = [evs[t][0].elapsed_time(evs[t][1]) * 1e3 for t in range(n)]
gap = [evs[t][1].elapsed_time(evs[t + 1][0]) * 1e3 for t in range(n - 1)]
print(f"C host-I/O steps: wall {wall_us:.0f} us/step; device span {statistics.median(span):.0f} us; "
      f"turnaround (end -> next start) {statistics.median(gap):.0f} us; launch call {statistics.median(launch):.0f} us")
