"""Steady-state timeline of one CUDA-graph decode step (cfg2, lanes): per
(lane, layer) the [start, end] span of the scan, chain and tail kernels
(globaltimer, recorded by the kernels when the debug timeline is on)."""
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

NL = int(sys.argv[1]) if len(sys.argv) > 1 else 8
lanes = int(sys.argv[2]) if len(sys.argv) > 2 else 8
b = int(sys.argv[3]) if len(sys.argv) > 3 else 8     # cfg3 geometry: 16 4
g = int(sys.argv[4]) if len(sys.argv) > 4 else 8
h, d, s, C, T = 32, 128, 98304, 2048, 16
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
    tails.append((q[:, :, C:].contiguous(), k[:, :, s:].contiguous(), v[:, :, s:].contiguous()))
    del q, k, v
lib = N.lib()
lib.ctkv_debug_kernel_timeline(1)
lib.ctkv_debug_phase_timing(1, None, 0)   # chain phase marks (a launch parameter: on before capture)
eng = DecodeEngine(built, P.DecodeConfig(4, 512), lanes=lanes)


def load(t):
    for li in range(NL):
        eng.q[li].copy_(tails[li][0][:, :, t])
        eng.k[li].copy_(tails[li][1][:, :, t])
        eng.v[li].copy_(tails[li][2][:, :, t])


buf = (ctypes.c_uint64 * 8)()
for t in range(6):
    load(t)
    if t == 2:
        eng.capture()
    if t >= 4:
        torch.cuda.synchronize()
        for L in eng.layers:
            lay, sd, idd, args, ws, wsn = L.call
            lib.ctkv_debug_timeline_rw(lay, L.index.capacity, L.index.rho, 4, ws, None, 1)
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.replay() if t >= 3 else eng.step()
    e1.record()
    torch.cuda.synchronize()
    if t == 5:
        rows = []
        for k_ in range(lanes):
            for li in range(NL):
                L = eng.lane_layers[k_][li]
                lay, sd, idd, args, ws, wsn = L.call
                lib.ctkv_debug_timeline_rw(lay, L.index.capacity, L.index.rho, 4, ws, buf, 0)
                rows.append((k_, li, list(buf)))
        t0 = min(r[2][0] for r in rows)
        print(f"step {e0.elapsed_time(e1) * 1e3:.0f} us (events), {NL} layers x {lanes} lanes")
        span = {0: [], 1: [], 2: []}
        for k_, li, v in rows:
            for kind in range(3):
                span[kind].append((v[2 * kind + 1] - v[2 * kind]) / 1e3)
        for kind, nm in enumerate(["scan", "chain", "tail"]):
            a = np.array(span[kind])
            print(f"  {nm:6s} span per launch: median {np.median(a):6.1f}  p90 {np.percentile(a, 90):6.1f} us")
        for k_ in range(lanes):
            line = []
            for li in range(NL):
                v = rows[k_ * NL + li][2]
                line.append(f"L{li}: s[{(v[0]-t0)/1e3:.0f},{(v[1]-t0)/1e3:.0f}] c[{(v[2]-t0)/1e3:.0f},{(v[3]-t0)/1e3:.0f}] t[{(v[4]-t0)/1e3:.0f},{(v[5]-t0)/1e3:.0f}]")
            print(f"  lane {k_}: " + "  ".join(line))
        # gaps on a lane's critical path: chain(l) end -> scan(l+1) start, scan end -> chain start
        g1, g2 = [], []
        for k_ in range(lanes):
            for li in range(NL):
                v = rows[k_ * NL + li][2]
                g1.append((v[2] - v[1]) / 1e3)
                if li + 1 < NL:
                    w = rows[k_ * NL + li + 1][2]
                    g2.append((w[0] - v[3]) / 1e3)
        print(f"  gap scan->chain median {np.median(g1):.1f} us; chain->next scan median {np.median(g2):.1f} us")
        sk = [(r[2][7] - r[2][2]) / 1e3 for r in rows]
        print(f"  chain CTA start skew (last start - first start): median {np.median(sk):.1f} us, p90 {np.percentile(sk, 90):.1f}")
n = 512 * 16
pb = (ctypes.c_uint64 * n)()
lib.ctkv_debug_phase_timing(0, pb, n)
a = np.frombuffer(pb, dtype=np.uint64).reshape(512, 16).astype(np.int64)[:min(512, eng.bl * g * 4)]
names = ["start", "q + slots", "lists+survivors", "sync2", "pull ids", "logits", "sync3",
         "pull keys", "threshold", "compaction", "attention", "sync4+merge"]
print("  chain phases under load (last writer per CTA slot): median / p90 / max us")
for kk in range(1, 12):
    rows = a[:, kk] > 0
    dd = (a[rows, kk] - a[rows, kk - 1]) / 1e3
    if kk == 11:
        dd = (a[0::4, 11] - a[0::4, 10]) / 1e3
    print(f"    {names[kk]:18s} {np.median(dd):7.2f} {np.percentile(dd, 90):7.2f} {dd.max():7.2f}")
tot = (a[0::4, 11] - a[0::4, 0]) / 1e3
print(f"  chain CTA-0 start->merge end: median {np.median(tot):.2f} p90 {np.percentile(tot, 90):.2f} max {tot.max():.2f} us")
# per cluster: the slowest rank's attention end vs the fastest's
cl = a.reshape(-1, 4, 16)
lag = (cl[:, :, 10].max(axis=1) - cl[:, :, 10].min(axis=1)) / 1e3
print(f"  cluster imbalance at attention end (max - min rank): median {np.median(lag):.2f} p90 {np.percentile(lag, 90):.2f} us")
lib.ctkv_debug_kernel_timeline(0)
