"""Phase breakdown of ONE chain launch in the middle of a loaded 4-lane
step (cfg2 geometry, 8 layers): the engine enqueues eagerly, and the
chain's phase timestamps are switched on only for the chosen (lane, layer)
launch, so the marks describe a chain that shares the GPU with the other
lanes' scans and chains (the per-CTA-slot buffers otherwise hold whichever
launch ran last)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15550_b200 as P  # noqa: E402
from paper_2512_15550_b200 import _native as N  # noqa: E402
N.use_profile_library()
from paper_2512_15550_b200.engine import DecodeEngine  # noqa: E402
from paper_2512_15550_b200.index import QueryCentroidIndex  # noqa: E402
from paper_2512_15550_b200.store import KvStore  # noqa: E402

NL, LANES = 8, 4
want_lane, want_layer = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (1, 4)
b, h, g, d, s, C, T = 8, 32, 8, 128, 98304, 2048, 16
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
eng = DecodeEngine(built, P.DecodeConfig(4, 512), lanes=LANES)
iid = "iid" in sys.argv[3:]   # iid Gaussian inputs (alpha ~0.75) instead of drift


def load(t):
    if iid:
        eng.q.normal_()
        eng.k.normal_()
        eng.v.normal_()
        return
    for li in range(NL):
        eng.q[li].copy_(tails[li][0][:, :, t])
        eng.k[li].copy_(tails[li][1][:, :, t])
        eng.v[li].copy_(tails[li][2][:, :, t])


target = eng.lane_layers[want_lane][want_layer]
orig = eng._launch


def hooked(layer, phase, stream=None):
    on = layer is target and (phase & 2)
    if on:
        lib.ctkv_debug_phase_timing(1, None, 0)
    orig(layer, phase, stream)
    if on:
        lib.ctkv_debug_phase_timing(0, None, 0)


graph = "graph" in sys.argv[3:]
if graph:   # the debug bit is a kernel parameter: capture with it on for the target launch only
    for t in range(2):
        load(t)
        eng.step()
    torch.cuda.synchronize()
    eng._launch = hooked
    eng.capture()
    eng._launch = orig
    for t in range(2, 6):
        load(t)
        eng.replay()
        torch.cuda.synchronize()
else:
    for t in range(3):
        load(t)
        eng._launch = hooked if t == 2 else orig
        eng.step()
        torch.cuda.synchronize()
n = 512 * 16
buf = (ctypes.c_uint64 * n)()
lib.ctkv_debug_phase_timing(-1, buf, n)
a = np.frombuffer(buf, dtype=np.uint64).reshape(512, 16).astype(np.int64)[:eng.bl * g * 4]
names = ["start", "q + slots", "lists+survivors", "sync2", "pull ids", "logits", "sync3",
         "pull keys", "threshold", "compaction", "attention", "sync4+merge"]
t0 = a[:, 0].min()
print(f"chain (lane {want_lane}, layer {want_layer}{', iid inputs' if iid else ''}{', graph replay' if graph else ', eager'}) under load: {a.shape[0]} CTAs, "
      f"start spread {(a[:, 0].max() - t0) / 1e3:.2f} us, span {(a[0::4, 11].max() - t0) / 1e3:.2f} us")
for kk in range(1, 12):
    dd = (a[:, kk] - a[:, kk - 1]) / 1e3 if kk < 11 else (a[0::4, 11] - a[0::4, 10]) / 1e3
    print(f"  {names[kk]:18s} median {np.median(dd):6.2f}  max {dd.max():6.2f} us")
