"""cfg4 (BASELINE configs[3]): prefill centroid-index build sweep at the
Llama-3-8B geometry (32q/8kv, d=128), 96K context, C x rho, bf16, the
tcgen05 build (BUILD_FAST).  One JSON line per point: ms per (layer, seq)
(CUDA events, median of 3 after a warm-up), TFLOP/s and the fraction of the
measured sustained bf16 peak (MEASURED_PEAKS.json).  FLOPs = 2*h*C*n_off*d
per (layer, seq).

usage: python scripts/build_sweep.py [--batch B] [--C 256,512,...] [--rho 640,...]
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_15550_b200 as P  # noqa: E402
from paper_2512_15550_b200 import _native as N  # noqa: E402
from paper_2512_15550_b200.index import QueryCentroidIndex  # noqa: E402
from paper_2512_15550_b200.store import KvStore  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--seq", type=int, default=98304)
ap.add_argument("--C", default="256,512,1024,2048")
ap.add_argument("--rho", default="640,1280,2560")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--check", action="store_true", help="also compare against the exact build")
a = ap.parse_args()
try:
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops_sustained"]
except Exception:
    peak = 1407.0
b, h, g, d, s = a.batch, 32, 8, 128, a.seq
Cs = [int(x) for x in a.C.split(",")]
lay = P.HeadLayout(b, h, g, s, d)
q, k, v, _ = P.generate(P.DriftConfig(seed=42, s=s, decode_steps=0), lay, dtype=torch.bfloat16,
                        q_rows=(s - max(Cs), s))
st = KvStore(lay, 128, 1024, dtype=torch.bfloat16, capacity=s, host_api=False)
st.keys.copy_(k)
st.values.copy_(v)
st._set_total(s)
del k, v
n_off = s - 128 - 1024
for C in Cs:
    cq = q[:, :, max(Cs) - C:].contiguous()
    for rho in [int(x) for x in a.rho.split(",")]:
        times = []
        for r in range(a.reps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ix = QueryCentroidIndex.build(cq, st, C, rho, mode=N.BUILD_FAST)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            if r < a.reps:
                del ix
        ms = statistics.median(times[1:])
        flop = 2 * h * C * n_off * d * b
        rec = {"C": C, "rho": rho, "batch": b, "seq": s, "ms_per_layer": ms,
               "ms_per_layer_seq": ms / b, "tflops": flop / (ms * 1e-3) / 1e12,
               "frac": flop / (ms * 1e-3) / 1e12 / peak, "runs_ms": [round(t, 3) for t in times]}
        if a.check:
            ex = QueryCentroidIndex.build(cq, st, C, rho, mode=N.BUILD_EXACT)
            same = (torch.sort(ix.lists_dev, -1).values == torch.sort(ex.lists_dev, -1).values).all(-1)
            rec["rows_equal_to_exact"] = float(same.float().mean())
            del ex
        del ix
        print(json.dumps(rec), flush=True)
