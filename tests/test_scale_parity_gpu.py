"""Parity at the benchmarked configuration.

The bench's own path -- 96K context, C=2048, rho=1280, rho'=512, C'=4,
bf16 stores, the tcgen05 index build (BUILD_FAST), DecodeEngine with 4
micro-batch lanes, CUDA-graph replay with programmatic dependent launch and
deferred DCU tails -- against the reference package (when importable) and
the pinned oracle on sampled (layer, sequence) units, step by step from a
snapshot of the device state (oracle/unit_parity.py).

Bars (north_star): sparse sets bit-exact except swaps inside the 1e-6
relative tie window of the reference's f64 scores (recall parity >= 0.9 is
the headline bar; expected ~1.0), ranks likewise, outputs within 1e-3
norm-relative (f32 outputs over bf16 storage), post-DCU lists per written
slot by the same tie rule, centroid rows and FIFO cursors exact.
"""

import pytest
import torch

import paper_2512_15550_b200 as P
from oracle import unit_parity as UP
from paper_2512_15550_b200 import _native as N
from paper_2512_15550_b200.engine import DecodeEngine
from paper_2512_15550_b200.index import QueryCentroidIndex
from paper_2512_15550_b200.store import KvStore

pytestmark = pytest.mark.gpu

S, C, RHO, RP, CP, INIT, LOCAL = 98304, 2048, 1280, 512, 4, 128, 1024


def _layers(b, h, g, nl, T, s=S):
    lay = P.HeadLayout(b, h, g, s + T, 128)
    layers, inputs = [], []
    for li in range(nl):
        q, k, v, _ = P.generate(P.DriftConfig(seed=42 + li, s=s, decode_steps=T), lay,
                                dtype=torch.bfloat16, q_rows=(s - C, s + T))
        st = KvStore(P.HeadLayout(b, h, g, s, 128), INIT, LOCAL, dtype=torch.bfloat16,
                     capacity=s + T, host_api=False)
        st.keys[:, :, :s].copy_(k[:, :, :s])
        st.values[:, :, :s].copy_(v[:, :, :s])
        st._set_total(s)
        ix = QueryCentroidIndex.build(q[:, :, :C].contiguous(), st, C, RHO, mode=N.BUILD_FAST)
        layers.append((st, ix))
        inputs.append((q[:, :, C:].contiguous(), k[:, :, s:].contiguous(), v[:, :, s:].contiguous()))
        del q, k, v
    return layers, inputs


@pytest.mark.parametrize("b,h,g,units,s", [
    (8, 32, 8, [(0, 0), (1, 7), (1, 3)], S),     # cfg2 geometry (Llama-3-8B heads)
    (16, 32, 4, [(0, 15), (1, 5)], S),           # cfg3 geometry (Yi-9B heads, gs = 8)
    (4, 4, 1, [(0, 0), (1, 3)], 131072),         # cfg5: one GPU's slice at 128K (8-CTA chains)
])
def test_bench_path_matches_reference_at_96k(b, h, g, units, s):
    torch.cuda.set_device(0)
    nl, warm, steps = 2, 4, 8
    T = warm + steps + 1
    layers, inputs = _layers(b, h, g, nl, T, s)
    eng = DecodeEngine(layers, P.DecodeConfig(CP, RP), lanes=4)

    def load(t):
        for li, (q, k, v) in enumerate(inputs):
            eng.q[li].copy_(q[:, :, t])
            eng.k[li].copy_(k[:, :, t])
            eng.v[li].copy_(v[:, :, t])

    for t in range(warm):                         # eager, capture, graph replays
        load(t)
        if t == 2:
            eng.capture()
        eng.replay() if t >= 2 else eng.step()
    torch.cuda.synchronize()
    eng.check()
    snaps = UP.snapshot(eng, units)
    for t in range(warm, warm + steps):
        load(t)
        eng.replay()
        torch.cuda.synchronize()
        UP.record(eng, snaps)
    eng.check()
    UP.final_state(eng, snaps)
    res = UP.check(snaps, CP, RP)
    summary = {k: v for k, v in res.items() if not k.endswith("_times")}
    print(summary)
    assert res["ref_vs_oracle_digest_mismatch"] == 0, summary
    assert res["recall"] >= 0.99, summary
    assert res["hard_mismatches"] == 0 and res["order_hard"] == 0, summary
    assert res["selected_hard"] == 0, summary       # top-C' slots: ties only
    assert res["recall_len_mismatch"] == 0, summary
    assert res["out_nrel_max"] < 1e-3, summary
    assert res["dcu_hard"] == 0 and res["centroids_equal"] and res["fifo_equal"], summary
