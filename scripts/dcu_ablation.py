"""SPEC acceptance criterion 7 (Table 6 direction): on an 8-turn drift
workload (s = 8192, rho' = 128, C' = 4, rho = 2.5 rho', C = min(2048, s/16))
the mean recall@rho' against the flat oracle with FIFO centroid updates is
>= the mean without them, for every round >= 2, over 5 seeds.  Runs the
drop-in API (run_decode with the GPU FlatOracle) on one B200; prints one
JSON line with the per-round means."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15550_b200 as P  # noqa: E402

SEEDS = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 3, 4, 5]
TURNS, PER = 8, 16
b, h, g, d, s = 1, 32, 8, 128, 8192
rp = 128
rho, C, T = int(round(2.5 * rp)), min(2048, s // 16), TURNS * PER


def run(seed, use_dcu):
    lay = P.HeadLayout(b, h, g, s + T, d)
    q, k, v, _ = P.generate(P.DriftConfig(seed=seed, s=s, decode_steps=T, turns=TURNS), lay,
                            device="cuda", dtype=torch.float32)
    store, index = P.prefill(q[:, :, :s].contiguous(), k[:, :, :s].contiguous(), v[:, :, :s].contiguous(),
                             P.PrefillParams(128, 1024, C, rho), reserve=T)
    cfg = P.DecodeConfig(4, rp, use_dcu=use_dcu)
    _, trace = P.run_decode(store, index, cfg, q[:, :, s:], k[:, :, s:], v[:, :, s:], with_oracle=True)
    rec = np.array([r.recall_at_k for r in trace], np.float64)
    return rec.reshape(TURNS, PER).mean(axis=1)


with_dcu = np.mean([run(sd, True) for sd in SEEDS], axis=0)
without = np.mean([run(sd, False) for sd in SEEDS], axis=0)
print(json.dumps({"seeds": SEEDS, "rounds": TURNS, "steps_per_round": PER,
                  "recall_with_dcu": [round(x, 4) for x in with_dcu],
                  "recall_without_dcu": [round(x, 4) for x in without],
                  "dcu_ge_without_rounds_2_plus": bool(np.all(with_dcu[1:] >= without[1:]))}))
