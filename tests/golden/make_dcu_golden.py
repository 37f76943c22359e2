"""Golden trace of the reference on a multi-turn drift workload (SPEC.md
acceptance criterion 7's setting: 8 turns, s = 8192, rho' = 128, C' = 4,
rho = 2.5 rho' = 320, C = 512; 32q/8kv, d = 128, f32), with and without the
FIFO centroid update: per step the sparse-set digest, recall length and
recall@rho' against the reference FlatOracle.  Run HERE (needs
/root/reference):  python tests/golden/make_dcu_golden.py
Inputs are the drift workload of ck/workload.py:156-242 (reproduced bit for
bit by oracle.ctkv_oracle.generate, so the GPU test regenerates them)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
import centroidkv as ck  # noqa: E402
from oracle import ctkv_oracle as O  # noqa: E402

SEED, TURNS, PER = 1, 8, 16
b, h, g, d, s = 1, 32, 8, 128, 8192
RP, RHO, C, T = 128, 320, 512, TURNS * PER

q, k, v = O.generate(O.Drift(seed=SEED, s=s, decode_steps=T, turns=TURNS), b, h, g, d)
out = {"seed": SEED, "turns": TURNS, "s": s, "steps": T, "c_prime": 4, "rho_prime": RP, "rho": RHO,
       "capacity": C, "init_len": 128, "local_len": 1024, "geometry": [b, h, g, d]}
for dcu in (True, False):
    store, index = ck.prefill(q[:, :, :s].copy(), k[:, :, :s].copy(), v[:, :, :s].copy(),
                              ck.PrefillParams(128, 1024, C, RHO))
    state = ck.DecodeState(store, index, ck.DecodeConfig(4, RP, use_dcu=dcu), oracle=ck.FlatOracle(store))
    rows = []
    for t in range(T):
        store.append(k[:, :, s + t], v[:, :, s + t])
        _, row = ck.decode_step(state, q[:, :, s + t])
        rows.append({"digest": row.sparse_digest, "recall_len": int(row.recall_len),
                     "recall_at_k": float(row.recall_at_k)})
    out["dcu" if dcu else "no_dcu"] = rows
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dcu_turns_seed1.json")
with open(path, "w") as fh:
    json.dump(out, fh)
print("wrote", path)
