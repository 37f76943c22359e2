"""Recall (union) length per (b, kv-head) unit at cfg2 for one decode query:
the L that sizes the chain's rerank gather."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2512_15550_b200 as P
from paper_2512_15550_b200.index import QueryCentroidIndex
from paper_2512_15550_b200.store import KvStore
b, h, g, d, s, C, T = 8, 32, 8, 128, 98304, 2048, 4
lay = P.HeadLayout(b, h, g, s + T, d)
q, k, v, _ = P.generate(P.DriftConfig(seed=42, s=s, decode_steps=T), lay, dtype=torch.bfloat16, q_rows=(s - C, s + T))
st = KvStore(P.HeadLayout(b, h, g, s, d), 128, 1024, dtype=torch.bfloat16, capacity=s + T, host_api=False)
st.keys[:, :, :s].copy_(k[:, :, :s]); st.values[:, :, :s].copy_(v[:, :, :s]); st._set_total(s)
ix = QueryCentroidIndex.build(q[:, :, :C].contiguous(), st, C, 1280)
r = P.recall(ix, q[:, :, C], 4)
print("recall len: mean %.0f min %d max %d" % (r.recall_len.mean(), r.recall_len.min(), r.recall_len.max()))
