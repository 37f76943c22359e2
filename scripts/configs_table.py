"""profiles/r2_configs.jsonl + the table rows of profiles/r2_configs.md from
the bench lines `scripts/r2_configs.sh` leaves in gpurun_out/cov_<tag>.txt.

usage: python scripts/configs_table.py [gpurun_out]   (writes the jsonl,
prints the markdown rows)
"""
import json
import os
import sys

TAGS = ["cfg1", "cfg2_norerank", "cfg3"] + [f"cfg5_b{b}" for b in (1, 2, 4, 8, 16, 32, 64)]
src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lines = []
for tag in TAGS:
    path = os.path.join(src, f"cov_{tag}.txt")
    if not os.path.exists(path):
        continue
    js = [x for x in open(path) if x.startswith("{")]
    if not js:
        print(f"| {tag} | (no bench line) |")
        continue
    d = json.loads(js[-1])
    d["tag"] = tag
    lines.append(d)
    c = d["config"]
    layers = str(c["layers"])
    if c.get("physical_layers"):
        layers += f" ({c['physical_layers']} phys)"
    b = d["build"]
    par = d["parity"]
    print(f"| {tag} | {c['seq_len']} | {c['global_batch']} | {layers} | {c['query_heads']}q/{c['kv_heads']}kv "
          f"| {d['dtype']} | {'yes' if c['rerank'] else 'no'} | {d['value']:.1f} | {d['ms_per_step']:.3f} "
          f"| {d['e2e']['value']:.1f} | {d['roofline']['frac']:.3f} | {d['kernels']['step']['frac']:.3f} "
          f"| {b['ms_per_layer_seq']:.3f} ({b['frac']:.2f}) "
          f"| {par['recall']} / {par['hard_mismatches']} / {par['out_nrel_max']:.1e} "
          f"| {d['cpu_baseline']['value']:.3f} |")
with open(os.path.join(root, "profiles", "r2_configs.jsonl"), "w") as f:
    for d in lines:
        f.write(json.dumps(d) + "\n")
