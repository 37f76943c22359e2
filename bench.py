#!/usr/bin/env python
"""CTkvr decode benchmark on B200 (BASELINE.json configs[1], "cfg2").

Workload: Llama-3-8B head geometry (32 q / 8 kv heads, d=128), all 32
layers, 96K (98,304-token) synthetic drift context, batch 8 per GPU, bf16,
C=2048 centroids, rho=1280, rho'=512, C'=4, L_init=128, L_local=1024.
A "step" = one decode token for the whole batch through all 32 layers:
per layer append + recall + rerank + sparse/static attention + merge + DCU.
Metric: decode tokens/s = tokens produced / step time (whole job, all ranks).

Inputs are larger than L2 (6.6 GB of reads per step vs 126 MB L2), so no
flush is needed between steps.  Reference arm (`--impl reference`): the
reference algorithm's CPU implementation (the pinned numpy port under
oracle/; the reference is pure Python and cannot travel to the GPU box)
timed on the host's cores for one (layer, sequence) unit of the same
geometry and extrapolated to the full step.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--batch", type=int, default=8, help="sequences per GPU")
    ap.add_argument("--seq", type=int, default=98304)
    ap.add_argument("--query-heads", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--head-dim", type=int, default=128)
    ap.add_argument("--capacity", type=int, default=2048)
    ap.add_argument("--rho", type=int, default=1280)
    ap.add_argument("--rho-prime", type=int, default=512)
    ap.add_argument("--c-prime", type=int, default=4)
    ap.add_argument("--init-len", type=int, default=128)
    ap.add_argument("--local-len", type=int, default=1024)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-steps", type=int, default=6)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--build-mode", type=int, default=1, help="0 exact f64, 1 fast")
    ap.add_argument("--lanes", type=int, default=4,
                    help="micro-batch lanes per GPU (sequence groups on their own streams)")
    return ap.parse_args()


def ncu_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu summary
    (profiles/ncu_traffic.json, written by scripts/ncu_traffic.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            db = json.load(fh)
        for key in (kernel, kernel.split("::")[-1]):
            if key in db:
                return db[key]["dram_bytes_per_launch"]
    except Exception:
        pass
    return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), float(pk.get("bf16_tflops_sustained", 1407.1)), "measured"
    except Exception:
        return HBM_FALLBACK, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU reference (the pinned oracle port), one (layer, sequence) unit
# ---------------------------------------------------------------------------

def cpu_unit_decode(keys, values, cent, lists, dec_q, dec_k, dec_v, a, steps, warm=1):
    """Time the reference algorithm's decode_step (oracle port, f64 numpy)
    on one (layer, sequence) unit; returns per-step seconds (median)."""
    from oracle import ctkv_oracle as O
    s = keys.shape[2]
    store = O.partition(keys, values, a.init_len, a.local_len, cent.shape[1])
    index = O.Index(cent.copy(), lists.copy(), np.zeros(1, dtype=np.int64))
    times = []
    for t in range(warm + steps):
        store.append(dec_k[:, :, t], dec_v[:, :, t])
        t0 = time.perf_counter()
        O.decode_step(store, index, dec_q[:, :, t], a.c_prime, a.rho_prime)
        times.append(time.perf_counter() - t0)
    del s
    return statistics.median(times[warm:]), times


def run_reference(a):
    """--impl reference: the reference's CPU path on the host cores."""
    import torch
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ctkv_oracle as O
    from paper_2512_15550_b200.workload import DriftConfig, generate
    from paper_2512_15550_b200.tensor_ops import HeadLayout
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(cores))
    s, T = a.seq, a.warmup + a.steps + 1
    lay = HeadLayout(1, a.query_heads, a.kv_heads, s + T, a.head_dim)
    q, k, v, _ = generate(DriftConfig(seed=42, s=s, decode_steps=T), lay, device="cpu",
                          dtype=torch.float32, q_rows=(s - a.capacity, s + T))
    q, k, v = q.numpy(), k.numpy(), v.numpy()
    # bf16 inputs, widened to f32 for the f32-only reference
    q, k, v = O.bf16_round(q), O.bf16_round(k), O.bf16_round(v)
    t0 = time.perf_counter()
    store, index = O.prefill(np.concatenate([np.zeros((1, a.query_heads, s - a.capacity, a.head_dim),
                                                      np.float32), q[:, :, :a.capacity]], axis=2),
                             np.ascontiguousarray(k[:, :, :s]), np.ascontiguousarray(v[:, :, :s]),
                             a.init_len, a.local_len, a.capacity, a.rho)
    build_s = time.perf_counter() - t0
    times = []
    for t in range(a.warmup + a.steps):
        store.append(k[:, :, s + t], v[:, :, s + t])
        t1 = time.perf_counter()
        O.decode_step(store, index, q[:, :, a.capacity + t], a.c_prime, a.rho_prime)
        times.append(time.perf_counter() - t1)
    unit = statistics.median(times[a.warmup:])
    units_per_step = a.layers * a.batch * a.gpus
    tok_s = (a.batch * a.gpus) / (unit * units_per_step)
    line = {
        "impl": "reference", "metric": "decode_tokens_per_s", "value": tok_s, "unit": "tok/s",
        "higher_is_better": True, "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": unit * units_per_step * 1e3, "dtype": "f64",
        "data": "synthetic drift (GPU-generator distribution, CPU torch RNG), bf16-rounded",
        "config": _config(a, a.gpus),
        "cpu_baseline": {"value": tok_s, "unit": "tok/s", "cores": cores, "kind": "port",
                         "sample": f"oracle decode_step on 1 of {units_per_step} (layer, seq) units "
                                   f"per step at 96K, median of {a.steps}, linear extrapolation",
                         "build_s_per_unit": build_s},
        "e2e": {"value": tok_s, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def _config(a, n):
    return {"workload": "cfg2: Llama-3-8B geometry 32q/8kv d=128, 32 layers, 96K ctx, "
                        "batch 8 per GPU, bf16 (BASELINE configs[1])",
            "model": "llama3-8b-geometry", "global_batch": a.batch * n, "seq_len": a.seq,
            "layers": a.layers, "C": a.capacity, "rho": a.rho, "rho_prime": a.rho_prime,
            "c_prime": a.c_prime, "init_len": a.init_len, "local_len": a.local_len,
            "parallelism": f"kvhead x batch shards over {n} GPU(s), {a.lanes} micro-batch lanes per GPU", "l2": "inputs > L2 (no flush)"}


# ---------------------------------------------------------------------------
# ours
# ---------------------------------------------------------------------------

def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist

    import paper_2512_15550_b200 as P
    from paper_2512_15550_b200 import _native as N
    from paper_2512_15550_b200.engine import DecodeEngine
    from paper_2512_15550_b200.parallel import ShardPlan
    from paper_2512_15550_b200.store import KvStore
    from paper_2512_15550_b200.index import QueryCentroidIndex

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    N.lib()
    dev = torch.device("cuda", local)
    B = a.batch * world                       # weak scaling: 8 sequences per GPU
    plan = ShardPlan(world, rank, B, a.kv_heads, a.query_heads)
    b, g, h, d = plan.b_loc, plan.g_loc, plan.h_loc, a.head_dim
    s = a.seq
    T = a.warmup + a.steps + a.e2e_steps + 12 + a.cpu_steps + 2
    layout = P.HeadLayout(b, h, g, s + T, d)
    cfg = P.DecodeConfig(a.c_prime, a.rho_prime)

    # ---- setup: synthetic inputs + device prefill (index build) per layer ----
    layers, tails = [], []
    build_ms = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for li in range(a.layers):
        q, k, v, _ = P.generate(P.DriftConfig(seed=42 + li + 1000 * rank, s=s, decode_steps=T),
                                layout, dtype=torch.bfloat16, q_rows=(s - a.capacity, s + T))
        store = KvStore(P.HeadLayout(b, h, g, s, d), a.init_len, a.local_len, dtype=torch.bfloat16,
                        capacity=s + T, host_api=False)
        store.keys[:, :, :s].copy_(k[:, :, :s])
        store.values[:, :, :s].copy_(v[:, :, :s])
        store._set_total(s)
        tails.append((q[:, :, a.capacity:].contiguous(), k[:, :, s:].contiguous(),
                      v[:, :, s:].contiguous()))
        cent_q = q[:, :, :a.capacity].contiguous()
        del k, v
        torch.cuda.synchronize()
        ev0.record()
        index = QueryCentroidIndex.build(cent_q, store, a.capacity, min(a.rho, s - a.init_len - a.local_len),
                                         mode=a.build_mode)
        ev1.record()
        torch.cuda.synchronize()
        build_ms.append(ev0.elapsed_time(ev1))
        layers.append((store, index))
        del q
    nl = a.layers
    # all step inputs, device resident: [T, L, b, heads, d]
    Qall = torch.stack([t[0].permute(2, 0, 1, 3) for t in tails], dim=1).contiguous()
    Kall = torch.stack([t[1].permute(2, 0, 1, 3) for t in tails], dim=1).contiguous()
    Vall = torch.stack([t[2].permute(2, 0, 1, 3) for t in tails], dim=1).contiguous()
    del tails
    step_i = [0]

    def load_inputs(eng):
        t = step_i[0]
        eng.q.copy_(Qall[t])
        eng.k.copy_(Kall[t])
        eng.v.copy_(Vall[t])
        step_i[0] += 1

    # ---- per-kernel timing at full-layer size (one launch per kernel covers
    # all b*g units of a layer), eager, CUDA events on the launching stream;
    # run before the lanes engine, which then continues from this state ----
    nmeas = 3
    tengine = DecodeEngine(layers, cfg, plan=plan, group=group, lanes=1)
    load_inputs(tengine)
    tengine.step()
    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(nl)]
           for _ in range(nmeas)]
    rl_tot = 0
    for m in range(nmeas):
        load_inputs(tengine)
        tengine.step(events=evs[m])
        torch.cuda.synchronize()
        rl_tot += sum(int(L.bufs.recall_len.sum()) for L in tengine.layers)
    tengine.check()
    scan_ms = statistics.mean(e[0].elapsed_time(e[1]) for run_ in evs for e in run_)
    unit_ms = statistics.mean(e[1].elapsed_time(e[2]) for run_ in evs for e in run_)
    del tengine
    engine = DecodeEngine(layers, cfg, plan=plan, group=group, lanes=a.lanes)
    # ---- warm-up (eager), capture, more warm-up ----
    for _ in range(max(1, a.warmup // 2)):
        load_inputs(engine)
        engine.step()
    torch.cuda.synchronize()
    engine.check()
    use_graph = not a.no_graph
    if use_graph:
        try:
            engine.capture()
        except RuntimeError as exc:   # e.g. a collective that cannot be captured on this stack
            print(f"bench: graph capture failed ({exc}); eager steps", file=sys.stderr)
            torch.cuda.synchronize()
            use_graph = False
    run = engine.replay if use_graph else engine.step
    for _ in range(a.warmup - max(1, a.warmup // 2)):
        load_inputs(engine)
        run()
    torch.cuda.synchronize()

    # ---- timed region ----
    hbm, tf_peak, peak_kind = peaks()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        start.record()
        for _ in range(a.steps):
            load_inputs(engine)
            run()
        stop.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_total = start.elapsed_time(stop)
    if world > 1:
        t = torch.tensor([ms_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    engine.check()
    ms_step = ms_total / a.steps
    tok_s = B * a.steps / (ms_total / 1e3)

    Lbar = rl_tot / (nmeas * nl * b * g)      # mean recall length per (b, g) unit
    e = 2
    gs = h // g
    U = b * g                                  # units per kernel launch (timing pass: full layer)
    n_static = a.init_len + a.local_len
    C = a.capacity
    # algorithmic bytes per launch (full-layer launch: U = b*g units)
    ns = math.ceil(n_static / 128)                # static splits (bf16: 128 tokens)
    scan_bytes = U * (gs * C * d * e + gs * C * 4          # centroid rows + cached norms
                      + 2 * n_static * d * e               # static K, V
                      + gs * d * e + 2 * d * e             # query heads, appended K/V
                      + C * 8 + ns * gs * (d * 4 + 16))    # group-max cosines, static partials
    unit_bytes = U * (C * 8 + 4 * a.c_prime * a.rho                # cosines, selected lists
                      + e * d * Lbar + e * d * a.rho_prime          # K rows (rerank), V rows
                      + 16 * gs * Lbar + 12 * Lbar                  # logits w+r, keys, ids
                      + ns * gs * (d * 4 + 16) + 4 * gs * d)        # static partials, output
    # step total: SURVEY.md section 8(d)
    algo_bytes = b * g * (h // g * C * d * e + 4 * a.c_prime * a.rho + e * d * Lbar
                          + e * d * a.rho_prime + 2 * e * d * n_static + e * gs * d + 4 * gs * d
                          + e * gs * d + 4 * a.rho + 2 * e * d) * nl
    scan_gbs = scan_bytes / (scan_ms * 1e-3) / 1e9
    unit_gbs = unit_bytes / (unit_ms * 1e-3) / 1e9 if unit_ms > 1e-4 else 0.0

    # ---- e2e through host buffers (pinned H2D of q/k/v, D2H of outputs) ----
    hq = Qall[:a.e2e_steps + 1].cpu().pin_memory()
    hk = Kall[:a.e2e_steps + 1].cpu().pin_memory()
    hv = Vall[:a.e2e_steps + 1].cpu().pin_memory()
    # two graph slots with the host copies inside the step: each (layer,
    # lane)'s inputs are copied in ahead of it and its output copied out as it
    # finishes; the host fills the other slot's inputs while a step runs
    hbufs = None
    if use_graph:
        try:
            hbufs = engine.capture_host_io(2)
        except RuntimeError as exc:
            print(f"bench: host-I/O graph capture failed ({exc}); copies around the step", file=sys.stderr)
            torch.cuda.synchronize()
    hout = hbufs[0][3] if hbufs else torch.empty(engine.gathered.shape, dtype=torch.float32).pin_memory()
    h2d = (hq[0].numel() + hk[0].numel() + hv[0].numel()) * 2
    d2h = hout.numel() * 4

    def fill(slot, t):
        bq, bk, bv, _ = hbufs[slot]
        bq.copy_(hq[t])
        bk.copy_(hk[t])
        bv.copy_(hv[t])

    if hbufs:
        fill(0, 0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    for t in range(a.e2e_steps):
        if hbufs:
            engine.replay_host(t % 2)
            if t + 1 < a.e2e_steps:
                fill((t + 1) % 2, t + 1)
        else:
            engine.q.copy_(hq[t], non_blocking=True)
            engine.k.copy_(hk[t], non_blocking=True)
            engine.v.copy_(hv[t], non_blocking=True)
            run()
            hout.copy_(engine.gathered, non_blocking=True)
        torch.cuda.current_stream().synchronize()   # the token is needed on the host
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_tok_s = B * a.e2e_steps / (e2e_ms / 1e3)
    engine.check()

    # ---- CPU baseline: oracle decode on one unit of the same state ----
    cpu = None
    if rank == 0 and not a.no_cpu:
        st0, ix0 = layers[0]
        tot = st0.total_tokens
        kk = st0.keys[:1, :, :tot].float().cpu().numpy()
        vv = st0.values[:1, :, :tot].float().cpu().numpy()
        cent = ix0.cent[:1].float().cpu().numpy()
        lists = ix0.lists_dev[:1].cpu().numpy()
        i0 = step_i[0]
        dq = Qall[i0:i0 + a.cpu_steps + 1, 0, :1].permute(1, 2, 0, 3).float().cpu().numpy()
        dk = Kall[i0:i0 + a.cpu_steps + 1, 0, :1].permute(1, 2, 0, 3).float().cpu().numpy()
        dv = Vall[i0:i0 + a.cpu_steps + 1, 0, :1].permute(1, 2, 0, 3).float().cpu().numpy()
        cores = len(os.sched_getaffinity(0))

        class A2:
            pass
        a2 = A2()
        a2.init_len, a2.local_len, a2.c_prime, a2.rho_prime = a.init_len, a.local_len, a.c_prime, a.rho_prime
        unit_s, _ = cpu_unit_decode(kk, vv, cent, lists, dq, dk, dv, a2, a.cpu_steps)
        units = nl * B
        cpu = {"value": B / (unit_s * units), "unit": "tok/s", "cores": cores, "kind": "port",
               "sample": f"oracle (numpy f64 port of the reference) decode_step on 1 of {units} "
                         f"(layer, seq) units, index state copied from the device build, median of "
                         f"{a.cpu_steps} steps = {unit_s * 1e3:.1f} ms/unit, extrapolated x{units}"}

    if rank == 0:
        build_avg = statistics.mean(build_ms)
        build_flop = 2 * a.query_heads // world * a.capacity * (s - a.init_len - a.local_len) * d * b
        line = {
            "metric": "decode_tokens_per_s", "value": tok_s, "unit": "tok/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic drift workload (GPU generator: spectral decay, drift, RoPE, needles)",
            "config": _config(a, world),
            "roofline": {"bound": "hbm",
                         "kernel": "scan2_kernel (centroid cosines + static attention), "
                                   "full-layer launch",
                         "achieved": scan_gbs, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": scan_gbs / hbm, "traffic": ncu_traffic("ctkv::scan2_kernel"),
                         "bytes_per_launch": scan_bytes, "ms_per_launch": scan_ms},
            "kernels": {
                "scan_kernel": {"ms": scan_ms, "bytes": scan_bytes, "gbs": scan_gbs},
                "unit_kernel": {"name": "chain_kernel", "ms": unit_ms, "bytes": unit_bytes,
                                "gbs": unit_gbs, "mean_recall_len": Lbar,
                                "alpha": Lbar / (a.c_prime * a.rho)},
                "step": {"algorithmic_bytes": algo_bytes,
                         "gbs": algo_bytes / (ms_step * 1e-3) / 1e9,
                         "frac": algo_bytes / (ms_step * 1e-3) / 1e9 / hbm},
            },
            "build": {"ms_per_layer": build_avg, "ms_per_layer_seq": build_avg / b,
                      "tflops": build_flop / (build_avg * 1e-3) / 1e12,
                      "mode": "fast" if a.build_mode else "exact-f64"},
            "e2e": {"value": e2e_tok_s, "unit": "tok/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            # per (lane, layer): scan + chain + deferred tail kernels
            "gpu_launches": 3 * nl * a.lanes * a.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "graph": use_graph,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
