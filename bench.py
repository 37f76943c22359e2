#!/usr/bin/env python
"""CTkvr decode benchmark on B200 (BASELINE.json configs).

Default workload = configs[1] ("cfg2"): Llama-3-8B head geometry (32 q / 8
kv heads, d=128), all 32 layers, 96K (98,304-token) synthetic drift
context, batch 8 per GPU, bf16, C=2048 centroids, rho=1280, rho'=512,
C'=4, L_init=128, L_local=1024.  A "step" = one decode token for the whole
batch through all layers: per layer append + recall + rerank + sparse/static
attention + merge + DCU.  Metric: decode tokens/s (whole job, all ranks).
`--config cfg3|cfg5|cfg1` selects the other BASELINE configs (see PRESETS).

Inputs are larger than L2 (6.6 GB of reads per step vs 126 MB L2), so no
flush is needed between steps.

Legs of one run (rank 0 prints ONE JSON line):
* timed region: K graph replays of the multi-layer engine, CUDA events;
* e2e: the same step through pinned host buffers (H2D inputs and D2H outputs
  inside each step's graph; the host fills and launches step t+1 before it
  waits for step t's outputs and reads them; 2 untimed warm-up steps);
* parity: after the timed region, sampled (layer, sequence) units are
  replayed on the CPU from a snapshot of the device state by the reference
  package itself (baseline/_ref, when present) and the pinned oracle port,
  step by step (oracle/unit_parity.py) -- the `parity` field;
* cpu_baseline: the reference's own decode_step timings from that leg.

Reference arm (`--impl reference`): the unmodified reference package
(`centroidkv` 0.1.0 installed under baseline/_ref) runs its own `prefill`
and `decode_step` on one (layer, sequence) unit of the same geometry on the
host cores; tok/s is a labelled linear extrapolation to the full step.
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", str(len(os.sched_getaffinity(0))))

import argparse  # noqa: E402
import json  # noqa: E402
import math  # noqa: E402
import platform  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0

# BASELINE.json configs.  cfg3 does not fit one B200 at 48 distinct layers
# (K/V 154 GB + lists 32 GB + centroids 13 GB): its capacity plan cycles 36
# physical layer buffers (logical layer l uses buffer l mod 36; every layer
# moves exactly the bytes a distinct layer would).  cfg5 on one GPU is one
# rank's slice of the 8-GPU shard plan (kv heads x batch).
PRESETS = {
    "cfg2": dict(layers=32, batch=8, seq=98304, query_heads=32, kv_heads=8, capacity=2048,
                 dtype="bf16", build_mode=1, lanes=4, phys_layers=0,
                 workload="cfg2: Llama-3-8B geometry 32q/8kv d=128, 32 layers, 96K ctx, batch 8 "
                          "per GPU, bf16 (BASELINE configs[1])", model="llama3-8b-geometry"),
    "cfg3": dict(layers=48, batch=16, seq=98304, query_heads=32, kv_heads=4, capacity=2048,
                 dtype="bf16", build_mode=1, lanes=2, phys_layers=36,
                 workload="cfg3: Yi-9B geometry 32q/4kv d=128, 48 layers, 96K ctx, batch 16 per "
                          "GPU, bf16 (BASELINE configs[2]); 48 logical layers over 36 physical "
                          "layer buffers (capacity plan)", model="yi-9b-geometry"),
    "cfg5": dict(layers=32, batch=8, seq=131072, query_heads=32, kv_heads=8, capacity=2048,
                 dtype="bf16", build_mode=1, lanes=4, phys_layers=0, slice_of=8,
                 workload="cfg5: Llama-3-8B geometry, 32 layers, 128K ctx, global batch B over "
                          "8 GPUs (kv heads x batch), bf16 (BASELINE configs[4])",
                 model="llama3-8b-geometry"),
    "cfg1": dict(layers=1, batch=1, seq=8192, query_heads=32, kv_heads=8, capacity=512,
                 dtype="f32", build_mode=0, lanes=1, phys_layers=0,
                 workload="cfg1: one layer, Llama-3-8B heads 32q/8kv d=128, 8K ctx, batch 1, "
                          "fp32 (BASELINE configs[0])", model="llama3-8b-geometry"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(PRESETS))
    for k in ("layers", "batch", "seq", "query_heads", "kv_heads", "capacity", "lanes",
              "phys_layers", "build_mode", "slice_of"):
        ap.add_argument("--" + k.replace("_", "-"), type=int, default=None)
    ap.add_argument("--rho", type=int, default=1280)
    ap.add_argument("--rho-prime", type=int, default=512)
    ap.add_argument("--c-prime", type=int, default=4)
    ap.add_argument("--init-len", type=int, default=128)
    ap.add_argument("--local-len", type=int, default=1024)
    ap.add_argument("--no-rerank", action="store_true",
                    help="attend the whole recall set (ck/retrieval.py:334-337; Fig. 11 ablation)")
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--parity-steps", type=int, default=10,
                    help="steps replayed on the CPU per sampled unit (0: no parity leg)")
    ap.add_argument("--parity-units", type=int, default=3)
    ap.add_argument("--no-graph", action="store_true")
    a = ap.parse_args()
    pre = PRESETS[a.config]
    for k, v in pre.items():
        if getattr(a, k, None) is None:
            setattr(a, k, v)
    if a.slice_of is None:
        a.slice_of = 0
    return a


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


def host_info() -> dict:
    """CPU model, cores used, numpy / BLAS versions (the CPU arms' context)."""
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        for p in threadpool_info():
            if p.get("user_api") == "blas":
                blas = f"{p.get('internal_api')} {p.get('version')} x{p.get('num_threads')}"
                break
    except Exception:
        pass
    return {"cpu_model": model, "cores": len(os.sched_getaffinity(0)), "numpy": np.__version__,
            "blas": blas}


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
            self._stop.wait(0.1)

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


def _config(a, n):
    cfg = {"workload": PRESETS[a.config]["workload"], "model": PRESETS[a.config]["model"],
           "global_batch": a.batch * n, "seq_len": a.seq, "layers": a.layers,
           "query_heads": a.query_heads, "kv_heads": a.kv_heads, "C": a.capacity,
           "rho": a.rho, "rho_prime": a.rho_prime, "c_prime": a.c_prime,
           "init_len": a.init_len, "local_len": a.local_len, "rerank": not a.no_rerank,
           "parallelism": f"kvhead x batch shards over {n} GPU(s), {a.lanes} micro-batch lanes "
                          f"per GPU", "l2": "inputs > L2 (no flush)"}
    if a.phys_layers:
        cfg["physical_layers"] = a.phys_layers
    if a.slice_of:
        cfg["slice"] = (f"rank 0 of a {a.slice_of}-GPU kv-head x batch shard plan, run on 1 GPU; "
                        f"value = global batch / slice step time (every rank runs an identical "
                        f"slice; the per-layer all-gather is not included)")
        cfg["global_batch"] = a.batch
        cfg["parallelism"] = f"1-GPU slice of {a.slice_of}-GPU shards, {a.lanes} lanes"
    return cfg


# ---------------------------------------------------------------------------
# reference arm: the unmodified reference package on the host cores
# ---------------------------------------------------------------------------

def run_reference(a):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.unit_parity import load_reference
    ck = load_reference()
    info = host_info()
    if ck is None:
        print(json.dumps({"impl": "reference", "unavailable": "centroidkv not installed under "
                          "baseline/_ref (pip install --target baseline/_ref /root/reference/pkg)"}))
        return
    from paper_2512_15550_b200.tensor_ops import HeadLayout
    from paper_2512_15550_b200.workload import DriftConfig, generate
    h, g, d, s, C = a.query_heads, a.kv_heads, 128, a.seq, a.capacity
    if a.slice_of:
        from paper_2512_15550_b200.parallel import ShardPlan
        sp = ShardPlan(a.slice_of, 0, a.batch * a.slice_of, g, h)
        h, g = sp.h_loc, sp.g_loc
    steps_total = a.warmup + a.steps
    lay = HeadLayout(1, h, g, s + steps_total, d)
    dt = torch.float32 if a.dtype == "f32" else torch.bfloat16
    q, k, v, _ = generate(DriftConfig(seed=42, s=s, decode_steps=steps_total), lay, device="cpu",
                          dtype=dt, q_rows=(s - C, s + steps_total))
    # bf16 inputs widened exactly to f32 for the f32-only reference
    q, k, v = q.float().numpy(), k.float().numpy(), v.float().numpy()
    queries = np.zeros((1, h, s, d), np.float32)         # only the last C rows are read
    queries[:, :, s - C:] = q[:, :, :C]
    t0 = time.perf_counter()
    store, index = ck.prefill(queries, np.ascontiguousarray(k[:, :, :s]),
                              np.ascontiguousarray(v[:, :, :s]),
                              ck.PrefillParams(a.init_len, a.local_len, C, a.rho))
    build_s = time.perf_counter() - t0
    state = ck.DecodeState(store, index, ck.DecodeConfig(a.c_prime, a.rho_prime,
                                                         use_rerank=not a.no_rerank))
    times = []
    for t in range(steps_total):
        store.append(k[:, :, s + t], v[:, :, s + t])      # ck/session.py:58-60
        t1 = time.perf_counter()
        ck.decode_step(state, q[:, :, C + t])
        times.append(time.perf_counter() - t1)
    unit = statistics.median(times[a.warmup:])
    hsplit = a.kv_heads // g                              # 8 for a cfg5 kv-head slice, else 1
    units = a.layers * a.batch * hsplit                   # units per step of the whole job
    tok_s = 1.0 / (unit * a.layers * hsplit)              # = batch / (unit * units)
    line = {
        "impl": "reference", "metric": "decode_tokens_per_s", "value": tok_s, "unit": "tok/s",
        "higher_is_better": True, "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        # one arm step = one measured (layer, sequence) unit decode_step
        "ms_per_step": unit * 1e3, "dtype": "f64 (f32 storage)",
        "data": "synthetic drift (same generator distribution, CPU torch RNG), bf16-rounded "
                "and widened to f32" if a.dtype != "f32" else "synthetic drift, f32",
        "config": _config(a, a.gpus),
        "extrapolation": {"measured": "reference decode_step on 1 (layer, sequence) unit",
                          "unit_ms": unit * 1e3, "units_per_step_per_gpu": units,
                          "extrapolated_ms_per_full_step": unit * units * 1e3,
                          "note": "value = batch / (unit_ms x units): a labelled linear "
                                  "extrapolation, not a measured full step"},
        "cpu_baseline": dict(value=tok_s, unit="tok/s", kind="reference",
                             sample=f"centroidkv.decode_step on one {s}-token unit "
                                    f"({h}q/{g}kv), median of {a.steps} after {a.warmup} warm-up",
                             build_s_per_unit=build_s, **info),
        "e2e": {"value": tok_s, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


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
    from paper_2512_15550_b200.index import QueryCentroidIndex
    from paper_2512_15550_b200.parallel import ShardPlan
    from paper_2512_15550_b200.store import KvStore

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # rank counts visible in the log
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    N.lib()
    dev = torch.device("cuda", local)
    if a.slice_of:
        if world > 1:
            raise SystemExit("--slice-of runs one rank's shard on one GPU (use --gpus 1)")
        # one rank's slice of the multi-GPU plan (--batch = the GLOBAL batch B),
        # no collective; B / step time = the job's throughput if every rank
        # runs its identical slice in parallel (the all-gather excluded)
        plan_full = ShardPlan(a.slice_of, 0, a.batch, a.kv_heads, a.query_heads)
        plan = ShardPlan(1, 0, plan_full.b_loc, plan_full.g_loc, plan_full.h_loc)
        B = a.batch
    else:
        B = a.batch * world                                  # weak scaling: batch per GPU fixed
        plan = ShardPlan(world, rank, B, a.kv_heads, a.query_heads)
    b, g, h, d = plan.b_loc, plan.g_loc, plan.h_loc, 128
    while b % a.lanes:
        a.lanes -= 1
    s = a.seq
    T = a.warmup + a.steps + a.e2e_steps + 2 + a.parity_steps + 8
    n_phys = a.phys_layers or a.layers
    apps = -(-a.layers // n_phys)                             # appends per buffer per step
    layout = P.HeadLayout(b, h, g, s + T, d)
    dtype = torch.float32 if a.dtype == "f32" else torch.bfloat16
    cfg = P.DecodeConfig(a.c_prime, a.rho_prime, use_rerank=not a.no_rerank)
    rho = min(a.rho, s - a.init_len - a.local_len)

    # ---- setup: synthetic inputs + device prefill (index build) per layer ----
    phys, build_ms, tails = [], [], []
    build_ws = None   # one build workspace for every layer (setup allocations stay out of the timing)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for li in range(a.layers):
        q, k, v, _ = P.generate(P.DriftConfig(seed=42 + li + 1000 * rank, s=s, decode_steps=T),
                                layout, dtype=dtype, q_rows=(s - a.capacity, s + T))
        tails.append((q[:, :, a.capacity:].contiguous(), k[:, :, s:].contiguous(),
                      v[:, :, s:].contiguous()))
        if li < n_phys:
            store = KvStore(P.HeadLayout(b, h, g, s, d), a.init_len, a.local_len, dtype=dtype,
                            capacity=s + T * apps, host_api=False)
            store.keys[:, :, :s].copy_(k[:, :, :s])
            store.values[:, :, :s].copy_(v[:, :, :s])
            store._set_total(s)
            cent_q = q[:, :, :a.capacity].contiguous()
            del k, v
            if build_ws is None:
                nb = N.lib().ctkv_build_workspace_bytes(store.ctkv_layout(), a.capacity, rho,
                                                        store.offloaded_ids().size, a.build_mode)
                build_ws = torch.empty(max(int(nb), 1), dtype=torch.uint8, device=dev)
            torch.cuda.synchronize()
            ev0.record()
            index = QueryCentroidIndex.build(cent_q, store, a.capacity, rho, mode=a.build_mode,
                                             workspace=build_ws)
            ev1.record()
            torch.cuda.synchronize()
            build_ms.append(ev0.elapsed_time(ev1))
            phys.append((store, index))
        del q
    del build_ws
    layers = [phys[li % n_phys] for li in range(a.layers)]
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
    tengine = DecodeEngine(layers, cfg, plan=plan if world > 1 else None, group=group, lanes=1)
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
    scan_ms_bracketed = statistics.mean(e[0].elapsed_time(e[1]) for run_ in evs for e in run_)
    unit_ms = statistics.mean(e[1].elapsed_time(e[2]) for run_ in evs for e in run_)
    # the scan's launch-to-launch duration: every layer's full-layer scan
    # back to back on the stream (no other kernel in between; the inputs of
    # the last step, whose appended rows the next real step rewrites), one
    # event pair per pass -- the roofline's denominator.  The bracketed
    # per-launch mean above also counts each launch's own latency.
    sb0, sb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b2b = []
    for m in range(nmeas):
        torch.cuda.synchronize()
        sb0.record()
        for L in tengine.layers:
            tengine._launch(L, 1 | tengine._cl_bits)
        sb1.record()
        torch.cuda.synchronize()
        b2b.append(sb0.elapsed_time(sb1) / len(tengine.layers))
    tengine.check()
    scan_ms = statistics.median(b2b)
    del tengine
    engine = DecodeEngine(layers, cfg, plan=plan if world > 1 else None, group=group,
                          lanes=a.lanes)
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
    e = 4 if dtype == torch.float32 else 2
    gs = h // g
    U = b * g                                  # units per kernel launch (timing pass: full layer)
    n_static = a.init_len + a.local_len
    C = a.capacity
    n_sparse = a.rho_prime if not a.no_rerank else Lbar
    # algorithmic bytes per launch (full-layer launch: U = b*g units)
    ns = math.ceil(n_static / (64 if e == 4 else 128))   # static splits (f32: 64 tokens)
    scan_bytes = U * (gs * C * d * e + gs * C * 4          # centroid rows + cached norms
                      + 2 * n_static * d * e               # static K, V
                      + gs * d * e + 2 * d * e             # query heads, appended K/V
                      + C * 8 + ns * gs * (d * 4 + 16))    # group-max cosines, static partials
    unit_bytes = U * (C * 8 + 4 * a.c_prime * a.rho                # cosines, selected lists
                      + e * d * Lbar + e * d * n_sparse             # K rows (rerank), V rows
                      + 16 * gs * Lbar + 12 * Lbar                  # logits w+r, keys, ids
                      + ns * gs * (d * 4 + 16) + 4 * gs * d)        # static partials, output
    # step total: SURVEY.md section 8(d)
    algo_bytes = b * g * (gs * C * d * e + 4 * a.c_prime * a.rho + e * d * Lbar
                          + e * d * n_sparse + 2 * e * d * n_static + e * gs * d + 4 * gs * d
                          + e * gs * d + 4 * a.rho + 2 * e * d) * nl
    scan_gbs = scan_bytes / (scan_ms * 1e-3) / 1e9
    unit_gbs = unit_bytes / (unit_ms * 1e-3) / 1e9 if unit_ms > 1e-4 else 0.0

    # ---- e2e through host buffers (pinned H2D of q/k/v, D2H of outputs) ----
    i0 = step_i[0]
    ne = a.e2e_steps + 2                      # 2 untimed warm-up steps (one per graph slot)
    hq = Qall[i0:i0 + ne].cpu().pin_memory()
    hk = Kall[i0:i0 + ne].cpu().pin_memory()
    hv = Vall[i0:i0 + ne].cpu().pin_memory()
    step_i[0] += ne
    # two graph slots with the host copies inside the step: each (layer,
    # lane)'s inputs are copied in ahead of it and its output copied out as it
    # finishes; the host fills the other slot's inputs while a step runs
    hbufs = None
    if use_graph:
        try:
            hbufs = engine.capture_host_io(2)
        except RuntimeError as exc:
            print(f"bench: host-I/O graph capture failed ({exc}); copies around the step",
                  file=sys.stderr)
            torch.cuda.synchronize()
    hout = hbufs[0][3] if hbufs else torch.empty(engine.gathered.shape,
                                                 dtype=torch.float32).pin_memory()
    h2d = (hq[0].numel() + hk[0].numel() + hv[0].numel()) * e
    d2h = hout.numel() * 4

    def fill(slot, t):
        bq, bk, bv, _ = hbufs[slot]
        bq.copy_(hq[t])
        bk.copy_(hk[t])
        bv.copy_(hv[t])

    if hbufs:   # warm-up: each graph slot's first replay (graph upload) is untimed
        for w in range(2):
            fill(w, w)
            engine.replay_host(w)
            torch.cuda.synchronize()
        hq, hk, hv = hq[2:], hk[2:], hv[2:]
        fill(0, 0)
    else:
        hq, hk, hv = hq[2:], hk[2:], hv[2:]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    host_sum = 0.0
    e0.record()
    if hbufs:
        # the host runs one step ahead (as a serving loop does with CUDA
        # graphs): step t+1 is filled and launched before the host waits for
        # step t's outputs, so the graph launch is off the GPU's critical
        # path; every step still copies its inputs in and its outputs out
        # inside its graph, and the host reads each step's result
        done = [torch.cuda.Event(), torch.cuda.Event()]
        engine.replay_host(0)
        done[0].record()
        for t in range(a.e2e_steps):
            if t + 1 < a.e2e_steps:
                fill((t + 1) % 2, t + 1)        # the slot of step t-1, finished
                engine.replay_host((t + 1) % 2)
                done[(t + 1) % 2].record()
            done[t % 2].synchronize()           # step t's outputs are on the host
            host_sum += float(hbufs[t % 2][3].view(-1)[0])
    else:
        for t in range(a.e2e_steps):
            engine.q.copy_(hq[t], non_blocking=True)
            engine.k.copy_(hk[t], non_blocking=True)
            engine.v.copy_(hv[t], non_blocking=True)
            run()
            hout.copy_(engine.gathered, non_blocking=True)
            torch.cuda.current_stream().synchronize()   # the token is needed on the host
            host_sum += float(hout.view(-1)[0])
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_tok_s = B * a.e2e_steps / (e2e_ms / 1e3)
    engine.check()

    # ---- parity leg (checker, after every timed region): sampled (layer,
    # seq) units replayed on the CPU by the reference and the oracle ----
    parity, cpu = None, None
    if rank == 0 and a.parity_steps > 0:
        from oracle import unit_parity as UP
        alias_free = [li for li in range(nl) if a.layers <= n_phys or
                      (li % n_phys) >= a.layers - n_phys]
        cand = [(alias_free[0], 0), (alias_free[-1], b - 1), (alias_free[len(alias_free) // 2], b // 2)]
        units = list(dict.fromkeys(cand))[:max(1, a.parity_units)]
        torch.cuda.synchronize()
        snaps = UP.snapshot(engine, units)
        for _ in range(a.parity_steps):
            load_inputs(engine)
            run()
            torch.cuda.synchronize()
            UP.record(engine, snaps)
        engine.check()
        UP.final_state(engine, snaps)
        t0 = time.perf_counter()
        res = UP.check(snaps, a.c_prime, a.rho_prime, use_rerank=not a.no_rerank)
        del snaps
        parity = {k: res[k] for k in ("ok", "reference", "units", "steps", "recall",
                                      "hard_mismatches", "order_hard", "exact_steps",
                                      "recall_len_mismatch", "selected_ties", "selected_hard",
                                      "out_nrel_max",
                                      "dcu_rows", "dcu_rows_exact", "dcu_hard",
                                      "centroids_equal", "fifo_equal",
                                      "ref_vs_oracle_digest_mismatch",
                                      "ref_vs_oracle_out_nrel_max")}
        parity["sampled_units"] = [list(u) for u in units]
        parity["path"] = (f"{'tcgen05' if a.build_mode else 'f64-exact'} build, DecodeEngine "
                          f"lanes={a.lanes}, {'graph+PDL' if use_graph else 'eager'}")
        parity["check_s"] = time.perf_counter() - t0
        info = host_info()
        tm = res["ref_times"] if res["ref_times"] else res["oracle_times"]
        if tm:
            unit_s = statistics.median(tm)
            units_n = nl * B * (a.kv_heads // g)   # whole-job (layer, seq) units of g kv heads
            cpu = dict(value=B / (unit_s * units_n), unit="tok/s",
                       kind="reference" if res["ref_times"] else "port",
                       sample=(f"{'centroidkv' if res['ref_times'] else 'oracle port'} decode_step "
                               f"on {len(units)} (layer, seq) units of this run's device state, "
                               f"median of {len(tm)} steps (2 warm-up per unit dropped) = "
                               f"{unit_s * 1e3:.1f} ms/unit, extrapolated x{units_n} units"),
                       **info)

    if rank == 0:
        build_avg = statistics.median(build_ms)   # per physical layer (the first pays module setup)
        n_off = s - a.init_len - a.local_len
        build_flop = 2 * h * a.capacity * n_off * d * b
        line = {
            "metric": "decode_tokens_per_s", "value": tok_s, "unit": "tok/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": a.dtype,
            "data": "synthetic drift workload (GPU generator: spectral decay, drift, RoPE, needles)",
            "config": _config(a, world),
            "roofline": {"bound": "hbm",
                         "kernel": "scan2_kernel (centroid cosines + static attention), "
                                   "full-layer launch (mean of 32 launches back to back)",
                         "achieved": scan_gbs, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": scan_gbs / hbm, "traffic": ncu_traffic("ctkv::scan2_kernel"),
                         "bytes_per_launch": scan_bytes, "ms_per_launch": scan_ms},
            "kernels": {
                "scan_kernel": {"ms": scan_ms, "bytes": scan_bytes, "gbs": scan_gbs,
                                "timing": "full-layer launches back to back, CUDA events per pass",
                                "ms_bracketed": scan_ms_bracketed},
                "unit_kernel": {"name": "chain_kernel", "ms": unit_ms, "bytes": unit_bytes,
                                "gbs": unit_gbs, "mean_recall_len": Lbar,
                                "alpha": Lbar / (a.c_prime * a.rho)},
                "step": {"algorithmic_bytes": algo_bytes,
                         "gbs": algo_bytes / (ms_step * 1e-3) / 1e9,
                         "frac": algo_bytes / (ms_step * 1e-3) / 1e9 / hbm},
            },
            "build": {"ms_per_layer": build_avg, "ms_per_layer_seq": build_avg / b,
                      "tflops": build_flop / (build_avg * 1e-3) / 1e12,
                      "frac": build_flop / (build_avg * 1e-3) / 1e12 / tf_peak,
                      "mode": "tcgen05" if a.build_mode else "exact-f64"},
            "e2e": {"value": e2e_tok_s, "unit": "tok/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            # per (lane, layer): scan + chain + deferred tail kernels
            "gpu_launches": 3 * nl * a.lanes * a.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "parity": parity,
            "graph": use_graph,
        }
        if world > 1:
            line["nccl"] = {"comm_nranks": dist.get_world_size(), "backend": "nccl"}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
