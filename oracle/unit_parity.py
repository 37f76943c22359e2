"""Parity at the benchmarked configuration -- TEST INFRASTRUCTURE ONLY.

Checks a running `DecodeEngine` (the bench's own path: tcgen05-built index,
micro-batch lanes, CUDA-graph replay with programmatic dependent launch and
deferred DCU tails) against the CPU ground truth on sampled (layer,
sequence) units, step by step, from a snapshot of the device state:

1. `snapshot(engine, units)` copies, per sampled unit, the layer's K/V rows
   [0, total), centroids, lists and FIFO cursor of that sequence to host f32
   (bf16 values widened exactly);
2. after every engine step, `record(engine, units)` copies that step's
   inputs (q, k_new, v_new) and the engine's outputs for the unit (merged
   output, selected slots, recall lengths, ordered sparse ids);
3. `check(...)` replays the same steps on the CPU with the pinned oracle
   port (oracle/ctkv_oracle.py, which exposes the intermediate sets and f64
   scores) and -- when the real reference package is importable
   (`baseline/_ref/centroidkv`, or /root/reference in the build container)
   -- with the reference's own `decode_step` (ck/retrieval.py:304-378),
   asserting reference == oracle on digests and outputs first.

Comparator (north_star): sparse sets equal except for
swaps whose reference f64 scores lie within 1e-6 relative of the k-th
score; ranks compared the same way; outputs norm-relative; post-DCU lists
per written slot (same tie rule against the step's grouped scores),
centroid rows and FIFO cursors exact.

Nothing in the product package imports this module.
"""

from __future__ import annotations

import os
import sys

import numpy as np

from . import ctkv_oracle as O

TIE_REL = 1e-6
_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_reference():
    """The reference package `centroidkv` 0.1.0, or None.  Search order:
    the gpurun-travelling install under baseline/_ref, then the read-only
    source tree of the build container."""
    for p in (os.path.join(_ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "centroidkv")):
            if p not in sys.path:
                sys.path.insert(0, p)
            try:
                import centroidkv  # noqa: F401
                return centroidkv
            except Exception:
                return None
    return None


def _lane(engine, li, bi):
    k, r = divmod(bi, engine.bl)
    return engine.lane_layers[k][li], r


def snapshot(engine, units):
    """Host copies of the sampled units' device state (call with the
    device idle, i.e. after torch.cuda.synchronize())."""
    snaps = []
    for li, bi in units:
        L, r = _lane(engine, li, bi)
        st, ix = L.store, L.index
        tot = st.total_tokens
        snaps.append(dict(
            layer=li, seq=bi, total=tot, init_len=st.init_len, local_len=st.local_len,
            keys=st.keys[r:r + 1, :, :tot].float().cpu().numpy(),
            values=st.values[r:r + 1, :, :tot].float().cpu().numpy(),
            cent=ix.cent[r:r + 1].float().cpu().numpy(),
            lists=ix.lists_dev[r:r + 1].cpu().numpy(),
            fifo=ix.fifo_dev[r:r + 1].cpu().numpy(),
            steps=[]))
    return snaps


def record(engine, snaps) -> None:
    """Append the last engine step's inputs and outputs for every sampled
    unit (device idle)."""
    for sn in snaps:
        li, bi = sn["layer"], sn["seq"]
        L, r = _lane(engine, li, bi)
        bf = L.bufs
        sl = bf.sparse_len[r].cpu().numpy()
        sp = bf.sparse_ids[r].cpu().numpy()
        sn["steps"].append(dict(
            q=engine.q[li, bi:bi + 1].float().cpu().numpy(),
            k=engine.k[li, bi:bi + 1].float().cpu().numpy(),
            v=engine.v[li, bi:bi + 1].float().cpu().numpy(),
            out=engine.out[li, bi].cpu().numpy(),
            selected=bf.selected[r].cpu().numpy().astype(np.int64),
            recall_len=bf.recall_len[r].cpu().numpy().astype(np.int64),
            sparse=[sp[gi, :sl[gi]].astype(np.int64) for gi in range(sp.shape[0])]))


def final_state(engine, snaps) -> None:
    for sn in snaps:
        L, r = _lane(engine, sn["layer"], sn["seq"])
        ix = L.index
        sn["cent_final"] = ix.cent[r:r + 1].float().cpu().numpy()
        sn["lists_final"] = ix.lists_dev[r:r + 1].cpu().numpy()
        sn["fifo_final"] = ix.fifo_dev[r:r + 1].cpu().numpy()


def _nrel(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _set_hard(mine, ref, score, k) -> bool:
    """True when the sets differ beyond the tie window around the k-th score."""
    if set(mine) == set(ref):
        return False
    kth = sorted(score.values(), reverse=True)[k - 1]
    return any(abs(score.get(i, -np.inf) - kth) > TIE_REL * abs(kth) for i in set(mine) ^ set(ref))


def _order_hard(mine, ref, score) -> int:
    return sum(abs(score.get(a, -np.inf) - score[b]) > TIE_REL * abs(score[b])
               for a, b in zip(mine, ref) if a != b)


def check(snaps, c_prime: int, rho_prime: int, *, use_rerank: bool = True,
          use_reference: bool = True, timing_warmup: int = 2) -> dict:
    """Replay the recorded steps on the CPU and compare (see module doc).
    Also returns the per-step CPU times of the reference's decode_step
    (`ref_times`) and of the oracle port (`oracle_times`), the first
    `timing_warmup` steps of every unit dropped."""
    import time
    ref_pkg = load_reference() if use_reference else None
    res = dict(units=len(snaps), steps=0, sparse_hits=0, sparse_total=0, hard_mismatches=0,
               order_hard=0, exact_steps=0, recall_len_mismatch=0, selected_mismatch=0,
               out_nrel_max=0.0, dcu_rows=0, dcu_rows_exact=0, dcu_hard=0,
               centroids_equal=True, fifo_equal=True, reference=None,
               ref_vs_oracle_digest_mismatch=0, ref_vs_oracle_out_nrel_max=0.0,
               selected_ties=0, selected_hard=0, ref_times=[], oracle_times=[])
    if ref_pkg is not None:
        res["reference"] = f"centroidkv {getattr(ref_pkg, '__version__', '?')} (real package)"
    for sn in snaps:
        g = sn["keys"].shape[1]
        h = sn["cent"].shape[1]
        ost = O.partition(sn["keys"], sn["values"], sn["init_len"], sn["local_len"], h)
        oix = O.Index(sn["cent"].copy(), sn["lists"].copy(), sn["fifo"].copy())
        rst = rix = rstate = None
        if ref_pkg is not None:
            rst = ref_pkg.KvStore.partition(sn["keys"], sn["values"], sn["init_len"],
                                            sn["local_len"], query_heads=h)
            rix = ref_pkg.QueryCentroidIndex(rst.layout, sn["cent"].shape[2], sn["lists"].shape[3],
                                             sn["cent"].copy(), sn["lists"].copy(),
                                             sn["fifo"].copy())
            rstate = ref_pkg.DecodeState(rst, rix, ref_pkg.DecodeConfig(
                c_prime, rho_prime, use_rerank=use_rerank, keep_sets=True))
        written = []
        fin = sn["lists_final"][0]          # the device's post-DCU lists (no slot is
        for si, st in enumerate(sn["steps"]):   # rewritten within a run: steps < C)
            slot = int(oix.fifo_head[0] % oix.capacity)
            pre = (oix.centroids.copy(), oix.lists.copy(), oix.fifo_head.copy())
            ost.append(st["k"], st["v"])
            t0 = time.perf_counter()
            r = O.decode_step(ost, oix, st["q"], c_prime, rho_prime, use_rerank=use_rerank)
            if si >= timing_warmup:
                res["oracle_times"].append(time.perf_counter() - t0)
            # top-C' slots: a difference inside the tie window of the f64
            # group-max cosines is counted once and the device's slots are
            # injected (the oracle step is redone with them)
            forced = None
            for gi in range(g):
                mine, ref = st["selected"][gi], r.selected[0, gi]
                if np.array_equal(mine, ref):
                    continue
                cosg = r.cosines[0, gi]
                kth = cosg[ref[-1]]
                tie = all(abs(cosg[c] - kth) <= TIE_REL * abs(kth)
                          for c in set(mine.tolist()) ^ set(ref.tolist()))
                tie &= all(abs(cosg[a] - cosg[b_]) <= TIE_REL * abs(cosg[b_])
                           for a, b_ in zip(mine.tolist(), ref.tolist()) if a != b_)
                res["selected_ties" if tie else "selected_hard"] += 1
                forced = forced or [[None] * g]
                forced[0][gi] = mine
            if forced is not None:
                ost.total -= 1                      # redo the step from the pre-step state
                oix.centroids, oix.lists, oix.fifo_head = pre
                ost.append(st["k"], st["v"])
                r = O.decode_step(ost, oix, st["q"], c_prime, rho_prime, use_rerank=use_rerank,
                                  force_selected=forced)
            if rst is not None:
                rst.append(st["k"], st["v"])       # ck/session.py:58-60
                t0 = time.perf_counter()
                rout, rrow = ref_pkg.decode_step(rstate, st["q"])
                if si >= timing_warmup:
                    res["ref_times"].append(time.perf_counter() - t0)
                if forced is None:
                    res["ref_vs_oracle_digest_mismatch"] += int(rrow.sparse_digest != r.digest)
                    res["ref_vs_oracle_out_nrel_max"] = max(res["ref_vs_oracle_out_nrel_max"],
                                                            _nrel(rout, r.out))
                else:                               # keep the reference on the injected path
                    rix.lists[0, :, slot] = oix.lists[0, :, slot]
            res["steps"] += 1
            res["out_nrel_max"] = max(res["out_nrel_max"], _nrel(st["out"], r.out[0]))
            rlen = np.array([len(x) for x in r.recalled[0]], np.int64)
            res["recall_len_mismatch"] += int((st["recall_len"] != rlen).sum())
            res["selected_mismatch"] += int((st["selected"] != r.selected[0]).sum())
            exact = True
            for gi in range(g):
                mine, ref = st["sparse"][gi].tolist(), r.sparse[0][gi].tolist()
                ids = np.asarray(r.recalled[0][gi])
                score = dict(zip(ids.tolist(), np.asarray(r.grouped[0][gi]).tolist()))
                res["sparse_hits"] += len(set(mine) & set(ref))
                res["sparse_total"] += len(ref)
                if len(mine) != len(ref):
                    res["hard_mismatches"] += 1
                    exact = False
                    continue
                exact &= mine == ref
                res["hard_mismatches"] += int(_set_hard(mine, ref, score, len(ref)))
                res["order_hard"] += _order_hard(mine, ref, score)
            res["exact_steps"] += int(exact)
            if r.recall_len == 0:
                continue
            # the DCU row this step wrote (ck/index.py:103-133), judged by the
            # step's own f64 scores; a tie-window difference is counted once
            # and the device's row is injected into the CPU state (the oracle's
            # and the reference's) so later steps compare from equal state
            written.append(slot)
            for gi in range(g):
                mine, ref = fin[gi, slot], oix.lists[0, gi, slot]
                res["dcu_rows"] += 1
                if np.array_equal(mine, ref):
                    res["dcu_rows_exact"] += 1
                    continue
                ids = np.asarray(r.recalled[0][gi])
                score = dict(zip(ids.tolist(), np.asarray(r.grouped[0][gi]).tolist()))
                m, rf = [i for i in mine.tolist() if i >= 0], [i for i in ref.tolist() if i >= 0]
                res["dcu_hard"] += int(len(m) != len(rf) or _set_hard(m, rf, score, len(rf)))
                oix.lists[0, gi, slot] = mine
                if rix is not None:
                    rix.lists[0, gi, slot] = mine
        others = np.ones(fin.shape[1], bool)
        others[written] = False
        res["dcu_hard"] += int(not np.array_equal(fin[:, others], oix.lists[0][:, others]))
        res["centroids_equal"] &= bool(np.array_equal(sn["cent_final"], oix.centroids))
        res["fifo_equal"] &= bool(np.array_equal(sn["fifo_final"], oix.fifo_head))
    res["recall"] = res["sparse_hits"] / max(res["sparse_total"], 1)
    res["ok"] = bool(res["hard_mismatches"] == 0 and res["order_hard"] == 0
                     and res["selected_hard"] == 0
                     and res["recall_len_mismatch"] == 0 and res["dcu_hard"] == 0
                     and res["centroids_equal"] and res["fifo_equal"]
                     and res["ref_vs_oracle_digest_mismatch"] == 0)
    return res
