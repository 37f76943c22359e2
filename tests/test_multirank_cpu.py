"""Multi-rank (batch x kv-head) sharding on CPU with the gloo backend.

Each rank decodes its shard of (b, kv head) units -- here with the oracle,
since the CUDA kernels need a GPU; they are per-unit identical -- and the
outputs are reassembled per step with the same `all_gather_outputs` the
B200 engine uses (NCCL there).  The sharded result must equal the
unsharded run, including the replicated per-batch FIFO cursor."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ctkv_oracle as O
from paper_2512_15550_b200.parallel import ShardPlan, all_gather_outputs, gather_lane_outputs

B, H, G, D, S, T = 4, 8, 4, 32, 384, 5
PARAMS = dict(init_len=8, local_len=40, capacity=24, rho=48)
CP, RP = 3, 16


def _data():
    return O.generate(O.Drift(seed=21, s=S, decode_steps=T), B, H, G, D)


def _decode(q, k, v):
    store, index = O.prefill(np.ascontiguousarray(q[:, :, :S]), np.ascontiguousarray(k[:, :, :S]),
                             np.ascontiguousarray(v[:, :, :S]), **PARAMS)
    outs, recs = O.run_decode(store, index, q[:, :, S:], k[:, :, S:], v[:, :, S:], CP, RP)
    return outs, index


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = ShardPlan(world, rank, B, G, H)
        qq, kk, vv = _data()
        b0, b1 = plan.batch_range()
        g0, g1 = plan.kv_range()
        h0, h1 = plan.q_range()
        outs, index = _decode(np.ascontiguousarray(qq[b0:b1, h0:h1]), np.ascontiguousarray(kk[b0:b1, g0:g1]),
                              np.ascontiguousarray(vv[b0:b1, g0:g1]))
        full = []
        for t in range(T):
            local = torch.from_numpy(np.ascontiguousarray(outs[:, :, t]))
            full.append(all_gather_outputs(plan, local).numpy())
        fifo = torch.from_numpy(index.fifo_head.copy())
        if rank == 0:
            q.put((np.stack(full), fifo.numpy(), plan.b_loc, plan.g_loc))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_decode_equals_unsharded(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, fifo, b_loc, g_loc = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    qq, kk, vv = _data()
    ref, index = _decode(qq, kk, vv)
    assert b_loc * g_loc * world == B * G
    for t in range(T):
        np.testing.assert_array_equal(got[t], ref[:, :, t])
    np.testing.assert_array_equal(fifo, index.fifo_head[:b_loc])


def test_shard_plan_covers_units_once():
    for world, g in [(1, 8), (2, 8), (4, 8), (8, 8), (8, 4), (2, 4), (4, 4)]:
        bsz = 16
        seen = set()
        for r in range(world):
            p = ShardPlan(world, r, bsz, g, 4 * g)
            b0, b1 = p.batch_range()
            g0, g1 = p.kv_range()
            for bi in range(b0, b1):
                for gi in range(g0, g1):
                    assert (bi, gi) not in seen
                    seen.add((bi, gi))
            h0, h1 = p.q_range()
            assert (h1 - h0) == p.h_loc and h0 == g0 * 4
        assert len(seen) == bsz * g


def test_assemble_inverts_gather_layout():
    plan = ShardPlan(4, 0, 4, 8, 32)
    parts = []
    full = torch.randn(4, 32, 16)
    for r in range(4):
        b0, b1 = plan.batch_range(r)
        h0, h1 = plan.q_range(r)
        parts.append(full[b0:b1, h0:h1])
    assert torch.equal(plan.assemble(torch.stack(parts)), full)


def _lane_worker(rank, world, port, q, lanes):
    """The engine's collective path (DecodeEngine._gather ->
    gather_lane_outputs) with gloo: per layer and lane, in the engine's
    (layer, lane) order, every rank all-gathers its lane slice into the
    global [L, B, H, d] output."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Bg, Hg, Gg, Dg, NL = 8, 32, 8, 16, 3
        plan = ShardPlan(world, rank, Bg, Gg, Hg)
        full = torch.arange(NL * Bg * Hg * Dg, dtype=torch.float32).view(NL, Bg, Hg, Dg)
        b0, b1 = plan.batch_range()
        h0, h1 = plan.q_range()
        out = full[:, b0:b1, h0:h1].contiguous()           # this rank's engine.out
        bl = plan.b_loc // lanes
        gathered = torch.zeros_like(full)
        bufs = [torch.empty((world, bl, plan.h_loc, Dg)) for _ in range(lanes)]
        for li in range(NL):
            for k in range(lanes):
                gather_lane_outputs(plan, out[li, k * bl:(k + 1) * bl], bufs[k], gathered[li],
                                    k * bl)
        if rank == 0:
            q.put(torch.equal(gathered, full))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,lanes", [(2, 2), (4, 2), (8, 1)])
def test_engine_lane_gather_reassembles_every_layer(world, lanes):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lane_worker, args=(r, world, port, q, lanes)) for r in range(world)]
    for p in procs:
        p.start()
    ok = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok
