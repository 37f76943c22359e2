"""The engine's multi-rank path on the GPU: 2 or 4 ranks, each decoding its
(batch x kv-head) shard with the real kernels through DecodeEngine(plan=...)
-- the per-(layer, lane) all-gather issued on the engine's communication
stream in the fixed (layer, lane) order, lanes waiting on it -- must equal
the unsharded engine bit for bit.

The pool gives one GPU per job and NCCL refuses two ranks on one device, so
the ranks share cuda:0 over the gloo backend (which stages CUDA tensors
through the host); steps run eagerly (gloo collectives cannot be captured
into a CUDA graph).  On an 8-GPU node `bench.py --gpus 8` runs the same code
path over NCCL inside the step graph."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

B, H, G, D, S, T, NL = 2, 16, 4, 128, 3072, 4, 2
PARAMS = dict(init_len=32, local_len=256, capacity=256, rho=320)
CP, RP = 4, 128


def _layers(plan):
    import paper_2512_15550_b200 as P
    from oracle import ctkv_oracle as O
    b0, b1 = plan.batch_range()
    g0, g1 = plan.kv_range()
    h0, h1 = plan.q_range()
    built, inputs = [], []
    for li in range(NL):
        q, k, v = O.generate(O.Drift(seed=70 + li, s=S, decode_steps=T), B, H, G, D)
        q, k, v = O.bf16_round(q)[b0:b1, h0:h1], O.bf16_round(k)[b0:b1, g0:g1], O.bf16_round(v)[b0:b1, g0:g1]
        st, ix = P.prefill(np.ascontiguousarray(q[:, :, :S]), np.ascontiguousarray(k[:, :, :S]),
                           np.ascontiguousarray(v[:, :, :S]), P.PrefillParams(**PARAMS),
                           dtype=torch.bfloat16, reserve=T + 2, build_mode=0)
        built.append((st, ix))
        inputs.append((q, k, v))
    return built, inputs


def _run(plan, group=None, lanes=1):
    import paper_2512_15550_b200 as P
    from paper_2512_15550_b200.engine import DecodeEngine
    built, inputs = _layers(plan)
    eng = DecodeEngine(built, P.DecodeConfig(CP, RP), plan=plan if plan.world > 1 else None,
                       group=group, lanes=lanes)
    dev = eng.q.device
    outs = []
    for t in range(T):
        for li, (q, k, v) in enumerate(inputs):
            eng.q[li].copy_(torch.from_numpy(np.ascontiguousarray(q[:, :, S + t])).to(dev))
            eng.k[li].copy_(torch.from_numpy(np.ascontiguousarray(k[:, :, S + t])).to(dev))
            eng.v[li].copy_(torch.from_numpy(np.ascontiguousarray(v[:, :, S + t])).to(dev))
        eng.step()
        torch.cuda.synchronize()
        outs.append(eng.gathered.cpu().numpy().copy())
    eng.check()
    return np.stack(outs), [ix.fifo_head.copy() for _, ix in built]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_15550_b200.parallel import ShardPlan
        plan = ShardPlan(world, rank, B, G, H)
        outs, fifo = _run(plan, lanes=plan.b_loc)
        if rank == 0:
            q.put((outs, fifo))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4])
def test_engine_sharded_over_ranks_equals_unsharded(world):
    from paper_2512_15550_b200.parallel import ShardPlan
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    got, fifo = q.get(timeout=600)
    for p_ in procs:
        p_.join(timeout=600)
        assert p_.exitcode == 0
    torch.cuda.set_device(0)
    ref, ref_fifo = _run(ShardPlan(1, 0, B, G, H), lanes=2)
    np.testing.assert_array_equal(got, ref)
    for a, b in zip(fifo, ref_fifo):   # head shards: every rank holds all B cursors
        np.testing.assert_array_equal(a, b)
