"""GPU: the multi-layer DecodeEngine (CUDA-graph replay, micro-batch lanes,
deferred DCU tails on side streams) against the per-layer drop-in API
(`run_decode`, ck/session.py:42-64) and the CPU oracle on identical inputs.

Lanes split the batch into sequence groups on their own streams; every
(b, g) unit runs the same kernels with the same summation order, so the
engine's outputs, index lists, centroids and FIFO cursors must equal the
per-layer path bit for bit, whatever the lane count."""

import numpy as np
import pytest
import torch

import paper_2512_15550_b200 as P
from oracle import ctkv_oracle as O
from paper_2512_15550_b200.engine import DecodeEngine

pytestmark = pytest.mark.gpu

B, H, G, D, S, T, NL = 4, 8, 2, 128, 3072, 5, 2
PARAMS = dict(init_len=32, local_len=256, capacity=256, rho=320)
CP, RP = 4, 128


def _inputs(li, b=B):
    q, k, v = O.generate(O.Drift(seed=60 + li, s=S, decode_steps=T), b, H, G, D)
    return O.bf16_round(q), O.bf16_round(k), O.bf16_round(v)


def _prefill(q, k, v):
    return P.prefill(np.ascontiguousarray(q[:, :, :S]), np.ascontiguousarray(k[:, :, :S]),
                     np.ascontiguousarray(v[:, :, :S]), P.PrefillParams(**PARAMS),
                     dtype=torch.bfloat16, reserve=T + 2, build_mode=0)


@pytest.mark.parametrize("lanes,graph,b,nl", [(1, False, B, NL), (2, True, B, NL), (4, True, B, NL),
                                              (4, "host", B, NL), (2, "host", B, 6), (4, True, 12, NL)])
def test_engine_equals_per_layer_decode(lanes, graph, b, nl):
    """graph="host": steps from t = 1 run through capture_host_io's two
    graph slots (q/k/v copied in from pinned host buffers per (layer, lane)
    inside the step, outputs copied out 4 layers at a time).  b = 12
    (24 units, 6 per lane): the per-layer path takes 4-CTA chain clusters and
    so must every lane, although a lane alone would qualify for 8 (the engine
    passes the whole-batch choice, include/ctkv.h phase bits 32/64).  nl = 6
    with host I/O: outputs leave in a 4-layer copy and a 2-layer remainder."""
    torch.cuda.set_device(0)
    NL = nl
    data = [_inputs(li, b) for li in range(NL)]
    cfg = P.DecodeConfig(CP, RP)
    # per-layer drop-in path
    ref_out, ref_idx = [], []
    for q, k, v in data:
        st, ix = _prefill(q, k, v)
        outs, _ = P.run_decode(st, ix, cfg, np.ascontiguousarray(q[:, :, S:S + T]),
                               np.ascontiguousarray(k[:, :, S:S + T]),
                               np.ascontiguousarray(v[:, :, S:S + T]))
        ref_out.append(outs)
        ref_idx.append((ix.lists.copy(), ix.centroid_queries.copy(), ix.fifo_head.copy()))
    # engine
    built = [_prefill(q, k, v) for q, k, v in data]
    eng = DecodeEngine(built, cfg, lanes=lanes)
    dev = eng.q.device
    got = np.zeros((NL, b, H, T, D), np.float32)
    hbufs = None
    for t in range(T):
        if graph == "host" and t >= 1:
            if hbufs is None:
                hbufs = eng.capture_host_io(2)
            hq, hk, hv, hout = hbufs[t % 2]
            for li, (q, k, v) in enumerate(data):
                hq[li].copy_(torch.from_numpy(np.ascontiguousarray(q[:, :, S + t])))
                hk[li].copy_(torch.from_numpy(np.ascontiguousarray(k[:, :, S + t])))
                hv[li].copy_(torch.from_numpy(np.ascontiguousarray(v[:, :, S + t])))
            eng.replay_host(t % 2)
            torch.cuda.synchronize()
            got[:, :, :, t] = hout.numpy()
            continue
        for li, (q, k, v) in enumerate(data):
            eng.q[li].copy_(torch.from_numpy(np.ascontiguousarray(q[:, :, S + t])).to(dev))
            eng.k[li].copy_(torch.from_numpy(np.ascontiguousarray(k[:, :, S + t])).to(dev))
            eng.v[li].copy_(torch.from_numpy(np.ascontiguousarray(v[:, :, S + t])).to(dev))
        if graph and t == 1:
            eng.capture()
        if graph and t >= 1:
            eng.replay()
        else:
            eng.step()
        torch.cuda.synchronize()
        got[:, :, :, t] = eng.out.cpu().numpy()
    eng.check()
    for li, (st, ix) in enumerate(built):
        np.testing.assert_array_equal(got[li], ref_out[li])
        assert st.total_tokens == S + T and int(st.total_dev.item()) == S + T
        np.testing.assert_array_equal(ix.lists, ref_idx[li][0])
        np.testing.assert_array_equal(ix.centroid_queries, ref_idx[li][1])
        np.testing.assert_array_equal(ix.fifo_head, ref_idx[li][2])


def test_engine_matches_oracle_bf16():
    """Engine (4 lanes, graph) vs the f64 oracle on the same bf16-rounded
    inputs: outputs within 1e-3 norm-relative (bf16 decode tolerance)."""
    torch.cuda.set_device(0)
    data = [_inputs(li) for li in range(NL)]
    built = [_prefill(q, k, v) for q, k, v in data]
    eng = DecodeEngine(built, P.DecodeConfig(CP, RP), lanes=4)
    dev = eng.q.device
    orc = []
    for q, k, v in data:
        ost, oidx = O.prefill(np.ascontiguousarray(q[:, :, :S]), np.ascontiguousarray(k[:, :, :S]),
                              np.ascontiguousarray(v[:, :, :S]), **PARAMS)
        _, recs = O.run_decode(ost, oidx, q[:, :, S:S + T], k[:, :, S:S + T], v[:, :, S:S + T], CP, RP)
        orc.append(recs)
    for t in range(T):
        for li, (q, k, v) in enumerate(data):
            eng.q[li].copy_(torch.from_numpy(np.ascontiguousarray(q[:, :, S + t])).to(dev))
            eng.k[li].copy_(torch.from_numpy(np.ascontiguousarray(k[:, :, S + t])).to(dev))
            eng.v[li].copy_(torch.from_numpy(np.ascontiguousarray(v[:, :, S + t])).to(dev))
        if t == 1:
            eng.capture()
        eng.replay() if t >= 1 else eng.step()
        torch.cuda.synchronize()
        for li in range(NL):
            ref = orc[li][t].out
            err = np.linalg.norm(eng.out[li].cpu().numpy() - ref) / np.linalg.norm(ref)
            assert err < 1e-3, (t, li, err)


def test_engine_refuses_to_overrun_store_capacity():
    """The fused scan appends in place and never grows the store: the engine
    raises before enqueueing a step the stores have no room for,
    and reserve() drops graphs that captured the old storage pointers."""
    torch.cuda.set_device(0)
    q, k, v = _inputs(0)
    st, ix = P.prefill(np.ascontiguousarray(q[:, :, :S]), np.ascontiguousarray(k[:, :, :S]),
                       np.ascontiguousarray(v[:, :, :S]), P.PrefillParams(**PARAMS),
                       dtype=torch.bfloat16, reserve=2, build_mode=0)
    assert st.capacity - st.total_tokens == 2
    eng = DecodeEngine([(st, ix)], P.DecodeConfig(CP, RP), lanes=1)
    assert eng.room() == 2
    eng.step()
    eng.capture()
    eng.replay()
    torch.cuda.synchronize()
    assert eng.room() == 0
    with pytest.raises(P.ConfigError):
        eng.step()
    with pytest.raises(P.ConfigError):
        eng.replay()
    eng.reserve(3)
    assert eng.graph is None and eng.room() >= 3
    eng.step()
    torch.cuda.synchronize()
    eng.check()
    assert st.total_tokens == S + 3 and int(st.total_dev.item()) == S + 3


def test_stage_copy_moves_pinned_host_bytes_both_ways():
    """ctkv_stage_copy (the engine's in-graph host I/O): host -> device and
    device -> host through mapped pinned memory, byte-exact; misaligned or
    non-16-byte sizes are refused (CTKV_ECONFIG)."""
    from paper_2512_15550_b200 import _native as N
    torch.cuda.set_device(0)
    lib = N.lib()
    src = torch.arange(4096 * 3, dtype=torch.int32).pin_memory()
    dev = torch.empty(src.shape, dtype=torch.int32, device="cuda")
    back = torch.zeros(src.shape, dtype=torch.int32).pin_memory()
    st = torch.cuda.current_stream().cuda_stream
    assert lib.ctkv_stage_copy(dev.data_ptr(), src.data_ptr(), src.nbytes, st) == N.OK
    assert lib.ctkv_stage_copy(back.data_ptr(), dev.data_ptr(), dev.nbytes, st) == N.OK
    torch.cuda.synchronize()
    assert torch.equal(back, src) and torch.equal(dev.cpu(), src)
    assert lib.ctkv_stage_copy(dev.data_ptr(), src.data_ptr(), 20, st) == N.ECONFIG
    assert lib.ctkv_stage_copy(dev.data_ptr() + 4, src.data_ptr(), 32, st) == N.ECONFIG
    assert lib.ctkv_stage_copy(dev.data_ptr(), src.data_ptr(), 0, st) == N.OK
