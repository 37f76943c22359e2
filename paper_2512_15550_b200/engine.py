"""Multi-layer decode engine: the serving-shaped entry point.

One (KvStore, QueryCentroidIndex) pair per layer lives in HBM; a decode
step walks the layers in order and, per layer, enqueues the scan kernel
(append, centroid cosines, static partials) and the unit kernels (recall,
rerank, sparse attention, merge) on the main stream, and the layer's tail
(FIFO DCU, cursor/total advance) on a side stream that overlaps the next
layers.  No host synchronisation, so the whole step is captured once as a
CUDA graph and replayed per token.  Under a ShardPlan
each rank owns a (batch x kv-head) shard and all-gathers the head-sharded
outputs after every layer (captured in the same graph).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _native as N
from .index import QueryCentroidIndex
from .parallel import ShardPlan, all_gather_outputs
from .retrieval import DecodeConfig, StepBuffers
from .store import KvStore


@dataclass
class Layer:
    store: KvStore
    index: QueryCentroidIndex
    bufs: StepBuffers
    call: tuple | None = None   # cached ctypes arguments of ctkv_decode_step_phase


class DecodeEngine:
    def __init__(self, layers: list[tuple[KvStore, QueryCentroidIndex]], cfg: DecodeConfig, *,
                 plan: ShardPlan | None = None, group=None):
        if not layers:
            raise ValueError("DecodeEngine needs at least one layer")
        self.cfg = cfg
        self.plan = plan
        self.group = group
        st0 = layers[0][0]
        lay = st0.layout
        self.b, self.h, self.g, self.d = lay.batch, lay.query_heads, lay.kv_heads, lay.head_dim
        self.dtype = st0.dtype
        dev = st0.keys.device
        # one workspace per layer: a layer's deferred tail (DCU, cursor/total
        # advance) reads its workspace while later layers already run
        self.layers: list[Layer] = []
        for store, index in layers:
            self.layers.append(Layer(store, index, StepBuffers.allocate(store, index, cfg)))
        nl = len(self.layers)
        self._side = torch.cuda.Stream(device=dev) if dev.type == "cuda" else None
        self._tail_ev = [torch.cuda.Event() for _ in range(nl)] if self._side is not None else []
        # step inputs (device): q [L,b,h,d], k/v [L,b,g,d]
        self.q = torch.zeros((nl, self.b, self.h, self.d), dtype=self.dtype, device=dev)
        self.k = torch.zeros((nl, self.b, self.g, self.d), dtype=self.dtype, device=dev)
        self.v = torch.zeros((nl, self.b, self.g, self.d), dtype=self.dtype, device=dev)
        self.out = torch.zeros((nl, self.b, self.h, self.d), dtype=torch.float32, device=dev)
        for li, layer in enumerate(self.layers):
            layer.bufs.out = self.out[li]          # kernels write the layer output in place
        world = plan.world if plan else 1
        self.gathered = (torch.zeros((nl, plan.batch, plan.query_heads, self.d), dtype=torch.float32,
                                     device=dev) if world > 1 else self.out)
        self._gbuf = (torch.empty((world, self.b, self.h, self.d), dtype=torch.float32, device=dev)
                      if world > 1 else None)
        self.graph: torch.cuda.CUDAGraph | None = None
        self.steps_done = 0

    # -- one step -------------------------------------------------------------

    def _prepare(self) -> None:
        """Build every layer's ctypes argument block once (pointers are fixed
        for the engine's lifetime), so a launch costs one foreign call."""
        cfg = self.cfg
        for li, layer in enumerate(self.layers):
            st, ix, bf = layer.store, layer.index, layer.bufs
            if cfg.c_prime > ix.capacity:
                raise ValueError("c_prime exceeds the index capacity")
            args = N.StepArgs(self.q[li].data_ptr(), self.k[li].data_ptr(), self.v[li].data_ptr(),
                              cfg.c_prime, cfg.rho_prime, int(cfg.use_dcu), int(cfg.use_rerank),
                              bf.out.data_ptr(), bf.row_max.data_ptr(), bf.denom.data_ptr(),
                              bf.selected.data_ptr(), bf.recall_len.data_ptr(),
                              bf.sparse_ids.data_ptr(), bf.sparse_len.data_ptr(), bf.sparse_cap,
                              bf.flags.data_ptr())
            layer.call = (st.ctkv_layout(), st.desc(), ix.desc(), args, bf.ws.data_ptr(),
                          bf.ws.numel())

    def _launch(self, layer: Layer, phase: int) -> None:
        lay, sd, idd, args, ws, wsn = layer.call
        rc = self._fn(lay, sd, idd, args, phase, ws, wsn, torch.cuda.current_stream().cuda_stream)
        if rc:
            N.check(rc, "decode_step")

    def _enqueue(self, events=None) -> None:
        if self.layers[0].call is None:
            self._prepare()
            self._fn = N.lib().ctkv_decode_step_phase
        main = torch.cuda.current_stream()
        for li, layer in enumerate(self.layers):
            # phase bits: 1 scan, 2 unit, 8 defer the tail, 4 tail only
            if events is not None:
                events[li][0].record()
                self._launch(layer, 1)
                events[li][1].record()
                self._launch(layer, 2 | 8)
                events[li][2].record()
            else:
                self._launch(layer, 1 | 2 | 8)
            # the tail (DCU write, sparse ids, cursor/total advance) is only
            # read by this layer's next step: run it beside the next layers
            self._tail_ev[li].record(main)
            self._side.wait_event(self._tail_ev[li])
            with torch.cuda.stream(self._side):
                self._launch(layer, 4)
            if self._gbuf is not None:
                self.gathered[li].copy_(all_gather_outputs(self.plan, self.out[li], self.group,
                                                           self._gbuf))
        main.wait_stream(self._side)

    def _note(self) -> None:
        for layer in self.layers:
            layer.store.note_device_append()
        self.steps_done += 1

    def reserve(self, steps: int) -> None:
        for layer in self.layers:
            layer.store.ensure_room(steps)
            layer.call = None   # storage may have moved

    def step(self, events=None) -> None:
        """Enqueue one decode step (all layers) eagerly."""
        self._enqueue(events)
        self._note()

    def capture(self) -> None:
        """Capture one step as a CUDA graph (state is device-resident, so
        replays advance the stores, cursors and FIFO exactly like eager
        steps).  Call after at least one eager warm-up step."""
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        # the capture itself must not run the kernels: snapshot nothing, the
        # graph records launches only
        with torch.cuda.graph(g):
            self._enqueue()
        self.graph = g

    def replay(self) -> None:
        if self.graph is None:
            raise RuntimeError("capture() first")
        self.graph.replay()
        self._note()

    def flags(self) -> int:
        f = 0
        for layer in self.layers:
            f |= int(layer.bufs.flags.item())
        return f

    def check(self) -> None:
        N.raise_flags(self.flags(), "decode step")
