"""Multi-layer decode engine: the serving-shaped entry point.

One (KvStore, QueryCentroidIndex) pair per layer lives in HBM; a decode
step walks the layers in order and, per layer, enqueues the scan kernel
(append, centroid cosines, static partials) and the unit kernels (recall,
rerank, sparse attention, merge), and the layer's tail (FIFO DCU,
cursor/total advance) on a side stream that overlaps the next layers.  No
host synchronisation, so the whole step is captured once as a CUDA graph
and replayed per token.

Lanes (micro-batches).  The sequences of a batch are independent through
every layer (ck/retrieval.py:151-167 loops over (b, g) units with no
cross-sequence state except the per-sequence FIFO cursor), so the batch is
split into `lanes` groups of sequences, each walking the layers on its own
stream.  Per lane the layer order is kept (layer l+1 of a sequence starts
after its layer l), but while one lane runs the latency-bound part of a
layer (top-C' -> union -> rerank -> top-rho' -> attention) another lane's
bandwidth-bound centroid scan fills the GPU.  No data dependency is
relaxed; this is the two-batch-overlap of serving engines.

Under a ShardPlan each rank owns a (batch x kv-head) shard and all-gathers
the head-sharded outputs after every layer (captured in the same graph) on
one communication stream in a fixed (layer, lane) order, so every rank
issues the collectives identically; lane k's layer l+1 waits for its layer-l
gather.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _native as N
from .errors import ConfigError
from .index import QueryCentroidIndex
from .parallel import ShardPlan, gather_lane_outputs
from .retrieval import DecodeConfig, StepBuffers
from .store import KvStore


@dataclass
class Layer:
    store: KvStore
    index: QueryCentroidIndex
    bufs: StepBuffers
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    call: tuple | None = None   # cached ctypes arguments of ctkv_decode_step_phase


class DecodeEngine:
    def __init__(self, layers: list[tuple[KvStore, QueryCentroidIndex]], cfg: DecodeConfig, *,
                 plan: ShardPlan | None = None, group=None, lanes: int = 1):
        if not layers:
            raise ValueError("DecodeEngine needs at least one layer")
        self.cfg = cfg
        self.plan = plan
        self.group = group
        self.parents = list(layers)
        st0 = layers[0][0]
        lay = st0.layout
        self.b, self.h, self.g, self.d = lay.batch, lay.query_heads, lay.kv_heads, lay.head_dim
        if lanes < 1 or self.b % lanes:
            raise ValueError(f"lanes={lanes} must divide the batch {self.b}")
        self.nlanes = lanes
        self.bl = self.b // lanes
        # chain cluster size from the whole batch (phase bits 32/64), the
        # same for every lane (ctkv_decode_step_phase, include/ctkv.h)
        self._cl_bits = 32 | (64 if self.b * self.g <= 16 else 0)
        self.dtype = st0.dtype
        dev = st0.keys.device
        nl = len(layers)
        self.nl = nl
        # step inputs (device): q [L,b,h,d], k/v [L,b,g,d]; outputs [L,b,h,d] f32
        self.q = torch.zeros((nl, self.b, self.h, self.d), dtype=self.dtype, device=dev)
        self.k = torch.zeros((nl, self.b, self.g, self.d), dtype=self.dtype, device=dev)
        self.v = torch.zeros((nl, self.b, self.g, self.d), dtype=self.dtype, device=dev)
        self.out = torch.zeros((nl, self.b, self.h, self.d), dtype=torch.float32, device=dev)
        # lane_layers[k][l]: lane k's view of layer l.  One workspace per
        # (lane, layer): a layer's deferred tail reads its workspace while
        # later layers already run.
        # Layers may alias one (store, index) pair (a capacity plan that
        # cycles fewer physical layer buffers than logical layers, bench
        # cfg3): the aliases share one lane view (one token counter), and a
        # layer's scan waits for the previous alias's deferred tail.
        self._alias_prev: list[int | None] = []
        seen: dict[int, int] = {}
        for li, (store, _) in enumerate(layers):
            j = seen.get(id(store))
            if j is not None and li - j < 2:
                raise ValueError(f"layers {j} and {li} alias one store; aliases must be >= 2 apart")
            self._alias_prev.append(j)
            seen[id(store)] = li
        self._appends = {}                       # id(parent store) -> appends per step
        for store, _ in layers:
            self._appends[id(store)] = self._appends.get(id(store), 0) + 1
        self.lane_layers: list[list[Layer]] = []
        for k in range(lanes):
            b0, b1 = k * self.bl, (k + 1) * self.bl
            row = []
            views: dict[int, tuple] = {}
            for li, (store, index) in enumerate(layers):
                if lanes > 1:
                    if id(store) not in views:
                        views[id(store)] = (store.batch_view(b0, b1), index.batch_view(b0, b1))
                    store, index = views[id(store)]
                bufs = StepBuffers.allocate(store, index, cfg)
                bufs.out = self.out[li, b0:b1]      # kernels write the layer output in place
                row.append(Layer(store, index, bufs, self.q[li, b0:b1], self.k[li, b0:b1],
                                 self.v[li, b0:b1]))
            self.lane_layers.append(row)
        self.layers = [L for row in self.lane_layers for L in row]
        cuda = dev.type == "cuda"
        self._lane_st = [torch.cuda.Stream(device=dev) for _ in range(lanes)] if cuda else []
        self._tail_st = [torch.cuda.Stream(device=dev) for _ in range(lanes)] if cuda else []
        self._ev = ([[torch.cuda.Event() for _ in range(nl)] for _ in range(lanes)] if cuda else [])
        self._evs = ([[torch.cuda.Event() for _ in range(nl)] for _ in range(lanes)] if cuda else [])
        self._evt = ([[torch.cuda.Event() for _ in range(nl)] for _ in range(lanes)] if cuda else [])
        world = plan.world if plan else 1
        self.world = world
        self._comm = torch.cuda.Stream(device=dev) if (cuda and world > 1) else None
        self._gev = ([[torch.cuda.Event() for _ in range(nl)] for _ in range(lanes)]
                     if self._comm is not None else [])
        self.gathered = (torch.zeros((nl, plan.batch, plan.query_heads, self.d), dtype=torch.float32,
                                     device=dev) if world > 1 else self.out)
        self._gbuf = ([torch.empty((world, self.bl, self.h, self.d), dtype=torch.float32, device=dev)
                       for _ in range(lanes)] if world > 1 else None)
        self.graph: torch.cuda.CUDAGraph | None = None
        self._hgraphs: list | None = None
        self.steps_done = 0

    # -- one step -------------------------------------------------------------

    def _prepare(self) -> None:
        """Build every (lane, layer) ctypes argument block once (pointers are
        fixed for the engine's lifetime), so a launch costs one foreign call."""
        cfg = self.cfg
        for L in self.layers:
            st, ix, bf = L.store, L.index, L.bufs
            if cfg.c_prime > ix.capacity:
                raise ValueError("c_prime exceeds the index capacity")
            args = N.StepArgs(L.q.data_ptr(), L.k.data_ptr(), L.v.data_ptr(),
                              cfg.c_prime, cfg.rho_prime, int(cfg.use_dcu), int(cfg.use_rerank),
                              bf.out.data_ptr(), bf.row_max.data_ptr(), bf.denom.data_ptr(),
                              bf.selected.data_ptr(), bf.recall_len.data_ptr(),
                              bf.sparse_ids.data_ptr(), bf.sparse_len.data_ptr(), bf.sparse_cap,
                              bf.flags.data_ptr())
            L.call = (st.ctkv_layout(), st.desc(), ix.desc(), args, bf.ws.data_ptr(), bf.ws.numel())
        self._fn = N.lib().ctkv_decode_step_phase

    def _launch(self, layer: Layer, phase: int, stream=None) -> None:
        lay, sd, idd, args, ws, wsn = layer.call
        s = stream if stream is not None else torch.cuda.current_stream()
        rc = self._fn(lay, sd, idd, args, phase, ws, wsn, s.cuda_stream)
        if rc:
            N.check(rc, "decode_step")

    @staticmethod
    def _stage(dst: torch.Tensor, src: torch.Tensor, stream) -> None:
        """Host<->device staging copy by a kernel (ctkv_stage_copy): one side
        is pinned host memory, reached through unified addressing, so the
        step graph holds kernel nodes instead of host memcpy nodes (those make
        every launch of the graph hundreds of microseconds slower)."""
        assert dst.is_contiguous() and src.is_contiguous() and dst.nbytes == src.nbytes
        N.check(N.lib().ctkv_stage_copy(dst.data_ptr(), src.data_ptr(), src.nbytes,
                                        stream.cuda_stream), "stage copy")

    def _gather(self, k: int, li: int) -> None:
        """All-gather lane k's layer-li output slice [bl, h_loc, d] into the
        global [B, H, d] view (parallel.gather_lane_outputs)."""
        b0 = k * self.bl
        gather_lane_outputs(self.plan, self.out[li, b0:b0 + self.bl], self._gbuf[k],
                            self.gathered[li], b0, self.group)

    def _enqueue_timed(self, events) -> None:
        """Serial eager step on the current stream with CUDA events around
        each launch: events[i] = (start, after scan, after unit) for
        i = layer * lanes + lane."""
        for li in range(self.nl):
            for k in range(self.nlanes):
                L = self.lane_layers[k][li]
                ev = events[li * self.nlanes + k]
                ev[0].record()
                self._launch(L, 1 | self._cl_bits)
                ev[1].record()
                self._launch(L, 2 | 8 | self._cl_bits)
                ev[2].record()
                self._launch(L, 4 | self._cl_bits)
                if self.world > 1:
                    self._gather(k, li)

    def _enqueue(self, events=None, hio=None) -> None:
        if self.layers[0].call is None:
            self._prepare()
        if events is not None:
            self._enqueue_timed(events)
            return
        main = torch.cuda.current_stream()
        fork = torch.cuda.Event()
        fork.record(main)
        streams = self._lane_st + self._tail_st + ([self._comm] if self._comm is not None else [])
        if hio is not None:
            streams = streams + [self._cin, self._cout]
        for s in streams:
            s.wait_event(fork)
        if hio is not None:
            # host inputs: every (layer, lane) slice copied in issue order on
            # one stream, so the copies run ahead of the layers that use them
            hq, hk, hv, _ = hio
            # layer 0 alone first (the step starts as soon as it is in), then
            # chunks of _cin_chunk layers running ahead of their use
            bounds = [0, 1] + list(range(1 + self._cin_chunk, self.nl, self._cin_chunk)) + [self.nl]
            bounds = sorted(set(min(x, self.nl) for x in bounds))
            for c0, c1 in zip(bounds[:-1], bounds[1:]):
                self._stage(self.q[c0:c1], hq[c0:c1], self._cin)
                self._stage(self.k[c0:c1], hk[c0:c1], self._cin)
                self._stage(self.v[c0:c1], hv[c0:c1], self._cin)
                for li in range(c0, c1):
                    for k in range(self.nlanes):
                        self._cin_ev[k][li].record(self._cin)
        for li in range(self.nl):
            for k in range(self.nlanes):
                L = self.lane_layers[k][li]
                ls, ts = self._lane_st[k], self._tail_st[k]
                if hio is not None:
                    ls.wait_event(self._cin_ev[k][li])
                if self._comm is not None and li > 0:
                    ls.wait_event(self._gev[k][li - 1])
                j = self._alias_prev[li]
                if j is not None:
                    ls.wait_event(self._evt[k][j])      # the alias's DCU tail is done
                # phase bits: 1 scan, 2 unit, 8 defer the tail, 4 tail only, 16 PDL
                # allowed (the kernel before a scan on a lane stream is the
                # previous layer's chain, before a chain this layer's scan).
                # The previous layer's tail is released once this layer's scan
                # is done, so it shares the GPU with this chain, not this scan.
                self._launch(L, 1 | 16 | self._cl_bits, ls)
                if li > 0:
                    es = self._evs[k][li]
                    es.record(ls)
                    ts.wait_event(self._ev[k][li - 1])
                    ts.wait_event(es)
                    self._launch(self.lane_layers[k][li - 1], 4 | self._cl_bits, ts)
                    self._evt[k][li - 1].record(ts)
                self._launch(L, 2 | 8 | 16 | self._cl_bits, ls)
                ev = self._ev[k][li]
                ev.record(ls)
                if li == self.nl - 1:
                    ts.wait_event(ev)
                    self._launch(L, 4 | self._cl_bits, ts)
                    self._evt[k][li].record(ts)
                if self._comm is not None:
                    self._comm.wait_event(ev)
                    with torch.cuda.stream(self._comm):
                        self._gather(k, li)
                    self._gev[k][li].record(self._comm)
            if hio is not None and self._comm is None and ((li + 1) % self._cout_chunk == 0
                                                            or li == self.nl - 1):
                # every _cout_chunk layers' outputs leave in one copy once all
                # lanes have finished them, while later layers run
                c0 = li - (li % self._cout_chunk)
                for k in range(self.nlanes):
                    self._cout.wait_event(self._ev[k][li])
                self._stage(hio[3][c0:li + 1], self.out[c0:li + 1], self._cout)
            if hio is not None and self._comm is not None:
                self._cout.wait_event(self._gev[self.nlanes - 1][li])   # all lanes gathered
                self._stage(hio[3][li], self.gathered[li], self._cout)
        for s in streams:
            main.wait_stream(s)

    def _note(self) -> None:
        for L in self.layers:
            L.store.note_device_append()
        if self.nlanes > 1:
            for li, (store, _) in enumerate(self.parents):
                store.note_device_append()
        self.steps_done += 1

    def reserve(self, steps: int) -> None:
        if self.nlanes > 1:
            raise RuntimeError("reserve() before splitting into lanes (lane views share storage)")
        for L in self.layers:
            L.store.ensure_room(steps * self._appends[id(L.store)])
            L.call = None   # storage may have moved
        self.graph = None   # captured graphs hold the old pointers
        self._hgraphs = None

    def room(self) -> int:
        """Decode steps left before some layer's store is full (the fused
        scan appends in place and never grows the store)."""
        left = None
        for store, _ in self.parents:
            n = (store.capacity - store.total_tokens) // self._appends[id(store)]
            left = n if left is None else min(left, n)
        return left

    def _check_room(self) -> None:
        if self.room() < 1:
            raise ConfigError("decode step: a layer's KvStore is full (reserve() more rows "
                              "before capturing, or build the stores with a larger capacity)")

    def step(self, events=None) -> None:
        """Enqueue one decode step (all layers) eagerly."""
        self._check_room()
        self._enqueue(events)
        self._note()

    def capture(self) -> None:
        """Capture one step as a CUDA graph (state is device-resident, so
        replays advance the stores, cursors and FIFO exactly like eager
        steps).  Call after at least one eager warm-up step."""
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._enqueue()
        self.graph = g

    def replay(self) -> None:
        if self.graph is None:
            raise RuntimeError("capture() first")
        self._check_room()
        self.graph.replay()
        self._note()

    # -- host I/O inside the step -------------------------------------------

    def capture_host_io(self, slots: int = 2) -> list:
        """Capture `slots` step graphs whose inputs come from, and outputs go
        to, pinned host buffers: each (layer, lane)'s q/k/v slice is copied in
        on a copy stream ahead of its layer, and its output is copied out as
        soon as the layer finishes, so the transfers overlap the other
        layers.  Returns the host buffer sets (q [L,b,h,d], k/v [L,b,g,d],
        out like `gathered`); with two slots a caller fills one slot's inputs
        while the other slot's step runs (`replay_host(slot)`)."""
        if self.layers[0].call is None:
            self._prepare()
        dev = self.q.device
        self._cin = torch.cuda.Stream(device=dev)
        self._cout = torch.cuda.Stream(device=dev)
        self._cin_ev = [[torch.cuda.Event() for _ in range(self.nl)] for _ in range(self.nlanes)]
        self._cin_chunk = 4   # layers per input copy
        self._cout_chunk = 4  # layers per output copy
        bufs, graphs = [], []
        torch.cuda.synchronize()
        for _ in range(slots):
            hio = (torch.empty(self.q.shape, dtype=self.dtype).pin_memory(),
                   torch.empty(self.k.shape, dtype=self.dtype).pin_memory(),
                   torch.empty(self.v.shape, dtype=self.dtype).pin_memory(),
                   torch.empty(self.gathered.shape, dtype=torch.float32).pin_memory())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._enqueue(hio=hio)
            bufs.append(hio)
            graphs.append(g)
        self._hgraphs = graphs
        return bufs

    def replay_host(self, slot: int) -> None:
        """One step through host buffer set `slot` (see capture_host_io); the
        outputs are in that set's out buffer once the stream is synchronised."""
        if not self._hgraphs:
            raise RuntimeError("capture_host_io() first")
        self._check_room()
        self._hgraphs[slot].replay()
        self._note()

    def flags(self) -> int:
        f = 0
        for L in self.layers:
            f |= int(L.bufs.flags.item())
        return f

    def sync_parents(self) -> None:
        """Copy the lanes' token counters back into the layers' stores (the
        lanes share K/V, centroids, lists and cursors with them already)."""
        if self.nlanes > 1:
            for li, (store, _) in enumerate(self.parents):
                store.adopt_total(self.lane_layers[0][li].store)

    def check(self) -> None:
        N.raise_flags(self.flags(), "decode step")
        self.sync_parents()
