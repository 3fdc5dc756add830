"""The modality-masked batched forward on the device, and the serving-loop
worker that runs it.

``MaskedModel.forward(slots, masks)`` is one device pass over a batch of
requests with per-request modality masks:

  1. request compaction (``ms_compact``): per-modality stable index lists,
     inverse maps, counting sort by combo, and a gather of each present
     modality's clip rows from the resident clip pool into contiguous
     modality-grouped sub-batches;
  2. each modality's encoder program over its compacted rows only (absent
     modalities cost nothing);
  3. the fusion head reads the compacted features through the inverse maps
     (absent modalities contribute zeros) and writes logits in the original
     request order — the scatter is fused into the gather GEMM.

Each modality's encoder is a CUDA graph keyed by its compacted count and the
head a graph keyed by N; the present modalities' graphs replay concurrently
on side streams (fork after compaction, join before the head).

``DeviceExecutor`` plugs this into the serving loop's worker seam
(reference sim.py:365-397): each dispatched job's canonical parts
(strategy.py:54-60) become one masked batch (G2(i): requests fill parts in
index order), timed with CUDA events.
"""

from __future__ import annotations

import numpy as np

from . import device as dv
from .encoders import (CONV1_PAD, FEAT_DIM, SEGMENTS, TBN_MODALITIES, U8_BIAS, U8_SCALE,
                       BNInceptionEncoder, FusionHead, MLPEncoder)


def request_masks(parts, size: int) -> np.ndarray:
    """G2(i): requests 0..size-1 in index order fill the job's canonical
    parts in order.  A rounded-up strategy (scheduler.py:138-167) has more
    part rows than the job has requests: then the parts are taken in order
    of decreasing modality count (stable), so the rows left over are the
    least-informed subsets rather than, by the canonical bitmask order, the
    all-modality ones (oracle/selection.parts_for_requests, same rule)."""
    out = np.zeros(size, dtype=np.int16)
    if sum(b for _, b in parts) > size:
        parts = sorted(parts, key=lambda pb: -bin(int(pb[0])).count("1"))
    lo = 0
    for mask, batch in parts:
        hi = min(size, lo + batch)
        out[lo:hi] = mask
        lo = hi
        if lo >= size:
            break
    return out


class MaskedModel:
    """Encoders + fusion head + resident input pool + compaction buffers."""

    STAGE_RING = 4

    def __init__(self, encoders, head, pools, rows, max_req: int, device="cuda"):
        """``rows[k] = (lines, width, c_src, c_dst, pad_w)``: one request of
        modality k is ``lines`` x ``width`` pixels of ``c_src`` channels in the
        pool; in the encoder's input each pixel has ``c_dst`` channels and each
        line ``pad_w`` zero pixels on both ends (the gather pads)."""
        import torch
        self.torch = torch
        self.dev = torch.device(device)
        self.encoders = encoders
        self.head = head
        self.pools = pools  # per modality: [n_slots, ...] bf16, row = one request
        # (lines, width, c_src, c_dst, pad_w[, src_u8, u8_scale, u8_bias[, frame_h, pad_h]])
        self.rows = [tuple(r) + (0, 1.0, 0.0, 0, 0)[len(r) - 5:] for r in rows]
        # modality k's request -> pool-row map lives at slot_d[k*max_req : k*max_req + n]
        # + slot_off, + plane_stride (an encoder whose stem reads 4-channel planes)
        self.rows = [r[:10] + (k * max_req, int(getattr(e, "x_plane_stride", 0)))
                     for k, (r, e) in enumerate(zip(self.rows, encoders))]
        self.src_bytes = [1 if r[5] else 2 for r in self.rows]
        self.row_bytes = [int(r[0] * r[1] * r[2] * b) for r, b in zip(self.rows, self.src_bytes)]
        self.K = len(encoders)
        self.max_req = max_req
        K, n = self.K, max_req
        self.mask_d = torch.zeros(n, dtype=torch.int16, device=self.dev)
        self.slot_d = torch.zeros(K * n, dtype=torch.int32, device=self.dev)
        # compaction index outputs, one set per pass parity (pipelined passes:
        # the next pass's compaction runs while this pass's head still reads inv)
        self._ix = [tuple(torch.zeros(sz, dtype=torch.int32, device=self.dev)
                          for sz in (K * n, K * n, K, (1 << K) + 1, n)) for _ in range(2)]
        self.idx, self.inv, self.counts, self.offs, self.perm = self._ix[0]
        # pinned staging ring for stage_inputs: slot i is rewritten only after
        # the H2D copies that last read it have executed (its event)
        self._stage_h = [(torch.zeros(n, dtype=torch.int16).pin_memory(),
                          torch.zeros(K * n, dtype=torch.int32).pin_memory(), torch.cuda.Event())
                         for _ in range(self.STAGE_RING)]
        self._stage_i = 0
        # device mask ring for passes formed on the device (ms_pass_select
        # writes row i, the pass's compaction reads it; ring_ev[i] is recorded
        # after that compaction so the next writer of row i can wait on it)
        self.mask_ring = torch.zeros(self.STAGE_RING, n, dtype=torch.int16, device=self.dev)
        self.ring_ev = [torch.cuda.Event() for _ in range(self.STAGE_RING)]
        self.ring_used = [False] * self.STAGE_RING
        import ctypes
        self._X = (ctypes.c_void_p * K)(*[p.data_ptr() for p in pools])
        self._G = (ctypes.c_void_p * K)(*[e.x.data_ptr() for e in encoders])
        self._ROWS = (dv.RowDesc * K)(*[dv.RowDesc(*r) for r in self.rows])
        self._graphs = {}
        self._gexec = {}
        self.use_graphs = True
        self.parallel_modalities = True
        self._side = [torch.cuda.Stream() for _ in range(K)]
        self._ev_c = torch.cuda.Event()
        self._ev_k = [torch.cuda.Event() for _ in range(K)]
        # pipelined device-formed passes (run_ring_pipelined; MS_PIPELINE=0: off, for A/B)
        import os
        self._pipeline = os.environ.get("MS_PIPELINE", "1") != "0"
        self._parity = 0
        self._cstream = torch.cuda.Stream()
        # raw stream pointers + native events for the per-pass launch path
        self._side_p = [s.cuda_stream for s in self._side]
        self._cstream_p = self._cstream.cuda_stream
        self._nev_stem = [dv.Event() for _ in range(K)]
        self._nev_cpar = [dv.Event() for _ in range(2)]
        self._nev_k = [dv.Event() for _ in range(K)]
        self._nev_c = dv.Event()

    @property
    def n_slots(self) -> int:
        return self.pools[0].shape[0]

    # -- host-side bookkeeping ------------------------------------------
    def counts_for(self, masks: np.ndarray):
        m = masks.astype(np.int64)
        return tuple(int(((m >> k) & 1).sum()) for k in range(self.K))

    def stage_inputs(self, slots, masks, stream=None):
        """Copy one batch's slots/masks into the fixed device buffers (H2D
        from a pinned staging ring; stream-ordered).  The host rewrites a
        staging slot only after the copies that last read it have run."""
        n = len(masks)
        if n > self.max_req:
            raise ValueError(f"batch of {n} exceeds capacity {self.max_req}")
        mask_h, slot_h, ev = self._stage_h[self._stage_i]
        self._stage_i = (self._stage_i + 1) % len(self._stage_h)
        ev.synchronize()
        mask_h[:n] = self.torch.as_tensor(np.asarray(masks, dtype=np.int16))
        sl = np.asarray(slots, dtype=np.int32)
        if sl.ndim == 1:  # the same pool row for every modality
            sl = np.broadcast_to(sl, (self.K, n))
        sh = slot_h.numpy().reshape(self.K, self.max_req)
        sh[:, :n] = sl
        s = stream or self.torch.cuda.current_stream()
        with self.torch.cuda.stream(s):
            self.mask_d[:n].copy_(mask_h[:n], non_blocking=True)
            # the whole [K, max_req] block: one contiguous DMA (a strided [:, :n]
            # slice made torch launch an elementwise copy kernel on every pass)
            self.slot_d.copy_(slot_h, non_blocking=True)
            ev.record(s)

    # -- device pass ------------------------------------------------------
    def _compact(self, n: int):
        L = dv.lib()
        dv.check(L.ms_compact(self.mask_d.data_ptr(), n, self.K, self._X, self._ROWS,
                              self.slot_d.data_ptr(), self._G, self.idx.data_ptr(),
                              self.inv.data_ptr(), self.counts.data_ptr(), self.offs.data_ptr(),
                              self.perm.data_ptr(), dv.stream_ptr()), "ms_compact")

    def _compact_ring(self, n: int, mask_ptr: int, bases, parity: int = 0, stream=None, stream_p=None):
        """Compaction of a pass whose masks are already on the device
        (``mask_ptr``), modality k's compacted rows read from the pool ring
        at ``bases[k]`` (ms_compact_ring), index outputs of ``parity``."""
        import ctypes
        L = dv.lib()
        rb = (ctypes.c_int32 * self.K)(*[int(b) for b in bases])
        idx, inv, counts, offs, perm = self._ix[parity]
        dv.check(L.ms_compact_ring(mask_ptr, n, self.K, self._X, self._ROWS, rb, self.n_slots, self._G,
                                   idx.data_ptr(), inv.data_ptr(), counts.data_ptr(), offs.data_ptr(),
                                   perm.data_ptr(), stream_p if stream_p is not None else dv.stream_ptr(stream)),
                 "ms_compact_ring")

    def _head(self, n: int, parity: int = 0):
        inv = self._ix[parity][1][: self.K * n].view(self.K, n)
        return self.head.program(n, [e.outs[parity] if hasattr(e, "outs") else e.out for e in self.encoders], inv)

    def _launch(self, n: int, counts):
        """All kernels of one pass for a staged batch of n requests, eagerly."""
        self._compact(n)
        for enc, nk in zip(self.encoders, counts):
            if nk:
                enc.program(nk).run()
        self._head(n).run()

    def launches_per_pass(self, counts) -> int:
        n = 1 + sum(1 for c in counts if c)  # index kernel + one gather per present modality
        n += sum(e.program(c).n_launches for e, c in zip(self.encoders, counts) if c)
        return n + 2

    def _graph(self, key, fn):
        """CUDA graph of ``fn``'s launches, captured on first use."""
        g = self._graphs.get(key)
        if g is None:
            torch = self.torch
            torch.cuda.synchronize()  # the warm run shares activation buffers with in-flight passes
            fn()  # warm: builds plans and tensor maps outside capture
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    fn()
            torch.cuda.current_stream().wait_stream(s)
            self._graphs[key] = g
            self._gexec[key] = g.raw_cuda_graph_exec()
        return g

    def _exec(self, key, make_fn):
        """The instantiated graph (cudaGraphExec_t) of ``key``, captured from
        ``make_fn()``'s launches on first use -- launched by the serving paths
        with ms_graph_launch on a raw stream (no framework stream switching)."""
        e = self._gexec.get(key)
        if e is None:
            self._graph(key, make_fn())
            e = self._gexec[key]
        return e

    def ring_upload(self, host_pools, counts, bases, stream):
        """Host-IO path: DMA modality k's next ``counts[k]`` ring rows (from
        ``bases[k]``, wrapping) from the pinned host pools into the HBM pool
        on ``stream`` -- one copy per modality (two on wrap-around).
        Returns the bytes moved."""
        torch = self.torch
        ns = self.n_slots
        moved = 0
        with torch.cuda.stream(stream):
            for k in range(self.K):
                c = int(counts[k])
                if not c:
                    continue
                r0 = int(bases[k])
                first = min(c, ns - r0)
                self.pools[k][r0:r0 + first].copy_(host_pools[k][r0:r0 + first], non_blocking=True)
                if first < c:
                    self.pools[k][: c - first].copy_(host_pools[k][: c - first], non_blocking=True)
                moved += c * self.row_bytes[k]
        return moved

    @property
    def pipelined(self) -> bool:
        """Consecutive device-formed passes overlap (run_ring_pipelined)."""
        return (self._pipeline and self.use_graphs and self.parallel_modalities
                and all(getattr(e, "supports_parity", False) for e in self.encoders))

    def run_ring(self, n: int, counts, slot: int, bases, upload_ev=None):
        """One pass formed on the device: masks in ``mask_ring[slot]``
        (written by ms_pass_select), pool rows from the per-modality rings
        at ``bases``; ``ring_ev[slot]`` marks the row free again."""
        ptr = self.mask_ring[slot].data_ptr()
        if self.pipelined:
            self.run_ring_pipelined(n, counts, slot, bases, ptr, upload_ev)
            return

        def compact():
            self._compact_ring(n, ptr, bases)
            self.ring_ev[slot].record()
            self.ring_used[slot] = True

        self.run_staged(n, counts, compact=compact)

    def run_ring_pipelined(self, n: int, counts, slot: int, bases, mask_ptr: int, upload_ev=None):
        """Pass P+1 overlapping pass P.  Each modality's encoder always runs on
        its own stream (so P+1's encoder k follows P's encoder k), split into
        its stem graph (the only reader of the gathered input) and the rest;
        P+1's compaction runs on the compaction stream as soon as every
        modality's latest stem has consumed its input (and the pass's clips
        are uploaded), with index outputs and encoder features double-buffered
        by pass parity; only the fusion head runs on the calling stream, after
        its pass's encoders.  So P+1's gather overlaps P's encoders and P+1's
        encoders start while P's last layers and head still run."""
        par = self._parity
        self._parity ^= 1
        main_p = dv.stream_ptr()
        cs_p = self._cstream_p
        for ev in self._nev_stem:  # every gathered input consumed by its stem
            dv.stream_wait(cs_p, ev)
        if upload_ev is not None:
            dv.stream_wait(cs_p, upload_ev)
        self._compact_ring(n, mask_ptr, bases, parity=par, stream_p=cs_p)
        self._nev_cpar[par].record_on(cs_p)
        self.ring_ev[slot].record(self._cstream)
        self.ring_used[slot] = True
        present = [k for k, nk in enumerate(counts) if nk]
        # the encoders of a multi-modality pass share the GPU: their "rest"
        # graphs come from the shared plans (encoders.BNInception.program)
        sh = len(present) > 1
        for k in present:
            nk = counts[k]
            enc = self.encoders[k]
            shk = sh and getattr(enc, "supports_shared", False)
            ga = self._exec(("stem", k, nk, par), lambda: enc.program(nk, par).first().run)
            gb = self._exec(("rest", k, nk, par, shk), lambda: enc.program(nk, par, shared=True).tail().run
                            if shk else enc.program(nk, par).tail().run)
            sp = self._side_p[k]
            dv.stream_wait(sp, self._nev_cpar[par])
            dv.graph_launch(ga, sp)
            self._nev_stem[k].record_on(sp)
            dv.graph_launch(gb, sp)
            self._nev_k[k].record_on(sp)
        for k in present:
            dv.stream_wait(main_p, self._nev_k[k])
        dv.graph_launch(self._exec(("head", n, par), lambda: self._head(n, par).run), main_p)

    def run_staged(self, n: int, counts, compact=None):
        """Compaction (direct launches), then one graph per present
        modality's encoder (keyed by its compacted count) and one for the
        fusion head (keyed by n): O(K * max_req) captures in total."""
        if compact is None:
            compact = lambda: self._compact(n)  # noqa: E731
        if not self.use_graphs:
            compact()
            for enc, nk in zip(self.encoders, counts):
                if nk:
                    enc.program(nk).run()
            self._head(n).run()
            return
        compact()
        main_p = dv.stream_ptr()
        present = [k for k, nk in enumerate(counts) if nk]
        execs = [self._exec(("enc", k, counts[k]), lambda k=k: self.encoders[k].program(counts[k]).run)
                 for k in present]
        head = self._exec(("head", n), lambda: self._head(n).run)
        if not self.parallel_modalities or len(present) < 2:
            for e in execs:
                dv.graph_launch(e, main_p)
        else:
            # independent encoders run concurrently: fork after compaction,
            # join before the fusion head
            self._nev_c.record_on(main_p)
            for k, e in zip(present, execs):
                sp = self._side_p[k]
                dv.stream_wait(sp, self._nev_c)
                dv.graph_launch(e, sp)
                self._nev_k[k].record_on(sp)
            for k in present:
                dv.stream_wait(main_p, self._nev_k[k])
        dv.graph_launch(head, main_p)

    def ensure_warm(self, max_n: int | None = None):
        """warm_graphs once per model (a graph captured lazily while passes are
        in flight costs a device sync + capture: milliseconds of serving)."""
        top = min(max_n or self.max_req, self.max_req)
        if getattr(self, "_warm_top", 0) < top:
            self.warm_graphs(top)

    def warm_graphs(self, max_n: int | None = None):
        """Capture every encoder/head graph up to ``max_n`` requests."""
        top = min(max_n or self.max_req, self.max_req)
        self._warm_top = max(getattr(self, "_warm_top", 0), top)
        for k, enc in enumerate(self.encoders):
            for nk in range(1, top + 1):
                self._graph(("enc", k, nk), enc.program(nk).run)
        for n in range(1, top + 1):
            self._graph(("head", n), self._head(n).run)
        if self.pipelined:  # run_ring_pipelined's stem / rest / head graphs, both parities
            for par in (0, 1):
                for k, enc in enumerate(self.encoders):
                    for nk in range(1, top + 1):
                        sp = enc.program(nk, par)
                        self._graph(("stem", k, nk, par), sp.first().run)
                        self._graph(("rest", k, nk, par, False), sp.tail().run)
                        if getattr(enc, "supports_shared", False) and self.K > 1:
                            self._graph(("rest", k, nk, par, True), enc.program(nk, par, shared=True).tail().run)
                for n in range(1, top + 1):
                    self._graph(("head", n, par), self._head(n, par).run)
        self.torch.cuda.synchronize()

    def forward(self, slots, masks):
        """One masked pass; returns the logits view [N, 397] (async).
        ``slots``: pool row per request ([N]) or per modality and request ([K, N])."""
        masks = np.asarray(masks)
        n = len(masks)
        counts = self.counts_for(masks)
        self.stage_inputs(slots, masks)
        self.run_staged(n, counts)
        return self.head.logits[:n]

    def flops(self, masks) -> int:
        return self.flops_counts(self.counts_for(np.asarray(masks)), len(masks))

    def flops_counts(self, counts, n: int) -> int:
        """Algorithmic FLOP of one pass: every present modality's encoder over
        its compacted count (real channels) + the fusion head over n."""
        return sum(e.flops(c) for e, c in zip(self.encoders, counts) if c) + self.head.flops(n)

    def compaction_bytes_rw(self, masks):
        """(bytes read, bytes written) of compaction_bytes: the rows read with
        the masks and the index reads; the padded rows and index lists written."""
        counts = self.counts_for(np.asarray(masks))
        dst_lines = [r[0] + (r[0] // r[8]) * 2 * r[9] if r[8] and r[9] else r[0] for r in self.rows]
        rd = sum(rb * c for rb, c in zip(self.row_bytes, counts)) + 2 * len(masks)
        wr = sum(2 * dl * (r[1] + 2 * r[4]) * r[3] * c for r, dl, c in zip(self.rows, dst_lines, counts))
        return rd, wr + 4 * sum(counts)

    def compaction_bytes(self, masks) -> int:
        """per present (request, modality) the row read (real
        channels) + written (padded channels), + 2N mask bytes + 4*sum N_k
        index bytes."""
        counts = self.counts_for(np.asarray(masks))
        # written lines include the frame row padding (MsRowDesc frame_h / pad_h)
        dst_lines = [r[0] + (r[0] // r[8]) * 2 * r[9] if r[8] and r[9] else r[0] for r in self.rows]
        rows = sum((rb + 2 * dl * (r[1] + 2 * r[4]) * r[3]) * c
                   for r, rb, dl, c in zip(self.rows, self.row_bytes, dst_lines, counts))
        return rows + 2 * len(masks) + 4 * sum(counts)


def build_tbn_model(max_req: int, n_slots: int, seeds=(101, 102, 103), fusion_seed: int = 199,
                    segments: int = SEGMENTS, device="cuda", data_seed: int = 0) -> MaskedModel:
    """configs[1]: TBN-shaped rgb/flow/audio BN-Inception encoders over
    EPIC-shaped synthetic clips resident in HBM (N(0,1), bf16)."""
    import torch
    encs = [BNInceptionEncoder(m, max_req, s, segments, device) for m, s in zip(TBN_MODALITIES, seeds)]
    head = FusionHead(len(encs), max_req, fusion_seed, FEAT_DIM, device)
    g = torch.Generator(device=device)
    g.manual_seed(data_seed)
    pools, rows = [], []
    for m in TBN_MODALITIES:
        # compact NHWC (real channels); the compaction gather pads to m.cpad.
        # rgb frames and (TSN-style quantised) flow are uint8 and converted to
        # bf16 (u8/64 - 2, exact in bf16) by the gather; audio spectrograms bf16
        shape = (n_slots, segments, m.size, m.size, m.channels)
        if m.uint8:
            pools.append(torch.randint(0, 256, shape, generator=g, device=device, dtype=torch.uint8))
            rows.append((segments * m.size, m.size, m.channels, m.cpad, CONV1_PAD, 1, U8_SCALE, U8_BIAS,
                         m.size, m.row_pad))
        else:
            pools.append(torch.randn(shape, generator=g, device=device).to(torch.bfloat16))
            rows.append((segments * m.size, m.size, m.channels, m.cpad, CONV1_PAD, 0, 1.0, 0.0, m.size,
                         m.row_pad))
    return MaskedModel(encs, head, pools, rows, max_req, device)


def build_mlp_model(in_dims, max_req: int, n_slots: int, seeds=(201, 202, 203),
                    fusion_seed: int = 299, device="cuda", data_seed: int = 0) -> MaskedModel:
    """configs[0]: small per-modality MLP towers with the same fusion head."""
    import torch
    encs = [MLPEncoder(d, max_req, s, device=device) for d, s in zip(in_dims, seeds)]
    head = FusionHead(len(encs), max_req, fusion_seed, FEAT_DIM, device)
    g = torch.Generator(device=device)
    g.manual_seed(data_seed)
    pools, rows = [], []
    for e, d in zip(encs, in_dims):
        width = e.x.shape[1]
        p = torch.zeros(n_slots, width, dtype=torch.bfloat16, device=device)
        p[:, :d] = torch.randn(n_slots, d, generator=g, device=device).to(torch.bfloat16)
        pools.append(p)
        rows.append((1, 1, width, width, 0))
    return MaskedModel(encs, head, pools, rows, max_req, device)


class DeviceExecutor:
    """Serving-loop worker seam backed by the GPU.

    ``timing="virtual"``: the device pass runs but each part still takes
    ``max(1, round(predicted * d))`` (reference sim.py:375) so run() logs are
    bit-identical to the reference.  ``timing="measured"``: the job's pass is
    timed with CUDA events and that time is attributed to its parts in
    proportion to their predicted latency; those observations feed the
    latency-feedback EWMA (scheduler.py:86-91).
    """

    def __init__(self, model: MaskedModel, timing: str = "measured", slot_seed: int = 0, record: int = 0):
        """``record``: keep (job id, assigned credit, masks, slots) of every
        pass and the logits of the first ``record`` passes in ``trace``."""
        if timing not in ("virtual", "measured"):
            raise ValueError("timing must be 'virtual' or 'measured'")
        self.model = model
        self.record = record
        self.trace = [] if record else None
        self.timing = timing
        self.rng = np.random.default_rng(slot_seed)
        self.ev0, self.ev1 = dv.Event(), dv.Event()
        self.passes = 0
        self.requests = 0
        self.device_us = 0.0
        self.last_logits = None

    def execute(self, job, profile, discrepancy: float, now_us: int):
        parts = job.assigned.strategy.parts
        masks = request_masks(parts, job.size)
        slots = self.rng.integers(0, self.model.n_slots, size=job.size)
        self.ev0.record()
        logits = self.model.forward(slots, masks)
        self.ev1.record()
        us = self.ev0.elapsed_us(self.ev1)  # synchronises on the pass
        self.passes += 1
        self.requests += job.size
        self.device_us += us
        self.last_logits = logits
        if self.trace is not None:
            keep = logits[: job.size].float().cpu() if len(self.trace) < self.record else None
            self.trace.append((job.id, job.assigned.credit, masks.copy(), slots.copy(), keep))
        preds = [profile.part_latency_us(m, b) for m, b in parts]
        if self.timing == "virtual":
            return [(p, max(1, round(p * discrepancy))) for p in preds]
        total = max(1, int(round(us)))
        tot_pred = sum(preds)
        out, used = [], 0
        for i, p in enumerate(preds):
            a = total - used if i == len(preds) - 1 else max(1, int(round(total * p / tot_pred)))
            a = max(1, a)
            used += a
            out.append((p, a))
        return out
