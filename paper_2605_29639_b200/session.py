"""Host-side decode-step runtime: one attention layer's decode step for a fixed
batch, from pinned host buffers to pinned host buffers.

    sess = DecodeSession(cache, block_table, batch=B, num_q_heads=Hq)
    sess.submit(q_h, k_h, v_h, slots_h, lens_h, out_h)   # async, returns an event
    ...
    sess.synchronize()

Each step uploads its inputs (q, the new K/V rows, slot mapping, sequence
lengths) on a copy stream, runs K1 (quantize-on-append) + K2 (paged decode
attention) on the compute stream and downloads the output on a second copy
stream.  Device buffers are double-buffered, so step i+1's uploads and step
i-1's download overlap step i's kernels; stream-ordering events make every
reuse safe.  This is the serving-loop counterpart of the reference's
``_on_decode_step`` (simulator.py:504-517), with the KV write of the decoded
token that the reference never models.

``capture()`` returns CUDA graphs of the device part of one step (K1, K2) over
the session's own device buffers, for launch-bound small batches.
"""
from __future__ import annotations

from typing import List, Optional

import torch

from . import _lib
from .cache import PagedKVCache
from .ops import (decode_step, paged_decode_attention, paged_decode_attention_gathered, quantize_append,
                  workspace_bytes)


class DecodeSession:
    def __init__(self, cache: PagedKVCache, block_table: torch.Tensor, batch: int, num_q_heads: int,
                 *, total_pages: Optional[int] = None, out_dtype: torch.dtype = torch.bfloat16,
                 head_major: bool = False, sm_scale: Optional[float] = None, depth: int = 2,
                 gather_factory=None, pages_per_split: Optional[int] = None, graphs: bool = False,
                 peer=None, append_tail_only: bool = False, fused_append: bool = False):
        """With ``gather_factory`` (returning a
        :class:`paper_2605_29639_b200.shard.OutputGather`, one per buffer slot,
        for KV-head / 2-D sharding) the local head-major output
        ``[Hq_loc, B_r, d]`` is assembled into ``[Hq, B, d]`` on the compute
        stream before the download.

        With ``peer`` (a :class:`paper_2605_29639_b200.shard.PeerOutput`
        with ``slots >= depth``) the gather is fused into K2 instead: each
        buffer slot's K2 stores its rows into every rank's copy of the global
        output over peer memory, and the download reads the slot's copy.

        ``append_tail_only=True`` promises that each step's slots are the
        sequences' newest tokens (in their last page): K2 then streams every
        other page while K1 runs (``ops.decode_step``).  ``fused_append=True``
        makes the same promise with one row per sequence (row b = sequence b's
        newest token) and launches no K1 at all: K2 quantizes the rows itself
        (``KVQ_STEP_FUSED_APPEND``; ignored with ``peer``).

        With ``graphs=True`` each buffer slot's device work (K1, K2 and the
        gather) is captured once as a CUDA graph on first use and replayed by
        every later :meth:`submit`: one host call per step instead of one
        per kernel."""
        dev = cache.device
        self.peer = peer
        if peer is not None and (gather_factory is not None or peer.slots < depth):
            raise ValueError("DecodeSession: peer needs slots >= depth and no gather_factory")
        self.sharded = gather_factory is not None or peer is not None
        if self.sharded:
            head_major = True
        self.cache, self.block_table = cache, block_table
        self.B, self.Hq, self.Hkv = batch, num_q_heads, cache.spec.num_kv_heads
        self.head_major, self.sm_scale, self.out_dtype = head_major, sm_scale, out_dtype
        lib = _lib.load()
        max_blocks = block_table.shape[1]
        self.pps = int(pages_per_split or lib.kvq_decode_pages_per_split_rows(
            batch, self.Hkv, num_q_heads // self.Hkv,
            total_pages if total_pages is not None else batch * max_blocks, max_blocks))
        max_splits = -(-max_blocks // self.pps)
        self.depth = depth
        self.compute = torch.cuda.current_stream(dev)
        self.h2d = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        oshape = (num_q_heads, batch, 128) if head_major else (batch, num_q_heads, 128)
        # The step's inputs live in one packed blob per slot (q | k | v | slots |
        # lens, 16-byte aligned), mirrored by a pinned host staging blob, so a
        # staged step uploads with a single copy.
        shapes = (("q", (batch, num_q_heads, 128), torch.bfloat16), ("k", (batch, self.Hkv, 128), torch.bfloat16),
                  ("v", (batch, self.Hkv, 128), torch.bfloat16), ("slots", (batch,), torch.int32),
                  ("lens", (batch,), torch.int32))
        layout, off = [], 0
        for name, shape, dt in shapes:
            n = 1
            for x in shape:
                n *= x
            nbytes = n * torch.empty((), dtype=dt).element_size()
            layout.append((name, shape, dt, off, nbytes))
            off = (off + nbytes + 15) & ~15
        self.in_bytes = off
        pin = torch.cuda.is_available()

        def views(blob):
            return {name: blob[o: o + nb].view(dt).view(shape) for name, shape, dt, o, nb in layout}

        self.bufs = []
        for i in range(depth):
            dev_in = torch.empty(max(off, 16), dtype=torch.uint8, device=dev)
            host_in = torch.empty(max(off, 16), dtype=torch.uint8, pin_memory=pin)
            self.bufs.append(dict(
                **views(dev_in), dev_in=dev_in, host_in=host_in, host=views(host_in),
                out=torch.empty(oshape, dtype=out_dtype, device=dev),
                ws=torch.zeros(workspace_bytes(batch, num_q_heads, self.Hkv, max_splits),
                               dtype=torch.uint8, device=dev),
                in_ready=torch.cuda.Event(), done=torch.cuda.Event(), out_done=torch.cuda.Event(),
                gather=gather_factory() if gather_factory is not None else None, used=False, idx=i))
        self.step_idx = 0
        self.graphs = graphs
        self.append_tail_only = append_tail_only
        self.fused_append = fused_append and peer is None

    def k1(self, buf) -> None:
        """Quantize-on-append of the step's new K/V rows (device buffers)."""
        quantize_append(self.cache, buf["k"], buf["v"], buf["slots"])

    def k2(self, buf) -> None:
        """Paged decode attention over the cache into ``buf["out"]`` (or, with
        ``peer``, into every rank's copy of the slot's global output)."""
        if self.peer is not None:
            paged_decode_attention_gathered(buf["q"], self.cache, self.block_table, buf["lens"], self.peer,
                                            buf["idx"], sm_scale=self.sm_scale, pages_per_split=self.pps,
                                            workspace=buf["ws"])
            return
        paged_decode_attention(buf["q"], self.cache, self.block_table, buf["lens"], out=buf["out"],
                               head_major=self.head_major, sm_scale=self.sm_scale,
                               pages_per_split=self.pps, out_dtype=self.out_dtype,
                               workspace=buf["ws"])

    def step(self, buf) -> None:
        """K1 + K2 of one step in one call (``kvq_decode_step``: K2's launch and
        prologue overlap K1 through programmatic dependent launch)."""
        decode_step(self.cache, buf["k"], buf["v"], buf["slots"], buf["q"], self.block_table, buf["lens"],
                    sm_scale=self.sm_scale, pages_per_split=self.pps, out=buf["out"],
                    out_dtype=self.out_dtype, head_major=self.head_major, workspace=buf["ws"],
                    peer=self.peer, slot=buf["idx"], append_tail_only=self.append_tail_only,
                    fused_append=self.fused_append)

    def _kernels(self, buf, k1: bool = True) -> None:
        if k1:
            self.step(buf)
        else:
            self.k2(buf)

    def submit(self, q_h: torch.Tensor, k_h: torch.Tensor, v_h: torch.Tensor, slots_h: torch.Tensor,
               lens_h: torch.Tensor, out_h: torch.Tensor) -> torch.cuda.Event:
        """Enqueue one decode step.  Host tensors should be pinned; they must
        stay untouched until the returned event completes."""
        return self._submit((q_h, k_h, v_h, slots_h, lens_h), out_h)

    def _submit(self, inputs, out_h: torch.Tensor) -> torch.cuda.Event:
        buf = self.bufs[self.step_idx % self.depth]
        self.step_idx += 1
        if inputs is None and buf.get("graph") is not None and out_h.is_pinned() and out_h.is_contiguous():
            return self._submit_native(buf, out_h)
        with torch.cuda.stream(self.h2d):
            if buf["used"]:
                self.h2d.wait_event(buf["done"])      # previous kernels finished reading
            if inputs is None:
                buf["dev_in"].copy_(buf["host_in"], non_blocking=True)
            else:
                for name, t in zip(("q", "k", "v", "slots", "lens"), inputs):
                    buf[name].copy_(t, non_blocking=True)
            buf["in_ready"].record(self.h2d)
        self.compute.wait_event(buf["in_ready"])
        if buf["used"]:
            self.compute.wait_event(buf["out_done"])   # previous download of this out buffer
        with torch.cuda.stream(self.compute):
            full = self._device_step(buf)
        buf["done"].record(self.compute)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(buf["done"])
            out_h.copy_(full, non_blocking=True)
            buf["out_done"].record(self.d2h)
        buf["used"] = True
        return buf["out_done"]

    def _submit_native(self, buf, out_h: torch.Tensor) -> torch.cuda.Event:
        """A staged step whose slot graph exists: upload, graph launch and
        download are enqueued by one native call (``kvq_pipeline_submit``)."""
        import ctypes
        full = buf["graph_out"]
        nbytes = full.numel() * full.element_size()
        if out_h.numel() * out_h.element_size() != nbytes:
            raise ValueError(f"submit: out_h must hold {nbytes} bytes")
        st = buf.get("pipe")
        if st is None:
            st = _lib.PipeStep()
            st.h2d_stream, st.compute_stream = self.h2d.cuda_stream, self.compute.cuda_stream
            st.d2h_stream = self.d2h.cuda_stream
            st.graph_exec = buf["graph"].raw_cuda_graph_exec()
            st.dev_in, st.host_in, st.in_bytes = buf["dev_in"].data_ptr(), buf["host_in"].data_ptr(), self.in_bytes
            st.dev_out, st.out_bytes = full.data_ptr(), nbytes
            st.ev_in_ready, st.ev_done = buf["in_ready"].cuda_event, buf["done"].cuda_event
            st.ev_out_done = buf["out_done"].cuda_event
            buf["pipe"] = st
        st.host_out = out_h.data_ptr()
        st.reuse = 1 if buf["used"] else 0
        _lib.check("kvq_pipeline_submit", _lib.load().kvq_pipeline_submit(ctypes.byref(st)))
        buf["used"] = True
        return buf["out_done"]

    def next_inputs(self) -> dict:
        """Pinned host views ``{q, k, v, slots, lens}`` of the staging blob the
        next :meth:`submit_staged` uploads.  Waits (host side) until that
        slot's previous upload has finished, so the views may be overwritten."""
        buf = self.bufs[self.step_idx % self.depth]
        if buf["used"]:
            buf["in_ready"].synchronize()
        return buf["host"]

    def submit_staged(self, out_h: torch.Tensor) -> torch.cuda.Event:
        """Enqueue one step whose inputs were written into :meth:`next_inputs`:
        one host-to-device copy, the device step, one device-to-host copy."""
        return self._submit(None, out_h)

    def _result(self, buf) -> torch.Tensor:
        if self.peer is not None:
            return self.peer.out(buf["idx"])
        return buf["gather"](buf["out"]) if buf["gather"] is not None else buf["out"]

    def _device_step(self, buf) -> torch.Tensor:
        if not self.graphs:
            self._kernels(buf)
            return self._result(buf)
        g = buf.get("graph")
        if g is None:
            # Warm once eagerly (module load, NCCL communicator), then capture.
            self._kernels(buf)
            full = self._result(buf)
            self.compute.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=torch.cuda.Stream(self.cache.device)):
                self._kernels(buf)
                full = self._result(buf)
            buf["graph"], buf["graph_out"] = g, full
        buf["graph"].replay()
        return buf["graph_out"]

    def synchronize(self) -> None:
        for s in (self.h2d, self.compute, self.d2h):
            s.synchronize()

    def capture(self) -> List[torch.cuda.CUDAGraph]:
        """CUDA graphs [K1, K2] of one step over device buffer 0's contents."""
        buf = self.bufs[0]
        graphs = []
        for fn in (lambda: self.k1(buf), lambda: self.k2(buf)):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            graphs.append(g)
        return graphs

    def device_buffers(self, i: int = 0) -> dict:
        return self.bufs[i]
