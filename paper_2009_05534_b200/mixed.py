"""Mixed-size codeword batches (transport-block segmentation) in one replay.

A 5G uplink slot carries codewords of several (graph, Z, rows_used) shapes.
Each shape needs its own plan (graph tables, layout), so a mixed batch is
one decode per shape. ``MixedBatchDecoder``
allocates static device buffers per group and captures the whole batch once
into a CUDA graph; ``decode()`` then replays it, one host call for the batch.

Grouped launches (default): int8 groups whose plans share a kernel variant
and CTA size go into one multi-shape launch of up to five shapes
(``nrldpc_decode_multi``; each shape's tables ride in the launch's parameter
block). A mixed batch of many small shapes is limited by how many kernels a
replay runs concurrently (about 32 measured, tools/cfg4_probe.py), not by
their work: the 102 groups of config 4 become ~25 launches. The launches are
fanned out over side streams, longest first, so they run concurrently on the
SMs. ``grouped=False`` keeps one launch per group (float precisions always).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .decoder import INT8_SAT, DecodeConfig, DecodeResult, get_plan, unpack_bits


@dataclass
class Group:
    bg: object
    rows_used: int
    batch: int


class MixedBatchDecoder:
    def __init__(self, groups: list[Group], cfg: DecodeConfig, streams: int = 16, device: int = 0,
                 grouped: bool = True, coscheduled: bool = True):
        import torch

        self.cfg = cfg
        self.groups = groups
        # plans tuned for sharing SMs with each other's launches
        self.plans = [get_plan(g.bg, g.rows_used, cfg, device, coscheduled=coscheduled) for g in groups]
        dev = torch.device("cuda", device)
        dtype = {"int8": torch.int8, "f16": torch.float16, "f32": torch.float32}[cfg.precision.value]
        # static buffers: callers fill .inputs[i] (or pass arrays to decode())
        self.inputs = [torch.zeros((g.batch, p.n_c), dtype=dtype, device=dev)
                       for g, p in zip(groups, self.plans)]
        self.outputs = [p.alloc_outputs(g.batch) for g, p in zip(groups, self.plans)]
        # one status word for the whole batch (any group's int8 -128 flags it):
        # a single memset per replay instead of one per group
        self._status = torch.zeros(1, dtype=torch.int32, device=dev)
        for out in self.outputs:
            out["status"] = self._status
        self.grouped = bool(grouped) and cfg.precision.value == "int8"
        self.launches = self._pack() if self.grouped else [[i] for i in range(len(groups))]
        self._streams = [torch.cuda.Stream(device=dev) for _ in range(max(1, streams))]
        self._order = self._schedule(len(self._streams))
        self._args = [self._multi_args(lg) for lg in self.launches] if self.grouped else None
        self._graph = None
        self._device = dev

    # -- grouping ------------------------------------------------------------
    def _kernel_key(self, plan) -> tuple[int, int, int]:
        k, t, sm = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        _native.check(_native.load().nrldpc_plan_kernel(plan.handle, ctypes.byref(k), ctypes.byref(t),
                                                        ctypes.byref(sm)))
        return k.value, t.value, sm.value

    def _pack(self) -> list[list[int]]:
        """Groups -> launches: same (kernel variant, CTA size), at most
        MULTI_MAX shapes each, shapes of similar shared-memory size together
        (a launch requests the largest)."""
        keys = [self._kernel_key(p) for p in self.plans]
        by_key: dict = {}
        for i, (k, t, sm) in enumerate(keys):
            by_key.setdefault((k, t), []).append(i)
        launches = []
        for members in by_key.values():
            members.sort(key=lambda i: keys[i][2])
            for j in range(0, len(members), _native.MULTI_MAX):
                launches.append(members[j:j + _native.MULTI_MAX])
        return launches

    def _group_cost(self, i: int) -> float:
        g, p = self.groups[i], self.plans[i]
        ctas = -(-g.batch // max(1, p.codewords_per_cta))
        warps = -(-p.threads_per_cta // 32)
        per_cta = p.tables.n_edges * (1.0 + 0.05 * warps)
        return per_cta * -(-ctas // 148)

    def _schedule(self, n_streams: int) -> list[tuple[int, int]]:
        """Longest-first list scheduling of the launches onto the side streams.

        A launch runs its CTAs, whose duration grows with the edges each
        thread walks per iteration and the CTA's warp count. The longest
        launches go first, each to the stream with the least queued work, so
        the longest kernels are not stuck behind short ones."""
        costs = [max(self._group_cost(i) for i in lg) for lg in self.launches]
        queued = [0.0] * n_streams
        order = []
        for li in sorted(range(len(costs)), key=lambda i: -costs[i]):
            s = min(range(n_streams), key=lambda k: queued[k])
            queued[s] += costs[li]
            order.append((li, s))
        return order

    def _multi_args(self, members: list[int]):
        n = len(members)
        P = ctypes.c_void_p * n
        outs = [self.outputs[i] for i in members]
        crc = self.cfg.early_stop.value == "crc"
        return (
            (ctypes.c_void_p * n)(*[self.plans[i].handle.value for i in members]), n,
            P(*[self.inputs[i].data_ptr() for i in members]),
            (ctypes.c_int64 * n)(*[self.groups[i].batch for i in members]),
            P(*[o["bits"].data_ptr() for o in outs]), P(*[o["iters"].data_ptr() for o in outs]),
            P(*[o["synd"].data_ptr() for o in outs]), P(*[o["success"].data_ptr() for o in outs]),
            P(*[o["crc_ok"].data_ptr() for o in outs]) if crc else None,
            self._status.data_ptr())

    def describe(self) -> str:
        if self.grouped:
            return (f"one CUDA-graph replay: {len(self.plans)} shapes in {len(self.launches)} multi-shape "
                    f"launches (nrldpc_decode_multi, same kernel variant and CTA size per launch) over "
                    f"{len(self._streams)} streams, longest first")
        return (f"one CUDA-graph replay: {len(self.plans)} per-shape launches over "
                f"{len(self._streams)} streams (longest first)")

    # -- launch / replay ------------------------------------------------------
    def _launch_all(self):
        import torch
        cur = torch.cuda.current_stream(self._device)
        # the status word (int8 -128 seen) restarts at zero on every replay
        self._status.zero_()
        for s in self._streams:
            s.wait_stream(cur)
        lib = _native.load()
        for li, si in self._order:
            st = self._streams[si].cuda_stream
            if self.grouped:
                _native.check(lib.nrldpc_decode_multi(*self._args[li], st))
            else:
                i = self.launches[li][0]
                self.plans[i].decode_device(self.inputs[i], self.outputs[i], stream=st)
        for s in self._streams:
            cur.wait_stream(s)

    def capture(self):
        import torch
        self._launch_all()                      # warm-up: kernel attributes, lazy init
        torch.cuda.synchronize(self._device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._launch_all()
        self._graph = g
        return self

    def replay(self):
        """Decode whatever is in ``self.inputs`` (asynchronous)."""
        if self._graph is None:
            self.capture()
        self._graph.replay()

    def decode(self, llrs: list) -> list[DecodeResult]:
        """Host arrays (or tensors) in, one DecodeResult per group out.

        Inputs are validated like ``decode`` (decoder.py:287-288): a wider
        integer input outside [-127, 127] raises before anything runs, and an
        int8 -128 is flagged by the kernels and raises after the replay."""
        import torch
        if len(llrs) != len(self.inputs):
            raise ValueError(f"expected {len(self.inputs)} groups, got {len(llrs)}")
        int8 = self.cfg.precision.value == "int8"
        for x, src in zip(self.inputs, llrs):
            t = src if isinstance(src, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(src))
            if tuple(t.shape) != tuple(x.shape):
                raise ValueError(f"group input shape {tuple(t.shape)} != {tuple(x.shape)}")
            if int8 and t.dtype != torch.int8:
                wide = t.to(torch.int32)  # astype semantics, decoder.py:286
                if wide.numel() and int(wide.abs().max()) > INT8_SAT:
                    raise ValueError("int8 LLR magnitudes must be at most 127")
                t = wide
            x.copy_(t)
        self.replay()
        if int(self._status.item()):  # synchronizes with the replay
            raise ValueError("int8 LLR magnitudes must be at most 127")
        results = []
        for plan, out in zip(self.plans, self.outputs):
            h = {k: v.cpu().numpy() for k, v in out.items() if k in ("bits", "iters", "synd", "success", "crc_ok")}
            results.append(DecodeResult(
                bits=unpack_bits(h["bits"], plan.k), iterations=h["iters"].astype(np.int64),
                success=h["success"].astype(bool), syndrome_weight=h["synd"].astype(np.int64),
                crc_ok=h["crc_ok"].astype(bool) if self.cfg.early_stop.value == "crc" else None))
        return results
