"""Mixed-size codeword batches (transport-block segmentation) as one CUDA graph.

A 5G uplink slot carries codewords of several (graph, Z, rows_used) shapes.
Each shape needs its own plan, so a mixed batch is one kernel launch per
shape. Issued from Python, those launches are
host-bound: about 20 µs of launch overhead each against kernels of ~100 µs.
``MixedBatchDecoder`` fixes this. It allocates static device buffers per
group and captures all launches once into a CUDA graph, fanned out over
side streams so independent groups run concurrently on the SMs. Each
``decode()`` then replays the graph: one host call for the whole batch.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .decoder import INT8_SAT, DecodeConfig, DecodeResult, get_plan, unpack_bits


@dataclass
class Group:
    bg: object
    rows_used: int
    batch: int


class MixedBatchDecoder:
    def __init__(self, groups: list[Group], cfg: DecodeConfig, streams: int = 16, device: int = 0):
        import torch

        self.cfg = cfg
        self.groups = groups
        # plans tuned for sharing SMs with each other's launches
        self.plans = [get_plan(g.bg, g.rows_used, cfg, device, coscheduled=True) for g in groups]
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
        self._streams = [torch.cuda.Stream(device=dev) for _ in range(max(1, streams))]
        self._order = self._schedule(len(self._streams))
        self._graph = None
        self._device = dev

    def _schedule(self, n_streams: int) -> list[tuple[int, int]]:
        """Longest-first list scheduling of the groups onto the side streams.

        A group's kernel runs ceil(batch / codewords_per_cta) CTAs whose
        duration grows with the edges each thread walks per iteration and
        the CTA's warp count. The longest groups are launched first and each
        goes to the stream with the least queued work, so the longest
        kernels are not stuck behind short ones in launch order."""
        sms = 148
        costs = []
        for g, p in zip(self.groups, self.plans):
            ctas = -(-g.batch // max(1, p.codewords_per_cta))
            warps = -(-p.threads_per_cta // 32)
            per_cta = p.tables.n_edges * (1.0 + 0.05 * warps)
            costs.append(per_cta * -(-ctas // sms))
        queued = [0.0] * n_streams
        order = []
        for i in sorted(range(len(costs)), key=lambda i: -costs[i]):
            s = min(range(n_streams), key=lambda k: queued[k])
            queued[s] += costs[i]
            order.append((i, s))
        return order

    def _launch_all(self):
        import torch
        cur = torch.cuda.current_stream(self._device)
        # the status word (int8 -128 seen) restarts at zero on every replay
        self._status.zero_()
        for s in self._streams:
            s.wait_stream(cur)
        for i, si in self._order:
            self.plans[i].decode_device(self.inputs[i], self.outputs[i], stream=self._streams[si].cuda_stream)
        for s in self._streams:
            cur.wait_stream(s)

    def describe(self) -> str:
        return (f"one CUDA-graph replay: {len(self.plans)} per-shape launches over "
                f"{len(self._streams)} streams (longest first)")

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
        results = []
        if int(self._status.item()):  # synchronizes with the replay
            raise ValueError("int8 LLR magnitudes must be at most 127")
        for plan, out in zip(self.plans, self.outputs):
            h = {k: v.cpu().numpy() for k, v in out.items() if k in ("bits", "iters", "synd", "success", "crc_ok")}
            results.append(DecodeResult(
                bits=unpack_bits(h["bits"], plan.k), iterations=h["iters"].astype(np.int64),
                success=h["success"].astype(bool), syndrome_weight=h["synd"].astype(np.int64),
                crc_ok=h["crc_ok"].astype(bool) if self.cfg.early_stop.value == "crc" else None))
        return results
