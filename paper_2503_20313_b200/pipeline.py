"""Host-resident activations through the TP-MLP layer with copy/compute overlap.

`MLPPipeline.run` streams a sequence of pinned host X shards through `tl_mlp_forward`: the
host->device copy of batch i+1 and the device->host copy of batch i-1 run on their own CUDA
streams while batch i computes, so a serving loop pays max(PCIe in, compute, PCIe out) per
batch instead of their sum.  Plumbing only (streams, events, buffers); the layer itself is the
library's two kernels.
"""
from __future__ import annotations

import torch


class MLPPipeline:
    def __init__(self, comm, W1, W2, act: int, M_r: int, H: int, depth: int = 2):
        self.comm, self.W1, self.W2, self.act, self.depth = comm, W1, W2, act, depth
        dev = W1.device
        I_l = W2.shape[1]
        M = M_r * comm.world
        self.x = [torch.empty(M_r, H, device=dev, dtype=torch.bfloat16) for _ in range(depth)]
        self.out = [torch.empty(M_r, H, device=dev, dtype=torch.bfloat16) for _ in range(depth)]
        self.Z = torch.empty(M, I_l, device=dev, dtype=torch.bfloat16)
        self.s_in, self.s_comp, self.s_out = (torch.cuda.Stream(dev) for _ in range(3))
        mk = lambda: [torch.cuda.Event() for _ in range(depth)]
        self.ev_in, self.ev_comp, self.ev_out = mk(), mk(), mk()
        self.bytes_in = M_r * H * 2
        self.bytes_out = M_r * H * 2

    def run(self, host_x, host_out, start_event=None, end_event=None):
        """host_x / host_out: equal-length lists of pinned [M_r, H] bf16 CPU tensors."""
        d = self.depth
        if start_event is not None:
            start_event.record(self.s_in)
        for i, (xi, xo) in enumerate(zip(host_x, host_out)):
            b = i % d
            if i >= d:
                self.s_in.wait_event(self.ev_comp[b])      # compute(i-d) finished reading x[b]
            with torch.cuda.stream(self.s_in):
                self.x[b].copy_(xi, non_blocking=True)
            self.ev_in[b].record(self.s_in)
            self.s_comp.wait_event(self.ev_in[b])
            if i >= d:
                self.s_comp.wait_event(self.ev_out[b])     # D2H(i-d) finished reading out[b]
            self.comm.mlp_forward(self.x[b], self.W1, self.W2, self.out[b], act=self.act, Z=self.Z,
                                  stream=self.s_comp)
            self.ev_comp[b].record(self.s_comp)
            self.s_out.wait_event(self.ev_comp[b])
            with torch.cuda.stream(self.s_out):
                xo.copy_(self.out[b], non_blocking=True)
            self.ev_out[b].record(self.s_out)
        if end_event is not None:
            self.s_in.wait_stream(self.s_out)
            self.s_comp.wait_stream(self.s_out)
            end_event.record(self.s_out)
        return host_out


class StepPipeline:
    """Generic host-resident pipeline: each step copies its pinned host inputs to device buffers on an
    input stream, runs `fn(device_inputs, device_outputs, stream)` on a compute stream and copies the
    outputs back on an output stream; with `depth` buffer sets, the copies of neighbouring steps overlap
    the current step's kernels (as MLPPipeline, for any op of the library)."""

    def __init__(self, fn, in_like, out_like, depth: int = 2):
        import torch
        self.fn, self.depth = fn, depth
        dev = torch.device("cuda", torch.cuda.current_device())
        self.x = [[torch.empty(t.shape, dtype=t.dtype, device=dev) for t in in_like] for _ in range(depth)]
        self.o = [[torch.empty(t.shape, dtype=t.dtype, device=dev) for t in out_like] for _ in range(depth)]
        self.s_in, self.s_comp, self.s_out = (torch.cuda.Stream(dev) for _ in range(3))
        mk = lambda: [torch.cuda.Event() for _ in range(depth)]
        self.ev_in, self.ev_comp, self.ev_out = mk(), mk(), mk()
        self.bytes_in = sum(t.numel() * t.element_size() for t in in_like)
        self.bytes_out = sum(t.numel() * t.element_size() for t in out_like)

    def run(self, host_in, host_out, start_event=None, end_event=None):
        """host_in / host_out: per step, lists of pinned CPU tensors matching in_like / out_like."""
        import torch
        d = self.depth
        if start_event is not None:
            start_event.record(self.s_in)
        for i, (xi, xo) in enumerate(zip(host_in, host_out)):
            b = i % d
            if i >= d:
                self.s_in.wait_event(self.ev_comp[b])      # compute(i-d) finished reading x[b]
            with torch.cuda.stream(self.s_in):
                for dst, src in zip(self.x[b], xi):
                    dst.copy_(src, non_blocking=True)
            self.ev_in[b].record(self.s_in)
            self.s_comp.wait_event(self.ev_in[b])
            if i >= d:
                self.s_comp.wait_event(self.ev_out[b])     # D2H(i-d) finished reading o[b]
            self.fn(self.x[b], self.o[b], self.s_comp)
            self.ev_comp[b].record(self.s_comp)
            self.s_out.wait_event(self.ev_comp[b])
            with torch.cuda.stream(self.s_out):
                for dst, src in zip(xo, self.o[b]):
                    dst.copy_(src, non_blocking=True)
            self.ev_out[b].record(self.s_out)
        if end_event is not None:
            self.s_in.wait_stream(self.s_out)
            self.s_comp.wait_stream(self.s_out)
            end_event.record(self.s_out)
        return host_out
