"""Layer-stack driver.

Runs a chain of 3x3 / stride-1 / pad-1 LANCE conv layers with the fused bias +
ReLU epilogue and 2x2 max-pools between stages (F(2x2): fused into the
preceding conv's GEMM epilogue), device-resident end to end:
every layer's output buffer is the next layer's input, filters are prepared
once (K2), and the whole forward can be captured once into a CUDA graph and
replayed (one graph launch per batch instead of 3-4 kernel launches per layer).

Numerics per conv layer are exactly ``lance_gemm`` (engines.hpp:492-536) --
the batch-coupled PerPosition fit is recomputed on each layer's actual input --
followed by ``relu(y + bias)``; the reference has no bias / ReLU / pooling, so
the parity oracle for a stack is the oracle's lance_gemm chained on the host
with those applied in numpy (tests/test_gpu_stack.py).

VGG16_CIFAR is BASELINE.json configs[1].
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

from . import _lib
from .api import ConvSpec, LanceConfig, LanceConv, LanceError, _check, _stream_ptr

# (kind, C, K) for convs, ("pool",) for 2x2 max-pools: VGG-16 on 32x32 inputs.
VGG16_CIFAR = [("conv", 3, 64), ("conv", 64, 64), ("pool",),
               ("conv", 64, 128), ("conv", 128, 128), ("pool",),
               ("conv", 128, 256), ("conv", 256, 256), ("conv", 256, 256), ("pool",),
               ("conv", 256, 512), ("conv", 512, 512), ("conv", 512, 512), ("pool",),
               ("conv", 512, 512), ("conv", 512, 512), ("conv", 512, 512)]


@dataclass
class _Stage:
    kind: str
    n: int
    h: int
    w: int
    c: int
    k: int = 0
    conv: LanceConv | None = None
    out: object = None  # torch tensor
    fused: bool = False  # pool folded into the previous conv's epilogue


class LanceStack:
    """A chain of LANCE conv layers (+ bias / ReLU) and 2x2 max-pools.

    layers: list of ("conv", C, K) / ("pool",); the first conv's C must match
    the input channels, and every conv's C the previous layer's channels.
    """

    def __init__(self, layers, n: int, h: int, w: int, cfg: LanceConfig, device: int = 0,
                 tile_m: int = 2, relu: bool = True, fuse_pool: bool = True):
        import torch
        self.device = device
        self.relu = relu
        self.cfg = cfg
        self.stages: list[_Stage] = []
        dev = torch.device("cuda", device)
        c = None
        for layer in layers:
            if layer[0] == "conv":
                _, lc, lk = layer
                if c is not None and lc != c:
                    raise LanceError(f"stack: conv expects C={lc} but the previous layer has {c}")
                spec = ConvSpec(n, lc, h, w, lk, 1)
                st = _Stage("conv", n, h, w, lc, lk, LanceConv(spec, cfg, device, tile_m=tile_m))
                st.out = torch.empty((n, h, w, lk), dtype=torch.float32, device=dev)
                c = lk
            elif layer[0] == "pool":
                if c is None:
                    raise LanceError("stack: a pool needs an input layer")
                if h < 2 or w < 2:
                    raise LanceError("stack: pool on a map smaller than 2x2")
                st = _Stage("pool", n, h, w, c)
                h, w = h // 2, w // 2
                st.out = torch.empty((n, h, w, c), dtype=torch.float32, device=dev)
            else:
                raise LanceError(f"stack: unknown layer kind {layer[0]!r}")
            self.stages.append(st)
        if not self.stages or self.stages[0].kind != "conv":
            raise LanceError("stack: the first layer must be a conv")
        # A pool right after a conv is fused into that conv's GEMM epilogue
        # (F(2x2): a Winograd tile's 2x2 outputs are one pool window), which
        # then writes the pooled map directly; the pool stage becomes a no-op.
        self.fuse_pool = fuse_pool and tile_m == 2
        if self.fuse_pool:
            for prev, st in zip(self.stages, self.stages[1:]):
                if st.kind == "pool" and prev.kind == "conv":
                    st.fused = True
                    prev.out = st.out
        self.in_shape = (n, self.stages[0].h, self.stages[0].w, self.stages[0].c)
        self.out_shape = tuple(self.stages[-1].out.shape)
        self._graph = None
        self._static_in = None

    @property
    def convs(self):
        return [s for s in self.stages if s.kind == "conv"]

    def set_weights(self, weights, biases=None, stream=None):
        """weights[i]: [K,3,3,C] float32 CUDA tensor of the i-th conv; biases[i]:
        [K] tensor or None.  K2 runs once per layer here."""
        convs = self.convs
        if len(weights) != len(convs):
            raise LanceError(f"stack: {len(convs)} convs but {len(weights)} weight tensors")
        biases = biases if biases is not None else [None] * len(convs)
        self._bias = list(biases)  # keep alive: the plans hold raw pointers
        pooled = {id(prev) for prev, st in zip(self.stages, self.stages[1:]) if st.fused}
        for st, wt, b in zip(convs, weights, biases):
            st.conv.set_filters(wt, stream)
            st.conv.set_epilogue(b, self.relu, pool=id(st) in pooled)

    def forward(self, x, stream=None):
        """All layers on `stream` (default: torch's current stream); returns the
        last layer's output buffer (owned by the stack)."""
        cur = x
        for st in self.stages:
            if st.kind == "conv":
                st.conv.forward(cur, st.out, stream=stream)
            elif st.fused:
                pass  # written by the previous conv's epilogue
            else:
                _check(_lib.lib().lance_maxpool2x2_nhwc(ct.c_void_p(cur.data_ptr()),
                                                        ct.c_void_p(st.out.data_ptr()), st.n, st.h,
                                                        st.w, st.c, _stream_ptr(stream)))
            cur = st.out
        return cur

    def launches_per_forward(self) -> int:
        return sum(3 if s.kind == "conv" else (0 if s.fused else 1) for s in self.stages)

    def capture(self, x_example):
        """Record one forward into a CUDA graph (after an eager warm-up that also
        configures every kernel).  Later batches: ``replay(x)`` copies x into
        the captured input buffer and launches the graph."""
        import torch
        self._static_in = x_example.clone()
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.forward(self._static_in)
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        self._graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self._graph):
            self._out = self.forward(self._static_in)
        return self._out

    def replay(self, x=None):
        if self._graph is None:
            raise LanceError("stack: capture() first")
        if x is not None:
            self._static_in.copy_(x)
        self._graph.replay()
        return self._out

    def sync(self, stream=None):
        """Surface a NaN seen by any layer's range pass (the reference throws
        from fit_params)."""
        for st in self.convs:
            st.conv.sync(stream)

    def close(self):
        for st in self.convs:
            st.conv.close()
