"""CUDA-graph capture of launch-bound sweep loops.

A config-1 sweep (64^3, 4.4 MB, L2-resident) runs in a few microseconds on
the device, less than the host path of one launch (Python -> ctypes -> C ABI
validation -> cudaLaunchKernel).  The reference's iteration loops
(``run_serial``/``run_tuned``, stencil.py:55-94) are therefore captured once
into a CUDA graph and replayed: one graph launch per batch of sweeps.  The
C ABI launch path makes no synchronising or allocating calls, so every
kernel of the library can be captured.
"""
from __future__ import annotations


class SweepGraph:
    """Capture ``body()`` (which enqueues device work on the current stream)
    ``repeat`` times into one CUDA graph; ``replay()`` re-runs all of it."""

    def __init__(self, body, repeat: int = 1, warmup: int = 1):
        import torch
        self.repeat = repeat
        self.stream = torch.cuda.Stream()
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            for _ in range(warmup):
                body()
        torch.cuda.current_stream().wait_stream(self.stream)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            for _ in range(repeat):
                body()

    def replay(self) -> None:
        self.graph.replay()
