"""Single-domain time stepping of one nest on resident device arrays.

A *step* is `sweeps` launches of the nest with the buffers rotating between
launches the way the nest's time loop rotates them (``nests.ROTATIONS``:
Jacobi / D3Q19 ping-pong, wave4's up <- u <- un <- up).  ``capture`` records
one CUDA graph of a whole step (Jacobi's 100 sweeps: 100 launches) so a time
loop replays it with no per-launch host work; the bench's per-kernel table
and the full-size parity tests run the same object.
"""
from __future__ import annotations

from typing import Dict

from . import backend, nests


class Stepper:
    def __init__(self, k: backend.Kernel, arrays: Dict[str, object], scalars: Dict[str, float],
                 variant: str = "accsat", schedule="default", sweeps: int = 1):
        import torch
        self.torch = torch
        self.k = k
        self.arrays = arrays
        self.names = list(arrays)
        self.scalars = dict(scalars)
        self.variant, self.schedule = variant, schedule
        self.sweeps = sweeps
        self.nest = nests.kernel(k.kernel_id).nest
        self.period = nests.rotation_period(self.nest)
        self.t = 0                    # launches so far
        self.graph = None

    def _launch(self, t: int, stream) -> None:
        roles = nests.role_buffers(self.nest, self.names, t)
        self.k.launch({p: self.arrays[b] for p, b in roles.items()}, self.scalars, self.variant, self.schedule,
                      stream)

    @property
    def blocked(self) -> bool:
        """schedule "tb2": the whole step as acs_launch_steps with temporal
        blocking (two sweeps per launch, kernels/tblock.cuh)."""
        return self.schedule == "tb2"

    def capture(self, stream=None) -> None:
        """One CUDA graph of a step.  Needs `sweeps` to be a multiple of the
        rotation period (the graph's buffers are fixed) and a step count of
        whole periods so far."""
        torch = self.torch
        if self.sweeps % self.period or self.t % self.period:
            raise ValueError(f"capture: {self.sweeps} sweeps per step do not close the {self.period}-buffer rotation")
        stream = stream or torch.cuda.current_stream()
        self.step(stream)                 # warm: attributes, tensor maps
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        with torch.cuda.graph(g, stream=cs):
            if self.blocked:
                self._steps(cs)
            else:
                for t in range(self.sweeps):
                    self._launch(t, cs)
        stream.wait_stream(cs)
        torch.cuda.synchronize()
        self.graph = g

    def _steps(self, stream) -> None:
        if self.sweeps % 4:
            raise ValueError("tb2 steps: a multiple of 4 sweeps keeps the newest field in the ping-pong's buffer")
        names = self.names
        latest = self.k.launch_steps({n: self.arrays[n] for n in names}, self.scalars, self.variant, self.sweeps,
                                     True, stream)
        want = nests.role_buffers(self.nest, names, self.sweeps)[nests.ROTATIONS[self.nest][0][0]]
        if latest != want:
            raise RuntimeError(f"tb2 steps left the newest field in {latest}, the time loop expects {want}")

    def step(self, stream=None) -> None:
        torch = self.torch
        stream = stream or torch.cuda.current_stream()
        if self.graph is not None:
            with torch.cuda.stream(stream):
                self.graph.replay()
            self.t += self.sweeps
            return
        if self.blocked:
            self._steps(stream)
            self.t += self.sweeps
            return
        for _ in range(self.sweeps):
            self._launch(self.t, stream)
            self.t += 1

    def current(self, name: str):
        """Physical buffer holding parameter `name` after the launches so far."""
        return self.arrays[nests.role_buffers(self.nest, self.names, self.t)[name]]
