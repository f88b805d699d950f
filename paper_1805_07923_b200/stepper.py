"""Graph-captured time stepping (the fast path behind bench.py's MLSDC lines).

The drop-in orchestration in `mlsdc.py` / `sdc.py` issues only stream-ordered
device work (library kernels, no host synchronisation), so one complete time
step is captured once into a CUDA graph and replayed per step: the ~100-400
kernel launches of a step cost one graph launch, and Python is out of the
loop.  This replaces the reference's timed stepping loop
(harness.py:234-259) for one fixed configuration.

The per-step finiteness check of the reference (harness.py:257-258, raising
InstabilityError(step)) becomes one device flag per step, written inside the
graph and inspected once after the run (no per-step host sync).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib, mlsdc, sdc
from .spharm import _dev_guard, _ptr, _stream_ptr
from .swe import EvalCounters, PrognosticState


class InstabilityError(RuntimeError):
    """Non-finite state after step `step` (0-based, as the reference's
    run_simulation loop index; harness.py:31-36)."""

    def __init__(self, step: int, message: str | None = None):
        self.step = step
        super().__init__(message or f"non-finite state after step {step}")


def _counter_sum(levels) -> list[EvalCounters]:
    return [lv.rhs.counters.snapshot() for lv in levels]


class _GraphStep:
    """Shared capture/replay machinery: `body(x)` advances the static state x
    (a (..., 3, R+1, R+1) device tensor) by one step, in place."""

    def __init__(self, x_static: torch.Tensor, body, levels, use_graph: bool = True):
        self.x = x_static
        self.body = body
        self.levels = levels
        # device int: 1 if the last step produced a non-finite value (written by
        # the library's fused copy + finiteness kernel inside the graph)
        self.bad = torch.zeros((), dtype=torch.int32, device=x_static.device)
        self.graph = None
        # eager warm-up on a side stream: sizes every plan workspace and sets
        # kernel attributes before capture (nothing may allocate in capture)
        backup = self.x.clone()
        before = _counter_sum(levels)
        s = torch.cuda.Stream(device=x_static.device)
        s.wait_stream(torch.cuda.current_stream(x_static.device))
        with torch.cuda.stream(s):
            self._step()
        torch.cuda.current_stream(x_static.device).wait_stream(s)
        after = _counter_sum(levels)
        self.counts_per_step = [a.since(b) for a, b in zip(after, before)]
        self.x.copy_(backup)
        if use_graph:
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self._step()
            # capture-time Python side effects (counters) are not per replay
            for lv, b in zip(levels, after):
                lv.rhs.counters.solves = b.solves
                lv.rhs.counters.implicit_evals = b.implicit_evals
                lv.rhs.counters.explicit_evals = b.explicit_evals

    def _step(self):
        y = self.body(self.x)
        dev = self.x.device
        with _dev_guard(dev):
            _lib.check(_lib.load().swsdc_copy_finite(
                _ptr(y.contiguous()), _ptr(self.x), self.x.numel() * 2, _ptr(self.bad),
                _stream_ptr(dev)))

    def replay(self):
        if self.graph is not None:
            self.graph.replay()
        else:
            self._step()
        for lv, c in zip(self.levels, self.counts_per_step):
            lv.rhs.counters.solves += c.solves
            lv.rhs.counters.implicit_evals += c.implicit_evals
            lv.rhs.counters.explicit_evals += c.explicit_evals


class MLSDCStepper:
    """Fixed-iteration two-level MLSDC stepping (mlsdc.py:242-254) on the GPU.

    `members` > 1 advances an ensemble in lock-step (leading state axis);
    `n_coarse_sweeps` = 2 is BASELINE config 2's variant.
    """

    def __init__(self, hier: mlsdc.TwoLevelHierarchy, dt: float, n_iterations: int,
                 state0: PrognosticState, n_coarse_sweeps: int = 1, use_graph: bool = True):
        if n_iterations < 1:
            raise ValueError("at least one iteration is required")
        self.hier, self.dt, self.n_iter, self.n_cs = hier, dt, n_iterations, n_coarse_sweeps
        members = int(np.prod(state0.data.shape[:-3])) if state0.data.dim() > 3 else 1
        hier.fine.plan.reserve(5 * members + 8)
        hier.coarse.plan.reserve(5 * members * max(1, hier.coarse.n_nodes) + 8)
        x = state0.data.clone()

        def body(xt):
            return mlsdc.mlsdc_timestep(PrognosticState.from_tensor(xt), dt, n_iterations, hier,
                                        n_coarse_sweeps).data

        self._g = _GraphStep(x, body, [hier.fine, hier.coarse], use_graph)
        self.members = members

    @property
    def state(self) -> PrognosticState:
        return PrognosticState.from_tensor(self._g.x)

    def set_state(self, st: PrognosticState) -> None:
        self._g.x.copy_(st.data)

    def step(self) -> None:
        self._g.replay()

    def run(self, n_steps: int) -> PrognosticState:
        """Advance n_steps; raise InstabilityError for the first non-finite step."""
        flags = torch.empty(n_steps, dtype=torch.int32, device=self._g.x.device)
        for k in range(n_steps):
            self._g.replay()
            flags[k].copy_(self._g.bad)
        bad = torch.nonzero(flags)
        if bad.numel():
            raise InstabilityError(int(bad[0]))
        return self.state

    @property
    def counts_per_step(self):
        return self._g.counts_per_step

    def fine_sweeps_per_step(self) -> int:
        return self.n_iter * self.members


class SDCStepper:
    """Fixed-sweep single-level IMEX SDC stepping (sdc.py:236-253) on the GPU."""

    def __init__(self, level: mlsdc.Level, dt: float, n_sweeps: int, state0: PrognosticState,
                 use_graph: bool = True):
        if n_sweeps < 1:
            raise ValueError("at least one sweep is required")
        members = int(np.prod(state0.data.shape[:-3])) if state0.data.dim() > 3 else 1
        level.plan.reserve(5 * members + 8)

        def body(xt):
            return sdc.sdc_timestep(PrognosticState.from_tensor(xt), dt, n_sweeps, level.tables,
                                    level.rhs).data

        self._g = _GraphStep(state0.data.clone(), body, [level], use_graph)
        self.n_sweeps, self.members = n_sweeps, members

    @property
    def state(self) -> PrognosticState:
        return PrognosticState.from_tensor(self._g.x)

    def run(self, n_steps: int) -> PrognosticState:
        flags = torch.empty(n_steps, dtype=torch.int32, device=self._g.x.device)
        for k in range(n_steps):
            self._g.replay()
            flags[k].copy_(self._g.bad)
        bad = torch.nonzero(flags)
        if bad.numel():
            raise InstabilityError(int(bad[0]))
        return self.state
