"""Batched device API: many independent MPC problems in one solver object.

This is the shape of BASELINE config 3 (65,536 pendulum / cart-pole
problems): every problem keeps its own trust-region and outer-loop state on
the device, so the whole batch advances with one launch sequence per
iteration and no per-problem host work.  Inputs and outputs are torch
tensors, problem-major ``(B, T+1, nx)`` / ``(B, T, nu)``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._device import DeviceSolver, SolveSettings
from .newton import NewtonOptions, plan_chunks, rollout_mode
from .outer import AdmmOptions, BarrierOptions
from .problem import ControlProblem


@dataclass
class BatchResult:
    states: object          # (B, T+1, nx) device tensor
    controls: object        # (B, T, nu) device tensor
    status: object          # (B,) int32: 1 done, <0 error
    rounds: object          # (B,) outer rounds run
    round_iters: object     # (round_cap, B) Newton iterations per round
    round_term: object      # (round_cap, B) termination codes
    cost: object            # (B,) final augmented cost
    launches: int           # device iterations launched

    @property
    def inner_iterations(self):
        return self.round_iters.sum(0)


class BatchSolver:
    """Solve ``batch`` copies of ``problem`` (shared model, cost and
    constraints) from per-problem initial trajectories."""

    def __init__(self, problem: ControlProblem, batch: int, method: str = "barrier",
                 newton: NewtonOptions | None = None, barrier: BarrierOptions | None = None,
                 admm: AdmmOptions | None = None, dtype=None, hist_cap: int = 0,
                 chunk0: int = 0, chunk: int = 0):
        newton = newton or (barrier.newton if barrier else admm.newton if admm else NewtonOptions())
        barrier = barrier or BarrierOptions(newton=newton)
        admm = admm or AdmmOptions(newton=newton)
        if method == "barrier":
            m, rounds = N.METHOD_BARRIER, barrier.rounds()
        elif method == "admm":
            m, rounds = N.METHOD_ADMM, admm.max_outer
        elif method == "newton":
            m, rounds = N.METHOD_NEWTON, 1
        else:
            raise ValueError("method must be 'barrier', 'admm' or 'newton'")
        c0, c1 = (chunk0, chunk) if (chunk0 or chunk) else plan_chunks(newton.executor,
                                                                       problem.horizon)
        self.settings = SolveSettings(
            method=m, alpha0=newton.alpha0, nu0=newton.nu0, inner_tol=newton.inner_tol,
            max_iters=newton.max_iters, mu0=barrier.mu0, zeta=barrier.zeta,
            mu_tol=barrier.mu_tol, rho=admm.rho, residual_tol=admm.residual_tol,
            max_outer=admm.max_outer, hist_cap=hist_cap, round_cap=max(1, rounds),
            chunk0=c0, chunk=c1, rollout=rollout_mode(newton.executor))
        self.problem = problem
        self.solver = DeviceSolver(problem.dynamics, problem.cost, problem.constraints, batch,
                                   self.settings, dtype=dtype)
        self.torch = self.solver.torch

    @property
    def batch(self) -> int:
        return self.solver.B

    def rollout(self, x0, controls):
        """Device rollout of (B, nx) initial states under (B, T, nu) controls."""
        torch, s = self.torch, self.solver
        X = torch.zeros(s.B, s.T + 1, s.nx, dtype=s.dtype, device=s.device)
        X[:, 0] = torch.as_tensor(x0, dtype=s.dtype, device=s.device)
        s.load(X, controls)
        s.rollout()
        return s.field("states", s.T + 1, (s.nx,)).contiguous()

    def solve(self, states, controls, check: bool = False) -> BatchResult:
        s = self.solver
        s.load(states, controls)
        if check:
            bad = s.check_consistency()
            if (bad >= 0).any():
                raise ValueError(f"{int((bad >= 0).sum())} initial trajectories are not "
                                 "dynamically consistent")
        launches = s.run()
        return self._result(launches)

    def _result(self, launches: int) -> BatchResult:
        s = self.solver
        return BatchResult(
            states=s.states().contiguous(), controls=s.controls().contiguous(),
            status=s.read("status"), rounds=s.read("round"),
            round_iters=s.rounds("round_iters"), round_term=s.rounds("round_term"),
            cost=s.read("cur_cost"), launches=launches)

    @staticmethod
    def solve_concurrently(jobs, group: int = 16, priorities=None) -> list:
        """Advance several batches (e.g. the two models of config 3) at once,
        one CUDA stream each: ``jobs`` = [(BatchSolver, states, controls)].
        Every solver runs its whole loop on the device (one graph with a
        conditional WHILE node per stream, ptc_solver_loop), so one batch's
        stragglers never serialise the other's iterations and a host stall
        cannot drain a stream.  Without conditional graphs the host polls
        each stream every ``group`` iterations instead.  ``priorities``:
        per-job CUDA stream priorities (lower = higher priority)."""
        import torch
        streams = [torch.cuda.Stream(priority=p)
                   for p in (priorities or [0] * len(jobs))]
        for (bs, X, U), st in zip(jobs, streams):
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                bs.solver.load(X, U)
        launched = [0] * len(jobs)
        caps = [(bs.settings.max_iters + 2) * max(1, bs.settings.round_cap) + 16
                for bs, _, _ in jobs]
        # each batch as one device-resident graph loop on its own stream: the
        # host only waits at the end (ptc_solver_loop)
        counts = [torch.zeros(1, dtype=torch.int32).pin_memory() for _ in jobs]
        looped = []
        for i, ((bs, _, _), st) in enumerate(zip(jobs, streams)):
            with torch.cuda.stream(st):
                looped.append(bs.solver.device_loop(caps[i], 1, counts[i]))
        # the rest (drivers without conditional graphs): host-polled below
        # one group stays queued while the host reads the previous group's
        # running count (pinned copy + event), so the streams never drain
        # waiting for the host; a finished batch runs at most one extra
        # group of early-exit iterations.  16 iterations per group: with 4,
        # about one config-3 solve in five took ~1.35x as long (a host
        # hiccup longer than the queued work drains both streams); 16 and
        # 64 gave no outlier in 24 solves (profiles/r2v_bench.md)
        polls = [torch.zeros(1, dtype=torch.int32).pin_memory() for _ in jobs]
        events = [None] * len(jobs)
        active = {i for i in range(len(jobs)) if not looped[i]}
        n = 1
        while active:
            pending = []
            for i in sorted(active):
                with torch.cuda.stream(streams[i]):
                    jobs[i][0].solver.iterate(n)
                launched[i] += n
                pending.append((i, events[i]))
                ev = torch.cuda.Event()
                with torch.cuda.stream(streams[i]):
                    jobs[i][0].solver.running_async(polls[i])
                    ev.record(streams[i])
                # (this copy may land before the previous group's value is
                # read below: a later count, just as valid -- it only falls)
                events[i] = ev
            for i, prev in pending:
                if prev is None:
                    continue
                prev.synchronize()
                if int(polls[i][0]) == 0 or launched[i] >= caps[i]:
                    active.discard(i)
            n = group
        out = []
        for i, ((bs, _, _), st) in enumerate(zip(jobs, streams)):
            if looped[i]:
                st.synchronize()
                launched[i] = int(counts[i][0])
            with torch.cuda.stream(st):
                out.append(bs._result(launched[i]))
            torch.cuda.current_stream().wait_stream(st)
        return out

    @staticmethod
    def shift_controls(controls, shift: int):
        """Receding-horizon warm start: drop the first ``shift`` controls and
        repeat the last one (bench.py run_mpc shift rule, generalised)."""
        import torch
        tail = controls[:, -1:].expand(-1, shift, -1)
        return torch.cat([controls[:, shift:], tail], dim=1).contiguous()
