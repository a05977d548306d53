"""Multi-GPU decompositions of the LQR-scan solve (BASELINE configs 3 and 4).

* ``shard_problems``: independent problems split across ranks (config 3).
  No data-path collective -- each rank solves its slice.
* ``TimeShardedLqr``: one long horizon split into contiguous time blocks,
  one per rank (config 4).  The two scans of the LQR subproblem
  (value_pass, reference ``passes.py:291-323``, and propagation_pass,
  ``passes.py:338-361``) are associative, so each rank folds its block into
  one aggregate per scan, the aggregates are all-gathered (one NCCL
  all-gather per scan over NVLink), and every rank combines the gathered
  list into the carry entering its block and finishes the block locally:

      phase 0  local value up-sweep            -> block value aggregate
      gather   (world, 3nx^2+2nx, 1, B)
      phase 1  carry from later blocks, local value down-sweep + gains,
               local propagation up-sweep      -> block affine aggregate
      gather   (world, nx^2+nx, 1, B)
      phase 2  carry from earlier blocks, local forward sweep -> dx, du

The block arithmetic is behind a small ops interface so the same driver runs
the CUDA kernels (``CudaBlockOps``, the product) and, in the CPU tests, a
numpy stand-in with a gloo process group (test infrastructure only).
"""

from __future__ import annotations

import ctypes as C

from . import _native as N


def block_bounds(horizon: int, world: int, rank: int) -> tuple[int, int]:
    """(t_base, length) of rank's contiguous block; lengths differ by <= 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    if horizon < world:
        raise ValueError(f"horizon {horizon} shorter than world size {world}")
    q, r = divmod(horizon, world)
    t0 = rank * q + min(rank, r)
    return t0, q + (1 if rank < r else 0)


def shard_problems(batch: int, world: int, rank: int) -> slice:
    """Contiguous slice of a problem batch owned by rank (config 3)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    q, r = divmod(batch, world)
    b0 = rank * q + min(rank, r)
    return slice(b0, b0 + q + (1 if rank < r else 0))


def block_comps(nx: int) -> tuple[int, int]:
    """Components of one value aggregate (A, Y, C, eta, b) and one affine
    aggregate (F, e)."""
    return 3 * nx * nx + 2 * nx, nx * nx + nx


# ---------------------------------------------------------------- gathers

def nccl_gather(group=None):
    """All-gather over a torch.distributed group into one rank-major tensor."""
    import torch
    import torch.distributed as dist

    def gather(t):
        world = dist.get_world_size(group)
        out = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(out, t.contiguous(), group=group)
        else:  # gloo has no all_gather_into_tensor
            parts = list(out.unbind(0))
            dist.all_gather(parts, t.contiguous(), group=group)
            out = torch.stack(parts)
        return out
    return gather


# ------------------------------------------------------------------ driver

class TimeShardedLqr:
    """Drives the three block phases of one rank with a gather between them."""

    def __init__(self, ops, gather):
        self.ops = ops
        self.gather = gather

    def solve(self):
        vblk = self.ops.value_up()
        pblk = self.ops.value_down(self.gather(vblk))
        self.ops.propagate(self.gather(pblk))
        return self.ops


def emulate_ranks(ops_list):
    """Run the block phases of `world` ranks in one process, in rank order,
    with the all-gather replaced by a stack (single-device parity tests and
    the N=1 bench; no kernel ever waits on another)."""
    import torch
    vs = [o.value_up() for o in ops_list]
    V = torch.stack(vs)
    ps = [o.value_down(V) for o in ops_list]
    Pg = torch.stack(ps)
    for o in ops_list:
        o.propagate(Pg)
    return ops_list


class CudaBlockOps:
    """One rank's block of a time-sharded LQR-scan solve on the device.

    Inputs are the block's stages in SoA batch-minor layout (see
    include/pintoc_b200.h): P (nx*nx, T, B), R (nu*nu, T, B), M, d, Fx, Fu;
    PT (nx*nx, 1, B) on the last block; alpha float64 [B].  Outputs after
    ``propagate``: Gamma, gamma, dx (nx, T+1, B), du; S, s when requested.
    """

    def __init__(self, rank, world, t_base, P, R, M, d, Fx, Fu, PT, alpha, nx, nu,
                 with_value=False, chunk0=0, chunk=0, rows=None):
        torch = N.require_cuda()
        self.torch = torch
        self.lib = N.load_library()
        self.rank, self.world, self.t_base = int(rank), int(world), int(t_base)
        self.nx, self.nu = int(nx), int(nu)
        ref = rows if rows is not None else P
        self.T, self.B = (int(rows.shape[0]), 1) if rows is not None else (int(P.shape[1]),
                                                                            int(P.shape[2]))
        self.dtype = ref.dtype
        self.code = N.PTC_F64 if ref.dtype == torch.float64 else N.PTC_F32
        self.rows = rows.contiguous() if rows is not None else None
        self.inputs = (P, R, M, d, Fx, Fu, PT if rank == world - 1 else None, alpha)
        self.chunk0, self.chunk = int(chunk0), int(chunk)
        dev = ref.device
        nbytes = self.lib.ptc_lqr_block_workspace_bytes(self.code, self.B, self.T, self.nx,
                                                        self.nu, self.chunk0, self.chunk)
        N.check(0 if nbytes >= 0 else int(nbytes))
        self.workspace = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
        vc, pc = block_comps(self.nx)
        mk = lambda *s: torch.empty(*s, dtype=self.dtype, device=dev)
        self.vblock = mk(vc, 1, self.B)
        self.pblock = mk(pc, 1, self.B)
        T, B = self.T, self.B
        self.Gamma = mk(self.nu * self.nx, T, B)
        self.gamma = mk(self.nu, T, B)
        self.dx = mk(self.nx, T + 1, B)
        self.du = mk(self.nu, T, B)
        self.S = mk(self.nx * self.nx, T + 1, B) if with_value else None
        self.s = mk(self.nx, T + 1, B) if with_value else None
        self.flags = torch.zeros(B, dtype=torch.int32, device=dev)

    @classmethod
    def from_rows(cls, rank, world, t_base, rows, PT, alpha, nx, nu, **kw):
        """One long problem (batch 1, nx >= 8) whose block expansion is given
        as stage rows (T, SC): [P | R | M | d | Fx | Fu] per stage, the layout
        the wide kernels read (ptc_lqr_block_solve_rows: no transpose)."""
        return cls(rank, world, t_base, None, None, None, None, None, None, PT, alpha, nx, nu,
                   rows=rows, **kw)

    def _run(self, phase, blocks_in, block_out):
        ptr = lambda t: None if t is None else t.data_ptr()
        P, R, M, d, Fx, Fu, PT, alpha = self.inputs
        if self.rows is not None:
            N.check(self.lib.ptc_lqr_block_solve_rows(
                phase, self.code, self.T, self.nx, self.nu, self.t_base,
                int(self.rank == self.world - 1), self.rank, self.world, ptr(self.rows), ptr(PT),
                ptr(alpha), ptr(blocks_in), ptr(block_out), ptr(self.S), ptr(self.s),
                ptr(self.Gamma), ptr(self.gamma), ptr(self.dx), ptr(self.du), ptr(self.flags),
                ptr(self.workspace), self.workspace.numel(), self.chunk0, self.chunk,
                N.stream_ptr()))
            return
        N.check(self.lib.ptc_lqr_block_solve(
            phase, self.code, self.B, self.T, self.nx, self.nu, self.t_base,
            int(self.rank == self.world - 1), self.rank, self.world,
            ptr(P), ptr(R), ptr(M), ptr(d), ptr(Fx), ptr(Fu), ptr(PT), ptr(alpha),
            ptr(blocks_in), ptr(block_out), ptr(self.S), ptr(self.s), ptr(self.Gamma),
            ptr(self.gamma), ptr(self.dx), ptr(self.du), ptr(self.flags),
            ptr(self.workspace), self.workspace.numel(), self.chunk0, self.chunk,
            N.stream_ptr()))

    def value_up(self):
        self.flags.zero_()
        self._run(0, None, self.vblock)
        return self.vblock

    def value_down(self, gathered):
        self._run(1, gathered.contiguous(), self.pblock)
        return self.pblock

    def propagate(self, gathered):
        self._run(2, gathered.contiguous(), None)


# ------------------------------------------------- time-sharded Newton solve

# reduction layout of the exchanged vectors (include/pintoc_b200.h,
# ptc_solver_block_phase): (first row, end row, op) per phase
_RED_SPECS = {
    3: ((0, 2, "sum"), (2, 6, "max")),
    5: ((0, 4, "sum"), (4, 5, "max"), (5, 7, "min")),
    6: ((0, 2, "max"),),
}


def split_dynamics(dyn, world: int, rank: int):
    """(t_base, block dynamics) of rank's contiguous time block of a
    TimeVaryingLinearDynamics (config 4's time-varying affine model)."""
    from .systems import TimeVaryingLinearDynamics
    if not isinstance(dyn, TimeVaryingLinearDynamics):
        raise TypeError("time-sharded solves take a TimeVaryingLinearDynamics model")
    t0, m = block_bounds(dyn.horizon, world, rank)
    return t0, TimeVaryingLinearDynamics(dyn.A[t0:t0 + m], dyn.B[t0:t0 + m],
                                         dyn.offset[t0:t0 + m])


class BlockNewton:
    """One rank's time block of a Newton / barrier / ADMM solve: a
    block-mode device solver (stages [t_base, t_base + T) of the horizon)
    plus the buffers it exchanges with the other ranks."""

    def __init__(self, block_dynamics, cost, constraints, batch: int, settings, rank: int,
                 world: int, t_base: int, dtype=None):
        from dataclasses import replace
        from ._device import DeviceSolver
        torch = N.require_cuda()
        self.torch = torch
        self.rank, self.world, self.t_base = int(rank), int(world), int(t_base)
        st = replace(settings, block_mode=1, t_base=int(t_base),
                     block_last=int(rank == world - 1), keep_round_controls=False)
        self.solver = s = DeviceSolver(block_dynamics, cost, constraints, batch, st, dtype=dtype)
        nx, B = s.nx, s.B
        cc, vc = nx * nx + nx, 3 * nx * nx + 2 * nx
        mk = lambda c, dt: torch.empty(c, 1, B, dtype=dt, device=s.device)
        self.outs = {0: mk(cc, s.dtype), 1: mk(vc, s.dtype), 2: mk(cc, s.dtype),
                     3: mk(6, torch.float64), 4: mk(cc, s.dtype), 5: mk(7, torch.float64),
                     6: mk(2, torch.float64), 8: mk(cc, s.dtype)}
        self.x0 = None

    def phase(self, p: int, inp=None):
        out = self.outs.get(p)
        aux = self.x0 if p in (5, 9) else None
        self.solver.block_phase(p, None if inp is None else inp.contiguous(), out, aux,
                                self.rank, self.world)
        return out


class _Emulated:
    """All ranks' blocks in one process on one device, run phase by phase in
    rank order; gathers become stacks and all-reduces elementwise folds
    (no kernel ever waits on another rank's)."""

    def gather(self, outs):
        import torch
        g = torch.stack(outs)
        return [g] * len(outs)

    def reduce(self, outs, spec):
        import torch
        r = outs[0].clone()
        for a, b, op in spec:
            st = torch.stack([o[a:b] for o in outs])
            r[a:b] = {"sum": st.sum(0), "max": st.amax(0), "min": st.amin(0)}[op]
        return [r] * len(outs)


class _Distributed:
    """One block per process; NCCL (or gloo) collectives on the current
    stream between the phases."""

    def __init__(self, group=None):
        self.group = group
        self._gather = nccl_gather(group)

    def gather(self, outs):
        return [self._gather(outs[0])]

    def reduce(self, outs, spec):
        import torch.distributed as dist
        ops = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN}
        t = outs[0]
        for a, b, op in spec:
            part = t[a:b].contiguous()
            dist.all_reduce(part, op=ops[op], group=self.group)
            t[a:b] = part
        return [t]


class TimeShardedNewton:
    """Newton / barrier / ADMM solve of one long horizon split into time
    blocks (config 4): every scan of the iteration -- co-state, value,
    propagation, candidate rollout -- folds each block into one aggregate,
    the aggregates are all-gathered and each rank finishes its block from
    the carry; the trust-region and outer-loop scalars (cost, step norm,
    predicted reduction, ADMM residuals, subproblem flags) are all-reduced
    before the per-problem control runs, so every rank takes the same
    accept / reject and outer decisions (newton.py:157-208, outer.py).

    ``blocks`` are the BlockNewton objects this process drives: all ranks'
    (``emulate=True``, one device) or its own one (a torch.distributed group
    with one process per GPU)."""

    def __init__(self, blocks, emulate: bool = False, group=None):
        self.blocks = list(blocks)
        self.comm = _Emulated() if emulate else _Distributed(group)
        self._graph = None      # the captured iteration, reused by later solves

    def _round(self, p, outs):
        if p in _RED_SPECS:
            return self.comm.reduce(outs, _RED_SPECS[p])
        return self.comm.gather(outs)

    def set_initial_state(self, x0):
        """x0 (B, nx): the horizon's initial states (every rank passes the same)."""
        torch = self.blocks[0].torch
        for bl in self.blocks:
            s = bl.solver
            bl.x0 = torch.as_tensor(x0, dtype=s.dtype).reshape(s.B, s.nx).t().contiguous() \
                .unsqueeze(1).to(s.device)

    def rollout(self, controls):
        """problem.py:449 over the split horizon: ``controls`` = per-block
        (B, T_block, nu) arrays; returns per-block (B, T_block + 1, nx)
        device states (row 0 = the block's first state)."""
        torch = self.blocks[0].torch
        for bl, U in zip(self.blocks, controls):
            s = bl.solver
            X = torch.zeros(s.B, s.T + 1, s.nx, dtype=s.dtype)
            s.load(X, U)
        outs = [bl.phase(8) for bl in self.blocks]
        ins = self.comm.gather(outs)
        for bl, g in zip(self.blocks, ins):
            bl.phase(9, g)
        return [bl.solver.field("states", bl.solver.T + 1, (bl.solver.nx,)).contiguous()
                for bl in self.blocks]

    def iteration(self):
        outs = [bl.phase(0) for bl in self.blocks]
        for p in (1, 2, 3, 4, 5, 6):
            ins = self._round(p - 1, outs)
            outs = [bl.phase(p, g) for bl, g in zip(self.blocks, ins)]
        ins = self._round(6, outs)
        for bl, g in zip(self.blocks, ins):
            bl.phase(7, g)

    def _capture(self):
        """One iteration (every phase and collective) as a CUDA graph, or None
        when the stream cannot be captured (the iteration then runs eagerly)."""
        torch = self.blocks[0].torch
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.iteration()
            return g
        except Exception:  # e.g. a backend without graph-capturable collectives
            torch.cuda.synchronize()
            return None

    def solve(self, states, controls, z=None, v=None, group_iters: int = 4,
              graph: bool = True):
        """Load per-block trajectories (B, T_block + 1, nx) / (B, T_block, nu)
        and iterate until every problem is done.  Returns the number of
        device iterations launched.  With ``graph`` the iteration's ~60
        launches and its collectives are captured once (after a first eager
        iteration) and replayed as one CUDA graph."""
        for k, bl in enumerate(self.blocks):
            bl.solver.load(states[k], controls[k], None if z is None else z[k],
                           None if v is None else v[k])
        s0 = self.blocks[0].solver
        st = s0.settings
        rounds = max(1, st.max_outer if st.method == N.METHOD_ADMM else 64)
        cap = (st.max_iters + 2) * rounds + 16
        self.iteration()                 # eager: lazy kernel attributes, allocator
        launched = 1
        if s0.running() == 0:
            return launched
        # one process driving every block (no collectives): capture once,
        # same buffers on every solve.  With a process group the iteration
        # stays eager (collectives inside a captured graph are left out).
        if graph and self._graph is None and isinstance(self.comm, _Emulated):
            self._graph = self._capture()
        g = self._graph if graph else None
        step = g.replay if g is not None else self.iteration
        n = group_iters
        while launched < cap:
            for _ in range(n):
                step()
            launched += n
            if s0.running() == 0:
                break
        return launched
