"""Multi-rank decompositions of the LQR-scan solve (configs 3 and 4).

CPU: block / problem partitioning, and the time-sharded driver run by a
world-size-2 and -3 gloo process group with numpy block ops (the driver's
decomposition and all-gather plumbing) against the unsharded oracle solve.
GPU: the CUDA block phases (``ptc_lqr_block_solve`` through the C ABI)
emulating 1..5 ranks on one device, and the NCCL gather path at world 1,
against the oracle -- fp64 1e-9 relative, fp32 1e-4 (BASELINE north_star).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from conftest import rel_gap

from oracle import pintoc_oracle as O
from paper_2409_20027_b200.sharded import (TimeShardedLqr, block_bounds, emulate_ranks,
                                           nccl_gather, shard_problems)


def test_block_bounds_cover_horizon_contiguously():
    for T in (1, 2, 7, 64, 1000, 1 << 20):
        for world in (1, 2, 3, 4, 8):
            if T < world:
                with pytest.raises(ValueError):
                    block_bounds(T, world, 0)
                continue
            nxt = 0
            lens = []
            for r in range(world):
                t0, n = block_bounds(T, world, r)
                assert t0 == nxt and n >= 1
                nxt += n
                lens.append(n)
            assert nxt == T and max(lens) - min(lens) <= 1


def test_shard_problems_partitions_batch():
    for B in (1, 5, 65536, 65537):
        for world in (1, 2, 4, 8):
            got = [shard_problems(B, world, r) for r in range(world)]
            assert got[0].start == 0 and got[-1].stop == B
            assert all(a.stop == b.start for a, b in zip(got, got[1:]))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, T, nx, nu, seed, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from sharded_ref import NumpyBlockOps
        exp = O.random_lqr_expansion(np.random.default_rng(seed), T, nx, nu, alpha=0.5)
        t0, n = block_bounds(T, world, rank)
        ops = TimeShardedLqr(NumpyBlockOps(exp, rank, world, t0, n), nccl_gather()).solve()
        np.savez(os.path.join(out, f"r{rank}.npz"), S=ops.S, s=ops.s, Gamma=ops.Gamma,
                 gamma=ops.gamma, dx=ops.dx, du=ops.du, t0=t0, n=n)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_time_sharded_driver_gloo_matches_unsharded(world, tmp_path):
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    T, nx, nu, seed = 37, 3, 2, 11
    mp.spawn(_gloo_worker, args=(world, _free_port(), T, nx, nu, seed, str(tmp_path)),
             nprocs=world, join=True)
    exp = O.random_lqr_expansion(np.random.default_rng(seed), T, nx, nu, alpha=0.5)
    S, s, Gam, gam, dxs, dus = O.lqr_solve(exp)
    for r in range(world):
        f = np.load(tmp_path / f"r{r}.npz")
        t0, n = int(f["t0"]), int(f["n"])
        sl, sl1 = slice(t0, t0 + n), slice(t0, t0 + n + 1)
        for name, got, want in (("S", f["S"], S[sl1]), ("s", f["s"], s[sl1]),
                                ("Gamma", f["Gamma"], Gam[sl]), ("gamma", f["gamma"], gam[sl]),
                                ("dx", f["dx"], dxs[sl1]), ("du", f["du"], dus[sl])):
            assert rel_gap(got, want) < 1e-10, (r, name)


# ------------------------------------------------------------------- GPU

def _soa(a, comps, dtype):
    t = torch.as_tensor(np.asarray(a, float), dtype=dtype).reshape(a.shape[0], comps)
    return t.t().contiguous().unsqueeze(-1).cuda()


def _cuda_ranks(exp, world, dtype, chunk0=0, chunk=0):
    from paper_2409_20027_b200.sharded import CudaBlockOps
    n, nx, nu = exp.P.shape[0], exp.P.shape[1], exp.R.shape[1]
    full = dict(P=_soa(exp.P, nx * nx, dtype), R=_soa(exp.R, nu * nu, dtype),
                M=_soa(exp.M, nx * nu, dtype), d=_soa(exp.d, nu, dtype),
                Fx=_soa(exp.Fx, nx * nx, dtype), Fu=_soa(exp.Fu, nx * nu, dtype))
    PT = _soa(exp.PT[None], nx * nx, dtype)
    alpha = torch.full((1,), float(exp.alpha), dtype=torch.float64, device="cuda")
    ops = []
    for r in range(world):
        t0, m = block_bounds(n, world, r)
        loc = {k: v[:, t0:t0 + m].contiguous() for k, v in full.items()}
        ops.append(CudaBlockOps(r, world, t0, loc["P"], loc["R"], loc["M"], loc["d"], loc["Fx"],
                                loc["Fu"], PT, alpha, nx, nu, with_value=True, chunk0=chunk0,
                                chunk=chunk))
    return ops


def _assemble(ops):
    host = lambda t: t[..., 0].t().double().cpu().numpy()

    def cat(name, extra_row):
        # T+1-row fields: each block's last row is the next block's first
        parts = [host(getattr(o, name)) for o in ops]
        if extra_row:
            parts = [p[:-1] for p in parts[:-1]] + [parts[-1]]
        return np.concatenate(parts)

    nx, nu = ops[0].nx, ops[0].nu
    S = cat("S", 1).reshape(-1, nx, nx)
    s = cat("s", 1)
    Gam = cat("Gamma", 0).reshape(-1, nu, nx)
    gam = cat("gamma", 0)
    dx = cat("dx", 1)
    du = cat("du", 0)
    return S, s, Gam, gam, dx, du


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3, 5])
@pytest.mark.parametrize("nx,nu,T", [(2, 1, 301), (4, 2, 128), (12, 4, 64)])
def test_cuda_time_blocks_match_oracle(world, nx, nu, T):
    exp = O.random_lqr_expansion(np.random.default_rng(100 + nx + world), T, nx, nu, alpha=0.0)
    ref = O.lqr_solve(exp)
    for plan in ((0, 0), (2, 2), (T, 0)):
        ops = emulate_ranks(_cuda_ranks(exp, world, torch.float64, *plan))
        torch.cuda.synchronize()
        assert all(int(o.flags[0]) == 0 for o in ops)
        for name, got, want in zip(("S", "s", "Gamma", "gamma", "dx", "du"), _assemble(ops), ref):
            assert got.shape == want.shape, name
            assert rel_gap(got, want) < 1e-9, (world, plan, name)
        # block-boundary consistency: rank r's swept last dx row and rank
        # r+1's carried first row agree to rounding (different association)
        for a, b in zip(ops, ops[1:]):
            assert torch.allclose(a.dx[:, -1], b.dx[:, 0], rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
def test_cuda_time_blocks_fp32_tolerance():
    exp = O.random_lqr_expansion(np.random.default_rng(5), 256, 4, 2, alpha=0.0)
    ref = O.lqr_solve(exp)
    ops = emulate_ranks(_cuda_ranks(exp, 4, torch.float32))
    torch.cuda.synchronize()
    for name, got, want in zip(("S", "s", "Gamma", "gamma", "dx", "du"), _assemble(ops), ref):
        assert rel_gap(got, want) < 1e-4, name


@pytest.mark.gpu
def test_cuda_time_blocks_through_nccl_gather_world1():
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        exp = O.random_lqr_expansion(np.random.default_rng(9), 200, 4, 2, alpha=0.3)
        ref = O.lqr_solve(exp)
        (ops,) = _cuda_ranks(exp, 1, torch.float64)
        TimeShardedLqr(ops, nccl_gather()).solve()
        torch.cuda.synchronize()
        for name, got, want in zip(("S", "s", "Gamma", "gamma", "dx", "du"), _assemble([ops]),
                                   ref):
            assert rel_gap(got, want) < 1e-9, name
    finally:
        dist.destroy_process_group()


# ---------------------------------------- time-sharded Newton driver plumbing

class _FakeBlock:
    """Stands in for sharded.BlockNewton: deterministic per-(phase, rank)
    outputs of the real shapes, records what each phase received."""

    def __init__(self, rank, world, nx=3, B=2):
        self.rank, self.world, self.B = rank, world, B
        cc, vc = nx * nx + nx, 3 * nx * nx + 2 * nx
        self.rows = {0: cc, 1: vc, 2: cc, 3: 6, 4: cc, 5: 7, 6: 2, 8: cc}
        self.got = {}

    def phase(self, p, inp=None):
        self.got[p] = None if inp is None else inp.clone()
        if p not in self.rows:
            return None
        g = torch.Generator().manual_seed(1000 * p + self.rank)
        return torch.randn(self.rows[p], 1, self.B, generator=g, dtype=torch.float64)


def _expected_inputs(world):
    from paper_2409_20027_b200.sharded import _RED_SPECS
    fakes = [_FakeBlock(r, world) for r in range(world)]
    outs = {p: [f.phase(p) for f in fakes] for p in (0, 1, 2, 3, 4, 5, 6)}
    exp = {}
    for p in (1, 2, 3, 5):
        exp[p] = torch.stack(outs[p - 1])
    for p, src in ((4, 3), (6, 5), (7, 6)):
        r = outs[src][0].clone()
        for a, b, op in _RED_SPECS[src]:
            st = torch.stack([o[a:b] for o in outs[src]])
            r[a:b] = {"sum": st.sum(0), "max": st.amax(0), "min": st.amin(0)}[op]
        exp[p] = r
    return exp


def _newton_plumbing_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2409_20027_b200.sharded import TimeShardedNewton
        fb = _FakeBlock(rank, world)
        TimeShardedNewton([fb]).iteration()
        torch.save(fb.got, os.path.join(out, f"g{rank}.pt"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_time_sharded_newton_driver_collectives_gloo(world, tmp_path):
    """The driver's exchange plan over a real process group (gloo, CPU):
    after phases 0, 1, 2 and 4 every rank receives the rank-major stack of
    all ranks' block maps; after 3, 5 and 6 the trust-region vectors reduced
    with the per-row SUM / MAX / MIN of include/pintoc_b200.h -- identical to
    the single-process emulation the GPU parity tests use."""
    from paper_2409_20027_b200.sharded import TimeShardedNewton
    mp.spawn(_newton_plumbing_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
             join=True)
    exp = _expected_inputs(world)
    fakes = [_FakeBlock(r, world) for r in range(world)]
    TimeShardedNewton(fakes, emulate=True).iteration()
    for r in range(world):
        got = torch.load(os.path.join(tmp_path, f"g{r}.pt"))
        assert got[0] is None
        for p in range(1, 8):
            # gloo's ring sum associates differently: equal to the last ulp
            assert torch.allclose(got[p], exp[p], rtol=1e-14, atol=0), (r, p)
            assert torch.equal(fakes[r].got[p], exp[p]), (r, p)
