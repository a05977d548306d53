"""Thin owner of one C-ABI solver object: workspace (a torch tensor),
descriptor, loading, the iteration driver and typed buffer reads.

Layout at this boundary: user-facing tensors are problem-major
``(B, T+1, nx)`` / ``(B, T, nu)``; the library's HBM layout is SoA
batch-minor ``(nx, T+1, B)`` (see include/pintoc_b200.h), converted here with
one permute + contiguous copy on the device.
"""

from __future__ import annotations

import ctypes as C
import warnings
from dataclasses import dataclass

import numpy as np

from . import _native as N


@dataclass(frozen=True)
class SolveSettings:
    method: int = N.METHOD_NEWTON
    aug: int = N.AUG_ZERO
    aug_mu: float = 0.0
    alpha0: float = 1.0
    nu0: float = 2.0
    inner_tol: float = 1e-8
    max_iters: int = 100
    mu0: float = 0.1
    zeta: float = 0.2
    mu_tol: float = 1e-4
    rho: float = 1.0
    residual_tol: float = 1e-2
    max_outer: int = 200
    hist_cap: int = 0
    round_cap: int = 1
    keep_round_controls: bool = False
    chunk0: int = 0
    chunk: int = 0
    rollout: int = 0          # 0 auto, 1 sequential, 2 log-depth Newton sweeps
    block_mode: int = 0       # time-block mode (sharded.TimeShardedNewton)
    t_base: int = 0
    block_last: int = 0


def _dtype_code(torch, dtype) -> int:
    if dtype == torch.float64:
        return N.PTC_F64
    if dtype == torch.float32:
        return N.PTC_F32
    raise ValueError("dtype must be torch.float64 or torch.float32")


def _np_ptr(a) -> int | None:
    return None if a is None else a.ctypes.data


def _linear_device(dynamics, spec, torch, dtype, device):
    """Affine model data as device (comps, rows) tensors, cached on the
    (read-only) dynamics object: the stage-major host arrays are uploaded
    once and transposed on the GPU instead of by numpy."""
    cache = dynamics.__dict__.setdefault("_device_cache", {})
    key = (str(dtype), str(device))
    if key not in cache:
        out = []
        for name in ("lin_a", "lin_b", "lin_c"):
            with warnings.catch_warnings():   # read-only source, only ever read
                warnings.simplefilter("ignore", UserWarning)
                host = torch.from_numpy(np.ascontiguousarray(spec[name], dtype=np.float64))
            out.append(host.to(device=device, dtype=dtype).t().contiguous())
        torch.cuda.current_stream(device).synchronize()
        cache[key] = tuple(out)
    return cache[key]


class DeviceSolver:
    """`batch` independent problems sharing dynamics, cost and constraints."""

    def __init__(self, dynamics, cost, constraints, batch: int, settings: SolveSettings,
                 dtype=None, device=None):
        torch = N.require_cuda()
        self.torch = torch
        self.lib = N.load_library()
        self.dtype = dtype or torch.float64
        self.device = torch.device(device or "cuda")
        self.settings = settings
        self.B = int(batch)
        self.T = int(dynamics.horizon)
        self.nx, self.nu = int(dynamics.d_x), int(dynamics.d_u)
        npdt = np.float64 if self.dtype == torch.float64 else np.float32

        from .usermodel import DeviceConstraint, DeviceCost, DeviceDynamics
        ucost = cost if isinstance(cost, DeviceCost) else None
        ucon = constraints if isinstance(constraints, DeviceConstraint) else None
        if ucost is not None or ucon is not None:
            if not isinstance(dynamics, DeviceDynamics):
                raise ValueError("a DeviceCost / DeviceConstraint is compiled into the model "
                                 "library of a DeviceDynamics; write the dynamics as one too")
            spec = dynamics._device_spec(ucost, ucon)
        else:
            spec = dynamics._device_spec()
        cspec = cost._device_spec()
        bspec = constraints._device_spec() if constraints is not None else {}
        keep = []  # host arrays whose pointers the descriptor holds

        def dptr(a, dt=np.float64):
            if a is None:
                return None
            arr = np.ascontiguousarray(np.asarray(a, dtype=dt))
            keep.append(arr)
            return arr.ctypes.data

        d = N.ProblemDesc()
        d.dtype = _dtype_code(torch, self.dtype)
        d.batch, d.horizon, d.nx, d.nu = self.B, self.T, self.nx, self.nu
        d.model = spec["model"]
        for i, v in enumerate(spec.get("dyn_params", [])):
            d.dyn_params[i] = float(v)
        if spec["model"] == N.DYN_LINEAR:
            rows = spec["lin_rows"]
            lin = _linear_device(dynamics, spec, torch, self.dtype, self.device)
            d.lin_a, d.lin_b, d.lin_c = (t.data_ptr() for t in lin)
            keep.extend(lin)
            d.lin_rows, d.lin_batch = rows, 1
        if spec.get("user_data") is not None:
            ud = spec["user_data"]
            d.user_data = ud.data_ptr()
            keep.append(ud)
            self._user_data = ud
        for i, v in enumerate(cspec.get("cost_params", [])):
            d.cost_params[i] = float(v)
        if cspec.get("cost_data") is not None:
            d.cost_data = cspec["cost_data"].data_ptr()
            keep.append(cspec["cost_data"])
            self._cost_data = cspec["cost_data"]
        d.Q = dptr(cspec["Q"])
        d.R = dptr(cspec["R"])
        d.Qf = dptr(cspec["Qf"])
        d.goal = dptr(cspec["goal"])
        for k in ("state_lower", "state_upper", "control_lower", "control_upper"):
            setattr(d, k, dptr(bspec.get(k)))
        if "con_rows_state" in bspec:
            d.con_rows_state = bspec["con_rows_state"]
            d.con_rows_control = bspec["con_rows_control"]
            for i, v in enumerate(bspec["con_params"]):
                d.con_params[i] = float(v)
            if bspec.get("con_data") is not None:
                d.con_data = bspec["con_data"].data_ptr()
                keep.append(bspec["con_data"])
                self._con_data = bspec["con_data"]
        s = settings
        d.method, d.aug, d.aug_mu = s.method, s.aug, s.aug_mu
        d.alpha0, d.nu0, d.inner_tol, d.max_iters = s.alpha0, s.nu0, s.inner_tol, s.max_iters
        d.mu0, d.zeta, d.mu_tol = s.mu0, s.zeta, s.mu_tol
        d.rho, d.residual_tol, d.max_outer = s.rho, s.residual_tol, s.max_outer
        d.hist_cap, d.round_cap = s.hist_cap, max(1, s.round_cap)
        d.keep_round_controls = int(s.keep_round_controls)
        d.chunk0, d.chunk = s.chunk0, s.chunk
        d.rollout = s.rollout
        d.block_mode, d.t_base, d.block_last = s.block_mode, s.t_base, s.block_last
        self.desc = d
        nbytes = self.lib.ptc_solver_workspace_bytes(C.byref(d))
        if nbytes < 0:
            N.check(int(nbytes))
        self.workspace = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        handle = C.c_void_p()
        with torch.cuda.device(self.device):
            N.check(self.lib.ptc_solver_create(C.byref(d), self.workspace.data_ptr(),
                                               nbytes, C.byref(handle)))
        self.handle = handle
        self.W = 0 if constraints is None else int(constraints.n_total)
        del keep

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.lib.ptc_solver_destroy(h)
            except Exception:
                pass
            self.handle = None

    # ------------------------------------------------------------ conversions

    def to_soa(self, arr, rows: int, comps: int):
        """(B, rows, comps) array/tensor -> device (comps, rows, B) contiguous."""
        torch = self.torch
        if isinstance(arr, np.ndarray) and not arr.flags.writeable:
            arr = arr.copy()
        t = torch.as_tensor(arr, dtype=self.dtype)
        if t.dim() == 2:
            t = t.unsqueeze(0)
        if tuple(t.shape) != (self.B, rows, comps):
            raise ValueError(f"expected shape {(self.B, rows, comps)}, got {tuple(t.shape)}")
        return t.to(self.device, non_blocking=True).permute(2, 1, 0).contiguous()

    @staticmethod
    def from_soa(t, comps_shape=None):
        """device (comps, rows, B) -> (B, rows, *comps_shape)."""
        c, rows, B = t.shape
        out = t.permute(2, 1, 0)
        if comps_shape is not None:
            out = out.reshape(B, rows, *comps_shape)
        return out

    # ----------------------------------------------------------------- driver

    @property
    def stream(self) -> int:
        return N.stream_ptr()

    def load(self, states, controls, z=None, v=None):
        X = self.to_soa(states, self.T + 1, self.nx)
        U = self.to_soa(controls, self.T, self.nu)
        zz = self.to_soa(z, self.T, self.W) if z is not None else None
        vv = self.to_soa(v, self.T, self.W) if v is not None else None
        N.check(self.lib.ptc_solver_load(
            self.handle, X.data_ptr(), U.data_ptr(),
            zz.data_ptr() if zz is not None else None,
            vv.data_ptr() if vv is not None else None, 1, self.stream))
        self._keep = (X, U, zz, vv)

    def check_consistency(self) -> np.ndarray:
        bad = np.zeros(self.B, dtype=np.int32)
        N.check(self.lib.ptc_solver_check_consistency(self.handle, bad.ctypes.data, self.stream))
        return bad

    def iterate(self, n: int = 1):
        N.check(self.lib.ptc_solver_iterate(self.handle, int(n), self.stream))

    def block_phase(self, phase: int, inp=None, out=None, aux=None, rank: int = 0,
                    world: int = 1):
        """One phase of a time-sharded iteration (include/pintoc_b200.h)."""
        ptr = lambda t: None if t is None else t.data_ptr()
        N.check(self.lib.ptc_solver_block_phase(self.handle, int(phase), ptr(inp), ptr(out),
                                                ptr(aux), int(rank), int(world), self.stream))

    def running(self) -> int:
        out = C.c_int32(0)
        N.check(self.lib.ptc_solver_running(self.handle, C.byref(out), self.stream))
        return int(out.value)

    def running_async(self, dst) -> None:
        """Enqueue the running count into dst (pinned int32 host tensor)."""
        N.check(self.lib.ptc_solver_running_async(self.handle, dst.data_ptr(), self.stream))

    # False once the driver rejected the conditional graph (then the host
    # polls ptc_solver_running between iteration groups)
    _device_loop = True

    def device_loop(self, max_launch: int, group: int = 1, launched=None) -> bool:
        """Enqueue the device-resident loop unless PTC_HOST_LOOP=1 or the
        driver cannot build it; False = nothing was enqueued."""
        import os
        if os.environ.get("PTC_HOST_LOOP") == "1" or not self._device_loop:
            return False
        try:
            self.loop(max_launch, group, launched)   # a failed build enqueues nothing
        except N.NativeError as err:
            import warnings
            warnings.warn(f"device-resident solve loop unavailable ({err}); "
                          "polling from the host instead", RuntimeWarning, stacklevel=2)
            self._device_loop = False
            return False
        return True

    def loop(self, max_launch: int, group: int = 1, launched=None) -> None:
        """Enqueue the whole solve as one device-resident graph loop
        (ptc_solver_loop); ``launched``: pinned int32 host tensor that
        receives the iteration count once the stream reaches it."""
        ptr = None if launched is None else launched.data_ptr()
        N.check(self.lib.ptc_solver_loop(self.handle, int(group), int(max_launch), ptr,
                                         self.stream))

    def run(self, group: int = 4, max_launch: int | None = None) -> int:
        """Iterate until every problem is done; returns device iterations launched."""
        s = self.settings
        if max_launch is None:
            per_round = s.max_iters + 2
            rounds = max(1, s.max_outer if s.method == N.METHOD_ADMM else 64)
            max_launch = per_round * rounds + 16
        import torch
        cnt = torch.zeros(1, dtype=torch.int32).pin_memory()
        if self.device_loop(max_launch, 1, cnt):
            torch.cuda.current_stream().synchronize()
            return int(cnt[0])
        launched = 0
        n = 1
        while launched < max_launch:
            self.iterate(n)
            launched += n
            if self.running() == 0:
                break
            n = group
        return launched

    # ------------------------------------------------------------------ reads

    def info(self, name: str) -> tuple[int, int]:
        numel, es = C.c_int64(0), C.c_int32(0)
        N.check(self.lib.ptc_solver_buffer_info(self.handle, name.encode(), C.byref(numel),
                                                C.byref(es)))
        return int(numel.value), int(es.value)

    def read(self, name: str):
        """Device copy of a named buffer as a flat torch tensor."""
        torch = self.torch
        numel, es = self.info(name)
        if es == 4 and name not in ("states", "controls", "lam", "P", "R", "M", "d", "Fx",
                                    "Fu", "PT", "S", "s", "Gamma", "gamma", "dx", "du",
                                    "z", "v", "round_controls"):
            dt = torch.int32
        elif name in ("hist", "cur_cost", "cand_cost", "alpha", "nu", "mu", "bad_value", "round_mu",
                      "round_cost", "round_rp", "round_rd"):
            dt = torch.float64
        else:
            dt = self.dtype
        out = torch.empty(numel, dtype=dt, device=self.device)
        N.check(self.lib.ptc_solver_read(self.handle, name.encode(), out.data_ptr(),
                                         numel * es, 1, self.stream))
        return out

    def write(self, name: str, values) -> None:
        """Set per-problem loop state ("alpha", "nu", "mu": float64[B]) after
        load(): the solver then continues exactly as a reference loop that
        enters its next iteration with that state (ptc_solver_write)."""
        a = np.ascontiguousarray(np.broadcast_to(np.asarray(values, np.float64), (self.B,)))
        N.check(self.lib.ptc_solver_write(self.handle, name.encode(), a.ctypes.data, a.nbytes,
                                          0, self.stream))

    def field(self, name: str, rows: int, comps_shape: tuple):
        """Per-stage field as (B, rows, *comps_shape) device tensor."""
        comps = int(np.prod(comps_shape))
        t = self.read(name).view(comps, rows, self.B)
        return self.from_soa(t, comps_shape)

    def states(self):
        return self.field("states", self.T + 1, (self.nx,))[:, : self.T + 1]

    def controls(self):
        return self.field("controls", self.T, (self.nu,))

    def per_problem(self, name: str):
        return self.read(name)

    def rounds(self, name: str):
        """(round_cap, B) record of the outer loop."""
        t = self.read(name)
        return t.view(-1, self.B)

    def history(self):
        """(hist_cap, 5, B) Newton iteration records."""
        t = self.read("hist")
        return t.view(-1, 5, self.B)

    # -------------------------------------------------------------- passes

    def expand(self):
        N.check(self.lib.ptc_solver_expand(self.handle, self.stream))

    def lqr(self, alpha):
        a = np.ascontiguousarray(np.broadcast_to(np.asarray(alpha, np.float64), (self.B,)))
        N.check(self.lib.ptc_solver_lqr(self.handle, a.ctypes.data, self.stream))
        self.torch.cuda.current_stream().synchronize()

    def rollout(self):
        N.check(self.lib.ptc_solver_rollout(self.handle, self.stream))

    def total_cost(self):
        N.check(self.lib.ptc_solver_total_cost(self.handle, self.stream))


def propagate_law(law, exp, dtype=None):
    """Device forward scan of a given feedback law (ptc_propagate)."""
    torch = N.require_cuda()
    lib = N.load_library()
    dtype = dtype or torch.float64
    code = N.PTC_F64 if dtype == torch.float64 else N.PTC_F32
    n, nx, nu = exp.horizon, exp.d_x, exp.d_u
    dev = torch.device("cuda")

    def soa(a, comps):
        t = torch.as_tensor(np.asarray(a, float), dtype=dtype).reshape(n, comps)
        return t.t().contiguous().unsqueeze(-1).to(dev)

    Fx, Fu = soa(exp.Fx, nx * nx), soa(exp.Fu, nx * nu)
    G, g, d = soa(law.Gamma, nu * nx), soa(law.gamma, nu), soa(exp.d, nu)
    dx = torch.empty(nx, n + 1, 1, dtype=dtype, device=dev)
    du = torch.empty(nu, n, 1, dtype=dtype, device=dev)
    nbytes = lib.ptc_lqr_workspace_bytes(code, 1, n, nx, nu, 0, 0)
    ws = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
    N.check(lib.ptc_propagate(code, 1, n, nx, nu, Fx.data_ptr(), Fu.data_ptr(), G.data_ptr(),
                              g.data_ptr(), d.data_ptr(), dx.data_ptr(), du.data_ptr(),
                              ws.data_ptr(), ws.numel(), 0, 0, N.stream_ptr()))
    return (dx[..., 0].t().cpu().numpy(), du[..., 0].t().cpu().numpy())
