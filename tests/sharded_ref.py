"""Numpy block ops for the time-sharded driver -- TEST INFRASTRUCTURE ONLY.

Implements the same three block phases as ``CudaBlockOps`` with the CPU
oracle's element constructors and combine rules (oracle/pintoc_oracle.py),
so the sharded driver's decomposition and its all-gather plumbing can be
checked on CPU with a gloo process group.  Never used by the product.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import pintoc_oracle as O


def _flat_velem(e):
    A, Y, C, eta, b = e
    return np.concatenate([A.ravel(), Y.ravel(), C.ravel(), eta, b])


def _unflat_velem(v, nx):
    k = nx * nx
    return (v[:k].reshape(nx, nx), v[k:2 * k].reshape(nx, nx), v[2 * k:3 * k].reshape(nx, nx),
            v[3 * k:3 * k + nx], v[3 * k + nx:3 * k + 2 * nx])


class NumpyBlockOps:
    """Rank `rank`'s block [t_base, t_base + T) of a full expansion `exp`."""

    def __init__(self, exp, rank, world, t_base, T):
        self.exp, self.rank, self.world, self.t0, self.T = exp, rank, world, t_base, T
        self.nx = exp.P.shape[1]
        A, Y, C, eta, b = O.value_elements(exp)
        n = exp.P.shape[0]
        sl = slice(t_base, t_base + T)
        self.elems = [(A[t], Y[t], C[t], eta[t], b[t]) for t in range(n + 1)][sl]
        self.last = rank == world - 1
        if self.last:
            self.elems.append((A[n], Y[n], C[n], eta[n], b[n]))

    def value_up(self):
        acc = self.elems[-1]
        for e in reversed(self.elems[:-1]):
            acc = O.value_combine(e, acc)
        return torch.as_tensor(_flat_velem(acc))[:, None, None]

    def value_down(self, gathered):
        nx, exp = self.nx, self.exp
        g = gathered.reshape(self.world, -1).numpy()
        z = np.zeros((nx, nx))
        carry = (z, z, z, np.zeros(nx), np.zeros(nx))
        for r in range(self.world - 1, self.rank, -1):
            carry = O.value_combine(_unflat_velem(g[r], nx), carry)
            carry = (z, carry[1], z, carry[3], np.zeros(nx))
        T, t0 = self.T, self.t0
        S = np.empty((T + 1, nx, nx))
        s = np.empty((T + 1, nx))
        acc = carry
        if self.last:
            acc = O.value_combine(self.elems[-1], acc)
        S[T], s[T] = acc[1], -acc[3]
        for k in range(T - 1, -1, -1):
            acc = O.value_combine(self.elems[k], acc)
            S[k], s[k] = acc[1], -acc[3]
        sl = slice(t0, t0 + T)
        Fu, Fx, M, d = exp.Fu[sl], exp.Fx[sl], exp.M[sl], exp.d[sl]
        Rr = exp.Rr[sl]
        FuTS = np.swapaxes(Fu, 1, 2) @ S[1:]
        Q = 0.5 * (Rr + FuTS @ Fu + np.swapaxes(Rr + FuTS @ Fu, 1, 2))
        self.Gamma = -np.linalg.solve(Q, np.swapaxes(M, 1, 2) + FuTS @ Fx)
        self.gamma = -np.linalg.solve(Q, (d + np.einsum("tkj,tk->tj", Fu, s[1:]))[..., None])[..., 0]
        self.S, self.s = S, s
        self.F = Fx + Fu @ self.Gamma
        if t0 == 0:
            self.F[0] = 0.0
        self.e = np.einsum("tij,tj->ti", Fu, self.gamma)
        Fa, ea = np.eye(nx), np.zeros(nx)
        for k in range(T):
            Fa, ea = self.F[k] @ Fa, self.F[k] @ ea + self.e[k]
        return torch.as_tensor(np.concatenate([Fa.ravel(), ea]))[:, None, None]

    def propagate(self, gathered):
        nx = self.nx
        g = gathered.reshape(self.world, -1).numpy()
        x = np.zeros(nx)
        for r in range(self.rank):
            x = g[r][:nx * nx].reshape(nx, nx) @ x + g[r][nx * nx:]
        dx = np.empty((self.T + 1, nx))
        dx[0] = x
        for k in range(self.T):
            dx[k + 1] = self.F[k] @ dx[k] + self.e[k]
        self.dx = dx
        self.du = np.einsum("tij,tj->ti", self.Gamma, dx[:-1]) + self.gamma
