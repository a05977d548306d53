"""Reproducibility floors of the reference for the restart fixtures, from
more nudges: re-run each recorded Newton solve (config-2 outer steps,
config-3 barrier rounds) with the entering trajectory moved by k = 1, 2, 3
ulps either way (six runs) and record how far the reference's own result
moves and whether its iteration count changes.  Rewrites the `step_floor` /
`step_stable` (restart_cfg2.npz) and `<sys>_<leg>_floor` / `_stable`
(cfg3_sample.npz) arrays in place.

    python tests/golden/make_floors.py [--workers 7]
"""

import argparse
import math
import multiprocessing as mp
import os
import sys
import time

import numpy as np

OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, OUT)
sys.path.insert(0, os.path.dirname(OUT))
import make_restart as MR  # noqa: E402  (imports the reference, read-only)
from make_restart import (AdmmAugmentation, BarrierAugmentation, NewtonOptions,  # noqa: E402
                          newton_chain, rollout)

ULPS = (1, 2, 3)


def nudged(dyn, states, controls, k, sign):
    x0, u = states[0].copy(), controls.copy()
    d = np.inf if sign > 0 else -np.inf
    for _ in range(k):
        x0, u = np.nextafter(x0, d), np.nextafter(u, d)
    return rollout(dyn, x0, u)


def floor_of(dyn, cost, aug, states, controls, opts, count, out_x, out_u):
    fl, stable = 0.0, True
    for k in ULPS:
        for sign in (1, -1):
            try:
                t2, n2, _, _, _, err = newton_chain(dyn, cost, aug,
                                                    nudged(dyn, states, controls, k, sign), opts)
            except Exception:
                return math.inf, False
            if err:
                return math.inf, False
            stable = stable and n2 == count
            for a, b in ((t2.states, out_x), (t2.controls, out_u)):
                fl = max(fl, float(np.abs(a - b).max() / max(1.0, np.abs(b).max())))
    return fl, stable


_JOB = None


def _cfg2(k):
    g, zv, prob = _JOB
    z, v = zv[0][k], zv[1][k]
    aug = AdmmAugmentation(prob.constraints, 1.0, z, v)
    X, U = g["step_traj_x"], g["step_traj_u"]
    return floor_of(prob.dynamics, prob.cost, aug, X[k], U[k], NewtonOptions(), int(g["step_iters"][k]),
                    X[k + 1], U[k + 1])


def _cfg3(job):
    system, leg, j, r, mu = job
    g = _JOB
    prob = MR.cfg3_problem(system)
    p = f"{system}_{leg}_"
    nr = int(g[p + "nrounds"][j])
    last = r == nr - 1
    out_x = g[p + "final_x"][j] if last else g[p + "round_in_x"][j, r + 1]
    out_u = g[p + "final_u"][j] if last else g[p + "round_in_u"][j, r + 1]
    aug = BarrierAugmentation(prob.constraints, mu)
    return floor_of(prob.dynamics, prob.cost, aug, g[p + "round_in_x"][j, r],
                    g[p + "round_in_u"][j, r], MR.CFG3_OPTS.newton, int(g[p + "iters"][j, r]),
                    out_x, out_u)


def main():
    global _JOB
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=7)
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    if args.only in (None, "cfg3"):
        path = os.path.join(OUT, "cfg3_sample.npz")
        g = dict(np.load(path))
        _JOB = g
        mus = list(g["mu_schedule"])
        jobs = []
        for system in ("pendulum", "cartpole"):
            for leg in ("cold", "warm"):
                p = f"{system}_{leg}_"
                for j, nr in enumerate(g[p + "nrounds"]):
                    for r in range(int(nr)):
                        if r == nr - 1 and g[p + "status"][j] == -1:
                            continue
                        jobs.append((system, leg, j, r, mus[r]))
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(args.workers) as pool:
            res = pool.map(_cfg3, jobs, chunksize=1)
        for (system, leg, j, r, _), (fl, st) in zip(jobs, res):
            p = f"{system}_{leg}_"
            g[p + "floor"][j, r] = fl
            g[p + "stable"][j, r] = st
        np.savez_compressed(path, **g)
        print(f"cfg3 floors: {len(jobs)} rounds, {time.perf_counter() - t0:.0f}s", flush=True)
    if args.only in (None, "cfg2"):
        path = os.path.join(OUT, "restart_cfg2.npz")
        g = dict(np.load(path))
        sys.path.insert(0, os.path.join(os.path.dirname(OUT)))
        from restart_util import admm_states, cfg2_box_oracle
        zv = admm_states(g, cfg2_box_oracle())
        prob = MR.cartpole_cfg2(500)
        _JOB = (g, zv, prob)
        n = len(g["step_iters"])
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(args.workers) as pool:
            res = pool.map(_cfg2, range(n), chunksize=1)
        g["step_floor"] = np.array([f for f, _ in res])
        g["step_stable"] = np.array([s for _, s in res])
        np.savez_compressed(path, **g)
        print(f"cfg2 floors: {n} steps, {time.perf_counter() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    main()
