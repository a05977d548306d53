"""GPU parity of the fused co-state / expansion kernels (Alg. 1 + the
quadratic expansion) on the nonlinear models, all three augmentations,
against the reference's outputs."""

import math

import numpy as np
import pytest
from conftest import golden, rel_gap

pytestmark = pytest.mark.gpu


def _models(P):
    pend = P.PendulumDynamics(24, P.PendulumParams(damping=0.1, dt=0.05))
    pcost = P.QuadraticCost(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0]))
    pbox = P.BoxConstraint(2, 1, control_lower=-5.0, control_upper=5.0)
    cp = P.CartPoleDynamics(24, P.CartPoleParams(cart_mass=1.0, pole_mass=0.1,
                                                 pole_length=0.5, dt=0.02))
    Q = np.diag([1.0, 10.0, 0.1, 0.1])
    ccost = P.QuadraticCost(Q, np.diag([0.01]), 10 * Q, x_goal=np.array([0.0, math.pi, 0.0, 0.0]))
    cbox = P.BoxConstraint(4, 1, control_lower=-10.0, control_upper=10.0,
                           state_lower=[-1.5, -np.inf, -np.inf, -np.inf],
                           state_upper=[1.5, np.inf, np.inf, np.inf])
    return {"pendulum": (pend, pcost, pbox), "cartpole": (cp, ccost, cbox)}


@pytest.mark.parametrize("name", ["pendulum", "cartpole"])
@pytest.mark.parametrize("aug_name", ["zero", "barrier", "admm"])
def test_costate_and_expansion_match_reference(name, aug_name):
    import paper_2409_20027_b200 as P
    g = golden("passes_models")
    dyn, cost, box = _models(P)[name]
    traj = P.Trajectory(g[f"{name}_xs"], g[f"{name}_us"])
    aug = {"zero": P.ZeroAugmentation(),
           "barrier": P.BarrierAugmentation(box, 0.1),
           "admm": P.AdmmAugmentation(box, 0.7, g[f"{name}_z"], g[f"{name}_v"])}[aug_name]
    key = f"{name}_{aug_name}_"
    lam = P.costate_pass(traj, cost, aug, dyn)
    assert rel_gap(lam, g[key + "lam"]) < 1e-12
    exp = P.hamiltonian_expansion(traj, lam, cost, aug, dyn, alpha=0.5)
    for f, val in dict(P=exp.P, R=exp.R, M=exp.M, d=exp.d, Fx=exp.Fx, Fu=exp.Fu,
                       PT=exp.P_terminal).items():
        assert rel_gap(val, g[key + f]) < 1e-12, f
    c = P.total_cost(cost, aug, traj, dyn=dyn)
    ref = float(g[key + "cost"])
    assert abs(c - ref) <= 1e-11 * max(1.0, abs(ref))
