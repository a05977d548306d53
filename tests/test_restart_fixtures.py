"""CPU checks of the restart-parity fixtures (tests/golden/make_restart.py).

* The records form one consistent chain: each iteration enters with the
  trajectory and (alpha, nu) the previous one left.
* The oracle, restarted from every recorded config-0 state, takes the
  reference's step (the same restart test the device passes in
  test_gpu_restart.py, here pinning the oracle per iteration).
* Config 2's z, v entering each outer step are re-derived from the recorded
  trajectories exactly as the reference updates them; the re-derivation is
  bitwise equal to the reference's checkpoints.
"""

import math

import numpy as np
import pytest
from conftest import golden

from oracle import pintoc_oracle as O


def _chain_ok(g, prefix=""):
    tin, tout = g[prefix + "it_in"], g[prefix + "it_out"]
    aug = g[prefix + "it_aug"]
    term = g[prefix + "it_term"]
    for i in range(1, len(tin)):
        if aug[i] == aug[i - 1] and term[i - 1] == 0:      # same Newton solve, continuing
            assert tin[i] == tout[i - 1], i
            assert g[prefix + "it_alpha"][i] == g[prefix + "it_alpha_next"][i - 1], i
            assert g[prefix + "it_nu"][i] == g[prefix + "it_nu_next"][i - 1], i


@pytest.mark.parametrize("name", ["restart_cfg0", "restart_cfg4"])
def test_chain_consistent(name):
    g = golden(name)
    _chain_ok(g)
    # the last record's trajectory is the reference's final solution
    assert np.array_equal(g["traj_u"][g["it_out"][-1]], g["final_u"])


def test_config0_oracle_takes_every_reference_step():
    g = golden("restart_cfg0")
    dyn = O.Pendulum(damping=0.1, dt=0.05)
    cost = O.Quadratic(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0]))
    box = O.Box(2, 1, control_lower=-5.0, control_upper=5.0)
    X, U = g["traj_x"], g["traj_u"]
    hist, tout = g["it_hist"], g["it_out"]
    flips = 0
    for i in range(0, len(hist), 3):      # every third iteration keeps the CPU suite short
        r = O.newton_solve(dyn, cost, ("barrier", box, float(g["it_aug"][i])),
                           X[g["it_in"][i]], U[g["it_in"][i]], alpha0=float(g["it_alpha"][i]),
                           nu0=float(g["it_nu"][i]), max_iters=1, check=False)
        c, a, ratio, step, acc = r.history[0]
        ref = hist[i]
        if bool(acc) != bool(ref[4]):
            flips += 1
            continue
        assert a == ref[1]
        assert abs(c - ref[0]) <= 1e-9 * max(1.0, abs(ref[0]))
        if math.isfinite(ref[3]):
            assert abs(step - ref[3]) <= 1e-9 * max(1.0, abs(ref[3]))
        assert np.abs(r.us - U[tout[i]]).max() <= 1e-9 * max(1.0, np.abs(U[tout[i]]).max())
    assert flips == 0


def test_config2_dual_states_rederived_bitwise():
    g = golden("restart_cfg2")
    from restart_util import admm_states, cfg2_box_oracle
    z, v = admm_states(g, cfg2_box_oracle())
    for k in (0, 1, 50, 100, 199):
        if f"z_{k}" in g.files and k < len(z):
            assert np.array_equal(z[k], g[f"z_{k}"]), k
            assert np.array_equal(v[k], g[f"v_{k}"]), k
    _chain_ok(g)


def test_config3_sample_fixture_shape():
    g = golden("cfg3_sample")
    stalled = sum(int((g[f"{s}_cold_status"] == -1).sum()) for s in ("pendulum", "cartpole"))
    assert stalled >= 16
    assert g["pendulum_cold_round_in_x"].shape[1:] == (8, 257, 2)
