"""User-defined device models used by the tests: the reference's own
user-model pattern (a DynamicsModel subclass, e.g. make_golden.py's
TVLinear) written against the device hook (usermodel.DeviceDynamics)."""

from paper_2409_20027_b200.usermodel import DeviceDynamics

# the reference pendulum (systems.py:161-231) as user code:
# prm = (g, l, m, b, dt)
PEND_STEP = """
    const R g = R(prm[0]), l = R(prm[1]), m = R(prm[2]), bd = R(prm[3]), dt = R(prm[4]);
    R acc = -(g / l) * sin(x[0]) + (u[0] - bd * x[1]) / (m * (l * l));
    xn[0] = x[0] + dt * x[1];
    xn[1] = x[1] + dt * acc;
"""
PEND_JAC = """
    const R g = R(prm[0]), l = R(prm[1]), m = R(prm[2]), bd = R(prm[3]), dt = R(prm[4]);
    fx[0][0] = R(1);
    fx[0][1] = dt;
    fx[1][0] = -dt * (g / l) * cos(x[0]);
    fx[1][1] = R(1) - dt * bd / (m * (l * l));
    fu[1][0] = dt / (m * (l * l));
"""
PEND_HESS = """
    const R g = R(prm[0]), l = R(prm[1]), dt = R(prm[4]);
    fxx[1][0][0] = dt * (g / l) * sin(x[0]);
"""


def user_pendulum(T, g=9.81, l=1.0, m=1.0, b=0.1, dt=0.05):
    return DeviceDynamics(T, 2, 1, step=PEND_STEP, jacobian=PEND_JAC, hessian=PEND_HESS,
                          params=(g, l, m, b, dt), name="pendulum")


# time-varying affine x' = A_t x + B_t u + c_t (make_golden.py TVLinear):
# data = [A (T, nx, nx) | B (T, nx, nu) | c (T, nx)], prm[0] = T
TVL_STEP = """
    const int T = int(prm[0]);
    const double* A = data + (size_t)t * NX * NX;
    const double* Bm = data + (size_t)T * NX * NX + (size_t)t * NX * NU;
    const double* c = data + (size_t)T * (NX * NX + NX * NU) + (size_t)t * NX;
    for (int i = 0; i < NX; ++i) {
      R ax = R(0), bu = R(0);
      for (int j = 0; j < NX; ++j) ax += R(A[i * NX + j]) * x[j];
      for (int k = 0; k < NU; ++k) bu += R(Bm[i * NU + k]) * u[k];
      xn[i] = ax + bu + R(c[i]);
    }
"""
TVL_JAC = """
    const int T = int(prm[0]);
    const double* A = data + (size_t)t * NX * NX;
    const double* Bm = data + (size_t)T * NX * NX + (size_t)t * NX * NU;
    for (int i = 0; i < NX; ++i) {
      for (int j = 0; j < NX; ++j) fx[i][j] = R(A[i * NX + j]);
      for (int k = 0; k < NU; ++k) fu[i][k] = R(Bm[i * NU + k]);
    }
"""


def user_tvlinear(A, B, c):
    import numpy as np
    T, nx, nu = B.shape
    data = np.concatenate([A.reshape(-1), B.reshape(-1), c.reshape(-1)])
    return DeviceDynamics(T, nx, nu, step=TVL_STEP, jacobian=TVL_JAC, params=(T,), data=data,
                          name="tvlinear")


def precompile():
    """Build the test models' libraries (build() does this so GPU runs load
    them without compiling)."""
    import numpy as np
    paths = [user_pendulum(8).library(), user_pendulum(8).library(user_cosine_cost()),
             user_pendulum(8).library(None, user_norm_constraints())]
    for nx, nu in ((4, 2),):
        z = np.zeros((3, nx, nx)), np.zeros((3, nx, nu)), np.zeros((3, nx))
        paths.append(user_tvlinear(*z).library())
    return paths


# make_golden.py's CosineCost (a user CostModel in pintoc) as device code:
# prm = (w0, w1, r, W0, W1)
COS_STAGE = "l = R(prm[0]) * (R(1) - cos(x[0])) + R(0.5 * prm[1]) * x[1] * x[1]" \
            " + R(0.5 * prm[2]) * u[0] * u[0];"
COS_GRAD = """
    lx[0] = R(prm[0]) * sin(x[0]);
    lx[1] = R(prm[1]) * x[1];
    lu[0] = R(prm[2]) * u[0];
    lxx[0][0] = R(prm[0]) * cos(x[0]);
    lxx[1][1] = R(prm[1]);
    luu[0][0] = R(prm[2]);
"""
COS_TERM = "V = R(prm[3]) * (R(1) - cos(x[0])) + R(0.5 * prm[4]) * x[1] * x[1];"
COS_TERM_GRAD = """
    Vx[0] = R(prm[3]) * sin(x[0]);
    Vx[1] = R(prm[4]) * x[1];
    Vxx[0][0] = R(prm[3]) * cos(x[0]);
    Vxx[1][1] = R(prm[4]);
"""


def user_cosine_cost(w0=10.0, w1=0.1, r=0.01, W0=100.0, W1=10.0):
    from paper_2409_20027_b200.usermodel import DeviceCost
    return DeviceCost(stage=COS_STAGE, gradients=COS_GRAD, terminal=COS_TERM,
                      terminal_gradients=COS_TERM_GRAD, params=(w0, w1, r, W0, W1),
                      name="cosine")


# make_golden.py's NormConstraints (a user ConstraintModel in pintoc):
# g(x) = [omega^2 - wmax^2], h(u) = [u^2 - umax^2]; prm = (wmax, umax)
NORM_G = "g[0] = x[1] * x[1] - R(prm[0] * prm[0]);"
NORM_G_D = "gx[0][1] = R(2) * x[1]; gxx[0][1][1] = R(2);"
NORM_H = "h[0] = u[0] * u[0] - R(prm[1] * prm[1]);"
NORM_H_D = "hu[0][0] = R(2) * u[0]; huu[0][0][0] = R(2);"


def user_norm_constraints(wmax=8.0, umax=5.0):
    from paper_2409_20027_b200.usermodel import DeviceConstraint
    return DeviceConstraint(1, 1, g=NORM_G, g_derivs=NORM_G_D, h=NORM_H, h_derivs=NORM_H_D,
                            params=(wmax, umax), name="norm")
