// Newton kernel sets of the pendulum and cart-pole models, double
#include "inst_common.cuh"
PTC_REG_PENDULUM(double)
PTC_REG_CARTPOLE(double)
