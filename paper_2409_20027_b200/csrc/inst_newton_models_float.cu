// Newton kernel sets of the pendulum and cart-pole models, float
#include "inst_common.cuh"
PTC_REG_PENDULUM(float)
PTC_REG_CARTPOLE(float)
