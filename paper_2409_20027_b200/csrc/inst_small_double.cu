// nx <= 4 kernel sets, double
#include "inst_common.cuh"
PTC_REG_PENDULUM(double)
PTC_REG_CARTPOLE(double)
PTC_REG_LQR(double, 1, 1) PTC_REG_LQR(double, 1, 2) PTC_REG_LQR(double, 1, 3)
PTC_REG_LQR(double, 2, 1) PTC_REG_LQR(double, 2, 2) PTC_REG_LQR(double, 2, 3)
PTC_REG_LQR(double, 3, 1) PTC_REG_LQR(double, 3, 2) PTC_REG_LQR(double, 3, 3)
PTC_REG_LQR(double, 4, 1) PTC_REG_LQR(double, 4, 2)
PTC_REG_AFFINE(double, 1, 1) PTC_REG_AFFINE(double, 1, 2) PTC_REG_AFFINE(double, 1, 3)
PTC_REG_AFFINE(double, 2, 1) PTC_REG_AFFINE(double, 2, 2) PTC_REG_AFFINE(double, 2, 3)
PTC_REG_AFFINE(double, 3, 1) PTC_REG_AFFINE(double, 3, 2) PTC_REG_AFFINE(double, 3, 3)
PTC_REG_AFFINE(double, 4, 1) PTC_REG_AFFINE(double, 4, 2)
