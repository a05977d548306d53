// nx = 12 kernel sets, double
#include "inst_common.cuh"
PTC_REG_LQR(double, 12, 4) PTC_REG_LQR(double, 12, 6)
PTC_REG_AFFINE(double, 12, 4) PTC_REG_AFFINE(double, 12, 6)
