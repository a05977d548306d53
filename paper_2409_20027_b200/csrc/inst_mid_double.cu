// nx = 6, 8 kernel sets, double
#include "inst_common.cuh"
PTC_REG_LQR(double, 6, 3) PTC_REG_LQR(double, 8, 4)
PTC_REG_AFFINE(double, 6, 3) PTC_REG_AFFINE(double, 8, 4)
