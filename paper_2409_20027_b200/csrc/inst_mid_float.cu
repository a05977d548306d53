// nx = 6, 8 kernel sets, float
#include "inst_common.cuh"
PTC_REG_LQR(float, 6, 3) PTC_REG_LQR(float, 8, 4)
PTC_REG_AFFINE(float, 6, 3) PTC_REG_AFFINE(float, 8, 4)
