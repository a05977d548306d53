// nx = 12 kernel sets, float
#include "inst_common.cuh"
PTC_REG_LQR(float, 12, 4) PTC_REG_LQR(float, 12, 6)
PTC_REG_AFFINE(float, 12, 4) PTC_REG_AFFINE(float, 12, 6)
