// Newton kernel sets of affine models nx = 6, 8, double
#include "inst_common.cuh"
PTC_REG_AFFINE(double, 6, 3) PTC_REG_AFFINE(double, 8, 4)
