// Newton kernel sets of affine models nx = 12, double
#include "inst_common.cuh"
PTC_REG_AFFINE(double, 12, 4) PTC_REG_AFFINE(double, 12, 6)
