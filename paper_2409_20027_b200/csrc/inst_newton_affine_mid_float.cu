// Newton kernel sets of affine models nx = 6, 8, float
#include "inst_common.cuh"
PTC_REG_AFFINE(float, 6, 3) PTC_REG_AFFINE(float, 8, 4)
