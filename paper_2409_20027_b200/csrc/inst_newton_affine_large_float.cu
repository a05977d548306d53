// Newton kernel sets of affine models nx = 12, float
#include "inst_common.cuh"
PTC_REG_AFFINE(float, 12, 4) PTC_REG_AFFINE(float, 12, 6)
