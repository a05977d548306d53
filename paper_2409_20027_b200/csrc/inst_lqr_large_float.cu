// LQR kernel sets nx = 12, float
#include "inst_common.cuh"
PTC_REG_LQR(float, 12, 4) PTC_REG_LQR(float, 12, 6)
