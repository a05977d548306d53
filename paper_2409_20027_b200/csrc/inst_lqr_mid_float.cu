// LQR kernel sets nx = 6, 8, float
#include "inst_common.cuh"
PTC_REG_LQR(float, 6, 3) PTC_REG_LQR(float, 8, 4)
