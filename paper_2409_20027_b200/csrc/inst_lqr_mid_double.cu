// LQR kernel sets nx = 6, 8, double
#include "inst_common.cuh"
PTC_REG_LQR(double, 6, 3) PTC_REG_LQR(double, 8, 4)
