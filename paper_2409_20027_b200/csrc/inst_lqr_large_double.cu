// LQR kernel sets nx = 12, double
#include "inst_common.cuh"
PTC_REG_LQR(double, 12, 4) PTC_REG_LQR(double, 12, 6)
