// LQR kernel sets nx <= 4, double
#include "inst_common.cuh"
PTC_REG_LQR(double, 1, 1) PTC_REG_LQR(double, 1, 2) PTC_REG_LQR(double, 1, 3)
PTC_REG_LQR(double, 2, 1) PTC_REG_LQR(double, 2, 2) PTC_REG_LQR(double, 2, 3)
PTC_REG_LQR(double, 3, 1) PTC_REG_LQR(double, 3, 2) PTC_REG_LQR(double, 3, 3)
PTC_REG_LQR(double, 4, 1) PTC_REG_LQR(double, 4, 2)
