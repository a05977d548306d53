// LQR kernel sets nx <= 4, float
#include "inst_common.cuh"
PTC_REG_LQR(float, 1, 1) PTC_REG_LQR(float, 1, 2) PTC_REG_LQR(float, 1, 3)
PTC_REG_LQR(float, 2, 1) PTC_REG_LQR(float, 2, 2) PTC_REG_LQR(float, 2, 3)
PTC_REG_LQR(float, 3, 1) PTC_REG_LQR(float, 3, 2) PTC_REG_LQR(float, 3, 3)
PTC_REG_LQR(float, 4, 1) PTC_REG_LQR(float, 4, 2)
