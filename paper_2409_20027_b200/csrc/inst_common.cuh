// Explicit instantiation helpers: each inst_*.cu registers the kernel sets
// it compiles (static registration objects run when the library loads).
#pragma once
#include "launch.cuh"

#define PTC_REG_LQR(R, NX, NU) \
  static ptc::RegisterLqr<R, NX, NU> _reg_lqr_##NX##_##NU##_##R;
#define PTC_REG_AFFINE(R, NX, NU) \
  static ptc::RegisterNewton<R, ptc::Affine<R, NX, NU>, ptc::DYN_LINEAR> _reg_aff_##NX##_##NU##_##R;
#define PTC_REG_PENDULUM(R) \
  static ptc::RegisterNewton<R, ptc::Pendulum<R>, ptc::DYN_PENDULUM> _reg_pend_##R;
#define PTC_REG_CARTPOLE(R) \
  static ptc::RegisterNewton<R, ptc::CartPole<R>, ptc::DYN_CARTPOLE> _reg_cp_##R;
