// Scan elements of the three Newton passes and their associative operators.
//
//  * value elements (A, Y, C, eta, b): dual form of a conditional value
//    function (reference passes.py:38-46, element init 244-261, combine
//    264-288).  `vcombine` is the general operator (tree interior nodes);
//    `vcombine_stage` the same with a single-stage left operand in Woodbury
//    form (level-0 up-sweep); `vstep` the operator specialised to a right
//    operand with A = C = b = 0 (every suffix containing the terminal has
//    that shape: tree down-sweep); `riccati_step` = vstep of a single stage
//    fused with that stage's gains (level-0 down-sweep).
//  * affine maps (F, e): x -> F x + e.  Propagation (passes.py:330-361) and
//    linear rollout compose them forwards; the co-state suffix
//    (passes.py:113-148) composes them backwards with F = fx^T.
#pragma once

#include "linalg.cuh"

namespace ptc {

// ---------------------------------------------------------------------------
// SoA field access: field[(c * rows + t) * B + b]
// ---------------------------------------------------------------------------

template <typename R>
PTC_D R ldf(const R* __restrict__ f, int c, int t, int rows, int B, int b) {
  return __ldg(f + ((size_t)c * rows + t) * B + b);
}

template <typename R>
PTC_D void stf(R* __restrict__ f, int c, int t, int rows, int B, int b, R v) {
  f[((size_t)c * rows + t) * B + b] = v;
}

template <int M, int N, typename R>
PTC_D void ld_mat(const R* f, int t, int rows, int B, int b, R (&A)[M][N], int c0 = 0) {
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) A[i][j] = ldf(f, c0 + i * N + j, t, rows, B, b);
}

template <int N, typename R>
PTC_D void ld_vec(const R* f, int t, int rows, int B, int b, R (&a)[N], int c0 = 0) {
#pragma unroll
  for (int i = 0; i < N; ++i) a[i] = ldf(f, c0 + i, t, rows, B, b);
}

template <int M, int N, typename R>
PTC_D void st_mat(R* f, int t, int rows, int B, int b, const R (&A)[M][N], int c0 = 0) {
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) stf(f, c0 + i * N + j, t, rows, B, b, A[i][j]);
}

template <int N, typename R>
PTC_D void st_vec(R* f, int t, int rows, int B, int b, const R (&a)[N], int c0 = 0) {
#pragma unroll
  for (int i = 0; i < N; ++i) stf(f, c0 + i, t, rows, B, b, a[i]);
}

// ---------------------------------------------------------------------------
// value elements
// ---------------------------------------------------------------------------

template <typename R, int NX>
struct VElem {
  R A[NX][NX], Y[NX][NX], C[NX][NX], eta[NX], b[NX];
  static constexpr int kComp = 3 * NX * NX + 2 * NX;
};

template <typename R, int NX>
struct VCarry {  // value function of a suffix containing the terminal
  R Y[NX][NX], eta[NX];
  static constexpr int kComp = NX * NX + NX;
};

template <typename R, int NX>
PTC_D void ld_velem(const R* f, int t, int rows, int B, int b, VElem<R, NX>& e) {
  ld_mat(f, t, rows, B, b, e.A, 0);
  ld_mat(f, t, rows, B, b, e.Y, NX * NX);
  ld_mat(f, t, rows, B, b, e.C, 2 * NX * NX);
  ld_vec(f, t, rows, B, b, e.eta, 3 * NX * NX);
  ld_vec(f, t, rows, B, b, e.b, 3 * NX * NX + NX);
}

template <typename R, int NX>
PTC_D void st_velem(R* f, int t, int rows, int B, int b, const VElem<R, NX>& e) {
  st_mat(f, t, rows, B, b, e.A, 0);
  st_mat(f, t, rows, B, b, e.Y, NX * NX);
  st_mat(f, t, rows, B, b, e.C, 2 * NX * NX);
  st_vec(f, t, rows, B, b, e.eta, 3 * NX * NX);
  st_vec(f, t, rows, B, b, e.b, 3 * NX * NX + NX);
}

template <typename R, int NX>
PTC_D void ld_vcarry(const R* f, int t, int rows, int B, int b, VCarry<R, NX>& c) {
  ld_mat(f, t, rows, B, b, c.Y, 0);
  ld_vec(f, t, rows, B, b, c.eta, NX * NX);
}

template <typename R, int NX>
PTC_D void st_vcarry(R* f, int t, int rows, int B, int b, const VCarry<R, NX>& c) {
  st_mat(f, t, rows, B, b, c.Y, 0);
  st_vec(f, t, rows, B, b, c.eta, NX * NX);
}

template <typename R, int NX>
PTC_D void vcarry_zero(VCarry<R, NX>& c) {
  set_zero(c.Y);
  set_zero(c.eta);
}

// Per-stage expansion data entering the subproblem (reference passes.py:62-97)
template <typename R, int NX, int NU>
struct Stage {
  R P[NX][NX], Rr[NU][NU], M[NX][NU], d[NU], Fx[NX][NX], Fu[NX][NU];
};

template <typename R, int NX, int NU>
PTC_D void ld_stage(const R* P, const R* Rm, const R* M, const R* d, const R* Fx, const R* Fu,
                    int t, int T, int B, int b, R alpha, Stage<R, NX, NU>& s) {
  // P and R are symmetric (reference passes.py:178-179 symmetrises them; the
  // StageExpansion invariant): load the upper triangles and mirror
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = i; j < NX; ++j) s.P[i][j] = s.P[j][i] = ldf(P, i * NX + j, t, T, B, b);
#pragma unroll
  for (int i = 0; i < NU; ++i)
#pragma unroll
    for (int j = i; j < NU; ++j) s.Rr[i][j] = s.Rr[j][i] = ldf(Rm, i * NU + j, t, T, B, b);
#pragma unroll
  for (int i = 0; i < NU; ++i) s.Rr[i][i] += alpha;
  ld_mat(M, t, T, B, b, s.M);
  ld_vec(d, t, T, B, b, s.d);
  ld_mat(Fx, t, T, B, b, s.Fx);
  ld_mat(Fu, t, T, B, b, s.Fu);
}

// Dual element of one stage (reference passes.py:192-228 / 244-261):
//   A = Fx - Fu Rr^-1 M^T,  Y = P - M Rr^-1 M^T,  C = Fu Rr^-1 Fu^T,
//   eta = M Rr^-1 d,        b = -Fu Rr^-1 d.
// Also returns the Cholesky factor of Rr (reused by the gains).
template <typename R, int NX, int NU>
PTC_D bool velem_from_stage(const Stage<R, NX, NU>& s, VElem<R, NX>& e, R (&L)[NU][NU]) {
#pragma unroll
  for (int i = 0; i < NU; ++i)
#pragma unroll
    for (int j = 0; j < NU; ++j) L[i][j] = s.Rr[i][j];
  bool ok = cholesky<NU>(L);
  R RiMt[NU][NX], RiFt[NU][NX], Rid[NU];
#pragma unroll
  for (int i = 0; i < NU; ++i) {
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      RiMt[i][j] = s.M[j][i];
      RiFt[i][j] = s.Fu[j][i];
    }
    Rid[i] = s.d[i];
  }
  chol_solve<NU, NX>(L, RiMt);
  chol_solve<NU, NX>(L, RiFt);
  chol_solve_vec<NU>(L, Rid);
  R tmp[NX][NX];
  mm<NX, NU, NX>(s.Fu, RiMt, tmp);
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) e.A[i][j] = s.Fx[i][j] - tmp[i][j];
  mm<NX, NU, NX>(s.M, RiMt, tmp);
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) e.Y[i][j] = s.P[i][j] - tmp[i][j];
  symmetrize<NX>(e.Y);
  mm<NX, NU, NX>(s.Fu, RiFt, e.C);
  symmetrize<NX>(e.C);
  mv<NX, NU>(s.M, Rid, e.eta);
  mv<NX, NU>(s.Fu, Rid, e.b);
#pragma unroll
  for (int i = 0; i < NX; ++i) e.b[i] = -e.b[i];
  return ok;
}

template <typename R, int NX>
PTC_D void velem_terminal(const R (&PT)[NX][NX], VElem<R, NX>& e) {
  set_zero(e.A);
  set_zero(e.C);
  set_zero(e.eta);
  set_zero(e.b);
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) e.Y[i][j] = PT[i][j];
}

// General combine  out = l (earlier) (x) r (later)  (reference passes.py:264-288)
//   G = I + C_l Y_r
//   X = G^-1 [A_l | C_l | b_l + C_l eta_r],   Z = G^-T [Y_r A_l | eta_r - Y_r b_l]
//   A = A_r X1,  Y = sym(A_l^T Z1 + Y_l),  C = sym(A_r X2 A_r^T + C_r),
//   eta = A_l^T z + eta_l,  b = A_r x + b_r
template <typename R, int NX>
PTC_D bool vcombine(const VElem<R, NX>& l, const VElem<R, NX>& r, VElem<R, NX>& o) {
  R G[NX][NX];
  mm<NX, NX, NX>(l.C, r.Y, G);
#pragma unroll
  for (int i = 0; i < NX; ++i) G[i][i] += R(1);
  int piv[NX];
  bool ok = lu_factor<NX>(G, piv);
  // right-hand sides of the transposed solve
  R Z[NX][NX + 1];
  {
    R YA[NX][NX];
    mm<NX, NX, NX>(r.Y, l.A, YA);
    R Yb[NX];
    mv<NX, NX>(r.Y, l.b, Yb);
#pragma unroll
    for (int i = 0; i < NX; ++i) {
#pragma unroll
      for (int j = 0; j < NX; ++j) Z[i][j] = YA[i][j];
      Z[i][NX] = r.eta[i] - Yb[i];
    }
  }
  lu_solve_t<NX, NX + 1>(G, piv, Z);
  // Y and eta (need only l and Z)
  {
    R Zs[NX][NX];
#pragma unroll
    for (int i = 0; i < NX; ++i)
#pragma unroll
      for (int j = 0; j < NX; ++j) Zs[i][j] = Z[i][j];
    mtm<NX, NX, NX>(l.A, Zs, o.Y);
#pragma unroll
    for (int i = 0; i < NX; ++i)
#pragma unroll
      for (int j = 0; j < NX; ++j) o.Y[i][j] += l.Y[i][j];
    symmetrize<NX>(o.Y);
    R z[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) z[i] = Z[i][NX];
    mtv<NX, NX>(l.A, z, o.eta);
#pragma unroll
    for (int i = 0; i < NX; ++i) o.eta[i] += l.eta[i];
  }
  // forward solve X = G^-1 [A_l | C_l | b_l + C_l eta_r]
  R X[NX][2 * NX + 1];
  {
    R Ce[NX];
    mv<NX, NX>(l.C, r.eta, Ce);
#pragma unroll
    for (int i = 0; i < NX; ++i) {
#pragma unroll
      for (int j = 0; j < NX; ++j) {
        X[i][j] = l.A[i][j];
        X[i][NX + j] = l.C[i][j];
      }
      X[i][2 * NX] = l.b[i] + Ce[i];
    }
  }
  lu_solve<NX, 2 * NX + 1>(G, piv, X);
  {
    R X1[NX][NX], X2[NX][NX], x[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) {
#pragma unroll
      for (int j = 0; j < NX; ++j) {
        X1[i][j] = X[i][j];
        X2[i][j] = X[i][NX + j];
      }
      x[i] = X[i][2 * NX];
    }
    mm<NX, NX, NX>(r.A, X1, o.A);
    R T2[NX][NX];
    mm<NX, NX, NX>(r.A, X2, T2);
    mmt<NX, NX, NX>(T2, r.A, o.C);
#pragma unroll
    for (int i = 0; i < NX; ++i)
#pragma unroll
      for (int j = 0; j < NX; ++j) o.C[i][j] += r.C[i][j];
    symmetrize<NX>(o.C);
    mv<NX, NX>(r.A, x, o.b);
#pragma unroll
    for (int i = 0; i < NX; ++i) o.b[i] += r.b[i];
  }
  return ok;
}

// Specialised combine  carry' = e (x) carry  for a carry with A = C = b = 0:
//   (I + Y_c C_e) Z = [Y_c A_e | eta_c - Y_c b_e]
//   Y' = sym(A_e^T Z1 + Y_e),  eta' = A_e^T z + eta_e
template <typename R, int NX>
PTC_D bool vstep(const VElem<R, NX>& e, const VCarry<R, NX>& c, VCarry<R, NX>& o) {
  R G[NX][NX];
  mm<NX, NX, NX>(c.Y, e.C, G);
#pragma unroll
  for (int i = 0; i < NX; ++i) G[i][i] += R(1);
  int piv[NX];
  bool ok = lu_factor<NX>(G, piv);
  R Z[NX][NX + 1];
  {
    R YA[NX][NX];
    mm<NX, NX, NX>(c.Y, e.A, YA);
    R Yb[NX];
    mv<NX, NX>(c.Y, e.b, Yb);
#pragma unroll
    for (int i = 0; i < NX; ++i) {
#pragma unroll
      for (int j = 0; j < NX; ++j) Z[i][j] = YA[i][j];
      Z[i][NX] = c.eta[i] - Yb[i];
    }
  }
  lu_solve<NX, NX + 1>(G, piv, Z);
  R Zs[NX][NX], z[NX];
#pragma unroll
  for (int i = 0; i < NX; ++i) {
#pragma unroll
    for (int j = 0; j < NX; ++j) Zs[i][j] = Z[i][j];
    z[i] = Z[i][NX];
  }
  mtm<NX, NX, NX>(e.A, Zs, o.Y);
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) o.Y[i][j] += e.Y[i][j];
  symmetrize<NX>(o.Y);
  mtv<NX, NX>(e.A, z, o.eta);
#pragma unroll
  for (int i = 0; i < NX; ++i) o.eta[i] += e.eta[i];
  return ok;
}

// One stage element (earlier, from its expansion) combined with a general
// aggregate r (later): vcombine(velem_from_stage(st), r) without forming
// the stage's dual element or the NX x NX system I + C_l Y_r.  The stage's
// C_l = Fu Rr^-1 Fu^T has rank NU, so by Woodbury
//   (I + C_l Y_r)^-1 = I - Fu Q^-1 Fu^T Y_r,  Q = Rr + Fu^T Y_r Fu  (NU x NU),
//   (I + C_l Y_r)^-1 C_l = Fu Q^-1 Fu^T,
// and with v = eta_r - Y_r b_l, q = Q^-1 Fu^T v, W = Q^-1 Fu^T Y_r A_l:
//   Y   = sym(A_l^T (Y_r A_l - Y_r Fu W) + Y_l),  eta = A_l^T (v - Y_r Fu q) + eta_l,
//   A   = A_r (A_l - Fu W),   C = sym(A_r Fu Q^-1 (A_r Fu)^T + C_r),
//   b   = A_r (b_l + Fu q) + b_r.
// det(I + C_l Y_r) = det(Q) / det(Rr): a singular combine is a singular Q
// (FLAG_COND); Rr failing its Cholesky raises FLAG_DEF_R as velem does.
template <typename R, int NX, int NU>
PTC_D int vcombine_stage(const Stage<R, NX, NU>& st, const VElem<R, NX>& r, VElem<R, NX>& o) {
  int fl = 0;
  R L[NU][NU];
#pragma unroll
  for (int i = 0; i < NU; ++i)
#pragma unroll
    for (int j = 0; j < NU; ++j) L[i][j] = st.Rr[i][j];
  if (!cholesky<NU>(L)) fl |= FLAG_DEF_R;
  R RiMt[NU][NX], Rid[NU];
#pragma unroll
  for (int i = 0; i < NU; ++i) {
#pragma unroll
    for (int j = 0; j < NX; ++j) RiMt[i][j] = st.M[j][i];
    Rid[i] = st.d[i];
  }
  chol_solve<NU, NX>(L, RiMt);
  chol_solve_vec<NU>(L, Rid);
  R Al[NX][NX], tmp[NX][NX];
  mm<NX, NU, NX>(st.Fu, RiMt, tmp);
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) Al[i][j] = st.Fx[i][j] - tmp[i][j];
  R Yl[NX][NX];
  mm<NX, NU, NX>(st.M, RiMt, tmp);
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) Yl[i][j] = st.P[i][j] - tmp[i][j];
  symmetrize<NX>(Yl);
  R etal[NX], bl[NX];
  mv<NX, NU>(st.M, Rid, etal);
  mv<NX, NU>(st.Fu, Rid, bl);
#pragma unroll
  for (int i = 0; i < NX; ++i) bl[i] = -bl[i];
  // Q = sym(Rr + Fu^T Y_r Fu), LU-factored (Q of a partial suffix may be
  // indefinite; only a singular one is an error)
  R YF[NX][NU];
  mm<NX, NX, NU>(r.Y, st.Fu, YF);
  R Q[NU][NU];
  mtm<NU, NX, NU>(st.Fu, YF, Q);
#pragma unroll
  for (int i = 0; i < NU; ++i)
#pragma unroll
    for (int j = 0; j < NU; ++j) Q[i][j] += st.Rr[i][j];
  symmetrize<NU>(Q);
  int piv[NU];
  if (!lu_factor<NU>(Q, piv)) fl |= FLAG_COND;
  // W = Q^-1 Fu^T Y_r A_l  (Fu^T Y_r = YF^T, Y_r symmetric)
  R W[NU][NX];
  mtm<NU, NX, NX>(YF, Al, W);
  lu_solve<NU, NX>(Q, piv, W);
  // v, q = Q^-1 Fu^T v
  R v[NX], Yb[NX];
  mv<NX, NX>(r.Y, bl, Yb);
#pragma unroll
  for (int i = 0; i < NX; ++i) v[i] = r.eta[i] - Yb[i];
  R q[NU][1];
  {
    R Ftv[NU];
    mtv<NU, NX>(st.Fu, v, Ftv);
#pragma unroll
    for (int i = 0; i < NU; ++i) q[i][0] = Ftv[i];
  }
  lu_solve<NU, 1>(Q, piv, q);
  // Y = sym(A_l^T (Y_r A_l - YF W) + Y_l)
  R Z1[NX][NX];
  mm<NX, NX, NX>(r.Y, Al, Z1);
  mm<NX, NU, NX>(YF, W, tmp);
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) Z1[i][j] -= tmp[i][j];
  mtm<NX, NX, NX>(Al, Z1, o.Y);
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) o.Y[i][j] += Yl[i][j];
  symmetrize<NX>(o.Y);
  // eta = A_l^T (v - YF q) + eta_l ;  x = b_l + Fu q
  R z[NX], x[NX];
#pragma unroll
  for (int i = 0; i < NX; ++i) {
    R yq = R(0), fq = R(0);
#pragma unroll
    for (int k = 0; k < NU; ++k) {
      yq = fma(YF[i][k], q[k][0], yq);
      fq = fma(st.Fu[i][k], q[k][0], fq);
    }
    z[i] = v[i] - yq;
    x[i] = bl[i] + fq;
  }
  mtv<NX, NX>(Al, z, o.eta);
#pragma unroll
  for (int i = 0; i < NX; ++i) o.eta[i] += etal[i];
  // A = A_r (A_l - Fu W)
  mm<NX, NU, NX>(st.Fu, W, tmp);
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) Al[i][j] -= tmp[i][j];
  mm<NX, NX, NX>(r.A, Al, o.A);
  // C = sym(AF Q^-1 AF^T + C_r),  AF = A_r Fu
  R AF[NX][NU], Y2[NU][NX];
  mm<NX, NX, NU>(r.A, st.Fu, AF);
#pragma unroll
  for (int i = 0; i < NU; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) Y2[i][j] = AF[j][i];
  lu_solve<NU, NX>(Q, piv, Y2);
  mm<NX, NU, NX>(AF, Y2, o.C);
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) o.C[i][j] += r.C[i][j];
  symmetrize<NX>(o.C);
  // b = A_r x + b_r
  mv<NX, NX>(r.A, x, o.b);
#pragma unroll
  for (int i = 0; i < NX; ++i) o.b[i] += r.b[i];
  return fl;
}

// One stage element folded into a terminal-containing suffix, fused with the
// gains of that stage: the reference's gains of stage t from the cost-to-go
// of stage t+1 (passes.py:316-323) together with vstep(velem(st), c)
// (element 192-228, combine 264-288), written without forming the dual
// element.  With
//   Q = sym(Rr + Fu^T S Fu),  Qux = M^T + Fu^T S Fx,  qu = d + Fu^T s
// the push-through identity  (I + S C)^-1 S = S - S Fu Q^-1 Fu^T S  (C =
// Fu Rr^-1 Fu^T) turns the combine into
//   Gamma = -Q^-1 Qux,  gamma = -Q^-1 qu,
//   S' = sym(P + Fx^T S Fx + Qux^T Gamma),  s' = Fx^T s + Qux^T gamma,
// exactly the suffix value of the dual scan (Y' = S', eta' = -s').  Since
// det(I + C S) = det(Q) / det(Rr), a singular combine is a Q that fails its
// Cholesky, so the two definiteness flags cover the conditioning case.
// Returns FLAG_DEF_R / FLAG_DEF_Q bits.
// kCheckR: also test R_t + alpha I (DefinitenessError).  Tree and block
// schedules have already tested every stage in the level-0 up-sweep.
// FxM, FuM: structural zeros of Fx and Fu (linalg.cuh kDense = none).
template <typename R, int NX, int NU, bool kCheckR = true, uint64_t FxM = kDense,
          uint64_t FuM = kDense>
PTC_D int riccati_step(const Stage<R, NX, NU>& st, const VCarry<R, NX>& c, R (&Gam)[NU][NX],
                       R (&gam)[NU], VCarry<R, NX>& o) {
  int fl = 0;
  if constexpr (kCheckR) {
    R L[NU][NU];
#pragma unroll
    for (int i = 0; i < NU; ++i)
#pragma unroll
      for (int j = 0; j < NU; ++j) L[i][j] = st.Rr[i][j];
    if (!cholesky<NU>(L)) fl |= FLAG_DEF_R;
  }
  R FtS[NU][NX];
  mtm<NU, NX, NX, R, FuM>(st.Fu, c.Y, FtS);
  R Q[NU][NU];
  mm<NU, NX, NU, R, FuM>(FtS, st.Fu, Q);
#pragma unroll
  for (int i = 0; i < NU; ++i)
#pragma unroll
    for (int j = 0; j < NU; ++j) Q[i][j] += st.Rr[i][j];
  symmetrize<NU>(Q);
  if (!cholesky<NU>(Q)) fl |= FLAG_DEF_Q;
  R Qux[NU][NX];
  mm<NU, NX, NX, R, FxM>(FtS, st.Fx, Qux);
#pragma unroll
  for (int i = 0; i < NU; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) Qux[i][j] += st.M[j][i];
  R Fe[NU];
  mtv<NU, NX, R, FuM>(st.Fu, c.eta, Fe);  // Fu^T eta = -Fu^T s
#pragma unroll
  for (int i = 0; i < NU; ++i) gam[i] = st.d[i] - Fe[i];
#pragma unroll
  for (int i = 0; i < NU; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) Gam[i][j] = Qux[i][j];
  chol_solve<NU, NX>(Q, Gam);
  chol_solve_vec<NU>(Q, gam);
#pragma unroll
  for (int i = 0; i < NU; ++i) {
#pragma unroll
    for (int j = 0; j < NX; ++j) Gam[i][j] = -Gam[i][j];
    gam[i] = -gam[i];
  }
  // S' = P + Fx^T (S Fx) + Qux^T Gamma
  R SF[NX][NX];
  mm<NX, NX, NX, R, FxM>(c.Y, st.Fx, SF);
  mtm<NX, NX, NX, R, FxM>(st.Fx, SF, o.Y);
  R QG[NX][NX];
  mtm<NX, NU, NX>(Qux, Gam, QG);
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) o.Y[i][j] += st.P[i][j] + QG[i][j];
  symmetrize<NX>(o.Y);
  // eta' = -s' = Fx^T eta - Qux^T gamma
  R Fte[NX], Qg[NX];
  mtv<NX, NX, R, FxM>(st.Fx, c.eta, Fte);
  mtv<NX, NU>(Qux, gam, Qg);
#pragma unroll
  for (int i = 0; i < NX; ++i) o.eta[i] = Fte[i] - Qg[i];
  return fl;
}

// ---------------------------------------------------------------------------
// affine maps
// ---------------------------------------------------------------------------

template <typename R, int NX>
struct Aff {
  R F[NX][NX], e[NX];
  static constexpr int kComp = NX * NX + NX;
};

template <typename R, int NX>
PTC_D void aff_identity(Aff<R, NX>& a) {
  set_identity(a.F);
  set_zero(a.e);
}

// o = outer o inner  (apply inner first):  F = F_o F_i,  e = F_o e_i + e_o
template <typename R, int NX>
PTC_D void aff_compose(const Aff<R, NX>& outer, const Aff<R, NX>& inner, Aff<R, NX>& o) {
  mm<NX, NX, NX>(outer.F, inner.F, o.F);
  mv<NX, NX>(outer.F, inner.e, o.e);
#pragma unroll
  for (int i = 0; i < NX; ++i) o.e[i] += outer.e[i];
}

template <typename R, int NX>
PTC_D void aff_apply(const Aff<R, NX>& a, const R (&x)[NX], R (&y)[NX]) {
  mv<NX, NX>(a.F, x, y);
#pragma unroll
  for (int i = 0; i < NX; ++i) y[i] += a.e[i];
}

template <typename R, int NX>
PTC_D void ld_aff(const R* f, int t, int rows, int B, int b, Aff<R, NX>& a) {
  ld_mat(f, t, rows, B, b, a.F, 0);
  ld_vec(f, t, rows, B, b, a.e, NX * NX);
}

template <typename R, int NX>
PTC_D void st_aff(R* f, int t, int rows, int B, int b, const Aff<R, NX>& a) {
  st_mat(f, t, rows, B, b, a.F, 0);
  st_vec(f, t, rows, B, b, a.e, NX * NX);
}

}  // namespace ptc
