// Device-side fp64 building blocks of the M-ABD step (sm_100a). No torch types, no host code.
//
// Paper references are PAPER.md line numbers (P:n). Conventions: q = [vec(A); t], vec column-major,
// q[3c+r] = A(r,c). A symmetric 3×3 is packed as (xx, xy, xz, yy, yz, zz).
#pragma once
#include <cstdint>

#include "mabd_internal.h"

namespace mabd {

// ------------------------------------------------------------------ small 3×3 helpers

__device__ __forceinline__ void sym_from_full(const double* M, double* S) {
  S[0] = M[0]; S[1] = M[1]; S[2] = M[2]; S[3] = M[4]; S[4] = M[5]; S[5] = M[8];
}
__device__ __forceinline__ void full_from_sym(const double* S, double* M) {
  M[0] = S[0]; M[1] = S[1]; M[2] = S[2];
  M[3] = S[1]; M[4] = S[3]; M[5] = S[4];
  M[6] = S[2]; M[7] = S[4]; M[8] = S[5];
}
// row-major 3×3: M[3*r + c]
__device__ __forceinline__ void mat3_mul(const double* A, const double* B, double* C) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) C[3 * r + c] = A[3 * r] * B[c] + A[3 * r + 1] * B[3 + c] + A[3 * r + 2] * B[6 + c];
}
// C = A * Bᵀ
__device__ __forceinline__ void mat3_mul_bt(const double* A, const double* B, double* C) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      C[3 * r + c] = A[3 * r] * B[3 * c] + A[3 * r + 1] * B[3 * c + 1] + A[3 * r + 2] * B[3 * c + 2];
}
// C = Aᵀ * B
__device__ __forceinline__ void mat3_mul_at(const double* A, const double* B, double* C) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) C[3 * r + c] = A[r] * B[c] + A[3 + r] * B[3 + c] + A[6 + r] * B[6 + c];
}
__device__ __forceinline__ void mat3_vec(const double* A, const double* x, double* y) {
#pragma unroll
  for (int r = 0; r < 3; ++r) y[r] = A[3 * r] * x[0] + A[3 * r + 1] * x[1] + A[3 * r + 2] * x[2];
}
__device__ __forceinline__ void mat3t_vec(const double* A, const double* x, double* y) {
#pragma unroll
  for (int r = 0; r < 3; ++r) y[r] = A[r] * x[0] + A[3 + r] * x[1] + A[6 + r] * x[2];
}
__device__ __forceinline__ void sym_vec(const double* S, const double* x, double* y) {
  y[0] = S[0] * x[0] + S[1] * x[1] + S[2] * x[2];
  y[1] = S[1] * x[0] + S[3] * x[1] + S[4] * x[2];
  y[2] = S[2] * x[0] + S[4] * x[1] + S[5] * x[2];
}

// 1/x: hardware approximation (MUFU.RCP64H, ~23 bits) refined by two Newton steps (e → e²) to full fp64
// precision (≤ 1 ulp; not IEEE-rounded, which the parity tolerance of 1e-9 does not need).
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// 1/√x: hardware approximation (MUFU.RSQ64H) refined by two Newton steps y ← y(3 − xy²)/2 to full fp64
// precision (≤ 1 ulp; not IEEE-rounded).
__device__ __forceinline__ double fast_rsqrt(double x) {
  double y = rsqrt(x);
  double e = fma(-x * y, y, 1.0);
  y = fma(0.5 * y, e, y);
  e = fma(-x * y, y, 1.0);
  return fma(0.5 * y, e, y);
}

// Inverse of an SPD 3×3 (packed sym) by its adjugate; returns false if a leading minor is ≤ 0
// (the dual matrix must be SPD: a failure means redundant joints, MABD_ESINGULAR).
__device__ __forceinline__ bool sym_inv_spd(const double* S, double* Si) {
  const double a = S[0], b = S[1], c = S[2], d = S[3], e = S[4], f = S[5];
  const double A00 = d * f - e * e, A01 = c * e - b * f, A02 = b * e - c * d;
  const double det = a * A00 + b * A01 + c * A02;
  const double m2 = a * d - b * b;
  const bool ok = (a > 0.0) && (m2 > 0.0) && (det > 0.0) && isfinite(det);
  const double id = fast_rcp(det);
  Si[0] = A00 * id;
  Si[1] = A01 * id;
  Si[2] = A02 * id;
  Si[3] = (a * f - c * c) * id;
  Si[4] = (b * c - a * e) * id;
  Si[5] = m2 * id;
  return ok;
}

// ------------------------------------------------------------------ polar decomposition
// R = A (AᵀA)^{-1/2}. With E = XᵀX − I, X ← X·p(E), p the degree-6 truncation of the series of (I+E)^{-1/2}
// (7th-order convergence: ‖E_new‖ ≈ 0.42‖E‖⁷, one step from ‖E‖ ≤ 1e-2 reaches ~1e-15; reading A5),
// preceded by determinant-scaled Newton steps X ← ½(ζX + ζ⁻¹X⁻ᵀ) while ‖E‖_F > 0.3, and followed, when
// ‖E‖_F ≥ 1e-2, by one third-order step X(I − E/2 + 3E²/8 − 5E³/16) instead of a second degree-6 step.
// A and R are row-major 3×3. Returns false for det A ≤ 1e-9 or non-finite input.

// C = S T for symmetric commuting S, T (packed sym): the product is symmetric, 6 entries.
__device__ __forceinline__ void symsym(const double* S, const double* T, double* C) {
  C[0] = S[0] * T[0] + S[1] * T[1] + S[2] * T[2];
  C[1] = S[0] * T[1] + S[1] * T[3] + S[2] * T[4];
  C[2] = S[0] * T[2] + S[1] * T[4] + S[2] * T[5];
  C[3] = S[1] * T[1] + S[3] * T[3] + S[4] * T[4];
  C[4] = S[1] * T[2] + S[3] * T[4] + S[4] * T[5];
  C[5] = S[2] * T[2] + S[4] * T[4] + S[5] * T[5];
}

__device__ __forceinline__ bool polar_rotation(const double* A, double* R) {
  const double detA = A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
                      A[2] * (A[3] * A[7] - A[4] * A[6]);
  if (!(detA > 1e-9) || !isfinite(detA)) {
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = (i % 4 == 0) ? 1.0 : 0.0;
    return false;
  }
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = A[i];
  for (int it = 0; it < 64; ++it) {
    // E = XᵀX − I (packed sym)
    double E[6];
    E[0] = R[0] * R[0] + R[3] * R[3] + R[6] * R[6] - 1.0;
    E[1] = R[0] * R[1] + R[3] * R[4] + R[6] * R[7];
    E[2] = R[0] * R[2] + R[3] * R[5] + R[6] * R[8];
    E[3] = R[1] * R[1] + R[4] * R[4] + R[7] * R[7] - 1.0;
    E[4] = R[1] * R[2] + R[4] * R[5] + R[7] * R[8];
    E[5] = R[2] * R[2] + R[5] * R[5] + R[8] * R[8] - 1.0;
    const double e2 = E[0] * E[0] + E[3] * E[3] + E[5] * E[5] + 2.0 * (E[1] * E[1] + E[2] * E[2] + E[4] * E[4]);
    if (e2 > 0.09) {  // scaled Newton step, far from orthogonal
      const double d = R[0] * (R[4] * R[8] - R[5] * R[7]) - R[1] * (R[3] * R[8] - R[5] * R[6]) +
                       R[2] * (R[3] * R[7] - R[4] * R[6]);
      // ζ = det^{-1/3} only sets the convergence speed (the iteration preserves the polar factor for any ζ > 0,
      // and a scalar error in 1/det merely rescales X⁻ᵀ), so single precision suffices for both scalars
      const double z = (double)cbrtf((float)fast_rcp(d));
      const double iz = fast_rcp(z * d);  // X⁻ᵀ = cof(X)/det
      double C[9];
      C[0] = R[4] * R[8] - R[5] * R[7]; C[1] = R[5] * R[6] - R[3] * R[8]; C[2] = R[3] * R[7] - R[4] * R[6];
      C[3] = R[2] * R[7] - R[1] * R[8]; C[4] = R[0] * R[8] - R[2] * R[6]; C[5] = R[1] * R[6] - R[0] * R[7];
      C[6] = R[1] * R[5] - R[2] * R[4]; C[7] = R[2] * R[3] - R[0] * R[5]; C[8] = R[0] * R[4] - R[1] * R[3];
#pragma unroll
      for (int i = 0; i < 9; ++i) R[i] = 0.5 * (z * R[i] + iz * C[i]);
      continue;
    }
    // p(E) − I by Horner: E(c1 + E(c2 + E(c3 + E(c4 + E(c5 + c6 E))))), c_k the series of (1+x)^{-1/2}
    // (a degree adapted to ‖E‖ saves up to 4 of the 5 products but measured slower on config 2: +4%, divergent lanes)
    double T[6], U[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) T[i] = (231.0 / 1024.0) * E[i];
    T[0] -= 63.0 / 256.0; T[3] -= 63.0 / 256.0; T[5] -= 63.0 / 256.0;
    symsym(E, T, U);
    U[0] += 35.0 / 128.0; U[3] += 35.0 / 128.0; U[5] += 35.0 / 128.0;
    symsym(E, U, T);
    T[0] -= 5.0 / 16.0; T[3] -= 5.0 / 16.0; T[5] -= 5.0 / 16.0;
    symsym(E, T, U);
    U[0] += 3.0 / 8.0; U[3] += 3.0 / 8.0; U[5] += 3.0 / 8.0;
    symsym(E, U, T);
    T[0] -= 0.5; T[3] -= 0.5; T[5] -= 0.5;
    symsym(E, T, U);  // p − I
    double X[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) X[i] = R[i];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      R[3 * r + 0] = X[3 * r] + X[3 * r] * U[0] + X[3 * r + 1] * U[1] + X[3 * r + 2] * U[2];
      R[3 * r + 1] = X[3 * r + 1] + X[3 * r] * U[1] + X[3 * r + 1] * U[3] + X[3 * r + 2] * U[4];
      R[3 * r + 2] = X[3 * r + 2] + X[3 * r] * U[2] + X[3 * r + 1] * U[4] + X[3 * r + 2] * U[5];
    }
#ifdef MABD_EXP_POLAR1
    break;
#endif
    if (e2 < 1e-4) break;  // ‖E_new‖ ≲ 0.42‖E‖⁷ < 5e-15
    {  // ‖E‖ ≤ 0.3: ‖E_new‖ ≲ 0.42‖E‖⁷ < 1e-4; one third-order step X ← X(I − E/2 + 3E²/8 − 5E³/16) leaves
       // (35/128)‖E_new‖⁴ < 1e-16 (one code path for every lane of a warp, instead of a second degree-6 step for
       // 1e-2 ≤ ‖E‖² and a first-order step below)
      double F[6];
      F[0] = R[0] * R[0] + R[3] * R[3] + R[6] * R[6] - 1.0;
      F[1] = R[0] * R[1] + R[3] * R[4] + R[6] * R[7];
      F[2] = R[0] * R[2] + R[3] * R[5] + R[6] * R[8];
      F[3] = R[1] * R[1] + R[4] * R[4] + R[7] * R[7] - 1.0;
      F[4] = R[1] * R[2] + R[4] * R[5] + R[7] * R[8];
      F[5] = R[2] * R[2] + R[5] * R[5] + R[8] * R[8] - 1.0;
#pragma unroll
      for (int i = 0; i < 6; ++i) T[i] = (-5.0 / 16.0) * F[i];
      T[0] += 3.0 / 8.0; T[3] += 3.0 / 8.0; T[5] += 3.0 / 8.0;
      symsym(F, T, U);
      U[0] -= 0.5; U[3] -= 0.5; U[5] -= 0.5;
      symsym(F, U, T);  // −E/2 + 3E²/8 − 5E³/16
#pragma unroll
      for (int i = 0; i < 9; ++i) X[i] = R[i];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        R[3 * r + 0] = X[3 * r] + X[3 * r] * T[0] + X[3 * r + 1] * T[1] + X[3 * r + 2] * T[2];
        R[3 * r + 1] = X[3 * r + 1] + X[3 * r] * T[1] + X[3 * r + 1] * T[3] + X[3 * r + 2] * T[4];
        R[3 * r + 2] = X[3 * r + 2] + X[3 * r] * T[2] + X[3 * r + 1] * T[4] + X[3 * r + 2] * T[5];
      }
      break;
    }
  }
  return true;
}

// ------------------------------------------------------------------ H̄⁻¹ in closed form
// For a central principal body frame M̄ = diag(a0,a1,a2,m) and K̄_A = V[μ(I₉+T₉) + λ vec(I)vec(I)ᵀ] ⊕ 0,
// H̄ = M_A/h² + K̄_A splits into: the 3×3 block G on the diagonal entries (A00, A11, A22), three 2×2
// blocks on the pairs (A_rc, A_cr), r < c, and (m/h²) I₃ on t. H̄⁻¹ keeps that pattern.

__device__ __forceinline__ void hinv_blocks(const Material& M, double mscale, double ih2, HinvBlk& H) {
  const double Vmu = M.V * M.mu, Vlam = M.V * M.lam;
  const double a0 = M.a0 * mscale * ih2, a1 = M.a1 * mscale * ih2, a2 = M.a2 * mscale * ih2;
  double G[6] = {a0 + 2.0 * Vmu + Vlam, Vlam, Vlam, a1 + 2.0 * Vmu + Vlam, Vlam, a2 + 2.0 * Vmu + Vlam};
  sym_inv_spd(G, H.g);
  const double ac[3][2] = {{a1, a0}, {a2, a0}, {a2, a1}};  // (mass of column c, mass of column r) per pair
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double x = ac[k][0] + Vmu, z = ac[k][1] + Vmu, y = Vmu;
    const double id = fast_rcp(x * z - y * y);
    H.pr[k][0] = z * id;
    H.pr[k][1] = -y * id;
    H.pr[k][2] = x * id;
  }
  H.tinv = fast_rcp(M.m * mscale * ih2);
}

// out = H̄⁻¹ v (12-vectors in q layout)
__device__ __forceinline__ void hinv_apply(const HinvBlk& H, const double* v, double* o) {
  const double d0 = v[0], d1 = v[4], d2 = v[8];
  o[0] = H.g[0] * d0 + H.g[1] * d1 + H.g[2] * d2;
  o[4] = H.g[1] * d0 + H.g[3] * d1 + H.g[4] * d2;
  o[8] = H.g[2] * d0 + H.g[4] * d1 + H.g[5] * d2;
  // pair (0,1): A01 = q[3], A10 = q[1]
  o[3] = H.pr[0][0] * v[3] + H.pr[0][1] * v[1];
  o[1] = H.pr[0][1] * v[3] + H.pr[0][2] * v[1];
  // pair (0,2): A02 = q[6], A20 = q[2]
  o[6] = H.pr[1][0] * v[6] + H.pr[1][1] * v[2];
  o[2] = H.pr[1][1] * v[6] + H.pr[1][2] * v[2];
  // pair (1,2): A12 = q[7], A21 = q[5]
  o[7] = H.pr[2][0] * v[7] + H.pr[2][1] * v[5];
  o[5] = H.pr[2][1] * v[7] + H.pr[2][2] * v[5];
  o[9] = H.tinv * v[9];
  o[10] = H.tinv * v[10];
  o[11] = H.tinv * v[11];
}

// H̄⁻¹ entry helpers for the 3×3 kernel P(y,y') = Γ(y) H̄⁻¹ Γ(y')ᵀ, Γ(y) = [y_augᵀ ⊗ I₃].
// self(a,c) = H̄⁻¹[3c+a, 3c+a] for a ≠ c;  cross(a,b) = H̄⁻¹[3b+a, 3a+b] for a ≠ b.
__device__ __forceinline__ double hinv_self(const HinvBlk& H, int a, int c) {
  const int lo = a < c ? a : c, hi = a < c ? c : a;
  const int k = lo + hi - 1;  // (0,1)→0, (0,2)→1, (1,2)→2
  return a < c ? H.pr[k][0] : H.pr[k][2];
}
__device__ __forceinline__ double hinv_cross(const HinvBlk& H, int a, int b) {
  const int lo = a < b ? a : b, hi = a < b ? b : a;
  return H.pr[lo + hi - 1][1];
}

// P_ab = y_a y'_b G⁻¹_ab + [a≠b] y_b y'_a cross(a,b) + [a=b](h²/m + Σ_{c≠a} y_c y'_c self(a,c))   (row-major)
__device__ __forceinline__ void pblock(const HinvBlk& H, const double* y, const double* yp, double* P) {
  const double Gf[9] = {H.g[0], H.g[1], H.g[2], H.g[1], H.g[3], H.g[4], H.g[2], H.g[4], H.g[5]};
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double v = y[a] * yp[b] * Gf[3 * a + b];
      if (a != b) {
        v += y[b] * yp[a] * hinv_cross(H, a, b);
      } else {
        v += H.tinv;
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (c != a) v += y[c] * yp[c] * hinv_self(H, a, c);
      }
      P[3 * a + b] = v;
    }
}

// Joint points on one principal axis (R18). If ȳ and ȳ' have no component off the body-frame axis k,
// every cross term of pblock vanishes: P(ȳ,ȳ') = (h²/m) I + ȳ_k ȳ'_k Q_k with Q_k = diag(q), q_k = G⁻¹_kk and
// q_a = self(a,k) for a ≠ k. All kernels of such a body are then tinv I + s Q_k, and R P Rᵀ = tinv I + s R Q_k Rᵀ:
// one rotated diagonal serves the body's D, D' and B blocks.
// axis of a point: 0-2 if it lies on that axis, 3 if it is zero (on every axis), −1 otherwise
__device__ __forceinline__ int point_axis(const double* y) {
  const bool z0 = y[0] == 0.0, z1 = y[1] == 0.0, z2 = y[2] == 0.0;
  if (z1 && z2) return z0 ? 3 : 0;
  if (z0 && z2) return 1;
  if (z0 && z1) return 2;
  return -1;
}
// the common axis of two points (−1: none)
__device__ __forceinline__ int common_axis(int a, int b) {
  if (a < 0 || b < 0) return -1;
  if (a == 3) return b == 3 ? 0 : b;
  if (b == 3 || b == a) return a;
  return -1;
}
// R Q_k Rᵀ (packed sym) for the axis k of pblock's special case above
__device__ __forceinline__ void axis_kernel_rot(const HinvBlk& H, const double* R, int k, double* Mq) {
  const double q0 = k == 0 ? H.g[0] : (k == 1 ? hinv_self(H, 0, 1) : hinv_self(H, 0, 2));
  const double q1 = k == 1 ? H.g[3] : (k == 0 ? hinv_self(H, 1, 0) : hinv_self(H, 1, 2));
  const double q2 = k == 2 ? H.g[5] : (k == 0 ? hinv_self(H, 2, 0) : hinv_self(H, 2, 1));
  double w[9];  // w[3j+c] = q_c R_jc
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    w[3 * j] = q0 * R[3 * j];
    w[3 * j + 1] = q1 * R[3 * j + 1];
    w[3 * j + 2] = q2 * R[3 * j + 2];
  }
  Mq[0] = R[0] * w[0] + R[1] * w[1] + R[2] * w[2];
  Mq[1] = R[0] * w[3] + R[1] * w[4] + R[2] * w[5];
  Mq[2] = R[0] * w[6] + R[1] * w[7] + R[2] * w[8];
  Mq[3] = R[3] * w[3] + R[4] * w[4] + R[5] * w[5];
  Mq[4] = R[3] * w[6] + R[4] * w[7] + R[5] * w[8];
  Mq[5] = R[6] * w[6] + R[7] * w[7] + R[8] * w[8];
}

// R P Rᵀ for symmetric P, packed sym out
__device__ __forceinline__ void rot_conj_sym(const double* R, const double* P, double* out) {
  double T[9];
  mat3_mul(R, P, T);
  out[0] = T[0] * R[0] + T[1] * R[1] + T[2] * R[2];
  out[1] = T[0] * R[3] + T[1] * R[4] + T[2] * R[5];
  out[2] = T[0] * R[6] + T[1] * R[7] + T[2] * R[8];
  out[3] = T[3] * R[3] + T[4] * R[4] + T[5] * R[5];
  out[4] = T[3] * R[6] + T[4] * R[7] + T[5] * R[8];
  out[5] = T[6] * R[6] + T[7] * R[7] + T[8] * R[8];
}

// R P Rᵀ (full 3×3 out)
__device__ __forceinline__ void rot_conj(const double* R, const double* P, double* out) {
  double T[9];
  mat3_mul(R, P, T);
  mat3_mul_bt(T, R, out);
}

// ------------------------------------------------------------------ per-body predict (stages 1-2)
// Computes R, q̃ − qⁿ = δq̃ = diag₄(R) H̄⁻¹ diag₄(Rᵀ) f_A with
// f_A = (1/h) M_A q̇ + M_A[0₉;g] − [V vec(R Π(RᵀA)); 0₃]   (Alg. 1 exact R).
// q̇ is fetched by qd_load(out12) and H̄⁻¹ by get_h(H) only when needed, so that neither is live during the polar
// decomposition (register pressure). Returns false if the polar decomposition failed.
// W (optional, world frame [τ; f; ȳ_f]): external wrench, f_A,ext = G(A)ᵀW: ½ τ × q_c on column c, f on t;
// f acts at the caller's frame origin, the material point ȳ_f of the canonical frame (0 unless the body was
// re-framed at create, R8), which adds ȳ_f,c f on column c.
// (‖v‖/‖M v‖) M v for row-major M (MT: Mᵀ v instead): Eq. len_preserving; 0 stays 0.
template <bool MT>
__device__ __forceinline__ void len_pres(const double* M, const double* v, double* o) {
  double w[3];
  if (MT)
    mat3t_vec(M, v, w);
  else
    mat3_vec(M, v, w);
  const double nv2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
  const double nw2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
  const double sc = nw2 > 0.0 ? sqrt(nv2) * fast_rsqrt(nw2) : 0.0;
#pragma unroll
  for (int e = 0; e < 3; ++e) o[e] = sc * w[e];
}

// Polar-free variant (LP = true, R9): no polar decomposition. R := A (returned, for the
// constraint-force operator diag₄(A)H̄⁻¹diag₄(Aᵀ) of stages 3-5, "A ≈ R"); the free solve is Alg. 1
// on the world-frame forces (inertia, gravity, wrench): each 3-block mapped by len_pres(Aᵀ); the elastic
// term enters in the body frame as the StVK stress −V Σ(E), Σ = 2μE + λ tr(E) I, E = ½(AᵀA − I) (the co-rotated
// method's −V Π); then H̄⁻¹, then each block of the result mapped by len_pres(A).
template <bool LP = false, class QdLoad, class GetH>
__device__ __forceinline__ bool predict_body_lazy(const double* q, QdLoad qd_load, const Material& M, double mscale,
                                                  GetH get_h, HinvBlk& H, double ih, const double* grav, double* R,
                                                  double* dqt, const double* W = nullptr) {
  double A[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) A[3 * r + c] = q[3 * c + r];
  if (LP) {
    const double detA = A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
                        A[2] * (A[3] * A[7] - A[4] * A[6]);
    double E[9];  // ½(AᵀA − I)
    mat3_mul_at(A, A, E);
#pragma unroll
    for (int i = 0; i < 9; ++i) E[i] = 0.5 * (E[i] - (i % 4 == 0 ? 1.0 : 0.0));
    const double trE = E[0] + E[4] + E[8];
    double Sg[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) Sg[i] = 2.0 * M.mu * E[i] + (i % 4 == 0 ? M.lam * trE : 0.0);
    const double ma[4] = {M.a0 * mscale * ih, M.a1 * mscale * ih, M.a2 * mscale * ih, M.m * mscale};
    double w[12], u[12], qd[12];
    qd_load(qd);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double fc[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) fc[r] = ma[c] * qd[3 * c + r];
      if (W) {
        const double* qc = q + 3 * c;
        fc[0] += 0.5 * (W[1] * qc[2] - W[2] * qc[1]) + W[6 + c] * W[3];
        fc[1] += 0.5 * (W[2] * qc[0] - W[0] * qc[2]) + W[6 + c] * W[4];
        fc[2] += 0.5 * (W[0] * qc[1] - W[1] * qc[0]) + W[6 + c] * W[5];
      }
      len_pres<true>(A, fc, w + 3 * c);
#pragma unroll
      for (int r = 0; r < 3; ++r) w[3 * c + r] -= M.V * Sg[3 * r + c];
    }
    {
      double ft[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) ft[r] = ma[3] * (qd[9 + r] * ih + grav[r]) + (W ? W[3 + r] : 0.0);
      len_pres<true>(A, ft, w + 9);
    }
    get_h(H);
    hinv_apply(H, w, u);
#pragma unroll
    for (int k = 0; k < 4; ++k) len_pres<false>(A, u + 3 * k, dqt + 3 * k);
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = A[i];
    return detA > 1e-9 && isfinite(detA) && isfinite(dqt[0] + dqt[4] + dqt[8] + dqt[9] + dqt[10] + dqt[11]);
  }
  const bool ok = polar_rotation(A, R);
  // F = RᵀA, Π(F) = μ(F+Fᵀ−2I) + λ tr(F−I) I, elastic force V vec(RΠ)
  double F[9];
  mat3_mul_at(R, A, F);
  const double tr = F[0] + F[4] + F[8] - 3.0;
  double Pi[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) Pi[3 * r + c] = M.mu * (F[3 * r + c] + F[3 * c + r]) + (r == c ? (M.lam * tr - 2.0 * M.mu) : 0.0);
  // w = diag₄(Rᵀ) f_A: the A-blocks are Rᵀ(m_c/h · q̇_c) − V Π[:,c] (Rᵀ R Π = Π), the t-block Rᵀ m (q̇_t/h + g)
  const double ma[4] = {M.a0 * mscale * ih, M.a1 * mscale * ih, M.a2 * mscale * ih, M.m * mscale};
  double w[12], u[12], qd[12];
  qd_load(qd);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double v[3], fc[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) fc[r] = ma[c] * qd[3 * c + r];
    if (W) {  // + ½ τ × q_c, + ȳ_f,c f (f acts at the material point ȳ_f: Γ(ȳ_f)ᵀ f)
      const double* qc = q + 3 * c;
      fc[0] += 0.5 * (W[1] * qc[2] - W[2] * qc[1]) + W[6 + c] * W[3];
      fc[1] += 0.5 * (W[2] * qc[0] - W[0] * qc[2]) + W[6 + c] * W[4];
      fc[2] += 0.5 * (W[0] * qc[1] - W[1] * qc[0]) + W[6 + c] * W[5];
    }
    mat3t_vec(R, fc, v);
#pragma unroll
    for (int r = 0; r < 3; ++r) w[3 * c + r] = v[r] - M.V * Pi[3 * r + c];
  }
  {
    double ft[3], v[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) ft[r] = ma[3] * (qd[9 + r] * ih + grav[r]) + (W ? W[3 + r] : 0.0);
    mat3t_vec(R, ft, v);
#pragma unroll
    for (int r = 0; r < 3; ++r) w[9 + r] = v[r];
  }
  get_h(H);
  hinv_apply(H, w, u);
#pragma unroll
  for (int k = 0; k < 4; ++k) mat3_vec(R, u + 3 * k, dqt + 3 * k);
  return ok && isfinite(dqt[0] + dqt[4] + dqt[8] + dqt[9] + dqt[10] + dqt[11]);
}

template <bool LP = false>
__device__ __forceinline__ bool predict_body(const double* q, const double* qd, const Material& M, double mscale,
                                             const HinvBlk& H, double ih, const double* grav, double* R,
                                             double* dqt, const double* W = nullptr) {
  HinvBlk Hc;
  return predict_body_lazy<LP>(
      q,
      [&](double* o) {
#pragma unroll
        for (int c = 0; c < 12; ++c) o[c] = qd[c];
      },
      M, mscale, [&](HinvBlk& o) { o = H; }, Hc, ih, grav, R, dqt, W);
}

// the wrench of body (SoA position) j (τ, f, ȳ_f: 9 doubles), or null
__device__ __forceinline__ const double* load_wrench(const BodyArrays& b, int64_t j, double* W) {
  if (!b.wr) return nullptr;
#pragma unroll
  for (int e = 0; e < 9; ++e) W[e] = b.wr[e * b.ld + j];
  return W;
}

// x(q; ȳ) = A ȳ + t
__device__ __forceinline__ void point_pos(const double* q, const double* y, double* x) {
#pragma unroll
  for (int r = 0; r < 3; ++r) x[r] = q[r] * y[0] + q[3 + r] * y[1] + q[6 + r] * y[2] + q[9 + r];
}

// g += s · (ȳ_aug ⊗ w): the body-frame generalized force of a point force w (= Γ(ȳ)ᵀ w)
__device__ __forceinline__ void add_point_force(double* g, const double* y, const double* w, double s) {
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    g[r] += s * y[0] * w[r];
    g[3 + r] += s * y[1] * w[r];
    g[6 + r] += s * y[2] * w[r];
    g[9 + r] += s * w[r];
  }
}

}  // namespace mabd
