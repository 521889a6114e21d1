// Chain solver of the M-ABD step on sm_100a: fused per-segment kernel (stages 1-4) and the hierarchical
// block-tridiagonal reduced-system kernels for chains longer than one segment.
//
// Paper: the chain dual is block tridiagonal (Eq. chain-btd); the paper solves it with block
// Thomas in O(K) on one thread. Here one 128-thread CTA owns a 256-slot segment of a chain and
// solves its 257-equation block-tridiagonal system by block cyclic reduction in shared memory
// (log₂ 256 = 8 levels), fused with the per-body stages in one pass over HBM:
//   phase 1, per body:  load qⁿ, q̇ⁿ → polar R → f_A → δq̃ (stages 1-2); δq̃ is parked in the
//                       q̇ buffer (q̇ⁿ is dead after f_A; the line stays in L2);
//            per joint: D, B, r = C(q̃) from the 3×3 kernels P(ȳ,ȳ') rotated by R
//   phase 2, per segment: cyclic reduction → λ
//   phase 3, per body:  re-read qⁿ, δq̃ (L2), recompute R, qⁿ⁺¹ = q̃ − diag₄(R)H̄⁻¹Σ±(ȳ_aug ⊗ Rᵀλ),
//                       q̇ⁿ⁺¹ = (qⁿ⁺¹ − qⁿ)/h
// Nothing per body is held in registers across the solve, so 4 CTAs (57 KB shared memory each) fit per SM.
// Chains spanning several segments are partitioned (SPIKE-style): each segment reduces its interior to a
// 2-equation "top" system on its end slots (REDUCE), the tops form a smaller block-tridiagonal system
// solved recursively by btd_kernel, and each segment then recomputes and back-substitutes (FINISH).
#include <cuda_runtime.h>

#include <algorithm>

#include "mabd_device.cuh"
#include "mabd_kernels.h"

namespace mabd {

// ------------------------------------------------------------------ shared-memory cyclic reduction
// Equations k = 0..256:  Bl_k λ_{k−s} + D_k λ_k + Br_k λ_{k+s} = r_k at stride s, with Bl_k = Br_{k−s}ᵀ.
// Component-major arrays D[6][NEQ] (sym; replaced by D⁻¹ once eliminated), B[9][NEQ] (Br), Bl[9][NEQ]
// (saved Br_{k−s} of an eliminated k), r[3][NEQ] (rhs, then λ). Equation k lives at position cr_pos(k):
// the equations eliminated at stride 2^l are stored contiguously (level-major order), so every CR level
// reads and writes contiguous positions (no shared-memory bank conflicts).
struct CRS {
  double* D;
  double* B;
  double* Bl;
  double* r;
};

__device__ __forceinline__ int cr_pos(int k) {
  if (k == 0) return SEG - 1;
  if (k >= SEG) return SEG;
  const int l = __ffs(k) - 1;
  return (SEG - (SEG >> l)) + (k >> (l + 1));
}

// strided view of one equation's components
struct SV {
  double* p;
  __device__ __forceinline__ double& operator[](int e) const { return p[e * NEQ]; }
};
__device__ __forceinline__ SV eqD(const CRS& s, int pos) { return SV{s.D + pos}; }
__device__ __forceinline__ SV eqB(const CRS& s, int pos) { return SV{s.B + pos}; }
__device__ __forceinline__ SV eqBl(const CRS& s, int pos) { return SV{s.Bl + pos}; }
__device__ __forceinline__ SV eqR(const CRS& s, int pos) { return SV{s.r + pos}; }
template <int N>
__device__ __forceinline__ void ldv(SV v, double* x) {
#pragma unroll
  for (int e = 0; e < N; ++e) x[e] = v[e];
}
template <int N>
__device__ __forceinline__ void stv(SV v, const double* x) {
#pragma unroll
  for (int e = 0; e < N; ++e) v[e] = x[e];
}

#ifdef MABD_EXP_CLOCK
__device__ unsigned long long g_phase_clk[16];
#define PH_MARK(i)                                                        \
  do {                                                                    \
    if (threadIdx.x == 0) {                                               \
      const long long now = clock64();                                    \
      atomicAdd(&g_phase_clk[i], (unsigned long long)(now - ph_last));    \
      ph_last = now;                                                      \
    }                                                                     \
  } while (0)
extern "C" int mabd_dbg_phases(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_phase_clk, sizeof(g_phase_clk));
}
extern "C" int mabd_dbg_reset() {
  unsigned long long z[16] = {0};
  return (int)cudaMemcpyToSymbol(g_phase_clk, z, sizeof(z));
}
#else
#define PH_MARK(i) \
  do {             \
  } while (0)
#endif

__device__ __forceinline__ void report(const StepConsts& k, int32_t flag) {
  atomicOr(k.err, flag);
  atomicMin(k.err + 1, k.step_index);
}

// invalidate one 128-byte L2 line without write-back (PTX discard.global.L2, sm_80+)
__device__ __forceinline__ void l2_discard128(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void l2_prefetch(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// update of the surviving equation kq at stride st (both neighbours already hold D⁻¹)
__device__ __forceinline__ void cr_update(const CRS& s, int kq, int st) {
  const int pk = cr_pos(kq);
  double Ds[6], D[9], Br[9], r[3];
  ldv<6>(eqD(s, pk), Ds);
  full_from_sym(Ds, D);
  ldv<9>(eqB(s, pk), Br);
  ldv<3>(eqR(s, pk), r);
  double nBr[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (kq >= st) {  // left neighbour i = kq − st:  α = Br_iᵀ D_i⁻¹;  D −= α Br_i;  r −= α r_i
    const int pi = cr_pos(kq - st);
    double Dis[6], Di[9], Bi[9], al[9], tmp[9], ri[3], ar[3];
    ldv<6>(eqD(s, pi), Dis);
    full_from_sym(Dis, Di);
    ldv<9>(eqB(s, pi), Bi);
    mat3_mul_at(Bi, Di, al);
    mat3_mul(al, Bi, tmp);
#pragma unroll
    for (int e = 0; e < 9; ++e) D[e] -= tmp[e];
    ldv<3>(eqR(s, pi), ri);
    mat3_vec(al, ri, ar);
#pragma unroll
    for (int e = 0; e < 3; ++e) r[e] -= ar[e];
  }
  if (kq < SEG) {  // right neighbour j = kq + st:  γ = Br_k D_j⁻¹;  D −= γ Br_kᵀ;  r −= γ r_j;  Br_k ← −γ Br_j
    const int pj = cr_pos(kq + st);
    double Djs[6], Dj[9], ga[9], tmp[9], Bj[9], rj[3], gr[3];
    ldv<6>(eqD(s, pj), Djs);
    full_from_sym(Djs, Dj);
    mat3_mul(Br, Dj, ga);
    mat3_mul_bt(ga, Br, tmp);
#pragma unroll
    for (int e = 0; e < 9; ++e) D[e] -= tmp[e];
    ldv<3>(eqR(s, pj), rj);
    mat3_vec(ga, rj, gr);
#pragma unroll
    for (int e = 0; e < 3; ++e) r[e] -= gr[e];
    ldv<9>(eqB(s, pj), Bj);
    mat3_mul(ga, Bj, tmp);
#pragma unroll
    for (int e = 0; e < 9; ++e) nBr[e] = -tmp[e];
    stv<9>(eqBl(s, pj), Br);  // j's left coupling at this level (Bl_j = Br_kᵀ), kept for back substitution
  }
  const double Dn[6] = {D[0], 0.5 * (D[1] + D[3]), 0.5 * (D[2] + D[6]), D[4], 0.5 * (D[5] + D[7]), D[8]};
  stv<6>(eqD(s, pk), Dn);
  stv<9>(eqB(s, pk), nBr);
  stv<3>(eqR(s, pk), r);
}

__device__ __forceinline__ void cr_invert(const CRS& s, int k, const StepConsts& ks) {
  const int p = cr_pos(k);
  double Ds[6], Di[6];
  ldv<6>(eqD(s, p), Ds);
  if (!sym_inv_spd(Ds, Di)) report(ks, ERR_SINGULAR);
  stv<6>(eqD(s, p), Di);
}

// Forward reduction. Precondition: every odd equation (eliminated at stride 1) already holds D⁻¹. A survivor
// that will be eliminated at the next level inverts its own D right after its update (no one else reads a
// survivor's D at this level), so each level needs one barrier.
__device__ void cr_forward(const CRS& s, int t, const StepConsts& k) {
  for (int st = 1; st < SEG; st <<= 1) {
    const int ne = SEG / (2 * st);
    for (int m = t; m <= ne; m += CT) {  // survivors k = 2st·m, m ≤ ne
      const int kq = 2 * st * m;
      cr_update(s, kq, st);
      if ((m & 1) && 2 * st < SEG) cr_invert(s, kq, k);
    }
    __syncthreads();
  }
}

// Solve the remaining 2-equation system [D0 B; Bᵀ D1][λ0; λ1] = [r0; r1] (one thread).
__device__ void cr_solve_top(const CRS& s, const StepConsts& k) {
  const int p0 = cr_pos(0), p1 = cr_pos(SEG);
  double D0s[6], D0i[6], D0[9], B[9], D1s[6], D1[9], r0[3], r1[3];
  ldv<9>(eqB(s, p0), B);
  ldv<3>(eqR(s, p0), r0);
  ldv<3>(eqR(s, p1), r1);
  ldv<6>(eqD(s, p0), D0s);
  ldv<6>(eqD(s, p1), D1s);
  if (!sym_inv_spd(D0s, D0i)) report(k, ERR_SINGULAR);
  full_from_sym(D0i, D0);
  full_from_sym(D1s, D1);
  double W[9], T[9];
  mat3_mul(D0, B, W);     // D0⁻¹ B
  mat3_mul_at(B, W, T);   // Bᵀ D0⁻¹ B
#pragma unroll
  for (int e = 0; e < 9; ++e) D1[e] -= T[e];
  double y[3], z[3];
  mat3_vec(D0, r0, y);
  mat3t_vec(B, y, z);
#pragma unroll
  for (int e = 0; e < 3; ++e) r1[e] -= z[e];
  D1s[0] = D1[0];
  D1s[1] = 0.5 * (D1[1] + D1[3]);
  D1s[2] = 0.5 * (D1[2] + D1[6]);
  D1s[3] = D1[4];
  D1s[4] = 0.5 * (D1[5] + D1[7]);
  D1s[5] = D1[8];
  double S1i[6], l1[3], l0[3], Bl1[3];
  if (!sym_inv_spd(D1s, S1i)) report(k, ERR_SINGULAR);
  sym_vec(S1i, r1, l1);
  mat3_vec(B, l1, Bl1);
#pragma unroll
  for (int e = 0; e < 3; ++e) r0[e] -= Bl1[e];
  mat3_vec(D0, r0, l0);
  stv<3>(eqR(s, p0), l0);
  stv<3>(eqR(s, p1), l1);
}

// Back substitution; λ of equations 0 and 256 are in r on entry, all λ on exit.
__device__ void cr_backward(const CRS& s, int t) {
  for (int st = SEG / 2; st >= 1; st >>= 1) {
    const int ne = SEG / (2 * st);
    for (int m = t; m < ne; m += CT) {
      const int i = st * (2 * m + 1);
      const int pi = cr_pos(i);
      double Bl[9], Br[9], Di[6], ll[3], lr[3], v[3], w[3];
      ldv<9>(eqBl(s, pi), Bl);
      ldv<9>(eqB(s, pi), Br);
      ldv<6>(eqD(s, pi), Di);
      ldv<3>(eqR(s, cr_pos(i - st)), ll);
      ldv<3>(eqR(s, cr_pos(i + st)), lr);
      ldv<3>(eqR(s, pi), v);
      mat3t_vec(Bl, ll, w);  // Bl_i λ_{i−s} = Br_{i−s}ᵀ λ_{i−s}
#pragma unroll
      for (int e = 0; e < 3; ++e) v[e] -= w[e];
      mat3_vec(Br, lr, w);
#pragma unroll
      for (int e = 0; e < 3; ++e) v[e] -= w[e];
      sym_vec(Di, v, w);
      stv<3>(eqR(s, pi), w);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ CRS cr_smem(double* smem) {
  CRS s;
  s.D = smem;
  s.B = s.D + NEQ * 6;
  s.Bl = s.B + NEQ * 9;
  s.r = s.Bl + NEQ * 9;
  return s;
}

__device__ __forceinline__ void write_top(const CRS& s, Top* o) {
  const int p0 = cr_pos(0), p1 = cr_pos(SEG);
  ldv<6>(eqD(s, p0), o->D0);
  ldv<6>(eqD(s, p1), o->D1);
  ldv<9>(eqB(s, p0), o->B);
  ldv<3>(eqR(s, p0), o->r0);
  ldv<3>(eqR(s, p1), o->r1);
}

__device__ __forceinline__ void body_material(const ChainArgs& a, int64_t slot, Material& M, double& msc,
                                              HinvBlk& H) {
  const int mid = a.b.mat_id ? __ldg(a.b.mat_id + slot) : 0;
  msc = a.b.mscale ? __ldg(a.b.mscale + slot) : 1.0;
  M = a.b.mats[mid];
  if (a.hinv_tab)
    H = a.hinv_tab[mid];
  else
    hinv_blocks(M, msc, a.k.ih2, H);
}

// ------------------------------------------------------------------ the fused chain segment kernel
// Persistent: each CTA loops over segments it ← blockIdx.x, += gridDim.x. While a segment is in the
// cyclic reduction (no memory traffic), the CTA prefetches the NEXT segment's state into L2, so its
// phase-1 loads are L2 hits (software pipeline across segments).
// FINISH = false: first pass (fused segments solve completely; long segments REDUCE to their top);
// FINISH = true: second pass of long segments (recompute, read the ends' λ, back-substitute, update).
__device__ __forceinline__ void prefetch_segment(const ChainArgs& a, int it, int tid) {
  if (it >= a.n_items) return;
  const int g = a.seg_list ? a.seg_list[it] : it;
  const int64_t base = (int64_t)g * SEG;
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    const int64_t sl = base + tid + b * CT;
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      l2_prefetch(a.b.q + c * a.b.ld + sl);
      l2_prefetch(a.b.qd + c * a.b.ld + sl);
    }
    if (a.b.mscale) l2_prefetch(a.b.mscale + sl);
    l2_prefetch(a.slot_info + sl);
  }
}

#ifndef MABD_CHAIN_MINB
#define MABD_CHAIN_MINB 4
#endif
template <bool FINISH>
__global__ void __launch_bounds__(CT, MABD_CHAIN_MINB) chain_kernel(ChainArgs a) {
  extern __shared__ double smem[];
  const CRS s = cr_smem(smem);
  const int tid = threadIdx.x;
  const StepConsts& k = a.k;
  if ((int)blockIdx.x < a.n_items) {  // first segment: its second body is fetched while the first is loaded
    const int g0 = a.seg_list ? a.seg_list[blockIdx.x] : (int)blockIdx.x;
    const int64_t s2 = (int64_t)g0 * SEG + tid + CT;
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      l2_prefetch(a.b.q + c * a.b.ld + s2);
      l2_prefetch(a.b.qd + c * a.b.ld + s2);
    }
  }
#ifdef MABD_EXP_CLOCK
  long long ph_last = clock64();
#endif
  for (int it = blockIdx.x; it < a.n_items; it += gridDim.x) {
    PH_MARK(7);
    const int g = a.seg_list ? a.seg_list[it] : it;
    const int flags = a.seg_flags[g];
    const bool is_long = (flags & SEG_LONG) != 0;
    const bool update = !is_long || FINISH;  // this pass writes the new state
    const int64_t base = (int64_t)g * SEG;

    // ---------------- phase 1: per body predict + joint contributions (thread tid: slots tid, tid+128)
    // Equation t is assembled in place: sD[t] = D part of body t, sR[t] = rhs part, sB[t] = B_t; body t's
    // contribution to equation t+1 goes to the scratch row sBl[t+1] and is added after the barrier.
    uint32_t infos[3];
    infos[0] = __ldg(a.slot_info + base + tid);
    infos[1] = __ldg(a.slot_info + base + tid + 1);
    infos[2] = __ldg(a.slot_info + base + tid + CT + 1);
#pragma unroll 1
    for (int b = 0; b < 2; ++b) {
      const int t = tid + b * CT;
      const int64_t slot = base + t;
      const uint32_t info = b == 0 ? infos[0] : __ldg(a.slot_info + slot);
      const uint32_t infoN = infos[1 + b];
      const bool has_body = slot_right(info) == SIDE_BODY;
      const bool eq_real = slot_real(info);
      const bool right_real = slot_real(infoN) && slot_left(infoN) == SIDE_BODY;
      const int pt = cr_pos(t);
      const SV sd = eqD(s, pt), sr = eqR(s, pt), sb = eqB(s, pt);
      const SV sx = eqBl(s, cr_pos(t + 1));  // scratch row: body t's contribution to equation t+1
      {
        const double one = eq_real ? 0.0 : 1.0;  // not a constraint: decoupled identity equation, λ = 0
        sd[0] = one; sd[1] = 0; sd[2] = 0; sd[3] = one; sd[4] = 0; sd[5] = one;
        double rr[3] = {0, 0, 0};
        if (eq_real) {
          const double* gp = a.geo + 6 * (size_t)slot_geo(info);
          if (slot_left(info) == SIDE_WORLD)  // start anchor: +p_world
#pragma unroll
            for (int e = 0; e < 3; ++e) rr[e] = __ldg(gp + e);
          if (slot_right(info) == SIDE_WORLD)  // end anchor: −p_world
#pragma unroll
            for (int e = 0; e < 3; ++e) rr[e] -= __ldg(gp + 3 + e);
        }
#pragma unroll
        for (int e = 0; e < 3; ++e) sr[e] = rr[e];
#pragma unroll
        for (int e = 0; e < 9; ++e) sb[e] = 0.0;
#pragma unroll
        for (int e = 0; e < 9; ++e) sx[e] = 0.0;
      }
      if (has_body) {
        double q[12], R[9];
        HinvBlk H;
        {
          double qd[12], dqt[12];
          double* qdb = a.b.qd + slot;
          const double* qb = a.b.q + slot;
#pragma unroll
          for (int c = 0; c < 12; ++c) q[c] = qb[c * a.b.ld];
#pragma unroll
          for (int c = 0; c < 12; ++c) qd[c] = qdb[c * a.b.ld];
          Material M;
          double msc;
          body_material(a, slot, M, msc, H);
          if (!predict_body(q, qd, M, msc, H, k.ih, k.grav, R, dqt)) report(k, ERR_NONFINITE);
          if (update) {
#pragma unroll
            for (int c = 0; c < 12; ++c) qdb[c * a.b.ld] = dqt[c];  // park δq̃ (q̇ⁿ is dead from here on)
#pragma unroll
            for (int c = 0; c < 9; ++c) a.b.rs[c * a.b.ld + slot] = R[c];  // park R (L2 scratch)
          }
#pragma unroll
          for (int c = 0; c < 12; ++c) q[c] += dqt[c];  // q̃
        }
        double P[9], F[6], yR[3], yL[3], x[3];
        if (eq_real) {  // joint to the left: this body is its right side (sign −)
          const double* gp = a.geo + 6 * (size_t)slot_geo(info);
#pragma unroll
          for (int e = 0; e < 3; ++e) yR[e] = __ldg(gp + 3 + e);
          pblock(H, yR, yR, P);
          rot_conj_sym(R, P, F);
#pragma unroll
          for (int e = 0; e < 6; ++e) sd[e] = F[e];
          point_pos(q, yR, x);
#pragma unroll
          for (int e = 0; e < 3; ++e) sr[e] -= x[e];
        }
        if (right_real) {  // joint to the right: this body is its left side (sign +)
          const double* gp = a.geo + 6 * (size_t)slot_geo(infoN);
#pragma unroll
          for (int e = 0; e < 3; ++e) yL[e] = __ldg(gp + e);
          pblock(H, yL, yL, P);
          rot_conj_sym(R, P, F);
#pragma unroll
          for (int e = 0; e < 6; ++e) sx[e] = F[e];
          point_pos(q, yL, x);
#pragma unroll
          for (int e = 0; e < 3; ++e) sx[6 + e] = x[e];
          if (eq_real) {  // B_t = −R P(ȳ_R, ȳ_L') Rᵀ  (signs −·+)
            double Fb[9];
            pblock(H, yR, yL, P);
            rot_conj(R, P, Fb);
#pragma unroll
            for (int e = 0; e < 9; ++e) sb[e] = -Fb[e];
          }
        }
      }
    }
    PH_MARK(0);
    __syncthreads();
    PH_MARK(1);
    // add the left neighbours' contributions (equation 0's left body lies in the previous segment: its part
    // of the interface equation is added by that segment's REDUCE output)
#pragma unroll 1
    for (int b = 0; b < 2; ++b) {
      const int t = tid + b * CT;
      const uint32_t info = b == 0 ? infos[0] : __ldg(a.slot_info + base + t);
      if (t > 0 && slot_real(info) && slot_left(info) == SIDE_BODY) {
        const int pt = cr_pos(t);
        const SV x = eqBl(s, pt), d = eqD(s, pt), r = eqR(s, pt);
#pragma unroll
        for (int e = 0; e < 6; ++e) d[e] += x[e];
#pragma unroll
        for (int e = 0; e < 3; ++e) r[e] += x[6 + e];
      }
      if (t & 1) cr_invert(s, t, k);  // eliminated at stride 1
    }
    if (tid == CT - 1) {  // equation 256: next segment's first slot (partial) or padding
      const bool real = (flags & SEG_RIGHT_IFACE) != 0;
      const SV x = eqBl(s, SEG);
      double D[6], r[3];
#pragma unroll
      for (int e = 0; e < 6; ++e) D[e] = real ? x[e] : ((e == 0 || e == 3 || e == 5) ? 1.0 : 0.0);
#pragma unroll
      for (int e = 0; e < 3; ++e) r[e] = real ? x[6 + e] : 0.0;
      const double Z[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      stv<6>(eqD(s, SEG), D);
      stv<9>(eqB(s, SEG), Z);
      stv<3>(eqR(s, SEG), r);
    }
    __syncthreads();

    // ---------------- phase 2: block cyclic reduction (the next segment's state streams into L2 meanwhile)
    PH_MARK(2);
    prefetch_segment(a, it + gridDim.x, tid);
#ifndef MABD_EXP_SKIP_CR
    cr_forward(s, tid, k);
#endif
    PH_MARK(3);
    if (!is_long) {
      if (tid == 0) cr_solve_top(s, k);
    } else if (!FINISH) {
      if (tid == 0) write_top(s, a.top_out + a.seg_red[g]);
      __syncthreads();
      continue;
    } else if (tid == 0) {
      const int u = a.seg_red[g];
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        eqR(s, cr_pos(0))[e] = a.lam_in[3 * u + e];
        eqR(s, SEG)[e] = (flags & SEG_RIGHT_IFACE) ? a.lam_in[3 * (u + 1) + e] : 0.0;
      }
    }
    __syncthreads();
    PH_MARK(4);
#ifndef MABD_EXP_SKIP_CR
    cr_backward(s, tid);
#endif
    PH_MARK(5);
#ifdef MABD_EXP_SKIP_P3
    __syncthreads();
    continue;
#endif

    // ---------------- phase 3: qⁿ⁺¹ = q̃ − diag₄(R) H̄⁻¹ Σ ±Γ(ȳ)ᵀ Rᵀλ
#pragma unroll 1
    for (int b = 0; b < 2; ++b) {
      const int t = tid + b * CT;
      const int64_t slot = base + t;
      const uint32_t info = b == 0 ? infos[0] : __ldg(a.slot_info + slot);
      const uint32_t infoN = infos[1 + b];
      double* qb = a.b.q + slot;
      double* qdb = a.b.qd + slot;
      // issue every load of this body first: R (parked), qⁿ, δq̃ (parked) — all L2 hits
      double R[9], q[12], dqt[12];
      const double* rp = a.b.rs + slot;
#pragma unroll
      for (int c = 0; c < 9; ++c) R[c] = __ldcg(rp + c * a.b.ld);
#pragma unroll
      for (int c = 0; c < 12; ++c) q[c] = __ldcs(qb + c * a.b.ld);
#pragma unroll
      for (int c = 0; c < 12; ++c) dqt[c] = __ldcs(qdb + c * a.b.ld);
      // all lanes have their R: discard the scratch lines (no DRAM write-back); the warp covers 32
      // consecutive, 256-B aligned slots = two 128-B lines per row
      __syncwarp();
      if ((threadIdx.x & 15) == 0) {
#pragma unroll
        for (int c = 0; c < 9; ++c) l2_discard128(rp + c * a.b.ld);
      }
      if (slot_right(info) != SIDE_BODY) continue;
      const bool eq_real = slot_real(info);
      const bool right_real = slot_real(infoN) && slot_left(infoN) == SIDE_BODY;
      double gq[12];
#pragma unroll
      for (int c = 0; c < 12; ++c) gq[c] = 0.0;
      double w[3], lam[3], y[3];
      if (eq_real) {
        const double* gp = a.geo + 6 * (size_t)slot_geo(info);
#pragma unroll
        for (int e = 0; e < 3; ++e) {
          y[e] = __ldg(gp + 3 + e);
          lam[e] = eqR(s, cr_pos(t))[e];
        }
        mat3t_vec(R, lam, w);
        add_point_force(gq, y, w, -1.0);
      }
      if (right_real) {
        const double* gp = a.geo + 6 * (size_t)slot_geo(infoN);
#pragma unroll
        for (int e = 0; e < 3; ++e) {
          y[e] = __ldg(gp + e);
          lam[e] = eqR(s, cr_pos(t + 1))[e];
        }
        mat3t_vec(R, lam, w);
        add_point_force(gq, y, w, 1.0);
      }
      Material M;
      double msc;
      HinvBlk H;
      body_material(a, slot, M, msc, H);
      double u[12];
      hinv_apply(H, gq, u);
#pragma unroll
      for (int kb = 0; kb < 4; ++kb) {
        double c3[3];
        mat3_vec(R, u + 3 * kb, c3);
#pragma unroll
        for (int e = 0; e < 3; ++e) {
          const int c = 3 * kb + e;
          const double dq = dqt[c] - c3[e];  // δq = δq̃ − correction
          __stcs(qb + c * a.b.ld, q[c] + dq);
          __stcs(qdb + c * a.b.ld, dq * k.ih);
        }
      }
    }
    PH_MARK(6);
    __syncthreads();  // shared memory is reused by the next segment
  }
}

// ------------------------------------------------------------------ reduced block-tridiagonal levels
// Unknown u of level L owns the equation built from the level-(L−1) tops:
//   D_u = top[u].D0 + (left(u) ? top[u−1].D1 : 0),  B_u = top[u].B,  r_u likewise.
// A window w of 256 unknowns is one CTA; its equation 256 is the first unknown of window w+1 (partial:
// D = 0, r = 0; its coupling from unknown 256w+255 is B_{256w+255}), or padding.
__global__ void __launch_bounds__(CT) btd_kernel(BtdArgs a) {
  extern __shared__ double smem[];
  const CRS s = cr_smem(smem);
  const int tid = threadIdx.x;
  const int64_t w = blockIdx.x;
  const int64_t nu = a.n_u;
  for (int b = 0; b < 2; ++b) {
    const int t = tid + b * CT;
    const int64_t u = w * SEG + t;
    double D[6] = {1, 0, 0, 1, 0, 1}, B[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, r[3] = {0, 0, 0};
    if (u < nu) {
      const Top& T = a.top_in[u];
      const bool left = a.left_iface ? (a.left_iface[u] != 0) : (u > 0);
#pragma unroll
      for (int e = 0; e < 6; ++e) D[e] = T.D0[e] + (left ? a.top_in[u - 1].D1[e] : 0.0);
#pragma unroll
      for (int e = 0; e < 3; ++e) r[e] = T.r0[e] + (left ? a.top_in[u - 1].r1[e] : 0.0);
#pragma unroll
      for (int e = 0; e < 9; ++e) B[e] = T.B[e];
    }
    const int pt = cr_pos(t);
    stv<6>(eqD(s, pt), D);
    stv<9>(eqB(s, pt), B);
    stv<3>(eqR(s, pt), r);
    if (t & 1) cr_invert(s, t, a.k);  // eliminated at stride 1
  }
  if (tid == CT - 1) {
    // equation 256: the next window's first unknown (partial, completed by that window), the next part's
    // first unknown (partial from this part's last unknown: its top D1, r1), or padding
    const bool real_next = (w + 1) * SEG < nu;
    const double Z[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (!real_next && a.right_open) {
      stv<6>(eqD(s, SEG), a.top_in[nu - 1].D1);
      stv<3>(eqR(s, SEG), a.top_in[nu - 1].r1);
    } else {
      const double dv = real_next ? 0.0 : 1.0;
      const double Dn[6] = {dv, 0, 0, dv, 0, dv};
      stv<6>(eqD(s, SEG), Dn);
      stv<3>(eqR(s, SEG), Z);
    }
    stv<9>(eqB(s, SEG), Z);
  }
  __syncthreads();
  cr_forward(s, tid, a.k);
  if (a.mode == BTD_REDUCE) {
    if (tid == 0) write_top(s, a.top_out + w);
    return;
  }
  if (a.mode == BTD_FUSED) {
    if (tid == 0) cr_solve_top(s, a.k);
  } else if (tid == 0) {
    const bool real_next = (w + 1) * SEG < nu;
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      eqR(s, cr_pos(0))[e] = a.lam_in[3 * w + e];
      eqR(s, SEG)[e] = real_next ? a.lam_in[3 * (w + 1) + e] : (a.right_open ? a.lam_remote[e] : 0.0);
    }
  }
  __syncthreads();
  cr_backward(s, tid);
  for (int b = 0; b < 2; ++b) {
    const int t = tid + b * CT;
    const int64_t u = w * SEG + t;
    if (u < nu) {
#pragma unroll
      for (int e = 0; e < 3; ++e) a.lam_out[3 * u + e] = eqR(s, cr_pos(t))[e];
    }
  }
}

// ------------------------------------------------------------------ multi-part chains: sequential part top
// A part (one rank's share of a long chain, or an emulated rank) reduces its n level unknowns u = 0..n−1 and
// the next part's first unknown ρ (partial, from this side) onto {0, ρ}: eliminate u = 1..n−1 in order,
// carrying the coupling X of equation 0 to the current frontier (block Thomas with a spike).
// n is small (≤ 256 by construction, typically ≤ 17), so one thread does it.
__device__ __forceinline__ void seq_eq(const SeqArgs& a, int u, double* D, double* r) {
  // equation u from the tops of the level below: D_u = top[u].D0 + top[u−1].D1 (u > 0), same for r;
  // u = n is the remote unknown ρ (partial: top[n−1].D1, r1 if right-open; else padding)
  const int n = a.n;
  if (u == n) {
    if (a.right_open) {
#pragma unroll
      for (int e = 0; e < 6; ++e) D[e] = a.top_in[n - 1].D1[e];
#pragma unroll
      for (int e = 0; e < 3; ++e) r[e] = a.top_in[n - 1].r1[e];
    } else {
      D[0] = 1; D[1] = 0; D[2] = 0; D[3] = 1; D[4] = 0; D[5] = 1;
      r[0] = r[1] = r[2] = 0;
    }
    return;
  }
#pragma unroll
  for (int e = 0; e < 6; ++e) D[e] = a.top_in[u].D0[e] + (u > 0 ? a.top_in[u - 1].D1[e] : 0.0);
#pragma unroll
  for (int e = 0; e < 3; ++e) r[e] = a.top_in[u].r0[e] + (u > 0 ? a.top_in[u - 1].r1[e] : 0.0);
}

__global__ void seq_top_kernel(SeqArgs a) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int n = a.n;
  double D0s[6], r0[3], X[9], Dks[6], rk[3];
  seq_eq(a, 0, D0s, r0);
#pragma unroll
  for (int e = 0; e < 9; ++e) X[e] = a.top_in[0].B[e];  // coupling 0 → 1 (or → ρ when n = 1)
  seq_eq(a, n == 1 ? 1 : 1, Dks, rk);
  for (int k = 1; k < n; ++k) {
    double Di[6], Dif[9], Bk[9];
    if (!sym_inv_spd(Dks, Di)) report(a.k, ERR_SINGULAR);
    full_from_sym(Di, Dif);
#pragma unroll
    for (int e = 0; e < 9; ++e) Bk[e] = a.top_in[k].B[e];  // k → k+1 (ρ when k = n−1)
    double* sc = a.scratch + 27 * (size_t)k;
#pragma unroll
    for (int e = 0; e < 6; ++e) sc[e] = Di[e];
#pragma unroll
    for (int e = 0; e < 9; ++e) { sc[6 + e] = X[e]; sc[15 + e] = Bk[e]; }
#pragma unroll
    for (int e = 0; e < 3; ++e) sc[24 + e] = rk[e];
    // eq 0:  D0 −= X D⁻¹ Xᵀ,  r0 −= X D⁻¹ r_k,  X ← −X D⁻¹ B_k
    double XD[9], T[9], v[3];
    mat3_mul(X, Dif, XD);
    mat3_mul_bt(XD, X, T);
    double D0f[9];
    full_from_sym(D0s, D0f);
#pragma unroll
    for (int e = 0; e < 9; ++e) D0f[e] -= T[e];
    D0s[0] = D0f[0]; D0s[1] = 0.5 * (D0f[1] + D0f[3]); D0s[2] = 0.5 * (D0f[2] + D0f[6]);
    D0s[3] = D0f[4]; D0s[4] = 0.5 * (D0f[5] + D0f[7]); D0s[5] = D0f[8];
    mat3_vec(XD, rk, v);
#pragma unroll
    for (int e = 0; e < 3; ++e) r0[e] -= v[e];
    double nX[9];
    mat3_mul(XD, Bk, nX);
#pragma unroll
    for (int e = 0; e < 9; ++e) X[e] = -nX[e];
    // eq k+1:  D −= B_kᵀ D⁻¹ B_k,  r −= B_kᵀ D⁻¹ r_k
    double Dn[6], rn[3], DB[9], BDB[9], Dnf[9], w[3], bw[3];
    seq_eq(a, k + 1, Dn, rn);
    mat3_mul(Dif, Bk, DB);
    mat3_mul_at(Bk, DB, BDB);
    full_from_sym(Dn, Dnf);
#pragma unroll
    for (int e = 0; e < 9; ++e) Dnf[e] -= BDB[e];
    Dks[0] = Dnf[0]; Dks[1] = 0.5 * (Dnf[1] + Dnf[3]); Dks[2] = 0.5 * (Dnf[2] + Dnf[6]);
    Dks[3] = Dnf[4]; Dks[4] = 0.5 * (Dnf[5] + Dnf[7]); Dks[5] = Dnf[8];
    mat3_vec(Dif, rk, w);
    mat3t_vec(Bk, w, bw);
#pragma unroll
    for (int e = 0; e < 3; ++e) rk[e] = rn[e] - bw[e];
  }
  Top* o = a.top_out;
#pragma unroll
  for (int e = 0; e < 6; ++e) { o->D0[e] = D0s[e]; o->D1[e] = Dks[e]; }
#pragma unroll
  for (int e = 0; e < 9; ++e) o->B[e] = X[e];
#pragma unroll
  for (int e = 0; e < 3; ++e) { o->r0[e] = r0[e]; o->r1[e] = rk[e]; }
}

__global__ void seq_finish_kernel(SeqArgs a) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int n = a.n;
  double l0[3], lnext[3];
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    l0[e] = a.lam_ends[e];
    lnext[e] = a.right_open ? a.lam_ends[3 + e] : 0.0;
    a.lam_out[e] = l0[e];
  }
  for (int k = n - 1; k >= 1; --k) {  // λ_k = D'_k⁻¹ (r'_k − X_kᵀ λ_0 − B_k λ_{k+1})
    const double* sc = a.scratch + 27 * (size_t)k;
    double v[3], w[3];
#pragma unroll
    for (int e = 0; e < 3; ++e) v[e] = sc[24 + e];
    mat3t_vec(sc + 6, l0, w);
#pragma unroll
    for (int e = 0; e < 3; ++e) v[e] -= w[e];
    mat3_vec(sc + 15, lnext, w);
#pragma unroll
    for (int e = 0; e < 3; ++e) v[e] -= w[e];
    sym_vec(sc, v, w);
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      a.lam_out[3 * k + e] = w[e];
      lnext[e] = w[e];
    }
  }
}

cudaError_t launch_seq_top(const SeqArgs& a, cudaStream_t st) {
  seq_top_kernel<<<1, 32, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_seq_finish(const SeqArgs& a, cudaStream_t st) {
  seq_finish_kernel<<<1, 32, 0, st>>>(a);
  return cudaGetLastError();
}

size_t cr_smem_bytes() { return sizeof(double) * NEQ * (6 + 9 + 9 + 3); }

static int g_num_sms = 0;

cudaError_t launch_chain(const ChainArgs& a0, int nitems, bool finish, cudaStream_t st) {
  if (nitems <= 0) return cudaSuccess;
  ChainArgs a = a0;
  a.n_items = nitems;
  const size_t sm = cr_smem_bytes();
  const int grid = std::min(nitems, MABD_CHAIN_MINB * std::max(g_num_sms, 1));
  if (finish)
    chain_kernel<true><<<grid, CT, sm, st>>>(a);
  else
    chain_kernel<false><<<grid, CT, sm, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_btd(const BtdArgs& a, int nblocks, cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
  btd_kernel<<<nblocks, CT, cr_smem_bytes(), st>>>(a);
  return cudaGetLastError();
}

cudaError_t chain_kernels_init() {
  const int sm = (int)cr_smem_bytes();
  cudaError_t e;
  int dev = 0;
  if ((e = cudaGetDevice(&dev))) return e;
  if ((e = cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev))) return e;
  if ((e = cudaFuncSetAttribute(chain_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm))) return e;
  if ((e = cudaFuncSetAttribute(chain_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm))) return e;
  if ((e = cudaFuncSetAttribute(btd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm))) return e;
  // favour shared memory in the unified L1/shared carve-out so that 4 segment CTAs fit per SM
  cudaFuncSetAttribute(chain_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(chain_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  return cudaSuccess;
}

// prefactor: per-material closed-form H̄⁻¹ ("pre-factorized")
__global__ void hinv_table_kernel(const Material* mats, int nm, double ih2, HinvBlk* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nm) hinv_blocks(mats[i], 1.0, ih2, out[i]);
}

cudaError_t launch_hinv_table(const Material* mats, int nm, double ih2, HinvBlk* out, cudaStream_t st) {
  if (nm <= 0) return cudaSuccess;
  hinv_table_kernel<<<(nm + 127) / 128, 128, 0, st>>>(mats, nm, ih2, out);
  return cudaGetLastError();
}

// state gather / scatter between the caller's AoS order and the internal SoA positions
__global__ void gather_state_kernel(const double* q, const double* qd, int64_t ld, const int64_t* perm, int64_t n,
                                    double* qo, double* qdo) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * 12) return;
  const int64_t b = i / 12, c = i % 12;
  const int64_t sidx = perm[b];
  if (qo) qo[i] = q[c * ld + sidx];
  if (qdo) qdo[i] = qd[c * ld + sidx];
}
__global__ void scatter_state_kernel(double* q, double* qd, int64_t ld, const int64_t* perm, int64_t n,
                                     const double* qi, const double* qdi) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * 12) return;
  const int64_t b = i / 12, c = i % 12;
  const int64_t sidx = perm[b];
  if (qi) q[c * ld + sidx] = qi[i];
  if (qdi) qd[c * ld + sidx] = qdi[i];
}

cudaError_t launch_gather(const double* q, const double* qd, int64_t ld, const int64_t* perm, int64_t n, double* qo,
                          double* qdo, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t tot = n * 12;
  gather_state_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(q, qd, ld, perm, n, qo, qdo);
  return cudaGetLastError();
}
cudaError_t launch_scatter(double* q, double* qd, int64_t ld, const int64_t* perm, int64_t n, const double* qi,
                           const double* qdi, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t tot = n * 12;
  scatter_state_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(q, qd, ld, perm, n, qi, qdi);
  return cudaGetLastError();
}

}  // namespace mabd
