// Loop breakers: the paper's Case III on the GPU chain / tree solvers (DESIGN.md
// reading R12).
//
// A few joints close loops ("breakers"); without them the joint graph is a forest the chain or tree solver handles.
// Partition the KKT into that forest's block 𝒜 and the breakers' multipliers λ_B (Eq. loop): the step is
// affine in λ_B, because the breakers act on their bodies as the external point forces −s Γ(ȳ)ᵀλ_B (the first line
// of Eq. kkt with ∇C_Bᵀλ_B moved to the right-hand side). So per Newton iteration, from the same qⁿ, the forest
// solver runs 1 + 3b times — with λ_B = 0 and with λ_B = each unit vector (b breaker points, 3 rows each) — and the
// breaker residuals C_B(q(λ_B)) give the affine map c₀ + M λ_B: M is the Schur complement 𝒮 = 𝒟 − 𝒞𝒜⁻¹𝒞ᵀ of
// Eq. loop up to sign, formed column by column through 𝒜⁻¹ (the forest solve) instead of by assembling 𝒞. Then
// M λ_B = −c₀ (one thread, ≤ 3·LOOP_MAX_PTS unknowns) and a last forest run with that λ_B gives qⁿ⁺¹: the exact KKT
// solution (the loop joints close like any other, pin P3). The breaker forces ride on the per-body wrench buffer
// (force f = −s λ at the material point ȳ), so a body may carry one breaker point and the caller's wrenches are
// not available in this mode.
#include <cuda_runtime.h>

#include <algorithm>
#include <numeric>
#include <string>
#include <vector>

#include "mabd_device.cuh"
#include "mabd_plan.h"

namespace mabd {

// ------------------------------------------------------------------------------------------ host: split
// Breakers: joints (between two bodies) whose bodies a spanning forest already connects, in joint order
// (union-find). Anchors never close a loop for the forest solvers (the chain solver takes anchors at path ends, the
// tree solver as child joints of their body).
bool loop_split(const mabd_joints* J, int64_t n, LoopPlan* L, std::string* msg) {
  std::vector<int64_t> par(n);
  std::iota(par.begin(), par.end(), 0);
  auto find = [&](int64_t x) {
    while (par[x] != x) x = par[x] = par[par[x]];
    return x;
  };
  for (int64_t k = 0; J->kind && k < J->n_joints; ++k)
    if (J->kind[k] != 0) return *msg = "nonlinear joints (five-row hinges, universal, prismatic) need the sparse solver", false;
  L->keep.clear();
  L->breakers.clear();
  for (int64_t k = 0; k < J->n_joints; ++k) {
    const int64_t a = J->body_a[k], b = J->body_b[k];
    if (b < 0) {
      L->keep.push_back(k);
      continue;
    }
    const int64_t ra = find(a), rb = find(b);
    if (ra == rb) {
      L->breakers.push_back(k);
    } else {
      par[ra] = rb;
      L->keep.push_back(k);
    }
  }
  if (L->breakers.empty()) return *msg = "no loops: use the chain or tree solver", false;
  // breaker points: ≤ LOOP_MAX_PTS, each body carries at most one
  std::vector<int64_t> pt_off(J->n_joints + 1, 0);
  for (int64_t k = 0; k < J->n_joints; ++k) pt_off[k + 1] = pt_off[k] + J->npts[k];
  std::vector<char> busy(n, 0);
  L->pa.clear();
  L->pb.clear();
  L->ya.clear();
  L->yb.clear();
  for (int64_t k : L->breakers)
    for (int q = 0; q < J->npts[k]; ++q) {
      const int64_t a = J->body_a[k], b = J->body_b[k], pt = pt_off[k] + q;
      if (busy[a] || busy[b]) return *msg = "a body carries two loop-breaker points (use the sparse solver)", false;
      busy[a] = busy[b] = 1;
      L->pa.push_back((int32_t)a);
      L->pb.push_back((int32_t)b);
      for (int e = 0; e < 3; ++e) {
        L->ya.push_back(J->ybar_a[3 * pt + e]);
        L->yb.push_back(J->ybar_b[3 * pt + e]);
      }
    }
  if ((int)L->pa.size() > LOOP_MAX_PTS)
    return *msg = "more than " + std::to_string(LOOP_MAX_PTS) + " loop-breaker points (use the sparse solver)", false;
  // the forest's joints as a joint list of their own (points copied in order)
  L->fa.clear();
  L->fb.clear();
  L->fn.clear();
  L->fya.clear();
  L->fyb.clear();
  for (int64_t k : L->keep) {
    L->fa.push_back(J->body_a[k]);
    L->fb.push_back(J->body_b[k]);
    L->fn.push_back(J->npts[k]);
    for (int64_t pt = pt_off[k]; pt < pt_off[k + 1]; ++pt)
      for (int e = 0; e < 3; ++e) {
        L->fya.push_back(J->ybar_a[3 * pt + e]);
        L->fyb.push_back(J->ybar_b[3 * pt + e]);
      }
  }
  L->forest.n_joints = (int64_t)L->keep.size();
  L->forest.body_a = L->fa.data();
  L->forest.body_b = L->fb.data();
  L->forest.npts = L->fn.data();
  L->forest.ybar_a = L->fya.data();
  L->forest.ybar_b = L->fyb.data();
  return true;
}

// ------------------------------------------------------------------------------------------ device
struct LoopArgs {
  double* wr;              // [9][ld] wrench buffer (τ, f, ȳ_f)
  const double* q;         // [12][ld]
  int64_t ld;
  int32_t np;              // breaker points
  const int32_t* pa;       // [np] internal positions
  const int32_t* pb;
  const double* ya;        // [np][3]
  const double* yb;
  double* M;               // [1 + 3np][3np] residual columns (column i of pass i)
  double* lam;             // [3np]
};

// pass `col` (0: λ_B = 0; 1 + i: unit vector e_i; −1: the solved λ_B) → the breaker bodies' point forces
__global__ void loop_force_kernel(LoopArgs a, int col) {
  const int p = threadIdx.x;
  if (p >= a.np) return;
  double lam[3];
#pragma unroll
  for (int e = 0; e < 3; ++e)
    lam[e] = col < 0 ? a.lam[3 * p + e] : (col >= 1 && col - 1 == 3 * p + e ? 1.0 : 0.0);
  for (int side = 0; side < 2; ++side) {  // body a: −Γ(ȳ_a)ᵀλ, body b: +Γ(ȳ_b)ᵀλ
    const int64_t j = side == 0 ? a.pa[p] : a.pb[p];
    const double* y = side == 0 ? a.ya + 3 * p : a.yb + 3 * p;
    const double sg = side == 0 ? -1.0 : 1.0;
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      a.wr[e * a.ld + j] = 0.0;                 // τ
      a.wr[(3 + e) * a.ld + j] = sg * lam[e];   // f
      a.wr[(6 + e) * a.ld + j] = y[e];          // ȳ_f
    }
  }
}

// C_B(q) of every breaker point → column `col` of M
__global__ void loop_residual_kernel(LoopArgs a, int col) {
  const int p = threadIdx.x;
  if (p >= a.np) return;
  double x[3] = {0, 0, 0};
  for (int side = 0; side < 2; ++side) {
    const int64_t j = side == 0 ? a.pa[p] : a.pb[p];
    const double* y = side == 0 ? a.ya + 3 * p : a.yb + 3 * p;
    const double sg = side == 0 ? 1.0 : -1.0;
    double qj[12], xp[3];
#pragma unroll
    for (int c = 0; c < 12; ++c) qj[c] = a.q[c * a.ld + j];
    point_pos(qj, y, xp);
#pragma unroll
    for (int e = 0; e < 3; ++e) x[e] += sg * xp[e];
  }
#pragma unroll
  for (int e = 0; e < 3; ++e) a.M[(size_t)col * 3 * a.np + 3 * p + e] = x[e];
}

// (M_i − M_0) λ = −M_0: Gaussian elimination with partial pivoting (one thread; ≤ 3·LOOP_MAX_PTS unknowns)
__global__ void loop_solve_kernel(LoopArgs a, StepConsts k) {
  if (threadIdx.x != 0) return;
  const int m = 3 * a.np;
  double A[3 * LOOP_MAX_PTS][3 * LOOP_MAX_PTS + 1];
  for (int r = 0; r < m; ++r) {
    for (int c = 0; c < m; ++c) A[r][c] = a.M[(size_t)(1 + c) * m + r] - a.M[r];
    A[r][m] = -a.M[r];
  }
  bool ok = true;
  for (int c = 0; c < m; ++c) {
    int piv = c;
    for (int r = c + 1; r < m; ++r)
      if (fabs(A[r][c]) > fabs(A[piv][c])) piv = r;
    if (!(fabs(A[piv][c]) > 0.0)) {
      ok = false;
      break;
    }
    if (piv != c)
      for (int e = 0; e <= m; ++e) {
        const double t = A[c][e];
        A[c][e] = A[piv][e];
        A[piv][e] = t;
      }
    const double inv = 1.0 / A[c][c];
    for (int r = c + 1; r < m; ++r) {
      const double f = A[r][c] * inv;
      for (int e = c; e <= m; ++e) A[r][e] -= f * A[c][e];
    }
  }
  for (int c = m - 1; c >= 0 && ok; --c) {
    double v = A[c][m];
    for (int e = c + 1; e < m; ++e) v -= A[c][e] * a.lam[e];
    a.lam[c] = v / A[c][c];
  }
  if (!ok) {
    atomicOr(k.err, ERR_SINGULAR);
    for (int c = 0; c < m; ++c) a.lam[c] = 0.0;
  }
}

cudaError_t loop_step(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st,
                      cudaError_t (*forest_step)(const Plan&, const DevPtrs&, const StepConsts&, cudaStream_t)) {
  const LoopPlan& L = p.loop;
  LoopArgs a;
  a.wr = d.wr_buf;
  a.q = d.b.q;
  a.ld = d.b.ld;
  a.np = (int32_t)L.pa.size();
  a.pa = d.loop_pa;
  a.pb = d.loop_pb;
  a.ya = d.loop_ya;
  a.yb = d.loop_yb;
  a.M = d.loop_M;
  a.lam = d.loop_lam;
  const size_t bytes = sizeof(double) * 12 * (size_t)p.ld;
  cudaError_t e;
  // qⁿ (and the velocity buffer) saved once; every pass starts from them
  if ((e = cudaMemcpyAsync(d.loop_save, d.b.q, bytes, cudaMemcpyDeviceToDevice, st))) return e;
  if ((e = cudaMemcpyAsync(d.loop_save + 12 * p.ld, d.b.qd, bytes, cudaMemcpyDeviceToDevice, st))) return e;
  const int passes = 1 + 3 * a.np;
  for (int c = 0; c < passes; ++c) {
    loop_force_kernel<<<1, 32, 0, st>>>(a, c);
    if ((e = forest_step(p, d, k, st))) return e;
    loop_residual_kernel<<<1, 32, 0, st>>>(a, c);
    if ((e = cudaMemcpyAsync(d.b.q, d.loop_save, bytes, cudaMemcpyDeviceToDevice, st))) return e;
    if ((e = cudaMemcpyAsync(d.b.qd, d.loop_save + 12 * p.ld, bytes, cudaMemcpyDeviceToDevice, st))) return e;
  }
  loop_solve_kernel<<<1, 32, 0, st>>>(a, k);
  loop_force_kernel<<<1, 32, 0, st>>>(a, -1);
  if ((e = forest_step(p, d, k, st))) return e;
  return cudaGetLastError();
}

}  // namespace mabd
