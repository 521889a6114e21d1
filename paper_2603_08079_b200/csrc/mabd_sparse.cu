// Sparse (loops / irregular networks) solver of the M-ABD step on sm_100a.
//
// The dual S λ = r, S = ∇C̃ H̃⁻¹ ∇C̃ᵀ, r = C(q̃) (P:563-566 with the footnote P:459), is solved by
// preconditioned conjugate gradients with an EXACT matrix-free product (reading A1: the dual
// changes every step because H_j⁻¹ = diag₄(R_j) H̄⁻¹ diag₄(R_jᵀ) rotates; the paper says "any linear solver
// like Cholesky"). Iterations run to ‖r − Sλ‖ ≤ 1e-12‖r‖, so the result agrees with a direct solve
// to the parity tolerance. Preconditioner: the exact 3×3 diagonal blocks of S (block Jacobi).
//
// S·p without forming S (two passes over HBM-resident arrays per product):
//   bodies:  v_j = H_j⁻¹ Σ_{points p on j} s_p Γ(ȳ_p)ᵀ p_p          (12 doubles per body)
//   points:  (S p)_p = s_a Γ(ȳ_a) v_a + s_b Γ(ȳ_b) v_b
// The whole PCG loop is one persistent cooperative kernel (grid.sync between passes); dot products are
// reduced per block and summed by every block in a fixed order (deterministic, no floating atomics).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "mabd_device.cuh"
#include "mabd_plan.h"

namespace cg = cooperative_groups;

namespace mabd {

constexpr int SP_THREADS = 256;

__device__ __forceinline__ void sreport(const StepConsts& k, int32_t flag) {
  atomicOr(k.err, flag);
  atomicMin(k.err + 1, k.step_index);
}

// ---------------------------------------------------------------------------- per-step preparation
// bodies: predict; R → rs scratch, δq̃ parked in the q̇ buffer
__global__ void sparse_predict_kernel(SparseArgs a) {
  const int64_t ld = a.b.ld;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < a.n; j += (int64_t)gridDim.x * blockDim.x) {
    double q[12], qd[12], R[9], dqt[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      q[c] = a.b.q[c * ld + j];
      qd[c] = a.b.qd[c * ld + j];
    }
    const int mid = a.b.mat_id ? a.b.mat_id[j] : 0;
    const double msc = a.b.mscale ? a.b.mscale[j] : 1.0;
    const Material M = a.b.mats[mid];
    HinvBlk H;
    if (a.hinv_tab)
      H = a.hinv_tab[mid];
    else
      hinv_blocks(M, msc, a.k.ih2, H);
    if (!predict_body(q, qd, M, msc, H, a.k.ih, a.k.grav, R, dqt)) sreport(a.k, ERR_NONFINITE);
#pragma unroll
    for (int c = 0; c < 9; ++c) a.b.rs[c * ld + j] = R[c];
#pragma unroll
    for (int c = 0; c < 12; ++c) a.b.qd[c * ld + j] = dqt[c];
  }
}

__device__ __forceinline__ void body_hinv(const SparseArgs& a, int64_t j, HinvBlk& H) {
  const int mid = a.b.mat_id ? a.b.mat_id[j] : 0;
  if (a.hinv_tab)
    H = a.hinv_tab[mid];
  else
    hinv_blocks(a.b.mats[mid], a.b.mscale ? a.b.mscale[j] : 1.0, a.k.ih2, H);
}
__device__ __forceinline__ void body_R(const SparseArgs& a, int64_t j, double* R) {
#pragma unroll
  for (int c = 0; c < 9; ++c) R[c] = a.b.rs[c * a.b.ld + j];
}

// points: r = C(q̃) and the inverse diagonal block D_p⁻¹ of S (block-Jacobi preconditioner)
__global__ void sparse_rhs_kernel(SparseArgs a) {
  const int64_t ld = a.b.ld;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < a.np; p += (int64_t)gridDim.x * blockDim.x) {
    double D[6] = {0, 0, 0, 0, 0, 0}, r[3] = {0, 0, 0};
    for (int side = 0; side < 2; ++side) {
      const int64_t j = side == 0 ? a.pa[p] : a.pb[p];
      const double* y = a.py + 6 * p + 3 * side;
      const double sg = side == 0 ? 1.0 : -1.0;
      if (j < 0) {  // world point
#pragma unroll
        for (int e = 0; e < 3; ++e) r[e] += sg * y[e];
        continue;
      }
      double qt[12], R[9], x[3], P[9], F[6];
#pragma unroll
      for (int c = 0; c < 12; ++c) qt[c] = a.b.q[c * ld + j] + a.b.qd[c * ld + j];
      body_R(a, j, R);
      HinvBlk H;
      body_hinv(a, j, H);
      point_pos(qt, y, x);
#pragma unroll
      for (int e = 0; e < 3; ++e) r[e] += sg * x[e];
      pblock(H, y, y, P);
      rot_conj_sym(R, P, F);
#pragma unroll
      for (int e = 0; e < 6; ++e) D[e] += F[e];
    }
    double Di[6];
    if (!sym_inv_spd(D, Di)) sreport(a.k, ERR_SINGULAR);
#pragma unroll
    for (int e = 0; e < 6; ++e) a.dinv[e * a.np + p] = Di[e];
#pragma unroll
    for (int e = 0; e < 3; ++e) a.rhs[e * a.np + p] = r[e];
  }
}

// v_j = H_j⁻¹ Σ s Γ(ȳ)ᵀ x_p over the points incident to body j (x: [3][np] component-major)
__device__ __forceinline__ void body_apply(const SparseArgs& a, int64_t j, const double* x, const double* z,
                                           double beta, double* out12) {
  double g[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) g[c] = 0.0;
  double R[9];
  body_R(a, j, R);
  for (int i = a.inc_off[j]; i < a.inc_off[j + 1]; ++i) {
    const int32_t e = a.inc[i];
    const int64_t p = e >> 1;
    const int side = e & 1;
    double w[3], wl[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) w[c] = z ? z[c * a.np + p] + beta * x[c * a.np + p] : x[c * a.np + p];
    mat3t_vec(R, w, wl);  // body frame
    add_point_force(g, a.py + 6 * p + 3 * side, wl, side == 0 ? 1.0 : -1.0);
  }
  HinvBlk H;
  body_hinv(a, j, H);
  double u[12];
  hinv_apply(H, g, u);
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) mat3_vec(R, u + 3 * kb, out12 + 3 * kb);
}

// block reduction of NV values into part[blockIdx.x * NV + v]
template <int NV>
__device__ __forceinline__ void block_reduce_store(double (&v)[NV], double* part) {
  __shared__ double red[NV][SP_THREADS / 32];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double x = v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) red[i][threadIdx.x >> 5] = x;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int w = 0; w < SP_THREADS / 32; ++w) s += red[threadIdx.x][w];
    part[blockIdx.x * NV + threadIdx.x] = s;
  }
  __syncthreads();
}

// every block sums the partials in the same order (deterministic). A block may start the next pass (and
// write partials) while others still sum: each reduction kind therefore has its own buffer, and two grid
// syncs separate consecutive uses of the same buffer.
template <int NV>
__device__ __forceinline__ void grid_sum(const double* part, int nblk, double* out) {
  __shared__ double tot[NV];
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += part[b * NV + threadIdx.x];
    tot[threadIdx.x] = s;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) out[i] = tot[i];
  __syncthreads();
}

__global__ void __launch_bounds__(SP_THREADS) sparse_pcg_kernel(SparseArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int nblk = gridDim.x;
  const int64_t np = a.np;
  double* X = a.lam;   // λ
  double* Rr = a.res;  // residual
  double* Z = a.zz;    // preconditioned residual
  double* Pp = a.pp;   // search direction
  double* Ap = a.ap;
  double* V = a.vv;    // [12][n]
  // init: λ = 0, r = rhs, z = D⁻¹r, p = z; partials of r·z and r·r
  {
    double acc[2] = {0.0, 0.0};
    for (int64_t p = tid; p < np; p += nth) {
      double r[3], di[6], z[3];
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        r[e] = a.rhs[e * np + p];
        X[e * np + p] = 0.0;
        Rr[e * np + p] = r[e];
      }
#pragma unroll
      for (int e = 0; e < 6; ++e) di[e] = a.dinv[e * np + p];
      sym_vec(di, r, z);
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        Z[e * np + p] = z[e];
        Pp[e * np + p] = z[e];
        acc[0] += r[e] * z[e];
        acc[1] += r[e] * r[e];
      }
    }
    block_reduce_store<2>(acc, a.part);
  }
  grid.sync();
  double s2[2];
  grid_sum<2>(a.part, nblk, s2);
  double rz = s2[0];
  const double bnorm2 = s2[1];
  const double tol2 = a.tol * a.tol * bnorm2;
  double beta = 0.0, last_r2 = bnorm2;
  bool first = true;
  int it = 0;
  if (bnorm2 > 0.0) {
    for (it = 0; it < a.max_iter; ++it) {
      // pass 1 (bodies): v = H⁻¹ Jᵀ p with p = z + βp (first iteration: p already set)
      for (int64_t j = tid; j < a.n; j += nth) {
        double v[12];
        body_apply(a, j, Pp, first ? nullptr : Z, beta, v);
#pragma unroll
        for (int c = 0; c < 12; ++c) V[c * a.n + j] = v[c];
      }
      grid.sync();
      // pass 2 (points): p ← z + βp (materialised), Ap = J v, partial p·Ap
      {
        double acc[1] = {0.0};
        for (int64_t p = tid; p < np; p += nth) {
          double pv[3], s[3] = {0, 0, 0};
#pragma unroll
          for (int e = 0; e < 3; ++e) {
            pv[e] = first ? Pp[e * np + p] : Z[e * np + p] + beta * Pp[e * np + p];
            Pp[e * np + p] = pv[e];
          }
          for (int side = 0; side < 2; ++side) {
            const int64_t j = side == 0 ? a.pa[p] : a.pb[p];
            if (j < 0) continue;
            const double* y = a.py + 6 * p + 3 * side;
            const double sg = side == 0 ? 1.0 : -1.0;
#pragma unroll
            for (int e = 0; e < 3; ++e)
              s[e] += sg * (V[(0 + e) * a.n + j] * y[0] + V[(3 + e) * a.n + j] * y[1] + V[(6 + e) * a.n + j] * y[2] +
                            V[(9 + e) * a.n + j]);
          }
#pragma unroll
          for (int e = 0; e < 3; ++e) {
            Ap[e * np + p] = s[e];
            acc[0] += pv[e] * s[e];
          }
        }
        block_reduce_store<1>(acc, a.part + 2 * SPARSE_MAX_BLOCKS);
      }
      grid.sync();
      double pAp[1];
      grid_sum<1>(a.part + 2 * SPARSE_MAX_BLOCKS, nblk, pAp);
      const double alpha = rz / pAp[0];
      // pass 3 (points): λ += αp, r −= αAp, z = D⁻¹r; partials r·z, r·r
      {
        double acc[2] = {0.0, 0.0};
        for (int64_t p = tid; p < np; p += nth) {
          double r[3], di[6], z[3];
#pragma unroll
          for (int e = 0; e < 3; ++e) {
            X[e * np + p] += alpha * Pp[e * np + p];
            r[e] = Rr[e * np + p] - alpha * Ap[e * np + p];
            Rr[e * np + p] = r[e];
          }
#pragma unroll
          for (int e = 0; e < 6; ++e) di[e] = a.dinv[e * np + p];
          sym_vec(di, r, z);
#pragma unroll
          for (int e = 0; e < 3; ++e) {
            Z[e * np + p] = z[e];
            acc[0] += r[e] * z[e];
            acc[1] += r[e] * r[e];
          }
        }
        block_reduce_store<2>(acc, a.part);
      }
      grid.sync();
      grid_sum<2>(a.part, nblk, s2);
      beta = s2[0] / rz;
      rz = s2[0];
      first = false;
      last_r2 = s2[1];
      if (s2[1] <= tol2) {
        ++it;
        break;
      }
    }
  }
  if (tid == 0) {
    a.iters[0] = it;
    // the recursive residual stagnates at the fp64 floor (~1e-13 relative for these duals); only a residual
    // still above 1e-9 of ‖b‖ after max_iter is a failure
    if (it >= a.max_iter && last_r2 > 1e-18 * bnorm2) sreport(a.k, ERR_SINGULAR);
  }
}

// bodies: qⁿ⁺¹ = q̃ − H⁻¹ Jᵀ λ, q̇ⁿ⁺¹ = δq/h
__global__ void sparse_update_kernel(SparseArgs a) {
  const int64_t ld = a.b.ld;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < a.n; j += (int64_t)gridDim.x * blockDim.x) {
    double v[12];
    body_apply(a, j, a.lam, nullptr, 0.0, v);
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      const double dq = a.b.qd[c * ld + j] - v[c];
      a.b.q[c * ld + j] += dq;
      a.b.qd[c * ld + j] = dq * a.k.ih;
    }
  }
}

static int g_sparse_grid = 0;

cudaError_t sparse_init() {
  int dev = 0, nsm = 0, per = 0;
  cudaError_t e;
  if ((e = cudaGetDevice(&dev))) return e;
  if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev))) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sparse_pcg_kernel, SP_THREADS, 0))) return e;
  g_sparse_grid = std::max(1, std::min(per, 4) * nsm);
  return cudaSuccess;
}

int sparse_grid_blocks() { return g_sparse_grid; }

cudaError_t sparse_step(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st) {
  SparseArgs a = d.sparse;
  a.k = k;
  const int nb = (int)std::min<int64_t>((a.n + 255) / 256, 148 * 8);
  const int npb = (int)std::min<int64_t>((a.np + 255) / 256, 148 * 8);
  sparse_predict_kernel<<<std::max(nb, 1), 256, 0, st>>>(a);
  sparse_rhs_kernel<<<std::max(npb, 1), 256, 0, st>>>(a);
  void* args[] = {&a};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)sparse_pcg_kernel, dim3(g_sparse_grid), dim3(SP_THREADS), args,
                                              0, st);
  if (e != cudaSuccess) return e;
  sparse_update_kernel<<<std::max(nb, 1), 256, 0, st>>>(a);
  (void)p;
  return cudaGetLastError();
}

// ============================================================================ host: point lists and incidence
bool sparse_build(const mabd_joints* J, int64_t n, Plan* p, std::vector<int64_t>* pos_of_body, std::string* msg) {
  const int64_t K = J->n_joints;
  SparsePlan& s = p->sparse;
  s = SparsePlan();
  int64_t P = 0;
  for (int64_t k = 0; k < K; ++k) P += J->npts[k];
  s.np = P;
  s.pa.resize(P);
  s.pb.resize(P);
  s.py.resize(6 * P);
  std::vector<int32_t> cnt(n + 1, 0);
  int64_t pt = 0;
  for (int64_t k = 0; k < K; ++k)
    for (int q = 0; q < J->npts[k]; ++q, ++pt) {
      s.pa[pt] = J->body_a[k];
      s.pb[pt] = J->body_b[k];
      for (int e = 0; e < 3; ++e) {
        s.py[6 * pt + e] = J->ybar_a[3 * pt + e];
        s.py[6 * pt + 3 + e] = J->ybar_b[3 * pt + e];
      }
      cnt[J->body_a[k] + 1]++;
      if (J->body_b[k] >= 0) cnt[J->body_b[k] + 1]++;
    }
  s.inc_off.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) s.inc_off[i + 1] = s.inc_off[i] + cnt[i + 1];
  s.inc.assign(s.inc_off[n], 0);
  std::vector<int32_t> fill(n, 0);
  for (int64_t q = 0; q < P; ++q) {
    const int64_t a = s.pa[q], b = s.pb[q];
    s.inc[s.inc_off[a] + fill[a]++] = (int32_t)(2 * q);
    if (b >= 0) s.inc[s.inc_off[b] + fill[b]++] = (int32_t)(2 * q + 1);
  }
  if (2 * P > (int64_t)INT32_MAX) return *msg = "too many joint points", false;
  pos_of_body->resize(n);
  for (int64_t i = 0; i < n; ++i) (*pos_of_body)[i] = i;  // caller order (grids are already local)
  p->ld = n;
  p->n_dual_rows = 3 * P;
  p->launches_per_step = 4;
  return true;
}

}  // namespace mabd
