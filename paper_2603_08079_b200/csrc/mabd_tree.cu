// Tree solver of the M-ABD step on sm_100a: exact leaf-to-root elimination of the dual (reading A12;
// the exact form of the paper's ABD-ABA, Alg. 2).
//
// Every joint k hangs from a "parent" body p_k and has a child body c_k (or the world, for an anchor);
// C_k = x_p(ȳ_p) − x_c(ȳ_c) (or − p_world), 3 rows per point (ball: 1 point, linear hinge: 2 points).
// Up (deepest bodies first), for body b with child joints X and up joint u, the frontal matrix
//   F = G H_b⁻¹ Gᵀ + diag(Ŝ_k, k ∈ X),  G = stacked ±Γ(ȳ) rows of the points on b,  H_b⁻¹ = diag₄(R)H̄⁻¹diag₄(Rᵀ)
// (blocks ±R P(ȳ,ȳ') Rᵀ, P the constant 3×3 kernels of mabd_device.cuh) is factored on X:
//   Ŝ_u = F_uu − F_uX F_XX⁻¹ F_Xu,  r̂_u = r_u − F_uX F_XX⁻¹ r_X        (condensed child side of joint u)
// Down (root first): λ_X = F_XX⁻¹(r_X − F_Xu λ_u), then qⁿ⁺¹ = q̃ − diag₄(R)H̄⁻¹Σ±Γᵀ Rᵀλ.
// The dual graph of a tree is chordal in this order, so the elimination has no fill (PROBE in SURVEY A12).
//
// Parallel schedule: bodies are grouped into CTA-local subtrees (≤ 256 bodies; levels separated by
// __syncthreads) plus one top group (bodies whose subtree is larger) processed by a single CTA.
// Launches per step: up(bottom) → up+down(top) → down(bottom), or one fused launch when there is no top.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "mabd_device.cuh"
#include "mabd_plan.h"

namespace mabd {

constexpr int TMAXM = TREE_MAXN + 6;

__device__ __forceinline__ void treport(const StepConsts& k, int32_t flag) {
  atomicOr(k.err, flag);
  atomicMin(k.err + 1, k.step_index);
}

// Body b's frontal matrix is ordered: the points of its child joints (sign +, b is their parent side), then
// the points of its up joint (sign −, b is its child side).
__device__ void tree_up(const TreeArgs& a, int b) {
  const StepConsts& k = a.k;
  const int64_t ld = a.b.ld;
  // ---- stage 1-2: predict
  double q[12], R[9], dqt[12];
  HinvBlk H;
  {
    double qd[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      q[c] = a.b.q[c * ld + b];
      qd[c] = a.b.qd[c * ld + b];
    }
    const int mid = a.b.mat_id ? a.b.mat_id[b] : 0;
    const double msc = a.b.mscale ? a.b.mscale[b] : 1.0;
    const Material M = a.b.mats[mid];
    if (a.hinv_tab)
      H = a.hinv_tab[mid];
    else
      hinv_blocks(M, msc, k.ih2, H);
    if (!predict_body(q, qd, M, msc, H, k.ih, k.grav, R, dqt)) treport(k, ERR_NONFINITE);
    double* sc = a.bscr + 21 * (int64_t)b;
#pragma unroll
    for (int c = 0; c < 9; ++c) sc[c] = R[c];
#pragma unroll
    for (int c = 0; c < 12; ++c) sc[9 + c] = dqt[c];
#pragma unroll
    for (int c = 0; c < 12; ++c) q[c] += dqt[c];  // q̃
  }
  // ---- frontal matrix
  const int c0 = a.child_off[b], c1 = a.child_off[b + 1];
  const int u = a.up_joint[b];
  int N = 0;
  for (int j = c0; j < c1; ++j) N += 3 * a.jnpts[a.child_joint[j]];
  const int nu = u >= 0 ? 3 * a.jnpts[u] : 0;
  const int M = N + nu;
  double F[TMAXM * TMAXM];
  double rhs[TMAXM];
  // point list
  const int npt = M / 3;
  for (int i = 0; i < npt; ++i) {
    int ji, pi;
    double si;
    const double* yi;
    {
      int row = 3 * i, jj = c0;
      if (row < N) {
        while (true) {
          const int n3 = 3 * a.jnpts[a.child_joint[jj]];
          if (row < n3) break;
          row -= n3;
          ++jj;
        }
        ji = a.child_joint[jj];
        pi = row / 3;
        si = 1.0;
        yi = a.jy + 12 * (int64_t)ji + 3 * pi;
      } else {
        ji = u;
        pi = (row - N) / 3;
        si = -1.0;
        yi = a.jy + 12 * (int64_t)ji + 6 + 3 * pi;
      }
    }
    // rhs: this body's side of C(q̃) plus the condensed child side
    double x[3];
    point_pos(q, yi, x);
    if (si > 0) {
      if (a.jchd[ji] < 0) {  // anchor: C = x_b(ȳ) − p_world
        const double* pw = a.jy + 12 * (int64_t)ji + 6 + 3 * pi;
#pragma unroll
        for (int e = 0; e < 3; ++e) rhs[3 * i + e] = x[e] - pw[e];
      } else {
#pragma unroll
        for (int e = 0; e < 3; ++e) rhs[3 * i + e] = x[e] + a.rhat[6 * (int64_t)ji + 3 * pi + e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < 3; ++e) rhs[3 * i + e] = -x[e];
    }
    for (int j = 0; j <= i; ++j) {
      int jj2, pj;
      double sj;
      const double* yj;
      {
        int row = 3 * j, jj = c0;
        if (row < N) {
          while (true) {
            const int n3 = 3 * a.jnpts[a.child_joint[jj]];
            if (row < n3) break;
            row -= n3;
            ++jj;
          }
          jj2 = a.child_joint[jj];
          pj = row / 3;
          sj = 1.0;
          yj = a.jy + 12 * (int64_t)jj2 + 3 * pj;
        } else {
          jj2 = u;
          pj = (row - N) / 3;
          sj = -1.0;
          yj = a.jy + 12 * (int64_t)jj2 + 6 + 3 * pj;
        }
      }
      double P[9], Bk[9];
      pblock(H, yi, yj, P);
      rot_conj(R, P, Bk);
      const double sg = si * sj;
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          double v = sg * Bk[3 * r + c];
          if (si > 0 && sj > 0 && ji == jj2 && a.jchd[ji] >= 0)  // + condensed child side Ŝ_k
            v += a.Shat[36 * (int64_t)ji + 6 * (3 * pi + r) + 3 * pj + c];
          F[(3 * i + r) * TMAXM + 3 * j + c] = v;
          F[(3 * j + c) * TMAXM + 3 * i + r] = v;
        }
    }
  }
  // ---- Cholesky of F_XX (lower, in place)
  for (int c = 0; c < N; ++c) {
    double d = F[c * TMAXM + c];
    for (int m = 0; m < c; ++m) d -= F[c * TMAXM + m] * F[c * TMAXM + m];
    if (!(d > 0.0)) {
      treport(k, ERR_SINGULAR);
      d = 1.0;
    }
    const double l = sqrt(d), il = 1.0 / l;
    F[c * TMAXM + c] = l;
    for (int r = c + 1; r < N; ++r) {
      double v = F[r * TMAXM + c];
      for (int m = 0; m < c; ++m) v -= F[r * TMAXM + m] * F[c * TMAXM + m];
      F[r * TMAXM + c] = v * il;
    }
  }
  // solve F_XX Z = [r_X | F_Xu] for Z = [y | W] (columns: 0 = rhs, 1..nu = F_Xu columns)
  double* ws = a.ws + a.ws_off[b];  // y [N], W [N][nu]
  for (int col = 0; col <= nu; ++col) {
    double z[TREE_MAXN];
    for (int r = 0; r < N; ++r) z[r] = col == 0 ? rhs[r] : F[r * TMAXM + N + col - 1];
    for (int r = 0; r < N; ++r) {  // L z' = z
      double v = z[r];
      for (int m = 0; m < r; ++m) v -= F[r * TMAXM + m] * z[m];
      z[r] = v / F[r * TMAXM + r];
    }
    for (int r = N - 1; r >= 0; --r) {  // Lᵀ z = z'
      double v = z[r];
      for (int m = r + 1; m < N; ++m) v -= F[m * TMAXM + r] * z[m];
      z[r] = v / F[r * TMAXM + r];
    }
    for (int r = 0; r < N; ++r) {
      if (col == 0)
        ws[r] = z[r];
      else
        ws[N + r * nu + col - 1] = z[r];
    }
  }
  if (u >= 0) {  // condensed child side of the up joint
    for (int r = 0; r < nu; ++r) {
      double rv = rhs[N + r];
      for (int m = 0; m < N; ++m) rv -= F[m * TMAXM + N + r] * ws[m];
      a.rhat[6 * (int64_t)u + r] = rv;
      for (int c = 0; c < nu; ++c) {
        double v = F[(N + r) * TMAXM + N + c];
        for (int m = 0; m < N; ++m) v -= F[m * TMAXM + N + r] * ws[N + m * nu + c];
        a.Shat[36 * (int64_t)u + 6 * r + c] = v;
      }
    }
  } else {  // root: λ_X = y
    int off = 0;
    for (int j = c0; j < c1; ++j) {
      const int kj = a.child_joint[j];
      const int n3 = 3 * a.jnpts[kj];
      for (int r = 0; r < n3; ++r) a.lam[6 * (int64_t)kj + r] = ws[off + r];
      off += n3;
    }
  }
}

__device__ void tree_down(const TreeArgs& a, int b) {
  const StepConsts& k = a.k;
  const int64_t ld = a.b.ld;
  const int c0 = a.child_off[b], c1 = a.child_off[b + 1];
  const int u = a.up_joint[b];
  int N = 0;
  for (int j = c0; j < c1; ++j) N += 3 * a.jnpts[a.child_joint[j]];
  const int nu = u >= 0 ? 3 * a.jnpts[u] : 0;
  const double* ws = a.ws + a.ws_off[b];
  double lu[6] = {0, 0, 0, 0, 0, 0};
  for (int r = 0; r < nu; ++r) lu[r] = a.lam[6 * (int64_t)u + r];
  if (u >= 0) {  // λ_X = y − W λ_u
    int off = 0;
    for (int j = c0; j < c1; ++j) {
      const int kj = a.child_joint[j];
      const int n3 = 3 * a.jnpts[kj];
      for (int r = 0; r < n3; ++r) {
        double v = ws[off + r];
        for (int c = 0; c < nu; ++c) v -= ws[N + (off + r) * nu + c] * lu[c];
        a.lam[6 * (int64_t)kj + r] = v;
      }
      off += n3;
    }
  }
  // stage 4: qⁿ⁺¹ = q̃ − diag₄(R) H̄⁻¹ Σ ±Γ(ȳ)ᵀ Rᵀλ
  const double* sc = a.bscr + 21 * (int64_t)b;
  double R[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) R[c] = sc[c];
  double gq[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) gq[c] = 0.0;
  for (int j = c0; j < c1; ++j) {
    const int kj = a.child_joint[j];
    for (int p = 0; p < a.jnpts[kj]; ++p) {
      double lam[3], w[3];
#pragma unroll
      for (int e = 0; e < 3; ++e) lam[e] = a.lam[6 * (int64_t)kj + 3 * p + e];
      mat3t_vec(R, lam, w);
      add_point_force(gq, a.jy + 12 * (int64_t)kj + 3 * p, w, 1.0);
    }
  }
  for (int p = 0; p < nu / 3; ++p) {
    double w[3];
    mat3t_vec(R, lu + 3 * p, w);
    add_point_force(gq, a.jy + 12 * (int64_t)u + 6 + 3 * p, w, -1.0);
  }
  HinvBlk H;
  const int mid = a.b.mat_id ? a.b.mat_id[b] : 0;
  if (a.hinv_tab)
    H = a.hinv_tab[mid];
  else
    hinv_blocks(a.b.mats[mid], a.b.mscale ? a.b.mscale[b] : 1.0, k.ih2, H);
  double uu[12];
  hinv_apply(H, gq, uu);
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    double c3[3];
    mat3_vec(R, uu + 3 * kb, c3);
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      const int c = 3 * kb + e;
      const double dq = sc[9 + c] - c3[e];
      a.b.q[c * ld + b] += dq;
      a.b.qd[c * ld + b] = dq * k.ih;
    }
  }
}

__global__ void __launch_bounds__(256) tree_kernel(TreeArgs a, int mode) {
  const int g = a.group0 + blockIdx.x;
  const int l0 = a.glev_ptr[g], l1 = a.glev_ptr[g + 1] - 1;  // levels l ∈ [l0, l1): [glev_off[l], glev_off[l+1])
  if (mode == TREE_UP || mode == TREE_BOTH) {
    for (int l = l0; l < l1; ++l) {  // deepest first
      for (int b = a.glev_off[l] + threadIdx.x; b < a.glev_off[l + 1]; b += blockDim.x) tree_up(a, b);
      __syncthreads();
    }
  }
  if (mode == TREE_DOWN || mode == TREE_BOTH) {
    for (int l = l1 - 1; l >= l0; --l) {  // shallowest first
      for (int b = a.glev_off[l] + threadIdx.x; b < a.glev_off[l + 1]; b += blockDim.x) tree_down(a, b);
      __syncthreads();
    }
  }
}

cudaError_t launch_tree(const TreeArgs& a, int ngroups, int mode, cudaStream_t st) {
  if (ngroups <= 0) return cudaSuccess;
  tree_kernel<<<ngroups, 256, 0, st>>>(a, mode);
  return cudaGetLastError();
}

cudaError_t tree_step(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st) {
  TreeArgs a = d.tree;
  a.k = k;
  const TreePlan& t = p.tree;
  cudaError_t e;
  if (!t.has_top) return launch_tree(a, t.n_bottom, TREE_BOTH, st);
  a.group0 = 0;
  if ((e = launch_tree(a, t.n_bottom, TREE_UP, st))) return e;
  a.group0 = t.n_bottom;
  if ((e = launch_tree(a, 1, TREE_BOTH, st))) return e;
  a.group0 = 0;
  return launch_tree(a, t.n_bottom, TREE_DOWN, st);
}

// ============================================================================ host: topology and ordering
bool tree_build(const mabd_joints* J, int64_t n, Plan* p, std::vector<int64_t>* pos_of_body, std::string* msg) {
  const int64_t K = J->n_joints;
  // union-find over inter-body joints: a repeated connection is a cycle
  std::vector<int64_t> uf(n);
  for (int64_t i = 0; i < n; ++i) uf[i] = i;
  auto find = [&](int64_t x) {
    while (uf[x] != x) x = uf[x] = uf[uf[x]];
    return x;
  };
  std::vector<int64_t> pt_off(K + 1, 0);
  std::vector<std::vector<std::pair<int64_t, int64_t>>> adj(n);  // (neighbour, joint)
  for (int64_t k = 0; k < K; ++k) {
    pt_off[k + 1] = pt_off[k] + J->npts[k];
    const int64_t a = J->body_a[k], b = J->body_b[k];
    if (b < 0) continue;
    const int64_t ra = find(a), rb = find(b);
    if (ra == rb) return *msg = "cycle in the joint graph (tree solver)", false;
    uf[ra] = rb;
    adj[a].push_back({b, k});
    adj[b].push_back({a, k});
  }
  // root every component at a centre (repeated leaf peeling) to minimise the depth
  std::vector<int64_t> deg(n);
  for (int64_t i = 0; i < n; ++i) deg[i] = (int64_t)adj[i].size();
  std::vector<int64_t> comp_root(n, -1);
  {
    std::vector<int64_t> layer;
    std::vector<int64_t> d2 = deg;
    std::vector<char> peeled(n, 0);
    for (int64_t i = 0; i < n; ++i)
      if (d2[i] <= 1) layer.push_back(i);
    std::vector<int64_t> order_peel;
    while (!layer.empty()) {
      std::vector<int64_t> next;
      for (int64_t v : layer) {
        peeled[v] = 1;
        order_peel.push_back(v);
        for (auto& e : adj[v])
          if (!peeled[e.first] && --d2[e.first] == 1) next.push_back(e.first);
      }
      layer.swap(next);
    }
    // the last peeled body of each component is a centre
    for (auto it = order_peel.rbegin(); it != order_peel.rend(); ++it) {
      const int64_t c = find(*it);
      if (comp_root[c] < 0) comp_root[c] = *it;
    }
  }
  std::vector<int64_t> parent(n, -1), upj(n, -1), depth(n, 0), bfs;
  bfs.reserve(n);
  std::vector<char> seen(n, 0);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t r = comp_root[find(i)];
    if (seen[r]) continue;
    seen[r] = 1;
    size_t h = bfs.size();
    bfs.push_back(r);
    while (h < bfs.size()) {
      const int64_t v = bfs[h++];
      for (auto& e : adj[v])
        if (!seen[e.first]) {
          seen[e.first] = 1;
          parent[e.first] = v;
          upj[e.first] = e.second;
          depth[e.first] = depth[v] + 1;
          bfs.push_back(e.first);
        }
    }
  }
  // subtree sizes and groups
  std::vector<int64_t> size(n, 1);
  for (auto it = bfs.rbegin(); it != bfs.rend(); ++it)
    if (parent[*it] >= 0) size[parent[*it]] += size[*it];
  std::vector<int64_t> local_roots;
  for (int64_t v : bfs)
    if (size[v] <= TREE_CAP && (parent[v] < 0 || size[parent[v]] > TREE_CAP)) local_roots.push_back(v);
  // children lists for subtree collection
  std::vector<std::vector<int64_t>> kids(n);
  for (int64_t v : bfs)
    if (parent[v] >= 0) kids[parent[v]].push_back(v);
  std::vector<std::vector<int64_t>> groups;
  std::vector<int64_t> cur;
  for (int64_t r : local_roots) {
    std::vector<int64_t> sub{r};
    for (size_t h = 0; h < sub.size(); ++h)
      for (int64_t c : kids[sub[h]]) sub.push_back(c);
    if (cur.size() + sub.size() > (size_t)TREE_CAP) {
      groups.push_back(cur);
      cur.clear();
    }
    cur.insert(cur.end(), sub.begin(), sub.end());
  }
  if (!cur.empty()) groups.push_back(cur);
  TreePlan& t = p->tree;
  t = TreePlan();
  t.n_bottom = (int32_t)groups.size();
  std::vector<int64_t> top;
  for (int64_t v : bfs)
    if (size[v] > TREE_CAP) top.push_back(v);
  if (!top.empty()) {
    groups.push_back(top);
    t.has_top = true;
  }
  // internal order: groups in sequence, each sorted by depth (deepest first). Level ranges: group g owns
  // levels l ∈ [glev_ptr[g], glev_ptr[g+1]−1), level l spans bodies [glev_off[l], glev_off[l+1]).
  pos_of_body->assign(n, -1);
  std::vector<int64_t> body_of(n);
  int64_t pos = 0;
  t.group_off.push_back(0);
  for (auto& gvec : groups) {
    std::stable_sort(gvec.begin(), gvec.end(), [&](int64_t x, int64_t y) { return depth[x] > depth[y]; });
    t.glev_ptr.push_back((int32_t)t.glev_off.size());
    for (size_t i = 0; i < gvec.size(); ++i) {
      if (i == 0 || depth[gvec[i]] != depth[gvec[i - 1]]) t.glev_off.push_back((int32_t)(pos + i));
      (*pos_of_body)[gvec[i]] = pos + (int64_t)i;
      body_of[pos + i] = gvec[i];
    }
    pos += (int64_t)gvec.size();
    t.glev_off.push_back((int32_t)pos);  // terminator of the group's last level
    t.group_off.push_back((int32_t)pos);
  }
  t.glev_ptr.push_back((int32_t)t.glev_off.size());
  // joints
  t.jnpts.assign(K, 0);
  t.jchd.assign(K, -1);
  t.jy.assign(12 * K, 0.0);
  std::vector<int64_t> jpar(K, -1);
  int64_t rows = 0;
  for (int64_t k = 0; k < K; ++k) {
    const int64_t a = J->body_a[k], b = J->body_b[k];
    const int np = J->npts[k];
    t.jnpts[k] = np;
    rows += 3 * np;
    const double* ya = J->ybar_a + 3 * pt_off[k];
    const double* yb = J->ybar_b + 3 * pt_off[k];
    const double *yp, *yc;
    if (b < 0) {
      jpar[k] = a;
      yp = ya;
      yc = yb;
    } else if (parent[b] == a && upj[b] == k) {
      jpar[k] = a;
      t.jchd[k] = (int32_t)(*pos_of_body)[b];
      yp = ya;
      yc = yb;
    } else {
      jpar[k] = b;
      t.jchd[k] = (int32_t)(*pos_of_body)[a];
      yp = yb;
      yc = ya;
    }
    for (int q = 0; q < 3 * np; ++q) {
      t.jy[12 * k + q] = yp[q];
      t.jy[12 * k + 6 + q] = yc[q];
    }
  }
  p->n_dual_rows = rows;
  // per internal body: up joint, child joints, workspace
  t.up_joint.assign(n, -1);
  std::vector<std::vector<int32_t>> cj(n);
  for (int64_t k = 0; k < K; ++k) cj[(*pos_of_body)[jpar[k]]].push_back((int32_t)k);
  t.child_off.assign(n + 1, 0);
  t.ws_off.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t v = body_of[i];
    t.up_joint[i] = (int32_t)upj[v];
    int N = 0;
    for (int32_t kk : cj[i]) N += 3 * t.jnpts[kk];
    if (N > TREE_MAXN) return *msg = "a body carries more than 24 child-joint rows (tree solver limit)", false;
    const int nu = upj[v] >= 0 ? 3 * t.jnpts[upj[v]] : 0;
    t.child_off[i + 1] = t.child_off[i] + (int32_t)cj[i].size();
    for (int32_t kk : cj[i]) t.child_joint.push_back(kk);
    t.ws_off[i + 1] = t.ws_off[i] + N + (int64_t)N * nu;
  }
  t.ws_total = t.ws_off[n];
  p->ld = n;
  p->launches_per_step = t.has_top ? (t.n_bottom > 0 ? 3 : 1) : 1;
  return true;
}

}  // namespace mabd
