// Host-side plan: topology analysis, ordering and the device memory layout (internal).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/mabd.h"
#include "mabd_internal.h"
#include "mabd_kernels.h"

namespace mabd {

struct BtdLevel {
  int64_t n_u;     // unknowns at this level
  int64_t windows; // CTAs
  bool fused;      // top level (n_u ≤ 256)
};

// Tree plan (leaf-to-root elimination, reading A12); see mabd_tree.cu.
struct TreePlan {
  int64_t n_levels = 0;
  std::vector<int64_t> level_off;    // [n_levels+1] body ranges per depth (internal order is by depth)
  std::vector<int32_t> parent;       // [n] internal parent index (−1 for roots)
  std::vector<int32_t> up_joint;     // [n] internal joint index of the joint to the parent (−1 if none)
  std::vector<int32_t> child_off;    // [n+1] CSR of the body's "child joints" (incl. anchors)
  std::vector<int32_t> child_joint;  // joint ids
  std::vector<int32_t> jrow_off;     // [K+1] dual row offset per joint (3 or 6 rows)
  std::vector<int32_t> jnpts;        // [K]
  std::vector<int32_t> jparent;      // [K] body the joint hangs from (internal index)
  std::vector<int32_t> jchild;       // [K] child body (internal) or −1 for anchors
  std::vector<double> jy_par;        // [K][2][3] material points on the parent body
  std::vector<double> jy_chd;        // [K][2][3] material points on the child body, or world points
  int32_t max_child_rows = 0;
};

struct Plan {
  int64_t n = 0, n_joints = 0, n_dual_rows = 0;
  int32_t solver = 0;
  int32_t launches_per_step = 0;
  double grav[3] = {0, 0, 0};
  // bodies
  std::vector<Material> mats;
  std::vector<int32_t> mat_id;   // [ld] (empty if one material)
  std::vector<double> mscale;    // [ld] (empty if all 1)
  std::vector<int64_t> perm;     // caller body → internal position
  int64_t ld = 0;                // SoA stride (positions)
  std::vector<double> q_soa, qd_soa;  // [12][ld]
  // chain solver
  int64_t n_windows = 0;
  std::vector<uint32_t> slot_info;   // [ld+1]
  std::vector<double> geo;           // [ng][6]
  std::vector<int32_t> seg_flags, seg_red, long_list, left_iface;
  int64_t n_long = 0;
  std::vector<BtdLevel> levels;      // levels[0] is BTD level 1
  // tree solver
  TreePlan tree;
  // device layout (byte offsets into the workspace)
  size_t workspace_bytes = 0;
  struct Off {
    size_t q, qd, rs, mat_id, mscale, mats, hinv, perm, io, err;
    size_t slot_info, geo, seg_flags, seg_red, long_list, left_iface;
    std::vector<size_t> tops, lams;  // per BTD level: tops[0] = chain tops (n_long), lams[i] = level i+1 λ
    size_t tree_base;
    std::vector<size_t> tree_off;
  } off{};
};

struct DevPtrs {
  BodyArrays b{};
  HinvBlk* hinv = nullptr;
  Material* mats = nullptr;
  int64_t* perm = nullptr;
  double* io = nullptr;
  int32_t* err = nullptr;
  uint32_t* slot_info = nullptr;
  double* geo = nullptr;
  int32_t *seg_flags = nullptr, *seg_red = nullptr, *long_list = nullptr, *left_iface = nullptr;
  std::vector<Top*> tops;
  std::vector<double*> lams;
  std::vector<void*> tree;           // tree arrays (see mabd_tree.cu)
};

mabd_status build_plan(const mabd_bodies* bodies, const mabd_joints* joints, const mabd_options* opts, Plan* p,
                       std::string* msg);
cudaError_t upload_plan(const Plan& p, char* ws, cudaStream_t st, DevPtrs* d);
cudaError_t prefactor_device(const Plan& p, const DevPtrs& d, double h, cudaStream_t st);
cudaError_t reset_err(const DevPtrs& d, cudaStream_t st);
cudaError_t launch_step(const Plan& p, const DevPtrs& d, double h, int32_t step, cudaStream_t st);

// tree solver hooks (mabd_tree.cu)
bool tree_build(const mabd_joints* joints, int64_t n, Plan* p, std::string* msg, std::vector<int64_t>* order);
void tree_layout(Plan* p, size_t* cursor);
cudaError_t tree_upload(const Plan& p, char* ws, cudaStream_t st, DevPtrs* d);
cudaError_t tree_step(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st);

}  // namespace mabd
