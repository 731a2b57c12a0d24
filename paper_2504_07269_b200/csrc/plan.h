// Plan = symbolic analysis of one spatial sparsity pattern (shared by all
// shifts) + device tables + per-batch numeric workspace.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>
#include <limits.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace stfem {

// One front (supernode) of the multifrontal elimination tree.  Front order
// n = p (pivots, contiguous in the new numbering from pbeg) + b (boundary rows,
// all belonging to ancestors).  Factor block: n x p column-major (ld n): for
// small fronts (shared-memory kernel) D on the diagonal and unit-lower L below;
// for large fronts the complex-symmetric Cholesky factor C (K = C C^T).
// Update block: b x b column-major (lower triangle used).
struct FrontDev {
  int32_t pbeg, p, n, nchild;
  int32_t child_beg;   // into child_ids
  int32_t ent_beg, ent_cnt;  // original (lower-triangle) entries of K owned by this front
  int32_t bidx_beg;    // into bidx: new indices of the b boundary rows
  int32_t relpos_beg;  // into relpos: position of each boundary row in the parent front
  int32_t parent, depth;
  int32_t inv_beg;     // into inv: nchild x n map parent row -> child boundary row (-1 if none)
  int32_t colptr_beg;  // into ent_colptr: p + 1 offsets (relative to ent_beg) of each pivot column's entries
  int64_t fofs;        // factor block offset (complex elements) within one shift
  int64_t uofs;        // update block offset within the pool of parity depth%2 (one shift)
  int64_t rofs;        // forward-RHS update offset (units of b, times nrhs) within its pool
};

// One spectrally eliminated subtree (csrc/spectral.cuh): root front, interior
// size m (pivots [first, first + m) of the plan numbering), boundary size g
// (= the root's boundary rows), offsets (in doubles) of V (m x m), theta (m),
// R then Q (g x m each, column-major), C0 then C1 (g x g each).
struct SubDev {
  int32_t front, m, g, first;
  int64_t vofs, tofs, rqofs, cofs;
};

struct Plan {
  // ---- symbolic (host) ----
  int32_t n = 0;
  int64_t nnz_pattern = 0;
  std::vector<int32_t> perm, iperm;       // perm[new] = old
  std::vector<FrontDev> fronts;           // postorder
  std::vector<int32_t> child_ids, bidx, relpos, ent_src, ent_dst, inv, ent_colptr;
  std::vector<int32_t> diag_src;           // CSR slot of the diagonal entry of every row (-1: none)
  std::vector<std::vector<int32_t>> levels;  // fronts per depth
  int32_t depth = 0, max_front = 0, max_pivots = 0;
  int64_t factor_stride = 0;               // complex per shift
  int64_t upool_stride[2] = {0, 0};        // complex per shift
  int64_t rpool_stride[2] = {0, 0};        // complex per shift per rhs
  int64_t nnz_factor = 0;
  double flops = 0;

  // ---- spectral subtrees (optional, stfem_plan_set_spectral) ----
  std::vector<std::vector<int32_t>> levels_all;   // every front per depth (levels = multifrontal ones)
  std::vector<SubDev> subs;
  std::vector<char> sub_rep;                      // subtree t computes its class's update block (others alias it)
  std::vector<int64_t> uofs0;                     // update-block offsets of the symbolic analysis (before aliasing)
  std::vector<std::vector<int32_t>> sub_levels;   // per depth: indices into subs
  std::vector<double> h_V, h_th, h_RQ, h_C01;
  int64_t spectral_flops_u = 0;                   // DMMA flops per shift of OP_U (4 E m)
  int64_t spectral_flops_rhs = 0;                 // per shift per rhs of F1+F2+B1+B2

  // ---- device tables (uploaded lazily) ----
  int device = -1;
  FrontDev* d_fronts = nullptr;
  int32_t* d_levels = nullptr;             // concatenated level lists
  std::vector<int64_t> level_off;          // offsets into d_levels
  std::vector<int32_t> level_nmax, level_pmax;  // per depth: max front order / pivots
  std::vector<int32_t> level_nsplit;       // per depth: fronts of order > BWD_SPLIT_N (a prefix: levels sorted by n)
  std::vector<int32_t> level_tail_nmax, level_tail_pmax;   // per depth: max order / pivots of the rest
  // tuning knobs (stfem_plan_set_options; measured defaults, C4 ms/step):
  //   fused_min_p  levels whose fronts have >= this many pivots fuse the children's extend-add into
  //                the Schur-update tiles (50 -> 899, 100 -> 902, no fusion -> 907; C5 neutral)
  //   panel_group  trailing pivot-column updates delayed over this many 32-wide panels
  //                (2 -> 96 ms of panel updates, 1 -> 111, 4 -> 108, 8 -> 121)
  //   asm_whole_n  asm_front_kernel assembles a whole front per CTA up to this order
  //                (160 -> 120 ms of assembly, 240 -> 118, every level -> 114)
  //   small_front_n levels of order <= this on the shared-memory small-front kernel (0: none)
  stfem_plan_options opt = default_options();
  static stfem_plan_options default_options() {
    stfem_plan_options o{};
    o.small_front_n = 100;
    o.fused_min_p = 0;
    o.panel_group = 2;
    o.asm_whole_n = INT32_MAX;
    o.level_timing = 0;
    o.tiles_per_cta = 16;
    o.ws_stages = 2;
    o.front_syrk_max_p = 32;
    o.bwd_dmma_min_p = 32;
    o.workspace_fraction = 0.70;
    o.pivot_tol = 1e-10;
    return o;
  }
  int32_t *d_child_ids = nullptr, *d_bidx = nullptr, *d_relpos = nullptr, *d_inv = nullptr;
  int32_t *d_ent_src = nullptr, *d_ent_dst = nullptr, *d_perm = nullptr, *d_ent_colptr = nullptr;
  double *d_ent_mv = nullptr, *d_ent_av = nullptr;   // M_x / A_x values gathered into entry order
  std::vector<int64_t> syrk32_off;         // per depth: offsets into d_syrk32_tiles
  int4* d_syrk32_tiles = nullptr;          // (front, ti, tj, 0) lower 32 x 32 Schur-update tiles of the large fronts
  std::vector<std::vector<int64_t>> panel_off;   // per depth, per panel step (+ end): offsets into d_panel_tiles
  int4* d_panel_tiles = nullptr;           // (front, ti, tj, 0) trailing-update tiles of every (level, panel step)
  std::vector<std::vector<int64_t>> step_off;    // per depth, per panel step (+ end): offsets into d_step_list
  std::vector<std::vector<int32_t>> step_nmax;   // per depth, per panel step: largest order of its fronts
  int32_t* d_step_list = nullptr;          // fronts with a panel at the step (p > kb)
  int* d_err = nullptr;
  int32_t* d_diag_src = nullptr;
  double* d_scale2 = nullptr;              // per shift of the batch: max_j |M_jj + lam A_jj|^2
  SubDev* d_subs = nullptr;
  double *d_V = nullptr, *d_th = nullptr, *d_RQ = nullptr, *d_C01 = nullptr;
  int4* d_spec_items = nullptr;
  std::vector<int64_t> spec_off;
  int spec_smem = 0;                       // dynamic shared memory of spectral_kernel           // (depth+1)*4 + 1: fwd1, fwd2, bwd1, bwd2 item ranges per depth

  // ---- numeric workspace (per batch of shifts) ----
  int32_t batch = 0;       // requested (0 = auto)
  int32_t ws_batch = 0;    // allocated for
  int32_t ws_nrhs = 0;
  int32_t last_batch = 0;  // batch size used by the last factor_solve
  int64_t last_launches = 0;  // kernel launches issued by the last factor_solve
  int32_t last_nbatches = 0;  // shift batches of the last factor_solve
  bool record_levels = false;   // record per-level CUDA-event times into level_ms
  std::vector<double> level_ms;
  std::vector<double> family_ms;   // per kernel family (record mode), summed over batches
  std::vector<int64_t> family_launches;
  cplx* d_factor = nullptr;
  cplx* d_upool[2] = {nullptr, nullptr};
  cplx* d_rpool[2] = {nullptr, nullptr};
  cplx* d_Z = nullptr;
  cplx* d_wbuf = nullptr;                   // spectral w = 1 / (theta + lam), sum(m) x batch
  bool io_permuted = false;                 // G / W of factor_solve are in the plan's (permuted) numbering
  int32_t* d_iperm = nullptr;               // iperm[old] = new, on the device (column maps of the transforms)
  int32_t shift_base = 0;                   // added to the shift index reported by stfem_plan_check
  int* h_err = nullptr;                     // pinned: the latched error flag read back by stfem_plan_check

  ~Plan();
  void free_device();
  void free_workspace();
};

// Leading dimension of a front's b x b update block: b rounded up to 8 complex (128 bytes), so
// every column starts on a cache line and the Schur-update epilogues can store whole lines (the
// DMMA accumulator layout -- 128-byte pieces at 16-byte alignment -- writes at 3.7 TB/s, aligned
// 256-byte pieces at 6 TB/s: tools/probe_store.py)
__host__ __device__ constexpr int ldu(int b) { return (b + 7) & ~7; }

// factor-block offsets (fofs) and factor_stride over the multifrontal fronts only
void assign_factor_offsets(Plan& P, const std::vector<char>& skip);

int build_symbolic(Plan& P, int32_t n, const int64_t* rowptr, const int32_t* colind,
                   const double* coords, int32_t dim, int32_t leaf_size);

}  // namespace stfem
