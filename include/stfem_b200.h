/*
 * stfem_b200 — C-ABI of the B200-native FDM space-time solver.
 *
 * Drop-in boundary for the reference's FDM hot path (arxiv 2504.07269).  The
 * reference has no FFI: its boundary is the in-process Python library API of
 * SPEC.md.  Each entry point below replaces one SPEC operation;
 * the Python host package (paper_2504_07269_b200) binds them with ctypes and
 * exposes the SPEC names.  Plain pointers and sizes only; every device buffer
 * is caller-owned (torch tensors on the Python side); all calls are
 * stream-ordered on the caller's stream (`stream` = cudaStream_t, NULL = legacy
 * default stream).
 *
 * Complex numbers are interleaved (re, im) float64 pairs ("c128"), exactly
 * torch.complex128 / numpy complex128 memory.
 *
 * Return value: STFEM_OK or an error code; stfem_last_error() gives the
 * message (thread-local).
 */
#ifndef STFEM_B200_H
#define STFEM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  STFEM_OK = 0,
  STFEM_ERR_ARG = 1,        /* invalid argument */
  STFEM_ERR_DIM = 2,        /* dimension mismatch */
  STFEM_ERR_SINGULAR = 3,   /* pivot collapse; see stfem_last_error for the shift */
  STFEM_ERR_CUDA = 4,
  STFEM_ERR_NOMEM = 5,
  STFEM_ERR_INTERNAL = 6,
  STFEM_ERR_NCCL = 7,
};

typedef struct stfem_plan stfem_plan;   /* symbolic analysis + device tables for one spatial pattern */
typedef struct stfem_asm stfem_asm;     /* mesh + CSR pattern + colouring for assembly */

const char* stfem_last_error(void);
int stfem_version(void);
int stfem_cuda_device_count(void);

/* ---------------------------------------------------------------------------
 * BlockVector addressing ("BlockVector", temporal index outer)
 * Element (rhs r, temporal/shift index l, spatial DoF j) lives at complex
 * offset   r*rhs_stride + l*shift_stride + (j / chunk_cols)*chunk_stride + j % chunk_cols.
 * A single (n_t, n_x) BlockVector: rhs_stride = n_t*n_x, shift_stride = n_x,
 * chunk_cols = n_x, chunk_stride = 0.  The chunked form addresses the receive
 * buffer of the spatial->temporal all-to-all without a repack.
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t rhs_stride;
  int64_t shift_stride;
  int64_t chunk_cols;
  int64_t chunk_stride;
} stfem_bv_layout;

/* ---------------------------------------------------------------------------
 * K3  transform_blocks (SPEC.md:392-400, steps 2 and 4 of solve, :377):
 *   out[b][l][j] = sum_k T[l][k] * in[b][k][j]     (complex128)
 * T: device, nt x nt row-major c128.  in/out: device, row stride ld_in/ld_out
 * (complex elements), `ncols` columns, `batch` matrices `bstride_*` apart.
 * Complex-fp64 GEMM on the FP64 tensor pipe (DMMA), cp.async-staged tiles.
 * ------------------------------------------------------------------------- */
int stfem_time_transform(const void* T, int nt, const void* in, int64_t ld_in,
                         void* out, int64_t ld_out, int64_t ncols, int batch,
                         int64_t bstride_in, int64_t bstride_out, void* stream);

/* ---------------------------------------------------------------------------
 * K3p  eigenpair-paired transforms (same contract as K3 for FD factors whose
 * eigenvalues pair as (lam, -conj(lam)) -- always the case for the real
 * temporal pencil of SPEC.md:181-189; host pairing and derivation in
 * paper_2504_07269_b200/paired_transform.py).  Half the flops of K3: a real
 * (M x n_t) x complex (n_t x ncols) product on DMMA.
 * Both A matrices are passed fragment-packed: P[mb][k][g][h] = A[16 mb + g + 8 h][k]
 * (rows zero-padded to a multiple of 16; paired_transform.pack_fragments).
 *   fwd:  G = Y F.  A: device float64 (mrows x nt), mrows a multiple of 16,
 *         rows in blocks of 16 = [Re y_l of 8 sources; Im y_l of the same 8];
 *         rows: int32 (nsrc, 2) = (l, p or -1); scale: c128 (nsrc,) with
 *         y_p = scale * conj(y_l).  Writes out rows l and p.
 *   back: Psi = X W.  A: device float64 (nt x nt), column l = Re x_l, column
 *         p = Im x_l (self-paired: the real part r of x_l = e^{i phi} r).
 *         `in` is CLOBBERED: an in-place pre-pass mixes each pair of rows
 *         [W_l; W_p] <- [[m00, m01], [m10, m11]] [W_l; W_p] (mix_coef c128
 *         (nmix, 4); p = -1: W_l <- m00 W_l).  in and out must not alias.
 * Replaces the two transform_blocks calls of solve on the FD path.
 * ------------------------------------------------------------------------- */
int stfem_transform_pair_fwd(const double* A, int mrows, int nt, const int32_t* rows,
                             const void* scale, int nsrc, const void* in, int64_t ld_in, void* out,
                             int64_t ld_out, int64_t ncols, int batch, int64_t bstride_in,
                             int64_t bstride_out, void* stream);
int stfem_transform_pair_back(const double* A, int nt, const int32_t* mix_rows, const void* mix_coef,
                              int nmix, void* in, int64_t ld_in, void* out, int64_t ld_out,
                              int64_t ncols, int batch, int64_t bstride_in, int64_t bstride_out,
                              void* stream);
/* The same two transforms with the spatial permutation of the shifted solves fused in (FD steps
 * 2 and 4 around stfem_factor_solve with stfem_plan_set_io_permuted(plan, 1)):
 *   _fwd_map : result column j is written at column out_cols[j] of `out` (out_cols = iperm, old -> new);
 *   _back_map: result column j reads operand column in_cols[j] of `in` (in_cols = iperm); with a
 *              map the pre-pass must have run over ALL columns of `in` first (stfem_pair_mix) and
 *              nmix is 0.  A NULL map is the identity.  A mapped side is addressed from its base
 *              pointer with absolute columns, so column blocks of the other side can be processed
 *              one at a time (pipelined host copies). */
int stfem_transform_pair_fwd_map(const double* A, int mrows, int nt, const int32_t* rows, const void* scale,
                                 int nsrc, const void* in, int64_t ld_in, void* out, int64_t ld_out, int64_t ncols,
                                 int batch, int64_t bstride_in, int64_t bstride_out, const int32_t* out_cols,
                                 void* stream);
int stfem_pair_mix(const int32_t* mix_rows, const void* mix_coef, int nmix, void* W, int64_t ld, int64_t ncols,
                   int batch, int64_t bstride, void* stream);
int stfem_transform_pair_back_map(const double* A, int nt, const int32_t* mix_rows, const void* mix_coef, int nmix,
                                  void* in, int64_t ld_in, void* out, int64_t ld_out, int64_t ncols, int batch,
                                  int64_t bstride_in, int64_t bstride_out, const int32_t* in_cols, void* stream);

/* Column block [0, ncols) of `rows` rows between host and device
 * (cudaMemcpy2DAsync; leading dimensions in complex128 elements; kind 0 =
 * host->device, 1 = device->host).  The pipelined host-buffer solve overlaps
 * these copies with the time transforms of neighbouring column blocks. */
int stfem_copy_cols(void* dst, int64_t ld_dst, const void* src, int64_t ld_src, int64_t ncols,
                    int64_t rows, int32_t kind, void* stream);

/* ---------------------------------------------------------------------------
 * Symbolic analysis (host, once per spatial sparsity pattern; SPEC.md:326,
 * :343 "fill-reducing ordering computed once per sparsity pattern and reused
 * across shifts").  Geometric nested dissection on the DoF coordinates,
 * supernodal elimination tree (fronts = separators / leaf regions), extend-add
 * maps.  `rowptr/colind`: symmetric CSR pattern of M_x / A_x (n rows, may
 * include the diagonal).  `coords`: n x 2 (dim 2) or n x 1 (dim 1) float64.
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t n;              /* spatial DoFs */
  int32_t num_fronts;
  int32_t depth;          /* tree depth (root = 0) */
  int32_t max_front;      /* max front order */
  int32_t max_pivots;
  int64_t nnz_factor;     /* nnz(L) incl. diagonal, per shift */
  int64_t factor_elems;   /* complex elements of factor storage per shift (sum n*p) */
  int64_t update_elems;   /* complex elements of the two update pools per shift */
  double flops_factor;    /* algorithmic real flops per shift: sum_j 4*c_j^2 */
  int64_t nnz_pattern;
} stfem_plan_stats;

int stfem_plan_create(int32_t n, const int64_t* rowptr, const int32_t* colind,
                      const double* coords, int32_t dim, int32_t leaf_size,
                      stfem_plan** out);
int stfem_plan_destroy(stfem_plan* plan);
int stfem_plan_stats_get(const stfem_plan* plan, stfem_plan_stats* out);
/* perm[new] = old (host array of n int32) */
int stfem_plan_perm(const stfem_plan* plan, int32_t* perm);
/* per-front table export for tests: rows of (pbeg, p, n, parent, depth) */
int stfem_plan_fronts(const stfem_plan* plan, int32_t* table5);
/* row index lists (new numbering) of every front: pivots then boundary rows;
 * offsets has num_fronts + 1 entries (call with rows = NULL for the sizes) */
int stfem_plan_front_rows(const stfem_plan* plan, int64_t* offsets, int32_t* rows);

/* ---------------------------------------------------------------------------
 * K4+K5  factor + solve, batched over shifts (FD step 3 :377):
 *   (M_x + lam[s] A_x) w[r][s] = g[r][s]      for s < nshift, r < nrhs
 * Complex-symmetric multifrontal LDL^T (transpose, not conjugate), numeric
 * phase on the GPU, forward substitution fused into the factorization,
 * backward substitution level by level.  Mvals/Avals: device CSR values in
 * the plan's pattern (nnz_pattern).  lam: device c128[nshift].  G read, W
 * written (may not alias), both in `layout`.  Factors are transient (streamed
 * in batches of shifts, never kept: SURVEY.md §7 hard part 4).  Stream-ordered:
 * see stfem_plan_check below for how a singular shift is reported.
 * ------------------------------------------------------------------------- */
int stfem_factor_solve(stfem_plan* plan, const double* Mvals, const double* Avals,
                       const void* lam, int32_t nshift, int32_t nrhs,
                       const void* G, void* W, stfem_bv_layout layout,
                       void* stream);
/* stfem_factor_solve only enqueues work on `stream`: it does not wait for the
 * GPU.  A pivot collapse met by its kernels (|pivot| <= pivot_tol
 * * max_j |M_jj + lam A_jj| in the multifrontal fronts, |theta_k + lam| <=
 * pivot_tol * (|theta_k| + |lam|) in a spectral subtree, or a non-finite
 * pivot) is latched in the plan (first offender wins).  stfem_plan_check
 * waits for the work issued so far on `stream`, clears the latch and returns
 * STFEM_ERR_SINGULAR (stfem_last_error names the shift: base + index within
 * the offending call) or STFEM_OK.  stfem_plan_set_shift_base sets the number
 * added to the reported index by the following calls (the Bartels-Stewart
 * sweep reports its sweep index l this way). */
int stfem_plan_check(stfem_plan* plan, void* stream);
int stfem_plan_set_shift_base(stfem_plan* plan, int32_t base);
/* G and W of the following stfem_factor_solve calls are indexed in the plan's own numbering
 * (column new = iperm[old]) instead of the operators': pivot rows are then contiguous, and the
 * permutation is applied by the transforms around the solves (the _map variants above).
 * The setting stays in the plan until it is changed; stfem_fdm_solve, whose transforms carry no
 * maps, clears it.
 * stfem_plan_device_iperm: the device copy of iperm (int32[n]); valid until the next
 * stfem_plan_set_spectral / stfem_plan_set_options. */
int stfem_plan_set_io_permuted(stfem_plan* plan, int32_t on);
int stfem_plan_device_iperm(stfem_plan* plan, const int32_t** iperm);
/* Allocate the numeric workspace for calls of up to `nshift` shifts and `nrhs`
 * right-hand sides now (the batch size is fixed here: equal batches from
 * workspace_fraction of the free memory, or stfem_plan_set_batch), so that
 * later stfem_factor_solve calls never allocate.  Without it the first call
 * (and any call that needs more than is reserved) allocates, which
 * synchronises the device once. */
int stfem_plan_reserve(stfem_plan* plan, int32_t nshift, int32_t nrhs);
/* Concurrency: a plan owns ONE numeric workspace (factor storage, update pools, the latched
 * error flag).  Calls on the same plan must be issued from one host thread at a time and are
 * ordered on the device only through the stream they are given: enqueue them on one stream
 * (or order the streams yourself).  Independent concurrent solves need one plan each; the
 * symbolic analysis is cheap to repeat (C4: 0.2 s). */
/* Tuning knobs of one plan (no environment variables).  get -> modify -> set;
 * set rebuilds the device tables on the next call. */
typedef struct {
  int32_t small_front_n;     /* levels whose largest front has order <= this run on the shared-memory
                                small-front kernel (unit-L LDL^T); 0 = every front on the tile-parallel
                                large-front pipeline.  Default 100 */
  int32_t fused_min_p;       /* levels with >= this many pivots fuse the children's extend-add into the
                                Schur-update tiles (U never assembled).  Default 0: every level */
  int32_t panel_group;       /* trailing pivot-column updates are delayed over this many 32-wide panels.
                                Default 2 */
  int32_t asm_whole_n;       /* fronts of order <= this are assembled by one CTA.  Default INT32_MAX */
  int32_t level_timing;      /* 1: print per-launch CUDA-event times to stderr (diagnostics) */
  int32_t tiles_per_cta;     /* tiles a CTA of the update engine walks (1..16).  Default 16 */
  int32_t ws_stages;         /* ring depth of the update engine (2, 3 or 4).  Default 2 */
  int32_t front_syrk_max_p;  /* Schur updates of levels with at most this many pivots (one panel) run one CTA per
                                instance with L21 resident in shared memory (syrk_front_kernel).  Default 32; 0: never */
  int32_t bwd_dmma_min_p;    /* multi-RHS backward substitution of levels with more than this many pivots runs as
                                GEMMs over the right-hand sides on the FP64 tensor pipe (default 32: every
                                multi-panel level; INT32_MAX: column dot products everywhere) */
  double workspace_fraction; /* share of the free device memory the numeric workspace may take.  Default 0.70 */
  double pivot_tol;          /* relative pivot-collapse threshold (see stfem_plan_check).  Default 1e-10 */
} stfem_plan_options;
int stfem_plan_get_options(const stfem_plan* plan, stfem_plan_options* out);
int stfem_plan_set_options(stfem_plan* plan, const stfem_plan_options* opt);
/* per-level accounting: record CUDA-event times of every level launch on the
 * next calls (on != 0); report ms[2*(depth+1)] (factor launches by depth, then
 * backward launches by depth, summed over shift batches), the algorithmic
 * flops per shift of each depth (flops[depth+1]) and whether the depth runs
 * on the shared-memory small-front kernels (small[depth+1]) */
int stfem_plan_record_levels(stfem_plan* plan, int32_t on);
int stfem_plan_level_report(const stfem_plan* plan, double* ms, double* flops, int32_t* small);
/* per-kernel-family accounting of the last recorded call: ms[f] (CUDA-event
 * time), launches[f], and algorithmic real flops per shift flops[f] for the families
 * 0 spectral (K6), 1 front assembly, 2 diagonal blocks, 3 TRSM, 4 trailing
 * pivot-column update, 5 SYRK (Schur update), 6 backward, 7 small-front factor */
int stfem_plan_kernel_report(const stfem_plan* plan, int32_t nfam, double* ms, double* flops,
                             int64_t* launches);
/* largest nrhs one stfem_factor_solve call accepts for this plan (<= 16) */
int stfem_plan_max_rhs(const stfem_plan* plan, int32_t* max_rhs);
/* shift batches used by the last stfem_factor_solve call */
int stfem_plan_last_batches(const stfem_plan* plan, int32_t* batches);
/* kernel launches of the last stfem_factor_solve call (for launch accounting) */
int stfem_plan_last_launches(const stfem_plan* plan, int64_t* launches);

/* ---------------------------------------------------------------------------
 * GPU uniform refinement of a conforming triangulation (spatial_mesh.refine_uniform,
 * /root/reference/pkg/src/stfem/spatial_mesh.py:121-156, with the boundary flags and
 * interior-DoF numbering of _finish :51-70): midpoints appended in first-encounter
 * order of the edges, four children per triangle, the P2 node table
 * (v0, v1, v2, m01, m12, m20) per parent.  All arrays are device memory;
 * outputs sized for the worst case nv + 3 ne vertices: verts_out double[2 (nv + 3 ne)],
 * elems_out int64[12 ne], p2_out int64[6 ne], boundary_out uint8[nv + 3 ne],
 * interior_dof_out int64[nv + 3 ne].  *nv_out / *ndof_out (host) receive the
 * refined vertex and interior-DoF counts.  Waits for the stream.
 * ------------------------------------------------------------------------- */
int stfem_mesh_refine2d(int32_t nv, const double* verts, int32_t ne, const int64_t* elems,
                        double* verts_out, int64_t* elems_out, int64_t* p2_out, uint8_t* boundary_out,
                        int64_t* interior_dof_out, int32_t* nv_out, int32_t* ndof_out, void* stream);

/* ---------------------------------------------------------------------------
 * K6  spectral subtree elimination (optional; replaces the bottom of the
 * elimination tree for every shift at once, csrc/spectral.cuh).  Call once
 * after assembly with host data computed from M_x / A_x (paper_2504_07269_b200
 * /spectral.py): for subtree t rooted at front root_front[t] with interior
 * pivots [first[t], first[t] + m_t) and boundary size g_t = the root's
 * boundary rows, offsets[4t..4t+3] give the double offsets of
 *   V (m x m, column-major; V^T A_II V = I, V^T M_II V = diag(theta)),
 *   theta (m), R then Q (g x m each, column-major), C0 then C1 (g x g each).
 * Fronts inside the subtrees leave the multifrontal levels; the roots' update
 * blocks, forward RHS and backward solves run as DMMA GEMMs over shifts.
 * nroots = 0 restores the plain multifrontal plan.  The data must come from
 * the same operators later passed to stfem_factor_solve.
 * ------------------------------------------------------------------------- */
int stfem_plan_set_spectral(stfem_plan* plan, int32_t nroots, const int32_t* root_front,
                            const int32_t* first, const int64_t* offsets, const double* V,
                            int64_t nV, const double* theta, int64_t ntheta, const double* RQ,
                            int64_t nRQ, const double* C01, int64_t nC01);
/* subtree count, DMMA flops per shift of the update blocks (4 E m summed),
 * flops per shift per RHS of the RHS GEMMs, and device bytes of the data */
int stfem_plan_spectral_stats(const stfem_plan* plan, int32_t* nroots, double* flops_u,
                              double* flops_rhs, int64_t* bytes);

/* ---------------------------------------------------------------------------
 * K1/K2/K7  assembly and the matrix-free residual
 * (apply_global) on the GPU.
 * degree 1: elems ne x 3 (P1 triangles); degree 2: ne x 6 (v0 v1 v2 m01 m12 m20).
 * interior_dof: nv int64 (-1 on the boundary).
 * ------------------------------------------------------------------------- */
int stfem_asm_create(int32_t degree, int32_t nv, const double* verts, int32_t ne,
                     const int64_t* elems, const int64_t* interior_dof,
                     stfem_asm** out);
int stfem_asm_destroy(stfem_asm* a);
/* host export of the CSR pattern: nnz via *nnz (call with NULL arrays first) */
int stfem_asm_pattern(const stfem_asm* a, int32_t* n, int64_t* nnz,
                      int64_t* rowptr, int32_t* colind);
/* M_x, A_x values into the pattern (device double[nnz] each), coloured scatter */
int stfem_asm_spatial(stfem_asm* a, double* Mvals, double* Avals, void* stream);
/* space-time load vector F (n_t x n_x c128 at F + l*ld) for a built-in source:
 * kind 1 = s(x)(i pi cos pi t + 2 pi^2 sin pi t)  (C1/C2 manufactured)
 * kind 2 = s(x) e^{-it}(i + t + 2 pi^2 t)         (C3 manufactured)
 * kind 3 = paper's e^{it} sin sin sin(t x y)
 * P1 in space and time; breakpoints: host double[N+1]. */
int stfem_asm_rhs(stfem_asm* a, int32_t kind, const double* breakpoints, int32_t N,
                  void* F, int64_t ld, void* stream);
/* y = alpha * A v (+ beta y): CSR SpMV on complex vectors, batched over
 * `nvec` vectors (row stride ld), real matrix values `vals` (device) */
int stfem_csr_spmv_c(const stfem_asm* a, const double* vals, const void* v,
                     int64_t ldv, void* y, int64_t ldy, int32_t nvec,
                     double alpha_re, double alpha_im, double beta, void* stream);
/* apply_global: out = (i B_t (x) M_x + M_t (x) A_x) v for a
 * banded M_t / B_t (P1 time: bw = 1; P2 time: bw = 2) given as device arrays
 * nt x (2 bw + 1), band[l][k - l + bw].  v/out: (nt, n_x) c128 row-major;
 * work: device scratch of 2 * nt * n_x c128. */
/* K8 spacetime_errors: (||psi - psi_h||_{L2(Q)},
 * |psi - psi_h|_{H1(Q)}) into host out2[2] for P1 x P1 coefficients
 * (N x n_x c128 at coeffs + l*ld, device) against a built-in exact solution
 * (kind as in stfem_asm_rhs), psi_h = sum coeff phi_j phi_l + psi0 (psi0:
 * device nv c128 nodal values or NULL).  7-point x 5-point quadrature per
 * prism, deterministic reduction. */
int stfem_spacetime_errors(const stfem_asm* a, int32_t kind, const double* breakpoints, int32_t N,
                           const void* coeffs, int64_t ld, const void* psi0, double* out2, void* stream);
/* Bartels-Stewart sweep update (Eq. 7, incremental form :418;
 * replaces the per-step "g_l - sum_{k>l} S[l,k] A_x w_k" of
 * kronecker_solver.solve(variant=BartelsStewart)):
 *   G[r][l'][j] -= scol[l'] * (A_x w_r)[j]   for l' < l, j < n_x, r < nrhs.
 * w: nrhs vectors of n_x c128 (stride ldw); scol: device S[0:l, l] (c128);
 * G: device c128 with strides g_rhs_stride (between RHS) and g_shift_stride
 * (between temporal rows). */
int stfem_bs_update(const stfem_asm* a, const double* Avals, const void* w, int64_t ldw, int32_t nrhs,
                    const void* scol, int32_t l, void* G, int64_t g_rhs_stride, int64_t g_shift_stride,
                    void* stream);
int stfem_apply_global(const stfem_asm* a, const double* Mvals, const double* Avals,
                       const double* Mt_band, const double* Bt_band, int32_t bw, int32_t nt,
                       const void* v, void* out, void* work, void* stream);

/* ---------------------------------------------------------------------------
 * The whole FD solve behind one call (kronecker_solver.solve, SPEC.md:374-382,
 * steps 2-4; step 1 -- the temporal eigendecomposition -- is host work whose
 * result arrives in stfem_fd_factors), single-GPU or sharded over NCCL
 * (SURVEY.md §8b "fdm_solve(plan, comm, ...)" and "comm_init(unique_id[128],
 * nranks, rank)", §8e partitioning).
 *
 * stfem_comm: one NCCL communicator per process / GPU.  Rank 0 calls
 * stfem_comm_unique_id and hands the 128 bytes to every rank through the
 * launcher's own channel (the torch.distributed store under torchrun); every
 * rank then calls stfem_comm_init with the CUDA device it will use current.
 * NCCL is bound at run time (dlopen libnccl.so.2); STFEM_ERR_NCCL if absent.
 * stfem_comm_all_to_all: block q (count c128) of send -> rank q.
 * ------------------------------------------------------------------------- */
typedef struct stfem_comm stfem_comm;
int stfem_comm_unique_id(uint8_t unique_id[128]);
int stfem_comm_init(const uint8_t unique_id[128], int32_t nranks, int32_t rank, stfem_comm** out);
int stfem_comm_destroy(stfem_comm* comm);
int stfem_comm_info(const stfem_comm* comm, int32_t* nranks, int32_t* rank, int32_t* nccl_version);
int stfem_comm_all_to_all(stfem_comm* comm, const void* send, void* recv, int64_t count, void* stream);

/* Temporal factors of the FD solve in device memory (TemporalFactors).
 * Either the K3p tables (stfem_transform_pair_fwd / _back arguments, built by
 * paired_transform.py) or the dense X, Y of K3; lam always. */
typedef struct {
  int32_t nt;
  const void* lam;          /* c128[nt], ordered as the rows of Y / columns of X */
  const void* X;            /* c128 nt x nt row-major, or NULL with the paired tables */
  const void* Y;
  const double* A_fwd;      /* K3p forward: see stfem_transform_pair_fwd */
  int32_t mrows_fwd;
  const int32_t* rows_fwd;
  const void* scale_fwd;
  int32_t nsrc;
  const double* A_back;     /* K3p back: see stfem_transform_pair_back */
  const int32_t* mix_rows;
  const void* mix_coef;
  int32_t nmix;
} stfem_fd_factors;

/* Psi = A^{-1} F, A = i B_t (x) M_x + M_t (x) A_x.
 * comm == NULL: F, Psi, work are (nrhs, n_t, n_x) c128 BlockVectors.
 * comm with P ranks: they are this rank's (n_t, nrhs, c) shard, c = ceil(n_x / P)
 *   spatial columns [rank c, (rank + 1) c) (zero padded), n_t divisible by P; the
 *   rank factors shifts [rank n_t / P, (rank + 1) n_t / P) of tf->lam.
 * F is read only; Psi and work are overwritten (work is scratch); the three must
 * be distinct.  Stream-ordered; pivot collapse via stfem_plan_check(plan). */
int stfem_fdm_solve(stfem_plan* plan, stfem_comm* comm, const double* Mvals, const double* Avals,
                    const stfem_fd_factors* tf, const void* F, void* Psi, void* work, int32_t nrhs,
                    void* stream);

#ifdef __cplusplus
}
#endif
#endif /* STFEM_B200_H */
