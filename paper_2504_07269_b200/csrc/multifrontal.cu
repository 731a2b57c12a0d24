// K4/K5 — batched multifrontal complex-symmetric LDL^T factor + solve of the
// n_t shifted spatial systems (M_x + lam_l A_x) w_l = g_l (SPEC.md:323-340,
// FD step 3 SPEC.md:377; factor/solve contract SPEC.md:319).
//
// One symbolic tree (plan) is shared by every shift, so a depth level of the
// tree times a batch of shifts is a set of independent, identically-shaped
// dense front problems.  One CTA owns one (front, shift) instance per level.
// Fronts of order <= SMALL_N take the shared-memory path of
// multifrontal_small.cuh (unit-L LDL^T).  Larger fronts (this file) live in
// HBM/L2 and use the complex-symmetric Cholesky form K = C C^T, c_jj = d_j^{1/2}:
//   1. assemble by gathering: every front entry is written once as the sum of
//      at most two children's update entries (inverse relpos maps in shared
//      memory), then the original entries M + lam*A are added (deterministic,
//      no atomics, no zero fill);
//   2. factor the p pivot columns, right-looking in panels of NB=32: diagonal
//      block by one warp in shared memory, row-parallel TRSM (8-column register
//      blocks) for the rows below with the forward substitution of the RHS
//      fused in, trailing pivot-column update on the FP64 tensor pipe (DMMA);
//   3. Schur update U = F22 - L21 L21^T (lower tiles, K = p, DMMA).
// Backward substitution walks the levels root-first; each instance gathers
// x_B of its boundary rows (already final), applies L21^T and the transposed
// triangle, and writes x both to the permuted work vector and (un-permuted)
// to the caller's BlockVector.  Transpose, not conjugate transpose: K is
// complex symmetric.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <array>
#include <string>

#include "plan.h"

namespace stfem {
namespace {

int upload(Plan& P);
int ensure_workspace(Plan& P, int batch, int nrhs);
int auto_batch(Plan& P, int nshift, int nrhs);
int ensure_workspace_backoff(Plan& P, int* batch, int nrhs);

constexpr int NT = 256;
constexpr int NB = 32;            // panel width
constexpr int LDD = NB + 1;       // diagonal block column stride
constexpr int MAXR = 16;          // max RHS per call (bv chunks of 16 in the host loop)

constexpr int BWD_XS_MAX = 192 * 1024;   // backward_level_kernel: staged x (n x nrhs) per front
constexpr int BWD_SPLIT_N = 256;         // backward: fronts above this order launch separately

// kernel families of the per-family accounting (stfem_plan_kernel_report)
enum { FAM_SPECTRAL = 0, FAM_ASM, FAM_DIAG, FAM_TRSM, FAM_PANEL, FAM_SYRK, FAM_BACKWARD, FAM_SMALL, NFAM };

struct LevelArgs {
  const FrontDev* fronts;
  const int32_t* list;
  int32_t nlist, nbatch;
  const int32_t *child_ids, *relpos, *bidx, *ent_src, *ent_dst, *perm, *inv;
  const double *Mv, *Av;
  const cplx* lam;
  cplx* factor;
  int64_t fstride;
  cplx* ucur;
  int64_t ucur_stride;
  const cplx* uchild;
  int64_t uchild_stride;
  cplx* rcur;
  int64_t rcur_stride;  // per shift per rhs
  const cplx* rchild;
  int64_t rchild_stride;
  cplx* Z;
  int32_t nx, nrhs;
  const cplx* G;
  cplx* W;
  stfem_bv_layout lay;
  int32_t shift0;
  int* err;
  int err_base;               // added to the shift index latched in err (stfem_plan_set_shift_base)
  const double* scale2;       // per local shift: (pivot_tol * max_j |M_jj + lam A_jj|)^2, the pivot-collapse bound
  const int32_t* ent_colptr;  // per front (p + 1): first sorted original entry of each pivot column
  int unit_diag;              // backward: 1 = unit-L LDL^T fronts, 0 = C C^T fronts
  int asm_pivots_only;        // asm_front_kernel: pivot columns only (U assembled by syrk_gather_kernel)
  int asm_cpc;                // asm_front_kernel: columns per CTA (a multiple of ASM_COLS)
};

__device__ __forceinline__ int64_t bv_off(const stfem_bv_layout& L, int r, int64_t shift, int64_t j) {
  // un-chunked BlockVectors (chunk_cols >= n_x: every single-GPU call) skip the 64-bit division
  int64_t q = 0;
  if (j >= L.chunk_cols) {
    q = j / L.chunk_cols;
    j -= q * L.chunk_cols;
  }
  return r * L.rhs_stride + shift * L.shift_stride + q * L.chunk_stride + j;
}

#include "multifrontal_large.cuh"

// Geometry of the 32 x 32-tile DMMA update engine: shared K chunks [16][32 + 2] complex (the
// 2-element pad keeps the fragment loads of the 32 lanes on 8 distinct 16-byte bank groups)
constexpr int S32_LD = 32 + 2, S32_STAGE = 16 * S32_LD;

constexpr int ST_MAXT = 16;                 // tiles per CTA (upper bound)
constexpr int ST_CS = 32 * S32_LD;          // one staged C tile: Cs[col * S32_LD + row] (complex)

struct __align__(16) StreamTile {
  const cplx* A;        // multiplier rows: element (r, kk) at A[r + kk * lda]
  cplx* C;              // C[row + col * ldC]
  const cplx* Uc[2];    // GATHER: the children's update blocks
  int lda, ldC, K, M, N, i0, c0;
  int bc[2];            // GATHER: children's boundary orders
  int inv_off[2];       // GATHER: a.inv offset of boundary row 0 for child s (-1: no such child)
  int pad;              // rows of C that may be stored (>= M: the update block's leading dimension; panel updates: M)
};

// ---------------------------------------------------------------------------
// Warp-specialised, TMA-fed update engine: C = Cinit - A A^T on lower 32 x 32
// tiles (Schur updates; DMMA).  One producer warp feeds a 4-stage ring of
// 16-deep K chunks with 1-D bulk copies (cp.async.bulk, the TMA engine: one
// 512-byte column segment per lane, completion counted in bytes on the
// stage's "full" mbarrier); four consumer warps (2 x 2 of 16 x 16) do nothing
// but wait on "full", LDS, DMMA and release the stage on its "empty" mbarrier
// -- no address arithmetic, no cp.async issue, no CTA-wide barrier in the
// DMMA warps, and every consumer warp runs on its own (a delayed warp stalls
// nobody else).  The ring runs across tile boundaries (a CTA walks up to 16
// tiles), so pipeline fill / drain and descriptor latency are paid once per
// CTA.  The tile's starting values -- the assembled block (bulk copies), or
// with GATHER the children's extend-add (16-byte cp.async through the inverse
// maps, completion forwarded to the "cfull" mbarrier) -- are staged in shared
// memory by the producer during the tile's K loop and added in the epilogue.
// A DMMA needs no second warp to hide its latency (measured: one warp per SM
// sub-partition with a single dependent accumulator chain reaches 36.8 of
// 37.1 TFLOP/s, tools/probe_dmma.py), so 3 CTAs x 4 consumer warps per SM
// keep the pipe busy through the other CTAs' epilogues.
// The complex product is formed from three real DMMAs instead of four ("3M":
// P1 = ar br, P2 = ai bi, P3 = (ar + ai)(br + bi); re = P1 - P2, im = P3 - P1 -
// P2), accumulated separately over K and combined in the epilogue: 6 DMMAs and 4
// DADDs per k step of a 16 x 16 block instead of 8 DMMAs.  The third
// accumulator set needs 104 registers in the DMMA warps; setmaxnreg moves them
// over from the copy warps (56), so the CTA keeps its 80-register launch
// footprint and 3 CTAs per SM.  Measured on C4: Schur updates 271 -> 246 ms,
// trailing updates 66 -> 58 ms per step (the DMMA-bound levels gain 12%, the
// short-K levels 2-5%); without the re-balancing (2 CTAs per SM) only 8% / -10%.
// ---------------------------------------------------------------------------
// warps 0-3: DMMA consumers (2 x 2 of 16 x 16); warp 4: bulk copies of the A rows of every chunk;
// warp 5: the B rows; warps 6, 7: the tile's starting values (GATHER: one warp per child -- a
// single staging warp was issue bound at the short-K levels, ncu had the consumers waiting on
// "cfull" in 22% of all samples: C4 Schur updates 278 -> 271 ms with two; otherwise warp 6 alone).
// (Measured on C4, 384 shifts, depths 1-6, ms per batch: one bulk-copy warp for A and B 91.0 --
// its 32 UBLKCPs per chunk issue one by one, their operands being uniform registers -- two warps
// 79.4, four 81.3; a cp.async producer 86.9; staging the starting values from the A warp instead
// of a third warp cost another 8 ms.)
constexpr int WS_THREADS = 256;
template <bool GATHER, int WS_STAGES>
constexpr int ws_smem_bytes() {
  return WS_STAGES * 2 * S32_STAGE * 16 + (GATHER ? 2 : 1) * ST_CS * 16 + ST_MAXT * (int)sizeof(StreamTile) +
         (2 * WS_STAGES + 2) * 8;
}

// resident CTAs per SM (shared memory: 71 KB with a 2-stage ring); the 2-CTA variants run at 128 registers
template <bool GATHER, int WS_STAGES>
constexpr int ws_ctas_per_sm() { return WS_STAGES <= (GATHER ? 2 : 3) ? 3 : 2; }

template <bool GATHER, int WS_STAGES>
__device__ __forceinline__ void ws_tiles(const StreamTile* __restrict__ desc, int nt, cplx* As, cplx* Bs, cplx* Cs,
                                         uint64_t* full, uint64_t* empty, uint64_t* cfull, uint64_t* cempty,
                                         const int32_t* __restrict__ inv) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // register re-balancing between the two warpgroups (80 per thread at launch, 3 CTAs per SM):
  // the copy warps give up registers, the DMMA warps take them for the third accumulator set
  // (ptxas allocates each role's code against its own limit)
  if constexpr (ws_ctas_per_sm<GATHER, WS_STAGES>() == 3) {
    if (warp >= 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n");
    else asm volatile("setmaxnreg.inc.sync.aligned.u32 104;\n");
  }
  if (warp >= 6) {
    // ---------------- starting values: one staging tile per child (GATHER) or one in all ----------------
    const int s = warp - 6;   // GATHER: this warp's child
    if (!GATHER && s == 1) return;
    uint32_t cphase = 0;
    if constexpr (GATHER) {
      // the child's extend-add through the inverse maps: lane = tile row; the column map is
      // loaded once (lane = column) and broadcast.  The maps of the next tile are fetched before
      // this tile's copies are issued, so their latency never sits between two tiles.
      int jn = 0;
      while (jn < nt && desc[jn].K <= 0) ++jn;
      int kr_n = -1, kc_n = -1;
      auto fetch = [&](int j) {
        const StreamTile& D = desc[j];
        const int off = D.inv_off[s];
        kr_n = (off >= 0 && D.i0 + lane < D.M) ? inv[off + D.i0 + lane] : -1;
        kc_n = (off >= 0 && D.c0 + lane < D.N) ? inv[off + D.c0 + lane] : -1;
      };
      if (jn < nt) fetch(jn);
      while (jn < nt) {
        const int j = jn;
        const int kr = kr_n, kcl = kc_n;
        do ++jn; while (jn < nt && desc[jn].K <= 0);
        if (jn < nt) fetch(jn);
        const StreamTile& D = desc[j];
        mbar_wait(cempty, cphase ^ 1);   // the consumers have read the previous tile's values
        cphase ^= 1;
        if (D.inv_off[s] >= 0) {
          const cplx* Uc = D.Uc[s];
          const int bc = D.bc[s], i0 = D.i0, c0 = D.c0;
          cplx* dst = Cs + s * ST_CS + lane;
#pragma unroll 8
          for (int cc = 0; cc < 32; ++cc) {
            const int kc = __shfl_sync(0xffffffffu, kcl, cc);
            const bool ok = kr >= 0 && kc >= 0 && i0 + lane >= c0 + cc;
            cp_async16(dst + cc * S32_LD, ok ? Uc + (int64_t)kc * bc + kr : Uc, ok);
          }
        }
        cp_async_mbar_arrive(cfull);   // 64 expected arrivals: one per lane of both warps, when its copies have landed
      }
    } else {
      for (int j = 0; j < nt; ++j) {
        const StreamTile& D = desc[j];
        if (D.K <= 0) continue;
        const int M = D.M, N = D.N, i0 = D.i0, c0 = D.c0;
        mbar_wait(cempty, cphase ^ 1);
        cphase ^= 1;
        const int ncol = min(32, N - c0), rows = min(32, M - i0);
        if (lane == 0) mbar_arrive_expect_tx(cfull, (uint32_t)ncol * (uint32_t)rows * 16u);
        __syncwarp();
        if (lane < ncol)
          bulk_g2s(Cs + lane * S32_LD, D.C + i0 + (int64_t)(c0 + lane) * D.ldC, (uint32_t)rows * 16u, cfull);
      }
    }
    return;
  }
  if (warp >= 4) {
    // ---------------- K chunks: warp 4 copies the A rows, warp 5 the B rows (lane = column) ----------------
    const int isB = warp - 4;
    cplx* ring = isB ? Bs : As;
    int stage = 0;
    uint32_t phase = 0;
    for (int j = 0; j < nt; ++j) {
      const StreamTile& D = desc[j];
      const int K = D.K, nk = (K + 15) >> 4;
      if (nk == 0) continue;
      const int lda = D.lda;
      const int r0 = isB ? D.c0 : D.i0, rows = min(32, (isB ? D.N : D.M) - r0);
      const cplx* src0 = D.A + r0 + (int64_t)lane * lda;
      const uint32_t myb = (uint32_t)rows * 16u;
      for (int c = 0; c < nk; ++c) {
        mbar_wait(&empty[stage], phase ^ 1);
        const int kv = min(16, K - c * 16);   // columns >= kv are not copied: the consumers mask them
        if (lane == 0) mbar_arrive_expect_tx(&full[stage], (uint32_t)kv * myb);
        __syncwarp();
        if (lane < kv) bulk_g2s(ring + stage * S32_STAGE + lane * S32_LD, src0 + (int64_t)(c * 16) * lda, myb, &full[stage]);
        if (++stage == WS_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }
  // ---------------- consumers ----------------
  const int g = lane >> 2, t = lane & 3, wm = warp & 1, wn = warp >> 1;
  int stage = 0;
  uint32_t phase = 0, cphase = 0;
  for (int j = 0; j < nt; ++j) {
    const StreamTile& D = desc[j];
    const int K = D.K, nk = (K + 15) >> 4;
    if (nk == 0) continue;
    const int M = D.M, N = D.N, i0 = D.i0, c0 = D.c0;
    // warps whose 16 x 16 block lies strictly above the diagonal (diagonal tiles) or outside
    // the block skip their DMMAs (warp-uniform; their outputs are never stored)
    const bool wact = (i0 + wm * 16 + 15 >= c0 + wn * 16) && (i0 + wm * 16 < M) && (c0 + wn * 16 < N);
    double cre[2][4], cim[2][4];
    double c3[2][4];
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        cre[ni][e] = cim[ni][e] = 0.0;
        c3[ni][e] = 0.0;
      }
    for (int c = 0; c < nk; ++c) {
      mbar_wait(&full[stage], phase);
      if (wact) {
        const cplx* as = As + stage * S32_STAGE + t * S32_LD + wm * 16 + g;
        const cplx* bs = Bs + stage * S32_STAGE + t * S32_LD + wn * 16 + g;
        const int kv = K - c * 16;   // valid k columns of this chunk (>= 16: all)
        if (kv >= 16) {
#pragma unroll
          for (int kk = 0; kk < 16; kk += 4) {
            const cplx a0 = as[kk * S32_LD], a1 = as[kk * S32_LD + 8];
            const cplx b0 = bs[kk * S32_LD], b1 = bs[kk * S32_LD + 8];
            // 3M complex product: P1 += ar br, P2 += ai bi, P3 += (ar + ai)(br + bi)
            {
              const double s0 = a0.re + a0.im, s1 = a1.re + a1.im;
              dmma_16x8x4(cre[0], a0.re, a1.re, b0.re);
              dmma_16x8x4(cim[0], a0.im, a1.im, b0.im);
              dmma_16x8x4(c3[0], s0, s1, b0.re + b0.im);
              dmma_16x8x4(cre[1], a0.re, a1.re, b1.re);
              dmma_16x8x4(cim[1], a0.im, a1.im, b1.im);
              dmma_16x8x4(c3[1], s0, s1, b1.re + b1.im);
            }
          }
        } else {
          // K tail: columns >= kv of the stage were not copied (stale data): masked out
          for (int kk = 0; kk < kv; kk += 4) {
            const bool ok = kk + t < kv;
            const cplx z = cmk(0.0, 0.0);
            const cplx a0 = ok ? as[kk * S32_LD] : z, a1 = ok ? as[kk * S32_LD + 8] : z;
            const cplx b0 = ok ? bs[kk * S32_LD] : z, b1 = ok ? bs[kk * S32_LD + 8] : z;
            // 3M complex product: P1 += ar br, P2 += ai bi, P3 += (ar + ai)(br + bi)
            {
              const double s0 = a0.re + a0.im, s1 = a1.re + a1.im;
              dmma_16x8x4(cre[0], a0.re, a1.re, b0.re);
              dmma_16x8x4(cim[0], a0.im, a1.im, b0.im);
              dmma_16x8x4(c3[0], s0, s1, b0.re + b0.im);
              dmma_16x8x4(cre[1], a0.re, a1.re, b1.re);
              dmma_16x8x4(cim[1], a0.im, a1.im, b1.im);
              dmma_16x8x4(c3[1], s0, s1, b1.re + b1.im);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == WS_STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
    // epilogue: C = Cinit + acc.  The DMMA accumulator layout would store 128-byte pieces at
    // 16-byte alignment (8 rows x 4 columns per instruction): measured 3.7 TB/s against 6 TB/s for
    // aligned 256-byte pieces (tools/probe_store.py).  So the warp writes its finished 16 x 16
    // block over its own corner of the first staging tile and stores it from there, two columns
    // of 16 rows per instruction.  Diagonal blocks are stored whole (their upper entries are the
    // mirror values and are never read); rows up to the block's leading dimension are written,
    // so that every touched line of an update block is written completely.
    mbar_wait(cfull, cphase);
    cphase ^= 1;
    cplx* C = D.C;
    const int ldC = D.ldC, rowlim = D.pad;
    const bool two = GATHER && D.inv_off[1] >= 0, one = !GATHER || D.inv_off[0] >= 0;
    if (wact) {
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int r = wm * 16 + g + 8 * h, cc = wn * 16 + ni * 8 + 2 * t + v;
            cplx o = cmk(0.0, 0.0);
            if (one) o = cadd(o, Cs[cc * S32_LD + r]);              // same sum order as asm_front_kernel
            if (two) o = cadd(o, Cs[ST_CS + cc * S32_LD + r]);
            const double p1 = cre[ni][2 * h + v], p2 = cim[ni][2 * h + v], p3 = c3[ni][2 * h + v];
            Cs[cc * S32_LD + r] = cmk(o.re - (p1 - p2), o.im - (p3 - p1 - p2));
          }
      __syncwarp();
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int r = wm * 16 + (lane & 15), cc = wn * 16 + 2 * it + (lane >> 4);
        const int row = i0 + r, col = c0 + cc;
        if (row < rowlim && col < N) stc(C + row + (int64_t)col * ldC, Cs[cc * S32_LD + r]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(cempty);
  }
}

template <bool GATHER, int WS_STAGES>
__device__ __forceinline__ void ws_init_barriers(uint64_t* full, uint64_t* empty, uint64_t* cfull, uint64_t* cempty) {
  for (int s = 0; s < WS_STAGES; ++s) {
    mbar_init(&full[s], 2);     // the A and the B warp's arrive.expect_tx (+ their copies' bytes)
    mbar_init(&empty[s], 4);    // one arrival per consumer warp
  }
  mbar_init(cfull, GATHER ? 64 : 1);
  mbar_init(cempty, 4);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

// Schur update of a level through the warp-specialised engine: tile q of the launch is
// (shift q / n32, tile q % n32 of the level's tile list); CTA x takes tiles [x T, (x + 1) T).
template <bool GATHER, int WS_STAGES>
__global__ void __launch_bounds__(WS_THREADS, ws_ctas_per_sm<GATHER, WS_STAGES>())
    syrk_ws_kernel(LevelArgs a, const int4* __restrict__ tiles, int n32, long long total, int T) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* As = reinterpret_cast<cplx*>(smem_raw);
  cplx* Bs = As + WS_STAGES * S32_STAGE;
  cplx* Cs = Bs + WS_STAGES * S32_STAGE;
  StreamTile* desc = reinterpret_cast<StreamTile*>(Cs + (GATHER ? 2 : 1) * ST_CS);
  uint64_t* bars = reinterpret_cast<uint64_t*>(desc + ST_MAXT);
  uint64_t *full = bars, *empty = bars + WS_STAGES, *cfull = bars + 2 * WS_STAGES, *cempty = cfull + 1;
  if (threadIdx.x == 0) ws_init_barriers<GATHER, WS_STAGES>(full, empty, cfull, cempty);
  const long long q0 = (long long)blockIdx.x * T;
  const int nt = (int)min((long long)T, total - q0);
  for (int j = threadIdx.x; j < nt; j += WS_THREADS) {
    const long long q = q0 + j;
    const int k = (int)(q / n32);
    const int4 tl = tiles[q - (long long)k * n32];
    const FrontDev F = a.fronts[tl.x];
    const int n = F.n, p = F.p, b = n - p;
    StreamTile D;
    D.A = a.factor + (int64_t)k * a.fstride + F.fofs + p;   // L21: row r, column kk at A[r + kk n]
    D.C = a.ucur + (int64_t)k * a.ucur_stride + F.uofs;
    D.lda = n;
    D.ldC = ldu(b);
    D.K = p;
    D.M = D.N = b;
    D.i0 = tl.y * 32;
    D.c0 = tl.z * 32;
    D.pad = ldu(b);   // rows stored: up to the leading dimension
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      D.Uc[s] = nullptr;
      D.bc[s] = 0;
      D.inv_off[s] = -1;
      if (GATHER && s < F.nchild) {
        const FrontDev Cf = a.fronts[a.child_ids[F.child_beg + s]];
        D.bc[s] = ldu(Cf.n - Cf.p);   // the child's update-block leading dimension
        D.Uc[s] = a.uchild + (int64_t)k * a.uchild_stride + Cf.uofs;
        D.inv_off[s] = F.inv_beg + s * n + p;
      }
    }
    desc[j] = D;
  }
  __syncthreads();
  ws_tiles<GATHER, WS_STAGES>(desc, nt, As, Bs, Cs, full, empty, cfull, cempty, a.inv);
}

// ---------------------------------------------------------------------------
// Schur update of the short-K levels (one pivot panel, K = p <= 32), one CTA per
// (front, shift) instance with the whole L21 (b x K) resident in shared memory.
// On these levels a 32 x 32 tile of the update engine above is one or two K chunks:
// its ring and staging handshakes (~1800 clocks per tile) and the serial gather of the
// starting values cost more than the DMMAs (C4 depths 7-9: DMMA pipe 31-50% active, DRAM
// 30-39%).  Here L21 arrives once per instance by K bulk copies (one mbarrier wait), after
// which every warp is on its own: it takes 16 x 16 blocks of the lower triangle from a shared
// counter, loads the children's entries of its block straight into registers through
// inverse maps staged in shared memory, runs the K loop from shared memory (3M product,
// as in the engine -- the results are bit-identical to the engine's) and stores the block.
// No per-tile protocol; the other warps of the SM cover a warp's load latency.
// ---------------------------------------------------------------------------
constexpr int SF_KMAX = 32;
__host__ __device__ constexpr int sf_ld(int b) { return ((b + 15) & ~15) + 2; }   // row pitch: = 2 mod 8, covers whole blocks
constexpr int SF_TS = 16 * 18;   // per-warp staging of a finished 16 x 16 block (pitch 18: = 2 mod 8)
__host__ __device__ constexpr int sf_smem_bytes(int bmax, int pmax, int nwarp) {
  return (pmax * sf_ld(bmax) + nwarp * SF_TS) * 16 + 2 * ((bmax + 15) & ~15) * 2 + 32;
}

template <int NTH>
__global__ void __launch_bounds__(NTH, NTH >= 256 ? 2 : 4) syrk_front_kernel(LevelArgs a) {
  extern __shared__ __align__(16) unsigned char sf_smem[];
  const int tid = threadIdx.x, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int inst = blockIdx.x;
  const int k = inst % a.nbatch;
  const FrontDev F = a.fronts[a.list[inst / a.nbatch]];
  const int n = F.n, K = F.p, b = n - K;
  if (b <= 0) return;
  const int LD = sf_ld(b), bp = (b + 15) & ~15;
  cplx* Ls = reinterpret_cast<cplx*>(sf_smem);                           // Ls[kk * LD + row] = L21[row][kk]
  cplx* Ts = Ls + (int64_t)K * LD + (tid >> 5) * SF_TS;                  // this warp's output staging
  int16_t* maps = reinterpret_cast<int16_t*>(Ls + (int64_t)K * LD + (NTH / 32) * SF_TS);   // maps[s * bp + row]
  uint64_t* bar = reinterpret_cast<uint64_t*>(maps + 2 * bp + (((2 * bp) & 3) ? 4 - ((2 * bp) & 3) : 0));
  int* next = reinterpret_cast<int*>(bar + 1);
  const cplx* L21 = a.factor + (int64_t)k * a.fstride + F.fofs + K;      // row r, column kk at L21[r + kk n]
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    *next = 0;
  }
  __syncthreads();
  if (tid < 32) {
    if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)K * (uint32_t)b * 16u);
    __syncwarp();
    if (lane < K) bulk_g2s(Ls + lane * LD, L21 + (int64_t)lane * n, (uint32_t)b * 16u, bar);
  }
  const cplx* Uc[2] = {nullptr, nullptr};
  int bc[2] = {0, 0};
#pragma unroll
  for (int s = 0; s < 2; ++s)
    if (s < F.nchild) {
      const FrontDev Cf = a.fronts[a.child_ids[F.child_beg + s]];
      bc[s] = ldu(Cf.n - Cf.p);   // leading dimension
      Uc[s] = a.uchild + (int64_t)k * a.uchild_stride + Cf.uofs;
    }
  for (int q = tid; q < 2 * bp; q += NTH) {
    const int s = q / bp, r = q - s * bp;
    maps[q] = (s < F.nchild && r < b) ? (int16_t)a.inv[F.inv_beg + s * n + K + r] : (int16_t)-1;
  }
  __syncthreads();
  mbar_wait(bar, 0);
  cplx* U = a.ucur + (int64_t)k * a.ucur_stride + F.uofs;
  const int nblk = bp >> 4, nwork = nblk * (nblk + 1) / 2;
  const cplx zero = cmk(0.0, 0.0);
  for (;;) {
    int wb = 0;
    if (lane == 0) wb = atomicAdd(next, 1);
    wb = __shfl_sync(0xffffffffu, wb, 0);
    if (wb >= nwork) break;
    int bi = (int)((sqrtf(8.0f * (float)wb + 1.0f) - 1.0f) * 0.5f);
    while (bi * (bi + 1) / 2 > wb) --bi;
    while ((bi + 1) * (bi + 2) / 2 <= wb) ++bi;
    const int bj = wb - bi * (bi + 1) / 2;
    const int rb = bi * 16, cb = bj * 16;
    double p1[2][4] = {}, p2[2][4] = {}, p3[2][4] = {};
    const cplx* as = Ls + t * LD + rb + g;
    const cplx* bs = Ls + t * LD + cb + g;
    for (int kk = 0; kk < K; kk += 4) {
      const bool ok = kk + t < K;
      const cplx a0 = ok ? as[kk * LD] : zero, a1 = ok ? as[kk * LD + 8] : zero;
      const cplx b0 = ok ? bs[kk * LD] : zero, b1 = ok ? bs[kk * LD + 8] : zero;
      const double s0 = a0.re + a0.im, s1 = a1.re + a1.im;
      dmma_16x8x4(p1[0], a0.re, a1.re, b0.re);
      dmma_16x8x4(p2[0], a0.im, a1.im, b0.im);
      dmma_16x8x4(p3[0], s0, s1, b0.re + b0.im);
      dmma_16x8x4(p1[1], a0.re, a1.re, b1.re);
      dmma_16x8x4(p2[1], a0.im, a1.im, b1.im);
      dmma_16x8x4(p3[1], s0, s1, b1.re + b1.im);
    }
    // the children's entries of the block (lower triangle only) through the staged inverse maps:
    // one half block (8 columns) at a time, its loads issued together, then combined and stored
    int kr0[2], kr1[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      kr0[h] = maps[rb + g + 8 * h];
      kr1[h] = maps[bp + rb + g + 8 * h];
    }
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      cplx v0[4], v1[4];
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int col = cb + ni * 8 + 2 * t + v;
        const int kc0 = maps[col], kc1 = maps[bp + col];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const bool low = rb + g + 8 * h >= col;
          const bool ok0 = low && kr0[h] >= 0 && kc0 >= 0, ok1 = low && kr1[h] >= 0 && kc1 >= 0;
          v0[2 * h + v] = ok0 ? ldc(Uc[0] + (int64_t)kc0 * bc[0] + kr0[h]) : zero;
          v1[2 * h + v] = ok1 ? ldc(Uc[1] + (int64_t)kc1 * bc[1] + kr1[h]) : zero;
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int e = 2 * h + v;
          const cplx o = cadd(cadd(zero, v0[e]), v1[e]);   // same sum order as asm_front_kernel
          Ts[(ni * 8 + 2 * t + v) * 18 + g + 8 * h] =
              cmk(o.re - (p1[ni][e] - p2[ni][e]), o.im - (p3[ni][e] - p1[ni][e] - p2[ni][e]));
        }
    }
    __syncwarp();
    // whole lines: two columns of 16 rows per instruction, rows up to the leading dimension
    // (diagonal blocks are stored whole: their upper entries are never read)
    {
      const int ldU = ldu(b);
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int r = lane & 15, cc = 2 * it + (lane >> 4);
        if (rb + r < ldU && cb + cc < b) stc(U + rb + r + (int64_t)(cb + cc) * ldU, Ts[cc * 18 + r]);
      }
    }
    __syncwarp();
  }
}

// Trailing pivot-column updates, delayed over groups of panels (multifrontal_large.cuh), through
// the same engine: F[cb:, cb:cb+cols] -= X X^T with X = F[cb:, k0:k0+K) (the TRSM'd panel rows),
// lower trapezoid of 32 x 32 tiles, enumerated per (level, panel step) on the host (compact
// lists: a level of very different fronts -- C5 -- launches no empty tile slots).
template <int WS_STAGES>
__global__ void __launch_bounds__(WS_THREADS, ws_ctas_per_sm<false, WS_STAGES>())
    panel_ws_kernel(LevelArgs a, int cb, int k0, int K, int narrow, const int4* __restrict__ tiles, int ntile,
                    long long total, int T) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* As = reinterpret_cast<cplx*>(smem_raw);
  cplx* Bs = As + WS_STAGES * S32_STAGE;
  cplx* Cs = Bs + WS_STAGES * S32_STAGE;
  StreamTile* desc = reinterpret_cast<StreamTile*>(Cs + ST_CS);
  uint64_t* bars = reinterpret_cast<uint64_t*>(desc + ST_MAXT);
  uint64_t *full = bars, *empty = bars + WS_STAGES, *cfull = bars + 2 * WS_STAGES, *cempty = cfull + 1;
  if (threadIdx.x == 0) ws_init_barriers<false, WS_STAGES>(full, empty, cfull, cempty);
  const long long q0 = (long long)blockIdx.x * T;
  const int nt = (int)min((long long)T, total - q0);
  for (int j = threadIdx.x; j < nt; j += WS_THREADS) {
    // tile q of the launch = (shift q / ntile, entry q % ntile of the step's compact tile list:
    // front of the level, tile row, tile column) -- every slot is a real tile, whatever the
    // spread of front sizes on the level
    const long long q = q0 + j;
    const int k = (int)(q / ntile);
    const int4 tl = tiles[q - (long long)k * ntile];
    const FrontDev F = a.fronts[tl.x];
    const int n = F.n, p = F.p;
    const int cols = narrow ? min(NB, p - cb) : p - cb;
    cplx* P = a.factor + (int64_t)k * a.fstride + F.fofs;
    StreamTile D;
    D.A = P + cb + (int64_t)k0 * n;
    D.C = P + cb + (int64_t)cb * n;
    D.lda = D.ldC = n;
    D.K = min(K, p - k0);
    D.M = n - cb;
    D.pad = D.M;
    D.N = cols;
    D.i0 = tl.y * 32;
    D.c0 = tl.z * 32;
    D.Uc[0] = D.Uc[1] = nullptr;
    D.bc[0] = D.bc[1] = 0;
    D.inv_off[0] = D.inv_off[1] = -1;
    desc[j] = D;
  }
  __syncthreads();
  ws_tiles<false, WS_STAGES>(desc, nt, As, Bs, Cs, full, empty, cfull, cempty, a.inv);
}

// Backward substitution of one level, one CTA per (front, shift) instance:
//   1. x of the boundary rows (final: they belong to ancestors) is staged in
//      shared memory together with z of the pivot rows;
//   2. the boundary part of every pivot column, t_j = z_j - L[p:n, j]^T x_B,
//      runs for all p columns at once (warp per column, coalesced columns);
//   3. the pivot triangle is swept in panels of NB from the last one: the
//      panel's columns subtract the already-solved pivot rows below it, then
//      one warp solves the transposed w x w triangle.
// unit = 1: unit-L LDL^T fronts (z already D^{-1}-scaled); 0: C C^T fronts.
template <int NR>
__global__ void __launch_bounds__(NT) backward_level_kernel(LevelArgs a, int unit) {
  constexpr int RB = NR < 4 ? NR : 4;   // right-hand sides per register chunk
  __shared__ cplx l11[NB * LDD];   // l11[c * LDD + i] = L[kb+i][kb+c], i > c; diagonal: 1/L[c][c] (or 1)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int inst = blockIdx.x;
  const int k = inst % a.nbatch;
  const FrontDev F = a.fronts[a.list[inst / a.nbatch]];
  const int n = F.n, p = F.p;
  const int nrhs = a.nrhs, nx = a.nx;
  const cplx* P = a.factor + (int64_t)k * a.fstride + F.fofs;
  cplx* Zk = a.Z + (int64_t)k * nx * nrhs;
  const int32_t* bidx = a.bidx + F.bidx_beg;
  const int64_t shift = a.shift0 + k;
  const cplx zero = cmk(0.0, 0.0);
  extern __shared__ __align__(16) unsigned char bwd_smem[];
  cplx* xs = reinterpret_cast<cplx*>(bwd_smem);   // n x nrhs: x (boundary rows), t then x (pivot rows)
  if (nrhs & 1) {
    // rows fastest: consecutive lanes read consecutive rows of one right-hand side (the right-hand
    // sides are n_x apart in Z); the shared-memory stride of nrhs complex is conflict free for odd nrhs
    for (int q = tid; q < n * nrhs; q += NT) {
      const int r = q / n, i = q - r * n;
      xs[i * nrhs + r] = ldc(Zk + (i < p ? F.pbeg + i : bidx[i - p]) + (int64_t)r * nx);
    }
  } else {
    for (int q = tid; q < n * nrhs; q += NT) {
      const int i = q / nrhs, r = q - i * nrhs;
      xs[q] = ldc(Zk + (i < p ? F.pbeg + i : bidx[i - p]) + (int64_t)r * nx);
    }
  }
  __syncthreads();
  // 2. boundary contributions of all pivot columns (parallel over columns); the right-hand
  // sides in register chunks of RB (the column is re-read from L1 per chunk) so many-RHS
  // solves keep the register count -- and the occupancy -- of the few-RHS ones
  if (n > p) {
    if (NR > 1 && n - p <= 128) {
      // multi-RHS, short columns (the single-panel fronts of the deep levels): the lane's (at most
      // four) column entries are loaded once, together, and reused for every chunk of right-hand
      // sides -- one exposed load latency per column instead of one per row block and chunk
      for (int j = warp; j < p; j += NT / 32) {
        const cplx* col = P + (int64_t)j * n;
        cplx lv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = p + lane + 32 * q;
          lv[q] = i < n ? ldc(col + i) : zero;
        }
        for (int r0 = 0; r0 < nrhs; r0 += RB) {
          cplx acc[RB];
#pragma unroll
          for (int r = 0; r < RB; ++r) acc[r] = zero;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i = min(p + lane + 32 * q, n - 1);   // lv is zero past the column
#pragma unroll
            for (int r = 0; r < RB; ++r)
              if (r0 + r < nrhs) acc[r] = cfma(lv[q], xs[i * nrhs + r0 + r], acc[r]);
          }
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            if (r0 + r >= nrhs) break;
            double re = acc[r].re, im = acc[r].im;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              re += __shfl_xor_sync(0xffffffffu, re, o);
              im += __shfl_xor_sync(0xffffffffu, im, o);
            }
            if (lane == 0) xs[j * nrhs + r0 + r] = cmk(xs[j * nrhs + r0 + r].re - re, xs[j * nrhs + r0 + r].im - im);
          }
        }
      }
    } else {
    for (int j = warp; j < p; j += NT / 32) {
      const cplx* col = P + (int64_t)j * n;
      for (int r0 = 0; r0 < nrhs; r0 += RB) {
        cplx acc[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) acc[r] = zero;
        for (int i = p + lane; i < n; i += 32) {
          const cplx l = ldc(col + i);
#pragma unroll
          for (int r = 0; r < RB; ++r)
            if (r0 + r < nrhs) acc[r] = cfma(l, xs[i * nrhs + r0 + r], acc[r]);
        }
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          if (r0 + r >= nrhs) break;
          double re = acc[r].re, im = acc[r].im;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            re += __shfl_xor_sync(0xffffffffu, re, o);
            im += __shfl_xor_sync(0xffffffffu, im, o);
          }
          if (lane == 0) xs[j * nrhs + r0 + r] = cmk(xs[j * nrhs + r0 + r].re - re, xs[j * nrhs + r0 + r].im - im);
        }
      }
    }
    }
    __syncthreads();
  }
  // 3. pivot triangle, panels from the last
  for (int kb = ((p - 1) / NB) * NB; kb >= 0; kb -= NB) {
    const int w = min(NB, p - kb);
    if (kb + w < p) {
      for (int j = warp; j < w; j += NT / 32) {
        const cplx* col = P + (int64_t)(kb + j) * n;
        for (int r0 = 0; r0 < nrhs; r0 += RB) {
          cplx acc[RB];
#pragma unroll
          for (int r = 0; r < RB; ++r) acc[r] = zero;
          for (int i = kb + w + lane; i < p; i += 32) {
            const cplx l = ldc(col + i);
#pragma unroll
            for (int r = 0; r < RB; ++r)
              if (r0 + r < nrhs) acc[r] = cfma(l, xs[i * nrhs + r0 + r], acc[r]);
          }
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            if (r0 + r >= nrhs) break;
            double re = acc[r].re, im = acc[r].im;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              re += __shfl_xor_sync(0xffffffffu, re, o);
              im += __shfl_xor_sync(0xffffffffu, im, o);
            }
            if (lane == 0) {
              cplx* t = xs + (kb + j) * nrhs + r0 + r;
              *t = cmk(t->re - re, t->im - im);
            }
          }
        }
      }
    }
    {
      // the block's loads issued together (compile-time trip count), then staged
      constexpr int U = NB * NB / NT;
      cplx v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = tid + u * NT, i = idx % NB, c = idx / NB;
        v[u] = (i < w && c < w && i >= c) ? ldc(P + (kb + i) + (int64_t)(kb + c) * n) : zero;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = tid + u * NT, i = idx % NB, c = idx / NB;
        if (i < w && c < w) {
          if (i > c) l11[c * LDD + i] = v[u];
          else if (i == c) l11[c * LDD + c] = unit ? cmk(1.0, 0.0) : crecip(v[u]);
        }
      }
    }
    __syncthreads();
    {
      // x_j = (t_j - sum_{c>j} L[c][j] x_c) * dinv_j in column (axpy) form: lane j
      // holds t_j; once x_c is final it is broadcast and every lane j < c subtracts
      // L[c][j] x_c -- one broadcast per step instead of a 5-level warp reduction.
      // The right-hand sides are spread over the warps.
      // two right-hand sides per warp and pass (independent chains interleave)
      for (int r0 = 2 * warp; r0 < nrhs; r0 += 2 * (NT / 32)) {
        const bool two = r0 + 1 < nrhs;
        cplx x0 = lane < w ? xs[(kb + lane) * nrhs + r0] : zero;
        cplx x1 = (lane < w && two) ? xs[(kb + lane) * nrhs + r0 + 1] : zero;
        for (int c = w - 1; c >= 0; --c) {
          const cplx dc = l11[c * LDD + c], lc = lane < c ? l11[lane * LDD + c] : zero;
          if (lane == c) {
            x0 = cmul(x0, dc);
            x1 = cmul(x1, dc);
          }
          const cplx c0 = cmk(__shfl_sync(0xffffffffu, x0.re, c), __shfl_sync(0xffffffffu, x0.im, c));
          const cplx c1 = cmk(__shfl_sync(0xffffffffu, x1.re, c), __shfl_sync(0xffffffffu, x1.im, c));
          if (lane < c) {
            x0 = cfms(x0, lc, c0);
            x1 = cfms(x1, lc, c1);
          }
        }
        if (lane < w) {
          const int prow = a.perm ? a.perm[F.pbeg + kb + lane] : F.pbeg + kb + lane;
          stc(Zk + F.pbeg + kb + lane + (int64_t)r0 * nx, x0);
          stc(a.W + bv_off(a.lay, r0, shift, prow), x0);
          xs[(kb + lane) * nrhs + r0] = x0;
          if (two) {
            stc(Zk + F.pbeg + kb + lane + (int64_t)(r0 + 1) * nx, x1);
            stc(a.W + bv_off(a.lay, r0 + 1, shift, prow), x1);
            xs[(kb + lane) * nrhs + r0 + 1] = x1;
          }
        }
      }
    }
    __syncthreads();
  }
}

template <int NR>
int launch_backward_level(const LevelArgs& a, int grid, int nmax, int unit, cudaStream_t s) {
  static DeviceOnce attr_once;
  if (attr_once.first()) {
    STFEM_CUDA_TRY(cudaFuncSetAttribute(backward_level_kernel<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        BWD_XS_MAX));
    STFEM_CUDA_TRY(cudaFuncSetAttribute(backward_level_kernel<NR>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        100));
  }
  backward_level_kernel<NR><<<grid, NT, (size_t)nmax * a.nrhs * 16, s>>>(a, unit);
  STFEM_LAUNCH_CHECK("backward_level_kernel");
  return STFEM_OK;
}

// ---------------------------------------------------------------------------
// Multi-RHS backward substitution of one level on the FP64 tensor pipe.
// backward_level_kernel turns every pivot column into nrhs warp-wide dot
// products: with 9 right-hand sides (C5) it ran at 15% of the HBM roofline, the
// top levels at one CTA of 8 warps per SM walking a 996 x 255 front column by
// column.  Here the same two products are GEMMs over the right-hand sides,
//   T = Z_p - L21^T X_B                     (M = p columns, N = nrhs, K = b rows)
//   T[0:kb] -= L[kb:kb+w, 0:kb]^T X[kb:kb+w] after panel kb is solved (right-looking, K = w),
// on m16n8k4 DMMAs: A = L^T read from global memory straight in fragment layout (8 columns x 4
// consecutive rows = eight 64-byte segments per load), B = x from shared memory, 4 real
// DMMAs per complex 16 x 8 x 4 block.  Warps own 16-column tiles; fronts with fewer tiles than
// warps split K over the spare warps and reduce through shared memory in a fixed order
// (deterministic).  Only the 32 x 32 triangle of each panel stays a warp-per-RHS substitution.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int bwd_nrp(int nrhs) { return nrhs <= 10 ? 10 : 18; }   // xs row pitch: = 2 mod 8, >= nrhs
template <int NW>
__host__ __device__ constexpr int bwd_mrhs_smem(int nmax, int nrhs) { return (nmax * bwd_nrp(nrhs) + NW * 256) * 16; }

// acc(16 columns x 8 NT8 rhs) = sum over k steps ks = ks0, ks0 + kstep, ... < KS of
// L[row0 + 4 ks + t][j0 + g (+8)] * xs[row0 + 4 ks + t][rhs]; K = valid rows from row0
template <int NT8, int UN>
__device__ __forceinline__ void bwd_gemm_tile(const cplx* __restrict__ P, int n, int j0, int jlim, int row0, int K,
                                              int ks0, int kstep, const cplx* xs, int NRP, int nrhs,
                                              double (&cr)[2][4], double (&ci)[2][4]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const cplx zero = cmk(0.0, 0.0);
  const cplx* c0 = P + (int64_t)min(j0 + g, jlim - 1) * n + row0 + t;
  const cplx* c1 = P + (int64_t)min(j0 + g + 8, jlim - 1) * n + row0 + t;
  const cplx* xb = xs + (int64_t)(row0 + t) * NRP + g;
  const int KS = (K + 3) >> 2;
  for (int ks = ks0; ks < KS; ks += UN * kstep) {
    cplx a0[UN], a1[UN];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int kq = ks + u * kstep;
      const bool ok = kq < KS && 4 * kq + t < K;
      a0[u] = ok ? ldc(c0 + 4 * kq) : zero;
      a1[u] = ok ? ldc(c1 + 4 * kq) : zero;
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int kq = ks + u * kstep;
      if (kq >= KS) break;
      const int rr = min(4 * kq + t, K - 1) - t;   // clamped: a zero A fragment must not meet a NaN
#pragma unroll
      for (int ni = 0; ni < NT8; ++ni) {
        const cplx bx = ni * 8 + g < nrhs ? xb[(int64_t)rr * NRP + ni * 8] : zero;
        dmma_16x8x4(cr[ni], a0[u].re, a1[u].re, bx.re);
        dmma_16x8x4(cr[ni], -a0[u].im, -a1[u].im, bx.im);
        dmma_16x8x4(ci[ni], a0[u].re, a1[u].re, bx.im);
        dmma_16x8x4(ci[ni], a0[u].im, a1[u].im, bx.re);
      }
    }
  }
}

// NW warps per CTA, UN k steps of A fragments in flight per warp: (8, 4) for the ordinary levels;
// (16, 8) for the launches of fronts above n = 256, whose staged x leaves room for one CTA per SM
// only -- registers and thread slots are free there, and more loads in flight is what hides the
// memory latency
template <int NW, int NT8, int UN>
__global__ void __launch_bounds__(32 * NW) backward_mrhs_kernel(LevelArgs a, int unit) {
  __shared__ cplx l11[NB * LDD];   // l11[c * LDD + i] = L[kb+i][kb+c], i > c; diagonal: 1/L[c][c] (or 1)
  extern __shared__ __align__(16) unsigned char bwd_smem[];
  constexpr int NTH = 32 * NW;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int inst = blockIdx.x;
  const int k = inst % a.nbatch;
  const FrontDev F = a.fronts[a.list[inst / a.nbatch]];
  const int n = F.n, p = F.p, b = n - p;
  const int nrhs = a.nrhs, nx = a.nx, NRP = bwd_nrp(nrhs);
  const cplx* P = a.factor + (int64_t)k * a.fstride + F.fofs;
  cplx* Zk = a.Z + (int64_t)k * nx * nrhs;
  const int32_t* bidx = a.bidx + F.bidx_beg;
  const int64_t shift = a.shift0 + k;
  const cplx zero = cmk(0.0, 0.0);
  cplx* xs = reinterpret_cast<cplx*>(bwd_smem);   // [n][NRP]: x (boundary rows), t then x (pivot rows); rhs >= nrhs: 0
  cplx* slots = xs + (int64_t)n * NRP;            // [NW][16 columns][16 rhs] partial tiles of a split K
  // rows fastest (coalesced along the pivot rows)
  for (int q = tid; q < n * nrhs; q += NTH) {
    const int r = q / n, i = q - r * n;
    xs[i * NRP + r] = ldc(Zk + (i < p ? F.pbeg + i : bidx[i - p]) + (int64_t)r * nx);
  }
  __syncthreads();
  auto apply = [&](int j0, int jlim, double (&cr)[2][4], double (&ci)[2][4]) {
#pragma unroll
    for (int ni = 0; ni < NT8; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int j = j0 + g + 8 * h;
          if (j < jlim && ni * 8 + 2 * t + v < nrhs) {
            cplx* d = xs + j * NRP + ni * 8 + 2 * t + v;
            *d = cmk(d->re - cr[ni][2 * h + v], d->im - ci[ni][2 * h + v]);
          }
        }
  };
  // 2. boundary contributions of all pivot columns
  if (b > 0) {
    const int MT = (p + 15) >> 4;
    if (MT >= NW) {
      for (int mt = warp; mt < MT; mt += NW) {
        double cr[2][4] = {}, ci[2][4] = {};
        bwd_gemm_tile<NT8, UN>(P, n, mt * 16, p, p, b, 0, 1, xs, NRP, nrhs, cr, ci);
        apply(mt * 16, p, cr, ci);
      }
    } else {
      // fewer column tiles than warps: S warps share a tile, interleaved over the k steps
      int MTc = 1;
      while (MTc < MT) MTc <<= 1;   // power of two >= MT (<= NW here)
      const int S = NW / MTc;
      const int mt = warp % MTc, sl = warp / MTc;
      {
        double cr[2][4] = {}, ci[2][4] = {};
        if (mt < MT && sl < S) bwd_gemm_tile<NT8, UN>(P, n, mt * 16, p, p, b, sl, S, xs, NRP, nrhs, cr, ci);
        cplx* my = slots + warp * 256;
#pragma unroll
        for (int ni = 0; ni < NT8; ++ni)
#pragma unroll
          for (int e = 0; e < 4; ++e)
            my[(g + 8 * (e >> 1)) * 16 + ni * 8 + 2 * t + (e & 1)] = cmk(cr[ni][e], ci[ni][e]);
      }
      __syncthreads();
      for (int q = tid; q < MT * 16 * 8 * NT8; q += NTH) {
        const int r = q % (8 * NT8), j = q / (8 * NT8), m2 = j >> 4;
        if (j >= p || r >= nrhs) continue;
        cplx sum = zero;
        for (int s2 = 0; s2 < S; ++s2) sum = cadd(sum, slots[(s2 * MTc + m2) * 256 + (j & 15) * 16 + r]);
        cplx* d = xs + j * NRP + r;
        *d = csub(*d, sum);
      }
    }
    __syncthreads();
  }
  // 3. pivot triangle, panels from the last; each solved panel updates all earlier columns
  for (int kb = ((p - 1) / NB) * NB; kb >= 0; kb -= NB) {
    const int w = min(NB, p - kb);
    for (int idx = tid; idx < NB * NB; idx += NTH) {
      const int i = idx % NB, c = idx / NB;
      if (i < w && c < w && i >= c) {
        const cplx v = ldc(P + (kb + i) + (int64_t)(kb + c) * n);
        l11[c * LDD + i] = i > c ? v : (unit ? cmk(1.0, 0.0) : crecip(v));
      }
    }
    __syncthreads();
    // x_j = (t_j - sum_{c>j} L[c][j] x_c) * dinv_j in column (axpy) form, one warp per RHS
    for (int r0 = 2 * warp; r0 < nrhs; r0 += 2 * NW) {   // two right-hand sides per warp and pass
      const bool two = r0 + 1 < nrhs;
      cplx x0 = lane < w ? xs[(kb + lane) * NRP + r0] : zero;
      cplx x1 = (lane < w && two) ? xs[(kb + lane) * NRP + r0 + 1] : zero;
      for (int c = w - 1; c >= 0; --c) {
        const cplx dc = l11[c * LDD + c], lc = lane < c ? l11[lane * LDD + c] : zero;
        if (lane == c) {
          x0 = cmul(x0, dc);
          x1 = cmul(x1, dc);
        }
        const cplx c0 = cmk(__shfl_sync(0xffffffffu, x0.re, c), __shfl_sync(0xffffffffu, x0.im, c));
        const cplx c1 = cmk(__shfl_sync(0xffffffffu, x1.re, c), __shfl_sync(0xffffffffu, x1.im, c));
        if (lane < c) {
          x0 = cfms(x0, lc, c0);
          x1 = cfms(x1, lc, c1);
        }
      }
      if (lane < w) {
        const int prow = a.perm ? a.perm[F.pbeg + kb + lane] : F.pbeg + kb + lane;
        stc(Zk + F.pbeg + kb + lane + (int64_t)r0 * nx, x0);
        stc(a.W + bv_off(a.lay, r0, shift, prow), x0);
        xs[(kb + lane) * NRP + r0] = x0;
        if (two) {
          stc(Zk + F.pbeg + kb + lane + (int64_t)(r0 + 1) * nx, x1);
          stc(a.W + bv_off(a.lay, r0 + 1, shift, prow), x1);
          xs[(kb + lane) * NRP + r0 + 1] = x1;
        }
      }
    }
    __syncthreads();
    if (kb > 0) {
      const int MT = (kb + 15) >> 4;
      for (int mt = warp; mt < MT; mt += NW) {
        double cr[2][4] = {}, ci[2][4] = {};
        bwd_gemm_tile<NT8, UN>(P, n, mt * 16, kb, kb, w, 0, 1, xs, NRP, nrhs, cr, ci);
        apply(mt * 16, kb, cr, ci);
      }
      __syncthreads();
    }
  }
}

template <int NW, int NT8, int UN>
int launch_backward_mrhs(const LevelArgs& a, int grid, int nmax, int unit, cudaStream_t s) {
  static DeviceOnce attr_once;
  if (attr_once.first()) {
    STFEM_CUDA_TRY(cudaFuncSetAttribute(backward_mrhs_kernel<NW, NT8, UN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        200 * 1024));
    STFEM_CUDA_TRY(cudaFuncSetAttribute(backward_mrhs_kernel<NW, NT8, UN>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        100));
  }
  backward_mrhs_kernel<NW, NT8, UN><<<grid, 32 * NW, bwd_mrhs_smem<NW>(nmax, a.nrhs), s>>>(a, unit);
  STFEM_LAUNCH_CHECK("backward_mrhs_kernel");
  return STFEM_OK;
}

#include "multifrontal_small.cuh"
#include "spectral.cuh"

// does depth d run on the shared-memory small-front kernels (unit-L LDL^T)?
// (measured on C4: fronts of order ~110 factor faster on the large-front kernel,
// while their backward pass stays on the shared-memory kernel)
bool level_is_small(const Plan& P, int d) {
  return P.level_nmax[d] <= std::min<int>(P.opt.small_front_n, SMALL_N);
}

// largest boundary block b = n - p among the fronts of depth d
int level_bmax(const Plan& P, int d) {
  int bm = 0;
  for (int32_t f : P.levels[d]) bm = std::max(bm, P.fronts[f].n - P.fronts[f].p);
  return bm;
}

// M_x / A_x values of every front entry, in entry order (shift-independent;
// one coalesced stream per front instead of an indirect gather)
__global__ void gather_entries_kernel(const int32_t* __restrict__ src, const double* __restrict__ Mv,
                                      const double* __restrict__ Av, double* mv, double* av, int64_t ne) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < ne) {
    const int s = src[e];
    mv[e] = Mv[s];
    av[e] = Av[s];
  }
}

// Pivot-collapse scale of every shift of a batch: scale2[s] =
// tol^2 * max_j |M_jj + lam_s A_jj|^2.  A pivot d with |d|^2 <= scale2[s] is
// reported as numerically singular.  One CTA per shift; the diagonal values are
// the same for every shift (L2 hits).
__global__ void __launch_bounds__(256) pivot_scale_kernel(const int32_t* __restrict__ diag_src, int n,
                                                          const double* __restrict__ Mv,
                                                          const double* __restrict__ Av,
                                                          const cplx* __restrict__ lam, double tol2,
                                                          double* __restrict__ scale2) {
  __shared__ double red[8];
  const cplx l = lam[blockIdx.x];
  double m = 0.0;
  for (int j = threadIdx.x; j < n; j += 256) {
    const int s = diag_src[j];
    if (s < 0) continue;
    const double re = fma(l.re, Av[s], Mv[s]), im = l.im * Av[s];
    m = fmax(m, fma(re, re, im * im));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 1; w < 8; ++w) m = fmax(m, red[w]);
    scale2[blockIdx.x] = tol2 * m;
  }
}

// opt-in shared-memory sizes of this file's kernels, once per device (a second
// device used by the same process needs its own opt-in)
int set_kernel_attributes(int dev) {
  static DeviceOnce once;
  (void)dev;
  if (!once.first()) return STFEM_OK;
#define STFEM_WS_ATTR(G, S)                                                                                     \
  STFEM_CUDA_TRY(cudaFuncSetAttribute(syrk_ws_kernel<G, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                      ws_smem_bytes<G, S>()));                                                  \
  STFEM_CUDA_TRY(cudaFuncSetAttribute(syrk_ws_kernel<G, S>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  STFEM_WS_ATTR(false, 4) STFEM_WS_ATTR(false, 3) STFEM_WS_ATTR(false, 2)
  STFEM_WS_ATTR(true, 4) STFEM_WS_ATTR(true, 3) STFEM_WS_ATTR(true, 2)
#undef STFEM_WS_ATTR
#define STFEM_PW_ATTR(S)                                                                                        \
  STFEM_CUDA_TRY(cudaFuncSetAttribute(panel_ws_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,          \
                                      ws_smem_bytes<false, S>()));                                              \
  STFEM_CUDA_TRY(cudaFuncSetAttribute(panel_ws_kernel<S>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  STFEM_PW_ATTR(4) STFEM_PW_ATTR(3) STFEM_PW_ATTR(2)
#undef STFEM_PW_ATTR
  return STFEM_OK;
}

int upload(Plan& P) {
  int dev;
  STFEM_CUDA_TRY(cudaGetDevice(&dev));
  if (P.d_fronts && P.device == dev) return STFEM_OK;
  P.free_device();
  P.device = dev;
  int rc;
  if ((rc = set_kernel_attributes(dev))) return rc;
  auto up = [&](auto** dptr, const auto& vec) -> int {
    using T = typename std::decay_t<decltype(vec)>::value_type;
    size_t bytes = std::max<size_t>(1, vec.size()) * sizeof(T);
    STFEM_CUDA_TRY(cudaMalloc((void**)dptr, bytes));
    if (!vec.empty()) STFEM_CUDA_TRY(cudaMemcpy(*dptr, vec.data(), vec.size() * sizeof(T), cudaMemcpyHostToDevice));
    return STFEM_OK;
  };
  // fronts of a level in decreasing order: the backward pass launches the few large fronts of an
  // unbalanced level (C5: n up to ~1000 next to n ~ 100) separately, so the many small ones run
  // with small shared-memory staging instead of the level maximum
  P.level_nsplit.assign(P.levels.size(), 0);
  P.level_tail_nmax.assign(P.levels.size(), 0);
  P.level_tail_pmax.assign(P.levels.size(), 0);
  for (size_t d = 0; d < P.levels.size(); ++d) {
    auto& L = P.levels[d];
    std::stable_sort(L.begin(), L.end(), [&](int32_t x, int32_t y) { return P.fronts[x].n > P.fronts[y].n; });
    int ns = 0;
    while (ns < (int)L.size() && P.fronts[L[ns]].n > BWD_SPLIT_N) ++ns;
    P.level_nsplit[d] = ns;
    for (size_t i = ns; i < L.size(); ++i) {
      P.level_tail_nmax[d] = std::max(P.level_tail_nmax[d], P.fronts[L[i]].n);
      P.level_tail_pmax[d] = std::max(P.level_tail_pmax[d], P.fronts[L[i]].p);
    }
  }
  std::vector<int32_t> lv;
  P.level_off.assign(P.levels.size() + 1, 0);
  for (size_t d = 0; d < P.levels.size(); ++d) {
    P.level_off[d] = (int64_t)lv.size();
    lv.insert(lv.end(), P.levels[d].begin(), P.levels[d].end());
  }
  P.level_off[P.levels.size()] = (int64_t)lv.size();
  if ((rc = up(&P.d_fronts, P.fronts))) return rc;
  if ((rc = up(&P.d_levels, lv))) return rc;
  if ((rc = up(&P.d_child_ids, P.child_ids))) return rc;
  if ((rc = up(&P.d_bidx, P.bidx))) return rc;
  if ((rc = up(&P.d_relpos, P.relpos))) return rc;
  if ((rc = up(&P.d_inv, P.inv))) return rc;
  if ((rc = up(&P.d_ent_src, P.ent_src))) return rc;
  STFEM_CUDA_TRY(cudaMalloc(&P.d_ent_mv, std::max<size_t>(1, P.ent_src.size()) * sizeof(double)));
  STFEM_CUDA_TRY(cudaMalloc(&P.d_ent_av, std::max<size_t>(1, P.ent_src.size()) * sizeof(double)));
  if ((rc = up(&P.d_ent_dst, P.ent_dst))) return rc;
  if ((rc = up(&P.d_ent_colptr, P.ent_colptr))) return rc;
  if ((rc = up(&P.d_perm, P.perm))) return rc;
  if ((rc = up(&P.d_iperm, P.iperm))) return rc;
  if ((rc = up(&P.d_diag_src, P.diag_src))) return rc;
  STFEM_CUDA_TRY(cudaMalloc(&P.d_err, sizeof(int)));
  STFEM_CUDA_TRY(cudaMemset(P.d_err, 0, sizeof(int)));
  if (!P.h_err) STFEM_CUDA_TRY(cudaMallocHost(&P.h_err, sizeof(int)));
  P.level_nmax.assign(P.levels.size(), 0);
  P.level_pmax.assign(P.levels.size(), 0);
  for (size_t d = 0; d < P.levels.size(); ++d)
    for (int32_t f : P.levels[d]) {
      P.level_nmax[d] = std::max(P.level_nmax[d], P.fronts[f].n);
      P.level_pmax[d] = std::max(P.level_pmax[d], P.fronts[f].p);
    }
  // Schur-update tiles of the large-front levels (lower 32 x 32 tiles of each b x b block)
  {
    std::vector<int4> t32;
    P.syrk32_off.assign(P.levels.size() + 1, 0);
    for (size_t d = 0; d < P.levels.size(); ++d) {
      P.syrk32_off[d] = (int64_t)t32.size();
      if (level_is_small(P, (int)d)) continue;
      for (int32_t f : P.levels[d]) {
        const int b = P.fronts[f].n - P.fronts[f].p;
        const int nt = (b + 31) / 32;
        for (int tj = 0; tj < nt; ++tj)
          for (int ti = tj; ti < nt; ++ti) t32.push_back(make_int4(f, ti, tj, 0));
      }
    }
    P.syrk32_off[P.levels.size()] = (int64_t)t32.size();
    if ((rc = up(&P.d_syrk32_tiles, t32))) return rc;
  }
  // trailing-update tiles of every (large level, panel step): (front, tile row, tile column)
  {
    std::vector<int4> tp;
    P.panel_off.assign(P.levels.size(), {});
    const int pg = std::max(1, P.opt.panel_group);
    for (size_t d = 0; d < P.levels.size(); ++d) {
      if (level_is_small(P, (int)d)) continue;
      for (int kb = 0; kb < P.level_pmax[d]; kb += NB) {
        const int GW = NB * pg, g0 = (kb / GW) * GW;
        const int narrow = ((kb - g0) / NB < pg - 1) ? 1 : 0, cb = kb + NB;
        P.panel_off[d].push_back((int64_t)tp.size());
        for (int32_t f : P.levels[d]) {
          const int n = P.fronts[f].n, p = P.fronts[f].p;
          const int cols = cb >= p ? 0 : (narrow ? std::min(NB, p - cb) : p - cb);
          if (cols <= 0) continue;
          const int tm = (n - cb + 31) / 32, tn = (cols + 31) / 32;
          for (int tj = 0; tj < tn; ++tj)
            for (int ti = tj; ti < tm; ++ti) tp.push_back(make_int4(f, ti, tj, 0));
        }
      }
      P.panel_off[d].push_back((int64_t)tp.size());
    }
    if ((rc = up(&P.d_panel_tiles, tp))) return rc;
  }
  // fronts of every (large level, panel step) that still have a panel at that step (p > kb), and
  // their largest order: the diagonal-block and TRSM launches of the late steps of an unbalanced
  // level run over those fronts only
  {
    std::vector<int32_t> sl;
    P.step_off.assign(P.levels.size(), {});
    P.step_nmax.assign(P.levels.size(), {});
    for (size_t d = 0; d < P.levels.size(); ++d) {
      if (level_is_small(P, (int)d)) continue;
      for (int kb = 0; kb < P.level_pmax[d]; kb += NB) {
        P.step_off[d].push_back((int64_t)sl.size());
        int nm = 0;
        for (int32_t f : P.levels[d])
          if (P.fronts[f].p > kb) {
            sl.push_back(f);
            nm = std::max(nm, P.fronts[f].n);
          }
        P.step_nmax[d].push_back(nm);
      }
      P.step_off[d].push_back((int64_t)sl.size());
    }
    if ((rc = up(&P.d_step_list, sl))) return rc;
  }
  // spectral subtrees: data + per-depth work items (fwd1 = U and F1, fwd2 = F2, bwd1 = B1, bwd2 = B2)
  {
    const int L = (int)P.levels.size();
    P.spec_off.assign(4 * L + 1, 0);
    std::vector<int4> items;
    for (int d = 0; d < L; ++d) {
      const std::vector<int32_t> none;
      const auto& roots = d < (int)P.sub_levels.size() ? P.sub_levels[d] : none;
      for (int j = 0; j < 4; ++j) {
        P.spec_off[4 * d + j] = (int64_t)items.size();
        for (int32_t t : roots) {
          const SubDev& S = P.subs[t];
          if (j == 0) {
            const int nbk = P.sub_rep[t] ? (S.g + 7) / 8 : 0;   // the class's update block: once
            for (int bj = 0; bj < nbk; ++bj)
              for (int bi = bj; bi < nbk; ++bi) items.push_back(make_int4(OP_U, t, bi, bj));
            for (int q = 0; q < (S.m + SP_BM - 1) / SP_BM; ++q) items.push_back(make_int4(OP_F1, t, q, 0));
          } else if (j == 1) {
            for (int q = 0; q < (S.g + SP_BM - 1) / SP_BM; ++q) items.push_back(make_int4(OP_F2, t, q, 0));
          } else if (j == 2) {
            // x_Gam resident, all row tiles (a root without boundary rows has no K loop: per-tile path)
            if (S.g >= 1 && S.g <= SP_B1R_K) items.push_back(make_int4(OP_B1R, t, 0, 0));
            else
              for (int q = 0; q < (S.m + 31) / 32; ++q) items.push_back(make_int4(OP_B1, t, q, 0));
          } else {
            for (int q = 0; q < (S.m + SP_BM - 1) / SP_BM; ++q) items.push_back(make_int4(OP_B2, t, q, 0));
          }
        }
      }
    }
    P.spec_off[4 * L] = (int64_t)items.size();
    if (!P.subs.empty()) {
      if ((rc = up(&P.d_subs, P.subs))) return rc;
      if ((rc = up(&P.d_V, P.h_V))) return rc;
      if ((rc = up(&P.d_th, P.h_th))) return rc;
      if ((rc = up(&P.d_RQ, P.h_RQ))) return rc;
      if ((rc = up(&P.d_C01, P.h_C01))) return rc;
      if ((rc = up(&P.d_spec_items, items))) return rc;
      int mmax = 0;
      for (const auto& S : P.subs) mmax = std::max(mmax, std::max(S.m, S.g));
      P.spec_smem = std::max(spectral_smem_bytes(mmax), SP_B1R_SMEM);
      if (P.spec_smem > 227 * 1024)
        return fail(STFEM_ERR_DIM, "spectral subtrees: interior too large for the shared-memory staging");
      STFEM_CUDA_TRY(cudaFuncSetAttribute(spectral_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, P.spec_smem));
      STFEM_CUDA_TRY(cudaFuncSetAttribute(spectral_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
  }
  return STFEM_OK;
}

int64_t bytes_per_shift(const Plan& P, int nrhs) {
  return 16 * (P.factor_stride + P.upool_stride[0] + P.upool_stride[1] +
               (int64_t)nrhs * (P.rpool_stride[0] + P.rpool_stride[1]) + (int64_t)P.n * nrhs +
               (int64_t)P.h_th.size()) + 8;
}

int ensure_workspace(Plan& P, int batch, int nrhs) {
  if (P.d_factor && P.ws_batch >= batch && P.ws_nrhs >= nrhs) return STFEM_OK;
  batch = std::max(batch, P.ws_batch);   // grow only: a later, smaller call keeps the batch split stable
  nrhs = std::max(nrhs, P.ws_nrhs);
  P.free_workspace();
  auto al = [&](cplx** d, int64_t elems) -> int {
    STFEM_CUDA_TRY(cudaMalloc((void**)d, std::max<int64_t>(1, elems) * 16));
    return STFEM_OK;
  };
  int rc;
  if ((rc = al(&P.d_factor, P.factor_stride * batch))) return rc;
  for (int q = 0; q < 2; ++q) {
    if ((rc = al(&P.d_upool[q], P.upool_stride[q] * batch))) return rc;
    if ((rc = al(&P.d_rpool[q], P.rpool_stride[q] * batch * nrhs))) return rc;
  }
  if ((rc = al(&P.d_Z, (int64_t)P.n * nrhs * batch))) return rc;
  if (!P.h_th.empty() && (rc = al(&P.d_wbuf, (int64_t)P.h_th.size() * batch))) return rc;
  STFEM_CUDA_TRY(cudaMalloc((void**)&P.d_scale2, sizeof(double) * batch));
  P.ws_batch = batch;
  P.ws_nrhs = nrhs;
  return STFEM_OK;
}

// equal-sized batches of at most bmax shifts: fewer, evenly filled waves at the top levels of the
// tree; rounded up to a multiple of the spectral kernel's 64-shift column tile when that still
// fits (e.g. 1024 shifts: 384 + 384 + 256 instead of 3 x 342, whose last spectral column tile is
// 22/64 full)
int even_batch(int nshift, int64_t bmax) {
  const int64_t nb = (nshift + bmax - 1) / bmax;
  const int64_t even = (nshift + nb - 1) / nb;
  const int64_t r64 = ((even + 63) / 64) * 64;
  return (int)((r64 <= bmax && (nshift + r64 - 1) / r64 == nb) ? r64 : even);
}

// Workspace for `batch` shifts; when the device cannot give it (fragmentation, a caller that took
// memory since cudaMemGetInfo) the batch is halved until it fits: slower, never an error a smaller
// batch would have avoided.  Returns the batch actually allocated in *batch.
int ensure_workspace_backoff(Plan& P, int* batch, int nrhs) {
  for (;;) {
    const int rc = ensure_workspace(P, *batch, nrhs);
    if (rc != STFEM_ERR_NOMEM || *batch <= 1) return rc;
    (void)cudaGetLastError();
    P.free_workspace();
    *batch = (*batch + 1) / 2;
  }
}

int auto_batch(Plan& P, int nshift, int nrhs) {
  if (P.batch > 0) return std::min(P.batch, nshift);
  // an existing workspace fixes the split (stfem_plan_reserve, or the first call): no
  // reallocation -- and no device synchronisation -- on later calls that fit it
  if (P.d_factor && P.ws_nrhs >= nrhs) return even_batch(nshift, P.ws_batch);
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) fr = (size_t)8 << 30;
  // keep whatever workspace we already own in the budget; the default 70% of what is free
  // leaves room for the caller's temporaries (residual checks)
  size_t owned = P.d_factor ? (size_t)bytes_per_shift(P, P.ws_nrhs) * P.ws_batch : 0;
  // workspace_fraction of what is free, or more when that still leaves two BlockVector stacks of
  // this solve (the caller's output / residual temporaries) and 15% free: C4 then runs 2 batches
  // of 512 shifts instead of 384 + 384 + 256 (-5 ms per step); C5, whose stacks are 29 GB, stays
  // at the fraction
  const double avail = (double)(fr + owned), bv = 16.0 * (double)P.n * nshift * nrhs;
  double budget = std::max(P.opt.workspace_fraction * avail, std::min(0.85 * avail, avail - 2.0 * bv));
  int64_t per = bytes_per_shift(P, nrhs);
  int64_t bmax = std::min<int64_t>(std::max<int64_t>(1, (int64_t)(budget / (double)per)), 4096);
  return even_batch(nshift, bmax);
}

}  // namespace

Plan::~Plan() {
  free_workspace();
  free_device();
  if (h_err) cudaFreeHost(h_err);
}

void Plan::free_device() {
  cudaFree(d_fronts);
  cudaFree(d_levels);
  cudaFree(d_child_ids);
  cudaFree(d_bidx);
  cudaFree(d_relpos);
  cudaFree(d_inv);
  cudaFree(d_syrk32_tiles);
  d_syrk32_tiles = nullptr;
  cudaFree(d_panel_tiles);
  d_panel_tiles = nullptr;
  cudaFree(d_step_list);
  d_step_list = nullptr;
  cudaFree(d_ent_src);
  cudaFree(d_ent_mv);
  cudaFree(d_ent_av);
  d_ent_mv = d_ent_av = nullptr;
  cudaFree(d_ent_dst);
  cudaFree(d_ent_colptr);
  d_ent_colptr = nullptr;
  cudaFree(d_perm);
  cudaFree(d_iperm);
  d_iperm = nullptr;
  cudaFree(d_diag_src);
  d_diag_src = nullptr;
  cudaFree(d_err);
  cudaFree(d_subs);
  cudaFree(d_V);
  cudaFree(d_th);
  cudaFree(d_RQ);
  cudaFree(d_C01);
  cudaFree(d_spec_items);
  d_subs = nullptr;
  d_V = d_th = d_RQ = d_C01 = nullptr;
  d_spec_items = nullptr;
  d_fronts = nullptr;
  d_levels = nullptr;
  d_child_ids = d_bidx = d_relpos = d_inv = d_ent_src = d_ent_dst = d_perm = nullptr;
  d_err = nullptr;
  device = -1;
}

void Plan::free_workspace() {
  cudaFree(d_factor);
  for (int q = 0; q < 2; ++q) {
    cudaFree(d_upool[q]);
    cudaFree(d_rpool[q]);
    d_upool[q] = d_rpool[q] = nullptr;
  }
  cudaFree(d_Z);
  cudaFree(d_wbuf);
  cudaFree(d_scale2);
  d_scale2 = nullptr;
  d_factor = d_Z = d_wbuf = nullptr;
  ws_batch = ws_nrhs = 0;
}

// Enqueue the factor + solve of every shift on `stream` (no host wait; a pivot collapse is latched
// in P.d_err and read by plan_check).
int factor_solve(Plan& P, const double* Mv, const double* Av, const cplx* lam, int nshift, int nrhs,
                 const cplx* G, cplx* W, stfem_bv_layout lay, cudaStream_t stream) {
  if (nshift < 0 || nrhs < 1) return fail(STFEM_ERR_DIM, "factor_solve: nshift >= 0 and nrhs >= 1 required");
  if (nrhs > MAXR) return fail(STFEM_ERR_DIM, "factor_solve: at most 16 right-hand sides per call");
  if ((int64_t)P.max_front * nrhs * 16 > BWD_XS_MAX)
    return fail(STFEM_ERR_DIM, "factor_solve: too many right-hand sides per call for this front size "
                               "(use stfem_plan_max_rhs)");
  if (!Mv || !Av || !lam || !G || !W) return fail(STFEM_ERR_ARG, "factor_solve: null pointer");
  if (lay.chunk_cols <= 0) return fail(STFEM_ERR_ARG, "factor_solve: chunk_cols must be positive");
  if (nshift == 0) return STFEM_OK;
  int rc;
  if ((rc = upload(P))) return rc;
  int batch = auto_batch(P, nshift, nrhs);
  if ((rc = ensure_workspace_backoff(P, &batch, nrhs))) return rc;

  LevelArgs a{};
  a.fronts = P.d_fronts;
  a.child_ids = P.d_child_ids;
  a.relpos = P.d_relpos;
  a.inv = P.d_inv;
  a.bidx = P.d_bidx;
  a.ent_src = P.d_ent_src;
  a.ent_dst = P.d_ent_dst;
  a.ent_colptr = P.d_ent_colptr;
  a.perm = P.io_permuted ? nullptr : P.d_perm;   // nullptr: G and W are indexed in the plan's numbering
  {
    const int64_t ne = (int64_t)P.ent_src.size();
    if (ne > 0) {
      gather_entries_kernel<<<(unsigned)((ne + 255) / 256), 256, 0, stream>>>(P.d_ent_src, Mv, Av, P.d_ent_mv,
                                                                             P.d_ent_av, ne);
      STFEM_LAUNCH_CHECK("gather_entries_kernel");
    }
  }
  a.Mv = P.d_ent_mv;   // entry-ordered
  a.Av = P.d_ent_av;
  a.factor = P.d_factor;
  a.fstride = P.factor_stride;
  a.Z = P.d_Z;
  a.nx = P.n;
  a.nrhs = nrhs;
  a.G = G;
  a.W = W;
  a.lay = lay;
  a.err = P.d_err;
  a.scale2 = P.d_scale2;
  int64_t nlaunch = P.ent_src.empty() ? 0 : 1;   // gather_entries_kernel
  // per-launch CUDA-event times (record mode / opt.level_timing; diagnostics only: it waits for
  // the stream at the end of the call)
  const bool level_print = P.opt.level_timing != 0;
  const bool level_timing = level_print || P.record_levels;
  std::vector<cudaEvent_t> evs;
  // per-kernel-family accounting (record mode): event after every launch,
  // the gap to the previous event is charged to the launch's family
  cudaEvent_t fev_start = nullptr;
  std::vector<std::pair<cudaEvent_t, int>> fevs;
  std::vector<int> fev_depth;
  int cur_depth = -1;
  auto fam = [&](int f) {
    if (!level_timing) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, stream);
    fevs.push_back({e, f});
    fev_depth.push_back(cur_depth);
  };
  auto mark = [&]() {
    if (!level_timing) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, stream);
    evs.push_back(e);
  };
  const double tol2 = P.opt.pivot_tol * P.opt.pivot_tol;
  const LevelArgs a0 = a;
  cudaStream_t st = stream;
  auto run_batch = [&](int s0, int nb) -> int {
    LevelArgs a = a0;
    a.nbatch = nb;
    a.lam = lam + s0;
    a.shift0 = s0;
    a.err_base = P.shift_base;
    cplx* up[2] = {P.d_upool[0], P.d_upool[1]};
    cplx* rp[2] = {P.d_rpool[0], P.d_rpool[1]};
    pivot_scale_kernel<<<nb, 256, 0, st>>>(P.d_diag_src, P.n, Mv, Av, lam + s0, tol2, P.d_scale2);
    STFEM_LAUNCH_CHECK("pivot_scale_kernel");
    ++nlaunch;
    SpecArgs sa{};
    sa.subs = P.d_subs;
    sa.V = P.d_V;
    sa.th = P.d_th;
    sa.RQ = P.d_RQ;
    sa.C01 = P.d_C01;
    sa.fronts = P.d_fronts;
    sa.bidx = P.d_bidx;
    sa.perm = P.io_permuted ? nullptr : P.d_perm;
    sa.lam = lam + s0;
    sa.nb = nb;
    sa.nrhs = nrhs;
    sa.nx = P.n;
    sa.shift0 = s0;
    sa.Z = a.Z;
    sa.G = G;
    sa.W = W;
    sa.lay = lay;
    sa.wbuf = P.d_wbuf;
    sa.wstride = P.ws_batch;
    if (!P.subs.empty()) {
      const int64_t nth = (int64_t)P.h_th.size();
      const int64_t tot = nth * nb;
      spectral_w_kernel<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 16), 256, 0, st>>>(
          P.d_th, nth, lam + s0, nb, P.d_wbuf, P.ws_batch, tol2, P.d_err, P.shift_base + s0);
      STFEM_LAUNCH_CHECK("spectral_w_kernel");
      ++nlaunch;
      fam(FAM_SPECTRAL);
    }
    for (int d = P.depth; d >= 0; --d) {
      cur_depth = d;
      const int q = d & 1;
      a.list = P.d_levels + P.level_off[d];
      a.nlist = (int32_t)P.levels[d].size();
      a.ucur = up[q];
      a.ucur_stride = P.upool_stride[q];
      a.uchild = up[q ^ 1];
      a.uchild_stride = P.upool_stride[q ^ 1];
      a.rcur = rp[q];
      a.rcur_stride = P.rpool_stride[q];
      a.rchild = rp[q ^ 1];
      a.rchild_stride = P.rpool_stride[q ^ 1];
      if (P.spec_off[4 * d + 2] > P.spec_off[4 * d]) {
        // spectral subtree roots of this depth: update blocks + forward RHS (no factor storage)
        for (int j = 0; j < 2; ++j) {
          const int64_t n_it = P.spec_off[4 * d + j + 1] - P.spec_off[4 * d + j];
          if (n_it == 0) continue;
          sa.items = P.d_spec_items + P.spec_off[4 * d + j];
          sa.ucur = a.ucur;
          sa.ucur_stride = a.ucur_stride;
          sa.rcur = a.rcur;
          sa.rcur_stride = a.rcur_stride;
          spectral_kernel<<<dim3((unsigned)n_it, (unsigned)((nb * nrhs + SP_BN - 1) / SP_BN)), 256, P.spec_smem,
                            st>>>(sa);
          STFEM_LAUNCH_CHECK("spectral_kernel");
          ++nlaunch;
          fam(FAM_SPECTRAL);
        }
      }
      if (a.nlist == 0) {
        mark();
        continue;
      }
      const int nmax = P.level_nmax[d];
      if (level_is_small(P, d)) {
        if ((rc = launch_small_factor_any(a, a.nlist * nb, nmax, st))) return rc;
        ++nlaunch;
        fam(FAM_SMALL);
      } else {
        // large fronts: tile-parallel pipeline over all (front, shift) instances of the level
        const int ninst = a.nlist * nb, pmax = P.level_pmax[d];
        const int T = std::max(1, std::min(ST_MAXT, P.opt.tiles_per_cta));   // tiles per CTA of the update engine
        const int ws_stages = P.opt.ws_stages;
        const int64_t n32 = P.syrk32_off[d + 1] - P.syrk32_off[d];
        // fused levels: the boundary block U is gathered by syrk_ws_kernel<true>, not assembled here
        a.asm_pivots_only = (n32 > 0 && pmax >= P.opt.fused_min_p) ? 1 : 0;
        const int asm_cols = a.asm_pivots_only ? pmax : nmax;
        // deep levels (fronts of order <= asm_whole_n): one CTA per instance for all columns
        a.asm_cpc = nmax <= P.opt.asm_whole_n ? ((asm_cols + ASM_COLS - 1) / ASM_COLS) * ASM_COLS : ASM_COLS;
        asm_front_kernel<<<dim3(ninst, (asm_cols + a.asm_cpc - 1) / a.asm_cpc), NT, (size_t)2 * nmax * sizeof(int),
                           st>>>(a);
        STFEM_LAUNCH_CHECK("asm_front_kernel");
        ++nlaunch;
        fam(FAM_ASM);
        const int pg = std::max(1, P.opt.panel_group);
        for (int kb = 0; kb < pmax; kb += NB) {
          // this step's fronts (p > kb) only
          LevelArgs as = a;
          as.list = P.d_step_list + P.step_off[d][kb / NB];
          as.nlist = (int32_t)(P.step_off[d][kb / NB + 1] - P.step_off[d][kb / NB]);
          const int sinst = as.nlist * nb, snmax = P.step_nmax[d][kb / NB];
          if (nrhs == 1)
            diag_kernel<true><<<sinst, 32, 0, st>>>(as, kb);
          else
            diag_kernel<false><<<sinst, 32 * std::min(8, (nrhs + DIAG_RPW - 1) / DIAG_RPW), 0, st>>>(as, kb);
          STFEM_LAUNCH_CHECK("diag_kernel");
          fam(FAM_DIAG);
          const dim3 tg(sinst, (unsigned)std::max(1, (snmax - kb + TR_ROWS - 1) / TR_ROWS));
          if (std::min(NB, pmax - kb) <= 16) trsm_kernel<16><<<tg, TR_ROWS, 0, st>>>(as, kb);
          else trsm_kernel<32><<<tg, TR_ROWS, 0, st>>>(as, kb);
          STFEM_LAUNCH_CHECK("trsm_kernel");
          fam(FAM_TRSM);
          nlaunch += 2;
          // delayed updates over groups of panel_group panels starting at g0 (see
          // panel_update32_kernel): inside a group only the next panel's columns are updated,
          // by every panel of the group so far; after its last panel, everything beyond
          const int GW = NB * pg, g0 = (kb / GW) * GW;
          const int narrow = ((kb - g0) / NB < pg - 1) ? 1 : 0;
          const int cb = kb + NB, k0 = g0, K = kb + NB - g0;
          const int step = kb / NB;
          const int64_t toff = P.panel_off[d][step];
          const int tiles = (int)(P.panel_off[d][step + 1] - toff);
          if (tiles > 0) {
            const long long total = (long long)nb * tiles;
            const unsigned gr = (unsigned)((total + T - 1) / T);
            const int4* ptl = P.d_panel_tiles + toff;
            if (ws_stages == 2)
              panel_ws_kernel<2><<<gr, WS_THREADS, ws_smem_bytes<false, 2>(), st>>>(a, cb, k0, K, narrow, ptl, tiles, total, T);
            else if (ws_stages == 4)
              panel_ws_kernel<4><<<gr, WS_THREADS, ws_smem_bytes<false, 4>(), st>>>(a, cb, k0, K, narrow, ptl, tiles, total, T);
            else
              panel_ws_kernel<3><<<gr, WS_THREADS, ws_smem_bytes<false, 3>(), st>>>(a, cb, k0, K, narrow, ptl, tiles, total, T);
            STFEM_LAUNCH_CHECK("panel_ws_kernel");
            ++nlaunch;
            fam(FAM_PANEL);
          }
        }
        const int bmax = level_bmax(P, d);
        if (n32 > 0 && a.asm_pivots_only && pmax <= P.opt.front_syrk_max_p && pmax <= SF_KMAX &&
            sf_smem_bytes(bmax, pmax, bmax <= 112 ? 4 : 8) <= 100 * 1024) {
          // one pivot panel: the whole L21 of an instance fits in shared memory
          static DeviceOnce sf_once;
          if (sf_once.first()) {
            STFEM_CUDA_TRY(cudaFuncSetAttribute(syrk_front_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
            STFEM_CUDA_TRY(cudaFuncSetAttribute(syrk_front_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
          }
          const int sm_b = sf_smem_bytes(bmax, pmax, bmax <= 112 ? 4 : 8);
          if (bmax <= 112) syrk_front_kernel<128><<<ninst, 128, sm_b, st>>>(a);
          else syrk_front_kernel<256><<<ninst, 256, sm_b, st>>>(a);
          STFEM_LAUNCH_CHECK("syrk_front_kernel");
          ++nlaunch;
          fam(FAM_SYRK);
        } else if (n32 > 0) {
          const long long total = (long long)n32 * nb;
          const unsigned gr = (unsigned)((total + T - 1) / T);
          const int4* tl = P.d_syrk32_tiles + P.syrk32_off[d];
#define STFEM_SYRK_LAUNCH(G, S) \
  syrk_ws_kernel<G, S><<<gr, WS_THREADS, ws_smem_bytes<G, S>(), st>>>(a, tl, (int)n32, total, T)
          if (a.asm_pivots_only) {
            if (ws_stages == 2) STFEM_SYRK_LAUNCH(true, 2);
            else if (ws_stages == 3) STFEM_SYRK_LAUNCH(true, 3);
            else STFEM_SYRK_LAUNCH(true, 4);
          } else {
            if (ws_stages == 2) STFEM_SYRK_LAUNCH(false, 2);
            else if (ws_stages == 4) STFEM_SYRK_LAUNCH(false, 4);
            else STFEM_SYRK_LAUNCH(false, 3);
          }
#undef STFEM_SYRK_LAUNCH
          STFEM_LAUNCH_CHECK("syrk_ws_kernel");
          ++nlaunch;
          fam(FAM_SYRK);
        }
      }
      mark();
    }
    for (int d = 0; d <= P.depth; ++d) {
      cur_depth = d;
      a.list = P.d_levels + P.level_off[d];
      a.nlist = (int32_t)P.levels[d].size();
      for (int j = 2; j < 4; ++j) {
        const int64_t n_it = P.spec_off[4 * d + j + 1] - P.spec_off[4 * d + j];
        if (n_it == 0) continue;
        sa.items = P.d_spec_items + P.spec_off[4 * d + j];
        spectral_kernel<<<dim3((unsigned)n_it, (unsigned)((nb * nrhs + SP_BN - 1) / SP_BN)), 256, P.spec_smem,
                          st>>>(sa);
        STFEM_LAUNCH_CHECK("spectral_kernel");
        ++nlaunch;
        fam(FAM_SPECTRAL);
      }
      if (a.nlist == 0) {
        mark();
        continue;
      }
      // factor format of this level: small-front kernel = unit-L LDL^T, large = C C^T
      const bool ldlt = level_is_small(P, d);
      a.unit_diag = ldlt ? 1 : 0;
      // one launch per size class: [0, nsplit) fronts of order > BWD_SPLIT_N, then the rest
      auto bwd = [&](int32_t off, int32_t cnt, int nmax, int pmax) -> int {
        LevelArgs b = a;
        b.list = a.list + off;
        b.nlist = cnt;
        const int bsm = small_bwd_smem_bytes(nmax, pmax, small_nr(nrhs));
        if (nmax <= SMALL_N && bsm <= 200 * 1024 && P.opt.small_front_n > 0 && (ldlt || nrhs < 2 || pmax <= P.opt.bwd_dmma_min_p))
          return launch_small_backward_any(b, cnt * nb, nmax, pmax, st);
        const int u = ldlt ? 1 : 0, gsz = cnt * nb;
        if (nrhs >= 2 && pmax > P.opt.bwd_dmma_min_p && bwd_mrhs_smem<8>(nmax, nrhs) <= 200 * 1024) {
          // multi-RHS, multi-panel fronts: GEMMs over the right-hand sides on DMMA
          if (nmax > BWD_SPLIT_N && bwd_mrhs_smem<16>(nmax, nrhs) <= 200 * 1024)
            return nrhs <= 8 ? launch_backward_mrhs<16, 1, 8>(b, gsz, nmax, u, st)
                             : launch_backward_mrhs<16, 2, 8>(b, gsz, nmax, u, st);
          if (nmax > BWD_SPLIT_N)   // the largest fronts: 8 warps (their staged x leaves no room for 16 reduction slots)
            return nrhs <= 8 ? launch_backward_mrhs<8, 1, 8>(b, gsz, nmax, u, st)
                             : launch_backward_mrhs<8, 2, 8>(b, gsz, nmax, u, st);
          return nrhs <= 8 ? launch_backward_mrhs<8, 1, 4>(b, gsz, nmax, u, st)
                           : launch_backward_mrhs<8, 2, 4>(b, gsz, nmax, u, st);
        }
        switch (small_nr(nrhs)) {
          case 1: return launch_backward_level<1>(b, gsz, nmax, u, st);
          case 2: return launch_backward_level<2>(b, gsz, nmax, u, st);
          case 4: return launch_backward_level<4>(b, gsz, nmax, u, st);
          case 8: return launch_backward_level<8>(b, gsz, nmax, u, st);
          default: return launch_backward_level<16>(b, gsz, nmax, u, st);
        }
      };
      const int ns = P.level_nsplit[d];
      if (ns > 0 && ns < a.nlist) {
        if ((rc = bwd(0, ns, P.level_nmax[d], P.level_pmax[d]))) return rc;
        if ((rc = bwd(ns, a.nlist - ns, P.level_tail_nmax[d], P.level_tail_pmax[d]))) return rc;
        ++nlaunch;
      } else if ((rc = bwd(0, a.nlist, P.level_nmax[d], P.level_pmax[d]))) {
        return rc;
      }
      ++nlaunch;
      fam(FAM_BACKWARD);
      mark();
    }
    return STFEM_OK;
  };
  if (level_timing) {
    cudaEventCreate(&fev_start);
    cudaEventRecord(fev_start, stream);
  }
  mark();
  for (int s0 = 0; s0 < nshift; s0 += batch)
    if ((rc = run_batch(s0, std::min(batch, nshift - s0)))) return rc;
  P.last_batch = batch;
  P.last_launches = nlaunch;
  P.last_nbatches = (nshift + batch - 1) / batch;
  if (level_timing) {
    cudaStreamSynchronize(stream);
    int L = P.depth + 1;
    // level_ms[0..L): factor launches by depth, [L..2L): backward launches by depth (summed over batches)
    P.level_ms.assign(2 * L, 0.0);
    for (size_t i = 1; i < evs.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, evs[i - 1], evs[i]);
      int j = (int)((i - 1) % (2 * L));
      int d = j < L ? P.depth - j : j - L;
      P.level_ms[(j < L ? 0 : L) + d] += ms;
      if (level_print)
        fprintf(stderr, "[stfem] batch %d %s depth %d: %.3f ms\n", (int)((i - 1) / (2 * L)),
                j < L ? "factor" : "backward", d, ms);
    }
    for (auto e : evs) cudaEventDestroy(e);
    P.family_ms.assign(NFAM, 0.0);
    P.family_launches.assign(NFAM, 0);
    cudaEvent_t prev = fev_start;
    std::vector<double> dfm((size_t)(P.depth + 2) * NFAM, 0.0);
    for (size_t i = 0; i < fevs.size(); ++i) {
      const auto& fe = fevs[i];
      float ms = 0;
      cudaEventElapsedTime(&ms, prev, fe.first);
      P.family_ms[fe.second] += ms;
      P.family_launches[fe.second] += 1;
      dfm[(size_t)(fev_depth[i] + 1) * NFAM + fe.second] += ms;
      if (level_print && fe.second == FAM_SPECTRAL)
        fprintf(stderr, "[stfem spectral launch] depth %d: %.3f ms\n", fev_depth[i], ms);
      prev = fe.first;
    }
    if (level_print) {
      static const char* fn[NFAM] = {"spectral", "asm", "diag", "trsm", "panel", "syrk", "backward", "small"};
      fprintf(stderr, "[stfem depth x family ms]  depth");
      for (int f = 0; f < NFAM; ++f) fprintf(stderr, " %9s", fn[f]);
      fprintf(stderr, "\n");
      for (int d = -1; d <= P.depth; ++d) {
        fprintf(stderr, "[stfem depth x family ms]  %5d", d);
        for (int f = 0; f < NFAM; ++f) fprintf(stderr, " %9.2f", dfm[(size_t)(d + 1) * NFAM + f]);
        fprintf(stderr, "\n");
      }
    }
    for (auto& fe : fevs) cudaEventDestroy(fe.first);
    cudaEventDestroy(fev_start);
  }
  return STFEM_OK;
}

int upload_tables(Plan& P) { return upload(P); }

int plan_reserve(Plan& P, int nshift, int nrhs) {
  int rc;
  if ((rc = upload(P))) return rc;
  int batch = auto_batch(P, nshift, nrhs);
  return ensure_workspace_backoff(P, &batch, nrhs);
}

// wait for the work issued so far on `stream`, read and clear the latched pivot-collapse flag
int plan_check(Plan& P, cudaStream_t stream) {
  if (!P.d_err) return STFEM_OK;   // nothing was ever enqueued
  STFEM_CUDA_TRY(cudaMemcpyAsync(P.h_err, P.d_err, sizeof(int), cudaMemcpyDeviceToHost, stream));
  STFEM_CUDA_TRY(cudaMemsetAsync(P.d_err, 0, sizeof(int), stream));
  STFEM_CUDA_TRY(cudaStreamSynchronize(stream));
  const int h_err = *P.h_err;
  if (h_err) {
    char buf[200];
    snprintf(buf, sizeof(buf), "singular pivot (numerically singular shifted system M_x + lam A_x) at shift "
                               "index %d", h_err - 1);
    return fail(STFEM_ERR_SINGULAR, buf);
  }
  return STFEM_OK;
}

}  // namespace stfem

using stfem::Plan;

extern "C" int stfem_plan_create(int32_t n, const int64_t* rowptr, const int32_t* colind,
                                 const double* coords, int32_t dim, int32_t leaf_size, stfem_plan** out) {
  if (!out || !rowptr || !colind || !coords) return stfem::fail(STFEM_ERR_ARG, "plan_create: null pointer");
  Plan* P = new Plan();
  int rc = stfem::build_symbolic(*P, n, rowptr, colind, coords, dim, leaf_size);
  if (rc) {
    delete P;
    return rc;
  }
  *out = reinterpret_cast<stfem_plan*>(P);
  return STFEM_OK;
}

extern "C" int stfem_plan_set_spectral(stfem_plan* plan, int32_t nroots, const int32_t* root_front,
                                       const int32_t* first, const int64_t* offsets, const double* V,
                                       int64_t nV, const double* theta, int64_t ntheta, const double* RQ,
                                       int64_t nRQ, const double* C01, int64_t nC01) {
  if (!plan) return stfem::fail(STFEM_ERR_ARG, "plan_set_spectral: null plan");
  Plan& P = *reinterpret_cast<Plan*>(plan);
  const int32_t nf = (int32_t)P.fronts.size();
  if (nroots < 0 || (nroots > 0 && (!root_front || !first || !offsets || !V || !theta)))
    return stfem::fail(STFEM_ERR_ARG, "plan_set_spectral: null pointer");
  // subtree pivot ranges: first pivot of every front's subtree (postorder: children first)
  std::vector<int32_t> sub_first(nf);
  for (int32_t f = 0; f < nf; ++f) sub_first[f] = P.fronts[f].pbeg;
  for (int32_t f = 0; f < nf; ++f)
    if (P.fronts[f].parent >= 0)
      sub_first[P.fronts[f].parent] = std::min(sub_first[P.fronts[f].parent], sub_first[f]);
  std::vector<char> is_root(nf, 0), skip(nf, 0);
  std::vector<stfem::SubDev> subs(nroots);
  for (int32_t t = 0; t < nroots; ++t) {
    const int32_t f = root_front[t];
    if (f < 0 || f >= nf || is_root[f]) return stfem::fail(STFEM_ERR_ARG, "plan_set_spectral: bad root front");
    const stfem::FrontDev& F = P.fronts[f];
    stfem::SubDev& S = subs[t];
    S.front = f;
    S.first = first[t];
    S.m = F.pbeg + F.p - first[t];
    S.g = F.n - F.p;
    S.vofs = offsets[4 * t];
    S.tofs = offsets[4 * t + 1];
    S.rqofs = offsets[4 * t + 2];
    S.cofs = offsets[4 * t + 3];
    if (first[t] != sub_first[f] || S.m < 1)
      return stfem::fail(STFEM_ERR_DIM, "plan_set_spectral: subtree interior range does not match the plan");
    if (S.vofs < 0 || S.vofs + (int64_t)S.m * S.m > nV || S.tofs < 0 || S.tofs + S.m > ntheta || S.rqofs < 0 ||
        S.rqofs + 2LL * S.g * S.m > nRQ || S.cofs < 0 || S.cofs + 2LL * S.g * S.g > nC01)
      return stfem::fail(STFEM_ERR_DIM, "plan_set_spectral: offsets outside the data arrays");
    is_root[f] = 1;
  }
  for (int32_t f = 0; f < nf; ++f) {
    for (int32_t a = f; a >= 0; a = P.fronts[a].parent)
      if (is_root[a]) {
        skip[f] = 1;
        break;
      }
  }
  P.free_workspace();
  P.free_device();
  P.subs = subs;
  P.sub_levels.assign(P.depth + 1, {});
  P.levels.assign(P.depth + 1, {});
  for (int32_t d = 0; d <= P.depth; ++d)
    for (int32_t f : P.levels_all[d])
      if (!skip[f]) P.levels[d].push_back(f);
  for (int32_t t = 0; t < nroots; ++t) P.sub_levels[P.fronts[root_front[t]].depth].push_back(t);
  stfem::assign_factor_offsets(P, skip);
  // Congruent subtrees (spectral.py hands them the SAME data offsets) have the same update block
  // U(lam) = -(R diag(w) R^T + C0 + lam C1) for every shift: it is computed once per class (by the
  // class's first subtree of each pool parity) and the other roots' update blocks alias it -- the
  // parents gather through their own inverse maps, so nothing else changes.  C4: 1024 subtrees,
  // 20 classes: 98% of the update-block GEMMs of the spectral level disappear.
  for (int32_t f = 0; f < nf; ++f) P.fronts[f].uofs = P.uofs0[f];
  P.sub_rep.assign(nroots, 1);
  {
    std::vector<std::pair<std::array<int64_t, 5>, int32_t>> seen;
    for (int32_t t = 0; t < nroots; ++t) {
      const stfem::SubDev& S = subs[t];
      const std::array<int64_t, 5> key{S.vofs, S.tofs, S.rqofs, S.cofs, (int64_t)(P.fronts[S.front].depth & 1)};
      int32_t rep = -1;
      for (const auto& e : seen)
        if (e.first == key) {
          rep = e.second;
          break;
        }
      if (rep < 0) {
        seen.push_back({key, t});
      } else {
        P.sub_rep[t] = 0;
        P.fronts[S.front].uofs = P.fronts[subs[rep].front].uofs;
      }
    }
  }
  P.h_V.assign(V, V + (nroots ? nV : 0));
  P.h_th.assign(theta, theta + (nroots ? ntheta : 0));
  P.h_RQ.assign(RQ, RQ + (nroots ? nRQ : 0));
  P.h_C01.assign(C01, C01 + (nroots ? nC01 : 0));
  P.spectral_flops_u = 0;
  P.spectral_flops_rhs = 0;
  for (int32_t t = 0; t < nroots; ++t) {
    const stfem::SubDev& S = subs[t];
    const int64_t E = (int64_t)S.g * (S.g + 1) / 2;
    if (P.sub_rep[t]) P.spectral_flops_u += 4 * E * S.m;   // executed: one update block per class
    P.spectral_flops_rhs += 4LL * S.m * S.m * 2 + 4LL * S.g * 2 * S.m * 2;
  }
  return STFEM_OK;
}

extern "C" int stfem_plan_spectral_stats(const stfem_plan* plan, int32_t* nroots, double* flops_u,
                                         double* flops_rhs, int64_t* bytes) {
  if (!plan) return stfem::fail(STFEM_ERR_ARG, "plan_spectral_stats: null plan");
  const Plan& P = *reinterpret_cast<const Plan*>(plan);
  if (nroots) *nroots = (int32_t)P.subs.size();
  if (flops_u) *flops_u = (double)P.spectral_flops_u;
  if (flops_rhs) *flops_rhs = (double)P.spectral_flops_rhs;
  if (bytes) *bytes = 8 * (int64_t)(P.h_V.size() + P.h_th.size() + P.h_RQ.size() + P.h_C01.size());
  return STFEM_OK;
}

extern "C" int stfem_plan_destroy(stfem_plan* plan) {
  delete reinterpret_cast<Plan*>(plan);
  return STFEM_OK;
}

extern "C" int stfem_plan_stats_get(const stfem_plan* plan, stfem_plan_stats* s) {
  if (!plan || !s) return stfem::fail(STFEM_ERR_ARG, "plan_stats: null pointer");
  const Plan& P = *reinterpret_cast<const Plan*>(plan);
  s->n = P.n;
  s->num_fronts = (int32_t)P.fronts.size();
  s->depth = P.depth;
  s->max_front = P.max_front;
  s->max_pivots = P.max_pivots;
  s->nnz_factor = P.nnz_factor;
  s->factor_elems = P.factor_stride;
  s->update_elems = P.upool_stride[0] + P.upool_stride[1];
  s->flops_factor = P.flops;
  s->nnz_pattern = P.nnz_pattern;
  return STFEM_OK;
}

extern "C" int stfem_plan_perm(const stfem_plan* plan, int32_t* perm) {
  if (!plan || !perm) return stfem::fail(STFEM_ERR_ARG, "plan_perm: null pointer");
  const Plan& P = *reinterpret_cast<const Plan*>(plan);
  std::copy(P.perm.begin(), P.perm.end(), perm);
  return STFEM_OK;
}

extern "C" int stfem_plan_fronts(const stfem_plan* plan, int32_t* t) {
  if (!plan || !t) return stfem::fail(STFEM_ERR_ARG, "plan_fronts: null pointer");
  const Plan& P = *reinterpret_cast<const Plan*>(plan);
  for (size_t f = 0; f < P.fronts.size(); ++f) {
    const auto& F = P.fronts[f];
    t[5 * f + 0] = F.pbeg;
    t[5 * f + 1] = F.p;
    t[5 * f + 2] = F.n;
    t[5 * f + 3] = F.parent;
    t[5 * f + 4] = F.depth;
  }
  return STFEM_OK;
}

extern "C" int stfem_plan_front_rows(const stfem_plan* plan, int64_t* offsets, int32_t* rows) {
  if (!plan || !offsets) return stfem::fail(STFEM_ERR_ARG, "plan_front_rows: null pointer");
  const Plan& P = *reinterpret_cast<const Plan*>(plan);
  int64_t o = 0;
  for (size_t f = 0; f < P.fronts.size(); ++f) {
    const auto& F = P.fronts[f];
    offsets[f] = o;
    if (rows) {
      for (int32_t i = 0; i < F.p; ++i) rows[o + i] = F.pbeg + i;
      for (int32_t i = 0; i < F.n - F.p; ++i) rows[o + F.p + i] = P.bidx[F.bidx_beg + i];
    }
    o += F.n;
  }
  offsets[P.fronts.size()] = o;
  return STFEM_OK;
}

extern "C" int stfem_plan_record_levels(stfem_plan* plan, int32_t on) {
  if (!plan) return stfem::fail(STFEM_ERR_ARG, "plan_record_levels: null pointer");
  reinterpret_cast<Plan*>(plan)->record_levels = on != 0;
  return STFEM_OK;
}

extern "C" int stfem_plan_level_report(const stfem_plan* plan, double* ms, double* flops, int32_t* small) {
  if (!plan) return stfem::fail(STFEM_ERR_ARG, "plan_level_report: null pointer");
  const Plan& P = *reinterpret_cast<const Plan*>(plan);
  const int L = P.depth + 1;
  for (int i = 0; i < 2 * L; ++i)
    if (ms) ms[i] = i < (int)P.level_ms.size() ? P.level_ms[i] : 0.0;
  if (flops) {
    for (int d = 0; d < L; ++d) flops[d] = 0.0;
    for (const auto& F : P.fronts)
      for (int32_t j = 0; j < F.p; ++j) {
        const double c = (double)(F.n - 1 - j);
        flops[F.depth] += 4.0 * c * c;
      }
  }
  if (small)
    for (int d = 0; d < L; ++d)
      small[d] = (d < (int)P.level_nmax.size() && stfem::level_is_small(P, d)) ? 1 : 0;
  return STFEM_OK;
}

extern "C" int stfem_plan_kernel_report(const stfem_plan* plan, int32_t nfam, double* ms, double* flops,
                                        int64_t* launches) {
  if (!plan) return stfem::fail(STFEM_ERR_ARG, "plan_kernel_report: null pointer");
  const Plan& P = *reinterpret_cast<const Plan*>(plan);
  const int nf = std::min<int>(nfam, stfem::NFAM);
  for (int i = 0; i < nf; ++i) {
    if (ms) ms[i] = i < (int)P.family_ms.size() ? P.family_ms[i] : 0.0;
    if (launches) launches[i] = i < (int)P.family_launches.size() ? P.family_launches[i] : 0;
    if (flops) flops[i] = 0.0;
  }
  if (flops) {
    // algorithmic real flops per shift of each family (1 RHS for the spectral RHS GEMMs)
    auto add = [&](int f, double v) {
      if (f < nf) flops[f] += v;
    };
    add(stfem::FAM_SPECTRAL, (double)P.spectral_flops_u + (double)P.spectral_flops_rhs);
    for (size_t d = 0; d < P.levels.size(); ++d) {
      const bool small = !P.level_nmax.empty() && stfem::level_is_small(P, (int)d);
      for (int32_t f : P.levels[d]) {
        const auto& F = P.fronts[f];
        const double n = F.n, p = F.p, b = F.n - F.p;
        if (small) {
          for (int j = 0; j < F.p; ++j) add(stfem::FAM_SMALL, 4.0 * (n - 1 - j) * (n - 1 - j));
          continue;
        }
        add(stfem::FAM_SYRK, 4.0 * b * b * p);
        for (int kb = 0; kb < F.p; kb += stfem::NB) {
          const double w = std::min(stfem::NB, F.p - kb), rows = n - kb - w;
          add(stfem::FAM_DIAG, 4.0 * w * w * w / 3.0);
          add(stfem::FAM_TRSM, 4.0 * rows * w * w);
          const double base = kb + w;
          if (base < p) add(stfem::FAM_PANEL, 8.0 * w * ((p - base) * (n - base) - (p - base) * (p - base - 1) / 2));
        }
      }
    }
  }
  return STFEM_OK;
}

extern "C" int stfem_plan_max_rhs(const stfem_plan* plan, int32_t* max_rhs) {
  if (!plan || !max_rhs) return stfem::fail(STFEM_ERR_ARG, "plan_max_rhs: null pointer");
  const Plan& P = *reinterpret_cast<const Plan*>(plan);
  *max_rhs = (int32_t)std::min<int64_t>(stfem::MAXR, stfem::BWD_XS_MAX / (16 * std::max(1, P.max_front)));
  return STFEM_OK;
}

extern "C" int stfem_plan_last_batches(const stfem_plan* plan, int32_t* batches) {
  if (!plan || !batches) return stfem::fail(STFEM_ERR_ARG, "plan_last_batches: null pointer");
  *batches = reinterpret_cast<const Plan*>(plan)->last_nbatches;
  return STFEM_OK;
}

extern "C" int stfem_plan_last_launches(const stfem_plan* plan, int64_t* launches) {
  if (!plan || !launches) return stfem::fail(STFEM_ERR_ARG, "plan_last_launches: null pointer");
  *launches = reinterpret_cast<const Plan*>(plan)->last_launches;
  return STFEM_OK;
}

extern "C" int stfem_plan_check(stfem_plan* plan, void* stream) {
  if (!plan) return stfem::fail(STFEM_ERR_ARG, "plan_check: null plan");
  return stfem::plan_check(*reinterpret_cast<Plan*>(plan), (cudaStream_t)stream);
}

// G and W of the following factor_solve calls are indexed in the plan's numbering (new = iperm[old])
// instead of the operators' -- the FD solver lets the time transforms apply the permutation
// (stfem_transform_pair_fwd_map / _back_map with the map from stfem_plan_device_iperm)
extern "C" int stfem_plan_set_io_permuted(stfem_plan* plan, int32_t on) {
  if (!plan) return stfem::fail(STFEM_ERR_ARG, "plan_set_io_permuted: null plan");
  reinterpret_cast<Plan*>(plan)->io_permuted = on != 0;
  return STFEM_OK;
}

extern "C" int stfem_plan_device_iperm(stfem_plan* plan, const int32_t** iperm) {
  if (!plan || !iperm) return stfem::fail(STFEM_ERR_ARG, "plan_device_iperm: null pointer");
  Plan& P = *reinterpret_cast<Plan*>(plan);
  int rc = stfem::upload_tables(P);
  if (rc) return rc;
  *iperm = P.d_iperm;
  return STFEM_OK;
}

extern "C" int stfem_plan_set_shift_base(stfem_plan* plan, int32_t base) {
  if (!plan) return stfem::fail(STFEM_ERR_ARG, "plan_set_shift_base: null plan");
  reinterpret_cast<Plan*>(plan)->shift_base = base;
  return STFEM_OK;
}

extern "C" int stfem_plan_reserve(stfem_plan* plan, int32_t nshift, int32_t nrhs) {
  if (!plan) return stfem::fail(STFEM_ERR_ARG, "plan_reserve: null plan");
  if (nshift < 1 || nrhs < 1 || nrhs > stfem::MAXR)
    return stfem::fail(STFEM_ERR_DIM, "plan_reserve: nshift >= 1 and 1 <= nrhs <= 16 required");
  return stfem::plan_reserve(*reinterpret_cast<Plan*>(plan), nshift, nrhs);
}

extern "C" int stfem_plan_get_options(const stfem_plan* plan, stfem_plan_options* out) {
  if (!plan || !out) return stfem::fail(STFEM_ERR_ARG, "plan_get_options: null pointer");
  *out = reinterpret_cast<const Plan*>(plan)->opt;
  return STFEM_OK;
}

extern "C" int stfem_plan_set_options(stfem_plan* plan, const stfem_plan_options* opt) {
  if (!plan || !opt) return stfem::fail(STFEM_ERR_ARG, "plan_set_options: null pointer");
  if (opt->panel_group < 1 || opt->small_front_n < 0 || !(opt->workspace_fraction > 0.0) ||
      opt->workspace_fraction > 1.0 || !(opt->pivot_tol >= 0.0))
    return stfem::fail(STFEM_ERR_ARG, "plan_set_options: value out of range");
  Plan& P = *reinterpret_cast<Plan*>(plan);
  P.opt = *opt;
  P.free_device();   // level classification and tile tables depend on the options
  return STFEM_OK;
}

extern "C" int stfem_plan_set_batch(stfem_plan* plan, int32_t batch, int64_t* bps) {
  if (!plan) return stfem::fail(STFEM_ERR_ARG, "plan_set_batch: null pointer");
  Plan& P = *reinterpret_cast<Plan*>(plan);
  P.batch = std::max(0, batch);
  if (bps) *bps = stfem::bytes_per_shift(P, 1);
  return STFEM_OK;
}

extern "C" int stfem_factor_solve(stfem_plan* plan, const double* Mvals, const double* Avals,
                                  const void* lam, int32_t nshift, int32_t nrhs, const void* G, void* W,
                                  stfem_bv_layout layout, void* stream) {
  if (!plan) return stfem::fail(STFEM_ERR_ARG, "factor_solve: null plan");
  return stfem::factor_solve(*reinterpret_cast<Plan*>(plan), Mvals, Avals, (const stfem::cplx*)lam, nshift,
                             nrhs, (const stfem::cplx*)G, (stfem::cplx*)W, layout, (cudaStream_t)stream);
}
