// K3 — time-axis transform (FD steps 2 and 4):
//   out[b][l][j] = sum_k T[l][k] * in[b][k][j]      complex128
//
// A complex-fp64 GEMM (M = K = n_t, N = n_x * n_rhs) on the FP64 tensor pipe:
// mma.sync.m16n8k4.f64 (SASS DMMA) with the 4-real-product complex scheme
//   Cre += Tre*Bre + (-Tim)*Bim ,  Cim += Tre*Bim + Tim*Bre
// Operand tiles are staged global->shared with 16-byte cp.async (one complex
// per copy) in a 3-stage pipeline.  CTA tile 64(l) x 64(j) complex, k-tile 16,
// 8 warps as 2 x 4, warp tile 32 x 16 complex (2 x 2 DMMA tiles, separate
// re/im accumulators: 32 fp64 registers per thread).
//
// Grid: x = M-tiles (fastest) so the n_t/64 CTAs that read the same column
// block of `in` run together and share it through L2 (in is read from HBM
// once; T (<= 16 MB) stays L2-resident).
#include "common.cuh"

#include <algorithm>

namespace stfem {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, STAGES = 3;
constexpr int LDA = BK + 4;   // As[m][k]: (g*LDA + t) mod 8 distinct -> conflict-free LDS.128
constexpr int LDB = BN + 2;   // Bs[k][n]: (t*LDB + g) mod 8 distinct
constexpr int A_STAGE = BM * LDA;
constexpr int B_STAGE = BK * LDB;
constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * 16;

// (Operand tiles by 1-D bulk copies, as in transform_rc_kernel<EPI, true> below, were measured on
// this kernel too: C4 64.0 ms against 62.4 ms with cp.async -- four DMMAs per fragment pair leave
// the mbarrier wait of every k tile less slack.  Not kept here.)
__global__ void __launch_bounds__(256, 2)
time_transform_kernel(const cplx* __restrict__ T, int nt, const cplx* __restrict__ in,
                      int64_t ld_in, cplx* __restrict__ out, int64_t ld_out, int64_t ncols,
                      int64_t bs_in, int64_t bs_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* As = reinterpret_cast<cplx*>(smem_raw);
  cplx* Bs = As + STAGES * A_STAGE;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  const int l0 = blockIdx.x * BM;
  const int64_t j0 = (int64_t)blockIdx.y * BN;
  in += (int64_t)blockIdx.z * bs_in;
  out += (int64_t)blockIdx.z * bs_out;

  const int nk = (nt + BK - 1) / BK;

  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * BK;
    cplx* as = As + stage * A_STAGE;
    cplx* bs = Bs + stage * B_STAGE;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int idx = tid + 256 * r;
      int m = idx >> 4, k = idx & 15;
      bool ok = (l0 + m < nt) && (k0 + k < nt);
      const cplx* src = ok ? T + (int64_t)(l0 + m) * nt + (k0 + k) : T;
      cp_async16(as + m * LDA + k, src, ok);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int idx = tid + 256 * r;
      int k = idx >> 6, n = idx & 63;
      bool ok = (k0 + k < nt) && (j0 + n < ncols);
      const cplx* src = ok ? in + (int64_t)(k0 + k) * ld_in + (j0 + n) : in;
      cp_async16(bs + k * LDB + n, src, ok);
    }
  };

  double cre[2][2][4], cim[2][2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) cre[i][j][v] = cim[i][j][v] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }

  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nxt = kt + STAGES - 1;
      if (nxt < nk) load_stage(nxt % STAGES, nxt);
      cp_async_commit();
    }
    const cplx* as = As + (kt % STAGES) * A_STAGE + (wm * 32 + g) * LDA + t;
    const cplx* bs = Bs + (kt % STAGES) * B_STAGE + t * LDB + wn * 16 + g;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      cplx a[2][2], b[2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        a[mi][0] = ldc(as + (mi * 16) * LDA + kk);
        a[mi][1] = ldc(as + (mi * 16 + 8) * LDA + kk);
      }
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) b[ni] = ldc(bs + kk * LDB + ni * 8);
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          dmma_16x8x4(cre[mi][ni], a[mi][0].re, a[mi][1].re, b[ni].re);
          dmma_16x8x4(cre[mi][ni], -a[mi][0].im, -a[mi][1].im, b[ni].im);
          dmma_16x8x4(cim[mi][ni], a[mi][0].re, a[mi][1].re, b[ni].im);
          dmma_16x8x4(cim[mi][ni], a[mi][0].im, a[mi][1].im, b[ni].re);
        }
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int row = l0 + wm * 32 + mi * 16 + g + 8 * h;
        int64_t col = j0 + wn * 16 + ni * 8 + 2 * t;
        if (row < nt) {
          cplx* dst = out + (int64_t)row * ld_out + col;
          if (col < ncols) stc(dst, cmk(cre[mi][ni][2 * h], cim[mi][ni][2 * h]));
          if (col + 1 < ncols) stc(dst + 1, cmk(cre[mi][ni][2 * h + 1], cim[mi][ni][2 * h + 1]));
        }
      }
}

// ---------------------------------------------------------------------------
// K3p — eigenpair-paired transforms (host side and derivation:
// paper_2504_07269_b200/paired_transform.py).  Both FD transforms become a
// REAL (M x K) x COMPLEX (K x N) product on DMMA: 2 real DMMAs (re, im) per
// real A fragment, half the work of the 4-product complex GEMM above.
//   EPI_PAIR  (forward G = Y F): A rows in blocks of 16 = [Re y of 8 sources;
//             Im y of the same 8], so one accumulator fragment holds u = c F
//             (row g) and v = d F (row g + 8) of source s; the epilogue writes
//             G_l = u + i v and G_p = s_p (u - i v).
//   EPI_PLAIN (back Psi = A W' after pair_mix_kernel): plain store.
// CTA tile 64 rows x 64 complex columns, k-tile 16, 3-stage cp.async, 8 warps
// as 2 x 4, warp tile 32 rows x 16 complex (2 x 2 fragments x re/im).
// A arrives PACKED from the host: A[mb][k][g][h] = A_logical[16 mb + g + 8 h][k], i.e. for
// every 16-row block and k the 8 (row g, row g + 8) pairs of one DMMA A fragment, so a
// thread fetches both fragment halves with one LDS.128 and the tile is a straight
// 16-byte cp.async copy.  Shared layout As[mb][k][20 doubles] (16 + 4 pad): the 32
// lanes' (t * 160 + 16 g) byte offsets cover 8 distinct 16-byte slots of each 128 B.
constexpr int RC_KS = 20;
// k-tile 16 in 3 stages (measured: a 32-deep tile in 2 stages, for half the barriers per
// DMMA, ran 33.7 vs 33.2 ms on C4)
constexpr int RC_BK = 16, RC_STAGES = 3;
constexpr int RC_A_STAGE = (BM / 16) * RC_BK * RC_KS;
constexpr int RC_B_STAGE = RC_BK * LDB;
constexpr int RC_SMEM = RC_STAGES * (RC_A_STAGE * 8 + RC_B_STAGE * 16);
enum { EPI_PLAIN = 0, EPI_PAIR = 1 };

// TMA: the operand tile's 16 rows of 64 contiguous complex columns arrive as 1-D bulk copies
// (cp.async.bulk, the TMA engine: one 1 KB row per lane of warp 0, completion counted in bytes on
// the stage's mbarrier) instead of 1024 16-byte cp.async issued by all 256 threads; used when the
// operand columns are not gathered through a map and K is a multiple of the k tile.  The packed A
// tile (its shared-memory rows are padded) stays on cp.async.  Measured neutral against the
// cp.async operand path (tools/prof_transform.py: C4 32.9 vs 32.7 ms, C5 221.7 vs 220.1 ms): the
// kernel is bound by DMMA issue (87-89% active), not by the copy instructions.
template <int EPI, bool TMA>
__global__ void __launch_bounds__(256, 2)
transform_rc_kernel(const double* __restrict__ A, int M, int K, const cplx* __restrict__ in, int64_t ld_in,
                    cplx* __restrict__ out, int64_t ld_out, int64_t ncols, int64_t bs_in, int64_t bs_out,
                    const int2* __restrict__ rows, const cplx* __restrict__ scale, int nsrc,
                    const int32_t* __restrict__ in_cols, const int32_t* __restrict__ out_cols) {
  // M: output rows (EPI_PLAIN) / A rows; A holds ceil(M / 16) packed 16-row blocks
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* As = reinterpret_cast<double*>(smem_raw);
  cplx* Bs = reinterpret_cast<cplx*>(As + RC_STAGES * RC_A_STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + RC_STAGES * RC_B_STAGE);   // TMA: one mbarrier per stage
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  const int m0 = blockIdx.x * BM;
  const int64_t j0 = (int64_t)blockIdx.y * BN;
  in += (int64_t)blockIdx.z * bs_in;
  out += (int64_t)blockIdx.z * bs_out;
  const int nk = (K + RC_BK - 1) / RC_BK;
  if constexpr (TMA) {
    if (tid == 0) {
      for (int s = 0; s < RC_STAGES; ++s) mbar_init(full + s, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
  }
  // TMA: bytes of one operand row of this column tile (the last tile of a launch may be partial:
  // its missing columns keep stale shared memory, and feed only accumulators that are never stored)
  const uint32_t row_bytes = (uint32_t)(16 * (ncols - j0 < BN ? ncols - j0 : (int64_t)BN));
  // Column maps (both optional): operand column j of this launch is read at column in_cols[j] of
  // `in`, result column j is written at column out_cols[j] of `out`.  The FD solve passes the
  // inverse nested-dissection permutation, so the spatial solves in between see G and W in
  // their own numbering (contiguous pivot rows) at no extra pass: the operand copies are 16-byte
  // cp.async per element either way, and the kernel is DMMA bound.  A thread's operand column
  // is the same for every k tile (tid & 63).
  const int64_t bcol = j0 + (tid & 63);
  const int64_t bsrc = (in_cols && bcol < ncols) ? (int64_t)in_cols[bcol] : bcol;

  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * RC_BK;
    double* as = As + stage * RC_A_STAGE;
    cplx* bs = Bs + stage * RC_B_STAGE;
    const int mblks = (M + 15) >> 4;
#pragma unroll
    for (int r = 0; r < RC_BK / 8; ++r) {   // 4 row blocks x RC_BK k x 8 fragment pairs (16-byte chunks)
      const int idx = tid + 256 * r;
      const int mb = idx / (RC_BK * 8), k = (idx >> 3) % RC_BK, gg = idx & 7;
      const int gmb = (m0 >> 4) + mb;
      const bool ok = (gmb < mblks) && (k0 + k < K);
      cp_async16(as + (mb * RC_BK + k) * RC_KS + 2 * gg, ok ? A + ((int64_t)gmb * K + (k0 + k)) * 16 + 2 * gg : A, ok);
    }
    if constexpr (TMA) {
      if (warp == 0) {
        if (lane == 0) mbar_arrive_expect_tx(full + stage, RC_BK * row_bytes);
        __syncwarp();
        if (lane < RC_BK) bulk_g2s(bs + lane * LDB, in + (int64_t)(k0 + lane) * ld_in + j0, row_bytes, full + stage);
      }
    } else {
#pragma unroll
      for (int r = 0; r < RC_BK / 4; ++r) {
        const int idx = tid + 256 * r;
        const int k = idx >> 6, n = idx & 63;
        const bool ok = (k0 + k < K) && (j0 + n < ncols);
        cp_async16(bs + k * LDB + n, ok ? in + (int64_t)(k0 + k) * ld_in + bsrc : in, ok);
      }
    }
  };

  double cre[2][2][4], cim[2][2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) cre[i][j][v] = cim[i][j][v] = 0.0;

#pragma unroll
  for (int s = 0; s < RC_STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<RC_STAGES - 2>();
    if constexpr (TMA) mbar_wait(full + kt % RC_STAGES, (kt / RC_STAGES) & 1);
    __syncthreads();
    {
      const int nxt = kt + RC_STAGES - 1;
      if (nxt < nk) load_stage(nxt % RC_STAGES, nxt);
      cp_async_commit();
    }
    const double* as = As + (kt % RC_STAGES) * RC_A_STAGE + ((wm * 2) * RC_BK + t) * RC_KS + 2 * g;
    const cplx* bs = Bs + (kt % RC_STAGES) * RC_B_STAGE + t * LDB + wn * 16 + g;
#pragma unroll
    for (int kk = 0; kk < RC_BK; kk += 4) {
      double a[2][2];
      cplx b[2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const cplx pr = ldc(reinterpret_cast<const cplx*>(as + (mi * RC_BK + kk) * RC_KS));   // rows g, g + 8
        a[mi][0] = pr.re;
        a[mi][1] = pr.im;
      }
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) b[ni] = ldc(bs + kk * LDB + ni * 8);
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          dmma_16x8x4(cre[mi][ni], a[mi][0], a[mi][1], b[ni].re);
          dmma_16x8x4(cim[mi][ni], a[mi][0], a[mi][1], b[ni].im);
        }
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const int64_t col = j0 + wn * 16 + ni * 8 + 2 * t;
      if constexpr (EPI == EPI_PAIR) {
        const int src = ((m0 + wm * 32 + mi * 16) >> 4) * 8 + g;
        if (src >= nsrc) continue;
        const int2 lp = rows[src];
        const cplx sc = scale[src];
#pragma unroll
        for (int cv = 0; cv < 2; ++cv) {
          if (col + cv >= ncols) continue;
          const int64_t oc = out_cols ? (int64_t)out_cols[col + cv] : col + cv;
          const cplx u = cmk(cre[mi][ni][cv], cim[mi][ni][cv]);        // c F
          const cplx v = cmk(cre[mi][ni][2 + cv], cim[mi][ni][2 + cv]);  // d F
          stc(out + (int64_t)lp.x * ld_out + oc, cmk(u.re - v.im, u.im + v.re));
          if (lp.y >= 0) stc(out + (int64_t)lp.y * ld_out + oc, cmul(sc, cmk(u.re + v.im, u.im - v.re)));
        }
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = m0 + wm * 32 + mi * 16 + g + 8 * h;
          if (row >= M) continue;
          cplx* dst = out + (int64_t)row * ld_out;
          if (col < ncols) stc(dst + (out_cols ? (int64_t)out_cols[col] : col), cmk(cre[mi][ni][2 * h], cim[mi][ni][2 * h]));
          if (col + 1 < ncols)
            stc(dst + (out_cols ? (int64_t)out_cols[col + 1] : col + 1), cmk(cre[mi][ni][2 * h + 1], cim[mi][ni][2 * h + 1]));
        }
      }
    }
}

// In-place pre-pass of the paired back transform: for every pair (l, p)
// [W_l; W_p] <- [[m00, m01], [m10, m11]] [W_l; W_p]; self-paired (p < 0):
// W_l <- m00 W_l.  Columns fastest (coalesced), one pair per grid row.
__global__ void pair_mix_kernel(cplx* __restrict__ W, int64_t ld, int64_t ncols, int64_t bs,
                                const int2* __restrict__ rows, const cplx* __restrict__ coef) {
  const int q = blockIdx.y;
  const int2 lp = rows[q];
  const cplx m00 = coef[4 * q], m01 = coef[4 * q + 1], m10 = coef[4 * q + 2], m11 = coef[4 * q + 3];
  cplx* wl = W + (int64_t)blockIdx.z * bs + (int64_t)lp.x * ld;
  cplx* wp = W + (int64_t)blockIdx.z * bs + (int64_t)lp.y * ld;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < ncols; j += (int64_t)gridDim.x * blockDim.x) {
    const cplx u = ldc(wl + j);
    if (lp.y >= 0) {
      const cplx v = ldc(wp + j);
      stc(wl + j, cadd(cmul(m00, u), cmul(m01, v)));
      stc(wp + j, cadd(cmul(m10, u), cmul(m11, v)));
    } else {
      stc(wl + j, cmul(m00, u));
    }
  }
}

template <int EPI>
int launch_rc(const double* A, int M, int K, const cplx* in, int64_t ld_in, cplx* out, int64_t ld_out,
              int64_t ncols, int batch, int64_t bs_in, int64_t bs_out, const int2* rows, const cplx* scale,
              int nsrc, const int32_t* in_cols, const int32_t* out_cols, cudaStream_t stream) {
  static DeviceOnce attr_once;
  if (attr_once.first()) {
    STFEM_CUDA_TRY(cudaFuncSetAttribute(transform_rc_kernel<EPI, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        RC_SMEM + RC_STAGES * 8));
    STFEM_CUDA_TRY(cudaFuncSetAttribute(transform_rc_kernel<EPI, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        RC_SMEM));
  }
  for (int64_t c0 = 0; c0 < ncols; c0 += 65535LL * BN) {
    const int64_t cn = ncols - c0 < 65535LL * BN ? ncols - c0 : 65535LL * BN;
    dim3 grid((M + BM - 1) / BM, (unsigned)((cn + BN - 1) / BN), batch);
    // a mapped side keeps its base pointer: the map holds absolute columns
    if (!in_cols && K % RC_BK == 0)
      transform_rc_kernel<EPI, true><<<grid, 256, RC_SMEM + RC_STAGES * 8, stream>>>(
          A, M, K, in + c0, ld_in, out_cols ? out : out + c0, ld_out, cn, bs_in, bs_out, rows, scale, nsrc, nullptr,
          out_cols ? out_cols + c0 : nullptr);
    else
      transform_rc_kernel<EPI, false><<<grid, 256, RC_SMEM, stream>>>(A, M, K, in_cols ? in : in + c0, ld_in,
                                                                      out_cols ? out : out + c0, ld_out, cn, bs_in, bs_out,
                                                                      rows, scale, nsrc, in_cols ? in_cols + c0 : nullptr,
                                                                      out_cols ? out_cols + c0 : nullptr);
    STFEM_LAUNCH_CHECK("transform_rc_kernel");
  }
  return STFEM_OK;
}

}  // namespace

int time_transform(const void* T, int nt, const void* in, int64_t ld_in, void* out,
                   int64_t ld_out, int64_t ncols, int batch, int64_t bs_in, int64_t bs_out,
                   cudaStream_t stream) {
  if (nt <= 0 || ncols < 0 || batch < 0 || ld_in < ncols || ld_out < ncols)
    return fail(STFEM_ERR_DIM, "time_transform: bad dimensions");
  if (!T || !in || !out) return fail(STFEM_ERR_ARG, "time_transform: null pointer");
  if (((uintptr_t)T | (uintptr_t)in | (uintptr_t)out) & 15)
    return fail(STFEM_ERR_ARG, "time_transform: buffers must be 16-byte aligned");
  if (ncols == 0 || batch == 0) return STFEM_OK;
  static DeviceOnce attr_once;
  if (attr_once.first()) {
    STFEM_CUDA_TRY(cudaFuncSetAttribute(time_transform_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
  }
  int64_t ntile = (ncols + BN - 1) / BN;
  if (ntile > 65535) {
    // split the column range into chunks of <= 65535 tiles
    for (int64_t c0 = 0; c0 < ncols; c0 += 65535LL * BN) {
      int64_t cn = ncols - c0 < 65535LL * BN ? ncols - c0 : 65535LL * BN;
      int rc = time_transform(T, nt, (const cplx*)in + c0, ld_in, (cplx*)out + c0, ld_out, cn,
                              batch, bs_in, bs_out, stream);
      if (rc) return rc;
    }
    return STFEM_OK;
  }
  dim3 grid((nt + BM - 1) / BM, (unsigned)ntile, batch);
  time_transform_kernel<<<grid, 256, SMEM_BYTES, stream>>>(
      (const cplx*)T, nt, (const cplx*)in, ld_in, (cplx*)out, ld_out, ncols, bs_in, bs_out);
  STFEM_LAUNCH_CHECK("time_transform_kernel");
  return STFEM_OK;
}

}  // namespace stfem

extern "C" int stfem_time_transform(const void* T, int nt, const void* in, int64_t ld_in,
                                    void* out, int64_t ld_out, int64_t ncols, int batch,
                                    int64_t bstride_in, int64_t bstride_out, void* stream) {
  return stfem::time_transform(T, nt, in, ld_in, out, ld_out, ncols, batch, bstride_in,
                               bstride_out, (cudaStream_t)stream);
}

extern "C" int stfem_transform_pair_fwd_map(const double* A, int mrows, int nt, const int32_t* rows,
                                            const void* scale, int nsrc, const void* in, int64_t ld_in, void* out,
                                            int64_t ld_out, int64_t ncols, int batch, int64_t bstride_in,
                                            int64_t bstride_out, const int32_t* out_cols, void* stream) {
  using namespace stfem;
  if (nt <= 0 || (nt & 1) || mrows <= 0 || (mrows & 15) || nsrc <= 0 || 2 * nsrc > mrows + 16 || ncols < 0 ||
      batch < 0 || ld_in < ncols || (!out_cols && ld_out < ncols))
    return fail(STFEM_ERR_DIM, "transform_pair_fwd: bad dimensions");
  if (!A || !rows || !scale || !in || !out) return fail(STFEM_ERR_ARG, "transform_pair_fwd: null pointer");
  if (((uintptr_t)A | (uintptr_t)in | (uintptr_t)out) & 15)
    return fail(STFEM_ERR_ARG, "transform_pair_fwd: buffers must be 16-byte aligned");
  if (ncols == 0 || batch == 0) return STFEM_OK;
  return launch_rc<EPI_PAIR>(A, mrows, nt, (const cplx*)in, ld_in, (cplx*)out, ld_out, ncols, batch, bstride_in,
                             bstride_out, (const int2*)rows, (const cplx*)scale, nsrc, nullptr, out_cols,
                             (cudaStream_t)stream);
}

extern "C" int stfem_transform_pair_fwd(const double* A, int mrows, int nt, const int32_t* rows,
                                        const void* scale, int nsrc, const void* in, int64_t ld_in, void* out,
                                        int64_t ld_out, int64_t ncols, int batch, int64_t bstride_in,
                                        int64_t bstride_out, void* stream) {
  return stfem_transform_pair_fwd_map(A, mrows, nt, rows, scale, nsrc, in, ld_in, out, ld_out, ncols, batch,
                                      bstride_in, bstride_out, nullptr, stream);
}

// in-place pre-pass of the paired back transform over `ncols` columns of W (all of them, before any
// column block is transformed, when the transform gathers its operand columns through a map)
extern "C" int stfem_pair_mix(const int32_t* mix_rows, const void* mix_coef, int nmix, void* W, int64_t ld,
                              int64_t ncols, int batch, int64_t bstride, void* stream) {
  using namespace stfem;
  if (nmix <= 0 || ncols < 0 || batch < 0 || ld < ncols) return fail(STFEM_ERR_DIM, "pair_mix: bad dimensions");
  if (!mix_rows || !mix_coef || !W) return fail(STFEM_ERR_ARG, "pair_mix: null pointer");
  if (ncols == 0 || batch == 0) return STFEM_OK;
  const int64_t gx = std::min<int64_t>((ncols + 255) / 256, 1024);
  pair_mix_kernel<<<dim3((unsigned)gx, nmix, batch), 256, 0, (cudaStream_t)stream>>>(
      (cplx*)W, ld, ncols, bstride, (const int2*)mix_rows, (const cplx*)mix_coef);
  STFEM_LAUNCH_CHECK("pair_mix_kernel");
  return STFEM_OK;
}

// nmix = 0: the pre-pass has been run already (stfem_pair_mix); in_cols (optional): result column j
// reads operand column in_cols[j] of `in`
extern "C" int stfem_transform_pair_back_map(const double* A, int nt, const int32_t* mix_rows, const void* mix_coef,
                                             int nmix, void* in, int64_t ld_in, void* out, int64_t ld_out,
                                             int64_t ncols, int batch, int64_t bstride_in, int64_t bstride_out,
                                             const int32_t* in_cols, void* stream) {
  using namespace stfem;
  if (nt <= 0 || (nt & 1) || nmix < 0 || nmix > nt || ncols < 0 || batch < 0 || (!in_cols && ld_in < ncols) ||
      ld_out < ncols)
    return fail(STFEM_ERR_DIM, "transform_pair_back: bad dimensions");
  if (!A || !in || !out || (nmix > 0 && (!mix_rows || !mix_coef)))
    return fail(STFEM_ERR_ARG, "transform_pair_back: null pointer");
  if (nmix > 0 && in_cols)
    return fail(STFEM_ERR_ARG, "transform_pair_back: with a column map run stfem_pair_mix over all of W first");
  if (((uintptr_t)A | (uintptr_t)in | (uintptr_t)out) & 15)
    return fail(STFEM_ERR_ARG, "transform_pair_back: buffers must be 16-byte aligned");
  if (in == out) return fail(STFEM_ERR_ARG, "transform_pair_back: in and out must not alias");
  if (ncols == 0 || batch == 0) return STFEM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (nmix > 0) {
    int rc = stfem_pair_mix(mix_rows, mix_coef, nmix, in, ld_in, ncols, batch, bstride_in, stream);
    if (rc) return rc;
  }
  return launch_rc<EPI_PLAIN>(A, nt, nt, (const cplx*)in, ld_in, (cplx*)out, ld_out, ncols, batch, bstride_in,
                              bstride_out, nullptr, nullptr, 0, in_cols, nullptr, st);
}

extern "C" int stfem_transform_pair_back(const double* A, int nt, const int32_t* mix_rows, const void* mix_coef,
                                         int nmix, void* in, int64_t ld_in, void* out, int64_t ld_out,
                                         int64_t ncols, int batch, int64_t bstride_in, int64_t bstride_out,
                                         void* stream) {
  if (nmix <= 0) return stfem::fail(STFEM_ERR_DIM, "transform_pair_back: bad dimensions");
  return stfem_transform_pair_back_map(A, nt, mix_rows, mix_coef, nmix, in, ld_in, out, ld_out, ncols, batch,
                                       bstride_in, bstride_out, nullptr, stream);
}
