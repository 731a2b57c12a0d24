// Spectral subtree elimination (included by multifrontal.cu inside its
// anonymous namespace; uses FrontDev/SubDev/bv_off/cplx helpers).
//
// The bottom of the elimination tree is where the multifrontal method is
// latency bound: millions of tiny (front, shift) instances per batch.  But
// every shifted system has the form K(lam) = M + lam A with M, A real SPD,
// so a whole subtree can be eliminated in closed form.  For a subtree with
// interior DoFs I (all pivots of the subtree, contiguous in the plan's
// numbering) and boundary rows Gam (the subtree root's boundary rows):
//   A_II V = M_II V diag(theta)^{-1}...   precisely  V^T A_II V = I,
//   V^T M_II V = diag(theta)             (host setup, once per mesh)
//   K_II(lam)^{-1} = V diag(w) V^T,      w_k = 1 / (theta_k + lam)
//   K_GI(lam) V = P + lam Q = R + (theta + lam) Q,  P = M_GI V, Q = A_GI V,
//   R = P - Q diag(theta)
// so the root's update block (the Schur complement the parent assembles) is
//   U(lam) = -K_GI K_II^{-1} K_IG = -( R diag(w) R^T + C0 + lam C1 ),
//   C1 = Q Q^T,  C0 = R Q^T + Q R^T + Q diag(theta) Q^T,
// the forward RHS contribution to the boundary rows is
//   c = V^T g_I (kept in Z),   r_Gam = -( R (w o c) + Q c ),
// and the backward solve of the interior is
//   y = w o (c - R^T x_Gam) - Q^T x_Gam,   x_I = V y.
// Every per-shift operation is a real x complex GEMM with the shifts (x RHS)
// as the N dimension: all of it runs on the FP64 tensor pipe (DMMA) with no
// per-shift factor storage and no per-front latency chains.
//
// One kernel, five operand generators (ops), one 64 x 64(complex) CTA tile:
//   OP_U  : U(lam)   rows = (i, j) pairs of an 8x8 block, K = m, B = w(k, shift)
//   OP_F1 : c = V^T g_I           rows = k_out, K = m, B = G gathered through perm
//   OP_F2 : r_Gam                 rows = i,     K = 2m, B = [w o c ; c]
//   OP_B1 : y                     rows = 8 R^T rows + 8 Q^T rows per 16, K = gam, B = x_Gam
//   OP_B2 : x_I = V y             rows = i,     K = m, B = y
// Register-prefetched double-buffered staging (operands are generated, not
// copied), 8 warps as 2 (M) x 4 (N), warp tile 32 x 16 complex,
// mma.sync.m16n8k4.f64: two DMMAs (re, im) per real A fragment.
#pragma once

constexpr int SP_BM = 64, SP_BN = 64, SP_BK = 16;
constexpr int SP_LDA = SP_BM + 4;   // As[k][row] doubles: (t*68 + g) mod 16 hits each bank pair twice
constexpr int SP_LDB = SP_BN + 2;   // Bs[k][col] complex: (t*66 + g) mod 8 hits each 16-B bank group 4x
constexpr int SP_A_STAGE = SP_BK * SP_LDA;   // doubles
constexpr int SP_B_STAGE = SP_BK * SP_LDB;   // complex
constexpr int SP_PF = 2;       // chunks ahead of the register prefetch that F2 / B2 pull their Z lines into L2
constexpr int SP_STAGES = 3;   // cp.async ring of the plain-copy ops (F1, B1); U, F2 and B2 use two
constexpr int SP_SMEM = SP_STAGES * (SP_A_STAGE * 8 + SP_B_STAGE * 16);
// + OP_U staging: the tile's 16 R rows over the subtree's m
__host__ __device__ constexpr int spectral_smem_bytes(int mmax) { return SP_SMEM + 4 * ((mmax + 3) & ~3); }   // + the staged index table
enum { OP_U = 0, OP_F1 = 1, OP_F2 = 2, OP_B1 = 3, OP_B2 = 4, OP_B1R = 5 };
// OP_B1R: B1 of a whole subtree whose root has at most SP_B1R_K boundary rows, one CTA per column
// tile: x_Gam of the tile (K = gam rows x 64 columns, gathered through the boundary index table)
// is staged ONCE and stays resident while the CTA walks the subtree's row tiles, streaming only
// the R^T / Q^T tiles.  The per-tile B1 re-gathers x_Gam for each of its m / 32 row tiles and pays
// the index-table / gather / fill latency chain for 4 k chunks of work.
constexpr int SP_B1R_K = 64;
constexpr int SP_B1R_SMEM = SP_STAGES * SP_A_STAGE * 8 + (SP_B1R_K / SP_BK) * SP_B_STAGE * 16 + 4 * SP_B1R_K;

__device__ __forceinline__ cplx spec_w(double th, cplx l) { return crecip_fast(cmk(th + l.re, l.im)); }

struct SpecArgs {
  const SubDev* subs;
  const int4* items;          // (op, subtree, tile_a, tile_b)
  const double *V, *th, *RQ, *C01;
  const FrontDev* fronts;
  const int32_t *bidx, *perm;
  const cplx* lam;            // this batch's shifts
  int32_t nb, nrhs, nx, shift0;
  cplx* ucur;
  int64_t ucur_stride;
  cplx* rcur;
  int64_t rcur_stride;
  cplx* Z;
  const cplx* G;
  cplx* W;
  stfem_bv_layout lay;
  const cplx* wbuf;           // w[(tofs + k) * wstride + s] = 1 / (theta_k + lam_s), this lane's shifts
  int64_t wstride;
};

// w_k(s) = 1 / (theta_k + lam_s) for every subtree interior index k and shift s
// of the batch (shared by all row tiles of a subtree instead of recomputed)
// Pivot collapse: theta_k + lam_s are exactly the pivots of the
// subtree interior in the eigenbasis, so lam = -theta_k (an eigenvalue -mu of
// the subtree's (M_II, A_II) pencil) is reported like a vanishing LDL^T pivot:
// |theta_k + lam|^2 <= tol^2 (|theta_k| + |lam|)^2 latches shift0 + s + 1 in err.
__global__ void spectral_w_kernel(const double* __restrict__ th, int64_t nth, const cplx* __restrict__ lam,
                                  int nb, cplx* __restrict__ w, int64_t wstride, double tol2, int* err,
                                  int shift0) {
  const int64_t tot = nth * nb;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < tot;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = idx / nb;
    const int s = (int)(idx - k * nb);
    const double t = th[k];
    const cplx l = lam[s];
    const double dr = t + l.re, d2 = fma(dr, dr, l.im * l.im);
    const double sc = fabs(t) + sqrt(cabs2(l));
    if (!(d2 > tol2 * sc * sc) || !isfinite(d2)) atomicCAS(err, 0, shift0 + s + 1);
    stc(w + k * wstride + s, spec_w(t, l));
  }
}

template <int OP>
__device__ __forceinline__ void spectral_tile(const SpecArgs& a, const int4 it, double* As, cplx* Bs) {
  const SubDev S = a.subs[it.y];
  const FrontDev F = a.fronts[S.front];
  const int m = S.m, g = S.g, nrhs = a.nrhs, nx = a.nx;
  const int ncols = OP == OP_U ? a.nb : a.nb * nrhs;
  const int n0 = blockIdx.y * SP_BN;
  if (n0 >= ncols) return;
  const int K = OP == OP_F2 ? 2 * m : OP == OP_B1 ? g : m;
  const double* __restrict__ V = a.V + S.vofs;
  const double* __restrict__ Rm = a.RQ + S.rqofs;
  const double* __restrict__ Qm = Rm + (int64_t)g * m;
  const int32_t* __restrict__ bidx = a.bidx + F.bidx_beg;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3, wm = warp & 1, wn = warp >> 1;
  const cplx zero = cmk(0.0, 0.0);

  // OP_U operands R_ik R_jk are formed from the class's R (column-major, L2-resident: one copy
  // per class of congruent subtrees) -- two loads per A element; nothing of size m is staged, so
  // the subtree size does not limit the CTAs per SM
  const cplx* __restrict__ wsub = a.wbuf + (int64_t)S.tofs * a.wstride;   // w[k * wstride + s]
  // OP_F1 / OP_B1 gather their B operand through an index table (the permutation of the subtree's
  // interior DoFs / the root's boundary rows).  Staged once per tile: the per-chunk fetch is then
  // one global load deep instead of two dependent ones (ncu: the index loads were 23% of all
  // stall samples of the F1 launch, long scoreboard)
  int* idx_s = reinterpret_cast<int*>(Bs + SP_STAGES * SP_B_STAGE);
  if constexpr (OP == OP_F1 || OP == OP_B1) {
    const int cnt = OP == OP_F1 ? m : g;
    for (int q = tid; q < cnt; q += 256) idx_s[q] = OP == OP_F1 ? (a.perm ? a.perm[S.first + q] : S.first + q) : bidx[q];
    __syncthreads();
  }

  // ---- operand generators ----
  auto a_val = [&](int r, int k) -> double {
    if (k >= K) return 0.0;
    if (OP == OP_U) {
      const int i = it.z * 8 + (r >> 3), j = it.w * 8 + (r & 7);
      return (i < g && j < g) ? Rm[i + (int64_t)k * g] * Rm[j + (int64_t)k * g] : 0.0;
    } else if (OP == OP_F1) {
      const int ko = it.z * SP_BM + r;
      return ko < m ? V[k + (int64_t)ko * m] : 0.0;
    } else if (OP == OP_F2) {
      const int i = it.z * SP_BM + r;
      if (i >= g) return 0.0;
      return k < m ? Rm[i + (int64_t)k * g] : Qm[i + (int64_t)(k - m) * g];
    } else if (OP == OP_B1) {
      const int kk = it.z * 32 + (r >> 4) * 8 + (r & 7);
      if (kk >= m) return 0.0;
      return ((r >> 3) & 1 ? Qm : Rm)[k + (int64_t)kk * g];
    } else {
      const int i = it.z * SP_BM + r;
      return i < m ? V[i + (int64_t)k * m] : 0.0;
    }
  };
  auto b_val = [&](int k, int c) -> cplx {
    const int cg = n0 + c;
    if (k >= K || cg >= ncols) return zero;
    if (OP == OP_U) return ldc(wsub + (int64_t)k * a.wstride + cg);
    const int s = cg / nrhs, r = cg - s * nrhs;
    const cplx* Zs = a.Z + (int64_t)s * nx * nrhs + (int64_t)r * nx;
    if (OP == OP_F1) return ldc(a.G + bv_off(a.lay, r, a.shift0 + s, idx_s[k]));
    if (OP == OP_F2)
      return k < m ? cmul(ldc(wsub + (int64_t)k * a.wstride + s), ldc(Zs + S.first + k)) : ldc(Zs + S.first + k - m);
    if (OP == OP_B1) return ldc(Zs + idx_s[k]);
    return ldc(Zs + S.first + k);
  };

  // F2 / B2 (register path): a thread's four B elements of a chunk are row k0 + kq of the columns
  // bq + 16 u -- the same columns for every chunk, so their Z (and w) column pointers, with the
  // shift / RHS split of the column index, are formed once per tile
  const int kq = tid & 15;
  const cplx* zc[4] = {nullptr, nullptr, nullptr, nullptr};
  const cplx* wc[4] = {nullptr, nullptr, nullptr, nullptr};
  if constexpr (OP == OP_F2 || OP == OP_B2) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int cg = n0 + (tid >> 4) + 16 * u;
      if (cg < ncols) {
        const int s = cg / nrhs, r = cg - s * nrhs;
        zc[u] = a.Z + (int64_t)s * nx * nrhs + (int64_t)r * nx + S.first;
        wc[u] = wsub + s;
      }
    }
  }
  double ra[4];
  cplx rb[4];
  auto fetch = [&](int kc) {
    const int k0 = kc * SP_BK;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = tid + 256 * u;
      // OP_F1 reads rows of V^T (= columns of V, contiguous in k): k fastest
      if constexpr (OP == OP_F1) ra[u] = a_val(idx >> 4, k0 + (idx & 15));
      else ra[u] = a_val(idx & 63, k0 + (idx >> 6));
      if constexpr (OP == OP_U) {
        // w streamed straight into its shared-memory stage (16-byte cp.async, zero-filled
        // outside); the stage was last read before the previous iteration's barrier
        const int k = k0 + (idx >> 6), cg = n0 + (idx & 63);
        const bool ok = k < K && cg < ncols;
        cp_async16(Bs + (kc & 1) * SP_B_STAGE + (idx >> 6) * SP_LDB + (idx & 63),
                   ok ? wsub + (int64_t)k * a.wstride + cg : wsub, ok);
      } else if constexpr (OP == OP_F2 || OP == OP_B2) {
        // 16 consecutive lanes walk down k of one column (Z is contiguous in k: 256-byte runs
        // instead of 32 separate 16-byte pieces per warp)
        const int k = k0 + kq;
        // the register double buffer looks one chunk ahead; an L2 prefetch of the Z lines of the
        // chunk SP_PF further on covers the rest of the HBM latency (F2's second half re-reads
        // the lines of its first: no prefetch there)
        {
          const int kp = k + SP_PF * SP_BK;
          if (zc[u] != nullptr && kp < (OP == OP_B2 ? K : m) && (kq & 7) == 0)
            asm volatile("prefetch.global.L2 [%0];\n" ::"l"(zc[u] + kp));
        }
        if (zc[u] == nullptr || k >= K) rb[u] = zero;
        else if constexpr (OP == OP_B2) rb[u] = ldc(zc[u] + k);
        else rb[u] = k < m ? cmul(ldc(wc[u] + (int64_t)k * a.wstride), ldc(zc[u] + k)) : ldc(zc[u] + k - m);
      } else {
        rb[u] = b_val(k0 + (idx & 15), idx >> 4);
      }
    }
    if constexpr (OP == OP_U) cp_async_commit();
  };
  auto store = [&](int st) {
    double* as = As + st * SP_A_STAGE;
    cplx* bs = Bs + st * SP_B_STAGE;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = tid + 256 * u;
      if constexpr (OP == OP_F1) as[(idx & 15) * SP_LDA + (idx >> 4)] = ra[u];
      else as[(idx >> 6) * SP_LDA + (idx & 63)] = ra[u];
      if constexpr (OP != OP_U) stc(bs + (idx & 15) * SP_LDB + (idx >> 4), rb[u]);
    }
  };

  double acc[2][2][2][4];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[mi][ni][0][v] = acc[mi][ni][1][v] = 0.0;

  const int nk = (K + SP_BK - 1) / SP_BK;
  // the last column tile of a batch is partial (e.g. 342 shifts = 5 x 64 + 22): warps whose
  // 16 (or upper 8) columns are all past ncols skip their DMMAs (warp-uniform)
  const bool wact = n0 + wn * 16 < ncols, wact1 = n0 + wn * 16 + 8 < ncols;
  auto compute = [&](int st) {
    const double* as = As + st * SP_A_STAGE + tq * SP_LDA + wm * 32 + gq;
    const cplx* bs = Bs + st * SP_B_STAGE + tq * SP_LDB + wn * 16 + gq;
#pragma unroll
    for (int kk = 0; kk < SP_BK; kk += 4) {
      if (!wact) break;
      double af[2][2];
      cplx bf[2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        af[mi][0] = as[kk * SP_LDA + mi * 16];
        af[mi][1] = as[kk * SP_LDA + mi * 16 + 8];
      }
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) bf[ni] = ldc(bs + kk * SP_LDB + ni * 8);
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          if (ni == 1 && !wact1) continue;
          dmma_16x8x4(acc[mi][ni][0], af[mi][0], af[mi][1], bf[ni].re);
          dmma_16x8x4(acc[mi][ni][1], af[mi][0], af[mi][1], bf[ni].im);
        }
    }
  };
  if constexpr (OP == OP_F1 || OP == OP_B1) {
    // Plain-copy operands (matrix tiles of V / R / Q, vectors gathered through the staged index
    // table): a 3-stage cp.async ring, one barrier per K chunk, nothing staged through
    // registers.  The thread's B column is the same for every chunk: its base pointer (and
    // the shift / RHS split of the column) is formed once.  (Measured per batch, register
    // path -> ring: C4 F1 5.45 -> 5.61, B1 3.58 -> 3.69, B2 4.43 -> 5.43 ms; C5 (9 RHS) F1 11.4 ->
    // 10.0, B1 10.1 -> 8.9, B2 10.2 -> 10.0: B2 stays on the register path.)
    // B operand: 16 consecutive lanes walk down k of one column (contiguous in the plan's
    // numbering: 256-byte runs), a thread's four copies of a chunk are columns bq + 16 u
    const int kq = tid & 15, bq = tid >> 4;
    bool bcol_ok[4];
    int bs_[4], br[4];
    const cplx* bbase[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int bcg = n0 + bq + 16 * u;
      bcol_ok[u] = bcg < ncols;
      bs_[u] = bcol_ok[u] ? bcg / nrhs : 0;
      br[u] = bcol_ok[u] ? bcg - bs_[u] * nrhs : 0;
      bbase[u] = OP == OP_F1 ? a.G + bv_off(a.lay, br[u], a.shift0 + bs_[u], 0)
                             : a.Z + (int64_t)bs_[u] * nx * nrhs + (int64_t)br[u] * nx + (OP == OP_B2 ? S.first : 0);
    }
    const bool unchunked = a.lay.chunk_cols >= nx;
    auto issue = [&](int st, int kc) {
      const int k0 = kc * SP_BK;
      double* as = As + st * SP_A_STAGE;
      cplx* bs = Bs + st * SP_B_STAGE;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = tid + 256 * u;
        if constexpr (OP == OP_F1) {
          const int r = idx >> 4, k = k0 + (idx & 15), ko = it.z * SP_BM + r;
          const bool ok = ko < m && k < K;
          cp_async8(as + (idx & 15) * SP_LDA + r, ok ? V + k + (int64_t)ko * m : V, ok);
        } else if constexpr (OP == OP_B1) {
          // rows of R^T / Q^T = columns of R / Q, contiguous in k: k fastest (128-byte runs)
          const int r = idx >> 4, k = k0 + (idx & 15), kk = it.z * 32 + (r >> 4) * 8 + (r & 7);
          const bool ok = kk < m && k < K;
          cp_async8(as + (idx & 15) * SP_LDA + r, ok ? ((r >> 3) & 1 ? Qm : Rm) + k + (int64_t)kk * g : Rm, ok);
        } else {
          const int r = idx & 63, k = k0 + (idx >> 6), i = it.z * SP_BM + r;
          const bool ok = i < m && k < K;
          cp_async8(as + (idx >> 6) * SP_LDA + r, ok ? V + i + (int64_t)k * m : V, ok);
        }
        const int k = k0 + kq;
        const bool ok = bcol_ok[u] && k < K;
        const cplx* src = bbase[u];
        if (ok) {
          if constexpr (OP == OP_F1)
            src = unchunked ? bbase[u] + idx_s[k] : a.G + bv_off(a.lay, br[u], a.shift0 + bs_[u], idx_s[k]);
          else if constexpr (OP == OP_B1) src = bbase[u] + idx_s[k];
          else src = bbase[u] + k;
        }
        cp_async16(bs + kq * SP_LDB + bq + 16 * u, src, ok);
      }
    };
#pragma unroll
    for (int st = 0; st < SP_STAGES - 1; ++st) {
      if (st < nk) issue(st, st);
      cp_async_commit();
    }
    for (int kc = 0; kc < nk; ++kc) {
      cp_async_wait<SP_STAGES - 2>();
      __syncthreads();
      const int nxt = kc + SP_STAGES - 1;
      if (nxt < nk) issue(nxt % SP_STAGES, nxt);
      cp_async_commit();
      compute(kc % SP_STAGES);
    }
    cp_async_wait<0>();
  } else {
    if (nk > 0) {
      fetch(0);
      store(0);
    }
    if constexpr (OP == OP_U) cp_async_wait<0>();
    __syncthreads();
    for (int kc = 0; kc < nk; ++kc) {
      if (kc + 1 < nk) fetch(kc + 1);
      compute(kc & 1);
      if (kc + 1 < nk) store((kc + 1) & 1);
      if constexpr (OP == OP_U) cp_async_wait<0>();
      __syncthreads();
    }
  }

  // ---- epilogues ----
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const int rbase = wm * 32 + mi * 16 + gq;
#pragma unroll
      for (int cv = 0; cv < 2; ++cv) {
        const int cg = n0 + wn * 16 + ni * 8 + 2 * tq + cv;
        if (cg >= ncols) continue;
        if constexpr (OP == OP_B1) {
          // rows rbase (R^T x) and rbase + 8 (Q^T x) belong to the same interior index
          const int kk = it.z * 32 + (rbase >> 4) * 8 + (rbase & 7);
          if (kk >= m) continue;
          const int s = cg / nrhs, r = cg - s * nrhs;
          cplx* zp = a.Z + (int64_t)s * nx * nrhs + (int64_t)r * nx + S.first + kk;
          const cplx t1 = cmk(acc[mi][ni][0][cv], acc[mi][ni][1][cv]);
          const cplx t2 = cmk(acc[mi][ni][0][2 + cv], acc[mi][ni][1][2 + cv]);
          const cplx w = ldc(wsub + (int64_t)kk * a.wstride + s);
          stc(zp, csub(cmul(w, csub(ldc(zp), t1)), t2));
        } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = rbase + 8 * h;
          const cplx v = cmk(acc[mi][ni][0][2 * h + cv], acc[mi][ni][1][2 * h + cv]);
          if (OP == OP_U) {
            const int i = it.z * 8 + (row >> 3), j = it.w * 8 + (row & 7);
            if (i >= g || j > i) continue;
            const double* C0 = a.C01 + S.cofs;
            const double* C1 = C0 + (int64_t)g * g;
            const int64_t e = i + (int64_t)j * g;
            const cplx l = a.lam[cg];
            cplx* U = a.ucur + (int64_t)cg * a.ucur_stride + F.uofs;
            stc(U + i + (int64_t)j * ldu(g), cmk(-(v.re + C0[e] + l.re * C1[e]), -(v.im + l.im * C1[e])));
          } else if (OP == OP_F1) {
            const int ko = it.z * SP_BM + row;
            if (ko >= m) continue;
            const int s = cg / nrhs, r = cg - s * nrhs;
            stc(a.Z + (int64_t)s * nx * nrhs + (int64_t)r * nx + S.first + ko, v);
          } else if (OP == OP_F2) {
            const int i = it.z * SP_BM + row;
            if (i >= g) continue;
            const int s = cg / nrhs, r = cg - s * nrhs;
            cplx* Rp = a.rcur + ((int64_t)s * a.rcur_stride + F.rofs) * nrhs;
            stc(Rp + i + (int64_t)r * g, cmk(-v.re, -v.im));
          } else {
            const int i = it.z * SP_BM + row;
            if (i >= m) continue;
            const int s = cg / nrhs, r = cg - s * nrhs;
            stc(a.W + bv_off(a.lay, r, a.shift0 + s, a.perm ? a.perm[S.first + i] : S.first + i), v);
          }
        }
        }
      }
    }
}

__device__ __forceinline__ void spectral_b1_resident(const SpecArgs& a, const int4 it, double* As, cplx* Bs) {
  const SubDev S = a.subs[it.y];
  const FrontDev F = a.fronts[S.front];
  const int m = S.m, g = S.g, nrhs = a.nrhs, nx = a.nx;
  const int ncols = a.nb * nrhs;
  const int n0 = blockIdx.y * SP_BN;
  if (n0 >= ncols) return;
  const int K = g, nk = (K + SP_BK - 1) / SP_BK;   // <= SP_B1R_K / SP_BK resident chunks
  const double* __restrict__ Rm = a.RQ + S.rqofs;
  const double* __restrict__ Qm = Rm + (int64_t)g * m;
  const int32_t* __restrict__ bidx = a.bidx + F.bidx_beg;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3, wm = warp & 1, wn = warp >> 1;
  const cplx* __restrict__ wsub = a.wbuf + (int64_t)S.tofs * a.wstride;
  int* idx_s = reinterpret_cast<int*>(Bs + (SP_B1R_K / SP_BK) * SP_B_STAGE);
  for (int q = tid; q < g; q += 256) idx_s[q] = bidx[q];
  __syncthreads();
  // x_Gam of this column tile: every chunk at once (16 consecutive lanes walk down k of a column)
  const int kq = tid & 15, bq = tid >> 4;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int bcg = n0 + bq + 16 * u;
    const bool cok = bcg < ncols;
    const int s = cok ? bcg / nrhs : 0, r = cok ? bcg - s * nrhs : 0;
    const cplx* bbase = a.Z + (int64_t)s * nx * nrhs + (int64_t)r * nx;
    for (int kc = 0; kc < nk; ++kc) {
      const int k = kc * SP_BK + kq;
      const bool ok = cok && k < K;
      cp_async16(Bs + kc * SP_B_STAGE + kq * SP_LDB + bq + 16 * u, ok ? bbase + idx_s[k] : bbase, ok);
    }
  }
  cp_async_commit();
  const int ntile = (m + 31) / 32, total = ntile * nk;
  auto issue_a = [&](int c) {   // chunk c = (row tile c / nk, k chunk c % nk) into A stage c % SP_STAGES
    const int tile = c / nk, k0 = (c - tile * nk) * SP_BK;
    double* as = As + (c % SP_STAGES) * SP_A_STAGE;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = tid + 256 * u;
      const int r = idx >> 4, k = k0 + (idx & 15), kk = tile * 32 + (r >> 4) * 8 + (r & 7);
      const bool ok = kk < m && k < K;
      cp_async8(as + (idx & 15) * SP_LDA + r, ok ? ((r >> 3) & 1 ? Qm : Rm) + k + (int64_t)kk * g : Rm, ok);
    }
  };
#pragma unroll
  for (int c = 0; c < SP_STAGES - 1; ++c) {
    if (c < total) issue_a(c);
    cp_async_commit();
  }
  double acc[2][2][2][4];
  const bool wact = n0 + wn * 16 < ncols, wact1 = n0 + wn * 16 + 8 < ncols;
  for (int c = 0; c < total; ++c) {
    const int tile = c / nk, kc = c - tile * nk;
    if (kc == 0) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[mi][ni][0][v] = acc[mi][ni][1][v] = 0.0;
      // the tile's epilogue reads c (in Z, last touched by the forward sweep) and w: pull their
      // lines into L2 now, a whole K loop ahead (no registers held, unlike an early load)
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          const int rbase = wm * 32 + mi * 16 + gq;
          const int kk = tile * 32 + (rbase >> 4) * 8 + (rbase & 7);
#pragma unroll
          for (int cv = 0; cv < 2; ++cv) {
            const int cg = n0 + wn * 16 + ni * 8 + 2 * tq + cv;
            if (cg < ncols && kk < m) {
              const int s = cg / nrhs, r = cg - s * nrhs;
              asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a.Z + (int64_t)s * nx * nrhs + (int64_t)r * nx + S.first + kk));
              if (cv == 0) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(wsub + (int64_t)kk * a.wstride + s));
            }
          }
        }
    }
    cp_async_wait<SP_STAGES - 2>();
    __syncthreads();
    if (c + SP_STAGES - 1 < total) issue_a(c + SP_STAGES - 1);
    cp_async_commit();
    if (wact) {
      const double* as = As + (c % SP_STAGES) * SP_A_STAGE + tq * SP_LDA + wm * 32 + gq;
      const cplx* bs = Bs + kc * SP_B_STAGE + tq * SP_LDB + wn * 16 + gq;
#pragma unroll
      for (int kk = 0; kk < SP_BK; kk += 4) {
        double af[2][2];
        cplx bf[2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          af[mi][0] = as[kk * SP_LDA + mi * 16];
          af[mi][1] = as[kk * SP_LDA + mi * 16 + 8];
        }
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) bf[ni] = ldc(bs + kk * SP_LDB + ni * 8);
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) {
            if (ni == 1 && !wact1) continue;
            dmma_16x8x4(acc[mi][ni][0], af[mi][0], af[mi][1], bf[ni].re);
            dmma_16x8x4(acc[mi][ni][1], af[mi][0], af[mi][1], bf[ni].im);
          }
      }
    }
    if (kc == nk - 1) {
      // y = w o (c - R^T x_Gam) - Q^T x_Gam: rows rbase (R^T x) and rbase + 8 (Q^T x) belong to the
      // same interior index
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          const int rbase = wm * 32 + mi * 16 + gq;
          const int kk = tile * 32 + (rbase >> 4) * 8 + (rbase & 7);
#pragma unroll
          for (int cv = 0; cv < 2; ++cv) {
            const int cg = n0 + wn * 16 + ni * 8 + 2 * tq + cv;
            if (cg >= ncols || kk >= m) continue;
            const int s = cg / nrhs, r = cg - s * nrhs;
            cplx* zp = a.Z + (int64_t)s * nx * nrhs + (int64_t)r * nx + S.first + kk;
            const cplx t1 = cmk(acc[mi][ni][0][cv], acc[mi][ni][1][cv]);
            const cplx t2 = cmk(acc[mi][ni][0][2 + cv], acc[mi][ni][1][2 + cv]);
            const cplx w = ldc(wsub + (int64_t)kk * a.wstride + s);
            stc(zp, csub(cmul(w, csub(ldc(zp), t1)), t2));
          }
        }
    }
  }
  cp_async_wait<0>();
}

__global__ void __launch_bounds__(256, 2) spectral_kernel(SpecArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* As = reinterpret_cast<double*>(smem_raw);
  cplx* Bs = reinterpret_cast<cplx*>(As + SP_STAGES * SP_A_STAGE);
  const int4 it = a.items[blockIdx.x];
  switch (it.x) {
    case OP_U: spectral_tile<OP_U>(a, it, As, Bs); break;
    case OP_F1: spectral_tile<OP_F1>(a, it, As, Bs); break;
    case OP_F2: spectral_tile<OP_F2>(a, it, As, Bs); break;
    case OP_B1: spectral_tile<OP_B1>(a, it, As, Bs); break;
    case OP_B1R: spectral_b1_resident(a, it, As, Bs); break;
    default: spectral_tile<OP_B2>(a, it, As, Bs); break;
  }
}
