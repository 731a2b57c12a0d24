// Large-front path of the multifrontal factorization (included by
// multifrontal.cu inside its anonymous namespace; uses LevelArgs, sym_tile32,
// NB/NT/LDD/MAXR).
//
// A level of large fronts times a batch of shifts is factored by a pipeline of
// tile-parallel kernels, each launched over every (front, shift) instance of
// the level, so no kernel serialises a whole front on one CTA:
//   asm_front_kernel     (instance, 32-column block): gather-once assembly of
//                        the front (pivot block into the factor storage,
//                        boundary block into U) from the children's update
//                        blocks (inverse relpos maps), + M + lam A original
//                        entries (sorted column-major with per-column
//                        pointers), + the forward RHS (G through perm +
//                        children's RHS)
//   per 32-wide pivot panel kb:
//     diag_kernel        (instance): one warp factors the w x w diagonal block
//                        (complex-symmetric Cholesky, c_jj = sqrt(d_j)) and
//                        forward-solves the panel RHS y = C11^{-1} r
//     trsm_kernel<W>     (instance, 128-row tile): every row below the block
//                        solves x C11^T = b in registers (right-looking, W
//                        independent chains) and updates its RHS r -= x y
//     panel_update_kernel (instance, 64x64 tile): trailing pivot columns
//                        F[base:, base:p] -= X X^T on the FP64 tensor pipe,
//                        delayed over groups of panels (K up to 128)
//   syrk_level_kernel    (instance, 64x64 tile): U = F22 - L21 L21^T, K = p.
// Factor format: K = C C^T (transpose, not conjugate transpose).
#pragma once

constexpr int ASM_COLS = 32;
constexpr int TR_ROWS = 128;

__global__ void __launch_bounds__(NT, 4) asm_front_kernel(LevelArgs a) {
  extern __shared__ int inv_s[];   // nc x n inverse relpos maps
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int inst = blockIdx.x;
  const int k = inst % a.nbatch;
  const FrontDev F = a.fronts[a.list[inst / a.nbatch]];
  const int n = F.n, p = F.p, b = n - p;
  // this CTA assembles columns [cbeg, cstop) in blocks of ASM_COLS (a.asm_cpc columns per CTA:
  // one block on the wide top levels, the whole front on deep levels so the per-CTA setup
  // -- descriptor chain, inverse maps, barriers -- is paid once per instance)
  const int cbeg = blockIdx.y * a.asm_cpc;
  const int ncol = a.asm_pivots_only ? p : n;   // fused levels: U is gathered by syrk_gather_kernel
  if (cbeg >= ncol) return;
  const int cstop = min(ncol, cbeg + a.asm_cpc);
  cplx* U = a.ucur + (int64_t)k * a.ucur_stride + F.uofs;
  const int nrhs = a.nrhs, nx = a.nx;
  const cplx lam = a.lam[k];
  cplx* P = a.factor + (int64_t)k * a.fstride + F.fofs;
  const int64_t shift = a.shift0 + k;
  const int nc = min(F.nchild, 2);
  for (int q = tid; q < nc * n; q += NT) inv_s[q] = a.inv[F.inv_beg + q];
  const cplx* Ucs[2] = {nullptr, nullptr};
  const cplx* Rcs[2] = {nullptr, nullptr};
  int bcs[2] = {0, 0}, lcs[2] = {0, 0};   // children's boundary orders / update-block leading dimensions
  for (int s = 0; s < nc; ++s) {
    const FrontDev Cf = a.fronts[a.child_ids[F.child_beg + s]];
    bcs[s] = Cf.n - Cf.p;
    lcs[s] = ldu(bcs[s]);
    Ucs[s] = a.uchild + (int64_t)k * a.uchild_stride + Cf.uofs;
    Rcs[s] = a.rchild + ((int64_t)k * a.rchild_stride + Cf.rofs) * nrhs;
  }
  // original entries of pivot columns [cbeg, min(cstop, p)): one contiguous range of the sorted list
  const int* cp = a.ent_colptr + F.colptr_beg;
  const int ent_lo = cbeg < p ? cp[cbeg] : 0, ent_hi = cbeg < p ? cp[min(cstop, p)] : 0;
  // the first EP original entries of this thread: their (value, destination) loads are issued
  // now so their latency hides behind the gather below
  constexpr int EP = 1;
  double pm[EP], pa[EP];
  int pd[EP];
#pragma unroll
  for (int u = 0; u < EP; ++u) {
    const int e = ent_lo + tid + u * NT;
    const bool ok = e < ent_hi;
    pm[u] = ok ? a.Mv[F.ent_beg + e] : 0.0;
    pa[u] = ok ? a.Av[F.ent_beg + e] : 0.0;
    pd[u] = ok ? a.ent_dst[F.ent_beg + e] : -1;
  }
  __syncthreads();
  // gather: warp w owns columns c0 + w + 8u (u < 4), lanes run down the rows
  constexpr int CU = 4, NW = NT / 32;
  const cplx zero = cmk(0.0, 0.0);
  for (int c0 = cbeg; c0 < cstop; c0 += ASM_COLS) {
    const int cend = min(cstop, c0 + ASM_COLS);
    int k2[2][CU];
    cplx* dst[CU];
#pragma unroll
    for (int u = 0; u < CU; ++u) {
      const int c2 = min(c0 + warp + u * NW, cend - 1);
#pragma unroll
      for (int s = 0; s < 2; ++s) k2[s][u] = s < nc ? inv_s[s * n + c2] : -1;
      dst[u] = (c2 < p) ? P + (int64_t)c2 * n : U + (int64_t)(c2 - p) * ldu(b) - p;
    }
    // two row blocks per iteration: 16 independent child loads in flight per thread
    for (int rb = c0 + warp + lane; rb < n; rb += 64) {
      cplx v[2][CU];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r1 = rb + 32 * h;
        int k1[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) k1[s] = (s < nc && r1 < n) ? inv_s[s * n + r1] : -1;
#pragma unroll
        for (int u = 0; u < CU; ++u) {
          v[h][u] = zero;
#pragma unroll
          for (int s = 0; s < 2; ++s)
            if (k1[s] >= 0 && k2[s][u] >= 0)
              v[h][u] = cadd(v[h][u], ldc(Ucs[s] + (int64_t)k2[s][u] * lcs[s] + k1[s]));
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r1 = rb + 32 * h;
#pragma unroll
        for (int u = 0; u < CU; ++u) {
          const int c2 = c0 + warp + u * NW;
          if (c2 < cend && r1 < n && r1 >= c2) stc(dst[u] + r1, v[h][u]);
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < EP; ++u) {
    if (pd[u] < 0) continue;
    cplx* d = P + pd[u];
    const cplx o = ldc(d);
    stc(d, cmk(o.re + fma(lam.re, pa[u], pm[u]), o.im + lam.im * pa[u]));
  }
  for (int e = ent_lo + tid + EP * NT; e < ent_hi; e += NT) {
    const double mv = a.Mv[F.ent_beg + e], av = a.Av[F.ent_beg + e];   // entry-ordered values
    cplx* d = P + a.ent_dst[F.ent_beg + e];
    const cplx o = ldc(d);
    stc(d, cmk(o.re + fma(lam.re, av, mv), o.im + lam.im * av));
  }
  if (blockIdx.y == 0) {
    // forward RHS: pivot rows get G (through perm) + children, boundary rows children only
    cplx* R = a.rcur + ((int64_t)k * a.rcur_stride + F.rofs) * nrhs;
    cplx* Zk = a.Z + (int64_t)k * nx * nrhs;
    for (int q = tid; q < n * nrhs; q += NT) {
      const int r1 = q % n, r = q / n;
      cplx v = zero;
      if (r1 < p) v = ldc(a.G + bv_off(a.lay, r, shift, a.perm ? a.perm[F.pbeg + r1] : F.pbeg + r1));
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int kk = s < nc ? inv_s[s * n + r1] : -1;
        if (kk >= 0) v = cadd(v, ldc(Rcs[s] + kk + (int64_t)r * bcs[s]));
      }
      if (r1 < p) stc(Zk + F.pbeg + r1 + (int64_t)r * nx, v);
      else stc(R + (r1 - p) + (int64_t)r * b, v);
    }
  }
}

// w x w diagonal block of panel kb, one CTA per instance: warp 0 factors it
// (lane = row), then every warp forward-solves its share of the RHS
// (blockDim = 32 * min(8, nrhs))
// packed lower triangle of the w x w block (column-major): element (row r, column c), r >= c
__device__ __forceinline__ int lp(int c, int r) { return c * (2 * NB - c + 1) / 2 + r - c; }
constexpr int LP_SIZE = NB * (NB + 1) / 2;
constexpr int DIAG_RPW = 3;   // right-hand sides per warp in the panel forward solve

// PACK (one-warp CTAs, nrhs == 1): packed triangle, 8.4 KB instead of 17 KB of shared memory
// per instance -- those CTAs are shared-memory limited, so twice as many resident instances
// per SM.  Multi-RHS CTAs (up to 8 warps) are thread limited; they keep the padded square,
// whose constant column stride keeps integer work off the serial factorization chain.
template <bool PACK>
__device__ __forceinline__ int dix(int c, int r) { return PACK ? lp(c, r) : c * LDD + r; }

template <bool PACK>
__global__ void __launch_bounds__(256) diag_kernel(LevelArgs a, int kb) {
  __shared__ cplx Ld[PACK ? LP_SIZE : NB * LDD];
  __shared__ cplx dinv_s[NB], cdg[NB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int inst = blockIdx.x;
  const int k = inst % a.nbatch;
  const FrontDev F = a.fronts[a.list[inst / a.nbatch]];
  const int n = F.n, p = F.p;
  if (kb >= p) return;
  const int w = min(NB, p - kb);
  const int nrhs = a.nrhs, nx = a.nx;
  cplx* P = a.factor + (int64_t)k * a.fstride + F.fofs;
  cplx* Zk = a.Z + (int64_t)k * nx * nrhs;
  const int64_t shift = a.shift0 + k;
  const cplx zero = cmk(0.0, 0.0);
  if (warp == 0) {
    {
      // all of the lane's (row's) loads in flight at once, then staged: one global latency
      // per instance instead of one per column
      cplx v[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c)
        v[c] = (c < w && lane >= c && lane < w) ? ldc(P + (kb + lane) + (int64_t)(kb + c) * n) : zero;
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c < w && lane >= c && lane < w) Ld[dix<PACK>(c, lane)] = v[c];
    }
    __syncwarp();
    // step j: a_ic -= (a_ij / d_j) a_cj on unscaled values; then columns scale by 1/c_j = d_j^{-1/2}
    for (int j = 0; j < w; ++j) {
      const cplx d = Ld[dix<PACK>(j, j)];
      if (lane > j && lane < w) {
        const cplx f = cmul(Ld[dix<PACK>(j, lane)], crecip_fast(d));
        const cplx* __restrict__ colj = Ld + dix<PACK>(j, 0);   // colj[c] = (row c, column j), c >= j
        int c = j + 1;
        int o = dix<PACK>(c, lane);                       // (row lane, column c)
        for (; c + 3 <= lane; c += 4) {
          const int o1 = PACK ? o + NB - 1 - c : o + LDD, o2 = PACK ? o1 + NB - 2 - c : o1 + LDD,
                    o3 = PACK ? o2 + NB - 3 - c : o2 + LDD;
          const cplx x0 = Ld[o], x1 = Ld[o1], x2 = Ld[o2], x3 = Ld[o3];
          const cplx y0 = colj[c], y1 = colj[c + 1], y2 = colj[c + 2], y3 = colj[c + 3];
          Ld[o] = cfms(x0, f, y0);
          Ld[o1] = cfms(x1, f, y1);
          Ld[o2] = cfms(x2, f, y2);
          Ld[o3] = cfms(x3, f, y3);
          o = PACK ? o3 + NB - 4 - c : o3 + LDD;
        }
        for (; c <= lane; ++c) {
          Ld[o] = cfms(Ld[o], f, colj[c]);
          o += PACK ? NB - 1 - c : LDD;
        }
      }
      __syncwarp();
    }
    if (lane < w) {
      const cplx d = Ld[dix<PACK>(lane, lane)];
      const double m2 = cabs2(d);
      // pivot collapse: relative to the largest original diagonal entry of this shift
      if (!(m2 > a.scale2[k]) || !isfinite(m2)) atomicCAS(a.err, 0, a.err_base + (int)shift + 1);
      const cplx c = csqrt_(d);
      cdg[lane] = c;
      dinv_s[lane] = crecip(c);
    }
    __syncwarp();
    for (int j = 0; j < w; ++j) {
      if (lane == j) Ld[dix<PACK>(j, j)] = cdg[j];
      else if (lane > j && lane < w) Ld[dix<PACK>(j, lane)] = cmul(Ld[dix<PACK>(j, lane)], dinv_s[j]);
    }
    __syncwarp();
    for (int c = 0; c < w; ++c)
      if (lane >= c && lane < w) stc(P + (kb + lane) + (int64_t)(kb + c) * n, Ld[dix<PACK>(c, lane)]);
  }
  __syncthreads();
  // y = C11^{-1} r in column (axpy) form: lane i holds r_i; once y_j is final it
  // is broadcast and every lane i > j subtracts C[i][j] y_j (RHS over warps)
  // A warp carries RPW (3; single-RHS instances 1) right-hand sides through the 32-step chain at once (independent
  // chains interleave in the pipeline): 9 RHS need 3 warps, not 8 -- and a multi-RHS CTA of 96
  // instead of 256 threads leaves room for three times as many resident instances.
  constexpr int RPW = PACK ? 1 : DIAG_RPW;
  for (int r0 = warp * RPW; r0 < nrhs; r0 += nwarp * RPW) {
    cplx* z = Zk + F.pbeg + kb + (int64_t)r0 * nx;
    cplx yl[RPW];
#pragma unroll
    for (int q = 0; q < RPW; ++q) yl[q] = (lane < w && r0 + q < nrhs) ? ldc(z + (int64_t)q * nx + lane) : zero;
    for (int j = 0; j < w; ++j) {
      const cplx dj = dinv_s[j], lj = (lane > j && lane < w) ? Ld[dix<PACK>(j, lane)] : zero;
#pragma unroll
      for (int q = 0; q < RPW; ++q) {
        if (lane == j) yl[q] = cmul(yl[q], dj);
        const cplx yj = cmk(__shfl_sync(0xffffffffu, yl[q].re, j), __shfl_sync(0xffffffffu, yl[q].im, j));
        if (lane > j) yl[q] = cfms(yl[q], lj, yj);
      }
    }
#pragma unroll
    for (int q = 0; q < RPW; ++q)
      if (lane < w && r0 + q < nrhs) stc(z + (int64_t)q * nx + lane, yl[q]);
  }
}

// rows below panel kb: x C11^T = b per row (thread per row), then the row's
// forward RHS r -= x y.  The W-wide panel is solved in register blocks of 16
// columns (right-looking inside a block, independent update chains); a later
// block first subtracts the finished blocks, re-read from global (L1-hot).
// Measured on C4 (ms per step): blocks of 8 at 64 registers / 8 CTAs per SM 72.9,
// blocks of 16 at 96 registers / 5 CTAs 69.0 (48 instead of 80 loads per row),
// at 128 registers / 4 CTAs 76.8, at 80 registers / 6 CTAs it spills.
template <int W>
__global__ void __launch_bounds__(TR_ROWS, 5) trsm_kernel(LevelArgs a, int kb) {
  constexpr int WB = 16;
  constexpr int LW = W + 1;           // padded pitch: the column-wise staging below is conflict-free
  __shared__ cplx Ls[W * LW];         // Ls[c * LW + c'] = C[kb+c][kb+c'] (c' < c); Ls[c*LW+c] = 1 / c_cc
  __shared__ cplx ys[W * MAXR];
  const int tid = threadIdx.x;
  const int inst = blockIdx.x;
  const int k = inst % a.nbatch;
  const FrontDev F = a.fronts[a.list[inst / a.nbatch]];
  const int n = F.n, p = F.p, b = n - p;
  if (kb >= p) return;
  const int w = min(NB, p - kb);
  const int r0 = kb + w + blockIdx.y * TR_ROWS;
  if (r0 >= n) return;
  const int nrhs = a.nrhs, nx = a.nx;
  cplx* P = a.factor + (int64_t)k * a.fstride + F.fofs;
  cplx* Zk = a.Z + (int64_t)k * nx * nrhs;
  const cplx zero = cmk(0.0, 0.0);
  for (int idx = tid; idx < W * W; idx += TR_ROWS) {
    const int c = idx % W, c2 = idx / W;   // consecutive threads walk down column c2 (coalesced)
    cplx v = zero;
    if (c < w && c2 <= c) {
      v = ldc(P + (kb + c) + (int64_t)(kb + c2) * n);
      if (c2 == c) v = crecip(v);
    } else if (c2 == c) {
      v = cmk(1.0, 0.0);
    }
    Ls[c * LW + c2] = v;
  }
  for (int idx = tid; idx < W * nrhs; idx += TR_ROWS) {
    const int c = idx % W, r = idx / W;
    ys[c * MAXR + r] = c < w ? ldc(Zk + F.pbeg + kb + c + (int64_t)r * nx) : zero;
  }
  __syncthreads();
  const int i = r0 + tid;
  if (i >= n) return;
  cplx* prow = P + i + (int64_t)kb * n;
#pragma unroll 1
  for (int jb = 0; jb < W; jb += WB) {
    if (jb >= w) break;
    cplx x[WB];
#pragma unroll
    for (int c = 0; c < WB; ++c) x[c] = jb + c < w ? ldc(prow + (int64_t)(jb + c) * n) : zero;
    // subtract the finished blocks (their x are final in global memory)
    for (int c2 = 0; c2 < jb; ++c2) {
      const cplx xc = ldc(prow + (int64_t)c2 * n);
#pragma unroll
      for (int c = 0; c < WB; ++c) x[c] = cfms(x[c], xc, Ls[(jb + c) * LW + c2]);
    }
#pragma unroll
    for (int c = 0; c < WB; ++c) {
      x[c] = cmul(x[c], Ls[(jb + c) * LW + jb + c]);
#pragma unroll
      for (int c2 = c + 1; c2 < WB; ++c2) x[c2] = cfms(x[c2], x[c], Ls[(jb + c2) * LW + jb + c]);
    }
#pragma unroll
    for (int c = 0; c < WB; ++c)
      if (jb + c < w) stc(prow + (int64_t)(jb + c) * n, x[c]);
    if (nrhs == 1) {
      cplx* dst = (i < p) ? Zk + F.pbeg + i : a.rcur + ((int64_t)k * a.rcur_stride + F.rofs) + (i - p);
      cplx acc = ldc(dst);
#pragma unroll
      for (int c = 0; c < WB; ++c) acc = cfms(acc, x[c], ys[(jb + c) * MAXR]);
      stc(dst, acc);
    } else {
      // (measured: one update per RHS after the whole panel, x re-read from L1, is slower)
      cplx* dst0 = (i < p) ? Zk + F.pbeg + i : a.rcur + ((int64_t)k * a.rcur_stride + F.rofs) * nrhs + (i - p);
      const int64_t rs = (i < p) ? (int64_t)nx : (int64_t)b;
#pragma unroll 4
      for (int r = 0; r < nrhs; ++r) {
        cplx acc = ldc(dst0 + r * rs);
#pragma unroll
        for (int c = 0; c < WB; ++c) acc = cfms(acc, x[c], ys[(jb + c) * MAXR + r]);
        stc(dst0 + r * rs, acc);
      }
    }
  }
}

// Trailing pivot-column updates, delayed over groups of G panels (right-looking
// across groups, left-looking inside one): inside a group only the next
// panel's 32 columns are updated, by every panel of the group so far
// ("narrow"); after the group's last panel the columns beyond it receive all G
// panels at once ("wide", K = 32 G), so the trailing block is read and written
// once per 32 G pivots instead of once per 32.
// Region of one update: rows [cb, n), columns [cb, cb + cols) with
// cols = narrow ? min(NB, p - cb) : p - cb, updated by the panel columns [k0, k0 + K).
