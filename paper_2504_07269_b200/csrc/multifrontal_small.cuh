// Small-front path of the multifrontal factorization (included by
// multifrontal.cu inside its anonymous namespace; uses LevelArgs/bv_off).
//
// Fronts of order n <= SMALL_N live entirely in shared memory (packed lower
// triangle, column-major) for the whole factorization: one CTA per
// (front, shift) instance, one thread per front row, CTA width = the level's
// max n rounded up to a warp.  Right-looking LDL^T in panels of KB = 8 pivots
// with four barriers per panel:
//   1. the panel rows publish their forward-RHS values;
//   2. warp 0 factors the 8x8 diagonal block in place (warp-synchronous) and
//      forward-solves the panel RHS;
//   3. every row below the panel runs its TRSM in registers (L11 read as
//      shared-memory broadcasts), publishes d_j l_cj, updates its RHS;
//   4. trailing update F[i][c] -= sum_j l_ij d_j l_cj, 8 complex FMAs per
//      shared load/store, two columns per iteration (independent chains).
// Only the initial gather (original entries, children's update blocks) and
// the final write-out of L/D, U and the forward vectors touch global memory.
#pragma once

constexpr int SMALL_N = 128;   // max front order on the shared-memory path
constexpr int KB = 8;          // panel width

__device__ __forceinline__ int pk(int i, int c, int n) { return c * n - ((c * (c - 1)) >> 1) + (i - c); }

// per-warp scratch (complex): L11 (KB x KB), y (KB x nr), d, 1/d
__host__ __device__ constexpr int scr_size(int nr) { return KB * KB + KB * nr + 2 * KB; }

__host__ __device__ constexpr int small_smem_bytes(int nmax, int nr) {
  return ((nmax * (nmax + 1)) / 2 + nmax * KB + nmax * nr + ((nmax + 31) / 32) * scr_size(nr)) * 16;
}

__device__ __forceinline__ cplx shfl_c(cplx v, int src) {
  return cmk(__shfl_sync(0xffffffffu, v.re, src), __shfl_sync(0xffffffffu, v.im, src));
}

// trailing update of row i: F[i][c] -= sum_{jj<W} av[jj] * PB[c][jj] for c in [c0, i]
// (W = panel width, compile-time: narrow last panels do no padded work)
template <int W>
__device__ __forceinline__ void trailing_row_w(cplx* __restrict__ F, const cplx* __restrict__ PB,
                                               const cplx (&av)[KB], int i, int c0, int n) {
  int c = c0;
  int q = pk(i, c, n);
  const cplx* __restrict__ pb = PB + c * KB;
#pragma unroll 2
  for (; c + 1 <= i; c += 2) {
    const int q1 = q + (n - c - 1);
    cplx x0 = F[q], x1 = F[q1];
#pragma unroll
    for (int jj = 0; jj < W; ++jj) {
      x0 = cfms(x0, av[jj], pb[jj]);
      x1 = cfms(x1, av[jj], pb[KB + jj]);
    }
    F[q] = x0;
    F[q1] = x1;
    q = q1 + (n - c - 2);
    pb += 2 * KB;
  }
  if (c <= i) {
    cplx x0 = F[q];
#pragma unroll
    for (int jj = 0; jj < W; ++jj) x0 = cfms(x0, av[jj], pb[jj]);
    F[q] = x0;
  }
}

__device__ __forceinline__ void trailing_row(cplx* F, const cplx* PB, const cplx (&av)[KB], int i, int c0,
                                             int n, int w) {
  switch (w) {
    case 8: trailing_row_w<8>(F, PB, av, i, c0, n); break;
    case 7: trailing_row_w<7>(F, PB, av, i, c0, n); break;
    case 6: trailing_row_w<6>(F, PB, av, i, c0, n); break;
    case 5: trailing_row_w<5>(F, PB, av, i, c0, n); break;
    case 4: trailing_row_w<4>(F, PB, av, i, c0, n); break;
    case 3: trailing_row_w<3>(F, PB, av, i, c0, n); break;
    case 2: trailing_row_w<2>(F, PB, av, i, c0, n); break;
    default: trailing_row_w<1>(F, PB, av, i, c0, n); break;
  }
}

template <int NR>
__global__ void __launch_bounds__(SMALL_N) factor_small_kernel(LevelArgs a, int nmax) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* F = reinterpret_cast<cplx*>(smem_raw);
  cplx* PB = F + (nmax * (nmax + 1)) / 2;   // nmax x KB : d_j l_cj of the current panel
  cplx* Rsm = PB + nmax * KB;               // nmax x NR  : forward RHS
  cplx* scratch = Rsm + nmax * NR;          // per warp: L11 (KB x KB), y (KB x NR), d, 1/d

  const int i = threadIdx.x, lane = i & 31, warp = i >> 5;
  const int nt = blockDim.x, nwarp = nt >> 5;
  const int nrhs = a.nrhs, nx = a.nx;
  const cplx zero = cmk(0.0, 0.0);
  cplx* W8 = scratch + warp * scr_size(NR);
  cplx* Y8 = W8 + KB * KB;
  cplx* Dv = Y8 + KB * NR;
  cplx* Dinv = Dv + KB;
  // grid-stride over (front, shift) instances: amortises block launch and
  // keeps a fixed set of resident CTAs busy on levels with millions of fronts
  const int total = a.nlist * a.nbatch;
  for (int inst = blockIdx.x; inst < total; inst += gridDim.x) {
  const int k = inst % a.nbatch;
  const FrontDev Fr = a.fronts[a.list[inst / a.nbatch]];
  const int n = Fr.n, p = Fr.p, b = n - p;
  const cplx lam = a.lam[k];
  const int64_t shift = a.shift0 + k;

  // ---- gather ----
  // the global loads (original entries, pivot rows of the RHS via perm) are
  // issued first so their latency overlaps the zero fill of F
  constexpr int EP = 4;
  int edst[EP];
  cplx eval[EP];
#pragma unroll
  for (int u = 0; u < EP; ++u) {
    const int e = i + u * nt;
    edst[u] = -1;
    eval[u] = zero;
    if (e < Fr.ent_cnt) {
      edst[u] = a.ent_dst[Fr.ent_beg + e];
      const double mv = a.Mv[Fr.ent_beg + e], av = a.Av[Fr.ent_beg + e];   // entry-ordered values
      eval[u] = cmk(fma(lam.re, av, mv), lam.im * av);
    }
  }
  const int64_t jrow = (i < p) ? (a.perm ? a.perm[Fr.pbeg + i] : Fr.pbeg + i) : 0;
  const int tri = (n * (n + 1)) / 2;
  for (int q = i; q < tri; q += nt) F[q] = zero;
  for (int row = i; row < n; row += nt) {
    int64_t j = row < p ? (row == i ? jrow : (a.perm ? a.perm[Fr.pbeg + row] : Fr.pbeg + row)) : 0;
#pragma unroll
    for (int r = 0; r < NR; ++r)
      Rsm[row * NR + r] = (row < p && r < nrhs) ? a.G[bv_off(a.lay, r, shift, j)] : zero;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < EP; ++u)
    if (edst[u] >= 0) F[pk(edst[u] % n, edst[u] / n, n)] = eval[u];
  for (int e = i + EP * nt; e < Fr.ent_cnt; e += nt) {
    const int dst = a.ent_dst[Fr.ent_beg + e];
    const double mv = a.Mv[Fr.ent_beg + e], av = a.Av[Fr.ent_beg + e];   // entry-ordered values
    F[pk(dst % n, dst / n, n)] = cmk(fma(lam.re, av, mv), lam.im * av);
  }
  __syncthreads();
  for (int ci = 0; ci < Fr.nchild; ++ci) {
    const FrontDev Cf = a.fronts[a.child_ids[Fr.child_beg + ci]];
    const int bc = Cf.n - Cf.p;
    const cplx* Uc = a.uchild + (int64_t)k * a.uchild_stride + Cf.uofs;
    const cplx* Rc = a.rchild + ((int64_t)k * a.rchild_stride + Cf.rofs) * nrhs;
    const int32_t* rel = a.relpos + Cf.relpos_beg;
    // each warp owns 8 child columns at a time (k2 = k2b + u*nwarp), lanes run
    // over child rows: one relpos load + 8 independent U_c loads in flight per lane
    constexpr int CU = 8;
    for (int k2b = warp; k2b < bc; k2b += CU * nwarp) {
      int r2[CU];
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const int k2 = k2b + u * nwarp;
        r2[u] = k2 < bc ? rel[k2] : 0;
      }
      for (int k1 = k2b + lane; k1 < bc; k1 += 32) {
        const int r1 = rel[k1];
        cplx v[CU];
#pragma unroll
        for (int u = 0; u < CU; ++u) {
          const int k2 = k2b + u * nwarp;
          v[u] = (k2 < bc && k1 >= k2) ? ldc(Uc + (int64_t)k2 * ldu(bc) + k1) : zero;
        }
#pragma unroll
        for (int u = 0; u < CU; ++u) {
          const int k2 = k2b + u * nwarp;
          if (k2 < bc && k1 >= k2) {
            const int q = pk(r1, r2[u], n);
            F[q] = cadd(F[q], v[u]);
          }
        }
      }
    }
    for (int q = i; q < bc; q += nt) {
      const int row = rel[q];
#pragma unroll
      for (int r = 0; r < NR; ++r)
        if (r < nrhs) Rsm[row * NR + r] = cadd(Rsm[row * NR + r], ldc(Rc + q + (int64_t)r * bc));
    }
    __syncthreads();
  }
  cplx rv[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) rv[r] = i < n ? Rsm[i * NR + r] : zero;

  // ---- factor the p pivots, panels of KB, two barriers per panel ----
  for (int kb = 0; kb < p; kb += KB) {
    const int w = min(KB, p - kb);
    // (A) every warp factors the w x w diagonal block redundantly in registers
    //     (lane = panel row) and forward-solves the panel RHS; warp-private results
    {
      cplx ar[KB], yr[NR];
#pragma unroll
      for (int cc = 0; cc < KB; ++cc) ar[cc] = (lane < w && cc <= lane) ? F[pk(kb + lane, kb + cc, n)] : zero;
#pragma unroll
      for (int r = 0; r < NR; ++r) yr[r] = lane < w ? Rsm[(kb + lane) * NR + r] : zero;
#pragma unroll
      for (int jj = 0; jj < KB; ++jj) {
        if (jj < w) {
          const cplx d = shfl_c(ar[jj], jj);
          const cplx dinv = crecip_fast(d);
          const cplx l = lane > jj ? cmul(ar[jj], dinv) : zero;
#pragma unroll
          for (int r = 0; r < NR; ++r) {
            const cplx ys = shfl_c(yr[r], jj);
            if (lane > jj) yr[r] = cfms(yr[r], l, ys);
          }
          const cplx ld = cmul(l, d);
#pragma unroll
          for (int cc = jj + 1; cc < KB; ++cc) {
            if (cc < w) {
              const cplx lc = shfl_c(l, cc);
              if (lane >= cc) ar[cc] = cfms(ar[cc], ld, lc);
            }
          }
          if (lane > jj) ar[jj] = l;
          if (lane == 0) {
            Dv[jj] = d;
            Dinv[jj] = dinv;
            if (warp == 0) {
              double m2 = cabs2(d);
              if (!(m2 > a.scale2[k]) || !isfinite(m2)) atomicCAS(a.err, 0, a.err_base + (int)shift + 1);
            }
          }
        }
      }
      if (lane < w) {
#pragma unroll
        for (int cc = 0; cc < KB; ++cc) W8[lane * KB + cc] = ar[cc];
#pragma unroll
        for (int r = 0; r < NR; ++r) Y8[lane * NR + r] = yr[r];
      }
      __syncwarp();
    }
    // (B) rows: panel rows take their factored row; rows below run the TRSM
    cplx av[KB];
#pragma unroll
    for (int jj = 0; jj < KB; ++jj) av[jj] = zero;
    if (i >= kb && i < kb + w) {
      const int row = i - kb;
#pragma unroll
      for (int cc = 0; cc < KB; ++cc)
        if (cc <= row) F[pk(i, kb + cc, n)] = W8[row * KB + cc];
#pragma unroll
      for (int r = 0; r < NR; ++r) rv[r] = Y8[row * NR + r];
    } else if (i >= kb + w && i < n) {
#pragma unroll
      for (int jj = 0; jj < KB; ++jj)
        if (jj < w) av[jj] = F[pk(i, kb + jj, n)];
#pragma unroll
      for (int jj = 1; jj < KB; ++jj) {
        if (jj < w) {
#pragma unroll
          for (int cc = 0; cc < jj; ++cc) av[jj] = cfms(av[jj], av[cc], W8[jj * KB + cc]);
        }
      }
#pragma unroll
      for (int jj = 0; jj < KB; ++jj) {
        if (jj < w) {
          av[jj] = cmul(av[jj], Dinv[jj]);
          F[pk(i, kb + jj, n)] = av[jj];
          PB[i * KB + jj] = cmul(Dv[jj], av[jj]);
        } else {
          PB[i * KB + jj] = zero;
        }
      }
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        if (r < nrhs) {
#pragma unroll
          for (int jj = 0; jj < KB; ++jj)
            if (jj < w) rv[r] = cfms(rv[r], av[jj], Y8[jj * NR + r]);
        }
      }
      if (i < kb + w + KB) {   // the next panel's rows publish their forward values
#pragma unroll
        for (int r = 0; r < NR; ++r) Rsm[i * NR + r] = rv[r];
      }
    }
    __syncthreads();
    if (i >= kb + w && i < n) trailing_row(F, PB, av, i, kb + w, n, w);
    __syncthreads();
  }

  // ---- write out: L/D (n x p), U (b x b), z = D^{-1} y, forward RHS update ----
  cplx* Pg = a.factor + (int64_t)k * a.fstride + Fr.fofs;
  cplx* Ug = a.ucur + (int64_t)k * a.ucur_stride + Fr.uofs;
  cplx* Rg = a.rcur + ((int64_t)k * a.rcur_stride + Fr.rofs) * nrhs;
  cplx* Zk = a.Z + (int64_t)k * nx * nrhs;
  if (i < n) {
    const int cmax = min(i, p - 1);
    int q = i;  // pk(i, 0, n)
    for (int c = 0; c <= cmax; ++c) {
      stc(Pg + i + (int64_t)c * n, F[q]);
      q += n - c - 1;
    }
    if (i >= p) {
      q = pk(i, p, n);
      for (int c = p; c <= i; ++c) {
        stc(Ug + (i - p) + (int64_t)(c - p) * ldu(b), F[q]);
        q += n - c - 1;
      }
#pragma unroll
      for (int r = 0; r < NR; ++r)
        if (r < nrhs) stc(Rg + (i - p) + (int64_t)r * b, rv[r]);
    } else {
      const cplx dinv = crecip_fast(F[pk(i, i, n)]);
#pragma unroll
      for (int r = 0; r < NR; ++r)
        if (r < nrhs) stc(Zk + Fr.pbeg + i + (int64_t)r * nx, cmul(rv[r], dinv));
    }
  }
  __syncthreads();   // shared memory is reused by the next instance
  }
}

__host__ __device__ constexpr int small_bwd_smem_bytes(int nmax, int pmax, int nr) {
  return ((nmax | 1) * pmax + nmax * nr + KB * nr) * 16;
}

// Backward substitution for fronts with small n * p: the factor block is
// staged in shared memory (odd leading dimension: conflict-free column reads);
// one thread per pivot column applies the boundary part, then the transposed
// unit triangle is solved in blocks of KB (warp 0 solves the block, all
// threads apply it): three barriers per block.
template <int NR>
__global__ void __launch_bounds__(SMALL_N) backward_small_kernel(LevelArgs a, int nmax, int pmax) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ldl = nmax | 1;
  cplx* Ls = reinterpret_cast<cplx*>(smem_raw);   // Ls[c * ldl + i]
  cplx* xs = Ls + ldl * pmax;                      // nmax x NR : x of boundary rows
  cplx* Tsm = xs + nmax * NR;                      // KB x NR : current block

  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
  const int nrhs = a.nrhs, nx = a.nx;
  const int total = a.nlist * a.nbatch;
  for (int inst = blockIdx.x; inst < total; inst += gridDim.x) {
  const int k = inst % a.nbatch;
  const FrontDev Fr = a.fronts[a.list[inst / a.nbatch]];
  const int n = Fr.n, p = Fr.p;
  const cplx* Pg = a.factor + (int64_t)k * a.fstride + Fr.fofs;
  cplx* Zk = a.Z + (int64_t)k * nx * nrhs;
  const int32_t* bidx = a.bidx + Fr.bidx_beg;
  const int64_t shift = a.shift0 + k;

  // stage the n x p factor block (full columns; 4 loads in flight per thread)
  {
    const int tot = n * p;
    int q = tid;
    for (; q + 3 * nt < tot; q += 4 * nt) {
      const cplx v0 = ldc(Pg + q), v1 = ldc(Pg + q + nt), v2 = ldc(Pg + q + 2 * nt), v3 = ldc(Pg + q + 3 * nt);
      Ls[(q / n) * ldl + q % n] = v0;
      Ls[((q + nt) / n) * ldl + (q + nt) % n] = v1;
      Ls[((q + 2 * nt) / n) * ldl + (q + 2 * nt) % n] = v2;
      Ls[((q + 3 * nt) / n) * ldl + (q + 3 * nt) % n] = v3;
    }
    for (; q < tot; q += nt) Ls[(q / n) * ldl + q % n] = ldc(Pg + q);
  }
  for (int i = p + tid; i < n; i += nt) {
    const int64_t g = bidx[i - p];
#pragma unroll
    for (int r = 0; r < NR; ++r)
      if (r < nrhs) xs[i * NR + r] = ldc(Zk + g + (int64_t)r * nx);
  }
  __syncthreads();
  const int j = tid;
  cplx t[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) t[r] = cmk(0.0, 0.0);
  if (j < p) {
#pragma unroll
    for (int r = 0; r < NR; ++r)
      if (r < nrhs) t[r] = ldc(Zk + Fr.pbeg + j + (int64_t)r * nx);
    for (int i = p; i < n; ++i) {
      const cplx l = Ls[j * ldl + i];
#pragma unroll
      for (int r = 0; r < NR; ++r)
        if (r < nrhs) t[r] = cfms(t[r], l, xs[i * NR + r]);
    }
  }
  for (int kb = ((p - 1) / KB) * KB; kb >= 0; kb -= KB) {
    const int w = min(KB, p - kb);
    if (j >= kb && j < kb + w) {
#pragma unroll
      for (int r = 0; r < NR; ++r) Tsm[(j - kb) * NR + r] = t[r];
    }
    __syncthreads();
    if (tid < 32 && lane < nrhs && lane < NR) {
      for (int jj = w - 1; jj >= 0; --jj) {
        cplx x = Tsm[jj * NR + lane];
        for (int cc = jj + 1; cc < w; ++cc) x = cfms(x, Ls[(kb + jj) * ldl + kb + cc], Tsm[cc * NR + lane]);
        if (!a.unit_diag) x = cmul(x, crecip_fast(Ls[(kb + jj) * ldl + kb + jj]));   // C C^T fronts
        Tsm[jj * NR + lane] = x;
        const int col = Fr.pbeg + kb + jj;
        stc(Zk + col + (int64_t)lane * nx, x);
        a.W[bv_off(a.lay, lane, shift, a.perm ? a.perm[col] : col)] = x;
      }
    }
    __syncthreads();
    if (j < kb) {
#pragma unroll
      for (int jj = 0; jj < KB; ++jj) {
        if (jj < w) {
          const cplx l = Ls[j * ldl + kb + jj];
#pragma unroll
          for (int r = 0; r < NR; ++r)
            if (r < nrhs) t[r] = cfms(t[r], l, Tsm[jj * NR + r]);
        }
      }
    }
    __syncthreads();
  }
  }   // instance loop
}

template <int NR>
int launch_small_factor(const LevelArgs& a, int grid, int nmax, cudaStream_t s) {
  const int smem = small_smem_bytes(nmax, NR);
  static DeviceOnce attr_once;
  if (attr_once.first()) {
    STFEM_CUDA_TRY(cudaFuncSetAttribute(factor_small_kernel<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        small_smem_bytes(SMALL_N, NR)));
    // occupancy here is shared-memory bound: ask for the full 228 KB carveout
    STFEM_CUDA_TRY(cudaFuncSetAttribute(factor_small_kernel<NR>,
                                        cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  }
  // persistent-style grid: as many CTAs as can be resident, grid-striding over instances
  const int threads = (nmax + 31) / 32 * 32;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  int per_sm = 0;
  STFEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, factor_small_kernel<NR>, threads, smem));
  const int resident = std::max(1, per_sm) * nsm;
  // measured: one instance per CTA (grid = all instances) beats a resident-only
  // grid-striding launch by ~5% on the leaf levels; keep the loop for large grids only
  const int g = grid > 64 * resident ? 64 * resident : grid;
  factor_small_kernel<NR><<<g, threads, smem, s>>>(a, nmax);
  STFEM_LAUNCH_CHECK("factor_small_kernel");
  return STFEM_OK;
}

template <int NR>
int launch_small_backward(const LevelArgs& a, int grid, int nmax, int pmax, cudaStream_t s) {
  const int smem = small_bwd_smem_bytes(nmax, pmax, NR);
  static DeviceOnce attr_once;
  if (attr_once.first()) {
    STFEM_CUDA_TRY(cudaFuncSetAttribute(backward_small_kernel<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        200 * 1024));
    STFEM_CUDA_TRY(cudaFuncSetAttribute(backward_small_kernel<NR>,
                                        cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  }
  const int threads = (nmax + 31) / 32 * 32;
  int nsm = 0, dev = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  STFEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, backward_small_kernel<NR>, threads, smem));
  backward_small_kernel<NR><<<std::min(grid, std::max(1, per_sm) * nsm), threads, smem, s>>>(a, nmax, pmax);
  STFEM_LAUNCH_CHECK("backward_small_kernel");
  return STFEM_OK;
}

inline int small_nr(int nrhs) { return nrhs <= 1 ? 1 : nrhs <= 2 ? 2 : nrhs <= 4 ? 4 : nrhs <= 8 ? 8 : 16; }

int launch_small_factor_any(const LevelArgs& a, int grid, int nmax, cudaStream_t s) {
  switch (small_nr(a.nrhs)) {
    case 1: return launch_small_factor<1>(a, grid, nmax, s);
    case 2: return launch_small_factor<2>(a, grid, nmax, s);
    case 4: return launch_small_factor<4>(a, grid, nmax, s);
    case 8: return launch_small_factor<8>(a, grid, nmax, s);
    default: return launch_small_factor<16>(a, grid, nmax, s);
  }
}

int launch_small_backward_any(const LevelArgs& a, int grid, int nmax, int pmax, cudaStream_t s) {
  switch (small_nr(a.nrhs)) {
    case 1: return launch_small_backward<1>(a, grid, nmax, pmax, s);
    case 2: return launch_small_backward<2>(a, grid, nmax, pmax, s);
    case 4: return launch_small_backward<4>(a, grid, nmax, pmax, s);
    case 8: return launch_small_backward<8>(a, grid, nmax, pmax, s);
    default: return launch_small_backward<16>(a, grid, nmax, pmax, s);
  }
}
