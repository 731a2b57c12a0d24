// Small-front path of the multifrontal factorization (included by
// multifrontal.cu inside its anonymous namespace; uses LevelArgs/bv_off).
//
// Fronts of order n <= SMALL_N live entirely in shared memory (packed lower
// triangle, column-major) for the whole factorization: one CTA per
// (front, shift) instance, one thread per front row, CTA width = the level's
// max n rounded up to a warp.  Right-looking LDL^T in register panels of
// KB = 8 pivots: each thread keeps its row's panel entries in registers, the
// scaled panel rows d_j l_cj are published to shared memory, and the trailing
// update F[i][c] -= sum_j l_ij d_j l_cj runs as 8 complex FMAs per shared
// load/store (broadcast reads of the panel row c).  The forward substitution
// of the RHS rides along with the pivot steps (thread i keeps r_i).  Only the
// initial gather (original entries, children's update blocks) and the final
// write-out of L/D, U and the forward vectors touch global memory.
#pragma once

constexpr int SMALL_N = 128;   // max front order on the shared-memory path
constexpr int KB = 8;          // register panel width

__device__ __forceinline__ int pk(int i, int c, int n) { return c * n - ((c * (c - 1)) >> 1) + (i - c); }

__host__ __device__ constexpr int small_smem_bytes(int nmax, int nrhs) {
  return ((nmax * (nmax + 1)) / 2 + nmax * KB + KB + KB * MAXR + KB * KB + nmax * nrhs) * 16;
}

__global__ void __launch_bounds__(SMALL_N) factor_small_kernel(LevelArgs a, int nmax) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* F = reinterpret_cast<cplx*>(smem_raw);
  cplx* PB = F + (nmax * (nmax + 1)) / 2;   // nmax x KB : d_j * l_cj for the current panel
  cplx* dsm = PB + nmax * KB;               // KB pivots of the panel
  cplx* ysm = dsm + KB;                     // KB x MAXR forward values y_j of the panel pivots
  cplx* plsm = ysm + KB * MAXR;             // KB x KB: l_{kb+cc, kb+jj} inside the panel
  cplx* Rsm = plsm + KB * KB;               // nmax x nrhs RHS gather

  const int i = threadIdx.x;
  const int inst = blockIdx.x;
  const int k = inst % a.nbatch;
  const FrontDev Fr = a.fronts[a.list[inst / a.nbatch]];
  const int n = Fr.n, p = Fr.p, b = n - p;
  const int nrhs = a.nrhs, nx = a.nx;
  const cplx lam = a.lam[k];
  cplx* Pg = a.factor + (int64_t)k * a.fstride + Fr.fofs;
  cplx* Ug = a.ucur + (int64_t)k * a.ucur_stride + Fr.uofs;
  cplx* Rg = a.rcur + ((int64_t)k * a.rcur_stride + Fr.rofs) * nrhs;
  cplx* Zk = a.Z + (int64_t)k * nx * nrhs;
  const int64_t shift = a.shift0 + k;
  const int nt = blockDim.x;
  const cplx zero = cmk(0.0, 0.0);

  // ---- gather ----
  const int tri = (n * (n + 1)) / 2;
  for (int q = i; q < tri; q += nt) F[q] = zero;
  for (int q = i; q < n * nrhs; q += nt) {
    int row = q % n, r = q / n;
    cplx v = zero;
    if (row < p) v = a.G[bv_off(a.lay, r, shift, a.perm[Fr.pbeg + row])];
    Rsm[row * nrhs + r] = v;
  }
  __syncthreads();
  for (int e = i; e < Fr.ent_cnt; e += nt) {
    int src = a.ent_src[Fr.ent_beg + e];
    int dst = a.ent_dst[Fr.ent_beg + e];
    double mv = a.Mv[src], av = a.Av[src];
    F[pk(dst % n, dst / n, n)] = cmk(fma(lam.re, av, mv), lam.im * av);
  }
  __syncthreads();
  for (int ci = 0; ci < Fr.nchild; ++ci) {
    const FrontDev Cf = a.fronts[a.child_ids[Fr.child_beg + ci]];
    const int bc = Cf.n - Cf.p;
    const cplx* Uc = a.uchild + (int64_t)k * a.uchild_stride + Cf.uofs;
    const cplx* Rc = a.rchild + ((int64_t)k * a.rchild_stride + Cf.rofs) * nrhs;
    const int32_t* rel = a.relpos + Cf.relpos_beg;
    for (int q = i; q < bc * bc; q += nt) {
      int k1 = q % bc, k2 = q / bc;
      if (k1 < k2) continue;
      int r1 = rel[k1], r2 = rel[k2];
      int pq = pk(r1, r2, n);
      F[pq] = cadd(F[pq], ldc(Uc + q));
    }
    for (int q = i; q < bc * nrhs; q += nt) {
      int k1 = q % bc, r = q / bc;
      int row = rel[k1];
      Rsm[row * nrhs + r] = cadd(Rsm[row * nrhs + r], ldc(Rc + k1 + (int64_t)r * bc));
    }
    __syncthreads();
  }
  cplx rv[MAXR];
#pragma unroll
  for (int r = 0; r < MAXR; ++r) rv[r] = (r < nrhs && i < n) ? Rsm[i * nrhs + r] : zero;

  // ---- factor p pivots in register panels of KB ----
  for (int kb = 0; kb < p; kb += KB) {
    const int w = min(KB, p - kb);
    cplx av[KB];
#pragma unroll
    for (int jj = 0; jj < KB; ++jj)
      av[jj] = (jj < w && i < n && kb + jj <= i) ? F[pk(i, kb + jj, n)] : zero;
#pragma unroll
    for (int jj = 0; jj < KB; ++jj) {
      if (jj < w) {
        const int j = kb + jj;
        if (i == j) {
          dsm[jj] = av[jj];
#pragma unroll
          for (int r = 0; r < MAXR; ++r)
            if (r < nrhs) ysm[jj * MAXR + r] = rv[r];
          double m2 = cabs2(av[jj]);
          if (!(m2 > 1e-300) || !isfinite(m2)) atomicCAS(a.err, 0, (int)shift + 1);
        }
        __syncthreads();
        const cplx d = dsm[jj];
        if (i > j && i < n) {
          cplx l = cdiv(av[jj], d);
          av[jj] = l;
          if (i < kb + w) plsm[jj * KB + (i - kb)] = l;
#pragma unroll
          for (int r = 0; r < MAXR; ++r)
            if (r < nrhs) rv[r] = cfms(rv[r], l, ysm[jj * MAXR + r]);
        }
        __syncthreads();
        if (i > j && i < n) {
          const cplx ld = cmul(av[jj], d);
#pragma unroll
          for (int cc = jj + 1; cc < KB; ++cc)
            if (cc < w && kb + cc <= i) av[cc] = cfms(av[cc], ld, plsm[jj * KB + cc]);
        }
      }
    }
    // write the panel back; publish d_j l_cj for the trailing update
    if (i < n) {
#pragma unroll
      for (int jj = 0; jj < KB; ++jj)
        if (jj < w && kb + jj <= i) {
          F[pk(i, kb + jj, n)] = av[jj];
          if (i >= kb + w) PB[i * KB + jj] = cmul(dsm[jj], av[jj]);
        }
    }
    __syncthreads();
    if (i >= kb + w && i < n) {
      for (int c = kb + w; c <= i; ++c) {
        const int q = pk(i, c, n);
        cplx acc = F[q];
#pragma unroll
        for (int jj = 0; jj < KB; ++jj)
          if (jj < w) acc = cfms(acc, av[jj], PB[c * KB + jj]);
        F[q] = acc;
      }
    }
    __syncthreads();
  }

  // ---- write out: L/D (n x p), U (b x b), z = D^{-1} y, forward RHS update ----
  if (i < n) {
    const int cmax = min(i, p - 1);
    for (int c = 0; c <= cmax; ++c) stc(Pg + i + (int64_t)c * n, F[pk(i, c, n)]);
    if (i >= p)
      for (int c = p; c <= i; ++c) stc(Ug + (i - p) + (int64_t)(c - p) * b, F[pk(i, c, n)]);
    if (i < p) {
      cplx d = F[pk(i, i, n)];
#pragma unroll
      for (int r = 0; r < MAXR; ++r)
        if (r < nrhs) stc(Zk + Fr.pbeg + i + (int64_t)r * nx, cdiv(rv[r], d));
    } else {
#pragma unroll
      for (int r = 0; r < MAXR; ++r)
        if (r < nrhs) stc(Rg + (i - p) + (int64_t)r * b, rv[r]);
    }
  }
}

__host__ __device__ constexpr int small_bwd_smem_bytes(int nmax, int pmax, int nrhs) {
  return ((nmax | 1) * pmax + nmax * nrhs + nrhs) * 16;
}

// Backward substitution for fronts with n * p small: the n x p factor block is
// staged in shared memory (odd leading dimension: conflict-free column reads),
// one thread per pivot column.
__global__ void __launch_bounds__(SMALL_N) backward_small_kernel(LevelArgs a, int nmax, int pmax) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ldl = nmax | 1;
  cplx* Ls = reinterpret_cast<cplx*>(smem_raw);   // Ls[c * ldl + i]
  cplx* xs = Ls + ldl * pmax;                      // nmax x nrhs : x of boundary rows / solved pivots
  cplx* xj = xs + nmax * a.nrhs;                   // nrhs: value published at each step

  const int tid = threadIdx.x, nt = blockDim.x;
  const int inst = blockIdx.x;
  const int k = inst % a.nbatch;
  const FrontDev Fr = a.fronts[a.list[inst / a.nbatch]];
  const int n = Fr.n, p = Fr.p;
  const int nrhs = a.nrhs, nx = a.nx;
  const cplx* Pg = a.factor + (int64_t)k * a.fstride + Fr.fofs;
  cplx* Zk = a.Z + (int64_t)k * nx * nrhs;
  const int32_t* bidx = a.bidx + Fr.bidx_beg;
  const int64_t shift = a.shift0 + k;

  for (int q = tid; q < n * p; q += nt) {
    int i = q % n, c = q / n;
    Ls[c * ldl + i] = ldc(Pg + q);
  }
  for (int q = tid; q < (n - p) * nrhs; q += nt) {
    int i = q % (n - p), r = q / (n - p);
    xs[(p + i) * nrhs + r] = ldc(Zk + bidx[i] + (int64_t)r * nx);
  }
  __syncthreads();
  const int j = tid;
  cplx t[MAXR];
#pragma unroll
  for (int r = 0; r < MAXR; ++r) t[r] = cmk(0.0, 0.0);
  if (j < p) {
#pragma unroll
    for (int r = 0; r < MAXR; ++r)
      if (r < nrhs) t[r] = ldc(Zk + Fr.pbeg + j + (int64_t)r * nx);
    for (int i = p; i < n; ++i) {
      cplx l = Ls[j * ldl + i];
#pragma unroll
      for (int r = 0; r < MAXR; ++r)
        if (r < nrhs) t[r] = cfms(t[r], l, xs[i * nrhs + r]);
    }
  }
  for (int jj = p - 1; jj >= 0; --jj) {
    if (j == jj) {
#pragma unroll
      for (int r = 0; r < MAXR; ++r)
        if (r < nrhs) {
          xj[r] = t[r];
          stc(Zk + Fr.pbeg + j + (int64_t)r * nx, t[r]);
          a.W[bv_off(a.lay, r, shift, a.perm[Fr.pbeg + j])] = t[r];
        }
    }
    __syncthreads();
    if (j < jj) {
      cplx l = Ls[j * ldl + jj];
#pragma unroll
      for (int r = 0; r < MAXR; ++r)
        if (r < nrhs) t[r] = cfms(t[r], l, xj[r]);
    }
    __syncthreads();
  }
}
