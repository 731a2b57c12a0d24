// K1/K2/K7 — GPU assembly and the matrix-free global residual.
//
// K1 assemble_spatial (P2 is the north-star
//    extension): one thread per element computes the local mass / stiffness
//    matrix (P1 closed form; P2 by the 7-point degree-5 rule, exact for the
//    degree-4 mass integrand) and adds it into the CSR values through a
//    precomputed slot table.  Elements are greedily coloured so that no two
//    elements of a colour share a node: a launch per colour writes disjoint
//    slots -> no atomics, results reproducible bit for bit.
// K2 assemble_rhs: one thread per (triangle, time
//    interval) pair, 7-point triangle rule x 5-point Gauss; coloured in space
//    (element colours) and in time (even/odd intervals).
// K7 apply_global: two batched CSR SpMVs (M v, A v) and a
//    banded temporal combine  out_l = sum_k (i B_t[l,k] (M v)_k + M_t[l,k] (A v)_k).
#include <stdio.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace stfem {

struct Asm {
  int degree = 1, k = 3;  // nodes per element
  int nv = 0, ne = 0, n = 0;
  std::vector<double> verts;        // nv x 2
  std::vector<int32_t> elems;       // ne x k, sorted by colour
  std::vector<int32_t> dof;         // nv
  std::vector<int64_t> rowptr;
  std::vector<int32_t> colind;
  std::vector<int32_t> slot;        // ne x k x k CSR slot (or -1), same element order
  std::vector<int32_t> color_off;   // ncolor + 1
  // device
  int device = -1;
  double* d_verts = nullptr;
  int32_t *d_elems = nullptr, *d_dof = nullptr, *d_slot = nullptr, *d_colind = nullptr;
  int64_t* d_rowptr = nullptr;
  ~Asm() { free_device(); }
  void free_device() {
    cudaFree(d_verts);
    cudaFree(d_elems);
    cudaFree(d_dof);
    cudaFree(d_slot);
    cudaFree(d_colind);
    cudaFree(d_rowptr);
    d_verts = nullptr;
    d_elems = d_dof = d_slot = d_colind = nullptr;
    d_rowptr = nullptr;
    device = -1;
  }
};

namespace {

// degree-5 7-point triangle rule (weights sum to 1/2), Gauss-5 on [0,1]
__constant__ double c_tri_a[7], c_tri_b[7], c_tri_w[7];
__constant__ double c_gl_x[5], c_gl_w[5];

void host_rules(double* a, double* b, double* w, double* gx, double* gw) {
  double s15 = std::sqrt(15.0);
  double p = (6 - s15) / 21, q = (6 + s15) / 21;
  double wa = (155 - s15) / 1200, wb = (155 + s15) / 1200;
  double A[7] = {1.0 / 3, p, 1 - 2 * p, p, q, 1 - 2 * q, q};
  double B[7] = {1.0 / 3, p, p, 1 - 2 * p, q, q, 1 - 2 * q};
  double W[7] = {9.0 / 40, wa, wa, wa, wb, wb, wb};
  for (int i = 0; i < 7; ++i) {
    a[i] = A[i];
    b[i] = B[i];
    w[i] = 0.5 * W[i];
  }
  // Gauss-Legendre 5 on [-1,1] mapped to [0,1]
  double x0 = 0.0, x1 = std::sqrt(5.0 - 2.0 * std::sqrt(10.0 / 7.0)) / 3.0,
         x2 = std::sqrt(5.0 + 2.0 * std::sqrt(10.0 / 7.0)) / 3.0;
  double w0 = 128.0 / 225.0, w1 = (322.0 + 13.0 * std::sqrt(70.0)) / 900.0,
         w2 = (322.0 - 13.0 * std::sqrt(70.0)) / 900.0;
  double X[5] = {-x2, -x1, x0, x1, x2}, Wg[5] = {w2, w1, w0, w1, w2};
  for (int i = 0; i < 5; ++i) {
    gx[i] = 0.5 * (X[i] + 1.0);
    gw[i] = 0.5 * Wg[i];
  }
}

__device__ __forceinline__ void p2_basis(double l0, double l1, double l2, double* phi) {
  phi[0] = l0 * (2 * l0 - 1);
  phi[1] = l1 * (2 * l1 - 1);
  phi[2] = l2 * (2 * l2 - 1);
  phi[3] = 4 * l0 * l1;
  phi[4] = 4 * l1 * l2;
  phi[5] = 4 * l2 * l0;
}

__device__ __forceinline__ void p2_dbasis(double l0, double l1, double l2, double (*d)[3]) {
  d[0][0] = 4 * l0 - 1; d[0][1] = 0;          d[0][2] = 0;
  d[1][0] = 0;          d[1][1] = 4 * l1 - 1; d[1][2] = 0;
  d[2][0] = 0;          d[2][1] = 0;          d[2][2] = 4 * l2 - 1;
  d[3][0] = 4 * l1;     d[3][1] = 4 * l0;     d[3][2] = 0;
  d[4][0] = 0;          d[4][1] = 4 * l2;     d[4][2] = 4 * l1;
  d[5][0] = 4 * l2;     d[5][1] = 0;          d[5][2] = 4 * l0;
}

template <int KN>
__global__ void asm_spatial_kernel(const double* __restrict__ V, const int32_t* __restrict__ E,
                                   const int32_t* __restrict__ S, int e0, int e1, double* Mv,
                                   double* Av) {
  int e = e0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= e1) return;
  const int32_t* el = E + (int64_t)e * KN;
  double x0 = V[2 * el[0]], y0 = V[2 * el[0] + 1];
  double x1 = V[2 * el[1]], y1 = V[2 * el[1] + 1];
  double x2 = V[2 * el[2]], y2 = V[2 * el[2] + 1];
  double area = 0.5 * ((x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0));
  double bx[3] = {y1 - y2, y2 - y0, y0 - y1};
  double cy[3] = {x2 - x1, x0 - x2, x1 - x0};
  double Ml[KN][KN], Kl[KN][KN];
  if (KN == 3) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        Kl[a][b] = (bx[a] * bx[b] + cy[a] * cy[b]) / (4 * area);
        Ml[a][b] = area / 12 * (a == b ? 2.0 : 1.0);
      }
  } else {
    double gl[3][2];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      gl[a][0] = bx[a] / (2 * area);
      gl[a][1] = cy[a] / (2 * area);
    }
#pragma unroll
    for (int a = 0; a < KN; ++a)
#pragma unroll
      for (int b = 0; b < KN; ++b) Ml[a][b] = Kl[a][b] = 0;
    for (int q = 0; q < 7; ++q) {
      double l1 = c_tri_a[q], l2 = c_tri_b[q], l0 = 1 - l1 - l2;
      double phi[6], d[6][3], g[6][2];
      p2_basis(l0, l1, l2, phi);
      p2_dbasis(l0, l1, l2, d);
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        g[i][0] = d[i][0] * gl[0][0] + d[i][1] * gl[1][0] + d[i][2] * gl[2][0];
        g[i][1] = d[i][0] * gl[0][1] + d[i][1] * gl[1][1] + d[i][2] * gl[2][1];
      }
      double w = 2 * area * c_tri_w[q];
#pragma unroll
      for (int a = 0; a < KN; ++a)
#pragma unroll
        for (int b = 0; b < KN; ++b) {
          Ml[a][b] += w * phi[a] * phi[b];
          Kl[a][b] += w * (g[a][0] * g[b][0] + g[a][1] * g[b][1]);
        }
    }
  }
  const int32_t* sl = S + (int64_t)e * KN * KN;
#pragma unroll
  for (int a = 0; a < KN; ++a)
#pragma unroll
    for (int b = 0; b < KN; ++b) {
      int s = sl[a * KN + b];
      if (s >= 0) {
        Mv[s] += Ml[a][b];
        Av[s] += Kl[a][b];
      }
    }
}

__device__ cplx source_fn(int kind, double x, double y, double t) {
  const double PI = 3.141592653589793;
  double s = sin(PI * x) * sin(PI * y);
  if (kind == 1) {
    return cmk(2 * PI * PI * s * sin(PI * t), PI * s * cos(PI * t));
  } else if (kind == 2) {
    // s e^{-it} (i + t + 2 pi^2 t)
    double c = cos(t), sn = sin(t);
    double ar = t + 2 * PI * PI * t, ai = 1.0;
    return cmk(s * (c * ar + sn * ai), s * (c * ai - sn * ar));
  } else {
    // f = i dpsi/dt - lap psi,  psi = e^{it} s q,  q = sin(t x y)
    double q = sin(t * x * y), cq = cos(t * x * y);
    double sx = PI * cos(PI * x) * sin(PI * y), sy = PI * sin(PI * x) * cos(PI * y);
    double lap = -2 * PI * PI * s * q + 2 * cq * t * (y * sx + x * sy) - s * q * t * t * (x * x + y * y);
    // i*E*s*(i q + x y cq) - E*lap = E * ( -s q - lap + i s x y cq )
    double re0 = -s * q - lap, im0 = s * x * y * cq;
    double c = cos(t), sn = sin(t);
    return cmk(c * re0 - sn * im0, c * im0 + sn * re0);
  }
}

__global__ void asm_rhs_kernel(int kind, const double* __restrict__ V, const int32_t* __restrict__ E,
                               const int32_t* __restrict__ dof, int e0, int ecount,
                               const double* __restrict__ bp, int N, int parity, cplx* F, int64_t ld) {
  int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int nint = (N - parity + 1) / 2;  // intervals k = parity, parity+2, ...
  if (gid >= (int64_t)ecount * nint) return;
  int e = e0 + (int)(gid % ecount);
  int kidx = parity + 2 * (int)(gid / ecount);
  const int32_t* el = E + (int64_t)e * 3;
  double px[3], py[3];
  int dj[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    px[a] = V[2 * el[a]];
    py[a] = V[2 * el[a] + 1];
    dj[a] = dof[el[a]];
  }
  double area = 0.5 * ((px[1] - px[0]) * (py[2] - py[0]) - (px[2] - px[0]) * (py[1] - py[0]));
  double t0 = bp[kidx], ht = bp[kidx + 1] - bp[kidx];
  cplx acc[2][3];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int a = 0; a < 3; ++a) acc[i][a] = cmk(0, 0);
  for (int q = 0; q < 7; ++q) {
    double l1 = c_tri_a[q], l2 = c_tri_b[q], l0 = 1 - l1 - l2;
    double lam[3] = {l0, l1, l2};
    double x = l0 * px[0] + l1 * px[1] + l2 * px[2];
    double y = l0 * py[0] + l1 * py[1] + l2 * py[2];
    for (int gq = 0; gq < 5; ++gq) {
      double s = c_gl_x[gq];
      cplx f = source_fn(kind, x, y, t0 + ht * s);
      double w = 2 * area * c_tri_w[q] * ht * c_gl_w[gq];
      double wt[2] = {w * (1 - s), w * s};
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          acc[i][a].re += wt[i] * lam[a] * f.re;
          acc[i][a].im += wt[i] * lam[a] * f.im;
        }
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    int lt = kidx - 1 + i;
    if (lt < 0) continue;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (dj[a] < 0) continue;
      cplx* dst = F + (int64_t)lt * ld + dj[a];
      cplx o = ldc(dst);
      stc(dst, cadd(o, acc[i][a]));
    }
  }
}

// y[v][r] = alpha * sum_c A[r][c] x[v][c] + beta * y[v][r]   (one thread per (row, vector))
__global__ void spmv_c_kernel(int n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                              const double* __restrict__ val, const cplx* __restrict__ x, int64_t ldx,
                              cplx* y, int64_t ldy, int nvec, cplx alpha, double beta) {
  int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)n * nvec) return;
  int r = (int)(gid % n), v = (int)(gid / n);
  const cplx* xv = x + (int64_t)v * ldx;
  double sr = 0, si = 0;
  for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
    cplx xx = ldc(xv + ci[k]);
    sr = fma(val[k], xx.re, sr);
    si = fma(val[k], xx.im, si);
  }
  cplx s = cmul(alpha, cmk(sr, si));
  cplx* yp = y + (int64_t)v * ldy + r;
  if (beta != 0.0) {
    cplx o = ldc(yp);
    s = cmk(s.re + beta * o.re, s.im + beta * o.im);
  }
  stc(yp, s);
}

// Bartels-Stewart sweep update: after w_l is solved,
//   G[r][l'][j] -= S[l', l] * (A_x w_l^{(r)})[j]   for every pending row l' < l.
// One thread per (spatial row j, RHS r): the CSR row product is formed once
// and scattered down the l' rows with coalesced (along j) read-modify-writes.
// The S column is staged in shared memory in chunks of 1024.
__global__ void bs_update_kernel(int n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                 const double* __restrict__ val, const cplx* __restrict__ w, int64_t ldw,
                                 int nrhs, const cplx* __restrict__ scol, int l, cplx* G, int64_t g_rhs,
                                 int64_t g_shift) {
  __shared__ cplx ss[1024];
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = gid < (int64_t)n * nrhs;
  const int j = live ? (int)(gid % n) : 0, r = live ? (int)(gid / n) : 0;
  double sr = 0, si = 0;
  if (live) {
    const cplx* wr = w + (int64_t)r * ldw;
    for (int64_t k = rp[j]; k < rp[j + 1]; ++k) {
      const cplx x = ldc(wr + ci[k]);
      sr = fma(val[k], x.re, sr);
      si = fma(val[k], x.im, si);
    }
  }
  cplx* gp = G + (int64_t)r * g_rhs + j;
  for (int c0 = 0; c0 < l; c0 += 1024) {
    const int cn = min(1024, l - c0);
    __syncthreads();
    for (int q = threadIdx.x; q < cn; q += blockDim.x) ss[q] = ldc(scol + c0 + q);
    __syncthreads();
    if (!live) continue;
    for (int q = 0; q < cn; ++q) {
      const cplx s = ss[q];
      cplx* g = gp + (int64_t)(c0 + q) * g_shift;
      const cplx o = ldc(g);
      stc(g, cmk(o.re - (s.re * sr - s.im * si), o.im - (s.re * si + s.im * sr)));
    }
  }
}

__global__ void combine_kernel(int nt, int nx, int bw, const double* __restrict__ Mb,
                               const double* __restrict__ Bb, const cplx* __restrict__ MV,
                               const cplx* __restrict__ AV, cplx* out) {
  int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)nt * nx) return;
  int l = (int)(gid / nx), j = (int)(gid % nx);
  double re = 0, im = 0;
  for (int o = -bw; o <= bw; ++o) {
    int kk = l + o;
    if (kk < 0 || kk >= nt) continue;
    double bm = Mb[l * (2 * bw + 1) + o + bw], bb = Bb[l * (2 * bw + 1) + o + bw];
    cplx mv = ldc(MV + (int64_t)kk * nx + j), av = ldc(AV + (int64_t)kk * nx + j);
    // i*bb*mv + bm*av
    re += -bb * mv.im + bm * av.re;
    im += bb * mv.re + bm * av.im;
  }
  stc(out + gid, cmk(re, im));
}

// ---- K8: space-time error norms ---------------------------
// psi, d_t psi, grad_x psi of the built-in manufactured solutions
__device__ void exact_fn(int kind, double x, double y, double t, cplx& psi, cplx& dt, cplx& gx, cplx& gy) {
  const double PI = 3.141592653589793;
  const double sx = sin(PI * x), sy = sin(PI * y), cx = cos(PI * x), cy = cos(PI * y);
  const double s = sx * sy, dsx = PI * cx * sy, dsy = PI * sx * cy;
  if (kind == 1) {  // s sin(pi t)
    const double st = sin(PI * t), ct = cos(PI * t);
    psi = cmk(s * st, 0);
    dt = cmk(s * PI * ct, 0);
    gx = cmk(dsx * st, 0);
    gy = cmk(dsy * st, 0);
  } else if (kind == 2) {  // s t e^{-it}
    const cplx e = cmk(cos(t), -sin(t));
    psi = cmul(cmk(s * t, 0), e);
    dt = cmul(cmk(s, -s * t), e);  // s e^{-it} (1 - i t)
    gx = cmul(cmk(dsx * t, 0), e);
    gy = cmul(cmk(dsy * t, 0), e);
  } else {  // e^{it} s sin(t x y)
    const cplx e = cmk(cos(t), sin(t));
    const double q = sin(t * x * y), cq = cos(t * x * y);
    psi = cmul(cmk(s * q, 0), e);
    dt = cmul(cmk(s * x * y * cq, s * q), e);  // e^{it} s (i q + x y cq)
    gx = cmul(cmk(dsx * q + s * cq * t * y, 0), e);
    gy = cmul(cmk(dsy * q + s * cq * t * x, 0), e);
  }
}

// one thread per (triangle, time interval); 7-point x 5-point quadrature;
// deterministic two-level reduction (block tree, then a fixed-order pass)
__global__ void __launch_bounds__(256) errors_kernel(int kind, const double* __restrict__ V,
                                                     const int32_t* __restrict__ E, const int32_t* __restrict__ dof,
                                                     int ne, const double* __restrict__ bp, int N,
                                                     const cplx* __restrict__ C, int64_t ld,
                                                     const cplx* __restrict__ psi0, double* partial) {
  __shared__ double s1[256], s2[256];
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double l2 = 0, h1 = 0;
  if (gid < (int64_t)ne * N) {
    const int e = (int)(gid % ne), k = (int)(gid / ne);
    const int32_t* el = E + (int64_t)e * 3;
    double px[3], py[3];
    cplx u0[3], u1[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      px[a] = V[2 * el[a]];
      py[a] = V[2 * el[a] + 1];
      const int j = dof[el[a]];
      const cplx p0 = psi0 ? psi0[el[a]] : cmk(0, 0);
      u0[a] = (k > 0 && j >= 0) ? cadd(C[(int64_t)(k - 1) * ld + j], p0) : p0;
      u1[a] = (j >= 0) ? cadd(C[(int64_t)k * ld + j], p0) : p0;
    }
    const double area = 0.5 * ((px[1] - px[0]) * (py[2] - py[0]) - (px[2] - px[0]) * (py[1] - py[0]));
    const double bx[3] = {py[1] - py[2], py[2] - py[0], py[0] - py[1]};
    const double cy[3] = {px[2] - px[1], px[0] - px[2], px[1] - px[0]};
    const double t0 = bp[k], ht = bp[k + 1] - bp[k];
    for (int g = 0; g < 5; ++g) {
      const double s = c_gl_x[g], t = t0 + ht * s;
      cplx ut[3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
        ut[a] = cmk((1 - s) * u0[a].re + s * u1[a].re, (1 - s) * u0[a].im + s * u1[a].im);
      cplx gxh = cmk(0, 0), gyh = cmk(0, 0), dth[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        gxh = cadd(gxh, cmk(ut[a].re * bx[a] / (2 * area), ut[a].im * bx[a] / (2 * area)));
        gyh = cadd(gyh, cmk(ut[a].re * cy[a] / (2 * area), ut[a].im * cy[a] / (2 * area)));
        dth[a] = cmk((u1[a].re - u0[a].re) / ht, (u1[a].im - u0[a].im) / ht);
      }
      for (int q = 0; q < 7; ++q) {
        const double l1 = c_tri_a[q], l2q = c_tri_b[q], l0 = 1 - l1 - l2q;
        const double x = l0 * px[0] + l1 * px[1] + l2q * px[2], y = l0 * py[0] + l1 * py[1] + l2q * py[2];
        cplx ps, dt, gx, gy;
        exact_fn(kind, x, y, t, ps, dt, gx, gy);
        const cplx uh = cmk(l0 * ut[0].re + l1 * ut[1].re + l2q * ut[2].re, l0 * ut[0].im + l1 * ut[1].im + l2q * ut[2].im);
        const cplx duh = cmk(l0 * dth[0].re + l1 * dth[1].re + l2q * dth[2].re,
                             l0 * dth[0].im + l1 * dth[1].im + l2q * dth[2].im);
        const double w = 2 * area * c_tri_w[q] * ht * c_gl_w[g];
        l2 += w * cabs2(csub(ps, uh));
        h1 += w * (cabs2(csub(dt, duh)) + cabs2(csub(gx, gxh)) + cabs2(csub(gy, gyh)));
      }
    }
  }
  s1[threadIdx.x] = l2;
  s2[threadIdx.x] = h1;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s1[threadIdx.x] += s1[threadIdx.x + o];
      s2[threadIdx.x] += s2[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = s1[0];
    partial[2 * blockIdx.x + 1] = s2[0];
  }
}

__global__ void sum_partials_kernel(const double* partial, int nb, double* out) {
  __shared__ double s1[256], s2[256];
  double a = 0, b = 0;
  for (int i = threadIdx.x; i < nb; i += 256) {
    a += partial[2 * i];
    b += partial[2 * i + 1];
  }
  s1[threadIdx.x] = a;
  s2[threadIdx.x] = b;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s1[threadIdx.x] += s1[threadIdx.x + o];
      s2[threadIdx.x] += s2[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = s1[0];
    out[1] = s2[0];
  }
}

int upload(Asm& A) {
  int dev;
  STFEM_CUDA_TRY(cudaGetDevice(&dev));
  if (A.d_verts && A.device == dev) return STFEM_OK;
  A.free_device();
  A.device = dev;
  STFEM_CUDA_TRY(cudaMalloc(&A.d_verts, A.verts.size() * 8));
  STFEM_CUDA_TRY(cudaMemcpy(A.d_verts, A.verts.data(), A.verts.size() * 8, cudaMemcpyHostToDevice));
  STFEM_CUDA_TRY(cudaMalloc(&A.d_elems, A.elems.size() * 4));
  STFEM_CUDA_TRY(cudaMemcpy(A.d_elems, A.elems.data(), A.elems.size() * 4, cudaMemcpyHostToDevice));
  STFEM_CUDA_TRY(cudaMalloc(&A.d_dof, A.dof.size() * 4));
  STFEM_CUDA_TRY(cudaMemcpy(A.d_dof, A.dof.data(), A.dof.size() * 4, cudaMemcpyHostToDevice));
  STFEM_CUDA_TRY(cudaMalloc(&A.d_slot, A.slot.size() * 4));
  STFEM_CUDA_TRY(cudaMemcpy(A.d_slot, A.slot.data(), A.slot.size() * 4, cudaMemcpyHostToDevice));
  STFEM_CUDA_TRY(cudaMalloc(&A.d_colind, std::max<size_t>(1, A.colind.size()) * 4));
  STFEM_CUDA_TRY(cudaMemcpy(A.d_colind, A.colind.data(), A.colind.size() * 4, cudaMemcpyHostToDevice));
  STFEM_CUDA_TRY(cudaMalloc(&A.d_rowptr, A.rowptr.size() * 8));
  STFEM_CUDA_TRY(cudaMemcpy(A.d_rowptr, A.rowptr.data(), A.rowptr.size() * 8, cudaMemcpyHostToDevice));
  double a[7], b[7], w[7], gx[5], gw[5];
  host_rules(a, b, w, gx, gw);
  STFEM_CUDA_TRY(cudaMemcpyToSymbol(c_tri_a, a, sizeof(a)));
  STFEM_CUDA_TRY(cudaMemcpyToSymbol(c_tri_b, b, sizeof(b)));
  STFEM_CUDA_TRY(cudaMemcpyToSymbol(c_tri_w, w, sizeof(w)));
  STFEM_CUDA_TRY(cudaMemcpyToSymbol(c_gl_x, gx, sizeof(gx)));
  STFEM_CUDA_TRY(cudaMemcpyToSymbol(c_gl_w, gw, sizeof(gw)));
  return STFEM_OK;
}

}  // namespace

int asm_create(int degree, int nv, const double* verts, int ne, const int64_t* elems,
               const int64_t* interior_dof, Asm** out) {
  if (degree != 1 && degree != 2) return fail(STFEM_ERR_ARG, "asm_create: degree must be 1 or 2");
  if (nv <= 0 || ne <= 0) return fail(STFEM_ERR_DIM, "asm_create: empty mesh");
  Asm* A = new Asm();
  A->degree = degree;
  A->k = degree == 1 ? 3 : 6;
  const int k = A->k;
  A->nv = nv;
  A->ne = ne;
  A->verts.assign(verts, verts + 2 * (size_t)nv);
  A->dof.resize(nv);
  int n = 0;
  for (int v = 0; v < nv; ++v) {
    A->dof[v] = (int32_t)interior_dof[v];
    if (interior_dof[v] >= 0) n = std::max(n, (int)interior_dof[v] + 1);
  }
  A->n = n;
  for (int64_t i = 0; i < (int64_t)ne * k; ++i)
    if (elems[i] < 0 || elems[i] >= nv) {
      delete A;
      return fail(STFEM_ERR_ARG, "asm_create: element vertex out of range");
    }
  // greedy colouring: no two elements of a colour share any node
  std::vector<uint64_t> used(nv, 0);
  std::vector<int> col(ne);
  int ncol = 0;
  for (int e = 0; e < ne; ++e) {
    uint64_t m = 0;
    for (int a = 0; a < k; ++a) m |= used[elems[(int64_t)e * k + a]];
    int c = 0;
    while (c < 64 && (m >> c & 1ull)) ++c;
    if (c == 64) {
      delete A;
      return fail(STFEM_ERR_INTERNAL, "asm_create: more than 64 colours needed");
    }
    col[e] = c;
    ncol = std::max(ncol, c + 1);
    for (int a = 0; a < k; ++a) used[elems[(int64_t)e * k + a]] |= 1ull << c;
  }
  std::vector<int> order(ne);
  A->color_off.assign(ncol + 1, 0);
  for (int e = 0; e < ne; ++e) A->color_off[col[e] + 1]++;
  for (int c = 0; c < ncol; ++c) A->color_off[c + 1] += A->color_off[c];
  {
    std::vector<int> fill(A->color_off.begin(), A->color_off.end() - 1);
    for (int e = 0; e < ne; ++e) order[fill[col[e]]++] = e;
  }
  A->elems.resize((size_t)ne * k);
  for (int i = 0; i < ne; ++i)
    for (int a = 0; a < k; ++a) A->elems[(size_t)i * k + a] = (int32_t)elems[(int64_t)order[i] * k + a];
  // CSR pattern over interior DoFs: all pairs within an element
  std::vector<std::vector<int32_t>> rows(n);
  for (int e = 0; e < ne; ++e)
    for (int a = 0; a < k; ++a) {
      int i = A->dof[A->elems[(size_t)e * k + a]];
      if (i < 0) continue;
      for (int b = 0; b < k; ++b) {
        int j = A->dof[A->elems[(size_t)e * k + b]];
        if (j >= 0) rows[i].push_back(j);
      }
    }
  A->rowptr.assign(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    auto& r = rows[i];
    std::sort(r.begin(), r.end());
    r.erase(std::unique(r.begin(), r.end()), r.end());
    A->rowptr[i + 1] = A->rowptr[i] + (int64_t)r.size();
  }
  A->colind.resize(A->rowptr[n]);
  for (int i = 0; i < n; ++i) std::copy(rows[i].begin(), rows[i].end(), A->colind.begin() + A->rowptr[i]);
  rows.clear();
  A->slot.assign((size_t)ne * k * k, -1);
  for (int e = 0; e < ne; ++e)
    for (int a = 0; a < k; ++a) {
      int i = A->dof[A->elems[(size_t)e * k + a]];
      if (i < 0) continue;
      for (int b = 0; b < k; ++b) {
        int j = A->dof[A->elems[(size_t)e * k + b]];
        if (j < 0) continue;
        auto beg = A->colind.begin() + A->rowptr[i], end = A->colind.begin() + A->rowptr[i + 1];
        auto it = std::lower_bound(beg, end, j);
        A->slot[((size_t)e * k + a) * k + b] = (int32_t)(it - A->colind.begin());
      }
    }
  *out = A;
  return STFEM_OK;
}

int asm_spatial(Asm& A, double* Mv, double* Av, cudaStream_t s) {
  int rc;
  if ((rc = upload(A))) return rc;
  size_t nnz = A.colind.size();
  STFEM_CUDA_TRY(cudaMemsetAsync(Mv, 0, nnz * 8, s));
  STFEM_CUDA_TRY(cudaMemsetAsync(Av, 0, nnz * 8, s));
  for (size_t c = 0; c + 1 < A.color_off.size(); ++c) {
    int e0 = A.color_off[c], e1 = A.color_off[c + 1];
    if (e1 <= e0) continue;
    int blocks = (e1 - e0 + 127) / 128;
    if (A.k == 3)
      asm_spatial_kernel<3><<<blocks, 128, 0, s>>>(A.d_verts, A.d_elems, A.d_slot, e0, e1, Mv, Av);
    else
      asm_spatial_kernel<6><<<blocks, 128, 0, s>>>(A.d_verts, A.d_elems, A.d_slot, e0, e1, Mv, Av);
    STFEM_LAUNCH_CHECK("asm_spatial_kernel");
  }
  return STFEM_OK;
}

}  // namespace stfem

using stfem::Asm;

extern "C" int stfem_asm_create(int32_t degree, int32_t nv, const double* verts, int32_t ne,
                                const int64_t* elems, const int64_t* interior_dof, stfem_asm** out) {
  if (!verts || !elems || !interior_dof || !out) return stfem::fail(STFEM_ERR_ARG, "asm_create: null pointer");
  Asm* A = nullptr;
  int rc = stfem::asm_create(degree, nv, verts, ne, elems, interior_dof, &A);
  if (rc) return rc;
  *out = reinterpret_cast<stfem_asm*>(A);
  return STFEM_OK;
}

extern "C" int stfem_asm_destroy(stfem_asm* a) {
  delete reinterpret_cast<Asm*>(a);
  return STFEM_OK;
}

extern "C" int stfem_asm_pattern(const stfem_asm* a, int32_t* n, int64_t* nnz, int64_t* rowptr,
                                 int32_t* colind) {
  if (!a) return stfem::fail(STFEM_ERR_ARG, "asm_pattern: null");
  const Asm& A = *reinterpret_cast<const Asm*>(a);
  if (n) *n = A.n;
  if (nnz) *nnz = (int64_t)A.colind.size();
  if (rowptr) std::copy(A.rowptr.begin(), A.rowptr.end(), rowptr);
  if (colind) std::copy(A.colind.begin(), A.colind.end(), colind);
  return STFEM_OK;
}

extern "C" int stfem_asm_spatial(stfem_asm* a, double* Mvals, double* Avals, void* stream) {
  if (!a || !Mvals || !Avals) return stfem::fail(STFEM_ERR_ARG, "asm_spatial: null");
  return stfem::asm_spatial(*reinterpret_cast<Asm*>(a), Mvals, Avals, (cudaStream_t)stream);
}

extern "C" int stfem_asm_rhs(stfem_asm* a, int32_t kind, const double* breakpoints, int32_t N, void* F,
                             int64_t ld, void* stream) {
  if (!a || !breakpoints || !F) return stfem::fail(STFEM_ERR_ARG, "asm_rhs: null");
  Asm& A = *reinterpret_cast<Asm*>(a);
  if (A.degree != 1) return stfem::fail(STFEM_ERR_ARG, "asm_rhs: P1 space only");
  if (kind < 1 || kind > 3) return stfem::fail(STFEM_ERR_ARG, "asm_rhs: unknown source kind");
  if (N < 1 || ld < A.n) return stfem::fail(STFEM_ERR_DIM, "asm_rhs: bad N / ld");
  int rc;
  if ((rc = stfem::upload(A))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  double* d_bp = nullptr;
  STFEM_CUDA_TRY(cudaMallocAsync((void**)&d_bp, (N + 1) * 8, s));
  STFEM_CUDA_TRY(cudaMemcpyAsync(d_bp, breakpoints, (N + 1) * 8, cudaMemcpyHostToDevice, s));
  STFEM_CUDA_TRY(cudaMemsetAsync(F, 0, (size_t)N * ld * 16, s));
  for (size_t c = 0; c + 1 < A.color_off.size(); ++c) {
    int e0 = A.color_off[c], cnt = A.color_off[c + 1] - e0;
    for (int par = 0; par < 2; ++par) {
      int nint = (N - par + 1) / 2;
      int64_t tot = (int64_t)cnt * nint;
      if (tot <= 0) continue;
      stfem::asm_rhs_kernel<<<(unsigned)((tot + 127) / 128), 128, 0, s>>>(
          kind, A.d_verts, A.d_elems, A.d_dof, e0, cnt, d_bp, N, par, (stfem::cplx*)F, ld);
      STFEM_LAUNCH_CHECK("asm_rhs_kernel");
    }
  }
  STFEM_CUDA_TRY(cudaFreeAsync(d_bp, s));
  // host buffer must stay valid until the copy completes
  STFEM_CUDA_TRY(cudaStreamSynchronize(s));
  return STFEM_OK;
}

extern "C" int stfem_csr_spmv_c(const stfem_asm* a, const double* vals, const void* v, int64_t ldv, void* y,
                                int64_t ldy, int32_t nvec, double are, double aim, double beta, void* stream) {
  if (!a || !vals || !v || !y) return stfem::fail(STFEM_ERR_ARG, "spmv: null");
  Asm& A = *reinterpret_cast<Asm*>(const_cast<stfem_asm*>(a));
  int rc;
  if ((rc = stfem::upload(A))) return rc;
  int64_t tot = (int64_t)A.n * nvec;
  if (tot == 0) return STFEM_OK;
  stfem::spmv_c_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      A.n, A.d_rowptr, A.d_colind, vals, (const stfem::cplx*)v, ldv, (stfem::cplx*)y, ldy, nvec,
      stfem::cmk(are, aim), beta);
  STFEM_LAUNCH_CHECK("spmv_c_kernel");
  return STFEM_OK;
}

extern "C" int stfem_bs_update(const stfem_asm* a, const double* Avals, const void* w, int64_t ldw,
                               int32_t nrhs, const void* scol, int32_t l, void* G, int64_t g_rhs_stride,
                               int64_t g_shift_stride, void* stream) {
  if (!a || !Avals || !w || !G || (l > 0 && !scol)) return stfem::fail(STFEM_ERR_ARG, "bs_update: null");
  if (nrhs < 1 || l < 0 || ldw < 0) return stfem::fail(STFEM_ERR_DIM, "bs_update: bad nrhs / l / ldw");
  const Asm& A = *reinterpret_cast<const Asm*>(a);
  int rc;
  if ((rc = stfem::upload(const_cast<Asm&>(A)))) return rc;
  if (l == 0) return STFEM_OK;
  const int64_t tot = (int64_t)A.n * nrhs;
  stfem::bs_update_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      A.n, A.d_rowptr, A.d_colind, Avals, (const stfem::cplx*)w, ldw, nrhs, (const stfem::cplx*)scol, l,
      (stfem::cplx*)G, g_rhs_stride, g_shift_stride);
  STFEM_LAUNCH_CHECK("bs_update_kernel");
  return STFEM_OK;
}

extern "C" int stfem_apply_global(const stfem_asm* a, const double* Mvals, const double* Avals,
                                  const double* Mt_band, const double* Bt_band, int32_t bw, int32_t nt,
                                  const void* v, void* out, void* work, void* stream) {
  if (!a || !Mvals || !Avals || !Mt_band || !Bt_band || !v || !out || !work)
    return stfem::fail(STFEM_ERR_ARG, "apply_global: null");
  const Asm& A = *reinterpret_cast<const Asm*>(a);
  const int nx = A.n;
  stfem::cplx* MV = (stfem::cplx*)work;
  stfem::cplx* AV = MV + (int64_t)nt * nx;
  int rc;
  if ((rc = stfem_csr_spmv_c(a, Mvals, v, nx, MV, nx, nt, 1.0, 0.0, 0.0, stream))) return rc;
  if ((rc = stfem_csr_spmv_c(a, Avals, v, nx, AV, nx, nt, 1.0, 0.0, 0.0, stream))) return rc;
  int64_t tot = (int64_t)nt * nx;
  stfem::combine_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      nt, nx, bw, Mt_band, Bt_band, MV, AV, (stfem::cplx*)out);
  STFEM_LAUNCH_CHECK("combine_kernel");
  return STFEM_OK;
}

extern "C" int stfem_spacetime_errors(const stfem_asm* a, int32_t kind, const double* breakpoints, int32_t N,
                                      const void* coeffs, int64_t ld, const void* psi0, double* out2,
                                      void* stream) {
  if (!a || !breakpoints || !coeffs || !out2) return stfem::fail(STFEM_ERR_ARG, "spacetime_errors: null");
  Asm& A = *reinterpret_cast<Asm*>(const_cast<stfem_asm*>(a));
  if (A.degree != 1) return stfem::fail(STFEM_ERR_ARG, "spacetime_errors: P1 space only");
  if (kind < 1 || kind > 3) return stfem::fail(STFEM_ERR_ARG, "spacetime_errors: unknown exact solution");
  if (N < 1 || ld < A.n) return stfem::fail(STFEM_ERR_DIM, "spacetime_errors: bad N / ld");
  int rc;
  if ((rc = stfem::upload(A))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t tot = (int64_t)A.ne * N;
  const int nb = (int)((tot + 255) / 256);
  double *d_bp = nullptr, *d_part = nullptr;
  STFEM_CUDA_TRY(cudaMallocAsync((void**)&d_bp, (N + 1) * 8, s));
  STFEM_CUDA_TRY(cudaMallocAsync((void**)&d_part, (2 * (size_t)nb + 2) * 8, s));
  STFEM_CUDA_TRY(cudaMemcpyAsync(d_bp, breakpoints, (N + 1) * 8, cudaMemcpyHostToDevice, s));
  stfem::errors_kernel<<<nb, 256, 0, s>>>(kind, A.d_verts, A.d_elems, A.d_dof, A.ne, d_bp, N,
                                          (const stfem::cplx*)coeffs, ld, (const stfem::cplx*)psi0, d_part);
  STFEM_LAUNCH_CHECK("errors_kernel");
  stfem::sum_partials_kernel<<<1, 256, 0, s>>>(d_part, nb, d_part + 2 * (size_t)nb);
  STFEM_LAUNCH_CHECK("sum_partials_kernel");
  STFEM_CUDA_TRY(cudaMemcpyAsync(out2, d_part + 2 * (size_t)nb, 2 * 8, cudaMemcpyDeviceToHost, s));
  STFEM_CUDA_TRY(cudaFreeAsync(d_bp, s));
  STFEM_CUDA_TRY(cudaFreeAsync(d_part, s));
  STFEM_CUDA_TRY(cudaStreamSynchronize(s));
  out2[0] = sqrt(out2[0]);
  out2[1] = sqrt(out2[1]);
  return STFEM_OK;
}
