// Peak probes for the roofline denominators that MEASURED_PEAKS.json lacks:
// FP64 tensor (DMMA) and FP64 CUDA-core (DFMA) throughput.  Register-only
// loops with 8 independent accumulator chains per warp; one CTA of 256
// threads per SM x `ctas_per_sm`.
#include "common.cuh"

namespace stfem {
namespace {

__global__ void __launch_bounds__(256) dmma_probe_kernel(double* sink, int iters) {
  double c[8][4];
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, b0 = 1.0 - a0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int v = 0; v < 4; ++v) c[i][v] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_16x8x4(c[i], a0, a1, b0);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int v = 0; v < 4; ++v) s += c[i][v];
  if (s == 12345.678) sink[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) dfma_probe_kernel(double* sink, int iters) {
  double c[8];
  double a = threadIdx.x * 1e-9, b = 1.0 - a;
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345.678) sink[threadIdx.x] = s;
}

// DMMA and DFMA interleaved in every warp, equal pipe time each if both run at 16 FMA / clk /
// sub-partition (8 DMMAs = 256 issue cycles, 128 DFMAs = 256): do the two FP64 paths share one
// datapath (time doubles, ~37 TFLOP/s total) or add up (~70 TFLOP/s)?
__global__ void __launch_bounds__(256) mixed_probe_kernel(double* sink, int iters) {
  double c[8][4], d[16];
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, b0 = 1.0 - a0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int v = 0; v < 4; ++v) c[i][v] = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) d[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      dmma_16x8x4(c[i], a0, a1, b0);
#pragma unroll
      for (int j = 0; j < 16; ++j) d[j] = fma(d[j], b0, a0);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int v = 0; v < 4; ++v) s += c[i][v];
#pragma unroll
  for (int i = 0; i < 16; ++i) s += d[i];
  if (s == 12345.678) sink[threadIdx.x] = s;
}

// DMMA issue / latency characterisation: CHAINS independent accumulator chains per warp,
// blockDim.x / 32 warps per CTA.  How many DMMAs must be in flight per SM sub-partition to
// reach the pipe's peak decides the warp tile and occupancy of the update kernels.
template <int CHAINS>
__global__ void dmma_chain_probe_kernel(double* sink, int iters) {
  double c[CHAINS][4];
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, b0 = 1.0 - a0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i)
#pragma unroll
    for (int v = 0; v < 4; ++v) c[i][v] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8 / CHAINS; ++r)
#pragma unroll
      for (int i = 0; i < CHAINS; ++i) dmma_16x8x4(c[i], a0, a1, b0);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i)
#pragma unroll
    for (int v = 0; v < 4; ++v) s += c[i][v];
  if (s == 12345.678) sink[threadIdx.x] = s;
}

// Workspace-layout probe: CTA (front f, shift k) -- shifts fastest, as in every level kernel --
// reads (or writes) one contiguous chunk at buf + k * kstride + f * fstride (complex elements).
// "shift-major" (kstride = whole per-shift workspace) against "front-major" (kstride = chunk).
__global__ void __launch_bounds__(128) layout_probe_kernel(cplx* buf, long long kstride, long long fstride,
                                                           int chunk, int nshift, int write, double* sink) {
  const long long inst = blockIdx.x;
  const long long k = inst % nshift, f = inst / nshift;
  cplx* p = buf + k * kstride + f * fstride;
  double acc = 0.0;
  if (write) {
    for (int i = threadIdx.x; i < chunk; i += 128) stc(p + i, cmk(1.0, 2.0));
  } else {
    for (int i = threadIdx.x; i < chunk; i += 128) acc += ldc(p + i).re;
  }
  if (acc == 12345.678) sink[0] = acc;
}

// Store-pattern probe: one CTA per b x b column-major block (lower triangle), 8 warps.
// mode 0: DMMA-epilogue pattern -- a warp stores 16 x 16 sub-blocks, each instruction 8 rows x
// 4 columns (128 contiguous bytes per column); mode 1: the same bytes column by column, a warp
// per column segment (contiguous runs of up to 512 B per instruction).
__global__ void __launch_bounds__(256) store_probe_kernel(cplx* buf, int b, long long bstride, int mode) {
  cplx* U = buf + (long long)blockIdx.x * bstride;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const cplx v = cmk(1.0, 2.0);
  if (mode == 0 || mode == 2) {
    const int nblk = (b + 15) >> 4, nwork = nblk * (nblk + 1) / 2;
    for (int wb = warp; wb < nwork; wb += 8) {
      int bi = 0;
      while ((bi + 1) * (bi + 2) / 2 <= wb) ++bi;
      const int bj = wb - bi * (bi + 1) / 2, rb = bi * 16, cb = bj * 16;
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int row = rb + g + 8 * h, col = cb + ni * 8 + 2 * t + q;
            // mode 2: packed lower triangle, column c starts at c (2 b - c - 1) / 2
            if (row < b && col < b && row >= col)
              stc(U + row + (mode == 2 ? (long long)col * (2 * b - col - 1) / 2 : (long long)col * b), v);
          }
    }
  } else if (mode == 1) {
    for (int col = warp; col < b; col += 8)
      for (int row = col + lane; row < b; row += 32) stc(U + row + (long long)col * b, v);
  } else if (mode == 3) {
    // packed, column by column
    for (int col = warp; col < b; col += 8)
      for (int row = col + lane; row < b; row += 32) stc(U + row + (long long)col * (2 * b - col - 1) / 2, v);
  } else if (mode == 4) {
    // ld padded to a multiple of 8 (128-byte columns), lower part rounded down to an 8-row boundary
    const int ld = (b + 7) & ~7;
    for (int col = warp; col < b; col += 8)
      for (int row = (col & ~7) + lane; row < ld; row += 32) stc(U + row + (long long)col * ld, v);
  } else {
    // mode 5: ld padded to 8; 16 x 16 blocks stored as 256-byte column pieces (lanes 0-15 one column,
    // 16-31 the next): the transposed epilogue.  Diagonal blocks are written whole.
    const int ld = (b + 7) & ~7;
    const int nblk = (b + 15) >> 4, nwork = nblk * (nblk + 1) / 2;
    for (int wb = warp; wb < nwork; wb += 8) {
      int bi = 0;
      while ((bi + 1) * (bi + 2) / 2 <= wb) ++bi;
      const int bj = wb - bi * (bi + 1) / 2, rb = bi * 16, cb = bj * 16;
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int row = rb + (lane & 15), col = cb + 2 * it + (lane >> 4);
        if (row < ld && col < b) stc(U + row + (long long)col * ld, v);
      }
    }
  }
}

}  // namespace
}  // namespace stfem

extern "C" int stfem_probe_store(void* buf, int b, long long bstride, int nblocks, int mode, void* stream) {
  stfem::store_probe_kernel<<<nblocks, 256, 0, (cudaStream_t)stream>>>((stfem::cplx*)buf, b, bstride, mode);
  STFEM_LAUNCH_CHECK("store probe");
  return STFEM_OK;
}

extern "C" int stfem_probe_layout(void* buf, long long kstride, long long fstride, int chunk, int nshift,
                                  int nfront, int write, double* sink, void* stream) {
  stfem::layout_probe_kernel<<<(unsigned)((long long)nshift * nfront), 128, 0, (cudaStream_t)stream>>>(
      (stfem::cplx*)buf, kstride, fstride, chunk, nshift, write, sink);
  STFEM_LAUNCH_CHECK("layout probe");
  return STFEM_OK;
}

// 8 DMMAs per iteration per warp on `chains` (1, 2, 4 or 8) independent accumulators
extern "C" int stfem_probe_dmma_chains(int chains, int warps_per_cta, int blocks, int iters, double* sink,
                                       double* flops, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int th = 32 * warps_per_cta;
  switch (chains) {
    case 1: stfem::dmma_chain_probe_kernel<1><<<blocks, th, 0, s>>>(sink, iters); break;
    case 2: stfem::dmma_chain_probe_kernel<2><<<blocks, th, 0, s>>>(sink, iters); break;
    case 4: stfem::dmma_chain_probe_kernel<4><<<blocks, th, 0, s>>>(sink, iters); break;
    default: stfem::dmma_chain_probe_kernel<8><<<blocks, th, 0, s>>>(sink, iters); break;
  }
  *flops = (double)blocks * warps_per_cta * iters * 8.0 * (2.0 * 16 * 8 * 4);
  STFEM_LAUNCH_CHECK("probe");
  return STFEM_OK;
}

// kind 0 = DMMA (flops = 2*16*8*4 per mma per warp), 1 = DFMA, 2 = both interleaved.  Returns the
// real fp64 flop count executed in *flops; caller times it with events.
extern "C" int stfem_probe_launch(int kind, int blocks, int iters, double* sink, double* flops,
                                  void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  double warps = blocks * 8.0;
  if (kind == 0) {
    stfem::dmma_probe_kernel<<<blocks, 256, 0, s>>>(sink, iters);
    *flops = warps * iters * 8.0 * (2.0 * 16 * 8 * 4);
  } else if (kind == 2) {
    stfem::mixed_probe_kernel<<<blocks, 256, 0, s>>>(sink, iters);
    *flops = warps * iters * 8.0 * (2.0 * 16 * 8 * 4) + blocks * 256.0 * iters * 128.0 * 2.0;
  } else {
    stfem::dfma_probe_kernel<<<blocks, 256, 0, s>>>(sink, iters);
    *flops = blocks * 256.0 * iters * 8.0 * 2.0;
  }
  STFEM_LAUNCH_CHECK("probe");
  return STFEM_OK;
}
