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

}  // namespace
}  // namespace stfem

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
