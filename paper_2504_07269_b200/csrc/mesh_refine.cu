// GPU uniform (red) refinement of a conforming triangulation with the reference's
// numbering contract (/root/reference/pkg/src/stfem/spatial_mesh.py:121-156 and
// _finish :51-70):
//   * edge midpoints become vertices nv, nv + 1, ... in FIRST-ENCOUNTER order of the
//     edges while walking the elements in order, local edges (01, 12, 20);
//   * every triangle (v0, v1, v2) becomes (v0, m01, m20), (m01, v1, m12), (m20, m12, v2),
//     (m01, m12, m20); the P2 node table row is (v0, v1, v2, m01, m12, m20);
//   * boundary vertices = end points of edges owned by one element (on the refined mesh:
//     the parent's, plus the midpoints of the parent's boundary edges); interior DoFs are
//     numbered in vertex order.
// All of it is deterministic: an open-addressing hash table keyed by the edge
// (atomicCAS insert, atomicMin of the encounter position, atomicAdd of the owner
// count), a flag per encounter position "first encounter of its edge", and an
// exclusive scan of the flags (the rank).  No sort.
#include <stdint.h>

#include "common.cuh"

namespace stfem {
namespace {

constexpr unsigned long long EMPTY = ~0ull;

__device__ __forceinline__ uint32_t hash64(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return (uint32_t)k;
}

__global__ void edge_insert_kernel(const int64_t* __restrict__ el, int ne, int64_t nv, unsigned long long* keys,
                                   int* first, int* count, int* slot_of, uint32_t mask) {
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= 3 * ne) return;
  const int e = pos / 3, j = pos - 3 * e;
  const int64_t a = el[3 * e + j], b = el[3 * e + (j + 1) % 3];
  const unsigned long long key = (unsigned long long)(min(a, b) * nv + max(a, b));
  uint32_t s = hash64(key) & mask;
  for (;;) {
    const unsigned long long prev = atomicCAS(&keys[s], EMPTY, key);
    if (prev == EMPTY || prev == key) break;
    s = (s + 1) & mask;
  }
  atomicMin(&first[s], pos);
  atomicAdd(&count[s], 1);
  slot_of[pos] = s;
}

__global__ void first_flag_kernel(const int* __restrict__ first, const int* __restrict__ slot_of, int n, int* flag) {
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos < n) flag[pos] = first[slot_of[pos]] == pos ? 1 : 0;
}

// exclusive scan of int32 in three passes: 1024 items per block
constexpr int SCAN_ITEMS = 4, SCAN_THREADS = 256, SCAN_BLOCK = SCAN_ITEMS * SCAN_THREADS;
__device__ __forceinline__ int block_exclusive_scan(int v, int* total) {
  __shared__ int wsum[SCAN_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < SCAN_THREADS / 32 ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < SCAN_THREADS / 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < SCAN_THREADS / 32) wsum[lane] = w;
  }
  __syncthreads();
  const int base = warp ? wsum[warp - 1] : 0;
  if (total) *total = wsum[SCAN_THREADS / 32 - 1];
  __syncthreads();
  return base + x - v;
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_local_kernel(const int* __restrict__ in, int n, int* out,
                                                                  int* block_sums) {
  const int base = blockIdx.x * SCAN_BLOCK + threadIdx.x * SCAN_ITEMS;
  int v[SCAN_ITEMS], s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    v[i] = base + i < n ? in[base + i] : 0;
    s += v[i];
  }
  int total;
  int ex = block_exclusive_scan(s, &total);
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    if (base + i < n) out[base + i] = ex;
    ex += v[i];
  }
  if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

// one CTA: exclusive scan of the block sums in place (serial over chunks of SCAN_THREADS)
__global__ void __launch_bounds__(SCAN_THREADS) scan_sums_kernel(int* sums, int nb, int* grand_total) {
  int carry = 0;
  for (int c0 = 0; c0 < nb; c0 += SCAN_THREADS) {
    const int i = c0 + threadIdx.x;
    const int v = i < nb ? sums[i] : 0;
    int total;
    const int ex = block_exclusive_scan(v, &total);
    if (i < nb) sums[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) *grand_total = carry;
}

__global__ void scan_add_kernel(int* out, int n, const int* __restrict__ block_sums) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += block_sums[i / SCAN_BLOCK];
}

int exclusive_scan(const int* in, int n, int* out, int* sums, int* total, cudaStream_t s) {
  const int nb = (n + SCAN_BLOCK - 1) / SCAN_BLOCK;
  scan_local_kernel<<<nb, SCAN_THREADS, 0, s>>>(in, n, out, sums);
  scan_sums_kernel<<<1, SCAN_THREADS, 0, s>>>(sums, nb, total);
  scan_add_kernel<<<(n + 255) / 256, 256, 0, s>>>(out, n, sums);
  STFEM_LAUNCH_CHECK("exclusive_scan");
  return STFEM_OK;
}

// first encounters: midpoint vertex, its rank, its boundary flag
__global__ void midpoint_kernel(const int64_t* __restrict__ el, int ne, int64_t nv, const double* __restrict__ P,
                                const int* __restrict__ flag, const int* __restrict__ rank,
                                const int* __restrict__ slot_of, const int* __restrict__ count, int* mid_rank,
                                double* Pout, uint8_t* bnd) {
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= 3 * ne || !flag[pos]) return;
  const int e = pos / 3, j = pos - 3 * e;
  const int64_t a = el[3 * e + j], b = el[3 * e + (j + 1) % 3];
  const int64_t lo = min(a, b), hi = max(a, b);
  const int r = rank[pos], s = slot_of[pos];
  mid_rank[s] = r;
  Pout[2 * (nv + r)] = (P[2 * lo] + P[2 * hi]) / 2;
  Pout[2 * (nv + r) + 1] = (P[2 * lo + 1] + P[2 * hi + 1]) / 2;
  const bool once = count[s] == 1;
  bnd[nv + r] = once ? 1 : 0;
  if (once) {   // benign race: every writer stores 1
    bnd[lo] = 1;
    bnd[hi] = 1;
  }
}

__global__ void children_kernel(const int64_t* __restrict__ el, int ne, int64_t nv, const int* __restrict__ slot_of,
                                const int* __restrict__ mid_rank, int64_t* elo, int64_t* p2) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const int64_t v0 = el[3 * e], v1 = el[3 * e + 1], v2 = el[3 * e + 2];
  const int64_t m01 = nv + mid_rank[slot_of[3 * e]], m12 = nv + mid_rank[slot_of[3 * e + 1]],
                m20 = nv + mid_rank[slot_of[3 * e + 2]];
  int64_t* o = elo + 12 * (int64_t)e;
  o[0] = v0, o[1] = m01, o[2] = m20;
  o[3] = m01, o[4] = v1, o[5] = m12;
  o[6] = m20, o[7] = m12, o[8] = v2;
  o[9] = m01, o[10] = m12, o[11] = m20;
  int64_t* q = p2 + 6 * (int64_t)e;
  q[0] = v0, q[1] = v1, q[2] = v2, q[3] = m01, q[4] = m12, q[5] = m20;
}

__global__ void interior_flag_kernel(const uint8_t* __restrict__ bnd, int n, int* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = bnd[i] ? 0 : 1;
}

__global__ void interior_dof_kernel(const uint8_t* __restrict__ bnd, const int* __restrict__ rank, int n,
                                    int64_t* dof) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dof[i] = bnd[i] ? -1 : rank[i];
}

}  // namespace
}  // namespace stfem

// verts: device double[2 nv]; elems: device int64[3 ne].  Outputs (device, caller-owned, sized
// for the worst case nv + 3 ne vertices): verts_out double[2 (nv + 3 ne)], elems_out
// int64[12 ne], p2_out int64[6 ne], boundary_out uint8[nv + 3 ne], interior_dof_out
// int64[nv + 3 ne].  *nv_out / *ndof_out (host) receive the refined vertex and interior-DoF
// counts; the call waits for the stream.
extern "C" int stfem_mesh_refine2d(int32_t nv, const double* verts, int32_t ne, const int64_t* elems,
                                   double* verts_out, int64_t* elems_out, int64_t* p2_out, uint8_t* boundary_out,
                                   int64_t* interior_dof_out, int32_t* nv_out, int32_t* ndof_out, void* stream) {
  using namespace stfem;
  if (nv < 3 || ne < 1) return fail(STFEM_ERR_DIM, "mesh_refine2d: nv >= 3 and ne >= 1 required");
  if (!verts || !elems || !verts_out || !elems_out || !p2_out || !boundary_out || !interior_dof_out || !nv_out ||
      !ndof_out)
    return fail(STFEM_ERR_ARG, "mesh_refine2d: null pointer");
  if ((int64_t)3 * ne > (1 << 29)) return fail(STFEM_ERR_DIM, "mesh_refine2d: mesh too large");
  cudaStream_t s = (cudaStream_t)stream;
  const int npos = 3 * ne, nvmax = nv + npos;
  uint32_t cap = 1;
  while (cap < 2u * (uint32_t)npos) cap <<= 1;
  unsigned long long* keys = nullptr;
  int *first = nullptr, *count = nullptr, *mid_rank = nullptr, *slot_of = nullptr, *flag = nullptr, *rank = nullptr,
      *sums = nullptr, *totals = nullptr;
  const int nscan = nvmax > npos ? nvmax : npos;
  auto release = [&]() {
    cudaFree(keys), cudaFree(first), cudaFree(count), cudaFree(mid_rank), cudaFree(slot_of), cudaFree(flag),
        cudaFree(rank), cudaFree(sums), cudaFree(totals);
  };
#define STFEM_TRY_FREE(expr)                       \
  do {                                             \
    cudaError_t _e = (expr);                       \
    if (_e != cudaSuccess) {                       \
      release();                                   \
      return ::stfem::cuda_fail(_e, #expr);        \
    }                                              \
  } while (0)
  STFEM_TRY_FREE(cudaMalloc(&keys, (size_t)cap * 8));
  STFEM_TRY_FREE(cudaMalloc(&first, (size_t)cap * 4));
  STFEM_TRY_FREE(cudaMalloc(&count, (size_t)cap * 4));
  STFEM_TRY_FREE(cudaMalloc(&mid_rank, (size_t)cap * 4));
  STFEM_TRY_FREE(cudaMalloc(&slot_of, (size_t)npos * 4));
  STFEM_TRY_FREE(cudaMalloc(&flag, (size_t)nscan * 4));
  STFEM_TRY_FREE(cudaMalloc(&rank, (size_t)nscan * 4));
  STFEM_TRY_FREE(cudaMalloc(&sums, (size_t)(nscan / SCAN_BLOCK + 2) * 4));
  STFEM_TRY_FREE(cudaMalloc(&totals, 2 * sizeof(int)));
  STFEM_TRY_FREE(cudaMemsetAsync(keys, 0xff, (size_t)cap * 8, s));
  STFEM_TRY_FREE(cudaMemsetAsync(first, 0x7f, (size_t)cap * 4, s));
  STFEM_TRY_FREE(cudaMemsetAsync(count, 0, (size_t)cap * 4, s));
  STFEM_TRY_FREE(cudaMemsetAsync(boundary_out, 0, (size_t)nvmax, s));
  STFEM_TRY_FREE(cudaMemcpyAsync(verts_out, verts, (size_t)nv * 16, cudaMemcpyDeviceToDevice, s));
  const int tb = 256;
  edge_insert_kernel<<<(npos + tb - 1) / tb, tb, 0, s>>>(elems, ne, nv, keys, first, count, slot_of, cap - 1);
  first_flag_kernel<<<(npos + tb - 1) / tb, tb, 0, s>>>(first, slot_of, npos, flag);
  int rc = exclusive_scan(flag, npos, rank, sums, totals, s);
  if (rc) {
    release();
    return rc;
  }
  midpoint_kernel<<<(npos + tb - 1) / tb, tb, 0, s>>>(elems, ne, nv, verts, flag, rank, slot_of, count, mid_rank,
                                                      verts_out, boundary_out);
  children_kernel<<<(ne + tb - 1) / tb, tb, 0, s>>>(elems, ne, nv, slot_of, mid_rank, elems_out, p2_out);
  int h_tot[2] = {0, 0};
  STFEM_TRY_FREE(cudaMemcpyAsync(&h_tot[0], totals, sizeof(int), cudaMemcpyDeviceToHost, s));
  STFEM_TRY_FREE(cudaStreamSynchronize(s));
  const int nvr = nv + h_tot[0];
  interior_flag_kernel<<<(nvr + tb - 1) / tb, tb, 0, s>>>(boundary_out, nvr, flag);
  rc = exclusive_scan(flag, nvr, rank, sums, totals + 1, s);
  if (rc) {
    release();
    return rc;
  }
  interior_dof_kernel<<<(nvr + tb - 1) / tb, tb, 0, s>>>(boundary_out, rank, nvr, interior_dof_out);
  STFEM_TRY_FREE(cudaMemcpyAsync(&h_tot[1], totals + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  STFEM_TRY_FREE(cudaStreamSynchronize(s));
#undef STFEM_TRY_FREE
  release();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "mesh_refine2d");
  *nv_out = nvr;
  *ndof_out = h_tot[1];
  return STFEM_OK;
}
