// stfem_fdm_solve / stfem_comm_*: the whole FD solve (steps 2-4)
// behind one C call, single-GPU or sharded over an NCCL communicator
// (SURVEY.md §8b, §8e), so a host without Python can drive it.
//
// Sharded data path (P ranks, one process per GPU; matches distributed.py):
//   F_p (n_t, n_rhs, c), c = ceil(n_x / P): this rank's spatial columns
//   (2) G_p = Y F_p                      K3p / K3, N = n_rhs c
//   a2a #1: block q of G_p (its n_t / P shifts, one contiguous slab) -> rank q;
//       the receive buffer is (P, n_t / P, n_rhs, c) = every column of the local shifts
//   (3) factor + solve of the local shifts straight from the receive buffer
//       (chunked stfem_bv_layout, no repack)
//   a2a #2 returns the (n_t, n_rhs, c) shards
//   (4) Psi_p = X W_p
// The exchange is a grouped ncclSend / ncclRecv (all NCCL versions; NVLink /
// NVSwitch underneath).  NCCL is bound at run time (dlopen of libnccl.so.2 --
// the copy torch already loaded when there is one), so the library has no
// link-time NCCL dependency and single-GPU hosts need none at all.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <mutex>

#include "plan.h"

namespace stfem {
int factor_solve(Plan& P, const double* Mv, const double* Av, const cplx* lam, int nshift, int nrhs, const cplx* G,
                 cplx* W, stfem_bv_layout lay, cudaStream_t stream);
}

namespace {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  std::string error;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the copy already in the process (torch's)
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.error = std::string("NCCL not found: ") + (dlerror() ? dlerror() : "dlopen(libnccl.so.2) failed");
      return;
    }
    api.handle = h;
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p && api.error.empty()) api.error = std::string("NCCL symbol missing: ") + name;
      return p;
    };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    api.GetVersion = (decltype(api.GetVersion))sym("ncclGetVersion");
  });
  return api;
}

int nccl_fail(ncclResult_t r, const char* where) {
  NcclApi& n = nccl();
  return stfem::fail(STFEM_ERR_NCCL, std::string(where) + ": " + (n.GetErrorString ? n.GetErrorString(r) : "NCCL error"));
}

#define STFEM_NCCL_TRY(expr)                                \
  do {                                                      \
    ncclResult_t _r = (expr);                               \
    if (_r != ncclSuccess) return nccl_fail(_r, #expr);     \
  } while (0)

}  // namespace

struct stfem_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
};

extern "C" int stfem_comm_unique_id(uint8_t unique_id[128]) {
  if (!unique_id) return stfem::fail(STFEM_ERR_ARG, "comm_unique_id: null pointer");
  NcclApi& n = nccl();
  if (!n.error.empty()) return stfem::fail(STFEM_ERR_NCCL, n.error);
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  STFEM_NCCL_TRY(n.GetUniqueId(&id));
  memcpy(unique_id, &id, 128);
  return STFEM_OK;
}

extern "C" int stfem_comm_init(const uint8_t unique_id[128], int32_t nranks, int32_t rank, stfem_comm** out) {
  if (!out || !unique_id) return stfem::fail(STFEM_ERR_ARG, "comm_init: null pointer");
  if (nranks < 1 || rank < 0 || rank >= nranks) return stfem::fail(STFEM_ERR_ARG, "comm_init: bad rank / nranks");
  NcclApi& n = nccl();
  if (!n.error.empty()) return stfem::fail(STFEM_ERR_NCCL, n.error);
  ncclUniqueId id;
  memcpy(&id, unique_id, 128);
  stfem_comm* c = new stfem_comm();
  c->nranks = nranks;
  c->rank = rank;
  ncclResult_t r = n.CommInitRank(&c->comm, nranks, id, rank);   // binds the current CUDA device
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  *out = c;
  return STFEM_OK;
}

extern "C" int stfem_comm_destroy(stfem_comm* c) {
  if (!c) return STFEM_OK;
  if (c->comm) nccl().CommDestroy(c->comm);
  delete c;
  return STFEM_OK;
}

extern "C" int stfem_comm_info(const stfem_comm* c, int32_t* nranks, int32_t* rank, int32_t* nccl_version) {
  if (nranks) *nranks = c ? c->nranks : 1;
  if (rank) *rank = c ? c->rank : 0;
  if (nccl_version) {
    int v = 0;
    NcclApi& n = nccl();
    if (n.error.empty() && n.GetVersion) n.GetVersion(&v);
    *nccl_version = v;
  }
  return STFEM_OK;
}

// block q of `send` (count complex each) -> rank q; block p of `recv` <- rank p
extern "C" int stfem_comm_all_to_all(stfem_comm* c, const void* send, void* recv, int64_t count, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!send || !recv || count < 0) return stfem::fail(STFEM_ERR_ARG, "comm_all_to_all: bad argument");
  if (!c) {
    STFEM_CUDA_TRY(cudaMemcpyAsync(recv, send, (size_t)count * 16, cudaMemcpyDeviceToDevice, s));
    return STFEM_OK;
  }
  const int P = c->nranks;
  NcclApi& n = nccl();
  const char* sb = (const char*)send;
  char* rb = (char*)recv;
  STFEM_NCCL_TRY(n.GroupStart());
  for (int q = 0; q < P; ++q) {
    // complex128 travels as pairs of float64 (NCCL has no complex type)
    STFEM_NCCL_TRY(n.Send(sb + (size_t)q * count * 16, (size_t)count * 2, ncclFloat64, q, c->comm, s));
    STFEM_NCCL_TRY(n.Recv(rb + (size_t)q * count * 16, (size_t)count * 2, ncclFloat64, q, c->comm, s));
  }
  STFEM_NCCL_TRY(n.GroupEnd());
  return STFEM_OK;
}

extern "C" int stfem_fdm_solve(stfem_plan* plan, stfem_comm* comm, const double* Mvals, const double* Avals,
                               const stfem_fd_factors* tf, const void* F, void* Psi, void* work, int32_t nrhs,
                               void* stream) {
  if (!plan || !tf || !F || !Psi || !work || !Mvals || !Avals)
    return stfem::fail(STFEM_ERR_ARG, "fdm_solve: null pointer");
  if (F == Psi || F == work || Psi == work)
    return stfem::fail(STFEM_ERR_ARG, "fdm_solve: F, Psi and work must be three distinct buffers");
  stfem::Plan& P = *reinterpret_cast<stfem::Plan*>(plan);
  const int nt = tf->nt, nx = P.n;
  if (nt < 1 || nrhs < 1 || !tf->lam) return stfem::fail(STFEM_ERR_DIM, "fdm_solve: n_t >= 1, n_rhs >= 1 and lam required");
  const bool paired = tf->A_fwd && tf->A_back;
  if (!paired && !(tf->X && tf->Y))
    return stfem::fail(STFEM_ERR_ARG, "fdm_solve: either the paired tables or X and Y are required");
  const int R = comm ? comm->nranks : 1, rank = comm ? comm->rank : 0;
  if (nt % R) return stfem::fail(STFEM_ERR_DIM, "fdm_solve: n_t must be divisible by the number of ranks");
  const int ntl = nt / R;
  const bool sharded = comm != nullptr;                    // shard layout + exchange (also with one rank)
  const int64_t c = sharded ? (nx + R - 1) / R : nx;       // spatial columns of a shard
  // transforms: one GEMM over N = n_rhs c columns (shard layout (n_t, n_rhs, c)); the single-GPU
  // BlockVector layout (n_rhs, n_t, n_x) is a batch of n_rhs matrices instead
  const int64_t ncols = sharded ? (int64_t)nrhs * c : nx;
  const int batch = sharded ? 1 : nrhs;
  const int64_t ld = ncols, bstride = (int64_t)nt * nx;
  auto fwd = [&](const void* in, void* out) -> int {
    if (paired)
      return stfem_transform_pair_fwd(tf->A_fwd, tf->mrows_fwd, nt, tf->rows_fwd, tf->scale_fwd, tf->nsrc, in, ld,
                                      out, ld, ncols, batch, bstride, bstride, stream);
    return stfem_time_transform(tf->Y, nt, in, ld, out, ld, ncols, batch, bstride, bstride, stream);
  };
  auto back = [&](void* in, void* out) -> int {
    if (paired)
      return stfem_transform_pair_back(tf->A_back, nt, tf->mix_rows, tf->mix_coef, tf->nmix, in, ld, out, ld, ncols,
                                       batch, bstride, bstride, stream);
    return stfem_time_transform(tf->X, nt, in, ld, out, ld, ncols, batch, bstride, bstride, stream);
  };
  const stfem::cplx* lam = (const stfem::cplx*)tf->lam + (size_t)rank * ntl;
  int rc;
  // the transforms of this entry point carry no column maps: G and W are in the operators' numbering,
  // whatever an earlier stfem_plan_set_io_permuted call left in the plan
  P.io_permuted = false;
  // at most 16 right-hand sides per factor_solve call (and fewer for very large fronts)
  int32_t step = 16;
  if ((rc = stfem_plan_max_rhs(plan, &step))) return rc;
  if (!sharded) {
    if ((rc = fwd(F, Psi))) return rc;                                            // (2) F -> Psi
    const stfem_bv_layout lay{(int64_t)nt * nx, nx, nx, 0};
    for (int r0 = 0; r0 < nrhs; r0 += step) {                                      // (3) Psi -> work
      const int nr = std::min<int>(step, nrhs - r0);
      const size_t off = (size_t)r0 * lay.rhs_stride;
      if ((rc = stfem::factor_solve(P, Mvals, Avals, lam, nt, nr, (const stfem::cplx*)Psi + off,
                                    (stfem::cplx*)work + off, lay, (cudaStream_t)stream)))
        return rc;
    }
    return back(work, Psi);                                                        // (4) work -> Psi
  }
  const int64_t slab = (int64_t)ntl * nrhs * c;                                    // complex per peer
  if ((rc = fwd(F, Psi))) return rc;                                               // (2) G_p in Psi
  if ((rc = stfem_comm_all_to_all(comm, Psi, work, slab, stream))) return rc;      // a2a #1 -> work (P, ntl, nrhs, c)
  const stfem_bv_layout lay{c, (int64_t)nrhs * c, c, slab};
  for (int r0 = 0; r0 < nrhs; r0 += step) {                                        // (3) work -> Psi (same layout)
    const int nr = std::min<int>(step, nrhs - r0);
    const size_t off = (size_t)r0 * lay.rhs_stride;
    if ((rc = stfem::factor_solve(P, Mvals, Avals, lam, ntl, nr, (const stfem::cplx*)work + off,
                                  (stfem::cplx*)Psi + off, lay, (cudaStream_t)stream)))
      return rc;
  }
  if ((rc = stfem_comm_all_to_all(comm, Psi, work, slab, stream))) return rc;      // a2a #2 -> work (n_t, nrhs, c)
  return back(work, Psi);                                                          // (4)
}
