// Domain-decomposition halo exchange over NCCL, driven from the library on
// the caller's compute stream (no extra streams, events or host syncs per
// step).  Geometry/bookkeeping lives in paper_1506_00716_b200/dd.py; this
// file moves the bytes:
//   nbx_dd_exchange_positions: pack the home particles near the -x face ->
//       ncclSend to rank-1, ncclRecv the halo from rank+1 straight into the
//       tail of the local coordinate array (one NCCL group);
//   nbx_dd_reduce_forces: ncclSend the halo forces to rank+1, ncclRecv the
//       forces rank-1 computed on our face particles, add them (one kernel).
#include <nccl.h>

#include "internal.cuh"

struct nbx_dd {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  int64_t n_send = 0, n_home = 0, n_halo = 0;
  nbx::DBuf<int64_t> send_local;  // indices (in the local array) of particles sent to rank-1
  nbx::DBuf<double> sendbuf;      // packed coordinates (n_send x 3)
  nbx::DBuf<double> recvbuf;      // forces from rank-1 (n_send x 3)
};

namespace nbx {

__global__ void k_pack(const double* __restrict__ x, const int64_t* __restrict__ idx, int64_t n,
                       double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = idx[i];
  out[3 * i] = x[3 * s];
  out[3 * i + 1] = x[3 * s + 1];
  out[3 * i + 2] = x[3 * s + 2];
}

__global__ void k_unpack_add(double* __restrict__ f, const int64_t* __restrict__ idx, int64_t n,
                             const double* __restrict__ in) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = idx[i];  // unique per i: no atomics, deterministic
  f[3 * s] += in[3 * i];
  f[3 * s + 1] += in[3 * i + 1];
  f[3 * s + 2] += in[3 * i + 2];
}

}  // namespace nbx

using namespace nbx;

#define NCCL_TRY(x)                                                           \
  do {                                                                        \
    ncclResult_t r_ = (x);                                                    \
    if (r_ != ncclSuccess) {                                                  \
      set_error("%s: %s", #x, ncclGetErrorString(r_));                        \
      return NBX_ERR_CUDA;                                                    \
    }                                                                         \
  } while (0)

extern "C" int nbx_dd_unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  static_assert(sizeof(id.internal) == 128, "ncclUniqueId size");
  for (int i = 0; i < 128; ++i) out[i] = (uint8_t)id.internal[i];
  return NBX_OK;
}

extern "C" int nbx_dd_create(const uint8_t uid[128], int32_t nranks, int32_t rank, nbx_dd_t** out) {
  if (!uid || !out || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("nbx_dd_create: bad argument");
    return NBX_ERR_PARAM;
  }
  ncclUniqueId id;
  for (int i = 0; i < 128; ++i) id.internal[i] = (char)uid[i];
  nbx_dd* d = new nbx_dd();
  d->rank = rank;
  d->nranks = nranks;
  ncclResult_t r = ncclCommInitRank(&d->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    set_error("ncclCommInitRank: %s", ncclGetErrorString(r));
    delete d;
    return NBX_ERR_CUDA;
  }
  *out = d;
  return NBX_OK;
}

extern "C" int nbx_dd_set_layout(nbx_dd_t* d, const int64_t* send_local, int64_t n_send, int64_t n_home,
                                 int64_t n_halo, void* stream) {
  if (!d || (n_send > 0 && !send_local) || n_send < 0 || n_home < 0 || n_halo < 0) {
    set_error("nbx_dd_set_layout: bad argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  cudaError_t e;
  if (d->send_local.n < n_send && (e = d->send_local.alloc(n_send, s))) goto fail;
  if (d->sendbuf.n < 3 * n_send && (e = d->sendbuf.alloc(3 * n_send, s))) goto fail;
  if (d->recvbuf.n < 3 * n_send && (e = d->recvbuf.alloc(3 * n_send, s))) goto fail;
  if (n_send > 0 &&
      (e = cudaMemcpyAsync(d->send_local.p, send_local, sizeof(int64_t) * n_send, cudaMemcpyDeviceToDevice, s)))
    goto fail;
  d->n_send = n_send;
  d->n_home = n_home;
  d->n_halo = n_halo;
  return NBX_OK;
fail:
  set_error("nbx_dd_set_layout: %s", cudaGetErrorString(e));
  return NBX_ERR_CUDA;
}

extern "C" int nbx_dd_exchange_positions(nbx_dd_t* d, double* local_pos, void* stream) {
  if (!d || !local_pos) {
    set_error("nbx_dd_exchange_positions: bad argument");
    return NBX_ERR_PARAM;
  }
  if (d->nranks == 1) return NBX_OK;
  cudaStream_t s = to_stream(stream);
  if (d->n_send > 0) {
    count_launch();
    k_pack<<<(unsigned)((d->n_send + 255) / 256), 256, 0, s>>>(local_pos, d->send_local.p, d->n_send, d->sendbuf.p);
  }
  const int down = (d->rank - 1 + d->nranks) % d->nranks, up = (d->rank + 1) % d->nranks;
  NCCL_TRY(ncclGroupStart());
  if (d->n_send > 0) NCCL_TRY(ncclSend(d->sendbuf.p, (size_t)(3 * d->n_send), ncclDouble, down, d->comm, s));
  if (d->n_halo > 0)
    NCCL_TRY(ncclRecv(local_pos + 3 * d->n_home, (size_t)(3 * d->n_halo), ncclDouble, up, d->comm, s));
  NCCL_TRY(ncclGroupEnd());
  cudaError_t e = cudaGetLastError();
  if (e) {
    set_error("nbx_dd_exchange_positions: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  return NBX_OK;
}

extern "C" int nbx_dd_reduce_forces(nbx_dd_t* d, double* local_f, void* stream) {
  if (!d || !local_f) {
    set_error("nbx_dd_reduce_forces: bad argument");
    return NBX_ERR_PARAM;
  }
  if (d->nranks == 1) return NBX_OK;
  cudaStream_t s = to_stream(stream);
  const int down = (d->rank - 1 + d->nranks) % d->nranks, up = (d->rank + 1) % d->nranks;
  NCCL_TRY(ncclGroupStart());
  if (d->n_halo > 0) NCCL_TRY(ncclSend(local_f + 3 * d->n_home, (size_t)(3 * d->n_halo), ncclDouble, up, d->comm, s));
  if (d->n_send > 0) NCCL_TRY(ncclRecv(d->recvbuf.p, (size_t)(3 * d->n_send), ncclDouble, down, d->comm, s));
  NCCL_TRY(ncclGroupEnd());
  if (d->n_send > 0) {
    count_launch();
    k_unpack_add<<<(unsigned)((d->n_send + 255) / 256), 256, 0, s>>>(local_f, d->send_local.p, d->n_send,
                                                                      d->recvbuf.p);
  }
  cudaError_t e = cudaGetLastError();
  if (e) {
    set_error("nbx_dd_reduce_forces: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  return NBX_OK;
}

extern "C" int nbx_dd_allreduce_sum(nbx_dd_t* d, double* buf, int64_t n, void* stream) {
  if (!d || (n > 0 && !buf)) {
    set_error("nbx_dd_allreduce_sum: bad argument");
    return NBX_ERR_PARAM;
  }
  if (d->nranks == 1 || n == 0) return NBX_OK;
  NCCL_TRY(ncclAllReduce(buf, buf, (size_t)n, ncclDouble, ncclSum, d->comm, to_stream(stream)));
  return NBX_OK;
}

extern "C" void nbx_dd_free(nbx_dd_t* d) {
  if (!d) return;
  if (d->comm) ncclCommDestroy(d->comm);
  d->send_local.release(0);
  d->sendbuf.release(0);
  d->recvbuf.release(0);
  delete d;
}
