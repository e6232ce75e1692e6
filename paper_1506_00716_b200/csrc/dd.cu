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

// ---------------------------------------------------------------- rebuild-time bookkeeping
namespace nbx {

__global__ void k_dd_flags(const double* __restrict__ pos, int64_t n, double Lx, const double* __restrict__ bnd,
                           int nranks, int rank, double r_comm, uint8_t* __restrict__ f_home,
                           uint8_t* __restrict__ f_halo, uint8_t* __restrict__ f_send, int32_t* __restrict__ counts) {
  // per-rank home counts: shared-memory tallies, one global atomic per rank
  // per block (a global atomic per particle on N addresses serialises:
  // ~1 ms at 1.5M particles)
  __shared__ int32_t s_cnt[64];
  for (int r = threadIdx.x; r < nranks; r += blockDim.x) s_cnt[r] = 0;
  __syncthreads();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    const double x = wrap_coord(pos[3 * i], Lx);
    int own = 0;  // searchsorted(bnd[1:-1], x, side="right"), clipped
    while (own < nranks - 1 && x >= bnd[own + 1]) ++own;
    const int nb = (rank + 1) % nranks;
    f_home[i] = own == rank;
    f_send[i] = own == rank && (x - bnd[rank]) < r_comm;
    f_halo[i] = own == nb && (x - bnd[nb]) < r_comm;
    atomicAdd(&s_cnt[own], 1);
  }
  __syncthreads();
  for (int r = threadIdx.x; r < nranks; r += blockDim.x)
    if (s_cnt[r]) atomicAdd(&counts[r], s_cnt[r]);
}

__global__ void k_iota64(int64_t* v, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

__global__ void k_gather_flags(const int64_t* __restrict__ idx, int64_t n, const uint8_t* __restrict__ f,
                               uint8_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = f[idx[i]];
}

__global__ void k_pack_home(const int64_t* __restrict__ ids, const double* __restrict__ pos, int64_t n, int64_t cap,
                            double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= cap) return;
  if (i < n) {
    out[4 * i] = (double)ids[i];
    out[4 * i + 1] = pos[3 * i];
    out[4 * i + 2] = pos[3 * i + 1];
    out[4 * i + 3] = pos[3 * i + 2];
  } else {
    out[4 * i] = -1.0;
  }
}

__global__ void k_unpack_global(const double* __restrict__ in, int64_t n_rec, double* __restrict__ pos) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_rec) return;
  const double id = in[4 * i];
  if (id < 0.0) return;
  const int64_t o = (int64_t)id;
  pos[3 * o] = in[4 * i + 1];
  pos[3 * o + 1] = in[4 * i + 2];
  pos[3 * o + 2] = in[4 * i + 3];
}

}  // namespace nbx

#include <cub/cub.cuh>

template <typename F>
static cudaError_t select_flagged(const int64_t* in, const uint8_t* flags, int64_t* out, int32_t* n_out, int64_t n,
                                  cudaStream_t s) {
  size_t bytes = 0;
  cudaError_t e = cub::DeviceSelect::Flagged(nullptr, bytes, in, flags, out, n_out, (int)n, s);
  if (e) return e;
  void* tmp = nullptr;
  nbx::ensure_pool();
  if ((e = cudaMallocAsync(&tmp, bytes, s))) return e;
  e = cub::DeviceSelect::Flagged(tmp, bytes, in, flags, out, n_out, (int)n, s);
  cudaFreeAsync(tmp, s);
  return e;
}

// Home / halo / send sets of this rank from global positions (the logic of
// dd.SlabDecomposition.assign), ids ascending, plus every rank's home count.
// Outputs (device, capacity n): home, halo, send_local (indices into home).
// counts_out (host): {n_home, n_halo, n_send, home count of rank 0..N-1}.  Syncs once.
extern "C" int nbx_dd_assign(nbx_dd_t* d, const double* pos, int64_t n, double Lx, const double* boundaries,
                             double r_comm, int64_t* home, int64_t* halo, int64_t* send_local, int64_t* counts_out,
                             void* stream) {
  if (!d || (n > 0 && (!pos || !home || !halo || !send_local)) || !boundaries || !counts_out) {
    set_error("nbx_dd_assign: bad argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  const int N = d->nranks;
  DBuf<uint8_t> fh, fl, fs, fsh;
  DBuf<int64_t> iota;
  DBuf<int32_t> cnt;
  DBuf<double> bnd;
  int32_t hc[3 + 64] = {0};
  cudaError_t e;
  if (N > 64) {
    set_error("nbx_dd_assign: at most 64 ranks");
    return NBX_ERR_PARAM;
  }
  if ((e = fh.alloc(n, s)) || (e = fl.alloc(n, s)) || (e = fs.alloc(n, s)) || (e = fsh.alloc(n, s)) ||
      (e = iota.alloc(n, s)) || (e = cnt.alloc(3 + N, s)) || (e = bnd.alloc(N + 1, s)))
    goto fail;
  if ((e = cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * (3 + N), s))) goto fail;
  if ((e = cudaMemcpyAsync(bnd.p, boundaries, sizeof(double) * (N + 1), cudaMemcpyHostToDevice, s))) goto fail;
  if (n > 0) {
    count_launch(2);
    k_dd_flags<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(pos, n, Lx, bnd.p, N, d->rank, r_comm, fh.p, fl.p, fs.p,
                                                           cnt.p + 3);
    k_iota64<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(iota.p, n);
    if ((e = select_flagged<void>(iota.p, fh.p, home, cnt.p, n, s))) goto fail;
    if ((e = select_flagged<void>(iota.p, fl.p, halo, cnt.p + 1, n, s))) goto fail;
  }
  if ((e = cudaMemcpyAsync(hc, cnt.p, sizeof(int32_t) * (3 + N), cudaMemcpyDeviceToHost, s))) goto fail;
  if ((e = cudaStreamSynchronize(s))) goto fail;
  if (n > 0 && hc[0] > 0) {
    // send_local: positions inside the home list whose particle is on the -x face
    count_launch();
    k_gather_flags<<<(unsigned)((hc[0] + 255) / 256), 256, 0, s>>>(home, hc[0], fs.p, fsh.p);
    if ((e = select_flagged<void>(iota.p, fsh.p, send_local, cnt.p + 2, hc[0], s))) goto fail;
    if ((e = cudaMemcpyAsync(&hc[2], cnt.p + 2, sizeof(int32_t), cudaMemcpyDeviceToHost, s))) goto fail;
    if ((e = cudaStreamSynchronize(s))) goto fail;
  }
  counts_out[0] = hc[0];
  counts_out[1] = hc[1];
  counts_out[2] = hc[2];
  for (int r = 0; r < N; ++r) counts_out[3 + r] = hc[3 + r];
  fh.release(s); fl.release(s); fs.release(s); fsh.release(s); iota.release(s); cnt.release(s); bnd.release(s);
  return nbx_dd_set_layout(d, send_local, hc[2], hc[0], hc[1], stream);
fail:
  fh.release(s); fl.release(s); fs.release(s); fsh.release(s); iota.release(s); cnt.release(s); bnd.release(s);
  set_error("nbx_dd_assign: %s", cudaGetErrorString(e));
  return NBX_ERR_CUDA;
}

// Global positions (n x 3, device) from every rank's home rows: one
// ncclAllGather of fixed-capacity (id, x, y, z) records; cap >= every rank's
// home count (known to all ranks from the previous nbx_dd_assign).
extern "C" int nbx_dd_allgather_home(nbx_dd_t* d, const int64_t* home_ids, const double* home_pos, int64_t n_home,
                                     int64_t cap, double* pos_global, void* stream) {
  if (!d || cap < n_home || (n_home > 0 && (!home_ids || !home_pos)) || !pos_global) {
    set_error("nbx_dd_allgather_home: bad argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  DBuf<double> sb, rb;
  cudaError_t e;
  const int64_t tot = cap * d->nranks;
  if ((e = sb.alloc(4 * cap, s)) || (e = rb.alloc(4 * tot, s))) goto fail;
  if (cap > 0) {
    count_launch();
    k_pack_home<<<(unsigned)((cap + 255) / 256), 256, 0, s>>>(home_ids, home_pos, n_home, cap, sb.p);
  }
  if (d->nranks > 1) {
    NCCL_TRY(ncclAllGather(sb.p, rb.p, (size_t)(4 * cap), ncclDouble, d->comm, s));
  } else if (cap > 0 && (e = cudaMemcpyAsync(rb.p, sb.p, sizeof(double) * 4 * cap, cudaMemcpyDeviceToDevice, s))) {
    goto fail;
  }
  if (tot > 0) {
    count_launch();
    k_unpack_global<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(rb.p, tot, pos_global);
  }
  if ((e = cudaGetLastError())) goto fail;
  sb.release(s);
  rb.release(s);
  return NBX_OK;
fail:
  sb.release(s);
  rb.release(s);
  set_error("nbx_dd_allgather_home: %s", cudaGetErrorString(e));
  return NBX_ERR_CUDA;
}
