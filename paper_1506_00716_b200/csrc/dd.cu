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

#include <cstring>

#include "internal.cuh"

struct nbx_dd {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  int64_t n_send = 0, n_home = 0, n_halo = 0;
  nbx::DBuf<int64_t> send_local;  // indices (in the local array) of particles sent to rank-1
  nbx::DBuf<double> sendbuf;      // packed coordinates (n_send x 3)
  nbx::DBuf<double> recvbuf;      // forces from rank-1 (n_send x 3)
  // NVLink peer path (nbx_dd_p2p_*): one cudaMalloc'd, IPC-exported region
  // per rank = [halo positions in (cap x 3)][halo forces in (cap x 3)][flags]
  int p2p = 0;
  int64_t cap = 0;
  char* p2p_base = nullptr;       // own region
  char* peer_down = nullptr;      // rank-1's region (positions go there)
  char* peer_up = nullptr;        // rank+1's region (halo forces go there)
  unsigned long long seq_pos = 0, seq_f = 0;
  unsigned int* err = nullptr;    // device: set when a wait timed out
  unsigned int err_seen = 0;      // host copy of err[0] taken by nbx_dd_assign's sync
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

// ---- NVLink peer path: the sender stores straight into the receiver's
// region (P2P stores over NVLink), then publishes a sequence number with a
// system-scope release; the receiver's kernel acquires it and consumes the
// data in place (copy into the halo rows / add into the face atoms).  No
// NCCL kernel, proxy thread or host involvement per step.
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// gather rows idx (or the contiguous rows [0, n) when idx == NULL) of x into
// the peer buffer, then the last block to finish publishes `seq`
__global__ void k_p2p_put(const double* __restrict__ x, const int64_t* __restrict__ idx, int64_t n,
                          double* __restrict__ peer_buf, unsigned long long* peer_flag, unsigned long long seq,
                          unsigned int* __restrict__ done) {
  // one double per thread over the flat 3 n rows: every warp stores 256
  // contiguous bytes to the peer (NVLink writes at full width)
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 3 * n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / 3, c = k - 3 * i;
    const int64_t r = idx ? idx[i] : i;
    peer_buf[k] = x[3 * r + c];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(done, 1u);
    if (prev == gridDim.x - 1) {  // every block's stores are fenced
      *done = 0u;
      __threadfence_system();
      st_release_sys(peer_flag, seq);
    }
  }
}

// wait for `seq` in the own flag (bounded spin), then consume the received
// rows: mode 0 copies them to out[0:n), mode 1 adds them to out[idx[i]]
__global__ void k_p2p_take(const unsigned long long* flag, unsigned long long seq, const double* __restrict__ buf,
                           int64_t n, const int64_t* __restrict__ idx, double* __restrict__ out, int mode,
                           unsigned int* err) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    // bounded wait: ~5 s of SM clock, then flag the error instead of hanging
    const long long t0 = clock64();
    while (ld_acquire_sys(flag) < seq && clock64() - t0 < 10000000000ll) __nanosleep(100);
    ok = ld_acquire_sys(flag) >= seq;
    if (!ok) atomicOr(err, 1u);
  }
  __syncthreads();
  if (!ok) return;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 3 * n; k += (int64_t)gridDim.x * blockDim.x) {
    const double v = __ldcv(buf + k);  // written by the peer: bypass L1
    if (mode == 0) {
      out[k] = v;
    } else {
      const int64_t i = k / 3, c = k - 3 * i;
      out[3 * idx[i] + c] += v;  // rows unique per i: deterministic, no atomics
    }
  }
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
  if (d->p2p && (n_send > d->cap || n_halo > d->cap)) {
    // the peer regions hold cap rows each (nbx_dd_p2p_alloc); a larger layout
    // would write past them into the peer's flags
    set_error("nbx_dd_set_layout: n_send=%lld / n_halo=%lld exceed the P2P capacity %lld", (long long)n_send,
              (long long)n_halo, (long long)d->cap);
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

// P2P position exchange in two halves: put my face rows into rank-1's
// region (and publish the sequence number), take rank+1's rows into my halo
// rows (bounded wait on my flag)
// put / take grids: one double per thread over 3 n, at most 4 blocks per SM
// (r02: 16 blocks moved 1.6 MB in ~30 us, ~55 GB/s of NVLink)
static unsigned p2p_blocks(int64_t n) {
  return (unsigned)std::min<int64_t>(std::max<int64_t>((3 * n + 255) / 256, 1), 4 * 148);
}

static void p2p_put_positions(nbx_dd* d, const double* local_pos, cudaStream_t s) {
  const unsigned long long seq = ++d->seq_pos;
  const int64_t cap = d->cap;
  double* peer_pos = reinterpret_cast<double*>(d->peer_down);
  unsigned long long* peer_flag = reinterpret_cast<unsigned long long*>(d->peer_down + 48 * cap);
  count_launch();
  k_p2p_put<<<p2p_blocks(d->n_send), 256, 0, s>>>(local_pos, d->send_local.p, d->n_send, peer_pos, peer_flag, seq, d->err + 1);
}
static void p2p_take_positions(nbx_dd* d, double* local_pos, cudaStream_t s) {
  const int64_t cap = d->cap;
  const double* own = reinterpret_cast<const double*>(d->p2p_base);
  const unsigned long long* flag = reinterpret_cast<const unsigned long long*>(d->p2p_base + 48 * cap);
  count_launch();
  k_p2p_take<<<p2p_blocks(d->n_halo), 256, 0, s>>>(flag, d->seq_pos, own, d->n_halo, nullptr, local_pos + 3 * d->n_home, 0, d->err);
}

// halo forces to the +x owner (peer stores + flag); face forces from the -x
// neighbour added to the send rows (bounded wait on my flag)
static void p2p_put_forces(nbx_dd* d, const double* local_f, cudaStream_t s) {
  const unsigned long long seq = ++d->seq_f;
  const int64_t cap = d->cap;
  double* peer_f = reinterpret_cast<double*>(d->peer_up + 24 * cap);
  unsigned long long* peer_flag = reinterpret_cast<unsigned long long*>(d->peer_up + 48 * cap) + 1;
  count_launch();
  k_p2p_put<<<p2p_blocks(d->n_halo), 256, 0, s>>>(local_f + 3 * d->n_home, nullptr, d->n_halo, peer_f, peer_flag,
                                                  seq, d->err + 2);
}
static void p2p_take_forces(nbx_dd* d, double* local_f, cudaStream_t s) {
  const int64_t cap = d->cap;
  const double* own = reinterpret_cast<const double*>(d->p2p_base + 24 * cap);
  const unsigned long long* flag = reinterpret_cast<const unsigned long long*>(d->p2p_base + 48 * cap) + 1;
  count_launch();
  k_p2p_take<<<p2p_blocks(d->n_send), 256, 0, s>>>(flag, d->seq_f, own, d->n_send, d->send_local.p, local_f, 1,
                                                   d->err);
}

extern "C" int nbx_dd_exchange_positions(nbx_dd_t* d, double* local_pos, void* stream) {
  if (!d || !local_pos) {
    set_error("nbx_dd_exchange_positions: bad argument");
    return NBX_ERR_PARAM;
  }
  if (d->nranks == 1) return NBX_OK;
  cudaStream_t s = to_stream(stream);
  if (d->p2p) {
    p2p_put_positions(d, local_pos, s);
    p2p_take_positions(d, local_pos, s);
    cudaError_t e = cudaGetLastError();
    if (e) {
      set_error("nbx_dd_exchange_positions: %s", cudaGetErrorString(e));
      return NBX_ERR_CUDA;
    }
    return NBX_OK;
  }
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
  if (d->p2p) {
    p2p_put_forces(d, local_f, s);
    p2p_take_forces(d, local_f, s);
    cudaError_t e = cudaGetLastError();
    if (e) {
      set_error("nbx_dd_reduce_forces: %s", cudaGetErrorString(e));
      return NBX_ERR_CUDA;
    }
    return NBX_OK;
  }
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

// NVLink peer path, step 1 (every rank): allocate the own region for up to
// `cap` halo / face particles and export its CUDA IPC handle (64 bytes).
extern "C" int nbx_dd_p2p_alloc(nbx_dd_t* d, int64_t cap, uint8_t handle_out[64]) {
  if (!d || cap < 1 || !handle_out) {
    set_error("nbx_dd_p2p_alloc: bad argument");
    return NBX_ERR_PARAM;
  }
  cudaError_t e;
  cudaIpcMemHandle_t h;
  const size_t bytes = (size_t)48 * cap + 64;
  if ((e = cudaMalloc(reinterpret_cast<void**>(&d->p2p_base), bytes)) ||
      (e = cudaMemset(d->p2p_base, 0, bytes)) ||
      (e = cudaMalloc(reinterpret_cast<void**>(&d->err), 16)) || (e = cudaMemset(d->err, 0, 16)) ||
      (e = cudaIpcGetMemHandle(&h, d->p2p_base))) {
    set_error("nbx_dd_p2p_alloc: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
  memcpy(handle_out, &h, 64);
  d->cap = cap;
  return NBX_OK;
}

// step 2: map the neighbours' regions (rank-1 receives our face positions,
// rank+1 our halo forces) and switch the per-step exchanges to P2P stores.
extern "C" int nbx_dd_p2p_open(nbx_dd_t* d, const uint8_t down_handle[64], const uint8_t up_handle[64]) {
  if (d && !down_handle && !up_handle) {  // collective fallback: back to NCCL send/recv
    d->p2p = 0;
    return NBX_OK;
  }
  if (!d || !d->p2p_base || !down_handle || !up_handle) {
    set_error("nbx_dd_p2p_open: call nbx_dd_p2p_alloc first");
    return NBX_ERR_PARAM;
  }
  cudaIpcMemHandle_t hd, hu;
  memcpy(&hd, down_handle, 64);
  memcpy(&hu, up_handle, 64);
  cudaError_t e = cudaIpcOpenMemHandle(reinterpret_cast<void**>(&d->peer_down), hd, cudaIpcMemLazyEnablePeerAccess);
  if (!e) {
    if (memcmp(down_handle, up_handle, 64) == 0) d->peer_up = d->peer_down;  // N = 2: one neighbour
    else e = cudaIpcOpenMemHandle(reinterpret_cast<void**>(&d->peer_up), hu, cudaIpcMemLazyEnablePeerAccess);
  }
  if (e) {
    set_error("nbx_dd_p2p_open: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  d->p2p = 1;
  return NBX_OK;
}

// non-zero when a peer wait timed out (the exchanged data is then invalid)
extern "C" int nbx_dd_p2p_error(nbx_dd_t* d, int32_t* out) {
  if (!d || !out) return NBX_ERR_PARAM;
  unsigned int h = 0;
  if (d->err) cudaMemcpy(&h, d->err, 4, cudaMemcpyDeviceToHost);
  *out = (int32_t)h;
  return NBX_OK;
}

extern "C" int nbx_dd_p2p_error_seen(const nbx_dd_t* d, int32_t* out) {
  if (!d || !out) return NBX_ERR_PARAM;
  *out = (int32_t)d->err_seen;
  return NBX_OK;
}

extern "C" void nbx_dd_free(nbx_dd_t* d) {
  if (!d) return;
  if (d->peer_down) cudaIpcCloseMemHandle(d->peer_down);
  if (d->peer_up && d->peer_up != d->peer_down) cudaIpcCloseMemHandle(d->peer_up);
  if (d->p2p_base) cudaFree(d->p2p_base);
  if (d->err) cudaFree(d->err);
  if (d->comm) ncclCommDestroy(d->comm);
  d->send_local.drop(0);
  d->sendbuf.drop(0);
  d->recvbuf.drop(0);
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

// migration: new owner + face flag of this rank's particles (k_dd_flags' rule)
__global__ void k_dd_classify(const double* __restrict__ pos, int64_t n, double Lx, const double* __restrict__ bnd,
                              int nranks, double r_comm, int32_t* __restrict__ owner, uint8_t* __restrict__ face) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = wrap_coord(pos[3 * i], Lx);
  int own = 0;
  while (own < nranks - 1 && x >= bnd[own + 1]) ++own;
  owner[i] = own;
  face[i] = (x - bnd[own]) < r_comm;
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
  if ((e = pool_malloc(&tmp, bytes, s))) return e;
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
  if (d->err && (e = cudaMemcpyAsync(&d->err_seen, d->err, sizeof(unsigned int), cudaMemcpyDeviceToHost, s)))
    goto fail;
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

extern "C" int nbx_dd_classify(const double* pos, int64_t n, double Lx, const double* boundaries, int32_t nranks,
                               double r_comm, int32_t* owner, uint8_t* face, void* stream) {
  if (n < 0 || (n > 0 && (!pos || !owner || !face)) || !boundaries || nranks < 1 || nranks > 64) {
    set_error("nbx_dd_classify: bad argument");
    return NBX_ERR_PARAM;
  }
  if (n == 0) return NBX_OK;
  cudaStream_t s = to_stream(stream);
  DBuf<double> bnd;
  cudaError_t e;
  if ((e = bnd.alloc(nranks + 1, s)) ||
      (e = cudaMemcpyAsync(bnd.p, boundaries, sizeof(double) * (nranks + 1), cudaMemcpyHostToDevice, s))) {
    bnd.release(s);
    set_error("nbx_dd_classify: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  count_launch();
  k_dd_classify<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(pos, n, Lx, bnd.p, nranks, r_comm, owner, face);
  e = cudaGetLastError();
  bnd.release(s);
  if (e) {
    set_error("nbx_dd_classify: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  return NBX_OK;
}

__global__ void k_dd_gather_local(const double* __restrict__ pos, const double* __restrict__ q,
                                  const int64_t* __restrict__ typ, const int64_t* __restrict__ home, int64_t nh,
                                  const int64_t* __restrict__ halo, int64_t n_local, double* __restrict__ lpos,
                                  double* __restrict__ lq, int64_t* __restrict__ lt, uint8_t* __restrict__ lhalo) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_local) return;
  const int64_t id = i < nh ? home[i] : halo[i - nh];
  lpos[3 * i] = pos[3 * id];
  lpos[3 * i + 1] = pos[3 * id + 1];
  lpos[3 * i + 2] = pos[3 * id + 2];
  lq[i] = q[id];
  lt[i] = typ[id];
  lhalo[i] = i >= nh;
}

// nbx_dd_assign plus the rank's local arrays in [home; halo] order (the
// inputs of its list step and force pass): positions, charges, types and the
// halo flags, into caller buffers of capacity n.  One call, the syncs of
// nbx_dd_assign only.
extern "C" int nbx_dd_assign_local(nbx_dd_t* d, const double* pos, const double* charges, const int64_t* lj_type,
                                   int64_t n, double Lx, const double* boundaries, double r_comm, int64_t* home,
                                   int64_t* halo, int64_t* send_local, double* local_pos, double* local_q,
                                   int64_t* local_t, uint8_t* local_halo, int64_t* counts_out, void* stream) {
  if (n > 0 && (!charges || !lj_type || !local_pos || !local_q || !local_t || !local_halo)) {
    set_error("nbx_dd_assign_local: bad argument");
    return NBX_ERR_PARAM;
  }
  int st = nbx_dd_assign(d, pos, n, Lx, boundaries, r_comm, home, halo, send_local, counts_out, stream);
  if (st) return st;
  const int64_t nh = counts_out[0], n_local = counts_out[0] + counts_out[1];
  if (n_local > 0) {
    count_launch();
    k_dd_gather_local<<<(unsigned)((n_local + 255) / 256), 256, 0, to_stream(stream)>>>(
        pos, charges, lj_type, home, nh, halo, n_local, local_pos, local_q, local_t, local_halo);
    if (cudaError_t e = cudaGetLastError()) {
      set_error("nbx_dd_assign_local: %s", cudaGetErrorString(e));
      return NBX_ERR_CUDA;
    }
  }
  return NBX_OK;
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

// One domain's force pass with the halo exchange overlapped (NVLink peer
// path): the face rows go to rank-1 first, the work items that read no halo
// coordinate run while the halo travels, the halo rows are taken, the
// boundary work items run, and the halo forces go back / the face forces
// come in (nbx_dd_reduce_forces).  NCCL path and one rank: sequential.
// Sequential peer-path force step with the halo forces leaving early: halo
// rows in, force pass, k_reduce over the clusters that hold halo particles,
// their forces out to the +x owner, k_reduce over the rest, face forces in.
// Results bit-identical to nbx_dd_exchange_positions + nbx_force +
// nbx_dd_reduce_forces.
extern "C" int nbx_dd_force_seq(nbx_dd_t* d, const nbx_list_t* list, const nbx_grid_t* grid, double* local_pos,
                                const double* charges, const int64_t* lj_type, const nbx_params_t* params,
                                const double box[3], int32_t flags, double* f_out, double* e_out, int64_t* bad,
                                void* stream) {
  if (!d || !list || !grid || !local_pos || !params || !box || !f_out || (flags & NBX_FORCE_CANONICAL)) {
    set_error("nbx_dd_force_seq: bad argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  if (d->nranks == 1 || !d->p2p) {
    int st = nbx_dd_exchange_positions(d, local_pos, stream);
    if (!st) st = nbx_force(list, grid, local_pos, charges, lj_type, params, box, nullptr, 0, flags, f_out, e_out, bad,
                            stream);
    if (!st) st = nbx_dd_reduce_forces(d, f_out, stream);
    return st;
  }
  p2p_put_positions(d, local_pos, s);
  p2p_take_positions(d, local_pos, s);
  const std::function<int()> put = [&]() {
    p2p_put_forces(d, f_out, s);
    return NBX_OK;
  };
  int st = force_split(list, grid, local_pos, charges, lj_type, params, box, flags, f_out, e_out, bad, stream,
                       [] { return NBX_OK; }, &put, false);
  if (st) return st;
  p2p_take_forces(d, f_out, s);
  if (cudaError_t e = cudaGetLastError()) {
    set_error("nbx_dd_force_seq: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  return NBX_OK;
}

extern "C" int nbx_dd_force(nbx_dd_t* d, const nbx_list_t* list, const nbx_grid_t* grid, double* local_pos,
                            const double* charges, const int64_t* lj_type, const nbx_params_t* params,
                            const double box[3], int32_t flags, double* f_out, double* e_out, int64_t* bad,
                            void* stream) {
  if (!d || !list || !grid || !local_pos || !params || !box || !f_out || (flags & NBX_FORCE_CANONICAL)) {
    set_error("nbx_dd_force: bad argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  if (d->nranks == 1 || !d->p2p) {
    int st = nbx_dd_exchange_positions(d, local_pos, stream);
    if (!st) st = nbx_force(list, grid, local_pos, charges, lj_type, params, box, nullptr, 0, flags, f_out, e_out, bad,
                            stream);
    if (!st) st = nbx_dd_reduce_forces(d, f_out, stream);
    return st;
  }
  p2p_put_positions(d, local_pos, s);
  int st = force_split(list, grid, local_pos, charges, lj_type, params, box, flags, f_out, e_out, bad, stream,
                       [&]() {
                         p2p_take_positions(d, local_pos, s);
                         return NBX_OK;
                       });
  if (st) return st;
  return nbx_dd_reduce_forces(d, f_out, stream);
}
