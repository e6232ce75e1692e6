// Gridding: x/y column binning, z order inside columns, padding to whole
// clusters, bounding boxes.  Replaces gridder.build_cluster_grid
// (/root/reference/pkg/src/clustermd/gridder.py:69-146), bit-identical.
//
// Pipeline (all on `stream`):
//   k_bin       wrap (model.py:147-156), column id (gridder.py:92-94), counts
//   scans       first sorted atom / first cluster of every column
//   k_scatter   atoms into their column segment (unordered)
//   k_colsort   per-column rank by (z, index) == np.lexsort((idx, z, cell))
//               (gridder.py:97), slots, filler padding (gridder.py:104-117)
//   k_bbox      per-cluster AABB (gridder.py:132-134) + real-slot count
#include <atomic>
#include <cstdarg>
#include <cstring>
#include <map>
#include <mutex>
#include <type_traits>
#include <vector>

#include "internal.cuh"

namespace nbx {

__global__ void k_bin(const double* __restrict__ pos, int64_t n, Box box, int64_t cells,
                      double* __restrict__ wpos, int32_t* __restrict__ cell,
                      int32_t* __restrict__ col_count) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = wrap_coord(pos[3 * i + 0], box.L[0]);
  double y = wrap_coord(pos[3 * i + 1], box.L[1]);
  double z = wrap_coord(pos[3 * i + 2], box.L[2]);
  wpos[3 * i + 0] = x;
  wpos[3 * i + 1] = y;
  wpos[3 * i + 2] = z;
  // (pos / L * cells).astype(int64), clamped to cells - 1; pos >= 0 so the
  // truncation is a floor.
  const double c = (double)cells;
  int64_t ix = (int64_t)__dmul_rn(__ddiv_rn(x, box.L[0]), c);
  int64_t iy = (int64_t)__dmul_rn(__ddiv_rn(y, box.L[1]), c);
  ix = ix < cells - 1 ? ix : cells - 1;
  iy = iy < cells - 1 ? iy : cells - 1;
  int32_t cid = (int32_t)(ix * cells + iy);
  cell[i] = cid;
  // warp-aggregated count: neighbouring atoms mostly share a column
  const unsigned mm = __match_any_sync(__activemask(), cid);
  if ((threadIdx.x & 31) == __ffs(mm) - 1) atomicAdd(&col_count[cid], __popc(mm));
}

__global__ void k_col_clusters(const int32_t* __restrict__ col_count, int64_t n_cols, int m, int G,
                               int32_t* __restrict__ ncl, int32_t* __restrict__ ngr) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c < n_cols) {
    const int32_t k = (col_count[c] + m - 1) / m;
    ncl[c] = k;
    ngr[c] = (k + G - 1) / G;
  }
  if (c == n_cols) ncl[c] = ngr[c] = 0;
}

// groups of G consecutive clusters of one column (the search / force work unit)
__global__ void k_groups(const int32_t* __restrict__ col_first, int64_t n_cols, int G,
                         const int32_t* __restrict__ grp_col_first, int32_t* __restrict__ group_first,
                         int32_t* __restrict__ group_nmem) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n_cols) return;
  const int32_t f = col_first[c], ncl = col_first[c + 1] - f;
  const int32_t g0 = grp_col_first[c];
  for (int32_t t = 0; t * G < ncl; ++t) {
    group_first[g0 + t] = f + t * G;
    group_nmem[g0 + t] = min(G, ncl - t * G);
  }
}

__global__ void k_scatter(const int32_t* __restrict__ cell, int64_t n,
                          const int32_t* __restrict__ col_atom_first, int32_t* __restrict__ col_fill,
                          int32_t* __restrict__ sorted) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t c = cell[i];
  // warp-aggregated slot claim (the order inside a column is arbitrary here:
  // k_colsort ranks by (z, index))
  const unsigned mm = __match_any_sync(__activemask(), c);
  const int lane = threadIdx.x & 31, leader = __ffs(mm) - 1;
  int32_t base = 0;
  if (lane == leader) base = atomicAdd(&col_fill[c], __popc(mm));
  base = __shfl_sync(mm, base, leader);
  sorted[col_atom_first[c] + base + __popc(mm & ((1u << lane) - 1u))] = (int32_t)i;
}

constexpr int COLSORT_WARPS = 4;
constexpr int COLSORT_SMEM = 640;  // keys kept in shared memory up to this column size (1.5M tuned grid: ~290 per column)

// One warp per column: rank of every atom by (z, original index).
__global__ void __launch_bounds__(COLSORT_WARPS * 32)
k_colsort(const int32_t* __restrict__ sorted, const int32_t* __restrict__ col_atom_first,
          const int32_t* __restrict__ col_first, int64_t n_cols, int m,
          const double* __restrict__ wpos, int32_t* __restrict__ perm, uint8_t* __restrict__ fill,
          double* __restrict__ cpos, int32_t* __restrict__ inverse_perm,
          int32_t* __restrict__ cell_of_cluster) {
  __shared__ double s_z[COLSORT_WARPS][COLSORT_SMEM];
  __shared__ int32_t s_i[COLSORT_WARPS][COLSORT_SMEM];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = blockIdx.x * (int64_t)COLSORT_WARPS + w;
  if (c >= n_cols) return;
  const int32_t a0 = col_atom_first[c], k = col_atom_first[c + 1] - a0;
  if (k == 0) return;
  const int32_t cl0 = col_first[c], ncl = col_first[c + 1] - cl0;
  for (int t = lane; t < ncl; t += 32) cell_of_cluster[cl0 + t] = (int32_t)c;
  const bool in_smem = k <= COLSORT_SMEM;
  if (in_smem) {
    for (int t = lane; t < k; t += 32) {
      int32_t idx = sorted[a0 + t];
      s_i[w][t] = idx;
      s_z[w][t] = wpos[3 * (int64_t)idx + 2];
    }
  }
  __syncwarp();
  for (int t = lane; t < k; t += 32) {
    const int32_t idx = in_smem ? s_i[w][t] : sorted[a0 + t];
    const double z = in_smem ? s_z[w][t] : wpos[3 * (int64_t)idx + 2];
    int32_t rank = 0;
    if (in_smem) {  // broadcast shared-memory reads, 8 independent compares in flight
#pragma unroll 8
      for (int u = 0; u < k; ++u) {
        const int32_t iu = s_i[w][u];
        const double zu = s_z[w][u];
        rank += (zu < z) || (zu == z && iu < idx);
      }
    } else {
      for (int u = 0; u < k; ++u) {
        const int32_t iu = sorted[a0 + u];
        const double zu = wpos[3 * (int64_t)iu + 2];
        rank += (zu < z) || (zu == z && iu < idx);
      }
    }
    const int64_t base = (int64_t)cl0 * m;
    const double x0 = wpos[3 * (int64_t)idx], y0 = wpos[3 * (int64_t)idx + 1];
    auto put = [&](int32_t r, uint8_t f) {
      const int64_t slot = base + r;
      perm[slot] = idx;
      fill[slot] = f;
      cpos[3 * slot + 0] = x0;
      cpos[3 * slot + 1] = y0;
      cpos[3 * slot + 2] = z;
    };
    put(rank, 0);
    inverse_perm[idx] = (int32_t)(base + rank);
    if (rank == k - 1) {
      for (int32_t r = k; r < ncl * m; ++r) put(r, 1);
    }
  }
}

__global__ void k_bbox(const double* __restrict__ cpos, const uint8_t* __restrict__ fill,
                       int64_t n_clusters, int m, double* __restrict__ bbox, float2* __restrict__ zr,
                       float4* __restrict__ bbf, int8_t* __restrict__ nreal) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n_clusters) return;
  double lo[3], hi[3];
  int nr = 0;
  for (int d = 0; d < 3; ++d) lo[d] = hi[d] = cpos[3 * (c * m) + d];
  for (int a = 0; a < m; ++a) {
    const int64_t s = c * m + a;
    nr += fill[s] == 0;
    for (int d = 0; d < 3; ++d) {
      const double v = cpos[3 * s + d];
      lo[d] = fmin(lo[d], v);
      hi[d] = fmax(hi[d], v);
    }
  }
  for (int d = 0; d < 3; ++d) {
    bbox[6 * c + d] = lo[d];
    bbox[6 * c + 3 + d] = hi[d];
  }
  nreal[c] = (int8_t)nr;
  zr[c] = make_float2(__double2float_rd(lo[2]), __double2float_ru(hi[2]));  // outward-rounded z range
  bbf[2 * c] = make_float4(__double2float_rd(lo[0]), __double2float_rd(lo[1]), __double2float_rd(lo[2]), 0.f);
  bbf[2 * c + 1] = make_float4(__double2float_ru(hi[0]), __double2float_ru(hi[1]), __double2float_ru(hi[2]), 0.f);
}

__global__ void k_scatter_original(const double* __restrict__ in, const int32_t* __restrict__ perm,
                                   const uint8_t* __restrict__ fill, int64_t n_slots, int k,
                                   double* __restrict__ out) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n_slots || fill[s]) return;
  const int64_t o = perm[s];
  for (int d = 0; d < k; ++d) out[o * k + d] = in[s * k + d];
}

static int blocks(int64_t n, int t) { return (int)((n + t - 1) / t); }

}  // namespace nbx

using namespace nbx;

// ---------------------------------------------------------------- errors
static thread_local char g_err[1024] = "";
void nbx::set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
extern "C" const char* nbx_last_error(void) { return g_err; }
extern "C" int nbx_version(void) { return 1; }

// The library's own stream-ordered pool per device (never the device's
// default pool, whose attributes other cudaMallocAsync users in the process --
// torch's async allocator -- would inherit).  Release threshold = max, so
// freed blocks stay mapped across syncs, and pre-grown once so rebuilds do not
// map new pages in the middle of a step.  A 1.5M-atom list generation needs
// several GB (54 M built rows, 18 M entries + their partial forces); the
// default reserve is 24 GB (NBX_POOL_GB), capped at 40 % of free memory.
cudaMemPool_t nbx::device_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (pools[dev]) return pools[dev];
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) return nullptr;
  uint64_t thr = ~0ull;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  double gb = 24.0;
  if (const char* e = getenv("NBX_POOL_GB")) gb = atof(e);
  size_t want = (size_t)(gb * (double)(size_t(1) << 30));
  if (want > free_b / 10 * 4) want = free_b / 10 * 4;
  void* p = nullptr;
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess) {
    if (want > 0 && cudaMallocFromPoolAsync(&p, want, pool, s) == cudaSuccess) cudaFreeAsync(p, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
  cudaGetLastError();
  pools[dev] = pool;
  return pool;
}

namespace {
struct CacheKey {
  int dev;
  cudaStream_t s;
  size_t bytes;
  bool operator<(const CacheKey& o) const {
    if (dev != o.dev) return dev < o.dev;
    if (s != o.s) return s < o.s;
    return bytes < o.bytes;
  }
};
std::mutex g_cmu;
std::map<CacheKey, std::vector<void*>> g_cache;
size_t g_cached = 0;
constexpr size_t kCacheMax = size_t(4) << 30;  // held in the cache at most
}  // namespace

void* nbx::cache_take(size_t bytes, cudaStream_t s) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_cmu);
  auto it = g_cache.find(CacheKey{dev, s, bytes});
  if (it == g_cache.end() || it->second.empty()) return nullptr;
  void* p = it->second.back();
  it->second.pop_back();
  g_cached -= bytes;
  return p;
}

bool nbx::cache_put(void* p, size_t bytes, cudaStream_t s) {
  int dev = 0;
  if (!p || bytes == 0 || cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lk(g_cmu);
  if (g_cached + bytes > kCacheMax) return false;
  g_cache[CacheKey{dev, s, bytes}].push_back(p);
  g_cached += bytes;
  return true;
}

cudaError_t nbx::pool_malloc(void** p, size_t bytes, cudaStream_t s) {
  cudaMemPool_t pool = device_pool();
  if (!pool) return cudaMallocAsync(p, bytes, s);
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

static std::atomic<int64_t> g_launches{0};
void nbx::count_launch(int64_t k) { g_launches += k; }
extern "C" int64_t nbx_launch_count(void) { return g_launches.load(); }

static std::mutex g_tmu;
static bool g_timing = false;
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_events;
bool nbx::timing_enabled() { return g_timing; }
void nbx::timing_record(cudaEvent_t a, cudaEvent_t b) {
  std::lock_guard<std::mutex> lk(g_tmu);
  g_events.emplace_back(a, b);
}
extern "C" void nbx_timing_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_tmu);
  g_timing = on != 0;
}
extern "C" int nbx_timing_query(double* total_ms, int64_t* n_launches) {
  std::lock_guard<std::mutex> lk(g_tmu);
  double tot = 0.0;
  for (auto& ev : g_events) {
    float ms = 0.f;
    if (cudaEventSynchronize(ev.second) != cudaSuccess || cudaEventElapsedTime(&ms, ev.first, ev.second) != cudaSuccess) {
      set_error("nbx_timing_query: event failure");
      return NBX_ERR_CUDA;
    }
    tot += ms;
    cudaEventDestroy(ev.first);
    cudaEventDestroy(ev.second);
  }
  if (total_ms) *total_ms = tot;
  if (n_launches) *n_launches = (int64_t)g_events.size();
  g_events.clear();
  return NBX_OK;
}

// ---------------------------------------------------------------- API
extern "C" int nbx_grid_build(const double* positions, int64_t n, const double box[3], int32_t m,
                              int64_t cells, void* stream, nbx_grid_t** out) {
  if (!out || (n > 0 && !positions) || !box) {
    set_error("nbx_grid_build: null argument");
    return NBX_ERR_PARAM;
  }
  if (m != 1 && m != 2 && m != 4 && m != 8) {
    set_error("cluster size m must be one of (1, 2, 4, 8), got %d", m);
    return NBX_ERR_PARAM;
  }
  if (cells < 1 || n < 0 || n >= (int64_t(1) << 31) / 2) {
    set_error("nbx_grid_build: bad n=%lld or cells=%lld", (long long)n, (long long)cells);
    return NBX_ERR_PARAM;
  }
  for (int d = 0; d < 3; ++d)
    if (!(box[d] > 0.0)) {
      set_error("box lengths must be positive");
      return NBX_ERR_PARAM;
    }
  cudaStream_t s = to_stream(stream);
  nbx_grid* g = new nbx_grid();
  *out = nullptr;
  g->n = n;
  g->m = m;
  g->cells = cells;
  for (int d = 0; d < 3; ++d) g->L[d] = box[d];
  Box bx;
  for (int d = 0; d < 3; ++d) {
    bx.L[d] = box[d];
    bx.invL[d] = 1.0 / box[d];
  }
  const int64_t n_cols = cells * cells;
  DBuf<double> wpos;
  DBuf<int32_t> cell, col_count, col_atom_first, ncl, col_fill, sorted, ngr, grp_col_first;
  auto fail = [&](cudaError_t e) {
    set_error("nbx_grid_build: %s", cudaGetErrorString(e));
    wpos.release(s); cell.release(s); col_count.release(s); col_atom_first.release(s);
    ncl.release(s); col_fill.release(s); sorted.release(s); ngr.release(s); grp_col_first.release(s);
    nbx_grid_free(g);
    return NBX_ERR_CUDA;
  };
  cudaError_t e;
  if ((e = wpos.alloc(3 * n, s)) || (e = cell.alloc(n, s)) || (e = col_count.alloc(n_cols + 1, s)) ||
      (e = col_atom_first.alloc(n_cols + 1, s)) || (e = ncl.alloc(n_cols + 1, s)) ||
      (e = col_fill.alloc(n_cols, s)) || (e = g->col_first.alloc(n_cols + 1, s)) ||
      (e = sorted.alloc(n, s)) || (e = g->inverse_perm.alloc(n, s)) || (e = ngr.alloc(n_cols + 1, s)) ||
      (e = grp_col_first.alloc(n_cols + 1, s)))
    return fail(e);
  if ((e = cudaMemsetAsync(col_count.p, 0, sizeof(int32_t) * (n_cols + 1), s)) ||
      (e = cudaMemsetAsync(col_fill.p, 0, sizeof(int32_t) * n_cols, s)))
    return fail(e);
  if (n > 0) count_launch(), k_bin<<<blocks(n, 256), 256, 0, s>>>(positions, n, bx, cells, wpos.p, cell.p, col_count.p);
  count_launch();
  const int G = 16 / m;
  k_col_clusters<<<blocks(n_cols + 1, 256), 256, 0, s>>>(col_count.p, n_cols, m, G, ncl.p, ngr.p);
  if ((e = exclusive_scan_i32(col_count.p, col_atom_first.p, n_cols + 1, s)) ||
      (e = exclusive_scan_i32(ncl.p, g->col_first.p, n_cols + 1, s)) ||
      (e = exclusive_scan_i32(ngr.p, grp_col_first.p, n_cols + 1, s)))
    return fail(e);
  int32_t nc = 0, ngroups = 0;
  if ((e = cudaMemcpyAsync(&nc, g->col_first.p + n_cols, sizeof(int32_t), cudaMemcpyDeviceToHost, s)) ||
      (e = cudaMemcpyAsync(&ngroups, grp_col_first.p + n_cols, sizeof(int32_t), cudaMemcpyDeviceToHost, s)) ||
      (e = cudaStreamSynchronize(s)))
    return fail(e);
  g->n_clusters = nc;
  g->n_groups = ngroups;
  if ((e = g->group_first.alloc(ngroups, s)) || (e = g->group_nmem.alloc(ngroups, s))) return fail(e);
  if (n_cols > 0)
    count_launch(), k_groups<<<blocks(n_cols, 256), 256, 0, s>>>(g->col_first.p, n_cols, G, grp_col_first.p,
                                                  g->group_first.p, g->group_nmem.p);
  const int64_t ns = (int64_t)nc * m;
  if ((e = g->perm.alloc(ns, s)) || (e = g->fill.alloc(ns, s)) || (e = g->cpos.alloc(3 * ns, s)) ||
      (e = g->cell_of_cluster.alloc(nc, s)) || (e = g->bbox.alloc(6 * (int64_t)nc, s)) ||
      (e = g->zr.alloc(nc, s)) || (e = g->bbf.alloc(2 * (int64_t)nc, s)) ||
      (e = g->nreal.alloc(nc, s)))
    return fail(e);
  if (n > 0) {
    count_launch(3);
    k_scatter<<<blocks(n, 256), 256, 0, s>>>(cell.p, n, col_atom_first.p, col_fill.p, sorted.p);
    k_colsort<<<blocks(n_cols, COLSORT_WARPS), COLSORT_WARPS * 32, 0, s>>>(
        sorted.p, col_atom_first.p, g->col_first.p, n_cols, m, wpos.p, g->perm.p, g->fill.p,
        g->cpos.p, g->inverse_perm.p, g->cell_of_cluster.p);
    k_bbox<<<blocks(nc, 128), 128, 0, s>>>(g->cpos.p, g->fill.p, nc, m, g->bbox.p, g->zr.p, g->bbf.p, g->nreal.p);
  }
  if ((e = cudaGetLastError())) return fail(e);
  wpos.release(s); cell.release(s); col_count.release(s); col_atom_first.release(s);
  ncl.release(s); col_fill.release(s); sorted.release(s); ngr.release(s); grp_col_first.release(s);
  *out = g;
  return NBX_OK;
}

extern "C" int nbx_grid_info(const nbx_grid_t* g, int64_t out[5]) {
  if (!g || !out) {
    set_error("nbx_grid_info: null argument");
    return NBX_ERR_PARAM;
  }
  out[0] = g->n;
  out[1] = g->m;
  out[2] = g->cells;
  out[3] = g->n_clusters;
  out[4] = g->n_slots();
  return NBX_OK;
}

template <typename TD, typename TH>
static cudaError_t download_widen(const TD* d, int64_t count, TH* h, cudaStream_t s) {
  if (!h || count <= 0) return cudaSuccess;
  if (std::is_same<TD, TH>::value) {  // no widening: straight into the caller's buffer
    cudaError_t e = cudaMemcpyAsync(h, d, sizeof(TD) * (size_t)count, cudaMemcpyDeviceToHost, s);
    return e ? e : cudaStreamSynchronize(s);
  }
  TD* tmp = (TD*)malloc(sizeof(TD) * (size_t)count);
  cudaError_t e = cudaMemcpyAsync(tmp, d, sizeof(TD) * (size_t)count, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  if (!e)
    for (int64_t i = 0; i < count; ++i) h[i] = (TH)tmp[i];
  free(tmp);
  return e;
}

extern "C" int nbx_grid_download(const nbx_grid_t* g, int64_t* perm, int64_t* inverse_perm,
                                 uint8_t* fill_mask, int64_t* cell_of_cluster,
                                 double* clustered_positions, double* bboxes, void* stream) {
  if (!g) {
    set_error("nbx_grid_download: null grid");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  const int64_t ns = g->n_slots(), nc = g->n_clusters;
  cudaError_t e;
  if ((e = download_widen(g->perm.p, ns, perm, s)) ||
      (e = download_widen(g->inverse_perm.p, g->n, inverse_perm, s)) ||
      (e = download_widen(g->fill.p, ns, fill_mask, s)) ||
      (e = download_widen(g->cell_of_cluster.p, nc, cell_of_cluster, s)) ||
      (e = download_widen(g->cpos.p, 3 * ns, clustered_positions, s)) ||
      (e = download_widen(g->bbox.p, 6 * nc, bboxes, s))) {
    set_error("nbx_grid_download: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  return NBX_OK;
}

extern "C" const double* nbx_grid_clustered_positions(const nbx_grid_t* g) { return g ? g->cpos.p : nullptr; }

extern "C" int nbx_scatter_to_original(const nbx_grid_t* g, const double* clustered, int32_t k,
                                       double* out, void* stream) {
  if (!g || k < 1) {
    set_error("nbx_scatter_to_original: bad argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double) * (size_t)(g->n * k), s);
  if (!e && g->n_slots() > 0)
    count_launch(), k_scatter_original<<<blocks(g->n_slots(), 256), 256, 0, s>>>(clustered, g->perm.p, g->fill.p,
                                                                  g->n_slots(), k, out);
  if (!e) e = cudaGetLastError();
  if (e) {
    set_error("nbx_scatter_to_original: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  return NBX_OK;
}

extern "C" void nbx_grid_free(nbx_grid_t* g) {
  if (!g) return;
  cudaStream_t s = 0;
  g->perm.drop(s); g->inverse_perm.drop(s); g->fill.drop(s);
  g->cell_of_cluster.drop(s); g->col_first.drop(s); g->cpos.drop(s);
  g->bbox.drop(s); g->zr.drop(s); g->bbf.drop(s); g->nreal.drop(s);
  g->group_first.drop(s); g->group_nmem.drop(s);
  delete g;
}
