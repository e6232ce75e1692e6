// Internal (device-resident) data structures of the nbx library.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <vector>

#include "common.cuh"
#include "nbx.h"

namespace nbx {

// The library's private stream-ordered pool on the current device (grid.cu):
// freed memory stays mapped across syncs (the default release threshold of 0
// returns it to the driver at every sync and makes the next allocation re-map
// pages -- milliseconds per rebuild).  All library allocations go through it.
cudaMemPool_t device_pool();
cudaError_t pool_malloc(void** p, size_t bytes, cudaStream_t s);

// Per-call temporaries are recycled through a small host-side cache of freed
// blocks keyed by (device, stream, size class) before the stream-ordered pool:
// a list step allocates and frees ~60 temporaries, and the ~2 us host cost of
// each pool call was a visible share of the host time that leaves the GPU idle
// between the list step's small kernels.  A block is reused only on the
// stream it was freed on (stream order keeps that safe); long-lived buffers
// of grids and lists are returned to the pool directly (drop()).
void* cache_take(size_t bytes, cudaStream_t s);
bool cache_put(void* p, size_t bytes, cudaStream_t s);

// Device buffer with stream-ordered allocation.
template <typename T>
struct DBuf {
  T* p = nullptr;
  int64_t n = 0;
  size_t bytes = 0;
  cudaError_t alloc(int64_t count, cudaStream_t s) {
    release(s);
    n = count;
    if (count <= 0) return cudaSuccess;
    bytes = size_class(sizeof(T) * (size_t)count);
    if (void* c = cache_take(bytes, s)) {
      p = reinterpret_cast<T*>(c);
      return cudaSuccess;
    }
    return pool_malloc(reinterpret_cast<void**>(&p), bytes, s);
  }
  // round up to {1, 1.25, 1.5, 1.75} x 2^k so that the per-rebuild buffers of
  // slightly different sizes reuse the same pool blocks
  static size_t size_class(size_t b) {
    if (b <= 4096) return b;
    size_t p = 1;
    while ((p << 1) <= b) p <<= 1;
    const size_t q = p >> 2;
    return ((b + q - 1) / q) * q;
  }
  void release(cudaStream_t s) {
    if (p && !cache_put(p, bytes, s)) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
    bytes = 0;
  }
  void drop(cudaStream_t s) {  // back to the pool (buffers of grids / lists)
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
    bytes = 0;
  }
};

// Clustered layout (gridder.ClusterGrid, gridder.py:23-66).
struct Grid {
  int64_t n = 0;        // particles
  int m = 0;            // cluster size
  int64_t cells = 0;    // columns per side
  int64_t n_clusters = 0;
  double L[3] = {0, 0, 0};
  DBuf<int32_t> perm;           // (n_slots) slot -> original index
  DBuf<int32_t> inverse_perm;   // (n)
  DBuf<uint8_t> fill;           // (n_slots)
  DBuf<int32_t> cell_of_cluster;// (n_clusters)
  DBuf<int32_t> col_first;      // (cells^2 + 1) first cluster of each column
  DBuf<double> cpos;            // (n_slots, 3) wrapped build-time positions
  DBuf<double> bbox;            // (n_clusters, 6) lo xyz, hi xyz
  DBuf<float2> zr;              // (n_clusters) z range rounded outward (search prefilter)
  DBuf<float4> bbf;             // (n_clusters, 2) FP32 box rounded outward (search)
  DBuf<int8_t> nreal;           // (n_clusters) real (non-filler) slots
  // search / force groups: G = 16/m consecutive clusters of one column
  int64_t n_groups = 0;
  DBuf<int32_t> group_first;    // (n_groups) first member cluster
  DBuf<int32_t> group_nmem;     // (n_groups)
  int64_t n_slots() const { return n_clusters * m; }
};

// Force workspace cached on a list (lazily sized on first force call).
struct ForceWork {
  DBuf<float4> xyzq;      // (n_slots) cluster-local FP32 positions (near-build image) + charge
  DBuf<int32_t> type;     // (n_slots)
  DBuf<float4> part_i;    // (n_slots) i-side partial forces
  DBuf<float4> part_j;    // (n_entries * m) or (n_rows * m) j-side partials
  DBuf<double> e_grp;     // (2 * n_work_groups) per-group energies
  DBuf<unsigned int> scalars;   // [0] max displacement bits, [1..2] bad key (u64)
  bool scalars_clean = false;   // reset by the last call's k_energy (skip k_init_scalars)
  DBuf<float4> lj;        // (t*t) {6 c6, 12 c12, shift_lj, 0}
  std::vector<double> lj_key;  // host copy of what `lj` was built from (skip re-uploads)
  // transposed index: entries (or rows) sorted by j-cluster
  DBuf<int32_t> t_first;  // (n_clusters + 1)
  DBuf<int32_t> t_items;  // (n_entries)
  DBuf<int32_t> t_pos;    // (n_entries) inverse of t_items: entry -> its slot in j-cluster order
  bool t_ready = false;
  bool t_split = false;   // t_first has 2 n_clusters + 1 bounds (inner-list split, k_reduce)
  DBuf<int32_t> tc_first; // canonical-row transpose
  DBuf<int32_t> tc_items;
  bool tc_ready = false;
};

// Cluster-pair list (pairlist.ClusterPairList, pairlist.py:27-94) plus the
// grouped force layout: G = 16/m consecutive clusters of one column form a
// group; an entry is (group, j-cluster) with the masks of every member.
struct List {
  int m = 0;
  int G = 0;
  int64_t n_clusters = 0;
  int64_t n_rows = 0;
  int64_t n_groups = 0;
  int64_t n_entries = 0;         // entry storage (>= the live count when !entries_exact)
  bool entries_exact = true;      // n_live known on the host
  int64_t n_live = -1;            // live entries (-1: == n_entries)
  double r_list = 0.0;
  double L[3] = {0, 0, 0};
  const double* bbox = nullptr;  // the grid's boxes (frame of `delta`); the grid outlives its lists
  // canonical CSR: materialised from the entries on demand (ensure_rows);
  // the force path never needs it
  bool rows_ready = false;
  DBuf<int32_t> offsets;    // (n_clusters + 1)
  DBuf<int32_t> j;          // (n_rows)
  DBuf<uint64_t> mask;      // (n_rows)
  DBuf<float4> delta;       // (n_rows) j-local -> i-local offset (image included), lazy
  bool delta_ready = false;
  // groups / entries
  DBuf<int32_t> group_first;  // (n_groups) first member cluster
  DBuf<int32_t> group_nmem;   // (n_groups)
  DBuf<int32_t> group_order;  // (n_groups) force-kernel work order (descending entry count)
  DBuf<int32_t> ent_offsets;  // (n_groups + 1)
  DBuf<int32_t> ent_j;        // (n_entries)
  DBuf<float4> ent_delta;    // (n_entries) j-local -> group-local offset, w = slack
  DBuf<uint64_t> ent_mask;    // (n_entries * W), W = 2 for m == 8 else 1
  DBuf<uint16_t> ent_pres;    // (n_entries) members holding a (canonical) row with this j-cluster
  // dynamic pruning (r_inner > 0): force masks of the inner list -- members
  // with a pair within r_inner at the prune positions; entries are then
  // ordered by the inner pattern.  ent_mask stays the canonical r_list list.
  double r_inner = 0.0;
  DBuf<uint64_t> ent_fmask;   // (n_entries * W) or empty
  DBuf<int32_t> ent_fend;     // (n_groups) end of the group's entries with an inner member
  // rolling prune (NBX_FORCE_REPRUNE): inner masks redone in place at later
  // positions (xprune, the force-frame coordinates of that call); validity is
  // then measured from xprune (scalars[5]) and no entry tail is skipped
  DBuf<float4> xprune;
  int inner_ref = 0;          // scalar slot of the inner list's displacement: 0 build, 5 rolling prune
  bool tail_sorted = true;    // entries without an inner member sit past ent_fend
  // entries are stored in force order (member pattern) once ordered; the
  // t-th entry of a group in ascending-j order is ent_jorder[t] (empty: identity)
  DBuf<int32_t> ent_jorder;
  bool entries_ordered = false;
  // reference super layout (on demand)
  int64_t super_size = 0, super_groups = 0, super_entries = 0;
  DBuf<int32_t> super_offsets, super_j, super_pair;
  ForceWork work;
  bool ordered = false;  // finalize_force_layout done
  // domain lists: per-cluster halo bits and the number of interior work
  // items (groups touching no halo particle, first in group_order; -1: none)
  DBuf<uint8_t> halo_cl;
  int64_t n_interior = -1;
  int64_t halo_c0 = 0, halo_c1 = 0;  // domain lists: clusters [c0, c1) hold every halo particle
  int mask_words() const { return m == 8 ? 2 : 1; }
};

inline cudaStream_t to_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// count of kernels this library launched (nbx_launch_count)
void count_launch(int64_t k = 1);
// k_force event timing (nbx_timing_*)
bool timing_enabled();
void timing_record(cudaEvent_t a, cudaEvent_t b);

struct List;
cudaError_t finalize_force_layout(List* l, cudaStream_t s);
cudaError_t force_prepare(List* l, cudaStream_t s);  // force layout + j transpose (force.cu)
cudaError_t ensure_row_delta(List* l, cudaStream_t s);
cudaError_t ensure_rows(List* l, cudaStream_t s);
// rolling prune: inner masks of `l` at the force-frame coordinates xyzq
// (k_gather output; scalars[0] = their max displacement since the build)
cudaError_t reprune_inner(List* l, const float4* xyzq, const unsigned int* scalars, const double* bbox,
                          const double* cpos, const double box[3], cudaStream_t s);
// one force evaluation with a hook between the interior and the boundary
// work items of a domain list (force.cu; dd.cu runs the halo exchange there)
int force_split(const nbx_list_t* l, const nbx_grid_t* grid, const double* positions, const double* charges,
                const int64_t* lj_type, const nbx_params_t* p, const double box[3], int32_t flags, double* f_out,
                double* e_out, int64_t* bad, void* stream, const std::function<int()>& between,
                const std::function<int()>* after_halo = nullptr, bool split_launch = true);

// exclusive scan helpers (CUB), defined in scan.cu
cudaError_t exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, cudaStream_t s);
cudaError_t sort_pairs_i32(const int32_t* keys_in, int32_t* keys_out, const int32_t* vals_in,
                           int32_t* vals_out, int64_t n, int end_bit, cudaStream_t s);

}  // namespace nbx

struct nbx_grid : nbx::Grid {};
struct nbx_list : nbx::List {};
