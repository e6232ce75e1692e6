// Cluster-pair search, pruning, statistics and list layouts.
//
// Replaces pairlist.build_pair_list (pairlist.py:147-217), _build_masks
// (:106-112), prune_pair_list (:242-282), _build_super_layout (:115-144) and
// interaction_stats/_count_within (:303-346) of
// /root/reference/pkg/src/clustermd.  Every inclusion decision is the
// reference's FP64 expression in the reference's operation order
// (common.cuh), so the canonical list is bit-identical (set-identical rows
// and masks, same CSR order).
//
// The search runs per GROUP: G = 16/m consecutive clusters of one x/y column
// (a z-stack).  One warp enumerates the j-clusters of the columns within
// r_list of the group (ascending cluster index, so CSR order falls out), tests
// each against every member with the exact AABB gap, and emits in one pass
//   * the canonical rows (ci, cj >= ci) -- the parity object, and
//   * the grouped force layout: one ENTRY per (group, cj) carrying the
//     m x m masks of all members, a periodic shift and a slack for the
//     single-shift validity test (force.cu).
// Two passes (count, write) around a scan keep the output deterministic.
#include <cub/cub.cuh>
#include <algorithm>
#include <utility>

#include "internal.cuh"

namespace nbx {

struct Ranges {
  int64_t lo[2], hi[2];
  int n;
};

// Columns (along one axis) that can hold clusters within r of [lo, hi]:
// nominal column index range padded by one column each side (binning can
// place a particle a few ulp outside its nominal column), wrapped and split
// into at most two ascending segments.
__device__ __forceinline__ Ranges col_ranges(double lo, double hi, double r, double w, int64_t cells) {
  Ranges R;
  int64_t a = (int64_t)floor((lo - r) / w) - 1;
  int64_t b = (int64_t)floor((hi + r) / w) + 1;
  if (b - a + 1 >= cells) {
    R.n = 1; R.lo[0] = 0; R.hi[0] = cells - 1;
    return R;
  }
  int64_t am = ((a % cells) + cells) % cells;
  int64_t bm = ((b % cells) + cells) % cells;
  if (am <= bm) {
    R.n = 1; R.lo[0] = am; R.hi[0] = bm;
  } else {
    R.n = 2; R.lo[0] = 0; R.hi[0] = bm; R.lo[1] = am; R.hi[1] = cells - 1;
  }
  return R;
}

__host__ __device__ constexpr uint64_t column_mask_u64(int m) {
  uint64_t c = 0;
  for (int a = 0; a < m; ++a) c |= 1ull << (a * m);
  return c;
}

__device__ __forceinline__ uint64_t row_mask(int m, int nr_i, int nr_j, bool diag) {
  uint64_t jb = (nr_j >= 64) ? ~0ull : ((1ull << nr_j) - 1ull);
  uint64_t mk = 0;
  for (int a = 0; a < nr_i; ++a) {
    uint64_t row = jb;
    if (diag) row &= ~((2ull << a) - 1ull);  // b > a only (strict upper triangle)
    mk |= row << (a * m);
  }
  return mk;
}

// Periodic image of the j-cluster relative to the i-side box (bi) and the
// FP32 offset that maps j-local coordinates (relative to the j-cluster's
// bbox low corner) into the i-side frame (origin `oi`):
//   delta = lo_j + n L - oi  (FP64, rounded once),
// plus slack = min_d (L - ext_i - ext_j) for the single-image validity test.
__device__ __forceinline__ void image_delta(const double* bi, const double* oi, const double* bj,
                                            const Box& box, float4* delta, float* slack) {
  double dl[3];
  double sl = 1e300;
  for (int d = 0; d < 3; ++d) {
    const double ci = 0.5 * (bi[d] + bi[3 + d]);
    const double cj = 0.5 * (bj[d] + bj[3 + d]);
    double n = rint((ci - cj) * box.invL[d]);
    n = fmin(1.0, fmax(-1.0, n));
    dl[d] = (bj[d] + n * box.L[d]) - oi[d];
    const double s = box.L[d] - (bi[3 + d] - bi[d]) - (bj[3 + d] - bj[d]);
    sl = fmin(sl, s);
  }
  *delta = make_float4((float)dl[0], (float)dl[1], (float)dl[2], (float)sl);
  *slack = (float)sl;
}

constexpr int SEARCH_WARPS = 4;
constexpr int GMAX = 16;
#ifndef NBX_STASH
#define NBX_STASH 1024
#endif
constexpr int STASH = NBX_STASH;   // hits kept per group between the two passes (overflow: recompute;
                                   // 512 overflowed on relaxed-water MD boxes: pass 1 49 -> 170 us at 96k)

struct SearchOut {
  // fused prune (nbx_pairlist_build_pruned): positions the exact criterion uses
  const float4* xl = nullptr;     // cluster-local FP32 coordinates (bbox-corner frames)
  const double* ppos = nullptr;   // clustered FP64 positions (exact fallback)
  // pass 1
  int32_t* ent_count;   // (n_groups)
  int2* stash;          // (n_groups * STASH) {cj, member bits}
  // pass 2
  const int32_t* ent_offsets;
  int32_t* ent_j;
  float4* ent_delta;
  uint64_t* ent_mask;
  uint16_t* ent_pres;
};

// FP32 periodic gap of one dimension (same formula as gap_1d)
__device__ __forceinline__ float gap1f(float lo_i, float hi_i, float lo_j, float hi_j, float L) {
  const float a = lo_j - hi_i, b = lo_i - hi_j;
  const float g0 = fmaxf(0.f, fmaxf(a, b));
  const float gm = fmaxf(0.f, fmaxf(a - L, b + L));
  const float gp = fmaxf(0.f, fmaxf(a + L, b - L));
  return fminf(g0, fminf(gm, gp));
}

struct SearchCtx {
  int32_t first;
  int nmem;
  double r2;
  float r2_lo, r2_hi;          // FP32 decision band around r_list^2
  float Lf[3];
  const double* bbox;
  const float4* bbf;            // (n_clusters * 2) outward-rounded FP32 boxes
};

// exact FP64 AABB test of gridder.py:165-185 (rare: FP32 ambiguity band)
__device__ __noinline__ bool exact_gap_within(const double* bi, const double* __restrict__ bbox, int32_t cj,
                                              Box box, double r2) {
  double bj[6];
  for (int d = 0; d < 6; ++d) bj[d] = bbox[6 * (int64_t)cj + d];
  return gap_sq(bi, bj, box) <= r2;
}

// Member bits of candidate cj: FP32 gap^2 decides outside +-1e-4 r^2 (boxes
// rounded outward; the band covers FP32 rounding), the exact FP64 replay of
// gridder.py:165-185 decides inside it.
__device__ __forceinline__ uint32_t member_bits(const SearchCtx& C, const float4 (*s_bf)[2],
                                                const double (*s_bb)[6], int32_t cj, const Box& box) {
  const float4 lo = __ldg(C.bbf + 2 * (int64_t)cj), hi = __ldg(C.bbf + 2 * (int64_t)cj + 1);
  uint32_t bits = 0;
  for (int k = 0; k < C.nmem; ++k) {
    if (cj < C.first + k) break;
    const float gx = gap1f(s_bf[k][0].x, s_bf[k][1].x, lo.x, hi.x, C.Lf[0]);
    const float gy = gap1f(s_bf[k][0].y, s_bf[k][1].y, lo.y, hi.y, C.Lf[1]);
    const float gz = gap1f(s_bf[k][0].z, s_bf[k][1].z, lo.z, hi.z, C.Lf[2]);
    const float g2 = fmaf(gx, gx, fmaf(gy, gy, gz * gz));
    bool in;
    if (g2 < C.r2_lo) in = true;
    else if (g2 > C.r2_hi) in = false;
    else in = exact_gap_within(s_bb[k], C.bbox, cj, box, C.r2);
    bits |= (in ? 1u : 0u) << k;
  }
  return bits;
}

// Emit one batch of hits (ascending cj across lanes): canonical rows of every
// member (CSR position = member offset + running count) and the group entry.
// slot pairs (a, b) with both slots halo (domain decomposition: computed by
// the owner of the halo, never here)
__device__ __forceinline__ uint64_t halo_pair_mask(uint32_t hi, uint32_t hj, int m) {
  uint64_t x = 0;
  for (int a = 0; a < m; ++a)
    if ((hi >> a) & 1u) x |= (uint64_t)hj << (a * m);
  return x;
}

__device__ __forceinline__ void emit_batch(const SearchOut& out, const SearchCtx& C, const double (*s_bb)[6],
                                           const double* gb, int32_t cj, uint32_t bits, int lane, int32_t& ecnt,
                                           int32_t ent_base, int m, const int8_t* nreal, const Box& box,
                                           const uint8_t* __restrict__ halo) {
  const unsigned lt = (1u << lane) - 1u;
  const unsigned eb = __ballot_sync(0xffffffffu, bits != 0);
  if (!eb) return;
  if (bits) {
    const int ent_pos = ent_base + ecnt + __popc(eb & lt);
    const int W = (m == 8) ? 2 : 1;
    uint64_t emask[2] = {0ull, 0ull};
    double bj[6];
    for (int d = 0; d < 6; ++d) bj[d] = C.bbox[6 * (int64_t)cj + d];
    for (int k = 0; k < C.nmem; ++k) {
      if (!((bits >> k) & 1u)) continue;
      const int32_t ci = C.first + k;
      uint64_t mk = row_mask(m, nreal[ci], nreal[cj], ci == cj);
      if (halo) mk &= ~halo_pair_mask(halo[ci], halo[cj], m);
      if (W == 2) emask[k] = mk;
      else emask[0] |= mk << (k * m * m);
    }
    float4 e_delta;
    float e_slack;
    image_delta(gb, s_bb[0], bj, box, &e_delta, &e_slack);
    out.ent_j[ent_pos] = cj;
    out.ent_delta[ent_pos] = e_delta;
    out.ent_mask[(int64_t)ent_pos * W] = emask[0];
    if (W == 2) out.ent_mask[(int64_t)ent_pos * W + 1] = emask[1];
    out.ent_pres[ent_pos] = (uint16_t)bits;
  }
  ecnt += __popc(eb);
}

// Fused prune (pairlist.py:242-282): keep member k of a hit only if one of
// its admitted slot pairs with cj is within r_list (FP32 decision outside
// +-1e-4 r^2, exact FP64 replay inside), diagonal rows always.
__device__ __noinline__ bool exact_within(const double* __restrict__ pos, int64_t si, int64_t sj, Box box,
                                          double r2);
__device__ __forceinline__ uint32_t prune_bits(uint32_t bits, int32_t cj, const SearchCtx& C, const float4* s_xi,
                                               const double* gb, const double (*s_bb)[6], const SearchOut& out,
                                               const int8_t* __restrict__ nreal, const uint8_t* __restrict__ halo,
                                               int m, const Box& box) {
  if (!bits) return 0u;
  const float lo = (float)(C.r2 * (1.0 - 1e-4)), hi = (float)(C.r2 * (1.0 + 1e-4));
  double bj[6];
  for (int d = 0; d < 6; ++d) bj[d] = C.bbox[6 * (int64_t)cj + d];
  float4 dlt;
  float slack;
  image_delta(gb, s_bb[0], bj, box, &dlt, &slack);
  float4 xj[8];
  for (int b = 0; b < m; ++b) {
    xj[b] = __ldg(out.xl + (int64_t)cj * m + b);
    xj[b].x += dlt.x;
    xj[b].y += dlt.y;
    xj[b].z += dlt.z;
  }
  const int nr_j = nreal[cj];
  uint32_t keep = 0;
  for (int k = 0; k < C.nmem; ++k) {
    if (!((bits >> k) & 1u)) continue;
    const int32_t ci = C.first + k;
    if (ci == cj) {
      keep |= 1u << k;
      continue;
    }
    uint64_t mk = row_mask(m, nreal[ci], nr_j, false);
    if (halo) mk &= ~halo_pair_mask(halo[ci], halo[cj], m);
    bool found = false;
    for (int a = 0; a < m && !found; ++a) {
      const float4 xi = s_xi[k * m + a];
      for (int b = 0; b < m; ++b) {
        if (!((mk >> (a * m + b)) & 1ull)) continue;
        float dx = xi.x - xj[b].x, dy = xi.y - xj[b].y, dz = xi.z - xj[b].z;
        dx = fmaf(-C.Lf[0], rintf(dx / C.Lf[0]), dx);
        dy = fmaf(-C.Lf[1], rintf(dy / C.Lf[1]), dy);
        dz = fmaf(-C.Lf[2], rintf(dz / C.Lf[2]), dz);
        const float f = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        if (f < lo || (f <= hi && exact_within(out.ppos, (int64_t)ci * m + a, (int64_t)cj * m + b, box, C.r2))) {
          found = true;
          break;
        }
      }
    }
    if (found) keep |= 1u << k;
  }
  return keep;
}

// MODE 0: search + count (+ stash hits);  MODE 1: emit (from the stash, or
// by re-running the search for groups whose hits overflowed it).
// pass 0 (the scan) at 6 resident blocks; pass 1 (emit from the stash, a
// load/store chain) at 10 (1.5M: 582 -> ~535 us; pass 0 is slower at 10)
#ifndef NBX_SEARCH_MINB
#define NBX_SEARCH_MINB 6
#endif
template <int MODE, bool PRUNE>
__global__ void __launch_bounds__(SEARCH_WARPS * 32, MODE == 1 ? 10 : NBX_SEARCH_MINB)
k_search(const int32_t* __restrict__ group_first, const int32_t* __restrict__ group_nmem,
         int64_t n_groups, int m, int G, const double* __restrict__ bbox, const float4* __restrict__ bbf,
         const float2* __restrict__ zr, const int8_t* __restrict__ nreal, const int32_t* __restrict__ col_first,
         int64_t cells, Box box, double r_list, SearchOut out, const uint8_t* __restrict__ halo) {
  __shared__ double s_bb[SEARCH_WARPS][GMAX][6];
  __shared__ float4 s_bf[SEARCH_WARPS][GMAX][2];
  constexpr int ZU = 4;  // z-prefilter chunks per pass
  __shared__ int32_t s_q[SEARCH_WARPS][32 * ZU + 32];
  __shared__ float4 s_xi[SEARCH_WARPS][16];  // fused prune: the group's i-atoms in the group frame
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = blockIdx.x * (int64_t)SEARCH_WARPS + w;
  if (g >= n_groups) return;
  SearchCtx C;
  C.first = group_first[g];
  C.nmem = group_nmem[g];
  C.r2 = __dmul_rn(r_list, r_list);
  C.r2_lo = (float)(C.r2 * (1.0 - 1e-4));
  C.r2_hi = (float)(C.r2 * (1.0 + 1e-4));
  for (int d = 0; d < 3; ++d) C.Lf[d] = (float)box.L[d];
  C.bbox = bbox;
  C.bbf = bbf;
  if (lane < C.nmem) {
    for (int d = 0; d < 6; ++d) s_bb[w][lane][d] = bbox[6 * (int64_t)(C.first + lane) + d];
    s_bf[w][lane][0] = bbf[2 * (int64_t)(C.first + lane)];
    s_bf[w][lane][1] = bbf[2 * (int64_t)(C.first + lane) + 1];
  }
  __syncwarp();
  if (PRUNE) {
    for (int ia = lane; ia < 16; ia += 32) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ia < C.nmem * m) {
        const int k = ia / m;
        v = __ldg(out.xl + (int64_t)C.first * m + ia);
        v.x = (float)((s_bb[w][k][0] - s_bb[w][0][0]) + (double)v.x);
        v.y = (float)((s_bb[w][k][1] - s_bb[w][0][1]) + (double)v.y);
        v.z = (float)((s_bb[w][k][2] - s_bb[w][0][2]) + (double)v.z);
      }
      s_xi[w][ia] = v;
    }
    __syncwarp();
  }
  double gb[6];  // group AABB
  for (int d = 0; d < 3; ++d) {
    gb[d] = s_bb[w][0][d];
    gb[3 + d] = s_bb[w][0][3 + d];
    for (int k = 1; k < C.nmem; ++k) {
      gb[d] = fmin(gb[d], s_bb[w][k][d]);
      gb[3 + d] = fmax(gb[3 + d], s_bb[w][k][3 + d]);
    }
  }
  int32_t ecnt = 0, ent_base = 0;
  int2* stash = out.stash + g * (int64_t)STASH;
  if (MODE == 1) {
    ent_base = out.ent_offsets[g];
    const int32_t nst = out.ent_count[g];  // hits of this group (== its entry count)
    if (nst <= STASH) {
      for (int32_t base = 0; base < nst; base += 32) {
        int2 h = make_int2(0, 0);
        if (base + lane < nst) h = stash[base + lane];
        emit_batch(out, C, s_bb[w], gb, h.x, (uint32_t)h.y, lane, ecnt, ent_base, m, nreal, box, halo);
      }
      return;
    }
  }
  const float r2_pre = (float)(C.r2 * (1.0 + 1e-4)) + 1e-5f;
  const float gzlo = __double2float_rd(gb[2]), gzhi = __double2float_ru(gb[5]);
  const double wx = box.L[0] / (double)cells, wy = box.L[1] / (double)cells;
  Ranges RX = col_ranges(gb[0], gb[3], r_list, wx, cells);
  Ranges RY = col_ranges(gb[1], gb[4], r_list, wy, cells);
  const unsigned lt = (1u << lane) - 1u;
  int qn = 0;  // queued z-survivors (warp-uniform)

  auto process = [&](int n_items) {  // the first n_items of the queue
    const int32_t cj = lane < n_items ? s_q[w][lane] : 0;
    uint32_t bits = lane < n_items ? member_bits(C, s_bf[w], s_bb[w], cj, box) : 0u;
    if (PRUNE) bits = prune_bits(bits, cj, C, s_xi[w], gb, s_bb[w], out, nreal, halo, m, box);
    if (MODE == 0) {
      const unsigned eb = __ballot_sync(0xffffffffu, bits != 0);
      if (bits && ecnt + __popc(eb & lt) < STASH) stash[ecnt + __popc(eb & lt)] = make_int2(cj, (int)bits);
      ecnt += __popc(eb);
    } else {
      emit_batch(out, C, s_bb[w], gb, cj, bits, lane, ecnt, ent_base, m, nreal, box, halo);
    }
  };

  for (int sx = 0; sx < RX.n; ++sx) {
    for (int64_t ix = RX.lo[sx]; ix <= RX.hi[sx]; ++ix) {
      for (int sy = 0; sy < RY.n; ++sy) {
        const int32_t c0 = col_first[ix * cells + RY.lo[sy]];
        const int32_t c1 = col_first[ix * cells + RY.hi[sy] + 1];
        const int32_t start = c0 > C.first ? c0 : C.first;
        // ZU chunks of 32 candidates per pass: their z loads are in flight
        // together (the scan is a latency chain otherwise); survivors keep
        // ascending order in the queue, batches of 32 from its front
        for (int32_t base = start; base < c1; base += 32 * ZU) {
          bool keep[ZU];
#pragma unroll
          for (int u = 0; u < ZU; ++u) {
            const int32_t cj = base + 32 * u + lane;
            keep[u] = false;
            if (cj < c1) {  // conservative FP32 z prefilter against the whole group
              const float2 z = __ldg(zr + cj);
              const float gz = gap1f(gzlo, gzhi, z.x, z.y, C.Lf[2]);
              keep[u] = gz * gz <= r2_pre;
            }
          }
#pragma unroll
          for (int u = 0; u < ZU; ++u) {
            const unsigned kb = __ballot_sync(0xffffffffu, keep[u]);
            if (keep[u]) s_q[w][qn + __popc(kb & lt)] = base + 32 * u + lane;
            qn += __popc(kb);
          }
          __syncwarp();
          while (qn >= 32) {
            process(32);
            __syncwarp();
            for (int t0 = 0; t0 < qn - 32; t0 += 32) {  // shift the rest to the front
              const int t = t0 + lane;
              const int32_t v = t < qn - 32 ? s_q[w][32 + t] : 0;
              __syncwarp();
              if (t < qn - 32) s_q[w][t] = v;
              __syncwarp();
            }
            qn -= 32;
          }
        }
      }
    }
  }
  if (qn > 0) process(qn);
  if (MODE == 0 && lane == 0) out.ent_count[g] = ecnt;
}

__global__ void k_halo_bits(const uint8_t* __restrict__ halo, const int32_t* __restrict__ perm,
                            const uint8_t* __restrict__ fill, int64_t n_clusters, int m, uint8_t* __restrict__ hb) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n_clusters) return;
  uint32_t b = 0;
  for (int a = 0; a < m; ++a) {
    const int64_t s = c * m + a;
    if (!fill[s] && halo[perm[s]]) b |= 1u << a;
  }
  hb[c] = (uint8_t)b;
}

// ---------------------------------------------------------------- exact pair decisions
// d2 of slots (si, sj) of `pos` with the reference's min image
// (model.py:159-172) and einsum order (pairlist.py:236).
__device__ __forceinline__ double d2_exact(const double* __restrict__ pos, int64_t si, int64_t sj,
                                           const Box& box) {
  const double dx = min_image_np(__dsub_rn(pos[3 * si], pos[3 * sj]), box.L[0], box.invL[0]);
  const double dy = min_image_np(__dsub_rn(pos[3 * si + 1], pos[3 * sj + 1]), box.L[1], box.invL[1]);
  const double dz = min_image_np(__dsub_rn(pos[3 * si + 2], pos[3 * sj + 2]), box.L[2], box.invL[2]);
  return d2_einsum(dx, dy, dz);
}

// FP32 estimate of the same d2 (any image convention gives the same minimum
// for |d| < L/2; the margin covers FP32 rounding).
__device__ __forceinline__ float d2_fast(const double* __restrict__ pos, int64_t si, int64_t sj,
                                         const float Lf[3], const float iLf[3]) {
  float s = 0.f;
  for (int d = 0; d < 3; ++d) {
    float v = (float)__dsub_rn(pos[3 * si + d], pos[3 * sj + d]);
    v = v - Lf[d] * rintf(v * iLf[d]);
    s += v * v;
  }
  return s;
}

// Three-way decision d2 <= r2: the FP32 estimate decides unless it is inside
// +-1e-4 relative of r2, then the exact FP64 replay decides.
__device__ __forceinline__ bool within_exact(const double* __restrict__ pos, int64_t si, int64_t sj,
                                             const Box& box, double r2, float lo, float hi,
                                             const float Lf[3], const float iLf[3]) {
  const float f = d2_fast(pos, si, sj, Lf, iLf);
  if (f < lo) return true;
  if (f > hi) return false;
  return d2_exact(pos, si, sj, box) <= r2;
}

constexpr int ROWS_WARPS = 4;

// Positions for the row kernels: FP32, relative to the cluster's build-time
// box corner (the frame of the per-row `delta` offsets), ~1e-7 nm resolution.
__global__ void k_local_coords(const double* __restrict__ pos, const double* __restrict__ bbox, int64_t n_slots,
                               int m, float4* __restrict__ xl, const double* __restrict__ cpos = nullptr,
                               unsigned int* __restrict__ dmax = nullptr) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  float d = 0.f;
  if (s < n_slots) {
    const int64_t c = s / m;
    xl[s] = make_float4((float)(pos[3 * s] - bbox[6 * c]), (float)(pos[3 * s + 1] - bbox[6 * c + 1]),
                        (float)(pos[3 * s + 2] - bbox[6 * c + 2]), 0.f);
    if (dmax)  // largest coordinate displacement from the build positions (no wrapping: a wrap counts as L)
      for (int k = 0; k < 3; ++k) d = fmaxf(d, (float)fabs(pos[3 * s + k] - cpos[3 * s + k]));
  }
  if (dmax) {
    for (int o = 16; o; o >>= 1) d = fmaxf(d, __shfl_xor_sync(0xffffffffu, d, o));
    if ((threadIdx.x & 31) == 0) atomicMax(dmax, __float_as_uint(d * 1.0001f + 1e-6f));
  }
}

// Exact replay of the reference decision d^2 <= r^2 for slots (si, sj)
// (model.py:159-172 minimum image, pairlist.py:236 einsum order).  Rare.
__device__ __noinline__ bool exact_within(const double* __restrict__ pos, int64_t si, int64_t sj, Box box,
                                          double r2) {
  const double ex = min_image_np(__dsub_rn(pos[3 * si], pos[3 * sj]), box.L[0], box.invL[0]);
  const double ey = min_image_np(__dsub_rn(pos[3 * si + 1], pos[3 * sj + 1]), box.L[1], box.invL[1]);
  const double ez = min_image_np(__dsub_rn(pos[3 * si + 2], pos[3 * sj + 2]), box.L[2], box.invL[2]);
  return d2_einsum(ex, ey, ez) <= r2;
}

// Row kernels (prune: pairlist.py:242-282, count: pairlist.py:303-320): one
// warp per i-cluster, lane = (row slot r of 32/m, j-atom b).  i-atoms live in
// registers, j-atoms are coalesced float4 loads.  Each admitted pair's
// d^2 <= r^2 is decided by the FP32 estimate outside +-1e-4 relative of r^2
// and by the exact FP64 replay (min_image_np + einsum order) inside it.
template <int M, int MODE>  // MODE 0: prune, 1: count within
__global__ void __launch_bounds__(ROWS_WARPS * 32, 8)
k_rows(const int32_t* __restrict__ offsets, const int32_t* __restrict__ jv, const uint64_t* __restrict__ mask,
       const float4* __restrict__ rdelta, const int32_t* __restrict__ row_entry, int64_t n_clusters, int G, const double* __restrict__ pos,
       const float4* __restrict__ xl, Box box, double r2,
       const int32_t* __restrict__ cell_of_cluster, const int32_t* __restrict__ col_first,
       int32_t* __restrict__ keep, uint64_t* __restrict__ ent_mask, int32_t* __restrict__ ent_alive,
       unsigned long long* __restrict__ counts) {
  constexpr int R = 32 / M;
  const int64_t ci = blockIdx.x * (int64_t)ROWS_WARPS + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (ci >= n_clusters) return;
  const int r = lane / M, b = lane % M;
  const float lo = (float)(r2 * (1.0 - 1e-4)), hi = (float)(r2 * (1.0 + 1e-4));
  const float Lf[3] = {(float)box.L[0], (float)box.L[1], (float)box.L[2]};
  const float iLf[3] = {(float)box.invL[0], (float)box.invL[1], (float)box.invL[2]};
  float4 xi[M];
#pragma unroll
  for (int a = 0; a < M; ++a) xi[a] = __ldg(xl + ci * M + a);
  const int W = (M == 8) ? 2 : 1;
  const int k = MODE == 0 ? (int)((ci - col_first[cell_of_cluster[ci]]) % G) : 0;
  unsigned long long adm = 0, win = 0;
  const int32_t r0 = offsets[ci], r1 = offsets[ci + 1];
  // two-deep software pipeline: row words of batch k+2 and the j-atom of
  // batch k+1 are in flight while batch k is evaluated
  int32_t c1 = -1, c2 = -1;       // cj of batches k+1, k+2
  uint64_t m1 = 0, m2 = 0;
  float4 d1 = make_float4(0.f, 0.f, 0.f, 0.f), d2 = d1, x0 = d1;
  auto load_row = [&](int32_t row, int32_t& c, uint64_t& mm, float4& d) {
    if (row < r1) {
      c = __ldg(jv + row);
      mm = __ldg(mask + row);
      d = __ldg(rdelta + row);
    }
  };
  int32_t c0 = -1;
  uint64_t m0 = 0;
  float4 dd0 = d1;
  load_row(r0 + r, c0, m0, dd0);
  load_row(r0 + R + r, c1, m1, d1);
  if (r0 + r < r1) {
    x0 = __ldg(xl + (int64_t)c0 * M + b);
    x0.x += dd0.x;
    x0.y += dd0.y;
    x0.z += dd0.z;
  }
  for (int32_t base = r0; base < r1; base += R) {
    const int32_t row = base + r;
    const bool valid = row < r1;
    bool any = false;
    const int32_t cj = c0;
    const uint64_t mk = m0;
    const float4 xj = x0;
    load_row(row + 2 * R, c2, m2, d2);
    if (row + R < r1) {
      x0 = __ldg(xl + (int64_t)c1 * M + b);
      x0.x += d1.x;
      x0.y += d1.y;
      x0.z += d1.z;
    }
    c0 = c1;
    m0 = m1;
    c1 = c2;
    m1 = m2;
    d1 = d2;
    if (valid) {
      // FP32 decisions for this lane's M pairs; pairs inside the ambiguity
      // band are collected and decided exactly afterwards (rare, out of line)
      const uint32_t cm = (uint32_t)(mk >> b);
      uint32_t amb = 0;
#pragma unroll
      for (int a = 0; a < M; ++a) {
        float dx = xi[a].x - xj.x, dy = xi[a].y - xj.y, dz = xi[a].z - xj.z;
        dx = fmaf(-Lf[0], rintf(dx * iLf[0]), dx);
        dy = fmaf(-Lf[1], rintf(dy * iLf[1]), dy);
        dz = fmaf(-Lf[2], rintf(dz * iLf[2]), dz);
        const float f = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        const bool adm = (M == 8 && a >= 4) ? (((uint32_t)(mk >> (32 + b)) >> ((a - 4) * M)) & 1u)
                                            : ((cm >> (a * M)) & 1u);
        const bool in = adm && f < lo;
        amb |= (adm && f >= lo && f <= hi) ? (1u << a) : 0u;
        any |= in;
        if (MODE == 1) win += in;
      }
      while (amb) {
        const int a = __ffs(amb) - 1;
        amb &= amb - 1;
        const bool in = exact_within(pos, ci * M + a, (int64_t)cj * M + b, box, r2);
        any |= in;
        if (MODE == 1) win += in;
      }
      if (MODE == 1) adm += __popcll(mk & (column_mask_u64(M) << b));
    }
    if (MODE == 0) {
      // row decision: any pair of the row's m lanes within r_list (or diagonal)
      const unsigned bal = __ballot_sync(0xffffffffu, any);
      const unsigned seg = ((M == 32) ? 0xffffffffu : ((1u << M) - 1u)) << (r * M);
      const bool kp = (cj == ci) || (bal & seg) != 0u;
      if (valid && b == 0) {
        keep[row] = kp ? 1 : 0;
        const int32_t e = row_entry[row];
        if (kp) {
          ent_alive[e] = 1;
        } else if (mk) {
          if (W == 2) atomicAnd((unsigned long long*)&ent_mask[(int64_t)e * 2 + k], 0ull);
          else atomicAnd((unsigned long long*)&ent_mask[e], ~(unsigned long long)(mk << (k * M * M)));
        }
      }
    }
  }
  if (MODE == 1) {
    for (int o = 16; o; o >>= 1) {
      adm += __shfl_xor_sync(0xffffffffu, adm, o);
      win += __shfl_xor_sync(0xffffffffu, win, o);
    }
    if (lane == 0 && (adm || win)) {
      atomicAdd(&counts[0], adm);
      atomicAdd(&counts[1], win);
    }
  }
}

// Entry-wise prune (pairlist.py:242-282 decisions, bit-identical): one
// BLOCK per group, its warps striding over the group's entries; lane = (entry
// slot r of 32/m, j-atom b) as in the force kernel.  The group's 16 i-atoms
// sit in shared memory in the group frame, j-atoms are coalesced float4 loads
// shifted by the entry's frame offset.  Per entry the result is a G-bit
// "member kept" word (diagonal rows always kept); per group the number of
// surviving entries.
constexpr int PRUNE_WARPS = 4;

// One prune batch (R entries of a warp) against the group's i-atoms:
// branch-free over the member's pairs, members absent from the whole batch
// skipped warp-uniformly.  MI = per-pair minimum image (entries whose slack
// cannot guarantee the single shift at the current displacements).
template <int M, int G, int W, bool MI>
__device__ __forceinline__ float prune_r2(const float4& xi, const float4& xj, const float (&Lf)[3],
                                          const float (&iLf)[3]) {
  float dx = xi.x - xj.x, dy = xi.y - xj.y, dz = xi.z - xj.z;
  if (MI) {
    dx = fmaf(-Lf[0], rintf(dx * iLf[0]), dx);
    dy = fmaf(-Lf[1], rintf(dy * iLf[1]), dy);
    dz = fmaf(-Lf[2], rintf(dz * iLf[2]), dz);
  }
  return fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}

// Per member: the minimum FP32 r^2 over this lane's admitted pairs decides
// (min < lo: kept; min > hi: no pair of the lane within r_list); only a
// member whose minimum falls inside the +-1e-4 band lists its band pairs for
// the exact FP64 replay -- the same decisions as testing every pair, with a
// select + min per pair instead of two compares and two selects.
// hi_in (dynamic pruning, 0: off): a member whose minimum is <= hi_in also
// gets its bit in `ibits` -- the inner (force) list.  The test is one-sided
// and conservative (hi_in = r_inner^2 (1 + 1e-4), no FP64 replay): a member
// left out has no pair within r_inner.
template <int M, int G, int W, bool MI>
__device__ __forceinline__ void prune_batch(const float4* __restrict__ s_xi, const float4* __restrict__ s_xp,
                                            const float2* __restrict__ s_zp, const uint32_t (&wd)[2 * W],
                                            const float4& xj, float lo, float hi, float hi_in, const float (&Lf)[3],
                                            const float (&iLf)[3], uint32_t& inbits, uint32_t& ibits, uint32_t& amb) {
  constexpr int MM = M * M;
  const float inf = __int_as_float(0x7f800000);
  // packed FP32 over i-atom pairs (no per-pair minimum image): the same
  // IEEE operations per element as prune_r2, so the same values
  constexpr bool PACKED = !MI && (M % 2 == 0);
  const float2 nx = make_float2(-xj.x, -xj.x), ny = make_float2(-xj.y, -xj.y), nz = make_float2(-xj.z, -xj.z);
#pragma unroll
  for (int k = 0; k < G; ++k) {
    const int p0 = W == 2 ? k * 64 : k * MM;
    uint32_t cb = 0;  // this member's column bits (pairs (a, b) for this lane's b)
#pragma unroll
    for (int a = 0; a < M; ++a) cb |= (wd[(p0 + a * M) >> 5] >> ((p0 + a * M) & 31)) & 1u ? (1u << a) : 0u;
    if (!__any_sync(0xffffffffu, cb != 0u)) continue;
    float fmin = inf;
    if constexpr (PACKED) {
#pragma unroll
      for (int a = 0; a < M; a += 2) {
        const float4 xy = s_xp[(k * M + a) >> 1];
        const float2 zz = s_zp[(k * M + a) >> 1];
        const float2 dx = __fadd2_rn(make_float2(xy.x, xy.y), nx);
        const float2 dy = __fadd2_rn(make_float2(xy.z, xy.w), ny);
        const float2 dz = __fadd2_rn(zz, nz);
        const float2 f = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __fmul2_rn(dz, dz)));
        fmin = fminf(fmin, ((cb >> a) & 1u) ? f.x : inf);
        fmin = fminf(fmin, ((cb >> (a + 1)) & 1u) ? f.y : inf);
      }
    } else {
#pragma unroll
      for (int a = 0; a < M; ++a) {
        const float f = prune_r2<M, G, W, MI>(s_xi[k * M + a], xj, Lf, iLf);
        fmin = fminf(fmin, ((cb >> a) & 1u) ? f : inf);
      }
    }
    if (fmin <= hi_in) ibits |= 1u << k;
    if (fmin < lo) {
      inbits |= 1u << k;
    } else if (fmin <= hi) {  // rare: list the band pairs of this member
#pragma unroll
      for (int a = 0; a < M; ++a) {
        const float f = prune_r2<M, G, W, MI>(s_xi[k * M + a], xj, Lf, iLf);
        amb |= (((cb >> a) & 1u) && f >= lo && f <= hi) ? (1u << (k * M + a)) : 0u;
      }
    }
  }
}

// 8 resident blocks (<= 64 registers): the kernel is a chain of dependent
// loads per group, so occupancy hides it (96k: 105 -> 77 us, 1.5M: 1.69 -> 1.12 ms)
#ifndef NBX_PRUNE_MINB
#define NBX_PRUNE_MINB 8
#endif
template <int M, int G>
__global__ void __launch_bounds__(PRUNE_WARPS * 32, NBX_PRUNE_MINB)
k_prune_entries(const int32_t* __restrict__ grp_first, const int32_t* __restrict__ grp_nmem, int64_t n_groups,
                const int32_t* __restrict__ ent_off, const int32_t* __restrict__ ent_j,
                const float4* __restrict__ ent_delta, const uint64_t* __restrict__ ent_mask,
                const float4* __restrict__ xl, const double* __restrict__ bbox, const double* __restrict__ pos,
                Box box, double r2, double r2_inner, const unsigned int* __restrict__ dmax_bits, float slack_base,
                uint32_t* __restrict__ ent_keep, int32_t* __restrict__ grp_alive) {
  constexpr int R = 32 / M;
  constexpr int IA = G * M;
  constexpr int W = (G * M * M > 64) ? 2 : 1;
  constexpr int U = 2;  // batches in flight per warp
  __shared__ float4 s_xi[IA];
  __shared__ float4 s_xp[(IA + 1) / 2];  // i-atom pairs {x_a, x_b, y_a, y_b} (packed FP32 path)
  __shared__ float2 s_zp[(IA + 1) / 2];  // {z_a, z_b}
  __shared__ int32_t s_cnt[PRUNE_WARPS];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane / M, b = lane % M;
  const float lo = (float)(r2 * (1.0 - 1e-4)), hi = (float)(r2 * (1.0 + 1e-4));
  const float hi_in = r2_inner > 0.0 ? (float)(r2_inner * (1.0 + 1e-4)) : -1.f;
  const float Lf[3] = {(float)box.L[0], (float)box.L[1], (float)box.L[2]};
  const float iLf[3] = {(float)box.invL[0], (float)box.invL[1], (float)box.invL[2]};
  const float slack_thr = slack_base + 4.f * __uint_as_float(*dmax_bits);
  for (int64_t g = blockIdx.x; g < n_groups; g += gridDim.x) {
    const int32_t first = grp_first[g];
    const int nmem = grp_nmem[g];
    __syncthreads();
    for (int ia = threadIdx.x; ia < IA; ia += blockDim.x) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ia < nmem * M) {
        const int64_t c = first + ia / M;
        v = xl[(int64_t)first * M + ia];
        v.x = (float)((bbox[6 * c] - bbox[6 * (int64_t)first]) + (double)v.x);
        v.y = (float)((bbox[6 * c + 1] - bbox[6 * (int64_t)first + 1]) + (double)v.y);
        v.z = (float)((bbox[6 * c + 2] - bbox[6 * (int64_t)first + 2]) + (double)v.z);
      }
      s_xi[ia] = v;
      float* xp = reinterpret_cast<float*>(&s_xp[ia >> 1]);
      xp[ia & 1] = v.x;
      xp[2 + (ia & 1)] = v.y;
      reinterpret_cast<float*>(&s_zp[ia >> 1])[ia & 1] = v.z;
    }
    __syncthreads();
    const int32_t e_beg = ent_off[g], e_end = ent_off[g + 1];
    int32_t alive = 0;
    for (int32_t e0 = e_beg + w * R; e0 < e_end; e0 += PRUNE_WARPS * R * U) {
      // loads of U batches first (memory-level parallelism), then the math
      int32_t cj[U];
      float4 xj[U];
      uint32_t wd[U][2 * W];
      bool valid[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int32_t e = e0 + u * PRUNE_WARPS * R + r;
        valid[u] = e < e_end;
        cj[u] = valid[u] ? __ldg(ent_j + e) : -1;
        float4 d = make_float4(0.f, 0.f, 0.f, 3.0e38f);
        if (valid[u]) d = __ldg(ent_delta + e);
        xj[u] = d;
#pragma unroll
        for (int q = 0; q < W; ++q) {
          const uint64_t mw = valid[u] ? (__ldg(ent_mask + (int64_t)e * W + q) >> b) : 0ull;
          wd[u][2 * q] = (uint32_t)mw;
          wd[u][2 * q + 1] = (uint32_t)(mw >> 32);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (valid[u]) {
          const float4 x = __ldg(xl + (int64_t)cj[u] * M + b);
          xj[u] = make_float4(x.x + xj[u].x, x.y + xj[u].y, x.z + xj[u].z, xj[u].w);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!__any_sync(0xffffffffu, valid[u])) break;
        uint32_t inbits = 0, ibits = 0, amb = 0;
        if (!__any_sync(0xffffffffu, valid[u] && xj[u].w < slack_thr))
          prune_batch<M, G, W, false>(s_xi, s_xp, s_zp, wd[u], xj[u], lo, hi, hi_in, Lf, iLf, inbits, ibits, amb);
        else
          prune_batch<M, G, W, true>(s_xi, s_xp, s_zp, wd[u], xj[u], lo, hi, hi_in, Lf, iLf, inbits, ibits, amb);
        while (amb) {  // rare: exact FP64 replay of the reference decision
          const int ia = __ffs(amb) - 1;
          amb &= amb - 1;
          const int k = ia / M;
          if ((inbits >> k) & 1u) continue;
          if (exact_within(pos, (int64_t)first * M + ia, (int64_t)cj[u] * M + b, box, r2)) inbits |= 1u << k;
        }
        // OR over the entry's M lanes (canonical bits 0..15, inner bits 16..31)
        uint32_t both = inbits | (ibits << 16);
#pragma unroll
        for (int o = 1; o < M; o <<= 1) both |= __shfl_xor_sync(0xffffffffu, both, o);
        inbits = both & 0xffffu;
        if (valid[u] && b == 0) {
          if (cj[u] >= first && cj[u] < first + nmem) inbits |= 1u << (cj[u] - first);  // diagonal rows survive
          ent_keep[e0 + u * PRUNE_WARPS * R + r] = inbits | (both & ~0xffffu);
        }
        alive += __popc(__ballot_sync(0xffffffffu, valid[u] && b == 0 && inbits != 0u));
      }
    }
    if (lane == 0) s_cnt[w] = alive;
    __syncthreads();
    if (threadIdx.x == 0) {
      int32_t t = 0;
      for (int q = 0; q < PRUNE_WARPS; ++q) t += s_cnt[q];
      grp_alive[g] = t;
    }
  }
}

// ---------------------------------------------------------------- entry order
// Within each group, entries are stored by member-presence pattern (stable,
// then by j-cluster) so that the 32/m entries a force-kernel warp handles per
// iteration share their members: the kernel skips a member only when no entry
// of the iteration has it, so homogeneous iterations waste no lanes.
constexpr int SORT_SMEM = 1024;
constexpr int ORDER_WARPS = 4;

__device__ __forceinline__ uint32_t mask_pattern(const uint64_t* em, int m, int G) {
  uint32_t pat = 0;
  const int mm = m * m;
  for (int k = 0; k < G; ++k) {
    uint64_t bits;
    if (m == 8) bits = em[k];
    else bits = (em[0] >> (k * mm)) & (mm == 64 ? ~0ull : ((1ull << mm) - 1ull));
    pat |= (bits != 0ull ? 1u : 0u) << k;
  }
  return pat;
}

__device__ __forceinline__ uint64_t keep_mask(uint32_t kb, int m, int G) {
  const int mm = m * m;
  const uint64_t one = (mm == 64) ? ~0ull : ((1ull << mm) - 1ull);
  uint64_t km = 0;
  for (int k = 0; k < G; ++k)
    if ((kb >> k) & 1u) km |= one << (k * mm);
  return km;
}

// Stable order of one group's live entries by key (warp-cooperative, keys in
// shared memory, key 0xffffffff = dead): returns through `opos` each live
// entry's position among the live entries.  Iterations = distinct keys.
__device__ __forceinline__ void warp_order(const uint32_t* s_key, int32_t* s_pos, int n, int lane) {
  const unsigned lt = (1u << lane) - 1u;
  int32_t placed = 0;
  int64_t prev = -1;
  for (;;) {
    uint32_t mn = 0xffffffffu;
    for (int t = lane; t < n; t += 32) {
      const uint32_t k = s_key[t];
      if ((int64_t)k > prev && k < mn) mn = k;
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    if (mn == 0xffffffffu) break;
    for (int base = 0; base < n; base += 32) {
      const int t = base + lane;
      const bool hit = t < n && s_key[t] == mn;
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (hit) s_pos[t] = placed + __popc(bal & lt);
      placed += __popc(bal);
    }
    prev = mn;
  }
}

// Same result as warp_order for small key sets (G <= 4: member patterns
// < 2^G, plus the inner-list tail key 1 << 16): a stable counting sort --
// per 32-entry chunk one __match_any_sync groups equal keys, bin leaders
// count, an exclusive scan over the <= 17 bins, then the same pass places.
// Two passes over the keys instead of two per distinct key.
// Force order of member patterns within a group (G <= 4).  k_force_h runs a
// member's sweep for an iteration of R = 32/m consecutive entries when ANY of
// them holds the member, so an iteration that straddles two patterns pays for
// their union.  Patterns are therefore ordered so that neighbours mostly nest:
// for G = 4 the order below (a local search over the 15! orders on the 96k SPC
// inner list, tools/pattern_order.py) evaluates 0.895 admitted / evaluated
// slot pairs against 0.858 for ascending pattern values; G = 2: 01, 11, 10.
__device__ __forceinline__ uint32_t pattern_rank(uint32_t pat, int G) {
  constexpr uint8_t r4[16] = {15, 14, 12, 13, 7, 0, 2, 1, 9, 5, 10, 11, 8, 4, 6, 3};
  constexpr uint8_t r2[4] = {3, 0, 2, 1};
#ifdef NBX_NO_PATTERN_RANK  // A/B: ascending pattern values
  return pat;
#endif
  if (G == 4) return r4[pat & 15u];
  if (G == 2) return r2[pat & 3u];
  return pat;
}

__device__ __forceinline__ void warp_order_bins(const uint32_t* s_key, int32_t* s_pos, int n, int lane, int G,
                                                int32_t* s_cnt) {
  const int K = (1 << G) + 1;
  const unsigned lt = (1u << lane) - 1u;
  if (lane < K) s_cnt[lane] = 0;
  __syncwarp();
  for (int pass = 0; pass < 2; ++pass) {
    for (int base = 0; base < n; base += 32) {
      const int t = base + lane;
      const uint32_t k = t < n ? s_key[t] : 0xffffffffu;
      const int bin = k == 0xffffffffu ? -1 : (k >= (1u << G) ? K - 1 : (int)k);
      const unsigned mm = __match_any_sync(0xffffffffu, bin);
      if (pass == 1 && bin >= 0) s_pos[t] = s_cnt[bin] + __popc(mm & lt);
      __syncwarp();
      if (bin >= 0 && (mm & lt) == 0u) s_cnt[bin] += __popc(mm);  // one leader per bin
      __syncwarp();
    }
    if (pass == 0) {
      if (lane == 0) {
        int32_t run = 0;
        for (int b = 0; b < K; ++b) {
          const int32_t c = s_cnt[b];
          s_cnt[b] = run;
          run += c;
        }
      }
      __syncwarp();
    }
  }
}

// Pruned list from the keep words: surviving entries of each group written
// in force order (member pattern of the pruned masks), their masks reduced to
// the kept members, and the ascending-j index ent_jorder.  One warp per group.
#ifndef NBX_ORDER_MINB
#define NBX_ORDER_MINB 1
#endif
__global__ void __launch_bounds__(ORDER_WARPS * 32, NBX_ORDER_MINB)
k_compact_order(const int32_t* __restrict__ off_in, int64_t n_groups, const int32_t* __restrict__ jorder_in,
                const uint32_t* __restrict__ ent_keep, const int32_t* __restrict__ ej, const float4* __restrict__ ed, const uint64_t* __restrict__ em,
                int m, int G, const int32_t* __restrict__ off_out, int32_t* __restrict__ ej2,
                float4* __restrict__ ed2, uint64_t* __restrict__ em2, uint16_t* __restrict__ ep2,
                int32_t* __restrict__ jorder2, uint64_t* __restrict__ fm2, int32_t* __restrict__ fend) {
  __shared__ uint32_t s_key[ORDER_WARPS][SORT_SMEM];
  __shared__ int32_t s_pos[ORDER_WARPS][SORT_SMEM];
  __shared__ int32_t s_cnt[ORDER_WARPS][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = blockIdx.x * (int64_t)ORDER_WARPS + w;
  if (g >= n_groups) return;
  const int W = (m == 8) ? 2 : 1;
  const unsigned lt = (1u << lane) - 1u;
  const int32_t e0 = off_in[g], n = off_in[g + 1] - e0, o0 = off_out[g];
  const bool sorted = n <= SORT_SMEM;  // very long lists (needle clusters): keep j order
  if (sorted) {
    for (int t = lane; t < n; t += 32) {
      const int64_t e = jorder_in ? jorder_in[e0 + t] : e0 + t;  // t-th entry in ascending j
      const uint32_t kw = ent_keep[e], kb0 = kw & 0xffffu;
      // fm2 (dynamic pruning): order by the inner (force) pattern, entries
      // with no inner member last
      const uint32_t kb = fm2 ? (kw >> 16) & kb0 : kb0;
      uint32_t key = 0xffffffffu;
      if (kb0) {
        uint64_t mk[2];
        for (int q = 0; q < W; ++q) mk[q] = em[e * W + q];
        if (W == 2) {
          for (int q = 0; q < 2; ++q)
            if (!((kb >> q) & 1u)) mk[q] = 0ull;
        } else {
          mk[0] &= keep_mask(kb, m, G);
        }
        key = mask_pattern(mk, m, G);
        if (fm2 && key == 0u) key = 1u << 16;
        else if (G <= 4) key = pattern_rank(key, G);
      }
      s_key[w][t] = key;
    }
    __syncwarp();
    if (G <= 4) warp_order_bins(s_key[w], s_pos[w], n, lane, G, s_cnt[w]);
    else warp_order(s_key[w], s_pos[w], n, lane);
    __syncwarp();
  }
  int32_t jr = 0;  // live entries before this chunk (ascending j)
  int32_t ni = 0;  // live entries with an inner member (sorted before the others)
  for (int base = 0; base < n; base += 32) {
    const int t = base + lane;
    const int64_t e = t < n ? (jorder_in ? jorder_in[e0 + t] : e0 + t) : 0;
    const uint32_t kw = t < n ? ent_keep[e] : 0u, kb = kw & 0xffffu, ib = (kw >> 16) & kb;
    const unsigned bal = __ballot_sync(0xffffffffu, kb != 0u);
    if (kb) {
      const int32_t rank = jr + __popc(bal & lt);
      const int32_t p = o0 + (sorted ? s_pos[w][t] : rank);
      ej2[p] = ej[e];
      ed2[p] = ed[e];
      if (W == 2) {
        for (int q = 0; q < 2; ++q) {
          em2[(int64_t)p * 2 + q] = ((kb >> q) & 1u) ? em[e * 2 + q] : 0ull;
          if (fm2) fm2[(int64_t)p * 2 + q] = ((ib >> q) & 1u) ? em[e * 2 + q] : 0ull;
        }
      } else {
        em2[p] = em[e] & keep_mask(kb, m, G);
        if (fm2) fm2[p] = em[e] & keep_mask(ib, m, G);
      }
      ep2[p] = (uint16_t)kb;
      jorder2[o0 + rank] = p;
    }
    jr += __popc(bal);
    ni += __popc(__ballot_sync(0xffffffffu, ib != 0u));
  }
  // inner-list end of the group: entries past it have no inner member (only
  // when the group was sorted; very long groups keep j order, no tail)
  if (fend && lane == 0) fend[g] = o0 + (sorted ? ni : jr);
}

template <int MODE>
static void launch_rows(int m, int64_t nc, cudaStream_t s, const int32_t* offsets, const int32_t* jv,
                        const uint64_t* mask, const float4* rdelta, const int32_t* row_entry, int G, const double* pos, const float4* xl,
                        Box box, double r2, const int32_t* coc, const int32_t* col_first,
                        int32_t* keep, uint64_t* ent_mask, int32_t* ent_alive, unsigned long long* counts) {
  const int blocks = (int)((nc + ROWS_WARPS - 1) / ROWS_WARPS);
  count_launch();
#define NBX_ROWS(MM)                                                                                         \
  k_rows<MM, MODE><<<blocks, ROWS_WARPS * 32, 0, s>>>(offsets, jv, mask, rdelta, row_entry, nc, G, pos, xl, box, r2, \
                                                      coc, col_first, keep, ent_mask, ent_alive, counts)
  switch (m) {
    case 1: NBX_ROWS(1); break;
    case 2: NBX_ROWS(2); break;
    case 4: NBX_ROWS(4); break;
    default: NBX_ROWS(8); break;
  }
#undef NBX_ROWS
}

// ---------------------------------------------------------------- compaction helpers
__global__ void k_new_offsets(const int32_t* __restrict__ old_off, int64_t n,
                              const int32_t* __restrict__ scan, int32_t* __restrict__ new_off) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i <= n) new_off[i] = scan[old_off[i]];
}

__global__ void k_compact_rows(int64_t n_rows, const int32_t* __restrict__ keep,
                               const int32_t* __restrict__ scan, const int32_t* __restrict__ ent_scan,
                               const int32_t* j, const uint64_t* mask, const int32_t* row_entry, int32_t* j2,
                               uint64_t* mask2, int32_t* row_entry2) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_rows || !keep[r]) return;
  const int32_t p = scan[r];
  j2[p] = j[r];
  mask2[p] = mask[r];
  row_entry2[p] = ent_scan[row_entry[r]];
}

__global__ void k_compact_entries(int64_t n_ent, int W, const int32_t* __restrict__ alive,
                                  const int32_t* __restrict__ scan, const int32_t* ej,
                                  const float4* edelta, const uint64_t* emask,
                                  int32_t* ej2, float4* edelta2, uint64_t* emask2) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n_ent || !alive[e]) return;
  const int32_t p = scan[e];
  ej2[p] = ej[e];
  edelta2[p] = edelta[e];
  for (int w = 0; w < W; ++w) emask2[(int64_t)p * W + w] = emask[e * W + w];
}

// CSR "first" array from keys sorted ascending: first[c] = lower_bound(c).
__global__ void k_first_from_sorted(const int32_t* __restrict__ keys, int64_t n, int64_t n_keys,
                                    int32_t* __restrict__ first) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  const int32_t prev = i == 0 ? -1 : keys[i - 1];
  const int32_t cur = i == n ? (int32_t)n_keys : keys[i];
  for (int32_t c = prev + 1; c <= cur; ++c) first[c] = (int32_t)i;
}

// super layout (pairlist.py:115-144): rows sorted by (ci / size, cj)
__global__ void k_row_ci(const int32_t* __restrict__ offsets, int64_t n_clusters, int32_t* __restrict__ ci_of_row) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n_clusters) return;
  for (int32_t r = offsets[c]; r < offsets[c + 1]; ++r) ci_of_row[r] = (int32_t)c;
}

__global__ void k_super_keys(const int32_t* __restrict__ ci_of_row, const int32_t* __restrict__ j,
                             int64_t n_rows, int size, int64_t n_clusters, uint64_t* __restrict__ keys,
                             int32_t* __restrict__ vals) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  keys[r] = (uint64_t)(ci_of_row[r] / size) * (uint64_t)n_clusters + (uint64_t)j[r];
  vals[r] = (int32_t)r;
}

__global__ void k_super_heads(const uint64_t* __restrict__ keys, int64_t n, int32_t* __restrict__ head) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
  if (i == n) head[i] = 0;
}

__global__ void k_super_fill(const uint64_t* __restrict__ keys, const int32_t* __restrict__ rows,
                             const int32_t* __restrict__ head_scan, const int32_t* __restrict__ ci_of_row,
                             int64_t n, int size, int64_t n_clusters, int32_t* __restrict__ sj,
                             int32_t* __restrict__ spair, int32_t* __restrict__ group_count) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool head = (i == 0 || keys[i] != keys[i - 1]);
  const int32_t e = head_scan[i + 1] - 1;  // inclusive head count - 1
  const int32_t r = rows[i];
  const int32_t ci = ci_of_row[r];
  if (head) {
    sj[e] = (int32_t)(keys[i] % (uint64_t)n_clusters);
    atomicAdd(&group_count[ci / size], 1);
  }
  spair[(int64_t)e * size + (ci % size)] = r;
}


// force order of a built (unpruned) list's entries: newpos[e] = storage
// position of the e-th entry (ascending j) of its group
__global__ void __launch_bounds__(ORDER_WARPS * 32)
k_entry_order(const int32_t* __restrict__ ent_off, int64_t n_groups, const uint64_t* __restrict__ emask,
              int m, int G, int32_t* __restrict__ newpos) {
  __shared__ uint32_t s_key[ORDER_WARPS][SORT_SMEM];
  __shared__ int32_t s_pos[ORDER_WARPS][SORT_SMEM];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = blockIdx.x * (int64_t)ORDER_WARPS + w;
  if (g >= n_groups) return;
  const int W = (m == 8) ? 2 : 1;
  const int32_t e0 = ent_off[g], n = ent_off[g + 1] - e0;
  if (n > SORT_SMEM) {  // very long lists (needle clusters): keep j order
    for (int t = lane; t < n; t += 32) newpos[e0 + t] = e0 + t;
    return;
  }
  for (int t = lane; t < n; t += 32) {
    const uint32_t pat = mask_pattern(emask + (int64_t)(e0 + t) * W, m, G);
    s_key[w][t] = G <= 4 ? pattern_rank(pat, G) : pat;
  }
  __syncwarp();
  warp_order(s_key[w], s_pos[w], n, lane);
  __syncwarp();
  for (int t = lane; t < n; t += 32) newpos[e0 + t] = e0 + s_pos[w][t];
}

__global__ void k_permute_entries(int64_t n_ent, int W, const int32_t* __restrict__ newpos, const int32_t* ej,
                                  const float4* edelta, const uint64_t* emask, const uint16_t* epres, int32_t* ej2,
                                  float4* edelta2, uint64_t* emask2, uint16_t* epres2) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n_ent) return;
  const int32_t p = newpos[e];
  ej2[p] = ej[e];
  edelta2[p] = edelta[e];
  epres2[p] = epres[e];
  for (int w = 0; w < W; ++w) emask2[(int64_t)p * W + w] = emask[e * W + w];
}

static int nb(int64_t n, int t) { return (int)((n + t - 1) / t); }

__global__ void k_fill_i32(int32_t* __restrict__ v, int64_t n, int32_t x) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = x;
}

__global__ void k_group_keys(const int32_t* __restrict__ ent_off, const int32_t* __restrict__ nmem,
                             const int32_t* __restrict__ fend, int64_t n_groups, int32_t* __restrict__ keys,
                             int32_t* __restrict__ vals) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= n_groups) return;
  // estimated force-kernel cost: per entry ~1/8 of an iteration's fixed work
  // plus up to nmem member sweeps (measured ratio ~1 : 5 per present member);
  // with an inner list only its entries are evaluated (the tail is stores)
  const int32_t e_end = fend ? fend[g] : ent_off[g + 1];
  const int64_t cost = (int64_t)(e_end - ent_off[g]) * (2 + 5 * (nmem ? nmem[g] : 1)) +
                       (fend ? (ent_off[g + 1] - e_end) / 4 : 0);
  // ascending key = descending cost, 16 bits (cost / 4, saturated): two radix
  // passes instead of four for a 30-bit key
  keys[g] = 0xffff - (int32_t)min(cost >> 2, (int64_t)0xffff);
  vals[g] = (int32_t)g;
}

// force-kernel work order: groups by descending estimated cost (LPT)
// domain lists (halo bits): a group is BOUNDARY when one of its clusters or
// one of its entries' j-clusters holds a halo particle; bit 16 of its work
// key, so interior groups -- which read no halo coordinates -- come first
// and the halo exchange can overlap them (dd.cu nbx_dd_force).  One warp per
// group; counts the interior groups.
__global__ void k_group_boundary(const int32_t* __restrict__ grp_first, const int32_t* __restrict__ grp_nmem,
                                 int64_t n_groups, const int32_t* __restrict__ ent_off,
                                 const int32_t* __restrict__ ent_j, const uint8_t* __restrict__ halo_cl,
                                 int32_t* __restrict__ keys, unsigned int* __restrict__ n_interior) {
  const int64_t g = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= n_groups) return;
  const int lane = threadIdx.x & 31;
  bool b = lane < grp_nmem[g] && halo_cl[grp_first[g] + lane] != 0;
  for (int32_t e = ent_off[g] + lane; e < ent_off[g + 1]; e += 32) b = b || halo_cl[ent_j[e]] != 0;
  const bool boundary = __any_sync(0xffffffffu, b);
  if (lane == 0) {
    if (boundary) keys[g] |= 1 << 16;
    else atomicAdd(n_interior, 1u);
  }
}

// range of the clusters holding a halo particle (k_reduce does them first in
// the DD force step so that the halo forces can leave early)
__global__ void k_halo_range(const uint8_t* __restrict__ halo_cl, int64_t nc, unsigned int* __restrict__ range) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c < nc && halo_cl[c]) {
    atomicMin(range, (unsigned int)c);
    atomicMax(range + 1, (unsigned int)c);
  }
}

static cudaError_t order_groups(List* l, cudaStream_t s) {
  DBuf<int32_t> keys, keys2, vals;
  DBuf<unsigned int> nint;
  cudaError_t e;
  l->n_interior = -1;
  if ((e = l->group_order.alloc(l->n_groups, s))) return e;
  if (l->n_groups == 0) return cudaSuccess;
  if ((e = keys.alloc(l->n_groups, s)) || (e = keys2.alloc(l->n_groups, s)) || (e = vals.alloc(l->n_groups, s)))
    return e;
  count_launch();
  k_group_keys<<<nb(l->n_groups, 256), 256, 0, s>>>(l->ent_offsets.p, l->group_nmem.p, l->ent_fend.p, l->n_groups,
                                                     keys.p, vals.p);
  const bool split = l->halo_cl.p != nullptr;
  if (split) {
    const unsigned int init[3] = {0u, 0xffffffffu, 0u};  // interior count, halo cluster min, max
    if ((e = nint.alloc(3, s)) || (e = cudaMemcpyAsync(nint.p, init, 12, cudaMemcpyHostToDevice, s))) return e;
    if (l->n_clusters > 0)
      count_launch(), k_halo_range<<<nb(l->n_clusters, 256), 256, 0, s>>>(l->halo_cl.p, l->n_clusters, nint.p + 1);
    count_launch();
    k_group_boundary<<<nb(l->n_groups, 8), 256, 0, s>>>(l->group_first.p, l->group_nmem.p, l->n_groups,
                                                         l->ent_offsets.p, l->ent_j.p, l->halo_cl.p, keys.p, nint.p);
  }
  e = sort_pairs_i32(keys.p, keys2.p, vals.p, l->group_order.p, l->n_groups, split ? 17 : 16, s);
  if (!e && split) {
    unsigned int h[3] = {0u, 0u, 0u};
    if (!(e = cudaMemcpyAsync(h, nint.p, 12, cudaMemcpyDeviceToHost, s)) && !(e = cudaStreamSynchronize(s))) {
      l->n_interior = h[0];
      l->halo_c0 = h[1] <= h[2] ? (int64_t)h[1] : 0;
      l->halo_c1 = h[1] <= h[2] ? (int64_t)h[2] + 1 : 0;
    }
  }
  keys.release(s); keys2.release(s); vals.release(s); nint.release(s);
  return e;
}

// reorder a built list's entries into force order (pruned lists are written
// in force order by the prune itself)
static cudaError_t order_entries(List* l, cudaStream_t s) {
  const int64_t ne = l->n_entries;
  if (ne == 0 || l->n_groups == 0) {
    l->entries_ordered = true;
    return cudaSuccess;
  }
  const int W = l->mask_words();
  DBuf<int32_t> newpos, ej;
  DBuf<float4> ed;
  DBuf<uint64_t> em;
  DBuf<uint16_t> ep;
  cudaError_t e;
  if ((e = newpos.alloc(ne, s)) || (e = ej.alloc(ne, s)) || (e = ed.alloc(ne, s)) || (e = em.alloc(ne * W, s)) ||
      (e = ep.alloc(ne, s)))
    return e;
  count_launch(2);
  k_entry_order<<<nb(l->n_groups, ORDER_WARPS), ORDER_WARPS * 32, 0, s>>>(l->ent_offsets.p, l->n_groups,
                                                                           l->ent_mask.p, l->m, l->G, newpos.p);
  k_permute_entries<<<nb(ne, 256), 256, 0, s>>>(ne, W, newpos.p, l->ent_j.p, l->ent_delta.p, l->ent_mask.p,
                                                 l->ent_pres.p, ej.p, ed.p, em.p, ep.p);
  std::swap(l->ent_j, ej);
  std::swap(l->ent_delta, ed);
  std::swap(l->ent_mask, em);
  std::swap(l->ent_pres, ep);
  std::swap(l->ent_jorder, newpos);  // j-order position -> storage position
  ej.release(s); ed.release(s); em.release(s); ep.release(s); newpos.release(s);
  l->entries_ordered = true;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- canonical rows
// The canonical CSR (pairlist.py:185-201 order: rows of ci ascending in cj)
// from the entries: member k of a group has a row with cj iff bit k of the
// entry's ent_pres is set; walking the group's entries in ascending j gives
// every member's rows in order.  One warp per group.
__global__ void k_rows_count(const int32_t* __restrict__ grp_first, const int32_t* __restrict__ grp_nmem,
                             int64_t n_groups, const int32_t* __restrict__ ent_off,
                             const uint16_t* __restrict__ ent_pres, int32_t* __restrict__ row_count) {
  const int64_t g = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= n_groups) return;
  const int lane = threadIdx.x & 31;
  const int nmem = grp_nmem[g];
  int32_t cnt = 0;  // lane k: rows of member k
  for (int32_t e = ent_off[g] + lane; e - lane < ent_off[g + 1]; e += 32) {
    const uint32_t p = e < ent_off[g + 1] ? ent_pres[e] : 0u;
    for (int k = 0; k < nmem; ++k) {
      const int c = __popc(__ballot_sync(0xffffffffu, (p >> k) & 1u));
      if (lane == k) cnt += c;
    }
  }
  if (lane < nmem) row_count[grp_first[g] + lane] = cnt;
}

__global__ void k_rows_fill(const int32_t* __restrict__ grp_first, const int32_t* __restrict__ grp_nmem,
                            int64_t n_groups, const int32_t* __restrict__ ent_off, const int32_t* __restrict__ jorder,
                            const int32_t* __restrict__ ent_j, const uint64_t* __restrict__ ent_mask,
                            const uint16_t* __restrict__ ent_pres, int m, const int32_t* __restrict__ offsets,
                            int32_t* __restrict__ jv, uint64_t* __restrict__ mask) {
  const int64_t g = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= n_groups) return;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int nmem = grp_nmem[g];
  const int32_t first = grp_first[g];
  const int W = (m == 8) ? 2 : 1, mm = m * m;
  const uint64_t one = (mm == 64) ? ~0ull : ((1ull << mm) - 1ull);
  int32_t run = lane < nmem ? offsets[first + lane] : 0;  // lane k: next row of member k
  const int32_t e_beg = ent_off[g], e_end = ent_off[g + 1];
  for (int32_t t = e_beg + lane; t - lane < e_end; t += 32) {
    const bool valid = t < e_end;
    const int32_t e = valid ? (jorder ? jorder[t] : t) : 0;
    const uint32_t p = valid ? ent_pres[e] : 0u;
    const int32_t cj = valid ? ent_j[e] : 0;
    for (int k = 0; k < nmem; ++k) {
      const unsigned b = __ballot_sync(0xffffffffu, (p >> k) & 1u);
      if (!b) continue;
      const int32_t base = __shfl_sync(0xffffffffu, run, k);
      if ((p >> k) & 1u) {
        const int32_t row = base + __popc(b & lt);
        jv[row] = cj;
        mask[row] = (W == 2) ? ent_mask[(int64_t)e * 2 + k] : ((ent_mask[e] >> (k * mm)) & one);
      }
      if (lane == k) run += __popc(b);
    }
  }
}

cudaError_t ensure_rows(List* l, cudaStream_t s) {
  if (l->rows_ready) return cudaSuccess;
  const int64_t nc = l->n_clusters;
  DBuf<int32_t> cnt;
  int32_t h = 0;
  cudaError_t e;
  if ((e = cnt.alloc(nc + 1, s)) || (e = l->offsets.alloc(nc + 1, s))) goto out;
  if ((e = cudaMemsetAsync(cnt.p, 0, 4 * (nc + 1), s))) goto out;
  if (l->n_groups > 0) {
    count_launch();
    k_rows_count<<<nb(l->n_groups, 8), 256, 0, s>>>(l->group_first.p, l->group_nmem.p, l->n_groups,
                                                     l->ent_offsets.p, l->ent_pres.p, cnt.p);
  }
  if ((e = exclusive_scan_i32(cnt.p, l->offsets.p, nc + 1, s))) goto out;
  if ((e = cudaMemcpyAsync(&h, l->offsets.p + nc, 4, cudaMemcpyDeviceToHost, s))) goto out;
  if ((e = cudaStreamSynchronize(s))) goto out;
  l->n_rows = h;
  if ((e = l->j.alloc(l->n_rows, s)) || (e = l->mask.alloc(l->n_rows, s))) goto out;
  if (l->n_groups > 0 && l->n_rows > 0) {
    count_launch();
    k_rows_fill<<<nb(l->n_groups, 8), 256, 0, s>>>(l->group_first.p, l->group_nmem.p, l->n_groups,
                                                    l->ent_offsets.p, l->ent_jorder.p, l->ent_j.p, l->ent_mask.p,
                                                    l->ent_pres.p, l->m, l->offsets.p, l->j.p, l->mask.p);
  }
  if ((e = cudaGetLastError())) goto out;
  l->rows_ready = true;
  l->delta_ready = false;
out:
  cnt.release(s);
  return e;
}

// Per-row frame offsets (j-local -> i-local, image included, w = slack) for
// the canonical-row consumers (row statistics, canonical force path); built
// on demand, the grouped fast path never needs them.
__global__ void k_row_delta(const int32_t* __restrict__ offsets, const int32_t* __restrict__ jv, int64_t n_clusters,
                            const double* __restrict__ bbox, Box box, float4* __restrict__ delta) {
  const int64_t ci = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (ci >= n_clusters) return;
  double bi[6];
  for (int d = 0; d < 6; ++d) bi[d] = bbox[6 * ci + d];
  for (int32_t row = offsets[ci] + (threadIdx.x & 31); row < offsets[ci + 1]; row += 32) {
    double bj[6];
    const int64_t cj = jv[row];
    for (int d = 0; d < 6; ++d) bj[d] = bbox[6 * cj + d];
    float4 dl;
    float sl;
    image_delta(bi, bi, bj, box, &dl, &sl);
    delta[row] = dl;
  }
}

cudaError_t ensure_row_delta(List* l, cudaStream_t s) {
  cudaError_t e;
  if ((e = ensure_rows(l, s))) return e;
  if (l->delta_ready || l->n_rows == 0) return cudaSuccess;
  if ((e = l->delta.alloc(l->n_rows, s))) return e;
  Box bx;
  for (int d = 0; d < 3; ++d) {
    bx.L[d] = l->L[d];
    bx.invL[d] = 1.0 / l->L[d];
  }
  count_launch();
  k_row_delta<<<nb(l->n_clusters, 8), 256, 0, s>>>(l->offsets.p, l->j.p, l->n_clusters, l->bbox, bx, l->delta.p);
  if ((e = cudaGetLastError())) return e;
  l->delta_ready = true;
  return cudaSuccess;
}

// Force layout finishing touches, done once per list at its first force pass
// (lists that are only pruned never pay for them): entries ordered by member
// pattern within each group, groups ordered by descending size.
cudaError_t finalize_force_layout(List* l, cudaStream_t s) {
  if (l->ordered) return cudaSuccess;
  cudaError_t e;
  if (!l->entries_ordered && (e = order_entries(l, s))) return e;
  if ((e = order_groups(l, s))) return e;
  l->ordered = true;
  return cudaSuccess;
}

// rolling prune: force masks = canonical masks of the inner members
__global__ void k_reprune_apply(const uint64_t* __restrict__ em, const uint32_t* __restrict__ keep, int64_t cap,
                                const int32_t* __restrict__ live, int m, int G, uint64_t* __restrict__ fm) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= cap || e >= *live) return;
  const uint32_t ib = keep[e] >> 16;
  if (m == 8) {
    for (int q = 0; q < 2; ++q) fm[2 * e + q] = ((ib >> q) & 1u) ? em[2 * e + q] : 0ull;
  } else {
    fm[e] = em[e] & keep_mask(ib, m, G);
  }
}

cudaError_t reprune_inner(List* l, const float4* xyzq, const unsigned int* scalars, const double* bbox,
                          const double* cpos, const double box[3], cudaStream_t s) {
  if (!l->ent_fmask.p || l->r_inner <= 0.0 || l->n_groups == 0 || l->n_entries == 0) return cudaSuccess;
  const int64_t ne = l->n_entries, ng = l->n_groups, ns = l->n_clusters * l->m;
  DBuf<uint32_t> keep;
  DBuf<int32_t> alive;
  cudaError_t e;
  if ((e = keep.alloc(ne + 1, s)) || (e = alive.alloc(ng + 1, s))) goto out;
  {
    Box bx;
    for (int d = 0; d < 3; ++d) {
      bx.L[d] = box[d];
      bx.invL[d] = 1.0 / box[d];
    }
    const int pblocks = (int)std::min<int64_t>(ng, 148 * 64);
    const float slack_base = (float)(2.0 * l->r_list + 1e-3);
    const double r2i = l->r_inner * l->r_inner;
    // r2 = 0: only the inner bits are wanted (no canonical decisions, no FP64 replays)
    count_launch(2);
#define NBX_REPRUNE(MM, GG)                                                                                   \
  k_prune_entries<MM, GG><<<pblocks, PRUNE_WARPS * 32, 0, s>>>(l->group_first.p, l->group_nmem.p, ng,         \
                                                               l->ent_offsets.p, l->ent_j.p, l->ent_delta.p,  \
                                                               l->ent_mask.p, xyzq, bbox, cpos, bx, 0.0, r2i, \
                                                               scalars, slack_base, keep.p, alive.p)
    if (l->m == 4) NBX_REPRUNE(4, 4);
    else NBX_REPRUNE(8, 2);
#undef NBX_REPRUNE
    k_reprune_apply<<<nb(ne, 256), 256, 0, s>>>(l->ent_mask.p, keep.p, ne, l->ent_offsets.p + ng, l->m, l->G,
                                                 l->ent_fmask.p);
  }
  if ((e = cudaGetLastError())) goto out;
  // every entry is evaluated from now on (the inner pattern changed, the
  // order did not); validity counts from these coordinates
  if ((e = cudaMemcpyAsync(l->ent_fend.p, l->ent_offsets.p + 1, 4 * ng, cudaMemcpyDeviceToDevice, s))) goto out;
  if (!l->xprune.p && (e = l->xprune.alloc(ns, s))) goto out;
  if ((e = cudaMemcpyAsync(l->xprune.p, xyzq, sizeof(float4) * ns, cudaMemcpyDeviceToDevice, s))) goto out;
  l->tail_sorted = false;
  l->inner_ref = 5;
out:
  keep.release(s);
  alive.release(s);
  return e;
}

}  // namespace nbx

using namespace nbx;

static void list_release(nbx_list* l, cudaStream_t s) {
  l->offsets.drop(s); l->j.drop(s); l->mask.drop(s); l->delta.drop(s);
  l->group_first.drop(s);
  l->group_nmem.drop(s); l->group_order.drop(s); l->ent_offsets.drop(s); l->ent_j.drop(s);
  l->ent_delta.drop(s); l->ent_mask.drop(s); l->ent_pres.drop(s); l->ent_jorder.drop(s);
  l->halo_cl.drop(s);
  l->ent_fmask.drop(s); l->ent_fend.drop(s); l->xprune.drop(s);
  l->super_offsets.drop(s); l->super_j.drop(s); l->super_pair.drop(s);
  ForceWork& w = l->work;
  w.xyzq.drop(s); w.type.drop(s); w.part_i.drop(s); w.part_j.drop(s);
  w.e_grp.drop(s); w.scalars.drop(s); w.lj.drop(s); w.t_first.drop(s);
  w.t_items.drop(s); w.t_pos.drop(s); w.tc_first.drop(s); w.tc_items.drop(s);
}

extern "C" void nbx_list_free(nbx_list_t* l) {
  if (!l) return;
  list_release(l, 0);
  delete l;
}

static Box make_box(const double L[3]) {
  Box b;
  for (int d = 0; d < 3; ++d) {
    b.L[d] = L[d];
    b.invL[d] = 1.0 / L[d];
  }
  return b;
}

#define TRY(x)                                                      \
  do {                                                              \
    cudaError_t e_ = (x);                                           \
    if (e_ != cudaSuccess) {                                        \
      set_error("%s:%d %s", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      goto fail;                                                    \
    }                                                               \
  } while (0)

extern "C" int nbx_pairlist_build(const nbx_grid_t* grid, const double box[3], double r_list,
                                  void* stream, nbx_list_t** out) {
  return nbx_pairlist_build_ex(grid, box, r_list, nullptr, stream, out);
}

static int pairlist_build_impl(const nbx_grid_t* grid, const double box[3], double r_list, const uint8_t* halo,
                               const double* prune_pos, void* stream, nbx_list_t** out);

extern "C" int nbx_pairlist_build_ex(const nbx_grid_t* grid, const double box[3], double r_list,
                                     const uint8_t* halo, void* stream, nbx_list_t** out) {
  return pairlist_build_impl(grid, box, r_list, halo, nullptr, stream, out);
}

extern "C" int nbx_pairlist_build_pruned(const nbx_grid_t* grid, const double box[3], double r_list,
                                         const double* positions, const uint8_t* halo, void* stream,
                                         nbx_list_t** out) {
  if (!grid) {
    set_error("nbx_pairlist_build_pruned: null grid");
    return NBX_ERR_PARAM;
  }
  return pairlist_build_impl(grid, box, r_list, halo, positions ? positions : grid->cpos.p, stream, out);
}

static int pairlist_build_impl(const nbx_grid_t* grid, const double box[3], double r_list, const uint8_t* halo,
                               const double* prune_pos, void* stream, nbx_list_t** out) {
  if (!grid || !box || !out) {
    set_error("nbx_pairlist_build: null argument");
    return NBX_ERR_PARAM;
  }
  if (!(r_list > 0.0)) {
    set_error("r_list must be positive, got %g", r_list);
    return NBX_ERR_PARAM;
  }
  for (int d = 0; d < 3; ++d)
    if (box[d] < 2.0 * r_list) {
      set_error("every box edge must be >= 2*r_list=%g for the single-image convention", 2.0 * r_list);
      return NBX_ERR_PARAM;
    }
  cudaStream_t s = to_stream(stream);
  nbx_list* l = new nbx_list();
  *out = nullptr;
  const int m = grid->m, G = 16 / grid->m;
  const int64_t nc = grid->n_clusters, n_cols = grid->cells * grid->cells;
  l->m = m;
  l->G = G;
  l->n_clusters = nc;
  l->r_list = r_list;
  l->bbox = grid->bbox.p;
  for (int d = 0; d < 3; ++d) l->L[d] = box[d];
  Box bx = make_box(box);
  DBuf<int32_t> ent_count;
  DBuf<int2> stash;
  DBuf<uint8_t> hbits;
  DBuf<float4> xl;
  int32_t h[2] = {0, 0};
  SearchOut so{};
  (void)n_cols;
  l->n_groups = grid->n_groups;
  TRY(l->group_first.alloc(l->n_groups, s));
  TRY(l->group_nmem.alloc(l->n_groups, s));
  if (l->n_groups) {
    TRY(cudaMemcpyAsync(l->group_first.p, grid->group_first.p, 4 * l->n_groups, cudaMemcpyDeviceToDevice, s));
    TRY(cudaMemcpyAsync(l->group_nmem.p, grid->group_nmem.p, 4 * l->n_groups, cudaMemcpyDeviceToDevice, s));
  }
  TRY(ent_count.alloc(l->n_groups + 1, s));
  TRY(cudaMemsetAsync(ent_count.p, 0, 4 * (l->n_groups + 1), s));
  TRY(stash.alloc(l->n_groups * (int64_t)STASH, s));
  if (prune_pos && nc > 0) {
    TRY(xl.alloc(nc * m, s));
    count_launch();
    k_local_coords<<<nb(nc * m, 256), 256, 0, s>>>(prune_pos, grid->bbox.p, nc * m, m, xl.p);
    so.xl = xl.p;
    so.ppos = prune_pos;
  }
  if (halo && nc > 0) {
    TRY(hbits.alloc(nc, s));
    count_launch();
    k_halo_bits<<<nb(nc, 256), 256, 0, s>>>(halo, grid->perm.p, grid->fill.p, nc, m, hbits.p);
  }
  so.ent_count = ent_count.p;
  so.stash = stash.p;
  if (l->n_groups > 0)
  {
    count_launch();
    auto k0 = so.xl ? k_search<0, true> : k_search<0, false>;
    k0<<<nb(l->n_groups, SEARCH_WARPS), SEARCH_WARPS * 32, 0, s>>>(
        l->group_first.p, l->group_nmem.p, l->n_groups, m, G, grid->bbox.p, grid->bbf.p, grid->zr.p,
        grid->nreal.p, grid->col_first.p, grid->cells, bx, r_list, so, hbits.p);
  }
  TRY(cudaGetLastError());
  TRY(l->ent_offsets.alloc(l->n_groups + 1, s));
  TRY(exclusive_scan_i32(ent_count.p, l->ent_offsets.p, l->n_groups + 1, s));
  TRY(cudaMemcpyAsync(&h[1], l->ent_offsets.p + l->n_groups, 4, cudaMemcpyDeviceToHost, s));
  TRY(cudaStreamSynchronize(s));
  l->n_entries = h[1];
  TRY(l->ent_j.alloc(l->n_entries, s));
  TRY(l->ent_delta.alloc(l->n_entries, s));
  TRY(l->ent_mask.alloc(l->n_entries * l->mask_words(), s));
  TRY(l->ent_pres.alloc(l->n_entries, s));
  so.ent_offsets = l->ent_offsets.p;
  so.ent_j = l->ent_j.p;
  so.ent_delta = l->ent_delta.p;
  so.ent_mask = l->ent_mask.p;
  so.ent_pres = l->ent_pres.p;
  if (l->n_groups > 0)
  {
    count_launch();
    auto k1 = so.xl ? k_search<1, true> : k_search<1, false>;
    k1<<<nb(l->n_groups, SEARCH_WARPS), SEARCH_WARPS * 32, 0, s>>>(
        l->group_first.p, l->group_nmem.p, l->n_groups, m, G, grid->bbox.p, grid->bbf.p, grid->zr.p,
        grid->nreal.p, grid->col_first.p, grid->cells, bx, r_list, so, hbits.p);
  }
  TRY(cudaGetLastError());
  ent_count.release(s); stash.release(s);
  if (hbits.p) std::swap(l->halo_cl, hbits);  // per-cluster halo bits: interior / boundary work split
  hbits.release(s); xl.release(s);
  *out = l;
  return NBX_OK;
fail:
  ent_count.release(s); stash.release(s);
  hbits.release(s); xl.release(s);
  nbx_list_free(l);
  return NBX_ERR_CUDA;
}

extern "C" int nbx_pairlist_prune(const nbx_list_t* in, const nbx_grid_t* grid,
                                  const double* pos, const double box[3], void* stream,
                                  nbx_list_t** out) {
  return nbx_pairlist_prune_inner(in, grid, pos, box, 0.0, stream, out);
}

extern "C" int nbx_pairlist_prune_inner(const nbx_list_t* in, const nbx_grid_t* grid,
                                        const double* pos, const double box[3], double r_inner, void* stream,
                                        nbx_list_t** out) {
  if (!in || !grid || !pos || !box || !out) {
    set_error("nbx_pairlist_prune: null argument");
    return NBX_ERR_PARAM;
  }
  if (r_inner != 0.0 && !(r_inner > 0.0 && r_inner <= in->r_list)) {
    set_error("r_inner must be 0 (off) or in (0, r_list=%g], got %g", in->r_list, r_inner);
    return NBX_ERR_PARAM;
  }
  if (in->m < 4) r_inner = 0.0;  // the inner list feeds k_force_h (m = 4, 8) only
  if (r_inner != 0.0 && pos != grid->cpos.p) {  // the force pass measures d_max against the build positions
    set_error("dynamic pruning (r_inner) needs the grid's own build positions");
    return NBX_ERR_PARAM;
  }
  if (grid->n_clusters != in->n_clusters || grid->m != in->m) {
    set_error("nbx_pairlist_prune: grid does not match the list");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  nbx_list* l = new nbx_list();
  *out = nullptr;
  l->m = in->m;
  l->G = in->G;
  l->n_clusters = in->n_clusters;
  l->n_groups = in->n_groups;
  l->r_list = in->r_list;
  l->r_inner = r_inner;
  l->bbox = in->bbox;
  for (int d = 0; d < 3; ++d) l->L[d] = in->L[d];
  const int W = in->mask_words();
  const int64_t ne = in->n_entries, nc = in->n_clusters, ng = in->n_groups;
  Box bx = make_box(box);
  DBuf<int32_t> alive;
  DBuf<float4> xl;
  DBuf<uint32_t> ekeep, dmax;
  int32_t h = 0;
  TRY(dmax.alloc(1, s));
  TRY(cudaMemsetAsync(dmax.p, 0, 4, s));
  TRY(alive.alloc(ng + 1, s));
  TRY(cudaMemsetAsync(alive.p, 0, 4 * (ng + 1), s));
  TRY(ekeep.alloc(ne + 1, s));
  TRY(xl.alloc(nc * in->m, s));
  if (nc > 0 && ng > 0) {
    count_launch(2);
    k_local_coords<<<nb(nc * in->m, 256), 256, 0, s>>>(pos, grid->bbox.p, nc * in->m, in->m, xl.p, grid->cpos.p,
                                                       dmax.p);
    const int pblocks = (int)std::min<int64_t>(ng, 148 * 64);
    const float slack_base = (float)(2.0 * in->r_list + 1e-3);
    const double r2 = in->r_list * in->r_list, r2i = r_inner * r_inner;
#define NBX_PRUNE(MM, GG)                                                                                     \
  k_prune_entries<MM, GG><<<pblocks, PRUNE_WARPS * 32, 0, s>>>(in->group_first.p, in->group_nmem.p, ng,        \
                                                               in->ent_offsets.p, in->ent_j.p, in->ent_delta.p, \
                                                               in->ent_mask.p, xl.p, grid->bbox.p, pos, bx, r2,  \
                                                               r2i, dmax.p, slack_base, ekeep.p, alive.p)
    switch (in->m) {
      case 1: NBX_PRUNE(1, 16); break;
      case 2: NBX_PRUNE(2, 8); break;
      case 4: NBX_PRUNE(4, 4); break;
      default: NBX_PRUNE(8, 2); break;
    }
#undef NBX_PRUNE
  }
  TRY(cudaGetLastError());
  TRY(l->ent_offsets.alloc(ng + 1, s));
  TRY(exclusive_scan_i32(alive.p, l->ent_offsets.p, ng + 1, s));
  // no host sync: storage sized by the input's entries (an upper bound), the
  // live count stays on the device (ent_offsets[n_groups]); unused j slots
  // hold n_clusters so that they sort last in the force-layout transposes
  (void)h;
  l->n_entries = ne;
  l->entries_exact = (ne == 0);
  TRY(l->group_first.alloc(ng, s));
  TRY(l->group_nmem.alloc(ng, s));
  TRY(l->ent_j.alloc(l->n_entries, s));
  TRY(l->ent_delta.alloc(l->n_entries, s));
  TRY(l->ent_mask.alloc(l->n_entries * W, s));
  TRY(l->ent_pres.alloc(l->n_entries, s));
  TRY(l->ent_jorder.alloc(l->n_entries, s));
  if (r_inner > 0.0) {
    TRY(l->ent_fmask.alloc(l->n_entries * W, s));
    TRY(l->ent_fend.alloc(ng, s));
  }
  if (ne) count_launch(), k_fill_i32<<<nb(ne, 256), 256, 0, s>>>(l->ent_j.p, ne, (int32_t)nc);
  if (ng) {
    TRY(cudaMemcpyAsync(l->group_first.p, in->group_first.p, 4 * ng, cudaMemcpyDeviceToDevice, s));
    TRY(cudaMemcpyAsync(l->group_nmem.p, in->group_nmem.p, 4 * ng, cudaMemcpyDeviceToDevice, s));
    count_launch();
    k_compact_order<<<nb(ng, ORDER_WARPS), ORDER_WARPS * 32, 0, s>>>(
        in->ent_offsets.p, ng, in->ent_jorder.p, ekeep.p, in->ent_j.p, in->ent_delta.p, in->ent_mask.p, in->m, in->G,
        l->ent_offsets.p, l->ent_j.p, l->ent_delta.p, l->ent_mask.p, l->ent_pres.p, l->ent_jorder.p,
        r_inner > 0.0 ? l->ent_fmask.p : nullptr, r_inner > 0.0 ? l->ent_fend.p : nullptr);
  }
  TRY(cudaGetLastError());
  l->entries_ordered = true;
  if (in->halo_cl.p) {  // the domain's halo bits travel with the list
    TRY(l->halo_cl.alloc(nc, s));
    TRY(cudaMemcpyAsync(l->halo_cl.p, in->halo_cl.p, nc, cudaMemcpyDeviceToDevice, s));
  }
  alive.release(s); xl.release(s); ekeep.release(s); dmax.release(s);
  *out = l;
  return NBX_OK;
fail:
  alive.release(s); xl.release(s); ekeep.release(s); dmax.release(s);
  nbx_list_free(l);
  return NBX_ERR_CUDA;
}

extern "C" int nbx_list_info(const nbx_list_t* l, int64_t out[5]) {
  if (!l || !out) {
    set_error("nbx_list_info: null argument");
    return NBX_ERR_PARAM;
  }
  out[0] = l->n_clusters;
  out[1] = l->rows_ready ? l->n_rows : -1;  // canonical rows: nbx_list_rows
  out[2] = l->m;
  out[3] = l->n_groups;
  out[4] = l->entries_exact ? (l->n_live >= 0 ? l->n_live : l->n_entries) : -1;  // -1: nbx_list_entries
  return NBX_OK;
}

extern "C" int nbx_list_entries(nbx_list_t* l, void* stream, int64_t* n_entries) {
  if (!l || !n_entries) {
    set_error("nbx_list_entries: null argument");
    return NBX_ERR_PARAM;
  }
  if (!l->entries_exact) {  // live entry count of a pruned list (kept on the device until asked for)
    int32_t h = 0;
    cudaStream_t s = to_stream(stream);
    cudaError_t e = cudaMemcpyAsync(&h, l->ent_offsets.p + l->n_groups, 4, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e) {
      set_error("nbx_list_entries: %s", cudaGetErrorString(e));
      return NBX_ERR_CUDA;
    }
    l->n_live = h;
    l->entries_exact = true;
  }
  *n_entries = l->n_live >= 0 ? l->n_live : l->n_entries;
  return NBX_OK;
}

__global__ void k_popcount_live(const uint64_t* __restrict__ words, int64_t cap, int W,
                                const int32_t* __restrict__ live, unsigned long long* __restrict__ out) {
  const int64_t n = min((int64_t)*live * W, cap);
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += __popcll(words[i]);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

extern "C" int nbx_list_force_pairs(nbx_list_t* l, int32_t inner, void* stream, int64_t* n_pairs) {
  if (!l || !n_pairs) {
    set_error("nbx_list_force_pairs: null argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  const int W = l->mask_words();
  const uint64_t* words = (inner && l->r_inner > 0.0 && l->ent_fmask.p) ? l->ent_fmask.p : l->ent_mask.p;
  DBuf<unsigned long long> cnt;
  unsigned long long h = 0;
  cudaError_t e;
  if ((e = cnt.alloc(1, s)) || (e = cudaMemsetAsync(cnt.p, 0, 8, s))) goto out;
  if (l->n_entries > 0 && l->n_groups > 0) {
    count_launch();
    k_popcount_live<<<148 * 4, 256, 0, s>>>(words, l->n_entries * W, W, l->ent_offsets.p + l->n_groups, cnt.p);
  }
  if ((e = cudaGetLastError()) || (e = cudaMemcpyAsync(&h, cnt.p, 8, cudaMemcpyDeviceToHost, s)) ||
      (e = cudaStreamSynchronize(s)))
    goto out;
  *n_pairs = (int64_t)h;
out:
  cnt.release(s);
  if (e) {
    set_error("nbx_list_force_pairs: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  return NBX_OK;
}

template <typename TD, typename TH>
static cudaError_t dl(const TD* d, int64_t count, TH* h, cudaStream_t s) {
  if (!h || count <= 0) return cudaSuccess;
  TD* tmp = (TD*)malloc(sizeof(TD) * (size_t)count);
  cudaError_t e = cudaMemcpyAsync(tmp, d, sizeof(TD) * (size_t)count, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  if (!e)
    for (int64_t i = 0; i < count; ++i) h[i] = (TH)tmp[i];
  free(tmp);
  return e;
}

extern "C" int nbx_list_rows(nbx_list_t* l, void* stream, int64_t* n_rows) {
  if (!l || !n_rows) {
    set_error("nbx_list_rows: null argument");
    return NBX_ERR_PARAM;
  }
  cudaError_t e = ensure_rows(l, to_stream(stream));
  if (e) {
    set_error("nbx_list_rows: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  *n_rows = l->n_rows;
  return NBX_OK;
}

extern "C" int nbx_list_download(const nbx_list_t* l, int64_t* offsets, int64_t* j_idx,
                                 uint64_t* masks, void* stream) {
  if (!l) {
    set_error("nbx_list_download: null list");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  cudaError_t e;
  if ((e = ensure_rows(const_cast<nbx_list*>(static_cast<const nbx_list*>(l)), s)) || (e = dl(l->offsets.p, l->n_clusters + 1, offsets, s)) || (e = dl(l->j.p, l->n_rows, j_idx, s)) ||
      (e = dl(l->mask.p, l->n_rows, masks, s))) {
    set_error("nbx_list_download: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  return NBX_OK;
}

extern "C" int nbx_count_within(const nbx_list_t* l, const double* pos, const double box[3],
                                double r_cut, void* stream, int64_t out[2]) {
  if (!l || !pos || !box || !out) {
    set_error("nbx_count_within: null argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  DBuf<unsigned long long> cnt;
  DBuf<float4> xl;
  unsigned long long h[2] = {0, 0};
  TRY(cnt.alloc(2, s));
  TRY(xl.alloc(l->n_clusters * l->m, s));
  TRY(cudaMemsetAsync(cnt.p, 0, 16, s));
  TRY(ensure_row_delta(const_cast<nbx_list*>(static_cast<const nbx_list*>(l)), s));
  if (l->n_clusters > 0) {
    count_launch();
    k_local_coords<<<nb(l->n_clusters * l->m, 256), 256, 0, s>>>(pos, l->bbox, l->n_clusters * l->m, l->m, xl.p);
    launch_rows<1>(l->m, l->n_clusters, s, l->offsets.p, l->j.p, l->mask.p, l->delta.p, nullptr, l->G, pos, xl.p,
                   make_box(box), r_cut * r_cut, nullptr, nullptr, nullptr, nullptr, nullptr, cnt.p);
  }
  TRY(cudaGetLastError());
  TRY(cudaMemcpyAsync(h, cnt.p, 16, cudaMemcpyDeviceToHost, s));
  TRY(cudaStreamSynchronize(s));
  cnt.release(s);
  xl.release(s);
  out[0] = (int64_t)h[0];
  out[1] = (int64_t)h[1];
  return NBX_OK;
fail:
  cnt.release(s);
  xl.release(s);
  return NBX_ERR_CUDA;
}

extern "C" int nbx_super_layout(const nbx_list_t* lc, int32_t size, void* stream, int64_t* n_entries) {
  if (!lc || size < 1) {
    set_error("nbx_super_layout: bad argument");
    return NBX_ERR_PARAM;
  }
  nbx_list* l = const_cast<nbx_list*>(static_cast<const nbx_list*>(lc));
  cudaStream_t s = to_stream(stream);
  if (cudaError_t e0 = ensure_rows(l, s)) {
    set_error("nbx_super_layout: %s", cudaGetErrorString(e0));
    return NBX_ERR_CUDA;
  }
  const int64_t nr = l->n_rows, nc = l->n_clusters;
  const int64_t ngr = (nc + size - 1) / size;
  DBuf<int32_t> ci_of_row, vals, vals2, head, hscan, gcount;
  DBuf<uint64_t> keys, keys2;
  int32_t ne = 0;
  size_t bytes = 0;
  void* tmp = nullptr;
  TRY(ci_of_row.alloc(nr, s));
  TRY(vals.alloc(nr, s));
  TRY(vals2.alloc(nr, s));
  TRY(keys.alloc(nr, s));
  TRY(keys2.alloc(nr, s));
  TRY(head.alloc(nr + 1, s));
  TRY(hscan.alloc(nr + 1, s));
  TRY(gcount.alloc(ngr + 1, s));
  TRY(cudaMemsetAsync(gcount.p, 0, 4 * (ngr + 1), s));
  if (nc) count_launch(), k_row_ci<<<nb(nc, 256), 256, 0, s>>>(l->offsets.p, nc, ci_of_row.p);
  if (nr) {
    count_launch(), k_super_keys<<<nb(nr, 256), 256, 0, s>>>(ci_of_row.p, l->j.p, nr, size, nc, keys.p, vals.p);
    TRY(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, keys2.p, vals.p, vals2.p, (int)nr, 0, 64, s));
    TRY(pool_malloc(&tmp, bytes, s));
    TRY(cub::DeviceRadixSort::SortPairs(tmp, bytes, keys.p, keys2.p, vals.p, vals2.p, (int)nr, 0, 64, s));
    cudaFreeAsync(tmp, s);
  }
  count_launch(), k_super_heads<<<nb(nr + 1, 256), 256, 0, s>>>(keys2.p, nr, head.p);
  TRY(exclusive_scan_i32(head.p, hscan.p, nr + 1, s));
  TRY(cudaMemcpyAsync(&ne, hscan.p + nr, 4, cudaMemcpyDeviceToHost, s));
  TRY(cudaStreamSynchronize(s));
  TRY(l->super_j.alloc(ne, s));
  TRY(l->super_pair.alloc((int64_t)ne * size, s));
  TRY(l->super_offsets.alloc(ngr + 1, s));
  TRY(cudaMemsetAsync(l->super_pair.p, 0xff, 4 * (size_t)ne * size, s));
  if (nr)
    count_launch(), k_super_fill<<<nb(nr, 256), 256, 0, s>>>(keys2.p, vals2.p, hscan.p, ci_of_row.p, nr, size, nc,
                                             l->super_j.p, l->super_pair.p, gcount.p);
  TRY(exclusive_scan_i32(gcount.p, l->super_offsets.p, ngr + 1, s));
  TRY(cudaGetLastError());
  TRY(cudaStreamSynchronize(s));
  l->super_size = size;
  l->super_groups = ngr;
  l->super_entries = ne;
  *n_entries = ne;
  ci_of_row.release(s); vals.release(s); vals2.release(s); keys.release(s); keys2.release(s);
  head.release(s); hscan.release(s); gcount.release(s);
  return NBX_OK;
fail:
  ci_of_row.release(s); vals.release(s); vals2.release(s); keys.release(s); keys2.release(s);
  head.release(s); hscan.release(s); gcount.release(s);
  return NBX_ERR_CUDA;
}

extern "C" int nbx_super_download(const nbx_list_t* l, int64_t* super_offsets, int64_t* super_j,
                                  int64_t* super_pair_idx, void* stream) {
  if (!l || l->super_size == 0) {
    set_error("nbx_super_download: layout not built");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  cudaError_t e;
  if ((e = dl(l->super_offsets.p, l->super_groups + 1, super_offsets, s)) ||
      (e = dl(l->super_j.p, l->super_entries, super_j, s)) ||
      (e = dl(l->super_pair.p, l->super_entries * l->super_size, super_pair_idx, s))) {
    set_error("nbx_super_download: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  return NBX_OK;
}

// ---------------------------------------------------------------- row diagnostics
// pairlist.write_pairs_csv (pairlist.py:349-376) computes, per canonical row,
// the periodic bounding-box gap (gridder.py:165-185) and the exact minimum
// admitted slot distance at the build positions (_pair_min_dist_sq,
// pairlist.py:220-239: numpy min image, einsum order, +inf when no slot pair
// is admitted).  One thread per row, the reference's FP64 operation order
// (this TU is compiled with -fmad=false): the values are bit-identical, so
// the CSV text is too.
__global__ void k_row_diag(const int32_t* __restrict__ ci_of_row, const int32_t* __restrict__ jv,
                           const uint64_t* __restrict__ mask, int64_t n_rows, int m, const double* __restrict__ bbox,
                           const double* __restrict__ pos, Box box, double* __restrict__ gap_sq,
                           double* __restrict__ min_d2) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const int64_t ci = ci_of_row[r], cj = jv[r];
  gap_sq[r] = nbx::gap_sq(bbox + 6 * ci, bbox + 6 * cj, box);
  const uint64_t mk = mask[r];
  double best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  for (int a = 0; a < m; ++a) {
    const double* pi = pos + 3 * (ci * m + a);
    for (int b = 0; b < m; ++b) {
      if (!((mk >> (a * m + b)) & 1ull)) continue;
      const double* pj = pos + 3 * (cj * m + b);
      const double dx = min_image_np(__dsub_rn(pi[0], pj[0]), box.L[0], box.invL[0]);
      const double dy = min_image_np(__dsub_rn(pi[1], pj[1]), box.L[1], box.invL[1]);
      const double dz = min_image_np(__dsub_rn(pi[2], pj[2]), box.L[2], box.invL[2]);
      const double d2 = d2_einsum(dx, dy, dz);
      best = d2 < best ? d2 : best;
    }
  }
  min_d2[r] = best;
}

extern "C" int nbx_list_diagnostics(nbx_list_t* l, const nbx_grid_t* grid, const double* positions,
                                    const double box[3], double* gap_sq, double* min_d2, void* stream) {
  if (!l || !grid || !box || !gap_sq || !min_d2 || grid->m != l->m || grid->n_clusters != l->n_clusters) {
    set_error("nbx_list_diagnostics: bad argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  DBuf<int32_t> ci;
  const double* pos = positions ? positions : grid->cpos.p;
  TRY(ensure_rows(l, s));
  if (l->n_rows > 0) {
    TRY(ci.alloc(l->n_rows, s));
    count_launch(2);
    k_row_ci<<<nb(l->n_clusters, 256), 256, 0, s>>>(l->offsets.p, l->n_clusters, ci.p);
    k_row_diag<<<nb(l->n_rows, 256), 256, 0, s>>>(ci.p, l->j.p, l->mask.p, l->n_rows, l->m, grid->bbox.p, pos,
                                                   make_box(box), gap_sq, min_d2);
    TRY(cudaGetLastError());
  }
  ci.release(s);
  return NBX_OK;
fail:
  ci.release(s);
  return NBX_ERR_CUDA;
}

// ---------------------------------------------------------------- exclusions
// Intramolecular exclusions (extension; the reference masks only fillers and
// the diagonal, pairlist.py:106-112): slot pairs whose particles carry the
// same molecule id are removed from the masks, so rigid water (SPC, SETTLE)
// has no intramolecular non-bonded terms.  Applied to a finished list, in
// place: the canonical masks (ent_mask) and the inner force masks (ent_fmask)
// of every entry.  Member presence and the entry order are unchanged (a
// member row always keeps pairs with other molecules: a cluster pair never
// holds only one molecule's atoms when m >= 2 and molecules have <= m atoms
// ... and when it does, the row simply evaluates nothing).
// One thread per slot: for each partner atom of the slot's molecule that
// the half list pairs it with (cluster cj > ci, or cj == ci and b > a), find
// the entry (group of ci, cj) by binary search over the group's entries in
// ascending j (ent_jorder) and clear the bit; a pruned row is simply absent.
// The molecules come as a CSR (mol_first / mol_atoms: the atoms of each
// molecule) plus the per-atom id (atom_mol); any id layout works.
__global__ void k_cluster_group(const int32_t* __restrict__ grp_first, const int32_t* __restrict__ grp_nmem,
                                int64_t n_groups, int32_t* __restrict__ cgroup) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= n_groups) return;
  for (int k = 0; k < grp_nmem[g]; ++k) cgroup[grp_first[g] + k] = (int32_t)g;
}

// per group, the entries' j-clusters in ascending order (binary-search keys)
// (t < ent_off[n_groups]: a pruned list's storage may hold unused slots past the live entries)
__global__ void k_sorted_j(const int32_t* __restrict__ jorder, const int32_t* __restrict__ ent_j, int64_t n,
                           const int32_t* __restrict__ live_end, int32_t* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n && t < *live_end) out[t] = ent_j[jorder ? jorder[t] : t];
}

constexpr int EXCL_SPLIT = 3;  // threads per slot (partners q, q + 3, ...)
__global__ void k_exclude(const int32_t* __restrict__ perm, const int32_t* __restrict__ inv_perm,
                          const uint8_t* __restrict__ fill, int64_t n_slots, const int32_t* __restrict__ mol_atoms,
                          const int32_t* __restrict__ mol_first, const int32_t* __restrict__ atom_mol,
                          const int32_t* __restrict__ cgroup, const int32_t* __restrict__ grp_first,
                          const int32_t* __restrict__ ent_off, const int32_t* __restrict__ jorder,
                          const int32_t* __restrict__ sj_sorted, int m, uint64_t* __restrict__ ent_mask,
                          uint64_t* __restrict__ ent_fmask, unsigned long long* __restrict__ n_removed) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t si = tid / EXCL_SPLIT;
  const int part = (int)(tid - si * EXCL_SPLIT);
  unsigned long long removed = 0;
  if (si < n_slots && !fill[si]) {
    const int32_t oi = __ldg(perm + si), mo = __ldg(atom_mol + oi);
    const int64_t ci = si / m;
    const int a = (int)(si - ci * m);
    const int32_t g = __ldg(cgroup + ci), k = (int32_t)(ci - __ldg(grp_first + g));
    const int W = (m == 8) ? 2 : 1, mm = m * m;
    const int32_t t_lo = __ldg(ent_off + g), t_hi = __ldg(ent_off + g + 1);
    for (int32_t q = __ldg(mol_first + mo) + part; q < __ldg(mol_first + mo + 1); q += EXCL_SPLIT) {
      const int32_t op = __ldg(mol_atoms + q);
      if (op == oi) continue;
      const int64_t sj = __ldg(inv_perm + op);
      const int64_t cj = sj / m;
      const int b = (int)(sj - cj * m);
      if (cj < ci || (cj == ci && b <= a)) continue;  // held by the other atom's row (or nowhere)
      int32_t lo = t_lo, hi = t_hi;                    // first t with sorted j >= cj
      while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (__ldg(sj_sorted + mid) < cj) lo = mid + 1;
        else hi = mid;
      }
      if (lo >= t_hi || __ldg(sj_sorted + lo) != cj) continue;
      const int32_t e = jorder ? __ldg(jorder + lo) : lo;
      const int bit = (W == 2) ? a * m + b : k * mm + a * m + b;
      const int64_t w = (int64_t)e * W + (W == 2 ? k : 0);
      const uint64_t bm = 1ull << bit;
      const unsigned long long old = atomicAnd(reinterpret_cast<unsigned long long*>(ent_mask + w), ~bm);
      removed += (old & bm) ? 1ull : 0ull;
      if (ent_fmask) atomicAnd(reinterpret_cast<unsigned long long*>(ent_fmask + w), ~bm);
    }
  }
  for (int o = 16; o; o >>= 1) removed += __shfl_xor_sync(0xffffffffu, removed, o);
  if ((threadIdx.x & 31) == 0 && removed) atomicAdd(n_removed, removed);
}

extern "C" int nbx_list_exclude(nbx_list_t* l, const nbx_grid_t* grid, const int32_t* atom_mol,
                                const int32_t* mol_first, const int32_t* mol_atoms, void* stream, int64_t* n_removed) {
  if (!l || !grid || (grid->n > 0 && (!atom_mol || !mol_first || !mol_atoms)) || grid->m != l->m ||
      grid->n_clusters != l->n_clusters) {
    set_error("nbx_list_exclude: bad argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  DBuf<int32_t> cg, sj;
  DBuf<unsigned long long> cnt;
  unsigned long long h = 0;
  const int64_t ns = grid->n_slots();
  TRY(cnt.alloc(1, s));
  TRY(cudaMemsetAsync(cnt.p, 0, 8, s));
  if (ns > 0 && l->n_groups > 0 && l->n_entries > 0) {
    TRY(cg.alloc(l->n_clusters, s));
    TRY(sj.alloc(l->n_entries, s));
    count_launch(3);
    k_cluster_group<<<nb(l->n_groups, 256), 256, 0, s>>>(l->group_first.p, l->group_nmem.p, l->n_groups, cg.p);
    k_sorted_j<<<nb(l->n_entries, 256), 256, 0, s>>>(l->ent_jorder.p, l->ent_j.p, l->n_entries,
                                                      l->ent_offsets.p + l->n_groups, sj.p);
    k_exclude<<<nb(ns * EXCL_SPLIT, 128), 128, 0, s>>>(grid->perm.p, grid->inverse_perm.p, grid->fill.p, ns,
                                                        mol_atoms, mol_first, atom_mol, cg.p, l->group_first.p,
                                                        l->ent_offsets.p, l->ent_jorder.p, sj.p, l->m, l->ent_mask.p,
                                                        l->ent_fmask.p, cnt.p);
    TRY(cudaGetLastError());
  }
  // canonical rows and the reference super layout are re-derived from the
  // entries on their next use
  l->rows_ready = false;
  l->delta_ready = false;
  l->super_size = 0;
  if (n_removed) {
    TRY(cudaMemcpyAsync(&h, cnt.p, 8, cudaMemcpyDeviceToHost, s));
    TRY(cudaStreamSynchronize(s));
    *n_removed = (int64_t)h;
  }
  cg.release(s);
  sj.release(s);
  cnt.release(s);
  return NBX_OK;
fail:
  cg.release(s);
  sj.release(s);
  cnt.release(s);
  return NBX_ERR_CUDA;
}
