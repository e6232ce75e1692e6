// Non-bonded force + energy over the cluster-pair list (sm_100a).
//
// Replaces kernels.compute_nonbonded_into (kernels.py:328-396) with its numba
// kernels _kernel_blocks (:124-221) and _kernel_super_blocks (:224-312) of
// /root/reference/pkg/src/clustermd, and extends the pair potential
// (lj_coulomb_terms, :84-111) with reaction-field and Ewald real-space terms.
//
// Work unit: a GROUP of G consecutive i-clusters (16 i-atoms) and its ENTRIES
// (one per j-cluster, carrying every member's m x m mask; search.cu).  One
// warp per group.  Lane (r, b) = (entry slot r of 32/m, j-atom b of m): each
// lane holds one j-atom in registers and sweeps the group's 16 i-atoms, which
// live in shared memory (broadcast LDS).  Consequences:
//   * j-forces accumulate in registers across all members -> one float4 store
//     per (entry, j-atom): no atomics, no shuffles;
//   * i-forces accumulate in registers across all entries -> one shared-memory
//     transpose-reduce per group;
//   * members absent from every entry of an iteration are skipped
//     warp-uniformly.
// The j-side partials are summed per atom by k_reduce in a fixed order
// (entries sorted by j-cluster), so forces are bit-reproducible with no
// fixed-point or float atomics.  Energies: FP32 per pair, FP64 per lane,
// fixed-order reduction.
//
// Periodicity: every entry carries the image shift of its j-cluster relative
// to the group (search.cu); a per-pair FP32 minimum image is used instead for
// the (rare) iterations holding an entry whose slack cannot guarantee a single
// image at the current displacements.  Cutoff decisions within a narrow band
// around r_c are re-made in FP64 exactly as the reference (kernels.py:165-184)
// when the Coulomb force is discontinuous at r_c (cutoff / reaction-field).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <functional>

#include "internal.cuh"

namespace nbx {

enum { FE_RF = 0, FE_EWALD = 1 };

struct ForceArgs {
  // work items
  int64_t n_work;
  const int32_t* sel;         // optional: work item -> group / i-cluster
  const int32_t* grp_first;   // group -> first member cluster (NULL: identity, canonical)
  const int32_t* grp_nmem;    // group -> member count (NULL: 1)
  const int32_t* ent_off;     // group -> entry range
  const int32_t* ent_j;
  const float4* ent_delta;    // j-local -> group-local offset (image included)
  const uint64_t* ent_mask;
  const uint64_t* ent_fmask;  // k_force_h: inner-list masks (dynamic pruning; NULL: none)
  const int32_t* ent_fend;    // group -> end of its entries with an inner member
  float inner_dmax;           // inner masks valid while d_max (scalars[inner_slot]) <= this
  int inner_slot;             // 0: displacement since the build, 5: since the rolling prune
  const int32_t* ent_tpos;    // k_force_h: entry -> partial-force slot in j-cluster order (NULL: entry order)
  int split;                  // k_force_h: work items per group (1, 2, 4, 8: parts of its entry range)
  int64_t wbase;              // k_force_h: global index of this launch's first work item
  int64_t ns;                 // slots (one i-partial plane per part)
  // per-slot inputs
  const float4* xyzq;         // cluster-local coordinates (relative to bbox low corner)
  const double* bbox;         // grid bboxes (origins of the local frames)
  const int32_t* type;
  const float4* lj;           // (nt * nt) {6 c6, 12 c12, shift_lj, 0}
  int nt;
  // outputs
  float4* part_i;
  float4* part_j;
  double* e_grp;              // 2 per work item
  unsigned int* scalars;      // [0] max displacement (float bits); [2..3] bad key
  // physics
  float rc2, k2rf, krf, crf, coul;
  float beta, beta3, ew_shift, ew_a;
  float ew_f[16], ew_v[16];         // EW_DEG + 1 (<= 16) coefficients, highest first
  float ew_s[16];                   // -beta^3 * ew_f (k_force_h)
  float slack_base;           // 2 r_c + margin; unsafe if slack < base + 4 d_max
  float band;
  float L[3], invL[3];
  // exact re-check
  const double* pos;          // original order
  const int32_t* perm;
  double rc2d;
  Box box;
};

__device__ __forceinline__ void record_bad(unsigned int* scalars, int64_t si, int64_t sj) {
  unsigned long long key = ((unsigned long long)si << 32) | (unsigned long long)(sj & 0xffffffff);
  atomicMin(reinterpret_cast<unsigned long long*>(scalars + 2), key);
}

// Exact reference decision for one pair (kernels.py:165-184): raw gathered
// positions, numba min image, sequential r^2.  Returns 1 inside, 0 outside,
// -1 singular.
__device__ __noinline__ int exact_inside(const ForceArgs& A, int64_t si, int64_t sj) {
  const int64_t oi = A.perm[si], oj = A.perm[sj];
  double d[3];
  for (int k = 0; k < 3; ++k)
    d[k] = min_image_kernel(__dsub_rn(A.pos[3 * oi + k], A.pos[3 * oj + k]), A.box.L[k], A.box.invL[k]);
  const double r2 = d2_seq(d[0], d[1], d[2]);
  if (r2 > A.rc2d) return 0;
  if (r2 == 0.0) return -1;
  return 1;
}

constexpr int FW = 4;  // warps per block

template <int M>
__host__ __device__ constexpr uint64_t column_bits() {
  uint64_t c = 0;
  for (int a = 0; a < M; ++a) c |= 1ull << (a * M);
  return c;
}

// Ewald real space without transcendentals beyond the per-pair rsqrt: with
// z = beta r, w = z^2 and u = w (2 / w_max) - 1 in [-1, 1] (host-fitted
// Chebyshev series of functions ANALYTIC in w, ew_fit below):
//   Gf(u) ~ erf(z)/z^3 - 2 exp(-w) / (sqrt(pi) w)  ->  F_c/r = qq (1/r^3 - beta^3 Gf)
//   Gv(u) ~ erf(z)/z                               ->  E_c = qq (1/r - beta Gv - shift)
// (the GROMACS analytical-Ewald split).  The polynomial terms do not vanish
// with rinv, so they are masked through qm = inc ? qq : 0.
// degree 10 for the force term (force rel-RMS ~5e-6 vs FP64 on SPC water,
// tolerance 1e-4), 12 for the energy term (~2e-8, tolerance 1e-5)
#ifndef NBX_EW_ESTRIN
#define NBX_EW_ESTRIN 0
#endif
#ifndef NBX_EW_DEG_F
#define NBX_EW_DEG_F 10
#endif
constexpr int EW_DEG_F = NBX_EW_DEG_F;
constexpr int EW_DEG_V = 12;

// bits a*M + {0, 1}, a < M: one member's i-atoms against a lane's two j-atoms
template <int M>
__host__ __device__ constexpr uint64_t pair_column_bits() {
  uint64_t c = 0;
  for (int a = 0; a < M; ++a) c |= 3ull << (a * M);
  return c;
}

// One pair: F/r, plus energies when requested.  `inc` zeroes rinv, which
// masks every force term; energy shift terms are masked explicitly.
template <int ELEC, bool KRF, bool ENERGY>
__device__ __forceinline__ float pair_eval(const ForceArgs& A, const float4& xi, const float4& lj, float xjw,
                                           float r2, bool inc, float& elj, float& ec) {
  float rinv = rsqrtf(r2);
  rinv = inc ? rinv : 0.f;
  const float rinv2 = rinv * rinv;
  const float rinv6 = rinv2 * rinv2 * rinv2;
  const float qq = xi.w * xjw;
  const float flj = rinv6 * fmaf(lj.y, rinv6, -lj.x);  // 12 c12/r^12 - 6 c6/r^6
  const float qr = qq * rinv;
  float fscal;
  if (ELEC == FE_RF) {
    fscal = (flj + qr) * rinv2;
    if (KRF || ENERGY) {
      const float qm = inc ? qq : 0.f;
      if (KRF) fscal = fmaf(-qm, A.k2rf, fscal);
      if (ENERGY) ec = fmaf(qm, fmaf(A.krf, r2, -A.crf), qr);
    }
  } else {
    const float qm = inc ? qq : 0.f;
    const float u = fmaf(r2, A.ew_a, -1.f);
    float gf = A.ew_f[0];
#pragma unroll
    for (int k = 1; k <= EW_DEG_F; ++k) gf = fmaf(gf, u, A.ew_f[k]);
    const float t = fmaf(-A.beta3, gf, rinv * rinv2);
    fscal = fmaf(qm, t, flj * rinv2);
    if (ENERGY) {
      float gv = A.ew_v[0];
#pragma unroll
      for (int k = 1; k <= EW_DEG_V; ++k) gv = fmaf(gv, u, A.ew_v[k]);
      ec = qm * (rinv - fmaf(A.beta, gv, A.ew_shift));
    }
  }
  if (ENERGY) elj = inc ? fmaf(rinv6, fmaf(lj.y * (1.f / 12.f), rinv6, -lj.x * (1.f / 6.f)), -lj.z) : 0.f;
  return fscal;
}

template <bool MI>
__device__ __forceinline__ float pair_geom(const ForceArgs& A, const float4& xi, const float4& xj, float& dx,
                                           float& dy, float& dz) {
  dx = xi.x - xj.x;
  dy = xi.y - xj.y;
  dz = xi.z - xj.z;
  if (MI) {
    dx = fmaf(-A.L[0], rintf(dx * A.invL[0]), dx);
    dy = fmaf(-A.L[1], rintf(dy * A.invL[1]), dy);
    dz = fmaf(-A.L[2], rintf(dz * A.invL[2]), dz);
  }
  return fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}

// Lane-view of one entry: its j-cluster, the lane's j-atom (shifted into the
// group frame), and the entry masks pre-shifted by the lane's j-slot b and
// split into 32-bit words (bit k*m*m + a*m tests pair (member k, atom a)).
template <int W>
struct Entry {
  int32_t cj;
  float4 d;          // xyz: j-local -> group-local offset, w: slack
  uint32_t w[2 * W];
};

// Entry / j-atom staging through shared memory with cp.async: each lane
// copies its own entry fields (2 iterations ahead) and its j-atom (1 ahead)
// into per-lane ring slots, so no register ever waits on an in-flight global
// load (a register-rotation prefetch stalls on the rotation moves).
// Out-of-range slots copy the group's last entry (a valid address) and are
// disabled when used.
template <int W>
struct Stage {
  float4 ed[3][32];
  uint64_t em[3][W][32];
  int32_t cj[3][32];
  float4 xj[2][32];
  int32_t tj[2][32];
};

__device__ __forceinline__ void cp_async(void* smem, const void* gmem, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  if (bytes == 16) asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
  else if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int W>
__device__ __forceinline__ void stage_entry(const ForceArgs& A, Stage<W>& S, int slot, int lane, int32_t e,
                                            int32_t e_last) {
  const int32_t i = e < e_last ? e : e_last;
  cp_async(&S.ed[slot][lane], A.ent_delta + i, 16);
#pragma unroll
  for (int q = 0; q < W; ++q) cp_async(&S.em[slot][q][lane], A.ent_mask + (int64_t)i * W + q, 8);
  cp_async(&S.cj[slot][lane], A.ent_j + i, 4);
}

template <int M, int W>
__device__ __forceinline__ void stage_jatom(const ForceArgs& A, Stage<W>& S, int xslot, int lane, int32_t cj,
                                            int b) {
  cp_async(&S.xj[xslot][lane], A.xyzq + (int64_t)cj * M + b, 16);
  cp_async(&S.tj[xslot][lane], A.type + (int64_t)cj * M + b, 4);
}

template <int W>
__device__ __forceinline__ void read_entry(const Stage<W>& S, int slot, int lane, bool valid, int b, Entry<W>& E) {
  E.cj = S.cj[slot][lane];
  E.d = S.ed[slot][lane];
  if (!valid) E.d.w = 3.0e38f;
#pragma unroll
  for (int q = 0; q < W; ++q) {
    const uint64_t mw = valid ? (S.em[slot][q][lane] >> b) : 0ull;
    E.w[2 * q] = (uint32_t)mw;
    E.w[2 * q + 1] = (uint32_t)(mw >> 32);
  }
}

template <int M, int W>
__device__ __forceinline__ bool entry_bit(const Entry<W>& E, int p) {
  return (E.w[p >> 5] & (1u << (p & 31))) != 0u;  // one LOP3 with an immediate
}

// One iteration: this lane's entry against the group's i-atoms.  MI =
// per-pair minimum image (entries whose slack cannot guarantee one image).
template <int M, int G, int ELEC, bool KRF, bool ENERGY, bool BAND, bool MI, int W>
__device__ __forceinline__ void sweep(const ForceArgs& A, const float4* __restrict__ s_xi,
                                      const float4* __restrict__ s_ljt, const Entry<W>& E, unsigned wpres,
                                      const float4& xj, float (&fi)[G * M][3], float& fjx, float& fjy,
                                      float& fjz, float& elj, float& ec, uint32_t& near) {
  constexpr int MM = M * M;
#pragma unroll
  for (int k = 0; k < G; ++k) {
    if (!((wpres >> k) & 1u)) continue;
#pragma unroll
    for (int a = 0; a < M; ++a) {
      const int ia = k * M + a;
      const float4 xi = s_xi[ia];
      const float4 lj = s_ljt[ia];
      float dx, dy, dz;
      const float r2 = pair_geom<MI>(A, xi, xj, dx, dy, dz);
      const bool adm = entry_bit<M, W>(E, k * MM + a * M);
      const bool inc = adm && (r2 <= A.rc2);
      if (BAND) near |= (adm && fabsf(r2 - A.rc2) < A.band) ? (1u << ia) : 0u;
      float pe_lj = 0.f, pe_c = 0.f;
      const float fscal = pair_eval<ELEC, KRF, ENERGY>(A, xi, lj, xj.w, r2, inc, pe_lj, pe_c);
      if (ENERGY) {
        elj += pe_lj;
        ec += pe_c;
      }
      fi[ia][0] = fmaf(fscal, dx, fi[ia][0]);
      fi[ia][1] = fmaf(fscal, dy, fi[ia][1]);
      fi[ia][2] = fmaf(fscal, dz, fi[ia][2]);
      fjx = fmaf(-fscal, dx, fjx);
      fjy = fmaf(-fscal, dy, fjy);
      fjz = fmaf(-fscal, dz, fjz);
    }
  }
}

// The same iteration on PAIRS of i-atoms (2h, 2h+1) with Blackwell's packed
// FP32 instructions (FFMA2 / FMUL2 / FADD2: two lanes' worth of FP32 work per
// issue slot, j-atom operands broadcast from one register).  The FP32 pipe
// work is unchanged but the issue slots it needs halve, which is what bounds
// the scalar sweep (ncu: issue ~73 % busy, FMA pipe ~50 %).  i-atom data are
// pair-interleaved in shared memory: s_xy[h] = {x0, x1, y0, y1},
// s_zq[h] = {z0, z1, q0, q1}, s_l2[h] = {-6c6_0, -6c6_1, 12c12_0, 12c12_1}
// (for this lane's j-type), s_sh[h] = {shift_0, shift_1}.
__device__ __forceinline__ float2 bc2(float v) { return make_float2(v, v); }

template <int M, int G, int ELEC, bool KRF, bool ENERGY, bool BAND, bool MI, int W>
__device__ __forceinline__ void sweep2(const ForceArgs& A, const float4* __restrict__ s_xy,
                                       const float4* __restrict__ s_zq, const float4* __restrict__ s_l2,
                                       const float2* __restrict__ s_sh, const Entry<W>& E, unsigned wpres,
                                       const float4& xj, float2 (&fi)[G * M / 2][3], float2& fjx, float2& fjy,
                                       float2& fjz, float2& elj, float2& ec, uint32_t& near) {
  constexpr int IA = G * M, H = IA / 2, MM = M * M;
  const float2 nx = bc2(-xj.x), ny = bc2(-xj.y), nz = bc2(-xj.z), qj = bc2(xj.w);
  // one warp-uniform branch per member (per pair of members when m = 1), so
  // the member's pair-pairs share a basic block and their dependency chains
  // interleave
  constexpr int HB = M >= 2 ? M / 2 : 1;  // pair-pairs per branch
#pragma unroll
  for (int hb = 0; hb < H; hb += HB) {
    const int kb0 = (2 * hb) / M, kb1 = (2 * hb + 2 * HB - 1) / M;
    if (!(((wpres >> kb0) | (wpres >> kb1)) & 1u)) continue;
#pragma unroll
  for (int h = hb; h < hb + HB; ++h) {
    const int ia0 = 2 * h, ia1 = 2 * h + 1;
    const int k0 = ia0 / M, k1 = ia1 / M;
    const float4 xy = s_xy[h], zq = s_zq[h], l2 = s_l2[h];
    float2 dx = __fadd2_rn(make_float2(xy.x, xy.y), nx);
    float2 dy = __fadd2_rn(make_float2(xy.z, xy.w), ny);
    float2 dz = __fadd2_rn(make_float2(zq.x, zq.y), nz);
    if (MI) {
      dx.x = fmaf(-A.L[0], rintf(dx.x * A.invL[0]), dx.x);
      dx.y = fmaf(-A.L[0], rintf(dx.y * A.invL[0]), dx.y);
      dy.x = fmaf(-A.L[1], rintf(dy.x * A.invL[1]), dy.x);
      dy.y = fmaf(-A.L[1], rintf(dy.y * A.invL[1]), dy.y);
      dz.x = fmaf(-A.L[2], rintf(dz.x * A.invL[2]), dz.x);
      dz.y = fmaf(-A.L[2], rintf(dz.y * A.invL[2]), dz.y);
    }
    const float2 r2 = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __fmul2_rn(dz, dz)));
    const int p0 = (W == 2 ? k0 * 64 : k0 * MM) + (ia0 % M) * M;
    const int p1 = (W == 2 ? k1 * 64 : k1 * MM) + (ia1 % M) * M;
    const bool adm0 = entry_bit<M, W>(E, p0), adm1 = entry_bit<M, W>(E, p1);
    const bool inc0 = adm0 && (r2.x <= A.rc2), inc1 = adm1 && (r2.y <= A.rc2);
    if (BAND) {
      near |= (adm0 && fabsf(r2.x - A.rc2) < A.band) ? (1u << ia0) : 0u;
      near |= (adm1 && fabsf(r2.y - A.rc2) < A.band) ? (1u << ia1) : 0u;
    }
    float2 rinv = make_float2(rsqrtf(r2.x), rsqrtf(r2.y));
    rinv.x = inc0 ? rinv.x : 0.f;
    rinv.y = inc1 ? rinv.y : 0.f;
    const float2 rinv2 = __fmul2_rn(rinv, rinv);
    const float2 rinv6 = __fmul2_rn(__fmul2_rn(rinv2, rinv2), rinv2);
    const float2 c6n = make_float2(l2.x, l2.y), c12 = make_float2(l2.z, l2.w);
    const float2 flj = __fmul2_rn(rinv6, __ffma2_rn(c12, rinv6, c6n));  // 12 c12/r^12 - 6 c6/r^6
    const float2 qq = __fmul2_rn(make_float2(zq.z, zq.w), qj);
    float2 fscal;
    if (ELEC == FE_RF) {
      fscal = __fmul2_rn(__ffma2_rn(qq, rinv, flj), rinv2);
      if (KRF || ENERGY) {
        const float2 qm = make_float2(inc0 ? qq.x : 0.f, inc1 ? qq.y : 0.f);
        if (KRF) fscal = __ffma2_rn(qm, bc2(-A.k2rf), fscal);
        if (ENERGY)
          ec = __fadd2_rn(ec, __ffma2_rn(qm, __ffma2_rn(bc2(A.krf), r2, bc2(-A.crf)), __fmul2_rn(qq, rinv)));
      }
    } else {
      const float2 qm = make_float2(inc0 ? qq.x : 0.f, inc1 ? qq.y : 0.f);
      const float2 u = __ffma2_rn(r2, bc2(A.ew_a), bc2(-1.f));
      float2 gf = bc2(A.ew_f[0]);
#pragma unroll
      for (int k = 1; k <= EW_DEG_F; ++k) gf = __ffma2_rn(gf, u, bc2(A.ew_f[k]));
      const float2 t = __ffma2_rn(bc2(-A.beta3), gf, __fmul2_rn(rinv, rinv2));
      fscal = __ffma2_rn(qm, t, __fmul2_rn(flj, rinv2));
      if (ENERGY) {
        float2 gv = bc2(A.ew_v[0]);
#pragma unroll
        for (int k = 1; k <= EW_DEG_V; ++k) gv = __ffma2_rn(gv, u, bc2(A.ew_v[k]));
        ec = __ffma2_rn(qm, __fadd2_rn(rinv, __ffma2_rn(bc2(-A.beta), gv, bc2(-A.ew_shift))), ec);
      }
    }
    if (ENERGY) {
      const float2 sh = s_sh[h];
      const float2 shm = make_float2(inc0 ? -sh.x : 0.f, inc1 ? -sh.y : 0.f);
      const float2 e6 = __fmul2_rn(rinv6, __ffma2_rn(__fmul2_rn(c12, bc2(1.f / 12.f)), rinv6,
                                                     __fmul2_rn(c6n, bc2(1.f / 6.f))));
      elj = __fadd2_rn(elj, __fadd2_rn(e6, shm));
    }
    fi[h][0] = __ffma2_rn(fscal, dx, fi[h][0]);
    fi[h][1] = __ffma2_rn(fscal, dy, fi[h][1]);
    fi[h][2] = __ffma2_rn(fscal, dz, fi[h][2]);
    fjx = __ffma2_rn(fscal, dx, fjx);  // j-side sign applied once per iteration
    fjy = __ffma2_rn(fscal, dy, fjy);
    fjz = __ffma2_rn(fscal, dz, fjz);
  }
  }
}

// Rare path: pairs whose FP32 r^2 fell within `band` of r_c^2 get the exact
// FP64 reference decision; when it differs the pair's contribution is added
// or removed (i-side through shared-memory atomics).
template <int M, int G, int ELEC, bool KRF, bool ENERGY, bool MI>
__device__ __forceinline__ void band_fix(const ForceArgs& A, const float4* __restrict__ s_xi,
                                      const float4* __restrict__ s_ljt, float* s_corr, uint32_t near,
                                      const float4& xj, int32_t first, int32_t cj, int b, float& fjx,
                                      float& fjy, float& fjz, float& elj, float& ec) {
  while (near) {
    const int ia = __ffs(near) - 1;
    near &= near - 1;
    const float4 xi = s_xi[ia];
    float dx, dy, dz;
    const float r2 = pair_geom<MI>(A, xi, xj, dx, dy, dz);
    const bool inc32 = r2 <= A.rc2;
    const int ex = exact_inside(A, (int64_t)first * M + ia, (int64_t)cj * M + b);
    if (ex < 0) record_bad(A.scalars, (int64_t)first * M + ia, (int64_t)cj * M + b);
    const bool inc64 = ex > 0;
    if (inc64 == inc32) continue;
    float pe_lj = 0.f, pe_c = 0.f;
    const float fscal = pair_eval<ELEC, KRF, ENERGY>(A, xi, s_ljt[ia], xj.w, r2, true, pe_lj, pe_c);
    const float sg = inc64 ? 1.f : -1.f;
    atomicAdd(&s_corr[3 * ia + 0], sg * fscal * dx);
    atomicAdd(&s_corr[3 * ia + 1], sg * fscal * dy);
    atomicAdd(&s_corr[3 * ia + 2], sg * fscal * dz);
    fjx -= sg * fscal * dx;
    fjy -= sg * fscal * dy;
    fjz -= sg * fscal * dz;
    if (ENERGY) {
      elj += sg * pe_lj;
      ec += sg * pe_c;
    }
  }
}

#ifndef NBX_FORCE_MINB
#define NBX_FORCE_MINB 4
#endif
template <int M, int G, int ELEC, bool KRF, bool ENERGY, bool BAND>
__global__ void __launch_bounds__(FW * 32, NBX_FORCE_MINB)
k_force(const ForceArgs A) {
  constexpr int R = 32 / M;   // entries per iteration
  constexpr int IA = G * M;   // i-atoms per group
  constexpr int W = (G * M * M > 64) ? 2 : 1;
  constexpr int MM = M * M;
  constexpr bool PK = (IA % 2) == 0;  // packed FP32x2 sweep over i-atom pairs
  constexpr int H = PK ? IA / 2 : 1;
  // dynamic: [FW][nt][IA] float4 LJ per (j-type, i-atom) (scalar sweep and
  // band fixes), then [FW][nt][H] float4 pair-interleaved LJ, [FW][nt][H]
  // float2 pair-interleaved shifts
  extern __shared__ float4 s_dyn[];
  __shared__ float4 s_xi[FW][IA];
  __shared__ float4 s_xy[FW][H];
  __shared__ float4 s_zq[FW][H];
  // per-warp scratch: the staging ring during the entry loop, the i-force
  // transpose buffer after it
  union Scratch {
    Stage<W> st;
    float red[32][IA * 3 + 1];
  };
  __shared__ Scratch s_ws[FW];
  __shared__ float s_corr[FW][IA * 3];

  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane / M, b = lane % M;
  // persistent warps: groups are handed out dynamically (largest first via
  // A.sel), which removes the wave tail and the group-size imbalance
  for (;;) {
  int64_t wi = 0;
  if (lane == 0) wi = (int64_t)atomicAdd(A.scalars + 4, 1u);
  wi = __shfl_sync(0xffffffffu, wi, 0);
  if (wi >= A.n_work) break;
  const int32_t g = A.sel ? A.sel[wi] : (int32_t)wi;
  const int32_t first = A.grp_first ? A.grp_first[g] : g;
  const int nmem = A.grp_nmem ? A.grp_nmem[g] : 1;
  const int32_t e_beg = A.ent_off[g], e_end = A.ent_off[g + 1];
  float4* s_lj = s_dyn + (size_t)w * IA * A.nt;
  float4* s_l2 = s_dyn + (size_t)FW * IA * A.nt + (size_t)w * H * A.nt;
  float2* s_sh = reinterpret_cast<float2*>(s_dyn + (size_t)FW * (IA + H) * A.nt) + (size_t)w * H * A.nt;

  // software pipeline (cp.async into per-lane smem slots): entry data two
  // iterations ahead, j-atom one ahead
  const int32_t e_last = e_end > e_beg ? e_end - 1 : e_beg;
  Stage<W>& S = s_ws[w].st;
  if (e_end > e_beg) {
    stage_entry<W>(A, S, 0, lane, e_beg + r, e_last);
    stage_entry<W>(A, S, 1, lane, e_beg + R + r, e_last);
    cp_async_commit();
    cp_async_wait_all();
    stage_jatom<M, W>(A, S, 0, lane, S.cj[0][lane], b);
    cp_async_commit();
  }

  // stage the group's i-atoms (group frame) and their LJ parameters per j-type
  for (int ia = lane; ia < IA; ia += 32) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ia < nmem * M) {
      v = A.xyzq[(int64_t)first * M + ia];
      const int64_t c = first + ia / M;
      v.x = (float)((A.bbox[6 * c + 0] - A.bbox[6 * (int64_t)first + 0]) + (double)v.x);
      v.y = (float)((A.bbox[6 * c + 1] - A.bbox[6 * (int64_t)first + 1]) + (double)v.y);
      v.z = (float)((A.bbox[6 * c + 2] - A.bbox[6 * (int64_t)first + 2]) + (double)v.z);
      v.w *= A.coul;
    }
    s_xi[w][ia] = v;
    if (PK) {
      float* xyf = reinterpret_cast<float*>(&s_xy[w][0]);
      float* zqf = reinterpret_cast<float*>(&s_zq[w][0]);
      const int h = ia >> 1, o = ia & 1;
      xyf[4 * h + o] = v.x;
      xyf[4 * h + 2 + o] = v.y;
      zqf[4 * h + o] = v.z;
      zqf[4 * h + 2 + o] = v.w;
    }
  }
  if (!PK || BAND)
    for (int idx = lane; idx < IA * A.nt; idx += 32) {
      const int t = idx / IA, ia = idx - t * IA;
      const int ti = ia < nmem * M ? A.type[(int64_t)first * M + ia] : 0;
      s_lj[idx] = __ldg(&A.lj[ti * A.nt + t]);
    }
  if (PK)
    for (int idx = lane; idx < H * A.nt; idx += 32) {
      const int t = idx / H, h = idx - t * H;
      const int ti0 = 2 * h < nmem * M ? A.type[(int64_t)first * M + 2 * h] : 0;
      const int ti1 = 2 * h + 1 < nmem * M ? A.type[(int64_t)first * M + 2 * h + 1] : 0;
      const float4 a0 = __ldg(&A.lj[ti0 * A.nt + t]), a1 = __ldg(&A.lj[ti1 * A.nt + t]);
      s_l2[idx] = make_float4(-a0.x, -a1.x, a0.y, a1.y);
      s_sh[idx] = make_float2(a0.z, a1.z);
    }
  if (BAND)
    for (int c = lane; c < IA * 3; c += 32) s_corr[w][c] = 0.f;
  __syncwarp();

  const float slack_thr = A.slack_base + 4.f * __uint_as_float(A.scalars[0]);
  float fi[PK ? 1 : IA][3];
  float2 fi2[H][3];
  if constexpr (PK) {
#pragma unroll
    for (int h = 0; h < H; ++h) fi2[h][0] = fi2[h][1] = fi2[h][2] = make_float2(0.f, 0.f);
  } else {
#pragma unroll
    for (int ia = 0; ia < IA; ++ia) fi[ia][0] = fi[ia][1] = fi[ia][2] = 0.f;
  }
  double elj_acc = 0.0, ec_acc = 0.0;
  constexpr uint64_t colmask = column_bits<M>();

  int es = 0, xs = 0;
  for (int32_t e0 = e_beg; e0 < e_end; e0 += R) {
    const int32_t e = e0 + r;
    const bool valid = e < e_end;
    // this iteration's entry (slot es) and j-atom (slot xs) have landed;
    // stage the j-atom of the next iteration and the entry two ahead
    cp_async_wait_all();
    Entry<W> cur;
    read_entry<W>(S, es, lane, valid, b, cur);
    const float4 xr = S.xj[xs][lane];
    const int tj = S.tj[xs][lane];
    {
      const int es1 = es == 2 ? 0 : es + 1, es2 = es1 == 2 ? 0 : es1 + 1;
      stage_jatom<M, W>(A, S, xs ^ 1, lane, S.cj[es1][lane], b);
      stage_entry<W>(A, S, es2, lane, e + 2 * R, e_last);
      cp_async_commit();
      es = es1;
      xs ^= 1;
    }
    const float4 xj = make_float4(xr.x + cur.d.x, xr.y + cur.d.y, xr.z + cur.d.z, xr.w);

    unsigned pres = 0;
#pragma unroll
    for (int k = 0; k < G; ++k) {
      uint64_t word;
      if constexpr (W == 2) word = ((uint64_t)cur.w[2 * k + 1] << 32) | cur.w[2 * k];
      else word = (((uint64_t)cur.w[1] << 32) | cur.w[0]) >> (k * MM);
      pres |= ((word & colmask) != 0ull) ? (1u << k) : 0u;
    }
    const unsigned wpres = __reduce_or_sync(0xffffffffu, pres);
    const bool wunsafe = __any_sync(0xffffffffu, valid && cur.d.w < slack_thr);
    const float4* s_ljt = s_lj + tj * IA;
    float fjx = 0.f, fjy = 0.f, fjz = 0.f;
    float elj = 0.f, ec = 0.f;
    uint32_t near = 0;
    if constexpr (PK) {
      const float4* s_l2t = s_l2 + tj * H;
      const float2* s_sht = s_sh + tj * H;
      float2 gx = make_float2(0.f, 0.f), gy = gx, gz = gx, el2 = gx, ec2 = gx;
      if (!wunsafe)
        sweep2<M, G, ELEC, KRF, ENERGY, BAND, false, W>(A, s_xy[w], s_zq[w], s_l2t, s_sht, cur, wpres, xj, fi2, gx,
                                                        gy, gz, el2, ec2, near);
      else
        sweep2<M, G, ELEC, KRF, ENERGY, BAND, true, W>(A, s_xy[w], s_zq[w], s_l2t, s_sht, cur, wpres, xj, fi2, gx,
                                                       gy, gz, el2, ec2, near);
      fjx = -(gx.x + gx.y);
      fjy = -(gy.x + gy.y);
      fjz = -(gz.x + gz.y);
      if (ENERGY) {
        elj = el2.x + el2.y;
        ec = ec2.x + ec2.y;
      }
    } else {
      if (!wunsafe)
        sweep<M, G, ELEC, KRF, ENERGY, BAND, false, W>(A, s_xi[w], s_ljt, cur, wpres, xj, fi, fjx, fjy, fjz, elj, ec, near);
      else
        sweep<M, G, ELEC, KRF, ENERGY, BAND, true, W>(A, s_xi[w], s_ljt, cur, wpres, xj, fi, fjx, fjy, fjz, elj, ec, near);
    }
    if (BAND && __any_sync(0xffffffffu, near != 0)) {
      if (near) {
        if (!wunsafe)
          band_fix<M, G, ELEC, KRF, ENERGY, false>(A, s_xi[w], s_ljt, s_corr[w], near, xj, first, cur.cj, b, fjx, fjy, fjz, elj, ec);
        else
          band_fix<M, G, ELEC, KRF, ENERGY, true>(A, s_xi[w], s_ljt, s_corr[w], near, xj, first, cur.cj, b, fjx, fjy, fjz, elj, ec);
      }
      __syncwarp();
    }
    if (valid) A.part_j[(int64_t)e * M + b] = make_float4(fjx, fjy, fjz, 0.f);
    if (ENERGY) {
      elj_acc += (double)elj;
      ec_acc += (double)ec;
    }
  }

  cp_async_wait_all();  // nothing in flight into the slots the next group reuses
  __syncwarp();         // ... and every lane's copies landed before the scratch is reused

  // i-force transpose-reduce through shared memory
  if constexpr (PK) {
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        s_ws[w].red[lane][3 * (2 * h) + c] = fi2[h][c].x;
        s_ws[w].red[lane][3 * (2 * h + 1) + c] = fi2[h][c].y;
      }
  } else {
#pragma unroll
    for (int ia = 0; ia < IA; ++ia) {
      s_ws[w].red[lane][3 * ia + 0] = fi[ia][0];
      s_ws[w].red[lane][3 * ia + 1] = fi[ia][1];
      s_ws[w].red[lane][3 * ia + 2] = fi[ia][2];
    }
  }
  __syncwarp();
  for (int c = lane; c < IA * 3; c += 32) {
    float sacc = BAND ? s_corr[w][c] : 0.f;
#pragma unroll 8
    for (int l = 0; l < 32; ++l) sacc += s_ws[w].red[l][c];
    s_ws[w].red[0][c] = sacc;  // column c is read and written by this lane only
  }
  __syncwarp();
  if (lane < nmem * M) {
    A.part_i[(int64_t)first * M + lane] =
        make_float4(s_ws[w].red[0][3 * lane], s_ws[w].red[0][3 * lane + 1], s_ws[w].red[0][3 * lane + 2], 0.f);
  }
  if (ENERGY) {
    for (int o = 16; o; o >>= 1) {
      elj_acc += __shfl_xor_sync(0xffffffffu, elj_acc, o);
      ec_acc += __shfl_xor_sync(0xffffffffu, ec_acc, o);
    }
    if (lane == 0) {
      A.e_grp[2 * wi] = elj_acc;
      A.e_grp[2 * wi + 1] = ec_acc;
    }
  }
  __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// k_force_h: the grouped kernel with TWO j-atoms per lane (m = 4, 8).
//
// Lane (ih, r, jp) = (half, entry slot r of R = 32/m, j-atom pair jp of m/2)
// holds two j-atoms of entry r in registers and sweeps i-atom PAIRS from
// shared memory: half ih owns pairs pp < m/4 starting at atom 2 ih (m/4) of
// EVERY member, so the warp-uniform member branches skip exactly what
// k_force skips.  Against k_force (one j-atom per lane over all 16 i-atoms)
// every i-atom pair loaded from shared memory serves two j-atoms, the i-force
// accumulators halve, and the entry fields are staged once per entry rather
// than once per lane.  The lane's "a" j-atom is 2jp + ih and its "b" j-atom
// 2jp + 1 - ih, so after one shuffle per component (the partner half's
// partial of a) each lane owns the full force on its a-atom: one store per
// (entry, j-atom), k_reduce unchanged.
//
// Sign convention: d = x_j - x_i (i-atoms are staged negated), so the j-force
// fscal d accumulates with no negation and the i-accumulators hold -F_i,
// negated once per group.  Masked or out-of-range pairs get r^2 = +inf
// before the rsqrt (rinv = 0, hence every force term 0).  Ewald force term:
//   F/r = rinv2 (flj + qq (rinv + r2 Gs(u))),  Gs = -beta^3 Gf.
// Per-warp staging, one CHUNK of CH = 128/m entries at a time: entry fields
// in a 3-slot ring (staged two chunks ahead), j-atoms in a 2-slot ring (one
// chunk ahead), stored [q][entry][m/2] so that a lane's a/b atoms of one
// iteration are read conflict-free.
template <int M, int W>
struct StageH {
  static constexpr int CH = 128 / M;
  float4 ed[3][CH];
  uint64_t em[3][CH][W];
  int32_t cj[3][CH];
  int32_t tp[3][CH];
  float4 xj[2][128];
  int32_t tj[2][128];
};

// admit = mask bit set and r2 <= rc2; returns r2 or +inf (rinv = 0)
__device__ __forceinline__ float admit_r2(float r2, float rc2, uint64_t mw, int p) {
  float out;
  const uint32_t word = p < 32 ? (uint32_t)mw : (uint32_t)(mw >> 32);
  const uint32_t bit = 1u << (p & 31);
  asm("{\n\t.reg .pred pm, pc;\n\t"
      "setp.ne.b32 pm, %3, 0;\n\t"
      "setp.le.and.ftz.f32 pc, %1, %2, pm;\n\t"
      "selp.f32 %0, %1, 0f7F800000, pc;\n\t}"
      : "=f"(out)
      : "f"(r2), "f"(rc2), "r"(word & bit));
  return out;
}

template <bool MI>
__device__ __forceinline__ float2 geom2(const ForceArgs& A, const float4& xy, const float4& zq, const float4& xj,
                                        float2& dx, float2& dy, float2& dz) {
  dx = __fadd2_rn(make_float2(xy.x, xy.y), bc2(xj.x));
  dy = __fadd2_rn(make_float2(xy.z, xy.w), bc2(xj.y));
  dz = __fadd2_rn(make_float2(zq.x, zq.y), bc2(xj.z));
  if (MI) {
    dx.x = fmaf(-A.L[0], rintf(dx.x * A.invL[0]), dx.x);
    dx.y = fmaf(-A.L[0], rintf(dx.y * A.invL[0]), dx.y);
    dy.x = fmaf(-A.L[1], rintf(dy.x * A.invL[1]), dy.x);
    dy.y = fmaf(-A.L[1], rintf(dy.y * A.invL[1]), dy.y);
    dz.x = fmaf(-A.L[2], rintf(dz.x * A.invL[2]), dz.x);
    dz.y = fmaf(-A.L[2], rintf(dz.y * A.invL[2]), dz.y);
  }
  return __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __fmul2_rn(dz, dz)));
}

// F/r (and energies) of one i-atom pair against one j-atom; inc0/inc1 are
// the admitted-and-within-r_c decisions.
template <int ELEC, bool KRF, bool ENERGY>
__device__ __forceinline__ float2 pair2_eval(const ForceArgs& A, const float4& zq, const float4& l2, float qj,
                                             float2 r2, float2 r2m, const float2& sh, float2& elj, float2& ec) {
  // r2m = r2 where admitted and within r_c, +inf elsewhere
  const float inf = __int_as_float(0x7f800000);
  const bool inc0 = r2m.x != inf, inc1 = r2m.y != inf;
  float2 rinv = make_float2(rsqrtf(r2m.x), rsqrtf(r2m.y));
  const float2 rinv2 = __fmul2_rn(rinv, rinv);
  const float2 rinv6 = __fmul2_rn(__fmul2_rn(rinv2, rinv2), rinv2);
  const float2 c6n = make_float2(l2.x, l2.y), c12 = make_float2(l2.z, l2.w);
  const float2 flj = __fmul2_rn(rinv6, __ffma2_rn(c12, rinv6, c6n));  // 12 c12/r^12 - 6 c6/r^6
  const float2 qq = __fmul2_rn(make_float2(zq.z, zq.w), bc2(qj));
  float2 fscal;
  if (ELEC == FE_RF) {
    fscal = __fmul2_rn(__ffma2_rn(qq, rinv, flj), rinv2);
    if (KRF || ENERGY) {
      const float2 qm = make_float2(inc0 ? qq.x : 0.f, inc1 ? qq.y : 0.f);
      if (KRF) fscal = __ffma2_rn(qm, bc2(-A.k2rf), fscal);
      if (ENERGY)
        ec = __fadd2_rn(ec, __ffma2_rn(qm, __ffma2_rn(bc2(A.krf), r2, bc2(-A.crf)), __fmul2_rn(qq, rinv)));
    }
  } else {
    const float2 u = __ffma2_rn(r2, bc2(A.ew_a), bc2(-1.f));
    float2 gs;
#if NBX_EW_ESTRIN
    static_assert(EW_DEG_F == 10, "Estrin scheme written for degree 10");
    {  // depth 4 instead of 10 (a_i = ew_s[10 - i])
      const float* c = A.ew_s;
      const float2 u2 = __fmul2_rn(u, u), u4 = __fmul2_rn(u2, u2), u8 = __fmul2_rn(u4, u4);
      const float2 b0 = __ffma2_rn(bc2(c[9]), u, bc2(c[10])), b1 = __ffma2_rn(bc2(c[7]), u, bc2(c[8]));
      const float2 b2 = __ffma2_rn(bc2(c[5]), u, bc2(c[6])), b3 = __ffma2_rn(bc2(c[3]), u, bc2(c[4]));
      const float2 b4 = __ffma2_rn(bc2(c[1]), u, bc2(c[2]));
      const float2 c0 = __ffma2_rn(b1, u2, b0), c1 = __ffma2_rn(b3, u2, b2), c2 = __ffma2_rn(bc2(c[0]), u2, b4);
      gs = __ffma2_rn(c2, u8, __ffma2_rn(c1, u4, c0));
    }
#else
    gs = bc2(A.ew_s[0]);
#pragma unroll
    for (int k = 1; k <= EW_DEG_F; ++k) gs = __ffma2_rn(gs, u, bc2(A.ew_s[k]));
#endif
    const float2 sc = __ffma2_rn(r2, gs, rinv);
    fscal = __fmul2_rn(__ffma2_rn(qq, sc, flj), rinv2);
    if (ENERGY) {
      const float2 qm = make_float2(inc0 ? qq.x : 0.f, inc1 ? qq.y : 0.f);
      float2 gv = bc2(A.ew_v[0]);
#pragma unroll
      for (int k = 1; k <= EW_DEG_V; ++k) gv = __ffma2_rn(gv, u, bc2(A.ew_v[k]));
      ec = __ffma2_rn(qm, __fadd2_rn(rinv, __ffma2_rn(bc2(-A.beta), gv, bc2(-A.ew_shift))), ec);
    }
  }
  if (ENERGY) {
    const float2 shm = make_float2(inc0 ? -sh.x : 0.f, inc1 ? -sh.y : 0.f);
    const float2 e6 =
        __fmul2_rn(rinv6, __ffma2_rn(__fmul2_rn(c12, bc2(1.f / 12.f)), rinv6, __fmul2_rn(c6n, bc2(1.f / 6.f))));
    elj = __fadd2_rn(elj, __fadd2_rn(e6, shm));
  }
  return fscal;
}

// Bits of the lane mask words: member k at k*MB, atom s of the lane's pair
// pp at (2 pp + s) * M (one j-atom per word: ma for a, mb for b).
template <int M>
__host__ __device__ constexpr int member_stride_bits() { return M == 4 ? 16 : 32; }

template <int M, int ELEC, bool KRF, bool ENERGY, bool BAND, bool MI>
__device__ __forceinline__ void sweep_h(const ForceArgs& A, const float4* __restrict__ s_xy,
                                        const float4* __restrict__ s_zq, const float4* __restrict__ s_l2a,
                                        const float4* __restrict__ s_l2b, const float2* __restrict__ s_sha,
                                        const float2* __restrict__ s_shb, uint64_t ma, uint64_t mb, unsigned wpres,
                                        int ih, const float4& xa, const float4& xb, float2 (&fi)[4][3],
                                        float2 (&fa)[3], float2 (&fb)[3], float2& elj, float2& ec, uint32_t& near) {
  constexpr int G = 16 / M, PP = M / 4, MB = member_stride_bits<M>();
#pragma unroll
  for (int k = 0; k < G; ++k) {
    if (!((wpres >> k) & 1u)) continue;
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      const int hl = k * PP + pp;
      const int h = k * (M / 2) + ih * PP + pp;
      const int p0 = k * MB + (2 * pp) * M, p1 = p0 + M;
      const float4 xy = s_xy[h], zq = s_zq[h];
      const float4 la = s_l2a[h], lb = s_l2b[h];
      float2 sha = bc2(0.f), shb = bc2(0.f);
      if (ENERGY) {
        sha = s_sha[h];
        shb = s_shb[h];
      }
      float2 dxa, dya, dza, dxb, dyb, dzb;
      const float2 r2a = geom2<MI>(A, xy, zq, xa, dxa, dya, dza);
      const float2 r2b = geom2<MI>(A, xy, zq, xb, dxb, dyb, dzb);
      const float2 r2ma = make_float2(admit_r2(r2a.x, A.rc2, ma, p0), admit_r2(r2a.y, A.rc2, ma, p1));
      const float2 r2mb = make_float2(admit_r2(r2b.x, A.rc2, mb, p0), admit_r2(r2b.y, A.rc2, mb, p1));
      if (BAND) {
        const bool ma0 = (ma >> p0) & 1ull, ma1 = (ma >> p1) & 1ull;
        const bool mb0 = (mb >> p0) & 1ull, mb1 = (mb >> p1) & 1ull;
        near |= (ma0 && fabsf(r2a.x - A.rc2) < A.band) ? (1u << (4 * hl + 0)) : 0u;
        near |= (ma1 && fabsf(r2a.y - A.rc2) < A.band) ? (1u << (4 * hl + 2)) : 0u;
        near |= (mb0 && fabsf(r2b.x - A.rc2) < A.band) ? (1u << (4 * hl + 1)) : 0u;
        near |= (mb1 && fabsf(r2b.y - A.rc2) < A.band) ? (1u << (4 * hl + 3)) : 0u;
      }
      const float2 fsa = pair2_eval<ELEC, KRF, ENERGY>(A, zq, la, xa.w, r2a, r2ma, sha, elj, ec);
      const float2 fsb = pair2_eval<ELEC, KRF, ENERGY>(A, zq, lb, xb.w, r2b, r2mb, shb, elj, ec);
      fi[hl][0] = __ffma2_rn(fsa, dxa, fi[hl][0]);
      fi[hl][1] = __ffma2_rn(fsa, dya, fi[hl][1]);
      fi[hl][2] = __ffma2_rn(fsa, dza, fi[hl][2]);
      fa[0] = __ffma2_rn(fsa, dxa, fa[0]);
      fa[1] = __ffma2_rn(fsa, dya, fa[1]);
      fa[2] = __ffma2_rn(fsa, dza, fa[2]);
      fi[hl][0] = __ffma2_rn(fsb, dxb, fi[hl][0]);
      fi[hl][1] = __ffma2_rn(fsb, dyb, fi[hl][1]);
      fi[hl][2] = __ffma2_rn(fsb, dzb, fi[hl][2]);
      fb[0] = __ffma2_rn(fsb, dxb, fb[0]);
      fb[1] = __ffma2_rn(fsb, dyb, fb[1]);
      fb[2] = __ffma2_rn(fsb, dzb, fb[2]);
    }
  }
}

// group i-atom of the lane's pair hl (s = 0, 1)
template <int M>
__device__ __forceinline__ int lane_atom(int hl, int s, int ih) {
  constexpr int PP = M / 4;
  const int k = hl / PP, pp = hl - k * PP;
  return 2 * (k * (M / 2) + ih * PP + pp) + s;
}

// Band fixes for the two j-atoms of a lane: near bit 4hl + 2s + q = (atom s
// of the lane's pair hl, j-atom q: 0 = a, 1 = b).  Corrections go to the
// j-force sums fj[q] (+F on j) and, through shared-memory atomics, to the
// i-atoms (+F on i).
template <int M, int ELEC, bool KRF, bool ENERGY, bool MI>
__device__ __forceinline__ void band_fix_h(const ForceArgs& A, const float4* __restrict__ s_xi,
                                           const float4* __restrict__ s_lj, float* s_corr, uint32_t near,
                                           const float4 (&xj)[2], const int (&tj)[2], const int (&bj)[2], int ih,
                                           int32_t first, int32_t cj, float (&fj)[2][3], float& elj, float& ec) {
  while (near) {
    const int bit = __ffs(near) - 1;
    near &= near - 1;
    const int hl = bit >> 2, s = (bit >> 1) & 1, q = bit & 1;
    const int ia = lane_atom<M>(hl, s, ih);
    const int b = bj[q];
    const float4 xi = s_xi[ia];
    float dx, dy, dz;
    const float r2 = pair_geom<MI>(A, xi, xj[q], dx, dy, dz);
    const bool inc32 = r2 <= A.rc2;
    const int ex = exact_inside(A, (int64_t)first * M + ia, (int64_t)cj * M + b);
    if (ex < 0) record_bad(A.scalars, (int64_t)first * M + ia, (int64_t)cj * M + b);
    const bool inc64 = ex > 0;
    if (inc64 == inc32) continue;
    float pe_lj = 0.f, pe_c = 0.f;
    const float fscal = pair_eval<ELEC, KRF, ENERGY>(A, xi, s_lj[tj[q] * 16 + ia], xj[q].w, r2, true, pe_lj, pe_c);
    const float sg = inc64 ? 1.f : -1.f;
    atomicAdd(&s_corr[3 * ia + 0], sg * fscal * dx);
    atomicAdd(&s_corr[3 * ia + 1], sg * fscal * dy);
    atomicAdd(&s_corr[3 * ia + 2], sg * fscal * dz);
    fj[q][0] -= sg * fscal * dx;
    fj[q][1] -= sg * fscal * dy;
    fj[q][2] -= sg * fscal * dz;
    if (ENERGY) {
      elj += sg * pe_lj;
      ec += sg * pe_c;
    }
  }
}

#ifndef NBX_FORCEH_MINB
#define NBX_FORCEH_MINB 4
#endif
constexpr int LJS = 9;  // row stride (float4 / float2) of the per-type LJ tables: no bank conflicts between types

template <int M, int ELEC, bool KRF, bool ENERGY, bool BAND>
__global__ void __launch_bounds__(FW * 32, NBX_FORCEH_MINB)
k_force_h(const ForceArgs A) {
  constexpr int G = 16 / M;
  constexpr int R = 32 / M;   // entries per iteration
  constexpr int IA = 16;      // i-atoms per group
  constexpr int H = 8;        // i-atom pairs per group
  constexpr int JP = M / 2;   // j-atom pairs per entry
  constexpr int W = (G * M * M > 64) ? 2 : 1;
  // dynamic: [FW][nt][LJS] float4 pair-interleaved LJ, [FW][nt][LJS] float2
  // shifts, then (BAND) [FW][nt][IA] float4 scalar LJ
  extern __shared__ float4 s_dyn[];
  __shared__ float4 s_xi[FW][IA];
  __shared__ float4 s_xy[FW][H];
  __shared__ float4 s_zq[FW][H];
  union Scratch {
    StageH<M, W> st;
    float red[32][25];
  };
  constexpr int CH = StageH<M, W>::CH;  // entries per chunk
  constexpr int CJ = CH * JP;           // staged atoms per q plane
  __shared__ Scratch s_ws[FW];
  __shared__ float s_corr[FW][BAND ? IA * 3 : 1];

  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ih = lane >> 4, r = (lane & 15) / JP, jp = (lane & 15) % JP;
  const int ba = 2 * jp + ih, bb = 2 * jp + 1 - ih;  // this lane's a and b j-atoms
  const size_t tn = (size_t)LJS * A.nt;
  float4* s_l2 = s_dyn + (size_t)w * tn;
  float2* s_sh = reinterpret_cast<float2*>(s_dyn + (size_t)FW * tn) + (size_t)w * tn;
  float4* s_lj = s_dyn + (size_t)FW * tn + (FW * tn + 1) / 2 + (size_t)w * IA * A.nt;
  StageH<M, W>& S = s_ws[w].st;
  // dynamic pruning: the inner list while the atoms have not moved far enough
  // (since the build) for a dropped row to reach r_c; else the full masks
  const bool use_inner = A.ent_fmask && __uint_as_float(A.scalars[A.inner_slot]) <= A.inner_dmax;
  const uint64_t* emask = use_inner ? A.ent_fmask : A.ent_mask;

  for (;;) {
    int64_t wi = 0;
    if (lane == 0) wi = (int64_t)atomicAdd(A.scalars + 4, 1u);
    wi = __shfl_sync(0xffffffffu, wi, 0);
    if (wi >= A.n_work) break;
    // work item -> (group in work order, part of its entry range)
    const int64_t wg = A.wbase + wi;
    const int part = (int)(wg % A.split);
    const int64_t gi = wg / A.split;
    const int32_t g = A.sel ? A.sel[gi] : (int32_t)gi;
    const int32_t first = A.grp_first[g];
    const int nmem = A.grp_nmem[g];
    // inner list: entries past ent_fend have no member within r_inner; they
    // are not evaluated and k_reduce skips their (unwritten) partials (split
    // transpose: per j-cluster the entries with an inner member come first)
    const int32_t g_beg = A.ent_off[g];
    const int32_t g_end = use_inner ? A.ent_fend[g] : A.ent_off[g + 1];
    const int32_t g_cnt = g_end - g_beg;
    const int32_t e_beg = g_beg + (int32_t)(((int64_t)g_cnt * part) / A.split);
    const int32_t e_end = g_beg + (int32_t)(((int64_t)g_cnt * (part + 1)) / A.split);
    const int32_t e_last = e_end > e_beg ? e_end - 1 : e_beg;

    // chunk staging: entry fields of chunk c (lanes < CH), j-atoms of chunk
    // c (4 per lane, flat index f = u*32 + lane -> plane q, entry, pair)
    auto stage_entries = [&](int slot, int32_t ec0) {
      if (lane < CH) {
        const int32_t e = min(ec0 + lane, e_last);
        cp_async(&S.ed[slot][lane], A.ent_delta + e, 16);
#pragma unroll
        for (int q = 0; q < W; ++q) cp_async(&S.em[slot][lane][q], emask + (int64_t)e * W + q, 8);
        cp_async(&S.cj[slot][lane], A.ent_j + e, 4);
        cp_async(&S.tp[slot][lane], A.ent_tpos + e, 4);
      }
    };
    auto stage_jatoms = [&](int xslot, int eslot) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int f = u * 32 + lane, q = f / CJ, rem = f - q * CJ;
        const int ent = rem / JP, b = 2 * (rem - ent * JP) + q;
        cp_async(&S.xj[xslot][f], A.xyzq + (int64_t)S.cj[eslot][ent] * M + b, 16);
      }
      const int te = lane / (M / 4), tq = lane % (M / 4);
      cp_async(&S.tj[xslot][te * M + tq * 4], A.type + (int64_t)S.cj[eslot][te] * M + tq * 4, 16);
    };
    if (e_end > e_beg) {
      stage_entries(0, e_beg);
      stage_entries(1, e_beg + CH);
      cp_async_commit();
      cp_async_wait_all();
      __syncwarp();
      stage_jatoms(0, 0);
      cp_async_commit();
    }

    // the group's i-atoms: group frame (s_xi, band fixes), negated and
    // pair-interleaved (s_xy, s_zq; charges positive), LJ rows per j-type
    for (int ia = lane; ia < IA; ia += 32) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ia < nmem * M) {
        v = A.xyzq[(int64_t)first * M + ia];
        const int64_t c = first + ia / M;
        v.x = (float)((A.bbox[6 * c + 0] - A.bbox[6 * (int64_t)first + 0]) + (double)v.x);
        v.y = (float)((A.bbox[6 * c + 1] - A.bbox[6 * (int64_t)first + 1]) + (double)v.y);
        v.z = (float)((A.bbox[6 * c + 2] - A.bbox[6 * (int64_t)first + 2]) + (double)v.z);
        v.w *= A.coul;
      }
      s_xi[w][ia] = v;
      float* xyf = reinterpret_cast<float*>(&s_xy[w][0]);
      float* zqf = reinterpret_cast<float*>(&s_zq[w][0]);
      const int h = ia >> 1, o = ia & 1;
      xyf[4 * h + o] = -v.x;
      xyf[4 * h + 2 + o] = -v.y;
      zqf[4 * h + o] = -v.z;
      zqf[4 * h + 2 + o] = v.w;
    }
    for (int idx = lane; idx < H * A.nt; idx += 32) {
      const int t = idx / H, h = idx - t * H;
      const int ti0 = 2 * h < nmem * M ? A.type[(int64_t)first * M + 2 * h] : 0;
      const int ti1 = 2 * h + 1 < nmem * M ? A.type[(int64_t)first * M + 2 * h + 1] : 0;
      const float4 a0 = __ldg(&A.lj[ti0 * A.nt + t]), a1 = __ldg(&A.lj[ti1 * A.nt + t]);
      s_l2[t * LJS + h] = make_float4(-a0.x, -a1.x, a0.y, a1.y);
      s_sh[t * LJS + h] = make_float2(a0.z, a1.z);
    }
    if (BAND) {
      for (int idx = lane; idx < IA * A.nt; idx += 32) {
        const int t = idx / IA, ia = idx - t * IA;
        const int ti = ia < nmem * M ? A.type[(int64_t)first * M + ia] : 0;
        s_lj[idx] = __ldg(&A.lj[ti * A.nt + t]);
      }
      for (int c = lane; c < IA * 3; c += 32) s_corr[w][c] = 0.f;
    }
    __syncwarp();

    const float slack_thr = A.slack_base + 4.f * __uint_as_float(A.scalars[0]);
    float2 fi[4][3];
#pragma unroll
    for (int h = 0; h < 4; ++h) fi[h][0] = fi[h][1] = fi[h][2] = make_float2(0.f, 0.f);
    double elj_acc = 0.0, ec_acc = 0.0;
    const int sha_ = 8 * ih * (W == 1) + 32 * ih * (W == 2) + 2 * jp;  // mask shift of the lane's pairs

    int es = 0;
    for (int32_t ec0 = e_beg, c = 0; ec0 < e_end; ec0 += CH, ++c) {
      // chunk c's entries and j-atoms have landed; stage chunk c+1's
      // j-atoms and chunk c+2's entries
      cp_async_wait_all();
      __syncwarp();
      const int xs = c & 1;
      {
        const int es1 = es == 2 ? 0 : es + 1, es2 = es1 == 2 ? 0 : es1 + 1;
        if (ec0 + CH < e_end) stage_jatoms(xs ^ 1, es1);
        if (ec0 + 2 * CH < e_end) stage_entries(es2, ec0 + 2 * CH);
        cp_async_commit();
      }
      const float4* c_ed = S.ed[es];
      const uint64_t* c_em = &S.em[es][0][0];
      const int32_t* c_cj = S.cj[es];
      const int32_t* c_tp = S.tp[es];
      const float4* c_xa = &S.xj[xs][ih * CJ];
      const float4* c_xb = &S.xj[xs][(1 - ih) * CJ];
      const int32_t* c_ty = S.tj[xs];
      es = es == 2 ? 0 : es + 1;
      const int32_t c_end = min(ec0 + CH, e_end);
#pragma unroll 1
    for (int32_t e0 = ec0, ci = 0; e0 < c_end; e0 += R, ci += R) {
      const bool valid = e0 + r < e_end;
      const int ce = ci + r;  // entry within the chunk
      const float4 d = c_ed[ce];
      uint64_t ma, mb;
      unsigned wpres = 0;
      if constexpr (W == 2) {
        const uint64_t w0 = valid ? c_em[ce * 2] : 0ull, w1 = valid ? c_em[ce * 2 + 1] : 0ull;
        const uint32_t a0 = (uint32_t)(w0 >> (sha_ + ih)), a1 = (uint32_t)(w1 >> (sha_ + ih));
        const uint32_t b0 = (uint32_t)(w0 >> (sha_ + 1 - ih)), b1 = (uint32_t)(w1 >> (sha_ + 1 - ih));
        ma = (uint64_t)a0 | ((uint64_t)a1 << 32);
        mb = (uint64_t)b0 | ((uint64_t)b1 << 32);
        // member presence over the iteration's entries (uniform datapath)
        const unsigned p0 = __reduce_or_sync(0xffffffffu, (uint32_t)w0 | (uint32_t)(w0 >> 32));
        const unsigned p1 = __reduce_or_sync(0xffffffffu, (uint32_t)w1 | (uint32_t)(w1 >> 32));
        wpres = (p0 ? 1u : 0u) | (p1 ? 2u : 0u);
      } else {
        const uint64_t w0 = valid ? c_em[ce] : 0ull;
        ma = w0 >> (sha_ + ih);
        mb = w0 >> (sha_ + 1 - ih);
        const unsigned lo = __reduce_or_sync(0xffffffffu, (uint32_t)w0);
        const unsigned hi = __reduce_or_sync(0xffffffffu, (uint32_t)(w0 >> 32));
        wpres = ((lo & 0xffffu) ? 1u : 0u) | ((lo >> 16) ? 2u : 0u) | ((hi & 0xffffu) ? 4u : 0u) |
                ((hi >> 16) ? 8u : 0u);
      }
      const int32_t cj = BAND ? c_cj[ce] : 0;
      const int xo = ci * JP + (lane & 15);  // = (ci + r) * JP + jp
      float4 xj[2];
      int tj[2];
      xj[0] = c_xa[xo];
      xj[1] = c_xb[xo];
      tj[0] = c_ty[ce * M + ba];
      tj[1] = c_ty[ce * M + bb];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        xj[q].x += d.x;
        xj[q].y += d.y;
        xj[q].z += d.z;
      }
      const bool wunsafe = __any_sync(0xffffffffu, valid && d.w < slack_thr);
      float2 fa[3], fb[3];
      fa[0] = fa[1] = fa[2] = fb[0] = fb[1] = fb[2] = make_float2(0.f, 0.f);
      float2 el2 = make_float2(0.f, 0.f), ec2 = el2;
      uint32_t near = 0;
      const float4* la = s_l2 + tj[0] * LJS;
      const float4* lb = s_l2 + tj[1] * LJS;
      const float2* sa = s_sh + tj[0] * LJS;
      const float2* sbp = s_sh + tj[1] * LJS;
      if (!wunsafe)
        sweep_h<M, ELEC, KRF, ENERGY, BAND, false>(A, s_xy[w], s_zq[w], la, lb, sa, sbp, ma, mb, wpres, ih, xj[0],
                                                   xj[1], fi, fa, fb, el2, ec2, near);
      else
        sweep_h<M, ELEC, KRF, ENERGY, BAND, true>(A, s_xy[w], s_zq[w], la, lb, sa, sbp, ma, mb, wpres, ih, xj[0],
                                                  xj[1], fi, fa, fb, el2, ec2, near);
      float fj[2][3] = {{fa[0].x + fa[0].y, fa[1].x + fa[1].y, fa[2].x + fa[2].y},
                        {fb[0].x + fb[0].y, fb[1].x + fb[1].y, fb[2].x + fb[2].y}};
      float elj = 0.f, ec = 0.f;
      if (ENERGY) {
        elj = el2.x + el2.y;
        ec = ec2.x + ec2.y;
      }
      if (BAND && __any_sync(0xffffffffu, near != 0)) {
        if (near) {
          const int bj[2] = {ba, bb};
          if (!wunsafe)
            band_fix_h<M, ELEC, KRF, ENERGY, false>(A, s_xi[w], s_lj, s_corr[w], near, xj, tj, bj, ih, first, cj, fj,
                                                    elj, ec);
          else
            band_fix_h<M, ELEC, KRF, ENERGY, true>(A, s_xi[w], s_lj, s_corr[w], near, xj, tj, bj, ih, first, cj, fj,
                                                   elj, ec);
        }
        __syncwarp();
      }
      // the partner half's b-atom is this lane's a-atom
      float out[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) out[c] = fj[0][c] + __shfl_xor_sync(0xffffffffu, fj[1][c], 16);
      if (valid) {
        // partials land in j-cluster order (t_pos, always set for this
        // kernel), so k_reduce streams them (packed xyz, 12 B per partial)
        float* dst = reinterpret_cast<float*>(A.part_j) + ((int64_t)c_tp[ce] * M + ba) * 3;
        dst[0] = out[0];
        dst[1] = out[1];
        dst[2] = out[2];
      }
      if (ENERGY) {
        elj_acc += (double)elj;
        ec_acc += (double)ec;
      }
    }
    }

    cp_async_wait_all();
    __syncwarp();

    // i-forces: lane holds -F of atoms lane_atom(hl, s, ih) at t = 2 hl + s;
    // sum over the 16 lanes of each half in a fixed order
#pragma unroll
    for (int h = 0; h < 4; ++h)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        s_ws[w].red[lane][3 * (2 * h) + c] = fi[h][c].x;
        s_ws[w].red[lane][3 * (2 * h + 1) + c] = fi[h][c].y;
      }
    __syncwarp();
    float acc[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int o = lane + 32 * u;  // output o = 3 ia + c
      acc[u] = 0.f;
      if (o < IA * 3) {
        const int ia = o / 3, c = o - 3 * ia;
        const int h = ia >> 1, km = h / (M / 2), wm = h - km * (M / 2);
        const int hf = wm / (M / 4), t = 2 * (km * (M / 4) + wm % (M / 4)) + (ia & 1);
        float sacc = 0.f;
#pragma unroll 4
        for (int l = 0; l < 16; ++l) sacc += s_ws[w].red[16 * hf + l][3 * t + c];
        acc[u] = BAND ? s_corr[w][o] - sacc : -sacc;
      }
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int o = lane + 32 * u;
      if (o < IA * 3) s_ws[w].red[0][o] = acc[u];
    }
    __syncwarp();
    if (lane < nmem * M) {
      A.part_i[part * A.ns + (int64_t)first * M + lane] =
          make_float4(s_ws[w].red[0][3 * lane], s_ws[w].red[0][3 * lane + 1], s_ws[w].red[0][3 * lane + 2], 0.f);
    }
    if (ENERGY) {
      for (int o = 16; o; o >>= 1) {
        elj_acc += __shfl_xor_sync(0xffffffffu, elj_acc, o);
        ec_acc += __shfl_xor_sync(0xffffffffu, ec_acc, o);
      }
      if (lane == 0) {
        A.e_grp[2 * wi] = elj_acc;
        A.e_grp[2 * wi + 1] = ec_acc;
      }
    }
    __syncwarp();
  }
}

// Gather positions for this evaluation: clustered FP32 coordinates placed in
// the periodic image nearest to the build-time positions (so build-time shift
// vectors stay valid), charges, types, and the max displacement since build.
__global__ void k_gather(const double* __restrict__ pos, const double* __restrict__ q,
                         const int64_t* __restrict__ typ, const int32_t* __restrict__ perm,
                         const uint8_t* __restrict__ fill, const double* __restrict__ cpos,
                         const double* __restrict__ bbox, int m, int64_t n_slots, Box box,
                         float4* __restrict__ xyzq,
                         int32_t* __restrict__ type_out, unsigned int* __restrict__ scalars,
                         const float4* __restrict__ xprune) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  float disp = 0.f, dpr = 0.f;
  if (s < n_slots) {
    const int64_t o = perm[s];
    float v[3];
    double d2 = 0.0;
    for (int d = 0; d < 3; ++d) {
      const double x = pos[3 * o + d], xb = cpos[3 * s + d];
      const double xu = x - box.L[d] * rint((x - xb) * box.invL[d]);
      v[d] = (float)(xu - bbox[6 * (s / m) + d]);
      d2 += (xu - xb) * (xu - xb);
    }
    disp = (float)sqrt(d2);
    if (xprune) {  // same frames (float), rounded up past the FP32 error
      const float4 xp = xprune[s];
      const float ex = v[0] - xp.x, ey = v[1] - xp.y, ez = v[2] - xp.z;
      dpr = sqrtf(fmaf(ex, ex, fmaf(ey, ey, ez * ez))) * 1.0001f + 1e-6f;
    }
    xyzq[s] = make_float4(v[0], v[1], v[2], fill[s] ? 0.f : (float)q[o]);
    type_out[s] = (int32_t)typ[o];
  }
  for (int o = 16; o; o >>= 1) disp = fmaxf(disp, __shfl_xor_sync(0xffffffffu, disp, o));
  if ((threadIdx.x & 31) == 0 && disp > 0.f) atomicMax(&scalars[0], __float_as_uint(disp));
  if (xprune) {
    for (int o = 16; o; o >>= 1) dpr = fmaxf(dpr, __shfl_xor_sync(0xffffffffu, dpr, o));
    if ((threadIdx.x & 31) == 0 && dpr > 0.f) atomicMax(&scalars[5], __float_as_uint(dpr));
  }
}

// Final per-atom forces: own i-partial + j-partials of every entry whose
// j-cluster holds the atom.  One warp per cluster, lane = (stride s of 32/m,
// j-slot b): lane sums items s, s + 32/m, ... in FP64, then a fixed shuffle
// tree combines the strides -- the same order on every run (deterministic).
__global__ void k_reduce(const float4* __restrict__ part_i, const float4* __restrict__ part_j,
                         const int32_t* __restrict__ t_first, const int32_t* __restrict__ t_items,
                         const int32_t* __restrict__ perm, const uint8_t* __restrict__ fill,
                         int64_t n_clusters, int m, int flags, double* __restrict__ f_out,
                         unsigned int* __restrict__ flag, int split, float inner_dmax,
                         const unsigned int* __restrict__ dref, int parts, int64_t ns, int64_t c_off) {
  // clusters [c_off, n_clusters) (n_clusters: the end of this launch's range)
  const int64_t c = c_off + blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= n_clusters) return;
  const int S = 32 / m;
  const int sidx = lane / m, b = lane - sidx * m;
  double fx = 0.0, fy = 0.0, fz = 0.0;
  // split transpose (dynamic pruning): 2 n_clusters + 1 bounds, [2c, 2c+1)
  // the entries with an inner member, [2c+1, 2c+2) the others -- those are
  // read only when k_force_h evaluated them (full masks: d_max = *dref above
  // the inner list's margin; inner_dmax < 0 after a rolling prune)
  int32_t tb, t1;
  if (split) {
    tb = t_first[2 * c];
    t1 = __uint_as_float(*dref) <= inner_dmax ? t_first[2 * c + 1] : t_first[2 * c + 2];
  } else {
    tb = t_first[c];
    t1 = t_first[c + 1];
  }
  // U transposed items per lane in flight (index loads, then partial loads);
  // each lane sums its items (ascending t) in FP32 -- a handful of FP32
  // partials, no per-item FP64 conversions -- and the lanes' sums are
  // combined in FP64 by a fixed shuffle tree: the order never changes, so
  // forces stay bit-reproducible
#ifndef NBX_REDUCE_U
#define NBX_REDUCE_U 4
#endif
  constexpr int U = NBX_REDUCE_U;
  float sx = 0.f, sy = 0.f, sz = 0.f;
  for (int32_t t0 = tb + sidx; t0 < t1; t0 += S * U) {
    int32_t it[U];
#pragma unroll
    for (int u = 0; u < U; ++u) it[u] = t0 + u * S < t1 ? (t_items ? __ldg(t_items + t0 + u * S) : t0 + u * S) : -1;
    float4 pj[U];
    if (t_items) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        pj[u] = it[u] >= 0 ? __ldg(part_j + (int64_t)it[u] * m + b) : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {  // sorted mode: packed xyz partials (k_force_h)
      const float* pf = reinterpret_cast<const float*>(part_j);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t o = ((int64_t)it[u] * m + b) * 3;
        pj[u] = it[u] >= 0 ? make_float4(__ldg(pf + o), __ldg(pf + o + 1), __ldg(pf + o + 2), 0.f)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (it[u] < 0) break;
      sx += pj[u].x;
      sy += pj[u].y;
      sz += pj[u].z;
    }
  }
  fx = sx;
  fy = sy;
  fz = sz;
  for (int o = 16; o >= m; o >>= 1) {
    fx += __shfl_xor_sync(0xffffffffu, fx, o);
    fy += __shfl_xor_sync(0xffffffffu, fy, o);
    fz += __shfl_xor_sync(0xffffffffu, fz, o);
  }
  if (sidx != 0) return;
  const int64_t s = c * m + b;
  for (int q = 0; q < parts; ++q) {  // i-partials of the group's parts, fixed order
    const float4 pi = part_i[q * ns + s];
    fx += pi.x;
    fy += pi.y;
    fz += pi.z;
  }
  if (!isfinite(fx) || !isfinite(fy) || !isfinite(fz)) atomicOr(flag, 1u);
  int64_t o;
  if (flags & NBX_FORCE_CLUSTERED) {
    o = s;
  } else {
    if (fill[s]) return;
    o = perm[s];
  }
  if (flags & NBX_FORCE_ACCUMULATE) {
    f_out[3 * o] += fx;
    f_out[3 * o + 1] += fy;
    f_out[3 * o + 2] += fz;
  } else {
    f_out[3 * o] = fx;
    f_out[3 * o + 1] = fy;
    f_out[3 * o + 2] = fz;
  }
}

__global__ void k_energy(const double* __restrict__ e_grp, int64_t n, double* __restrict__ e_out,
                         const unsigned int* __restrict__ scalars, int64_t* __restrict__ bad,
                         unsigned int* __restrict__ reset) {
  __shared__ double s[2][256];
  double a = 0.0, c = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 256) {
    a += e_grp[2 * i];
    c += e_grp[2 * i + 1];
  }
  s[0][threadIdx.x] = a;
  s[1][threadIdx.x] = c;
  __syncthreads();
  for (int h = 128; h; h >>= 1) {
    if (threadIdx.x < h) {
      s[0][threadIdx.x] += s[0][threadIdx.x + h];
      s[1][threadIdx.x] += s[1][threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (e_out) {
      e_out[0] = s[0][0];
      e_out[1] = s[1][0];
    }
    if (bad) {
      const unsigned long long key = *reinterpret_cast<const unsigned long long*>(scalars + 2);
      if (key == ~0ull) {
        // non-finite forces without a located pair: the host runs
        // nbx_find_singular (exact scan) to name the coincident pair
        bad[0] = bad[1] = scalars[1] ? -2 : -1;
      } else {
        bad[0] = (int64_t)(key >> 32);
        bad[1] = (int64_t)(key & 0xffffffffull);
      }
    }
    // the next force call's k_init_scalars, done here (one launch fewer per call)
    if (reset)
      for (int i = 0; i < 7; ++i) reset[i] = (i == 2 || i == 3) ? 0xffffffffu : 0u;
  }
}

__global__ void k_init_scalars(unsigned int* scalars) {
  // [0] max displacement, [1] non-finite flag, [2..3] bad key, [4] work counter
  // [5] max displacement since the rolling prune
  if (threadIdx.x < 7) scalars[threadIdx.x] = (threadIdx.x == 2 || threadIdx.x == 3) ? 0xffffffffu : 0u;
}

__global__ void k_build_lj(const double* __restrict__ tab, int nt, double rc2, int shift,
                           float4* __restrict__ lj) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt * nt) return;
  const double eps = tab[2 * i], sig = tab[2 * i + 1];
  const double s2 = sig * sig, s6 = s2 * s2 * s2;
  const double c6 = 4.0 * eps * s6, c12 = 4.0 * eps * s6 * s6;
  double sh = 0.0;
  if (shift) {
    const double sr2 = s2 / rc2, sr6 = sr2 * sr2 * sr2;
    sh = 4.0 * eps * (sr6 * sr6 - sr6);
  }
  lj[i] = make_float4((float)(6.0 * c6), (float)(12.0 * c12), (float)sh, 0.f);
}

// ---------------------------------------------------------------- dispatch
template <int M, int G, int ELEC, bool KRF, bool ENERGY, bool BAND>
static cudaError_t launch_one(const ForceArgs& A, cudaStream_t s) {
  constexpr int IA = G * M;
  constexpr int H = (IA % 2) == 0 ? IA / 2 : 1;
  const size_t dyn = (sizeof(float4) * (size_t)(IA + H) + sizeof(float2) * (size_t)H) * FW * A.nt;
  auto kern = k_force<M, G, ELEC, KRF, ENERGY, BAND>;
  static size_t dyn_set = 0;  // static + dynamic may exceed the default 48 KB
  if (dyn > dyn_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    dyn_set = dyn;
  }
  // persistent grid: as many blocks as fit on the GPU at once
  static int max_blocks = 0;
  if (max_blocks == 0) {
    int dev = 0, n_sm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, FW * 32, dyn);
    max_blocks = n_sm * (per_sm > 0 ? per_sm : 1);
  }
  int64_t blocks = (A.n_work + FW - 1) / FW;
  if (blocks > max_blocks) blocks = max_blocks;
  if (blocks > 0) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    const bool tm = timing_enabled();
    if (tm) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
    }
    count_launch();
    kern<<<(unsigned)blocks, FW * 32, dyn, s>>>(A);
    if (tm) {
      cudaEventRecord(e1, s);
      timing_record(e0, e1);
    }
  }
  return cudaGetLastError();
}

template <int M, int G>
static cudaError_t launch_mg(const ForceArgs& A, int elec, bool krf, bool energy, bool band, cudaStream_t s) {
  if (elec == FE_EWALD)
    return energy ? launch_one<M, G, FE_EWALD, false, true, false>(A, s)
                  : launch_one<M, G, FE_EWALD, false, false, false>(A, s);
  if (krf) {
    if (band)
      return energy ? launch_one<M, G, FE_RF, true, true, true>(A, s) : launch_one<M, G, FE_RF, true, false, true>(A, s);
    return energy ? launch_one<M, G, FE_RF, true, true, false>(A, s) : launch_one<M, G, FE_RF, true, false, false>(A, s);
  }
  if (band)
    return energy ? launch_one<M, G, FE_RF, false, true, true>(A, s) : launch_one<M, G, FE_RF, false, false, true>(A, s);
  return energy ? launch_one<M, G, FE_RF, false, true, false>(A, s) : launch_one<M, G, FE_RF, false, false, false>(A, s);
}

template <int M, int ELEC, bool KRF, bool ENERGY, bool BAND>
static cudaError_t launch_h(const ForceArgs& A, cudaStream_t s) {
  constexpr int IA = 16;
  const size_t tn = (size_t)LJS * A.nt;
  const size_t dyn = sizeof(float4) * (FW * tn + (FW * tn + 1) / 2 + (BAND ? FW * IA * (size_t)A.nt : 0));
  auto kern = k_force_h<M, ELEC, KRF, ENERGY, BAND>;
  static size_t dyn_set = 0;
  if (dyn > dyn_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    dyn_set = dyn;
  }
  static int max_blocks = 0;
  if (max_blocks == 0) {
    int dev = 0, n_sm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, FW * 32, dyn);
    max_blocks = n_sm * (per_sm > 0 ? per_sm : 1);
  }
  int64_t blocks = (A.n_work + FW - 1) / FW;
  if (blocks > max_blocks) blocks = max_blocks;
  if (blocks > 0) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    const bool tm = timing_enabled();
    if (tm) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
    }
    count_launch();
    kern<<<(unsigned)blocks, FW * 32, dyn, s>>>(A);
    if (tm) {
      cudaEventRecord(e1, s);
      timing_record(e0, e1);
    }
  }
  return cudaGetLastError();
}

template <int M>
static cudaError_t launch_mh(const ForceArgs& A, int elec, bool krf, bool energy, bool band, cudaStream_t s) {
  if (elec == FE_EWALD)
    return energy ? launch_h<M, FE_EWALD, false, true, false>(A, s) : launch_h<M, FE_EWALD, false, false, false>(A, s);
  if (krf) {
    if (band) return energy ? launch_h<M, FE_RF, true, true, true>(A, s) : launch_h<M, FE_RF, true, false, true>(A, s);
    return energy ? launch_h<M, FE_RF, true, true, false>(A, s) : launch_h<M, FE_RF, true, false, false>(A, s);
  }
  if (band) return energy ? launch_h<M, FE_RF, false, true, true>(A, s) : launch_h<M, FE_RF, false, false, true>(A, s);
  return energy ? launch_h<M, FE_RF, false, true, false>(A, s) : launch_h<M, FE_RF, false, false, false>(A, s);
}

// NBX_FORCE_KERNEL=legacy selects k_force (one j-atom per lane) for the
// grouped layout at m = 4, 8 too (A/B measurements)
static bool use_legacy_force() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("NBX_FORCE_KERNEL");
    v = (e && strcmp(e, "legacy") == 0) ? 1 : 0;
  }
  return v == 1;
}

static cudaError_t launch_force(int m, bool grouped, const ForceArgs& A, int elec, bool krf, bool energy, bool band,
                                cudaStream_t s) {
  switch (m) {
    case 1: return grouped ? launch_mg<1, 16>(A, elec, krf, energy, band, s) : launch_mg<1, 1>(A, elec, krf, energy, band, s);
    case 2: return grouped ? launch_mg<2, 8>(A, elec, krf, energy, band, s) : launch_mg<2, 1>(A, elec, krf, energy, band, s);
    case 4:
      if (grouped && !use_legacy_force()) return launch_mh<4>(A, elec, krf, energy, band, s);
      return grouped ? launch_mg<4, 4>(A, elec, krf, energy, band, s) : launch_mg<4, 1>(A, elec, krf, energy, band, s);
    default:
      if (grouped && !use_legacy_force()) return launch_mh<8>(A, elec, krf, energy, band, s);
      return grouped ? launch_mg<8, 2>(A, elec, krf, energy, band, s) : launch_mg<8, 1>(A, elec, krf, energy, band, s);
  }
}

// Chebyshev fit of the Ewald correction functions (see EW_DEG above), in
// double precision on the host, converted to a power series in u.
static double ew_gf(double w) {  // erf(z)/z^3 - 2 exp(-w) / (sqrt(pi) w)
  if (w < 0.5) {  // series: (2/sqrt(pi)) sum_{n>=1} (-1)^(n+1) w^(n-1) 2n / (n! (2n+1))
    double s = 0.0, term = 1.0;  // term = w^(n-1) / n!
    for (int n = 1; n < 30; ++n) {
      term = (n == 1) ? 1.0 : term * w / n;
      s += ((n & 1) ? 1.0 : -1.0) * term * (2.0 * n) / (2.0 * n + 1.0);
    }
    return 2.0 / sqrt(M_PI) * s;
  }
  const double z = sqrt(w);
  return erf(z) / (z * w) - 2.0 / sqrt(M_PI) * exp(-w) / w;
}
static double ew_gv(double w) {  // erf(z)/z
  if (w < 1e-12) return 2.0 / sqrt(M_PI);
  const double z = sqrt(w);
  return erf(z) / z;
}
static void ew_fit(double (*f)(double), double wmax, int deg, float* out /* deg+1, highest first */,
                   double scale = 1.0) {
  const int N = deg + 1;
  double c[16] = {0};
  for (int k = 0; k < N; ++k) {
    double acc = 0.0;
    for (int j = 0; j < N; ++j) {
      const double x = cos(M_PI * (j + 0.5) / N);
      acc += f((x + 1.0) * 0.5 * wmax) * cos(M_PI * k * (j + 0.5) / N);
    }
    c[k] = acc * 2.0 / N;
  }
  c[0] *= 0.5;
  // Chebyshev -> power series in u: T_{k+1} = 2u T_k - T_{k-1}
  double Tprev[16] = {0}, Tcur[16] = {0}, p[16] = {0};
  Tprev[0] = 1.0;            // T_0
  Tcur[1] = 1.0;             // T_1
  p[0] += c[0];
  for (int i = 0; i <= deg; ++i) p[i] += c[1] * Tcur[i];
  for (int k = 2; k < N; ++k) {
    double Tn[16] = {0};
    for (int i = 0; i <= deg; ++i) {
      if (i > 0) Tn[i] += 2.0 * Tcur[i - 1];
      Tn[i] -= Tprev[i];
    }
    for (int i = 0; i <= deg; ++i) {
      p[i] += c[k] * Tn[i];
      Tprev[i] = Tcur[i];
      Tcur[i] = Tn[i];
    }
  }
  for (int i = 0; i <= deg; ++i) out[i] = (float)(scale * p[deg - i]);
}

// transposed index: items (entries or rows) sorted by j-cluster, stable
static cudaError_t build_transpose(const int32_t* keys, int64_t n, int64_t n_clusters, DBuf<int32_t>& first,
                                   DBuf<int32_t>& items, cudaStream_t s, DBuf<int32_t>* pos = nullptr);

static int nb(int64_t n, int t) { return (int)((n + t - 1) / t); }

__global__ void k_iota(int32_t* v, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)i;
}

// bucket starts of the sorted keys and (optional) the inverse permutation
// pos[items[i]] = i, in one pass
__global__ void k_first_sorted(const int32_t* __restrict__ keys, int64_t n, int64_t n_keys,
                               int32_t* __restrict__ first, const int32_t* __restrict__ items,
                               int32_t* __restrict__ pos) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  // keys >= n_keys are unused storage slots (sorted last)
  const int32_t prev = i == 0 ? -1 : min(keys[i - 1], (int32_t)n_keys);
  const int32_t cur = i == n ? (int32_t)n_keys : min(keys[i], (int32_t)n_keys);
  for (int32_t c = prev + 1; c <= cur; ++c) first[c] = (int32_t)i;
  if (pos && i < n) pos[items[i]] = (int32_t)i;
}

// split-transpose keys: 2 j + 1 for entries without an inner member (unused
// storage slots hold j = n_clusters and sort last either way)
__global__ void k_split_keys(const int32_t* __restrict__ ej, const uint64_t* __restrict__ fmask, int64_t n, int W,
                             int32_t* __restrict__ keys) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t any = fmask[i * W];
  if (W == 2) any |= fmask[i * W + 1];
  keys[i] = 2 * ej[i] + (any ? 0 : 1);
}

static cudaError_t build_transpose(const int32_t* keys, int64_t n, int64_t n_clusters, DBuf<int32_t>& first,
                                   DBuf<int32_t>& items, cudaStream_t s, DBuf<int32_t>* pos) {
  DBuf<int32_t> vals, skeys;
  cudaError_t e;
  if ((e = first.alloc(n_clusters + 1, s)) || (e = items.alloc(n, s)) || (e = vals.alloc(n, s)) ||
      (e = skeys.alloc(n, s)))
    return e;
  int end_bit = 1;
  while ((int64_t(1) << end_bit) <= n_clusters) ++end_bit;
  if (n > 0) {
    count_launch(), k_iota<<<nb(n, 256), 256, 0, s>>>(vals.p, n);
    if ((e = sort_pairs_i32(keys, skeys.p, vals.p, items.p, n, end_bit, s))) return e;
  }
  if (pos && (e = pos->alloc(n, s))) return e;
  count_launch(), k_first_sorted<<<nb(n + 1, 256), 256, 0, s>>>(skeys.p, n, n_clusters, first.p, items.p,
                                                               pos ? pos->p : nullptr);
  vals.release(s);
  skeys.release(s);
  return cudaGetLastError();
}

}  // namespace nbx

using namespace nbx;

namespace nbx {
// One force evaluation in phases, so that a caller (the domain decomposition,
// dd.cu) can interleave communication: force_setup (validation, workspace,
// force layout, LJ table, scalars, k_gather), force_launch over a range of
// work items, force_regather (k_gather again after halo rows changed),
// force_finish (k_reduce, energies, rolling prune).
struct ForceCall {
  nbx_list* l = nullptr;
  const nbx_grid_t* grid = nullptr;
  cudaStream_t s = nullptr;
  ForceArgs A{};
  const int32_t* sel0 = nullptr;
  double* e_grp0 = nullptr;
  bool canonical = false, sorted_j = false, ewald = false, band = false, use_krf = false;
  int m = 0, flags = 0, n_launched = 0;
  int64_t ns = 0, n_work = 0;
  const double* positions = nullptr;
  const double* charges = nullptr;
  const int64_t* lj_type = nullptr;
  Box bx{};
};

// The grouped force layout (work order, member-pattern entry order) and the
// j-cluster transpose k_reduce reads, built once per list -- by its first
// force call, or ahead of it by nbx_list_step.
cudaError_t force_prepare(List* l, cudaStream_t s) {
  ForceWork& wk = l->work;
  const int m = l->m;
  cudaError_t e;
  if (!l->ordered) {
    if ((e = finalize_force_layout(l, s))) return e;
    wk.t_ready = false;
  }
  if (wk.t_ready) return cudaSuccess;
  // with an inner list (k_force_h only): key 2 j + (no inner member), so
  // that k_reduce can stop before the entries k_force_h skipped
  wk.t_split = l->ent_fmask.p && (m == 4 || m == 8) && !use_legacy_force() && l->n_entries > 0;
  if (wk.t_split) {
    DBuf<int32_t> tkeys;
    if ((e = tkeys.alloc(l->n_entries, s))) return e;
    count_launch();
    k_split_keys<<<nb(l->n_entries, 256), 256, 0, s>>>(l->ent_j.p, l->ent_fmask.p, l->n_entries, l->mask_words(),
                                                        tkeys.p);
    e = build_transpose(tkeys.p, l->n_entries, 2 * l->n_clusters, wk.t_first, wk.t_items, s, &wk.t_pos);
    tkeys.release(s);
    if (e) return e;
  } else if ((e = build_transpose(l->ent_j.p, l->n_entries, l->n_clusters, wk.t_first, wk.t_items, s, &wk.t_pos))) {
    return e;
  }
  wk.t_ready = true;
  return cudaSuccess;
}

// work items per group of k_force_h: the smallest power of two (<= 8) that
// gives at least two work items per resident warp, while parts keep >= 32
// entries on average; NBX_FORCE_SPLIT=1|2|4|8 overrides (A/B)
static int force_parts(const List* l) {
  if (l->n_groups <= 0) return 1;
  if (const char* e = getenv("NBX_FORCE_SPLIT")) {
    const int v = atoi(e);
    if (v == 1 || v == 2 || v == 4 || v == 8) return v;
  }
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm <= 0) n_sm = 148;
  }
  const int64_t resident = (int64_t)n_sm * NBX_FORCEH_MINB * FW;
  int p = 1;
  while (p < 8 && l->n_groups * p < 2 * resident && l->n_entries >= (int64_t)64 * l->n_groups * p) p *= 2;
  return p;
}

static int force_setup(ForceCall& C, const nbx_list_t* lc, const nbx_grid_t* grid, const double* positions,
                       const double* charges, const int64_t* lj_type, const nbx_params_t* p, const double box[3],
                       const int32_t* i_sel, int64_t n_sel, int32_t flags, double* f_out, void* stream) {
  if (!lc || !grid || !p || !box || !f_out) {
    set_error("nbx_force: null argument");
    return NBX_ERR_PARAM;
  }
  nbx_list* l = const_cast<nbx_list*>(static_cast<const nbx_list*>(lc));
  if (grid->m != l->m || grid->n_clusters != l->n_clusters) {
    set_error("layout m=%d, grid m=%d, list m=%d must agree", l->m, grid->m, l->m);
    return NBX_ERR_PARAM;
  }
  if (p->n_types < 1 || p->n_types > 64 || !p->lj_table) {
    set_error("nbx_force: n_types must be in [1, 64]");
    return NBX_ERR_PARAM;
  }
  if (p->elec < 0 || p->elec > 2) {
    set_error("nbx_force: unknown electrostatics %d", p->elec);
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  C.l = l;
  C.grid = grid;
  C.s = s;
  C.flags = flags;
  C.positions = positions;
  C.charges = charges;
  C.lj_type = lj_type;
  ForceWork& wk = l->work;
  const int m = l->m;
  C.m = m;
  const int64_t ns = l->n_clusters * m;
  C.ns = ns;
  const bool canonical = (i_sel != nullptr) || (flags & NBX_FORCE_CANONICAL);
  C.canonical = canonical;
  if (canonical) {
    if (cudaError_t e0 = ensure_rows(l, s)) {
      set_error("nbx_force: %s", cudaGetErrorString(e0));
      return NBX_ERR_CUDA;
    }
  }
  const int64_t n_items = canonical ? l->n_rows : l->n_entries;
  // k_force_h: groups split into `parts` work items (consecutive entry
  // ranges) when there are too few groups to fill the GPU -- small boxes and
  // domain-decomposed ranks -- each part with its own i-partial plane
  const bool grouped_h = !canonical && (m == 4 || m == 8) && !use_legacy_force();
  const int parts = grouped_h ? force_parts(l) : 1;
  const int64_t n_work = canonical ? (i_sel ? n_sel : l->n_clusters) : l->n_groups * parts;
  C.n_work = n_work;
  Box bx;
  for (int d = 0; d < 3; ++d) {
    bx.L[d] = box[d];
    bx.invL[d] = 1.0 / box[d];
  }
  C.bx = bx;
  cudaError_t e;
  double* dtab = nullptr;
  // workspace (cached across calls on this list)
  if (wk.xyzq.n < ns) { if ((e = wk.xyzq.alloc(ns, s))) goto cuda_fail; }
  if (wk.type.n < ns) { if ((e = wk.type.alloc(ns, s))) goto cuda_fail; }
  if (wk.part_i.n < parts * ns) { if ((e = wk.part_i.alloc(parts * ns, s))) goto cuda_fail; }
  if (wk.part_j.n < n_items * m) { if ((e = wk.part_j.alloc(n_items * m, s))) goto cuda_fail; }
  if (wk.e_grp.n < 2 * n_work) { if ((e = wk.e_grp.alloc(2 * n_work + 2, s))) goto cuda_fail; }
  if (wk.scalars.n < 8) { if ((e = wk.scalars.alloc(8, s))) goto cuda_fail; }
  if (wk.lj.n < (int64_t)p->n_types * p->n_types) {
    if ((e = wk.lj.alloc((int64_t)p->n_types * p->n_types, s))) goto cuda_fail;
    wk.lj_key.clear();
  }
  if (!canonical && (e = force_prepare(l, s))) goto cuda_fail;
  if (canonical && (e = ensure_row_delta(l, s))) goto cuda_fail;
  if (canonical && !wk.tc_ready) {
    if ((e = build_transpose(l->j.p, l->n_rows, l->n_clusters, wk.tc_first, wk.tc_items, s))) goto cuda_fail;
    wk.tc_ready = true;
  }
  {
    // LJ table -> device only when it changed (no per-call host copies)
    const int nt = p->n_types;
    std::vector<double> key(p->lj_table, p->lj_table + 2 * nt * nt);
    key.push_back(p->r_cut);
    key.push_back((double)p->shift_potential);
    if (key != wk.lj_key) {
      if ((e = pool_malloc(reinterpret_cast<void**>(&dtab), sizeof(double) * 2 * nt * nt, s))) goto cuda_fail;
      if ((e = cudaMemcpyAsync(dtab, p->lj_table, sizeof(double) * 2 * nt * nt, cudaMemcpyHostToDevice, s))) goto cuda_fail;
      count_launch();
      k_build_lj<<<nb(nt * nt, 64), 64, 0, s>>>(dtab, nt, p->r_cut * p->r_cut, p->shift_potential, wk.lj.p);
      cudaFreeAsync(dtab, s);
      dtab = nullptr;
      wk.lj_key = key;
    }
    // scalars: [0] = 0 (max displacement), [1] = 0 (non-finite flag), [2..3] = ~0 (bad key)
    if (!wk.scalars_clean) count_launch(), k_init_scalars<<<1, 32, 0, s>>>(wk.scalars.p);
    wk.scalars_clean = false;  // (re-set by this call's k_energy when it resets them)
    if (ns > 0)
      count_launch(), k_gather<<<nb(ns, 256), 256, 0, s>>>(positions, charges, lj_type, grid->perm.p, grid->fill.p,
                                           grid->cpos.p, grid->bbox.p, m, ns, bx, wk.xyzq.p, wk.type.p,
                                           wk.scalars.p, canonical ? nullptr : l->xprune.p);
    if (canonical) {
      if (ns > 0 && (e = cudaMemsetAsync(wk.part_i.p, 0, sizeof(float4) * ns, s))) goto cuda_fail;
      if (i_sel && n_items > 0 && (e = cudaMemsetAsync(wk.part_j.p, 0, sizeof(float4) * n_items * m, s))) goto cuda_fail;
    }
    ForceArgs& A = C.A;
    A.n_work = n_work;
    A.split = parts;
    A.wbase = 0;
    A.ns = ns;
    A.sel = canonical ? i_sel : l->group_order.p;
    C.sel0 = A.sel;
    A.grp_first = canonical ? nullptr : l->group_first.p;
    A.grp_nmem = canonical ? nullptr : l->group_nmem.p;
    A.ent_off = canonical ? l->offsets.p : l->ent_offsets.p;
    A.ent_j = canonical ? l->j.p : l->ent_j.p;
    A.ent_delta = canonical ? l->delta.p : l->ent_delta.p;
    A.ent_mask = canonical ? l->mask.p : l->ent_mask.p;
    // k_force_h (grouped, m = 4, 8) writes partials in j-cluster order
    const bool sorted_j = !canonical && (m == 4 || m == 8) && !use_legacy_force();
    C.sorted_j = sorted_j;
    A.ent_tpos = sorted_j ? wk.t_pos.p : nullptr;
    // inner list only where it is safe by a margin over FP32 rounding
    // (r_inner >= r_c + 2e-4 nm); validity is decided on the device
    A.ent_fmask = (sorted_j && l->r_inner >= p->r_cut + 2e-4 && l->ent_fmask.p) ? l->ent_fmask.p : nullptr;
    A.ent_fend = l->ent_fend.p;
    A.inner_dmax = (float)(0.5 * (l->r_inner - p->r_cut) - 5e-5);
    A.inner_slot = l->inner_ref;
    A.xyzq = wk.xyzq.p;
    A.bbox = grid->bbox.p;
    A.type = wk.type.p;
    A.lj = wk.lj.p;
    A.nt = nt;
    A.part_i = wk.part_i.p;
    A.part_j = wk.part_j.p;
    A.e_grp = wk.e_grp.p;
    C.e_grp0 = wk.e_grp.p;
    A.scalars = wk.scalars.p;
    const double rc = p->r_cut;
    A.rc2 = (float)(rc * rc);
    A.rc2d = rc * rc;
    const bool ewald = p->elec == NBX_ELEC_EWALD;
    double krf = 0.0, crf = 0.0;
    if (p->elec == NBX_ELEC_REACTION_FIELD) {
      krf = p->k_rf;
      crf = p->c_rf;
    } else if (p->elec == NBX_ELEC_CUTOFF) {
      crf = p->shift_potential ? 1.0 / rc : 0.0;
    }
    A.krf = (float)krf;
    A.k2rf = (float)(2.0 * krf);
    A.crf = (float)crf;
    A.coul = (float)p->coulomb_scale;
    A.beta = (float)p->ewald_beta;
    A.beta3 = (float)(p->ewald_beta * p->ewald_beta * p->ewald_beta);
    A.ew_shift = p->shift_potential ? (float)(erfc(p->ewald_beta * rc) / rc) : 0.f;
    if (ewald) {
      // fit range: r^2 up to (r_c^2 + band) with margin.  The fits cost ~600
      // transcendental host calls: cached per (beta, r_c) (thread-local).
      struct EwCache {
        double beta = -1.0, rc = -1.0;
        float a, f[16], v[16], sc[16];
      };
      static thread_local EwCache ec;
      if (ec.beta != p->ewald_beta || ec.rc != rc) {
        const double wmax = p->ewald_beta * p->ewald_beta * rc * rc * 1.02;
        ec.a = (float)(2.0 / wmax * p->ewald_beta * p->ewald_beta);
        ew_fit(ew_gf, wmax, EW_DEG_F, ec.f);
        ew_fit(ew_gv, wmax, EW_DEG_V, ec.v);
        ew_fit(ew_gf, wmax, EW_DEG_F, ec.sc, -(double)p->ewald_beta * p->ewald_beta * p->ewald_beta);
        ec.beta = p->ewald_beta;
        ec.rc = rc;
      }
      A.ew_a = ec.a;
      for (int k = 0; k < 16; ++k) {
        A.ew_f[k] = ec.f[k];
        A.ew_v[k] = ec.v[k];
        A.ew_s[k] = ec.sc[k];
      }
    }
    A.slack_base = (float)(2.0 * rc + 1e-3);
    double Lmax = fmax(box[0], fmax(box[1], box[2]));
    A.band = (float)(64.0 * 5.96e-8 * (Lmax * rc + rc * rc));
    for (int d = 0; d < 3; ++d) {
      A.L[d] = (float)box[d];
      A.invL[d] = (float)(1.0 / box[d]);
    }
    A.pos = positions;
    A.perm = grid->perm.p;
    A.box = bx;
    C.ewald = ewald;
    // FP64 re-check of cutoff decisions near r_c only where the Coulomb force
    // jumps there: plain cutoff (the reference's physics) and a
    // reaction field with finite eps_rf.  eps_rf = inf (2 k_rf r_c^3 = 1) and
    // Ewald have F_c(r_c) ~ 0, so a rounding flip at r_c changes nothing.
    C.band = !ewald && fabs(1.0 - 2.0 * krf * rc * rc * rc) > 1e-6;
    C.use_krf = !ewald && krf != 0.0;
  }
  if ((e = cudaGetLastError())) goto cuda_fail;
  return NBX_OK;
cuda_fail:
  if (dtab) cudaFreeAsync(dtab, s);
  set_error("nbx_force: %s", cudaGetErrorString(e));
  return NBX_ERR_CUDA;
}

// the force kernel over work items [w0, w1) of the work order (persistent
// warps claim them through scalars[4], reset here; energies per item land at
// e_grp[2 (w0 + i)], so the ranges of one evaluation add up in k_energy)
static cudaError_t force_launch(ForceCall& C, int64_t w0, int64_t w1) {
  if (w1 <= w0) return cudaSuccess;
  ForceArgs A = C.A;
  if (C.sorted_j) {  // k_force_h: items index the work order through A.split
    A.sel = C.sel0;
    A.wbase = w0;
  } else {
    A.sel = C.sel0 ? C.sel0 + w0 : nullptr;
    if (!C.sel0 && w0 != 0) return cudaErrorInvalidValue;  // identity order: one range only
  }
  A.n_work = w1 - w0;
  A.e_grp = C.e_grp0 + 2 * w0;
  // the work counter is zero for a call's first launch (k_init_scalars or the
  // previous call's k_energy reset it); later launches of the call reset it
  cudaError_t e = C.n_launched++ ? cudaMemsetAsync(A.scalars + 4, 0, sizeof(unsigned int), C.s) : cudaSuccess;
  if (e) return e;
  return launch_force(C.m, !C.canonical, A, C.ewald ? FE_EWALD : FE_RF, C.use_krf,
                      (C.flags & NBX_FORCE_ENERGY) != 0, C.band, C.s);
}

static cudaError_t force_regather(ForceCall& C) {
  if (C.ns <= 0) return cudaSuccess;
  ForceWork& wk = C.l->work;
  count_launch();
  k_gather<<<nb(C.ns, 256), 256, 0, C.s>>>(C.positions, C.charges, C.lj_type, C.grid->perm.p, C.grid->fill.p,
                                           C.grid->cpos.p, C.grid->bbox.p, C.m, C.ns, C.bx, wk.xyzq.p, wk.type.p,
                                           wk.scalars.p, C.canonical ? nullptr : C.l->xprune.p);
  return cudaGetLastError();
}

static int force_finish(ForceCall& C, const double box[3], double* f_out, double* e_out, int64_t* bad,
                        const std::function<int()>* mid = nullptr) {
  nbx_list* l = C.l;
  ForceWork& wk = l->work;
  cudaStream_t s = C.s;
  const ForceArgs& A = C.A;
  cudaError_t e;
  // clusters [c0, c1) of each k_reduce launch; with a `mid` hook (the DD
  // force step) the halo clusters go first, then the hook (their forces
  // leave), then the rest -- the same per-cluster sums, any order
  auto reduce = [&](int64_t c0, int64_t c1) {
    if (c1 <= c0) return;
    count_launch();
    k_reduce<<<nb(c1 - c0, 8), 256, 0, s>>>(wk.part_i.p, wk.part_j.p, C.canonical ? wk.tc_first.p : wk.t_first.p,
                                            C.canonical ? wk.tc_items.p : (C.sorted_j ? nullptr : wk.t_items.p),
                                            C.grid->perm.p, C.grid->fill.p, c1, C.m, C.flags, f_out,
                                            wk.scalars.p + 1, !C.canonical && wk.t_split,
                                            (A.ent_fmask && l->tail_sorted) ? A.inner_dmax : -1.f,
                                            wk.scalars.p + A.inner_slot, C.canonical ? 1 : A.split, C.ns, c0);
  };
  if (C.ns > 0) {
    const int64_t nc = l->n_clusters;
    if (mid && l->halo_c1 > l->halo_c0) {
      reduce(l->halo_c0, l->halo_c1);
      if (int st = (*mid)()) return st;
      reduce(0, l->halo_c0);
      reduce(l->halo_c1, nc);
    } else {
      reduce(0, nc);
      if (mid)
        if (int st = (*mid)()) return st;
    }
  } else if (mid) {
    if (int st = (*mid)()) return st;
  }
  if (!(C.flags & NBX_FORCE_ENERGY) && e_out == nullptr && bad == nullptr) {
    // nothing else to produce
  } else {
    // the rolling prune reads the scalars after this kernel: no reset then
    unsigned int* reset = (C.flags & NBX_FORCE_REPRUNE) ? nullptr : wk.scalars.p;
    if (!(C.flags & NBX_FORCE_ENERGY)) {
      count_launch(), k_energy<<<1, 256, 0, s>>>(wk.e_grp.p, 0, nullptr, wk.scalars.p, bad, reset);
    } else {
      count_launch(), k_energy<<<1, 256, 0, s>>>(wk.e_grp.p, C.n_work, e_out, wk.scalars.p, bad, reset);
    }
    wk.scalars_clean = reset != nullptr;
  }
  if ((e = cudaGetLastError())) goto cuda_fail;
  // rolling prune at this call's coordinates (after the pass that used the old masks)
  if ((C.flags & NBX_FORCE_REPRUNE) && C.sorted_j && l->ent_fmask.p && C.ns > 0 &&
      (e = reprune_inner(l, wk.xyzq.p, wk.scalars.p, C.grid->bbox.p, C.grid->cpos.p, box, s)))
    goto cuda_fail;
  return NBX_OK;
cuda_fail:
  set_error("nbx_force: %s", cudaGetErrorString(e));
  return NBX_ERR_CUDA;
}

int force_split(const nbx_list_t* lc, const nbx_grid_t* grid, const double* positions, const double* charges,
                const int64_t* lj_type, const nbx_params_t* p, const double box[3], int32_t flags, double* f_out,
                double* e_out, int64_t* bad, void* stream, const std::function<int()>& between,
                const std::function<int()>* after_halo, bool split_launch) {
  ForceCall C;
  int st = force_setup(C, lc, grid, positions, charges, lj_type, p, box, nullptr, 0, flags, f_out, stream);
  if (st) return st;
  const int64_t n_int =
      C.canonical || !split_launch ? -1 : (C.l->n_interior < 0 ? -1 : C.l->n_interior * C.A.split);
  cudaError_t e;
  if (n_int < 0) {  // no interior / boundary split: one range, the caller's hook first
    if ((st = between())) return st;
    // (split_launch false: the positions were final before force_setup's gather)
    if ((split_launch && (e = force_regather(C))) || (e = force_launch(C, 0, C.n_work))) goto fail;
    return force_finish(C, box, f_out, e_out, bad, after_halo);
  }
  if ((e = force_launch(C, 0, n_int))) goto fail;
  if ((st = between())) return st;
  if ((e = force_regather(C)) || (e = force_launch(C, n_int, C.n_work))) goto fail;
  return force_finish(C, box, f_out, e_out, bad, after_halo);
fail:
  set_error("nbx_force: %s", cudaGetErrorString(e));
  return NBX_ERR_CUDA;
}
}  // namespace nbx

extern "C" int nbx_force(const nbx_list_t* lc, const nbx_grid_t* grid, const double* positions,
                         const double* charges, const int64_t* lj_type, const nbx_params_t* p,
                         const double box[3], const int32_t* i_sel, int64_t n_sel, int32_t flags,
                         double* f_out, double* e_out, int64_t* bad, void* stream) {
  ForceCall C;
  int st = force_setup(C, lc, grid, positions, charges, lj_type, p, box, i_sel, n_sel, flags, f_out, stream);
  if (st) return st;
  if (cudaError_t e = force_launch(C, 0, C.n_work)) {
    set_error("nbx_force: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  return force_finish(C, box, f_out, e_out, bad);
}

namespace nbx {
// Exact scan of every admitted pair (kernels.py:184-187 semantics): first
// coincident in-range pair in (i-cluster, row, a, b) order.
__global__ void k_find_singular(const int32_t* __restrict__ offsets, const int32_t* __restrict__ jv,
                                const uint64_t* __restrict__ mask, int64_t n_clusters, int m,
                                ForceArgs A) {
  const int64_t ci = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (ci >= n_clusters) return;
  for (int32_t row = offsets[ci]; row < offsets[ci + 1]; ++row) {
    const uint64_t mk = mask[row];
    for (int a = 0; a < m; ++a)
      for (int b = 0; b < m; ++b)
        if ((mk >> (a * m + b)) & 1ull) {
          const int64_t si = ci * m + a, sj = (int64_t)jv[row] * m + b;
          if (exact_inside(A, si, sj) < 0) {
            record_bad(A.scalars, si, sj);
            return;
          }
        }
  }
}
}  // namespace nbx

extern "C" int nbx_find_singular(const nbx_list_t* l, const nbx_grid_t* grid, const double* positions,
                                 double r_cut, const double box[3], void* stream, int64_t out[2]) {
  if (!l || !grid || !positions || !box || !out) {
    set_error("nbx_find_singular: null argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  DBuf<unsigned int> sc;
  unsigned int h[4] = {0u, 0u, 0xffffffffu, 0xffffffffu};
  cudaError_t e;
  ForceArgs A{};
  A.pos = positions;
  A.perm = grid->perm.p;
  A.rc2d = r_cut * r_cut;
  for (int d = 0; d < 3; ++d) {
    A.box.L[d] = box[d];
    A.box.invL[d] = 1.0 / box[d];
  }
  if ((e = ensure_rows(const_cast<nbx_list*>(static_cast<const nbx_list*>(l)), s))) goto fail;
  if ((e = sc.alloc(4, s))) goto fail;
  if ((e = cudaMemcpyAsync(sc.p, h, 16, cudaMemcpyHostToDevice, s))) goto fail;
  A.scalars = sc.p;
  if (l->n_clusters > 0)
    count_launch(), k_find_singular<<<nb(l->n_clusters, 128), 128, 0, s>>>(l->offsets.p, l->j.p, l->mask.p, l->n_clusters,
                                                            l->m, A);
  if ((e = cudaGetLastError())) goto fail;
  if ((e = cudaMemcpyAsync(h, sc.p, 16, cudaMemcpyDeviceToHost, s))) goto fail;
  if ((e = cudaStreamSynchronize(s))) goto fail;
  sc.release(s);
  {
    const unsigned long long key = ((unsigned long long)h[3] << 32) | h[2];
    if (key == ~0ull) {
      out[0] = out[1] = -1;
    } else {
      out[0] = (int64_t)(key >> 32);
      out[1] = (int64_t)(key & 0xffffffffull);
    }
  }
  return NBX_OK;
fail:
  sc.release(s);
  set_error("nbx_find_singular: %s", cudaGetErrorString(e));
  return NBX_ERR_CUDA;
}
