// Shared device helpers for the nbx (nbnxn) sm_100a library.
//
// FP64 decision helpers replay the reference's operation order exactly
// (/root/reference/pkg/src/clustermd: model.py:147-172, gridder.py:165-185,
// pairlist.py:220-239) using explicitly rounded intrinsics, so results do not
// depend on -fmad settings.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

namespace nbx {

constexpr int WARP = 32;

// ------------------------------------------------------------------ errors
void set_error(const char* fmt, ...);
#define NBX_CUDA(call)                                                        \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      ::nbx::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                       cudaGetErrorString(e_));                               \
      return NBX_ERR_CUDA;                                                    \
    }                                                                         \
  } while (0)

// ------------------------------------------------------------------ FP64 geometry
// np.mod(x, L) (npy_divmod: fmod, sign fix, +0 for exact zero) then the
// fold of model.py:156 (out >= L -> out - L).
__device__ __forceinline__ double wrap_coord(double x, double L) {
  double r = fmod(x, L);
  if (r != 0.0) {
    if ((L < 0.0) != (r < 0.0)) r = __dadd_rn(r, L);
  } else {
    r = 0.0;  // copysign(0, L) with L > 0
  }
  if (r >= L) r = __dsub_rn(r, L);
  return r;
}

// floor(dr / L + 0.5), bit-identical to numpy's (IEEE division).  The
// reciprocal product is used unless the rounded argument is within a few ulp
// of an integer, where the exact quotient decides.
__device__ __forceinline__ double image_count(double dr, double L, double invL) {
  double t = __dadd_rn(__dmul_rn(dr, invL), 0.5);
  double k = floor(t);
  double frac = __dsub_rn(t, k);
  double thr = 1e-12 * fmax(1.0, fabs(t));
  if (frac < thr || frac > 1.0 - thr) {
    k = floor(__dadd_rn(__ddiv_rn(dr, L), 0.5));
  }
  return k;
}

// model.py:167-171 minimum_image: dr - floor(dr/L + 0.5)*L, then folds
// (np.where twice: >= half -> -L, then < -half -> +L).
__device__ __forceinline__ double min_image_np(double dr, double L, double invL) {
  double out = __dsub_rn(dr, __dmul_rn(image_count(dr, L, invL), L));
  double half = __dmul_rn(0.5, L);
  if (out >= half) out = __dsub_rn(out, L);
  if (out < -half) out = __dadd_rn(out, L);
  return out;
}

// kernels.py:168-182: same expression with if/elif folds.
__device__ __forceinline__ double min_image_kernel(double d, double L, double invL) {
  d = __dsub_rn(d, __dmul_rn(image_count(d, L, invL), L));
  double half = __dmul_rn(0.5, L);
  if (d >= half) d = __dsub_rn(d, L);
  else if (d < -half) d = __dadd_rn(d, L);
  return d;
}

// gridder.py:177-183 one dimension of the periodic AABB gap.
__device__ __forceinline__ double gap_1d(double lo_i, double hi_i, double lo_j, double hi_j,
                                         double span) {
  double a = __dsub_rn(lo_j, hi_i);
  double b = __dsub_rn(lo_i, hi_j);
  double g0 = fmax(0.0, fmax(a, b));
  double gm = fmax(0.0, fmax(__dsub_rn(a, span), __dadd_rn(b, span)));
  double gp = fmax(0.0, fmax(__dadd_rn(a, span), __dsub_rn(b, span)));
  return fmin(g0, fmin(gm, gp));
}

struct Box {
  double L[3];
  double invL[3];
};

__device__ __forceinline__ double gap_sq(const double* bi, const double* bj, const Box& box) {
  // bboxes: [lo x, lo y, lo z, hi x, hi y, hi z]; ((0 + gx^2) + gy^2) + gz^2
  double s = 0.0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double g = gap_1d(bi[d], bi[3 + d], bj[d], bj[3 + d], box.L[d]);
    s = __dadd_rn(s, __dmul_rn(g, g));
  }
  return s;
}

// numpy einsum("pabd,pabd->pab") order on this numpy: (dx^2 + dz^2) + dy^2
__device__ __forceinline__ double d2_einsum(double dx, double dy, double dz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dz, dz)), __dmul_rn(dy, dy));
}

// numba kernel order (kernels.py:183): (dx^2 + dy^2) + dz^2, no contraction
__device__ __forceinline__ double d2_seq(double dx, double dy, double dz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace nbx
