// Device-side pieces of the MD step around the force pass.
//
//   nbx_max_displacement  oracle.update_drift (oracle.py:106-123): largest
//                         minimum-image displacement |cur - ref| (exact FP64
//                         replay of model.py:159-172 + einsum order; max is
//                         order independent, so the result is bit-identical)
//   nbx_vv_update         the two velocity-Verlet half steps of
//                         engine.velocity_verlet_step (engine.py:543-580):
//                         v += f * (0.5 dt / m); optionally x = wrap(x + v dt)
#include "internal.cuh"

namespace nbx {

__global__ void k_max_disp(const double* __restrict__ ref, const double* __restrict__ cur, int64_t n, Box box,
                           unsigned long long* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double d2 = 0.0;
  if (i < n) {
    const double dx = min_image_np(__dsub_rn(cur[3 * i], ref[3 * i]), box.L[0], box.invL[0]);
    const double dy = min_image_np(__dsub_rn(cur[3 * i + 1], ref[3 * i + 1]), box.L[1], box.invL[1]);
    const double dz = min_image_np(__dsub_rn(cur[3 * i + 2], ref[3 * i + 2]), box.L[2], box.invL[2]);
    d2 = d2_einsum(dx, dy, dz);
  }
  for (int o = 16; o; o >>= 1) d2 = fmax(d2, __shfl_xor_sync(0xffffffffu, d2, o));
  // d2 >= 0: the IEEE bit pattern is monotone as an unsigned integer
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(d2));
}

__global__ void k_vv(double* __restrict__ x, double* __restrict__ v, const double* __restrict__ f,
                     const double* __restrict__ mass, int64_t n, double half_dt, double dt, int move, Box box) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double s = __ddiv_rn(half_dt, mass[i]);  // (0.5 dt) / m  (engine.py:558)
  for (int d = 0; d < 3; ++d) {
    const double vn = __dadd_rn(v[3 * i + d], __dmul_rn(f[3 * i + d], s));
    v[3 * i + d] = vn;
    if (move) x[3 * i + d] = wrap_coord(__dadd_rn(x[3 * i + d], __dmul_rn(vn, dt)), box.L[d]);
  }
}

}  // namespace nbx

using namespace nbx;

extern "C" int nbx_max_displacement(const double* ref, const double* cur, int64_t n, const double box[3],
                                    double* out_d2, void* stream) {
  if ((n > 0 && (!ref || !cur)) || !box || !out_d2) {
    set_error("nbx_max_displacement: null argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  Box bx;
  for (int d = 0; d < 3; ++d) {
    bx.L[d] = box[d];
    bx.invL[d] = 1.0 / box[d];
  }
  cudaError_t e = cudaMemsetAsync(out_d2, 0, sizeof(double), s);
  if (!e && n > 0) {
    count_launch();
    k_max_disp<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ref, cur, n, bx, reinterpret_cast<unsigned long long*>(out_d2));
    e = cudaGetLastError();
  }
  if (e) {
    set_error("nbx_max_displacement: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  return NBX_OK;
}

extern "C" int nbx_vv_update(double* x, double* v, const double* f, const double* mass, int64_t n, double dt,
                             int32_t move, const double box[3], void* stream) {
  if ((n > 0 && (!x || !v || !f || !mass)) || !box) {
    set_error("nbx_vv_update: null argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  Box bx;
  for (int d = 0; d < 3; ++d) {
    bx.L[d] = box[d];
    bx.invL[d] = 1.0 / box[d];
  }
  if (n > 0) {
    count_launch();
    k_vv<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, v, f, mass, n, 0.5 * dt, dt, move, bx);
  }
  cudaError_t e = cudaGetLastError();
  if (e) {
    set_error("nbx_vv_update: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  return NBX_OK;
}
