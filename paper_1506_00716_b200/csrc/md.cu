// Device-side pieces of the MD step around the force pass.
//
//   nbx_max_displacement  oracle.update_drift (oracle.py:106-123): largest
//                         minimum-image displacement |cur - ref| (exact FP64
//                         replay of model.py:159-172 + einsum order; max is
//                         order independent, so the result is bit-identical)
//   nbx_vv_update         the two velocity-Verlet half steps of
//                         engine.velocity_verlet_step (engine.py:543-580):
//                         v += f * (0.5 dt / m); optionally x = wrap(x + v dt)
//   nbx_settle            rigid 3-site water (extension; the
//                         reference has no constraints): analytic SETTLE of
//                         the drifted positions (Miyamoto & Kollman 1992) with
//                         the matching velocity correction, and RATTLE's
//                         velocity stage after the second half kick
//                         (oracle/constraints.py restates both in numpy and
//                         checks SETTLE against iterated SHAKE)
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

// one-launch variant: block maxima into scratch[0], the last block (ticket
// in scratch[1]) writes the result -- sqrt'ed when asked -- and re-zeroes the
// scratch for the next call (no memset, no separate sqrt kernel)
__global__ void k_max_disp_once(const double* __restrict__ ref, const double* __restrict__ cur, int64_t n, Box box,
                                unsigned long long* __restrict__ scratch, double* __restrict__ out, int take_sqrt) {
  __shared__ double s_max[8];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double d2 = 0.0;
  if (i < n) {
    const double dx = min_image_np(__dsub_rn(cur[3 * i], ref[3 * i]), box.L[0], box.invL[0]);
    const double dy = min_image_np(__dsub_rn(cur[3 * i + 1], ref[3 * i + 1]), box.L[1], box.invL[1]);
    const double dz = min_image_np(__dsub_rn(cur[3 * i + 2], ref[3 * i + 2]), box.L[2], box.invL[2]);
    d2 = d2_einsum(dx, dy, dz);
  }
  for (int o = 16; o; o >>= 1) d2 = fmax(d2, __shfl_xor_sync(0xffffffffu, d2, o));
  if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = d2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = s_max[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) b = fmax(b, s_max[w]);
    // d2 >= 0: the IEEE bit pattern is monotone as an unsigned integer
    atomicMax(scratch, (unsigned long long)__double_as_longlong(b));
    __threadfence();
    const unsigned long long t = atomicAdd(scratch + 1, 1ull);
    if (t == gridDim.x - 1) {  // every block's maximum is in
      const double m = __longlong_as_double((long long)atomicExch(scratch, 0ull));
      *out = take_sqrt ? sqrt(m) : m;
      scratch[1] = 0ull;
    }
  }
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


// ---------------------------------------------------------------- SETTLE
// molecule k = atoms (3k, 3k+1, 3k+2) = (O, H1, H2); per-atom wrapped
// positions, so every intramolecular vector is a minimum image.
struct Settle {
  double mO, mH, wohh, ra, rb, rc, inv_dt;
};

__device__ __forceinline__ void mi3(const double* a, const double* b, const Box& box, double* out) {
  for (int d = 0; d < 3; ++d) {
    double r = a[d] - b[d];
    r -= box.L[d] * rint(r * box.invL[d]);
    out[d] = r;
  }
}
__device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}
__device__ __forceinline__ double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

// positions: x_old constrained (previous step), x drifted (unconstrained) ->
// x constrained (wrapped), v += displacement / dt
__device__ __forceinline__ void settle_mol(const double* A0, double* X, double* V, const Settle& P, const Box& box) {
  double b0[3], c0[3], B1[3], C1[3];
  mi3(A0 + 3, A0, box, b0);
  mi3(A0 + 6, A0, box, c0);
  mi3(X + 3, X, box, B1);
  mi3(X + 6, X, box, C1);
  double com[3], a1[3], b1[3], c1[3];
  for (int d = 0; d < 3; ++d) {
    com[d] = (P.mH * B1[d] + P.mH * C1[d]) / P.wohh;
    a1[d] = -com[d];
    b1[d] = B1[d] - com[d];
    c1[d] = C1[d] - com[d];
  }
  double n[3], ex[3], ey[3];
  cross3(b0, c0, n);
  cross3(a1, n, ex);
  cross3(n, ex, ey);
  const double ix = rsqrt(dot3(ex, ex)), iy = rsqrt(dot3(ey, ey)), iz = rsqrt(dot3(n, n));
  for (int d = 0; d < 3; ++d) {
    ex[d] *= ix;
    ey[d] *= iy;
    n[d] *= iz;
  }
  const double xb0d = dot3(b0, ex), yb0d = dot3(b0, ey);
  const double xc0d = dot3(c0, ex), yc0d = dot3(c0, ey);
  const double za1d = dot3(a1, n);
  const double xb1d = dot3(b1, ex), yb1d = dot3(b1, ey), zb1d = dot3(b1, n);
  const double xc1d = dot3(c1, ex), yc1d = dot3(c1, ey), zc1d = dot3(c1, n);
  const double sinphi = za1d / P.ra;
  const double cosphi = sqrt(1.0 - sinphi * sinphi);
  const double sinpsi = (zb1d - zc1d) / (2.0 * P.rc * cosphi);
  const double cospsi = sqrt(1.0 - sinpsi * sinpsi);
  const double ya2d = P.ra * cosphi, xb2d = -P.rc * cospsi;
  const double t1 = -P.rb * cosphi, t2 = P.rc * sinpsi * sinphi;
  const double yb2d = t1 - t2, yc2d = t1 + t2;
  const double alpha = xb2d * (xb0d - xc0d) + yb0d * yb2d + yc0d * yc2d;
  const double beta = xb2d * (yc0d - yb0d) + xb0d * yb2d + xc0d * yc2d;
  const double gamma = xb0d * yb1d - xb1d * yb0d + xc0d * yc1d - xc1d * yc0d;
  const double al2be2 = alpha * alpha + beta * beta;
  const double sinth = (alpha * gamma - beta * sqrt(al2be2 - gamma * gamma)) / al2be2;
  const double costh = sqrt(1.0 - sinth * sinth);
  const double a3[3] = {-ya2d * sinth, ya2d * costh, za1d};
  const double b3[3] = {xb2d * costh - yb2d * sinth, xb2d * sinth + yb2d * costh, zb1d};
  const double c3[3] = {-xb2d * costh - yc2d * sinth, -xb2d * sinth + yc2d * costh, zc1d};
  const double* loc[3] = {a3, b3, c3};
  const double* rel1[3] = {nullptr, B1, C1};
  for (int a = 0; a < 3; ++a) {
    for (int d = 0; d < 3; ++d) {
      const double r = com[d] + loc[a][0] * ex[d] + loc[a][1] * ey[d] + loc[a][2] * n[d];
      const double disp = r - (a ? rel1[a][d] : 0.0);
      V[3 * a + d] += disp * P.inv_dt;
      X[3 * a + d] = wrap_coord(X[3 * a + d] + disp, box.L[d]);
    }
  }
}

__global__ void k_settle(const double* __restrict__ x_old, double* __restrict__ x, double* __restrict__ v,
                         int64_t n_mol, Settle P, Box box) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n_mol) return;
  settle_mol(x_old + 9 * k, x + 9 * k, v + 9 * k, P, box);
}

// RATTLE velocity stage: r_b . (v_j - v_i) = 0 for the bonds (O,H1), (O,H2),
// (H1,H2); corrections v_i += l_b r_b / m_i, v_j -= l_b r_b / m_j with the
// multipliers from the 3x3 system (Cramer's rule)
__device__ __forceinline__ void rattle_mol(const double* X, double* V, const Settle& P, const Box& box) {
  const int bi[3] = {0, 0, 1}, bj[3] = {1, 2, 2};
  const double m[3] = {P.mO, P.mH, P.mH};
  double r[3][3];
  for (int b = 0; b < 3; ++b) mi3(X + 3 * bj[b], X + 3 * bi[b], box, r[b]);
  double A[3][3], rhs[3];
  for (int c = 0; c < 3; ++c) {
    double dv[3];
    for (int d = 0; d < 3; ++d) dv[d] = V[3 * bj[c] + d] - V[3 * bi[c] + d];
    rhs[c] = -dot3(r[c], dv);
    for (int b = 0; b < 3; ++b) {
      double coef = 0.0;
      if (bj[b] == bj[c]) coef -= 1.0 / m[bj[b]];
      if (bi[b] == bj[c]) coef += 1.0 / m[bi[b]];
      if (bj[b] == bi[c]) coef += 1.0 / m[bj[b]];
      if (bi[b] == bi[c]) coef -= 1.0 / m[bi[b]];
      A[c][b] = coef * dot3(r[c], r[b]);
    }
  }
  const double det = A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) -
                     A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
                     A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
  double lam[3];
  for (int c = 0; c < 3; ++c) {
    double M[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) M[i][j] = (j == c) ? rhs[i] : A[i][j];
    lam[c] = (M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) - M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
              M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0])) / det;
  }
  for (int b = 0; b < 3; ++b)
    for (int d = 0; d < 3; ++d) {
      V[3 * bi[b] + d] += lam[b] / m[bi[b]] * r[b][d];
      V[3 * bj[b] + d] -= lam[b] / m[bj[b]] * r[b][d];
    }
}

__global__ void k_rattle_v(const double* __restrict__ x, double* __restrict__ v, int64_t n_mol, Settle P, Box box) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n_mol) return;
  rattle_mol(x + 9 * k, v + 9 * k, P, box);
}

// One rigid-water molecule per thread, the velocity-Verlet halves fused with
// their constraint (k_vv's arithmetic, op for op, then k_settle / k_rattle_v):
// phase 0 -- half kick, drift + wrap, SETTLE against the pre-drift positions
// (kept in registers: no x_old copy); phase 1 -- half kick, RATTLE.
__global__ void k_vv_constrained(double* __restrict__ x, double* __restrict__ v, const double* __restrict__ f,
                                 const double* __restrict__ mass, int64_t n_mol, double half_dt, double dt,
                                 int phase, Settle P, Box box) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n_mol) return;
  double* X = x + 9 * k;
  double* V = v + 9 * k;
  double A0[9];
  for (int a = 0; a < 3; ++a) {
    const int64_t i = 3 * k + a;
    const double s = __ddiv_rn(half_dt, mass[i]);  // (0.5 dt) / m  (engine.py:558)
    for (int d = 0; d < 3; ++d) {
      const double vn = __dadd_rn(V[3 * a + d], __dmul_rn(f[3 * i + d], s));
      V[3 * a + d] = vn;
      if (phase == 0) {
        A0[3 * a + d] = X[3 * a + d];
        X[3 * a + d] = wrap_coord(__dadd_rn(X[3 * a + d], __dmul_rn(vn, dt)), box.L[d]);
      }
    }
  }
  if (phase == 0) settle_mol(A0, X, V, P, box);
  else rattle_mol(X, V, P, box);
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

extern "C" int nbx_max_displacement_ex(const double* ref, const double* cur, int64_t n, const double box[3],
                                       uint64_t* scratch, double* out, int32_t flags, void* stream) {
  if ((n > 0 && (!ref || !cur)) || !box || !out || !scratch) {
    set_error("nbx_max_displacement_ex: null argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  if (n == 0) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), s);
    if (e) {
      set_error("nbx_max_displacement_ex: %s", cudaGetErrorString(e));
      return NBX_ERR_CUDA;
    }
    return NBX_OK;
  }
  Box bx;
  for (int d = 0; d < 3; ++d) {
    bx.L[d] = box[d];
    bx.invL[d] = 1.0 / box[d];
  }
  count_launch();
  k_max_disp_once<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ref, cur, n, bx,
                                                              reinterpret_cast<unsigned long long*>(scratch), out,
                                                              flags & 1);
  if (cudaError_t e = cudaGetLastError()) {
    set_error("nbx_max_displacement_ex: %s", cudaGetErrorString(e));
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

static Settle make_settle(double m_o, double m_h, double d_oh, double d_hh, double dt, bool positions) {
  Settle P;
  P.mO = m_o;
  P.mH = m_h;
  P.wohh = m_o + 2.0 * m_h;
  P.rc = 0.5 * d_hh;
  const double h = sqrt(d_oh * d_oh - P.rc * P.rc);
  P.ra = 2.0 * m_h * h / P.wohh;
  P.rb = h - P.ra;
  P.inv_dt = positions ? 1.0 / dt : 0.0;
  return P;
}

extern "C" int nbx_vv_constrained(double* x, double* v, const double* f, const double* mass, int64_t n_mol,
                                  double m_o, double m_h, double d_oh, double d_hh, double dt, int32_t phase,
                                  const double box[3], void* stream) {
  if ((n_mol > 0 && (!x || !v || !f || !mass)) || !box || !(m_o > 0.0) || !(m_h > 0.0) || !(d_hh > 0.0) ||
      !(d_oh > 0.5 * d_hh) || !(dt > 0.0) || phase < 0 || phase > 1) {
    set_error("nbx_vv_constrained: bad argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  Box bx;
  for (int d = 0; d < 3; ++d) {
    bx.L[d] = box[d];
    bx.invL[d] = 1.0 / box[d];
  }
  const Settle P = make_settle(m_o, m_h, d_oh, d_hh, dt, phase == 0);
  if (n_mol > 0) {
    count_launch();
    k_vv_constrained<<<(unsigned)((n_mol + 127) / 128), 128, 0, s>>>(x, v, f, mass, n_mol, 0.5 * dt, dt, phase, P,
                                                                     bx);
  }
  if (cudaError_t e = cudaGetLastError()) {
    set_error("nbx_vv_constrained: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  return NBX_OK;
}

extern "C" int nbx_settle(const double* x_old, double* x, double* v, int64_t n_mol, double m_o, double m_h,
                          double d_oh, double d_hh, double dt, int32_t mode, const double box[3], void* stream) {
  if ((n_mol > 0 && (!x || !v || (mode == 0 && !x_old))) || !box || !(m_o > 0.0) || !(m_h > 0.0) ||
      !(d_hh > 0.0) || !(d_oh > 0.5 * d_hh) || (mode == 0 && !(dt > 0.0)) || mode < 0 || mode > 1) {
    set_error("nbx_settle: bad argument");
    return NBX_ERR_PARAM;
  }
  cudaStream_t s = to_stream(stream);
  Box bx;
  for (int d = 0; d < 3; ++d) {
    bx.L[d] = box[d];
    bx.invL[d] = 1.0 / box[d];
  }
  const Settle P = make_settle(m_o, m_h, d_oh, d_hh, dt, mode == 0);
  if (n_mol > 0) {
    count_launch();
    if (mode == 0)
      k_settle<<<(unsigned)((n_mol + 127) / 128), 128, 0, s>>>(x_old, x, v, n_mol, P, bx);
    else
      k_rattle_v<<<(unsigned)((n_mol + 127) / 128), 128, 0, s>>>(x, v, n_mol, P, bx);
  }
  cudaError_t e = cudaGetLastError();
  if (e) {
    set_error("nbx_settle: %s", cudaGetErrorString(e));
    return NBX_ERR_CUDA;
  }
  return NBX_OK;
}
