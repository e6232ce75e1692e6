// Throughput ceiling of the force kernel's pair arithmetic on one B200:
// the packed (FFMA2) LJ + Ewald-real-space pair evaluation of k_force_h
// (2 i-atoms x 2 j-atoms per lane per block) in a tight loop with all data in
// registers / broadcast shared memory -- no list, no staging, no stores.
// Reports pairs/s and the fraction of the FP32 peak at 52 flop per pair.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -ftz=true -prec-sqrt=false -o pair_math pair_math.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 bc2(float v) { return make_float2(v, v); }

struct Coef { float rc2, ew_a, s[11]; };
__constant__ Coef C;

__device__ __forceinline__ float admit_r2(float r2, float rc2, uint32_t word, uint32_t bit) {
  float out;
  asm("{\n\t.reg .pred pm, pc;\n\tsetp.ne.b32 pm, %3, 0;\n\tsetp.le.and.ftz.f32 pc, %1, %2, pm;\n\t"
      "selp.f32 %0, %1, 0f7F800000, pc;\n\t}" : "=f"(out) : "f"(r2), "f"(rc2), "r"(word & bit));
  return out;
}

template <int POLY>
__device__ __forceinline__ float2 eval(float2 r2, float2 r2m, float4 zq, float4 l2, float qj) {
  float2 rinv = make_float2(rsqrtf(r2m.x), rsqrtf(r2m.y));
  const float2 rinv2 = __fmul2_rn(rinv, rinv);
  const float2 rinv6 = __fmul2_rn(__fmul2_rn(rinv2, rinv2), rinv2);
  const float2 flj = __fmul2_rn(rinv6, __ffma2_rn(make_float2(l2.z, l2.w), rinv6, make_float2(l2.x, l2.y)));
  const float2 qq = __fmul2_rn(make_float2(zq.z, zq.w), bc2(qj));
  const float2 u = __ffma2_rn(r2, bc2(C.ew_a), bc2(-1.f));
  float2 gs = bc2(C.s[0]);
#pragma unroll
  for (int k = 1; k <= POLY; ++k) gs = __ffma2_rn(gs, u, bc2(C.s[k]));
  const float2 sc = __ffma2_rn(r2, gs, rinv);
  return __fmul2_rn(__ffma2_rn(qq, sc, flj), rinv2);
}

template <int NB, int POLY, int MINB>
__global__ void __launch_bounds__(128, MINB) k(float* out, int iters, uint32_t mask) {
  __shared__ float4 s_xy[8], s_zq[8], s_l[8];
  if (threadIdx.x < 8) {
    s_xy[threadIdx.x] = make_float4(-0.1f * threadIdx.x, -0.2f, 0.3f, -0.1f);
    s_zq[threadIdx.x] = make_float4(0.05f, -0.07f, 0.41f * 138.9f, -0.82f * 138.9f);
    s_l[threadIdx.x] = make_float4(-0.0026f, -0.0026f, 2.6e-6f, 2.6e-6f);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float4 xa = make_float4(0.3f + lane * 0.01f, 0.2f, 0.25f, 0.41f), xb = make_float4(0.1f, 0.35f + lane * 0.01f, 0.2f, -0.82f);
  float2 fi[NB][3], fa[3], fb[3];
  for (int b = 0; b < NB; ++b) fi[b][0] = fi[b][1] = fi[b][2] = bc2(0.f);
  for (int c = 0; c < 3; ++c) fa[c] = fb[c] = bc2(0.f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int h = (2 * b + (lane >> 4)) & 7;
      const float4 xy = s_xy[h], zq = s_zq[h], la = s_l[h], lb = s_l[(h + 1) & 7];
      float2 dxa = __fadd2_rn(make_float2(xy.x, xy.y), bc2(xa.x));
      float2 dya = __fadd2_rn(make_float2(xy.z, xy.w), bc2(xa.y));
      float2 dza = __fadd2_rn(make_float2(zq.x, zq.y), bc2(xa.z));
      float2 dxb = __fadd2_rn(make_float2(xy.x, xy.y), bc2(xb.x));
      float2 dyb = __fadd2_rn(make_float2(xy.z, xy.w), bc2(xb.y));
      float2 dzb = __fadd2_rn(make_float2(zq.x, zq.y), bc2(xb.z));
      const float2 r2a = __ffma2_rn(dxa, dxa, __ffma2_rn(dya, dya, __fmul2_rn(dza, dza)));
      const float2 r2b = __ffma2_rn(dxb, dxb, __ffma2_rn(dyb, dyb, __fmul2_rn(dzb, dzb)));
      const float2 r2ma = make_float2(admit_r2(r2a.x, C.rc2, mask, 1u << (4 * b)), admit_r2(r2a.y, C.rc2, mask, 1u << (4 * b + 1)));
      const float2 r2mb = make_float2(admit_r2(r2b.x, C.rc2, mask, 1u << (4 * b + 2)), admit_r2(r2b.y, C.rc2, mask, 1u << (4 * b + 3)));
      const float2 fsa = eval<POLY>(r2a, r2ma, zq, la, xa.w);
      const float2 fsb = eval<POLY>(r2b, r2mb, zq, lb, xb.w);
      fi[b][0] = __ffma2_rn(fsa, dxa, fi[b][0]); fi[b][1] = __ffma2_rn(fsa, dya, fi[b][1]); fi[b][2] = __ffma2_rn(fsa, dza, fi[b][2]);
      fa[0] = __ffma2_rn(fsa, dxa, fa[0]); fa[1] = __ffma2_rn(fsa, dya, fa[1]); fa[2] = __ffma2_rn(fsa, dza, fa[2]);
      fi[b][0] = __ffma2_rn(fsb, dxb, fi[b][0]); fi[b][1] = __ffma2_rn(fsb, dyb, fi[b][1]); fi[b][2] = __ffma2_rn(fsb, dzb, fi[b][2]);
      fb[0] = __ffma2_rn(fsb, dxb, fb[0]); fb[1] = __ffma2_rn(fsb, dyb, fb[1]); fb[2] = __ffma2_rn(fsb, dzb, fb[2]);
    }
    xa.x += 1e-7f;
    xb.y -= 1e-7f;
  }
  float s = fa[0].x + fa[1].y + fb[2].x + fb[0].y;
  for (int b = 0; b < NB; ++b) s += fi[b][0].x + fi[b][1].y + fi[b][2].x;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NB, int POLY, int MINB>
void run(float* out, int blocks_per_sm) {
  Coef h;
  h.rc2 = 1.0f; h.ew_a = 2.0f; for (int i = 0; i < 11; ++i) h.s[i] = 0.01f * (i + 1);
  cudaMemcpyToSymbol(C, &h, sizeof(h));
  const int iters = 4000, grid = 148 * blocks_per_sm;
  k<NB, POLY, MINB><<<grid, 128>>>(out, 10, 0xffffffffu);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<NB, POLY, MINB><<<grid, 128>>>(out, iters, 0xffffffffu);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaFuncAttributes a; cudaFuncGetAttributes(&a, k<NB, POLY, MINB>);
  const double pairs = (double)grid * 128 * iters * NB * 4;
  const double tf = pairs * 52 / (ms * 1e-3) / 1e12;
  int dev; cudaGetDevice(&dev); int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const double peak = 148.0 * 128 * 2 * 1965e6 / 1e12;
  printf("NB=%d poly=%2d regs=%3d warps/SM=%2d: %.1f Gpairs/s  %.2f TF/s(52/pair)  frac %.3f\n", NB, POLY, a.numRegs,
         blocks_per_sm * 4, pairs / (ms * 1e-3) / 1e9, tf, tf / peak);
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 64 * 128 * 4);
  for (int b : {4, 8, 12, 16}) run<1, 10, 1>(out, b);
  for (int b : {4, 8, 12, 16}) run<2, 10, 1>(out, b);
  for (int b : {4, 8}) run<4, 10, 1>(out, b);
  for (int b : {4, 8, 16}) run<1, 6, 1>(out, b);
  for (int b : {4, 8, 16}) run<2, 6, 1>(out, b);
  return 0;
}
