// single-warp and full-GPU throughput of FFMA2 operand patterns
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, long long* cyc, float a, int iters) {
  float2 acc[4], x[4], y[4];
  for (int i = 0; i < 4; ++i) {
    acc[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    x[i] = make_float2(a + i * 1e-3f, a - i * 1e-3f);
    y[i] = make_float2(1e-4f * i, 2e-4f * i);
  }
  const float s = a * 0.5f;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (MODE == 0) acc[i] = __ffma2_rn(x[i], y[i], acc[i]);             // 3 distinct 64-bit regs
        if (MODE == 1) acc[i] = __ffma2_rn(x[i], make_float2(s, s), acc[i]); // broadcast scalar
        if (MODE == 2) acc[i] = __ffma2_rn(acc[i], make_float2(a, a), make_float2(s, s));  // acc*const + const
        if (MODE == 3) { acc[i] = __ffma2_rn(x[i], y[i], acc[i]); x[i] = __ffma2_rn(x[i], make_float2(s, s), y[i]); }
      }
    }
  }
  long long t1 = clock64();
  float t = 0;
  for (int i = 0; i < 4; ++i) t += acc[i].x + acc[i].y + x[i].x + y[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 64 * 4);
  cudaMalloc(&cyc, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"a*b+c (3 regs)", "a*s+c (bcast)", "c*k+k (uniform)", "mix"};
  const int nper[] = {16, 16, 16, 32};
  for (int mode = 0; mode < 4; ++mode) {
    for (int cfg = 0; cfg < 2; ++cfg) {
      const int blocks = cfg == 0 ? 1 : 148 * 16, threads = cfg == 0 ? 32 : 128, iters = cfg == 0 ? 256 : 2048;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<blocks, threads>>>(out, cyc, 0.999f, iters);
        if (mode == 1) k<1><<<blocks, threads>>>(out, cyc, 0.999f, iters);
        if (mode == 2) k<2><<<blocks, threads>>>(out, cyc, 0.999f, iters);
        if (mode == 3) k<3><<<blocks, threads>>>(out, cyc, 0.999f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        if (rep) {
          if (cfg == 0) printf("%-18s 1 warp: %.2f cycles per FFMA2\n", names[mode], (double)c / (iters * nper[mode]));
          else printf("%-18s full GPU: %.1f TFLOP/s\n", names[mode], 4.0 * nper[mode] * (double)iters * blocks * threads / (ms * 1e-3) / 1e12);
        }
      }
    }
  }
  return 0;
}
