// FP32 issue/throughput microbenchmark: FFMA (3-reg), FFMA (imm), FFMA2.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, float a, float b, int iters) {
  float x[16];
  float2 y[8];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int i = 0; i < 8; ++i) y[i] = make_float2(x[2 * i], x[2 * i + 1]);
  const float2 a2 = make_float2(a, b), b2 = make_float2(b, a);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) x[i] = fmaf(x[i], a, b);            // 3-reg (a, b in regs)
      if (MODE == 1) x[i] = fmaf(x[i], 0.999f, 1e-4f);   // imm form
      if (MODE == 2 && i < 8) y[i] = __ffma2_rn(y[i], a2, b2);
      if (MODE == 4) x[i] = fmaf(x[i], x[(i + 5) & 15], x[(i + 9) & 15]);
      if (MODE == 3 && i < 8) y[i] = __ffma2_rn(y[i], a2, y[(i + 1) & 7]);
    }
  }
  float s = 0;
  for (int i = 0; i < 16; ++i) s += x[i];
  for (int i = 0; i < 8; ++i) s += y[i].x + y[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 64 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096, blocks = 148 * 8, threads = 256;
  for (int mode = 0; mode < 5; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(out, 0.999f, 1e-4f, iters);
      if (mode == 1) k<1><<<blocks, threads>>>(out, 0.999f, 1e-4f, iters);
      if (mode == 2) k<2><<<blocks, threads>>>(out, 0.999f, 1e-4f, iters);
      if (mode == 4) k<4><<<blocks, threads>>>(out, 0.999f, 1e-4f, iters);
      if (mode == 3) k<3><<<blocks, threads>>>(out, 0.999f, 1e-4f, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16 * (double)iters * blocks * threads;
      if (rep) printf("mode %d (%s): %.1f TFLOP/s\n", mode, mode == 0 ? "FFMA 3-reg" : mode == 1 ? "FFMA imm" : mode == 2 ? "FFMA2 const" : mode == 3 ? "FFMA2 3-reg" : "FFMA 3-reg true",
                      flops / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
