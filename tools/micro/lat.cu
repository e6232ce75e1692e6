// dependent-chain latency (cycles/instr) of FFMA, FFMA2, FMUL2, MUFU.RSQ, LDS, and
// throughput of a single warp with 2 / 4 independent FFMA2 chains
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, long long* cyc, float a) {
  __shared__ float sm[64];
  sm[threadIdx.x & 63] = a;
  __syncthreads();
  float x = threadIdx.x * 1e-3f + 1.f, y = x + 1.f, z = x + 2.f, w = x + 3.f;
  float2 x2 = make_float2(x, y), y2 = make_float2(z, w), z2 = make_float2(w, x), w2 = make_float2(y, z);
  const float2 a2 = make_float2(a, a);
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 256; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) x = fmaf(x, a, 0.5f);
      if (MODE == 1) x2 = __ffma2_rn(x2, a2, a2);
      if (MODE == 2) x = rsqrtf(x);
      if (MODE == 3) x = sm[__float_as_uint(x) & 63];
      if (MODE == 4) { x2 = __ffma2_rn(x2, a2, a2); y2 = __ffma2_rn(y2, a2, a2); }
      if (MODE == 5) { x2 = __ffma2_rn(x2, a2, a2); y2 = __ffma2_rn(y2, a2, a2); z2 = __ffma2_rn(z2, a2, a2); w2 = __ffma2_rn(w2, a2, a2); }
      if (MODE == 6) { x = fmaf(x, a, 0.5f); y = fmaf(y, a, 0.5f); z = fmaf(z, a, 0.5f); w = fmaf(w, a, 0.5f); }
      if (MODE == 7) x2 = __fmul2_rn(x2, a2);
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x + y + z + w + x2.x + x2.y + y2.x + y2.y + z2.x + z2.y + w2.x + w2.y;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4096);
  cudaMalloc(&cyc, 8);
  const char* names[] = {"FFMA chain", "FFMA2 chain", "MUFU.RSQ chain", "LDS chain", "2x FFMA2 chains", "4x FFMA2 chains", "4x FFMA chains", "FMUL2 chain"};
  const int per[] = {1, 1, 1, 1, 2, 4, 4, 1};
  for (int mode = 0; mode < 8; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (mode) {
        case 0: k<0><<<1, 32>>>(out, cyc, 0.999f); break;
        case 1: k<1><<<1, 32>>>(out, cyc, 0.999f); break;
        case 2: k<2><<<1, 32>>>(out, cyc, 0.999f); break;
        case 3: k<3><<<1, 32>>>(out, cyc, 0.0f); break;
        case 4: k<4><<<1, 32>>>(out, cyc, 0.999f); break;
        case 5: k<5><<<1, 32>>>(out, cyc, 0.999f); break;
        case 6: k<6><<<1, 32>>>(out, cyc, 0.999f); break;
        case 7: k<7><<<1, 32>>>(out, cyc, 0.999f); break;
      }
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      if (rep) printf("%-18s %.2f cycles per instruction (issue-to-issue, 1 warp)\n", names[mode], (double)c / (256 * 16 * per[mode]));
    }
  }
  return 0;
}
