// Throughput of fixed-point j-force accumulation by L2 atomics vs the
// partial-force stores + gather of the current path (synthetic 96k-like
// sizes: 1.17 M entries of m = 4 atoms over 24.3 k clusters).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_bench red_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

constexpr int M = 4;

// store variant: one float4 per (entry, atom)
__global__ void k_store(const int32_t* ej, int64_t n_ent, float4* part) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t e0 = w * 8; e0 < n_ent; e0 += nw * 8) {
    const int64_t e = e0 + lane / 4;
    if (e < n_ent) part[e * M + (lane & 3)] = make_float4(1.f + lane, 2.f, 3.f, 0.f);
  }
}

// atomic variant: SoA fixed point [3][n_slots], 3 RED.64 per (entry, atom)
__global__ void k_red(const int32_t* ej, int64_t n_ent, int64_t n_slots, unsigned long long* f) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t e0 = w * 8; e0 < n_ent; e0 += nw * 8) {
    const int64_t e = e0 + lane / 4;
    if (e < n_ent) {
      const int64_t s = (int64_t)ej[e] * M + (lane & 3);
      const float fx = 1.f + lane, fy = 2.f, fz = 3.f;
      atomicAdd(f + s, (unsigned long long)__float2ll_rn(fx * 4294967296.f));
      atomicAdd(f + n_slots + s, (unsigned long long)__float2ll_rn(fy * 4294967296.f));
      atomicAdd(f + 2 * n_slots + s, (unsigned long long)__float2ll_rn(fz * 4294967296.f));
    }
  }
}

// atomic variant, AoS-interleaved 32-bit pairs? no: fp32 red.v4 (non-deterministic, for reference)
__global__ void k_redf(const int32_t* ej, int64_t n_ent, float4* f) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t e0 = w * 8; e0 < n_ent; e0 += nw * 8) {
    const int64_t e = e0 + lane / 4;
    if (e < n_ent) {
      const int64_t s = (int64_t)ej[e] * M + (lane & 3);
      atomicAdd(&f[s], make_float4(1.f + lane, 2.f, 3.f, 0.f));
    }
  }
}

int main() {
  const int64_t n_ent = 1170728, n_cl = 24327, n_slots = n_cl * M;
  int32_t* h = (int32_t*)malloc(4 * n_ent);
  srand(1);
  // entries of a group point at nearby clusters; groups are visited in an arbitrary order
  for (int64_t e = 0; e < n_ent; ++e) h[e] = (int32_t)(((e / 183) * 4 + (rand() % 700)) % n_cl);
  int32_t* ej;
  cudaMalloc(&ej, 4 * n_ent);
  cudaMemcpy(ej, h, 4 * n_ent, cudaMemcpyHostToDevice);
  float4* part;
  cudaMalloc(&part, sizeof(float4) * n_ent * M);
  unsigned long long* f;
  cudaMalloc(&f, 8 * 3 * n_slots);
  float4* ff;
  cudaMalloc(&ff, sizeof(float4) * n_slots);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int v = 0; v < 3; ++v) {
    float best = 1e9f;
    for (int rep = 0; rep < 10; ++rep) {
      cudaMemset(f, 0, 8 * 3 * n_slots);
      cudaEventRecord(a);
      if (v == 0) k_store<<<592, 128>>>(ej, n_ent, part);
      else if (v == 1) k_red<<<592, 128>>>(ej, n_ent, n_slots, f);
      else k_redf<<<592, 128>>>(ej, n_ent, ff);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%s: %.1f us\n", v == 0 ? "store float4 partials" : v == 1 ? "RED.64 fixed point x3" : "RED.v4.f32", best * 1e3);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
