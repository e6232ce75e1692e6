// CUB-backed device-wide primitives (scan, stable radix sort) used by the
// build/prune bookkeeping.  Temp storage is stream-ordered (recycled through
// the temporaries cache, internal.cuh).
#include <cub/cub.cuh>

#include "internal.cuh"

namespace nbx {

cudaError_t exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  size_t bytes = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)n, s);
  if (e != cudaSuccess) return e;
  DBuf<char> tmp;  // recycled through the temporaries cache
  if ((e = tmp.alloc((int64_t)bytes, s)) != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, (int)n, s);
  tmp.release(s);
  return e;
}

cudaError_t sort_pairs_i32(const int32_t* keys_in, int32_t* keys_out, const int32_t* vals_in,
                           int32_t* vals_out, int64_t n, int end_bit, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  size_t bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys_in, keys_out, vals_in,
                                                  vals_out, (int)n, 0, end_bit, s);
  if (e != cudaSuccess) return e;
  DBuf<char> tmp;
  if ((e = tmp.alloc((int64_t)bytes, s)) != cudaSuccess) return e;
  e = cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys_in, keys_out, vals_in, vals_out, (int)n, 0,
                                      end_bit, s);
  tmp.release(s);
  return e;
}

}  // namespace nbx
