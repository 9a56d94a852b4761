// Device helpers shared by the sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "acp_internal.h"

namespace acp {

// Streaming 128-bit global accesses: M and E are touched once per kernel, so
// they bypass L1 retention (ld.global.cs / st.global.cs) and leave L1 to the
// r-column factors, which every row of a layer re-reads.
__device__ __forceinline__ float4 ld_cs4(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void st_cs4(float* p, float4 v) {
  __stcs(reinterpret_cast<float4*>(p), v);
}
// Factor loads: read-only for the whole kernel, L1-cached.
__device__ __forceinline__ float4 ld_f4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float f4dot(float4 a, float4 b) {
  return fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, a.w * b.w)));
}
__device__ __forceinline__ void f4fma(float4& acc, float s, float4 q) {
  acc.x = fmaf(s, q.x, acc.x);
  acc.y = fmaf(s, q.y, acc.y);
  acc.z = fmaf(s, q.z, acc.z);
  acc.w = fmaf(s, q.w, acc.w);
}
__device__ __forceinline__ float4 f4scale(float4 a, float s) {
  return make_float4(a.x * s, a.y * s, a.z * s, a.w * s);
}

// splitmix64 and the counter-based N(0,1) of DESIGN.md "Counter-based
// generator" (the oracle implements the same definition independently).
__device__ __forceinline__ uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t column_key(uint64_t seed, uint64_t tag, uint64_t layer,
                                               uint64_t step, uint64_t col) {
  uint64_t k = sm64(seed);
  k = sm64(k ^ tag);
  k = sm64(k ^ layer);
  k = sm64(k ^ step);
  return sm64(k ^ col);
}
__device__ __forceinline__ float gaussian_at(uint64_t key, uint64_t i) {
  const uint64_t a = sm64(key ^ (2ull * i));
  const uint64_t b = sm64(key ^ (2ull * i + 1ull));
  const double u1 = (double)((a >> 11) + 1ull) * 0x1p-53;
  const double u2 = (double)(b >> 11) * 0x1p-53;
  const double z = sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
  return (float)z;
}

constexpr int kTagQ0 = 1, kTagDegenerate = 2, kTagNoReuse = 3;

}  // namespace acp
