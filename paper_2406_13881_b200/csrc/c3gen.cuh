// c3gen.cuh -- configuration C3 synthetic CFG generator.
// Counter-based hashes so the CPU oracle (oracle/mfp_oracle.c) and the GPU
// generate identical inputs without transferring them.
#pragma once
#include <cstdint>

namespace dfx {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t c3_node_key(uint64_t seed, int64_t n) {
  return mix64(mix64(seed ^ 0x243F6A8885A308D3ull) + (uint64_t)n);
}
__host__ __device__ __forceinline__ int c3_is_kernel(uint64_t seed, int64_t n) {
  return (mix64(c3_node_key(seed, n) ^ 0x13198A2E03707344ull) % 5u) == 0u;
}
__host__ __device__ __forceinline__ int c3_n_extra(uint64_t seed, int64_t n) {
  // Poisson(1.5) inverse CDF scaled to 2^32
  const uint64_t cdf[11] = {958336740ull,  2395841851ull, 3473970684ull, 4013035101ull,
                            4215184257ull, 4275829004ull, 4290990191ull, 4294239016ull,
                            4294848171ull, 4294949697ull, 4294964926ull};
  if (n == 0) return 0;
  uint32_t u = (uint32_t)(mix64(c3_node_key(seed, n) ^ 0xA4093822299F31D0ull) >> 32);
  int k = 0;
  while (k < 11 && (uint64_t)u >= cdf[k]) k++;
  return k;
}
__host__ __device__ __forceinline__ int64_t c3_extra_pred(uint64_t seed, int64_t n, int j,
                                                          int64_t n_nodes) {
  uint64_t h = mix64(c3_node_key(seed, n) ^ (0x082EFA98EC4E6C89ull + (uint64_t)j));
  return (int64_t)(h % (uint64_t)n_nodes);
}
__host__ __device__ __forceinline__ void c3_word(uint64_t key, int w, uint32_t& R, uint32_t& W) {
  uint64_t base = mix64(key + 0x452821E638D01377ull * (uint64_t)(w + 1));
  uint64_t r0 = mix64(base + 1), r1 = mix64(base + 2), r2 = mix64(base + 3),
           r3 = mix64(base + 4), r4 = mix64(base + 5);
  uint32_t acc = (uint32_t)r0 & (uint32_t)(r0 >> 32) & (uint32_t)r1 & (uint32_t)(r1 >> 32) &
                 (uint32_t)r2;
  uint32_t u1 = (uint32_t)(r2 >> 32), u2 = (uint32_t)r3, u3 = (uint32_t)(r3 >> 32),
           u4 = (uint32_t)r4;
  uint32_t ronly = acc & u1, rest = acc & ~u1;
  uint32_t wsel = u2 | (u3 & u4);
  uint32_t wonly = rest & wsel, rw = rest & ~wsel;
  R = ronly | rw;
  W = wonly | rw;
}
__host__ __device__ __forceinline__ uint32_t c3_scalar_word(int w, int n_scalar) {
  int lo = w * 32;
  if (n_scalar <= lo) return 0u;
  if (n_scalar >= lo + 32) return 0xFFFFFFFFu;
  return (1u << (n_scalar - lo)) - 1u;
}

}  // namespace dfx
