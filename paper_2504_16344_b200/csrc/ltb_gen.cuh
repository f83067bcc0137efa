// ltb_gen.cuh -- counter-based synthetic inputs, keyed by (seed, stream,
// flat index).  Bit-identical to the oracle's orc_gen_* (integer mixing, then
// an exact integer->double conversion and an exact 2u-1), so the GPU can
// generate Cascadia-scale kernels (66 GB time domain) in place while the CPU
// oracle regenerates any shard of them for parity checks.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define LTB_HD __host__ __device__ __forceinline__
#else
#define LTB_HD inline
#endif

namespace ltb {

// stream ids (tensor identities); kernels use LTB tag + 1
enum : uint64_t {
  kStreamKernelF = 1,
  kStreamKernelFq = 2,
  kStreamKernelGstar = 3,
  kStreamKernelGqstar = 4,
  kStreamParam = 10,   // m
  kStreamData = 11,    // d
  kStreamFactor = 0x4C4F,
};

LTB_HD uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

LTB_HD uint64_t gen_key(uint64_t seed, uint64_t stream) {
  return splitmix64(seed ^ splitmix64(stream * 0xD1B54A32D192ED03ull));
}

LTB_HD double gen_uniform_keyed(uint64_t key, uint64_t index) {
  const uint64_t h = splitmix64(key ^ (index * 0xC2B2AE3D27D4EB4Full));
#ifdef __CUDA_ARCH__
  const double u = __dmul_rn(__ull2double_rn(h >> 11), 0x1.0p-53);
  return __dadd_rn(__dmul_rn(2.0, u), -1.0);
#else
  const double u = (double)(h >> 11) * 0x1.0p-53;
  return 2.0 * u - 1.0;
#endif
}

LTB_HD double gen_uniform(uint64_t seed, uint64_t stream, uint64_t index) {
  return gen_uniform_keyed(gen_key(seed, stream), index);
}

// synthetic lower Cholesky factor (oracle orc_gen_factor_entry)
LTB_HD double gen_factor_entry(uint64_t key, int n, double offdiag_scale, int i, int j) {
  if (j > i) return 0.0;
  const double u = gen_uniform_keyed(key, (uint64_t)i * (uint64_t)n + (uint64_t)j);
#ifdef __CUDA_ARCH__
  if (i == j) return __dadd_rn(1.0, __dmul_rn(0.5, __dadd_rn(u, 1.0)));
  return __dmul_rn(u, offdiag_scale);
#else
  if (i == j) return 1.0 + 0.5 * (u + 1.0);
  return u * offdiag_scale;
#endif
}

}  // namespace ltb
