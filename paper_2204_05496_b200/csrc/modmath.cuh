// Modular arithmetic on 32-bit residues (every q_i, t0, t1 < 2^31) and the
// shared-memory negacyclic NTT used by every kernel.
//
// Bit-exactness: all results are strictly reduced to [0, q), so any correct
// transform reproduces the reference's values exactly. The
// transform conventions follow the reference:
//   * forward: Cooley–Tukey, natural order in, bit-reversed order out,
//     zetas[k] = psi^{bitrev(k)} (proj/src/ring/ntt_tables.cpp:13-41,
//     proj/src/kernels/modops_scalar.cpp:45-63);
//   * inverse: Gentleman–Sande, bit-reversed in, natural out, scaled by n^-1
//     (modops_scalar.cpp:65-81). The n^-1 scaling is folded into the last
//     stage's constants, which is exact mod q.
// Shoup multiplication uses the 32-bit constant floor(w * 2^32 / q), the same
// constant the reference's AVX2 path derives (modops_avx2.cpp:8-11,36-42).
#pragma once
#include <cstdint>

namespace heb {

// x * w mod q with ws = floor(w * 2^32 / q); valid for any x < 2^32, w < q.
__device__ __forceinline__ uint32_t mul_shoup(uint32_t x, uint32_t w, uint32_t ws, uint32_t q) {
  uint32_t qh = __umulhi(x, ws);
  uint32_t r = x * w - qh * q;  // in [0, 2q)
  return min(r, r - q);
}
__device__ __forceinline__ uint32_t add_mod(uint32_t a, uint32_t b, uint32_t q) {
  uint32_t s = a + b;  // a, b < q < 2^31
  return min(s, s - q);
}
__device__ __forceinline__ uint32_t sub_mod(uint32_t a, uint32_t b, uint32_t q) {
  uint32_t d = a - b;
  return min(d, d + q);
}
// a * b mod q for a, b < q < 2^31 without a precomputed Shoup constant:
// Barrett with mu = floor(2^64 / q) (q > 2^1).
__device__ __forceinline__ uint32_t mul_barrett(uint32_t a, uint32_t b, uint32_t q, uint64_t mu) {
  uint64_t p = (uint64_t)a * b;
  uint64_t qh = __umul64hi(p, mu);
  uint64_t r = p - qh * q;  // < 2q (error of the estimate is at most 1)
  return (uint32_t)(r >= q ? r - q : r);
}

// Forward NTT of s[0..n) in shared memory; ends with __syncthreads().
// tw = (zeta, shoup) for this modulus, tw[m + i] used by block i of stage m.
__device__ __forceinline__ void ntt_fwd_smem(uint32_t* s, const uint2* __restrict__ tw, uint32_t q,
                                             uint32_t n, uint32_t logn) {
  const uint32_t half = n >> 1;
  uint32_t logt = logn - 1;
  for (uint32_t m = 1; m < n; m <<= 1, --logt) {
    const uint32_t t = 1u << logt;
    for (uint32_t b = threadIdx.x; b < half; b += blockDim.x) {
      const uint32_t i = b >> logt, j = b & (t - 1);
      const uint32_t x = (i << (logt + 1)) + j;
      const uint2 w = __ldg(&tw[m + i]);
      const uint32_t u = s[x];
      const uint32_t v = mul_shoup(s[x + t], w.x, w.y, q);
      s[x] = add_mod(u, v, q);
      s[x + t] = sub_mod(u, v, q);
    }
    __syncthreads();
  }
}

// Inverse NTT with the final n^-1 scaling fused into the last stage:
// last = (inv_zetas[1] * n^-1, shoup), ninv = (n^-1, shoup). Ends with a sync.
__device__ __forceinline__ void ntt_inv_smem(uint32_t* s, const uint2* __restrict__ itw, uint32_t q,
                                             uint32_t n, uint32_t logn, uint2 last, uint2 ninv) {
  const uint32_t half = n >> 1;
  uint32_t logt = 0;
  for (uint32_t m = half; m > 1; m >>= 1, ++logt) {
    const uint32_t t = 1u << logt;
    for (uint32_t b = threadIdx.x; b < half; b += blockDim.x) {
      const uint32_t i = b >> logt, j = b & (t - 1);
      const uint32_t x = (i << (logt + 1)) + j;
      const uint2 w = __ldg(&itw[m + i]);
      const uint32_t u = s[x], v = s[x + t];
      s[x] = add_mod(u, v, q);
      s[x + t] = mul_shoup(sub_mod(u, v, q), w.x, w.y, q);
    }
    __syncthreads();
  }
  // m = 1, t = n/2: both outputs scaled by n^-1
  for (uint32_t j = threadIdx.x; j < half; j += blockDim.x) {
    const uint32_t u = s[j], v = s[j + half];
    s[j] = mul_shoup(add_mod(u, v, q), ninv.x, ninv.y, q);
    s[j + half] = mul_shoup(sub_mod(u, v, q), last.x, last.y, q);
  }
  __syncthreads();
}

}  // namespace heb
