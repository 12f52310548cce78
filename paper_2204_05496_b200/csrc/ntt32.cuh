// Register-blocked negacyclic NTT with 32 residues per thread, N = 2^LOGN,
// LOGN in {13, 14}; one CTA of T = N/32 threads per polynomial.
//
// Same transform as ntt_fast.cuh (the reference's Cooley-Tukey forward with
// zetas[m + i] = psi^{bitrev(m + i)} and Gentleman-Sande inverse scaled by
// n^-1, proj/src/kernels/modops_scalar.cpp:45-81; every value strictly
// reduced where it feeds an add, so the output is bit-identical), but with
// twice the residues per thread the 13 (14) stages fit three register passes
// with no cross-thread stage:
//
//   pass A  stages 0..4          x = j + T*r                      (r < 32)
//   pass B  stages 5..9          x = blk*T + jj + (T/32)*r, blk = j / (T/32)
//   pass C  stages 10..LOGN-1    x = 32*j + r  (32 contiguous eval slots)
//
// Twiddle of the butterfly on (x, x + N >> (st+1)) at stage st:
// m = 2^st + (x >> (LOGN - st)). Pass A indices are compile-time (< 32); pass
// B reads the natural table (2-4 distinct indices per warp); pass C reads a
// per-thread transposed table (tc32[k * T + j], uint4 = two (w, shoup)).
//
// Shared memory (N words) is swizzled on bits 2..4 with
// h(x) = ((x >> 5) & 7) ^ (((x >> 8) & 3) << 1), conflict-free for all three
// access patterns at both sizes, 16-byte aligned for pass C's 128-bit accesses.
#pragma once
#include "ntt_fast.cuh"

namespace heb {

template <int LOGN>
struct Ntt32 {
  static_assert(LOGN == 13 || LOGN == 14, "Ntt32 covers N = 8192 and 16384");
  static constexpr uint32_t N = 1u << LOGN;
  static constexpr uint32_t T = N / 32;       // threads per polynomial
  static constexpr uint32_t JB = T / 32;      // pass-B threads per block (stride of r)
  static constexpr int NC = LOGN - 10;        // pass-C stages
  // pass-C twiddle entries per thread: sum over stages of 32 >> (LOGN - st)
  static constexpr int EC = (LOGN == 14) ? 30 : 28;
  static constexpr int KC = EC / 2;           // uint4 per thread
  static __device__ __forceinline__ uint32_t sw(uint32_t x) {
    return x ^ ((((x >> 5) & 7u) ^ (((x >> 8) & 3u) << 1)) << 2);
  }
  static __device__ __forceinline__ uint32_t posA(uint32_t j, uint32_t r) { return j + T * r; }
  static __device__ __forceinline__ uint32_t posB(uint32_t j, uint32_t r) {
    return (j / JB) * T + (j % JB) + JB * r;
  }
  static __device__ __forceinline__ uint32_t posC0(uint32_t j) { return 32 * j; }
  // first entry of pass-C stage `s` (0-based within pass C)
  static __device__ __forceinline__ constexpr int cbase(int s) {
    int e = 0;
    for (int k = 0; k < s; ++k) e += 32 >> (LOGN - 10 - k);
    return e;
  }

  static __device__ __forceinline__ void ct(uint32_t& u, uint32_t& v, uint2 w, uint32_t q, bool ru, bool rv) {
    Ntt<LOGN>::ct(u, v, w, q, ru, rv);
  }
  static __device__ __forceinline__ constexpr bool red(int x, int half) { return !(x & (half >> 1)); }

  template <bool LAZY_OUT = false, typename TW = const uint2*>
  static __device__ __forceinline__ void fwd(uint32_t (&e)[32], uint32_t* sm, TW tw, const uint2* __restrict__ twg,
                                             const uint4* __restrict__ tc32, uint32_t q) {
    const uint32_t j = threadIdx.x;
    // ---- pass A: stages 0..4
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const int half = 16 >> s;
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (!(r & half)) ct(e[r], e[r + half], load_tw(tw, (1 << s) + (r >> (5 - s))), q, red(r, half), red(r + half, half));
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 32; ++r) sm[sw(posA(j, r))] = e[r];
    __syncthreads();
    // ---- pass B: stages 5..9
#pragma unroll
    for (int r = 0; r < 32; ++r) e[r] = sm[sw(posB(j, r))];
    {
      const uint32_t blk = j / JB;
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        const int half = 16 >> s;
#pragma unroll
        for (int r = 0; r < 32; ++r)
          if (!(r & half))
            ct(e[r], e[r + half], __ldg(twg + (32u << s) + (blk << s) + (r >> (5 - s))), q, red(r, half),
               red(r + half, half));
      }
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) sm[sw(posB(j, r))] = e[r];
    __syncthreads();
    // ---- pass C: stages 10..LOGN-1 on 32 contiguous slots
    {
      const uint32_t x0 = posC0(j);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 v = *reinterpret_cast<const uint4*>(sm + sw(x0 + 4 * c));
        e[4 * c] = v.x;
        e[4 * c + 1] = v.y;
        e[4 * c + 2] = v.z;
        e[4 * c + 3] = v.w;
      }
    }
    const uint4* tcj = tc32 + j;
#pragma unroll
    for (int s = 0; s < NC; ++s) {
      const int half = 1 << (NC - 1 - s);  // register distance
      const int g = LOGN - 10 - s;         // log2 of the twiddle group size (2 * half)
      const bool last = s == NC - 1;
#pragma unroll
      for (int b = 0; b < (32 >> g); b += 2) {  // two groups share one uint4 of twiddles
        const int ent = cbase(s) + b;
        const uint4 v0 = __ldg(tcj + (ent >> 1) * T);
        const uint4 v1 = (ent & 1) ? __ldg(tcj + ((ent + 1) >> 1) * T) : v0;
        const uint2 w0 = (ent & 1) ? make_uint2(v0.z, v0.w) : make_uint2(v0.x, v0.y);
        const uint2 w1 = (ent & 1) ? make_uint2(v1.x, v1.y) : make_uint2(v0.z, v0.w);
#pragma unroll
        for (int h = 0; h < 2 && b + h < (32 >> g); ++h)
#pragma unroll
          for (int r = (b + h) << g; r < ((b + h) << g) + half; ++r)
            ct(e[r], e[r + half], h ? w1 : w0, q, last ? !LAZY_OUT : red(r, half), last ? !LAZY_OUT : red(r + half, half));
      }
    }
  }

  // Inverse: e in pass-C order (32 contiguous eval slots) -> pass-A order
  // (natural coefficients), scaled by n^-1. Begins and ends with a barrier.
  template <typename TW = const uint2*>
  static __device__ __forceinline__ void inv(uint32_t (&e)[32], uint32_t* sm, TW itw, const uint2* __restrict__ itwg,
                                             const uint4* __restrict__ itc32, uint32_t q, uint2 last, uint2 ninv) {
    const uint32_t j = threadIdx.x;
    {
      const uint4* tcj = itc32 + j;
#pragma unroll
      for (int s = NC - 1; s >= 0; --s) {
        const int half = 1 << (NC - 1 - s);
        const int g = LOGN - 10 - s;
#pragma unroll
        for (int b = 0; b < (32 >> g); b += 2) {
          const int ent = cbase(s) + b;
          const uint4 v0 = __ldg(tcj + (ent >> 1) * T);
          const uint4 v1 = (ent & 1) ? __ldg(tcj + ((ent + 1) >> 1) * T) : v0;
          const uint2 w0 = (ent & 1) ? make_uint2(v0.z, v0.w) : make_uint2(v0.x, v0.y);
          const uint2 w1 = (ent & 1) ? make_uint2(v1.x, v1.y) : make_uint2(v0.z, v0.w);
#pragma unroll
          for (int h = 0; h < 2 && b + h < (32 >> g); ++h)
#pragma unroll
            for (int r = (b + h) << g; r < ((b + h) << g) + half; ++r) Ntt<LOGN>::gs(e[r], e[r + half], h ? w1 : w0, q);
        }
      }
    }
    __syncthreads();
    {
      const uint32_t x0 = posC0(j);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4*>(sm + sw(x0 + 4 * c)) = make_uint4(e[4 * c], e[4 * c + 1], e[4 * c + 2], e[4 * c + 3]);
    }
    __syncthreads();
    // ---- pass B: stages 9..5
#pragma unroll
    for (int r = 0; r < 32; ++r) e[r] = sm[sw(posB(j, r))];
    {
      const uint32_t blk = j / JB;
#pragma unroll
      for (int s = 4; s >= 0; --s) {
        const int half = 16 >> s;
#pragma unroll
        for (int r = 0; r < 32; ++r)
          if (!(r & half)) Ntt<LOGN>::gs(e[r], e[r + half], __ldg(itwg + (32u << s) + (blk << s) + (r >> (5 - s))), q);
      }
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) sm[sw(posB(j, r))] = e[r];
    __syncthreads();
    // ---- pass A: stages 4..1, then stage 0 fused with the n^-1 scaling
#pragma unroll
    for (int r = 0; r < 32; ++r) e[r] = sm[sw(posA(j, r))];
#pragma unroll
    for (int s = 4; s >= 1; --s) {
      const int half = 16 >> s;
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (!(r & half)) Ntt<LOGN>::gs(e[r], e[r + half], load_tw(itw, (1 << s) + (r >> (5 - s))), q);
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t u = e[r], v = e[r + 16];
      e[r] = mul_shoup(u + v, ninv.x, ninv.y, q);
      e[r + 16] = mul_shoup(u - v + q, last.x, last.y, q);
    }
  }
};

}  // namespace heb
