// Register-blocked negacyclic NTT for N = 2^LOGN, LOGN in {12, 13, 14}.
//
// One CTA of T = N/16 threads transforms one polynomial; every thread keeps
// 16 residues in registers for the whole transform and the 13 (14) radix-2
// stages run as three register passes with two shared-memory exchanges (the
// A <-> B exchange spans the CTA; for LOGN <= 13 the B <-> C exchange stays
// inside each warp and needs only a warp barrier):
//
//   pass A  stages 0..3          thread j holds x = j + T*r          (r < 16)
//   pass B  stages 4..7          x = blk*(N/16) + jj + (N/256)*r
//   pass C  stages 8..LOGN-1     x = grp*G + 16*h + r, G = N/256; the first
//                                LOGN-12 stages of pass C pair threads and
//                                exchange through warp shuffles.
//
// The forward transform consumes pass-A order (natural coefficients, which
// coalesce in global memory) and leaves pass-C order (16 contiguous eval
// slots per thread); the inverse does the reverse. Shared memory is swizzled
// (x ^ (((x >> 5) & 7) << 2)) so all three access patterns are free of bank
// conflicts and pass C can use 128-bit accesses.
//
// The butterflies are the reference's (modops_scalar.cpp:45-81): forward
// Cooley–Tukey with zetas[m + i] = psi^{bitrev(m + i)}, inverse
// Gentleman–Sande with inv_zetas and a final n^-1 scaling folded into the
// last stage. Values stay congruent mod q throughout (lazy ones, < 2q, only
// ever feed a Shoup product) and the outputs are strictly reduced unless the
// caller asks for lazy ones, so results are bit-identical.
#pragma once
#include "modmath.cuh"

namespace heb {

__device__ __forceinline__ uint32_t swz(uint32_t x) { return x ^ (((x >> 5) & 7u) << 2); }

// Twiddle sources for passes A/B (indices 1..255): read-only global loads,
// or a table passed in the kernel's parameter space (constant bank), which
// keeps these warp-uniform reads off the L1 data pipe.
__device__ __forceinline__ uint2 load_tw(const uint2* __restrict__ p, uint32_t i) { return __ldg(p + i); }
struct ParamTw {
  const uint2* p;
};
__device__ __forceinline__ uint2 load_tw(ParamTw t, uint32_t i) { return t.p[i]; }

// NG > 1: the CTA holds NG independent thread groups of T threads, each
// transforming its own polynomial in its own shared buffer; the group
// barriers are named barriers 1..NG (barrier 0 stays __syncthreads).
template <int LOGN, int NG = 1>
struct Ntt {
  static constexpr uint32_t N = 1u << LOGN;
  static constexpr uint32_t T = N / 16;          // threads per polynomial
  static_assert(T >= 256, "pass-A addressing assumes the swizzle bits (2..7) lie inside j < T");
  static __device__ __forceinline__ uint32_t tid() { return NG == 1 ? threadIdx.x : threadIdx.x % T; }
  static __device__ __forceinline__ void sync() {
    if constexpr (NG == 1)
      __syncthreads();
    else
      asm volatile("bar.sync %0, %1;" ::"r"(1 + threadIdx.x / T), "r"(T) : "memory");
  }
  // The pass-B <-> pass-C exchange: for LOGN <= 13 pass B's 512-element block
  // (blk = j >> (LOGN - 8)) and pass C's slots (posC0) of a warp are the same
  // 512 words, so only the warp's own lanes meet there and a warp barrier
  // orders them (one CTA barrier fewer per transform). At LOGN = 14 two warps
  // share a pass-B block.
  static __device__ __forceinline__ void sync_bc() {
    if constexpr (LOGN <= 13)
      __syncwarp();
    else
      sync();
  }
  static constexpr uint32_t G = N >> 8;          // pass-C block size
  static constexpr uint32_t TPG = G / 16;        // threads per pass-C block
  static constexpr int XST = LOGN - 12;          // cross-thread stages in pass C
  // Pass-C twiddles are stored per thread, transposed for coalescing:
  // tc[k * T + j] (uint4 = two (w, shoup) entries). Entry order:
  // [pad][cross stages 0..XST-1][stage s0 (1)][s1 (2)][s2 (4)][s3 (8)],
  // with one pad entry when XST is even so every s>=1 group starts even.
  static constexpr int PAD = (XST % 2 == 0) ? 1 : 0;
  static constexpr int B0 = PAD + XST;           // entry of register stage 0
  static constexpr int KC = (PAD + XST + 15 + 1) / 2;  // uint4 per thread
  static __device__ __forceinline__ uint2 lo(uint4 v) { return make_uint2(v.x, v.y); }
  static __device__ __forceinline__ uint2 hi(uint4 v) { return make_uint2(v.z, v.w); }
  static __device__ __forceinline__ uint2 entry(const uint4* __restrict__ tc, int e) {
    const uint4 v = __ldg(tc + (e >> 1) * T);
    return (e & 1) ? hi(v) : lo(v);
  }

  // pass-A position of register r
  static __device__ __forceinline__ uint32_t posA(uint32_t j, uint32_t r) { return j + T * r; }
  // pass-B position
  static __device__ __forceinline__ uint32_t posB(uint32_t j, uint32_t r) {
    const uint32_t blk = j >> (LOGN - 8), jj = j & ((N >> 8) - 1);
    return blk * (N / 16) + jj + (N >> 8) * r;
  }
  // pass-C position (first of the 16 contiguous slots)
  static __device__ __forceinline__ uint32_t posC0(uint32_t j) {
    const uint32_t grp = j / TPG, h = j % TPG;
    return grp * G + 16 * h;
  }

  // Cooley-Tukey butterfly with lazy outputs: u must be reduced (< q), v may
  // be lazy (< 2q; Shoup accepts any x < 2^32). Each output is reduced only
  // if the next stage uses it as a `u` (ru / rv); a lazy value is < 2q < 2^32.
  // Every value stays congruent to the reference's, and each stage that
  // feeds an add sees reduced operands, so the final result is identical.
  static __device__ __forceinline__ void ct(uint32_t& u, uint32_t& v, uint2 w, uint32_t q, bool ru = true,
                                            bool rv = true) {
    const uint32_t t = mul_shoup(v, w.x, w.y, q);  // [0, q)
    uint32_t a = u + t, b = u - t + q;             // [0, 2q), (0, 2q)
    if (ru) a = min(a, a - q);
    if (rv) b = min(b, b - q);
    u = a;
    v = b;
  }
  // Gentleman-Sande: the difference feeds Shoup unreduced (u - v + q < 2q).
  static __device__ __forceinline__ void gs(uint32_t& u, uint32_t& v, uint2 w, uint32_t q) {
    const uint32_t d = u - v + q;
    u = add_mod(u, v, q);
    v = mul_shoup(d, w.x, w.y, q);
  }
  // reduce output x of a stage whose butterfly half-distance is `half` iff
  // the next stage (half / 2) uses it as the reduced operand u.
  static __device__ __forceinline__ constexpr bool red(int x, int half) { return !(x & (half >> 1)); }

  static __device__ __forceinline__ void store_pos(uint32_t* sm, uint32_t x, uint32_t v) { sm[swz(x)] = v; }
  static __device__ __forceinline__ void storeC(uint32_t* sm, uint32_t j, const uint32_t (&e)[16]) {
    const uint32_t x0 = posC0(j);
#pragma unroll
    for (int c = 0; c < 4; ++c)
      *reinterpret_cast<uint4*>(sm + swz(x0 + 4 * c)) = make_uint4(e[4 * c], e[4 * c + 1], e[4 * c + 2], e[4 * c + 3]);
  }
  static __device__ __forceinline__ void loadC(const uint32_t* sm, uint32_t j, uint32_t (&e)[16]) {
    const uint32_t x0 = posC0(j);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 v = *reinterpret_cast<const uint4*>(sm + swz(x0 + 4 * c));
      e[4 * c] = v.x;
      e[4 * c + 1] = v.y;
      e[4 * c + 2] = v.z;
      e[4 * c + 3] = v.w;
    }
  }

  // ---- The one cross-thread stage of LOGN = 13 (stage 8, butterflies x,
  // x + 16 inside each 32-word group) as its own warp-local pass through
  // shared memory instead of shuffles. A warp's pass-B block is 16 groups of
  // 32 words; lane (quarter qd, gi, hh) takes group g = 2 gi + (qd & 1) +
  // 8 (qd >> 1) and the 4-word chunks hh, hh + 2 of its first half (u) with
  // their partners 16 words up (v): eight butterflies per lane, four of them
  // (the chunk with offset bit 3 clear) feeding the next stage's `u` operands.
  // With the swizzle (chunk ^ (g & 7)) the eight lanes of a quarter-warp hit
  // eight distinct 16-byte bank groups in each 128-bit access.
  static __device__ __forceinline__ uint32_t x8_base(uint32_t j) {
    const uint32_t lane = j & 31u, qd = lane >> 3, gi = (lane >> 1) & 3u, hh = lane & 1u;
    const uint32_t g = 2 * gi + (qd & 1u) + 8 * (qd >> 1);
    // word offset of chunk hh of group g in the warp's block, swizzled ((x >> 5) & 7 = g & 7 for every word of the group)
    return (j & ~31u) * 16 + 32 * g + ((4 * hh) ^ ((g & 7u) << 2));
  }
  static __device__ __forceinline__ uint32_t x8_group(uint32_t j) {
    const uint32_t lane = j & 31u, qd = lane >> 3, gi = (lane >> 1) & 3u;
    return (j >> 5) * 16 + 2 * gi + (qd & 1u) + 8 * (qd >> 1);
  }
  // chunk c of the lane: c = 0, 1 -> u chunks hh, hh + 2; c = 2, 3 -> their v partners (+16 words).
  // (swizzled base ^ 8 flips chunk bit 1: chunk hh -> hh + 2; ^ 16 flips bit 2: +16 words)
  static __device__ __forceinline__ uint4* x8_ptr(uint32_t* sm, uint32_t b, int c) {
    return reinterpret_cast<uint4*>(sm + (b ^ ((c & 1) ? 8u : 0u) ^ ((c & 2) ? 16u : 0u)));
  }

  // Forward: e in pass-A order -> e in pass-C order. Begins and ends with a
  // barrier on the shared buffer (sm: N words).
  // LAZY_OUT: leave the final stage's outputs in [0, 2q) (for consumers that
  // only feed them to a Shoup multiply).
  // LEAD_SYNC = false: the caller guarantees no thread still reads `sm`
  // (e.g. consecutive transforms alternate between two buffers, so the
  // previous reader of this one has since passed two barriers).
  // X8_SMEM (LOGN = 13): the cross-thread stage runs as its own warp-local
  // pass through shared memory (x8_base) instead of the half-exchange
  // shuffles: ~50 fewer instructions per transform, one more shared-memory
  // round trip. Pays in the throughput kernels (C4 key switch 3.908 -> 3.855
  // ms); the latency kernels and the inverse keep the shuffles (the round
  // trip is on their critical path: C3 0.550 -> 0.567 ms, digits 0.652 ->
  // 0.666 ms when tried).
  template <bool LAZY_OUT = false, typename TW = const uint2*, bool LEAD_SYNC = true, bool X8_SMEM = false>
  static __device__ __forceinline__ void fwd(uint32_t (&e)[16], uint32_t* sm, TW tw, const uint4* __restrict__ twc,
                                             uint32_t q) {
    const uint32_t j = tid();
    // ---- pass A: stages 0..3
    // (the last stage's outputs stay lazy: pass B knows which of them it uses
    // as `u` operands and reduces only those, 8 instead of 16)
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int half = 8 >> s;
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (!(r & half))
          ct(e[r], e[r + half], load_tw(tw, (1 << s) + (r >> (4 - s))), q, s < 3 && red(r, half),
             s < 3 && red(r + half, half));
    }
    if constexpr (LEAD_SYNC) sync();
    {
      // swz only reads bits 5..7 and flips bits 2..4, all inside j < T, so
      // swz(j + T*r) = swz(j) + T*r: one base register, immediate offsets
      uint32_t* pa = sm + swz(j);
#pragma unroll
      for (int r = 0; r < 16; ++r) pa[T * r] = e[r];
    }
    sync();
    // ---- pass B: stages 4..7
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t v = sm[swz(posB(j, r))];
      e[r] = r < 8 ? min(v, v - q) : v;  // lazy pass-A outputs: stage 4's u operands are r < 8
    }
    {
      const uint32_t blk = j >> (LOGN - 8);
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int half = 8 >> s;
#pragma unroll
        for (int r = 0; r < 16; ++r)
          if (!(r & half))
            ct(e[r], e[r + half], load_tw(tw, (16u << s) + (blk << s) + (r >> (4 - s))), q, red(r, half), red(r + half, half));
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) sm[swz(posB(j, r))] = e[r];
    sync_bc();
    const uint32_t x0 = posC0(j);
    const uint4* tc = twc + j;
    constexpr bool X8 = X8_SMEM && XST == 1;
    if constexpr (X8) {
      // ---- stage 8 in its own layout (see x8_base), then back through shared memory
      const uint32_t b8 = x8_base(j);
      const uint2 w = lo(__ldg(twc + 2 * x8_group(j)));  // zetas[256 + group]
      uint4 u0 = *x8_ptr(sm, b8, 0), u1 = *x8_ptr(sm, b8, 1), v0 = *x8_ptr(sm, b8, 2), v1 = *x8_ptr(sm, b8, 3);
      // chunk hh (offset bit 3 clear): the next stage's u operands -> reduced; chunk hh + 2: its v operands -> lazy
      ct(u0.x, v0.x, w, q, true, true);
      ct(u0.y, v0.y, w, q, true, true);
      ct(u0.z, v0.z, w, q, true, true);
      ct(u0.w, v0.w, w, q, true, true);
      ct(u1.x, v1.x, w, q, false, false);
      ct(u1.y, v1.y, w, q, false, false);
      ct(u1.z, v1.z, w, q, false, false);
      ct(u1.w, v1.w, w, q, false, false);
      *x8_ptr(sm, b8, 0) = u0;
      *x8_ptr(sm, b8, 1) = u1;
      *x8_ptr(sm, b8, 2) = v0;
      *x8_ptr(sm, b8, 3) = v1;
      __syncwarp();
    }
    // ---- pass C: stages 8..LOGN-1
    loadC(sm, j, e);
#pragma unroll
    for (int s = 0; s < (X8 ? 0 : XST); ++s) {
      // stage st = 8 + s, t = G >> (s + 1) >= 16: partner thread h ^ (t / 16)
      const uint32_t t = G >> (s + 1);
      const uint32_t lanebit = t / 16;
      const bool upper = (x0 & t) != 0;
      const uint2 w = entry(tc, PAD + s);
      // Half exchange: each thread of a pair does 8 of the 16 butterflies
      // locally, then the outputs that belong to the partner go back (16
      // shuffles, no redundant products). Butterfly k leaves a_k in the lower
      // thread's e[k] and b_k in the upper's; the next stage pairs e[k] with
      // e[k + 8], so only butterflies k < 8 need reduced outputs when a
      // register stage follows. The lower thread takes k = 0..3, 8..11 and the
      // upper k + 4, so each issues the reductions for just four butterflies.
      const bool more = s + 1 < XST;  // another cross stage follows: reduce all
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int kl = p < 4 ? p : p + 4, ku = kl + 4;
        const uint32_t recv = __shfl_xor_sync(0xffffffffu, upper ? e[kl] : e[ku], lanebit);
        uint32_t u = upper ? recv : e[kl], v = upper ? e[ku] : recv;
        ct(u, v, w, q, more || p < 4, more || p < 4);
        const uint32_t back = __shfl_xor_sync(0xffffffffu, upper ? u : v, lanebit);
        e[kl] = upper ? back : u;
        e[ku] = upper ? v : back;
      }
    }
    {
      const uint2 w = entry(tc, B0);
#pragma unroll
      for (int r = 0; r < 8; ++r) ct(e[r], e[r + 8], w, q, red(r, 8), red(r + 8, 8));
    }
    {
      const uint4 v = __ldg(tc + ((B0 + 1) >> 1) * T);
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (!(r & 4)) ct(e[r], e[r + 4], (r >> 3) ? hi(v) : lo(v), q, red(r, 4), red(r + 4, 4));
    }
    {
      const uint4 v0 = __ldg(tc + ((B0 + 3) >> 1) * T), v1 = __ldg(tc + ((B0 + 5) >> 1) * T);
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & 2) continue;
        const int b = r >> 2;
        const uint4 v = b < 2 ? v0 : v1;
        ct(e[r], e[r + 2], (b & 1) ? hi(v) : lo(v), q, red(r, 2), red(r + 2, 2));
      }
    }
    {
      uint4 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = __ldg(tc + ((B0 + 7) / 2 + k) * T);
#pragma unroll
      for (int r = 0; r < 16; r += 2) {
        const int b = r >> 1;
        ct(e[r], e[r + 1], (b & 1) ? hi(v[b >> 1]) : lo(v[b >> 1]), q, !LAZY_OUT, !LAZY_OUT);
      }
    }
  }

  // Inverse: e in pass-C order (eval slots) -> e in pass-A order (natural
  // coefficients), scaled by n^-1. Begins and ends with a barrier.
  template <typename TW = const uint2*>
  static __device__ __forceinline__ void inv(uint32_t (&e)[16], uint32_t* sm, TW itw, const uint4* __restrict__ itwc,
                                             uint32_t q, uint2 last, uint2 ninv) {
    const uint32_t j = tid();
    const uint32_t x0 = posC0(j);
    const uint4* tc = itwc + j;
    // ---- pass C: stages LOGN-1 .. 8 (register stages first: t = 1, 2, 4, 8)
    {
      uint4 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = __ldg(tc + ((B0 + 7) / 2 + k) * T);
#pragma unroll
      for (int r = 0; r < 16; r += 2) {
        const int b = r >> 1;
        gs(e[r], e[r + 1], (b & 1) ? hi(v[b >> 1]) : lo(v[b >> 1]), q);
      }
    }
    {
      const uint4 v0 = __ldg(tc + ((B0 + 3) >> 1) * T), v1 = __ldg(tc + ((B0 + 5) >> 1) * T);
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & 2) continue;
        const int b = r >> 2;
        const uint4 v = b < 2 ? v0 : v1;
        gs(e[r], e[r + 2], (b & 1) ? hi(v) : lo(v), q);
      }
    }
    {
      const uint4 v = __ldg(tc + ((B0 + 1) >> 1) * T);
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (!(r & 4)) gs(e[r], e[r + 4], (r >> 3) ? hi(v) : lo(v), q);
    }
    {
      const uint2 w = entry(tc, B0);
#pragma unroll
      for (int r = 0; r < 8; ++r) gs(e[r], e[r + 8], w, q);
    }
#pragma unroll
    for (int s = XST - 1; s >= 0; --s) {
      const uint32_t t = G >> (s + 1);
      const uint32_t lanebit = t / 16;
      const bool upper = (x0 & t) != 0;
      const uint2 w = entry(tc, PAD + s);
#pragma unroll
      for (int k = 0; k < 8; ++k) {  // half exchange, as in the forward pass
        const uint32_t recv = __shfl_xor_sync(0xffffffffu, upper ? e[k] : e[k + 8], lanebit);
        uint32_t u = upper ? recv : e[k], v = upper ? e[k + 8] : recv;
        gs(u, v, w, q);
        const uint32_t back = __shfl_xor_sync(0xffffffffu, upper ? u : v, lanebit);
        e[k] = upper ? back : u;
        e[k + 8] = upper ? v : back;
      }
    }
    sync();
    storeC(sm, j, e);
    sync_bc();
    // ---- pass B: stages 7..4
#pragma unroll
    for (int r = 0; r < 16; ++r) e[r] = sm[swz(posB(j, r))];
    {
      const uint32_t blk = j >> (LOGN - 8);
#pragma unroll
      for (int s = 3; s >= 0; --s) {
        const int half = 8 >> s;
#pragma unroll
        for (int r = 0; r < 16; ++r)
          if (!(r & half)) gs(e[r], e[r + half], load_tw(itw, (16u << s) + (blk << s) + (r >> (4 - s))), q);
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) sm[swz(posB(j, r))] = e[r];
    sync();
    // ---- pass A: stages 3..1, then stage 0 fused with the n^-1 scaling
    {
      const uint32_t* pa = sm + swz(j);  // swz(j + T*r) = swz(j) + T*r
#pragma unroll
      for (int r = 0; r < 16; ++r) e[r] = pa[T * r];
    }
#pragma unroll
    for (int s = 3; s >= 1; --s) {
      const int half = 8 >> s;
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (!(r & half)) gs(e[r], e[r + half], load_tw(itw, (1 << s) + (r >> (4 - s))), q);
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const uint32_t u = e[r], v = e[r + 8];
      e[r] = mul_shoup(u + v, ninv.x, ninv.y, q);
      e[r + 8] = mul_shoup(u - v + q, last.x, last.y, q);
    }
  }
};

}  // namespace heb
