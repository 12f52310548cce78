// Standard (sample-batched) comparator on the device:
// hei::matmul::baseline_matmul (proj/src/matmul/matmul.cpp:273-344).
//
// Per feature k and sample block the reference encrypts the column x[:, k]
// with the public key (BfvContext::encrypt_parts, context.cpp:262-303) using
// its util::Prng stream (rng.hpp:19-68), multiplies it by the all-slot
// constant w(k, j) for every class j and sums. The device draws the SAME
// stream and sums by linearity (stdalg_kernels.cuh):
//   k_mt_chunks /   mt19937_64 replay: jump-ahead chunk generators, or one
//   k_mt_generate   sequential CTA per branch
//   k_bl_noise_p    u = v mod 3 - 1, (e0, e1) = Box-Muller pairs, llround
//   k_bl_encode     m = INTT_t(scatter(centered column residues))
//   k_bl_sums       exact int64 sums over features of w' u, w' e0, w' e1, w' m
//   k_bl_fold_sums  -> residues mod every q_i
//   k_bl_finish_lin c0 = NTT(A) pk0 + NTT(B) + bias, c1 = NTT(A) pk1 + NTT(C)
#pragma once

namespace heb_baseline {

constexpr uint64_t kMtUM = 0xFFFFFFFF80000000ULL, kMtLM = 0x7FFFFFFFULL, kMtA = 0xB5026F5AA96619E9ULL;

__device__ __forceinline__ uint64_t mt_temper(uint64_t x) {
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

// state: [2][313] (312 words + mti) for the two branches; block b advances
// branch b by `count` draws into out[b * count ...]. The twist runs as two
// 156-wide phases on ping-pong buffers (2 barriers per 312 outputs); each
// thread tempers and stores the word it produced.
__global__ void __launch_bounds__(320) k_mt_generate(uint64_t* __restrict__ state, uint64_t* __restrict__ out,
                                                     uint64_t count) {
  __shared__ uint64_t buf[2][312];
  const uint32_t b = blockIdx.x, t = threadIdx.x;
  uint64_t* st = state + (uint64_t)b * 313;
  uint64_t* o = out + (uint64_t)b * count;
  for (uint32_t i = t; i < 312; i += blockDim.x) buf[0][i] = st[i];
  uint32_t mti = (uint32_t)st[312];
  __syncthreads();
  // words of the current block not consumed yet
  const uint64_t rem = min((uint64_t)(312 - mti), count);
  if (t < rem) o[t] = mt_temper(buf[0][mti + t]);
  uint64_t pos = rem;
  mti += (uint32_t)rem;
  int cur = 0;
  while (pos < count) {
    const uint64_t* A = buf[cur];
    uint64_t* B = buf[cur ^ 1];
    if (t < 156) {
      const uint64_t y = (A[t] & kMtUM) | (A[t + 1] & kMtLM);
      const uint64_t v = A[t + 156] ^ (y >> 1) ^ ((y & 1) ? kMtA : 0);
      B[t] = v;
      if (pos + t < count) o[pos + t] = mt_temper(v);
    }
    __syncthreads();
    if (t >= 156 && t < 312) {
      const uint64_t y = (A[t] & kMtUM) | ((t == 311 ? B[0] : A[t + 1]) & kMtLM);
      const uint64_t v = B[t - 156] ^ (y >> 1) ^ ((y & 1) ? kMtA : 0);
      B[t] = v;
      if (pos + t < count) o[pos + t] = mt_temper(v);
    }
    __syncthreads();
    cur ^= 1;
    const uint64_t nw = min((uint64_t)312, count - pos);
    pos += nw;
    mti = (uint32_t)nw;
  }
  for (uint32_t i = t; i < 312; i += blockDim.x) st[i] = buf[cur][i];
  if (t == 0) st[312] = mti;
}

// One Prng::gaussian pair (rng.hpp:47-62: cos first, sin cached as the spare)
// scaled by sigma = 3.2, clamped at 6 sigma and rounded with llround
// (sample_gaussian, sampling.cpp:24-34). Returns false on the u1 == 0
// rejection, which would shift the stream.
__device__ __forceinline__ bool box_muller_pair(uint64_t r1, uint64_t r2, int8_t& a, int8_t& b) {
  const double sigma = 3.2, bound = 6.0 * sigma, two_pi = 6.283185307179586476925286766559;
  const double u1 = (double)(r1 >> 11) * 0x1.0p-53;
  const double u2 = (double)(r2 >> 11) * 0x1.0p-53;
  const double mag = sqrt(-2.0 * log(u1));
  double sn, cs;
  sincos(two_pi * u2, &sn, &cs);
  double x0 = mag * cs * sigma, x1 = mag * sn * sigma;
  x0 = x0 > bound ? bound : (x0 < -bound ? -bound : x0);
  x1 = x1 > bound ? bound : (x1 < -bound ? -bound : x1);
  a = (int8_t)llround(x0);
  b = (int8_t)llround(x1);
  return u1 > 0.0;
}

// Noise of one encryption per (e, branch): raw draws [3][N] -> i8 [3][N]
// (sample_ternary, sample_gaussian twice; sampling.cpp:16-34). The Box-Muller
// pair (cos first, sin as the cached spare) follows Prng::gaussian. Any
// rejection (v == 2^64 - 1 for the ternary draw, u1 == 0) would shift the
// stream; it is flagged and the call fails rather than diverge.
__global__ void k_bl_noise(const uint64_t* __restrict__ raw, uint64_t count, uint32_t n, uint32_t encs,
                           int8_t* __restrict__ noise, uint32_t* err) {
  const uint32_t e = blockIdx.x, b = blockIdx.y;
  const uint64_t* d = raw + (uint64_t)b * count + (uint64_t)e * 3 * n;
  int8_t* o = noise + ((uint64_t)e * 2 + b) * 3 * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
    const uint64_t v = d[x];
    if (v == ~0ull) *err = 1;
    o[x] = (int8_t)((int)(v % 3) - 1);
  }
  for (uint32_t s = 0; s < 2; ++s) {
    const uint64_t* g = d + n + (uint64_t)s * n;
    int8_t* og = o + n + s * n;
    for (uint32_t k = threadIdx.x; k < n / 2; k += blockDim.x)
      if (!box_muller_pair(g[2 * k], g[2 * k + 1], og[2 * k], og[2 * k + 1])) *err = 1;
  }
  (void)encs;
}

// ---- jump-ahead (parallel replay of one sequential stream) ----------------
// A window state S_o = (W_o .. W_{o+311}) of the word recurrence
// W_{k+312} = W_{k+156} ^ T(W_k, W_{k+1}) is exactly the generator array when
// mti == 312. Advancing by J words is S -> p(A) S with p = x^J mod phi (phi
// the characteristic polynomial of mt19937_64), and p(A) S is a sliding XOR
// of the word sequence: (p(A) S)[k] = XOR_{i: p_i = 1} W_{o+k+i}.
// One block per branch; writes the K chunk start windows (mti = 312) spaced
// J words apart. smem: the 20249-word window sequence.
constexpr int kMtDeg = 19937;
constexpr int kMtSeq = kMtDeg + 312;  // words needed by one jump

// One jump step is three launches so the XOR convolution runs on the whole
// GPU: k_mt_wseq extends each branch's current window to the 20249-word
// sequence (sequential twists, one block per branch), k_mt_xor computes
// partial windows over slices of the polynomial (many blocks), and
// k_mt_xor_reduce folds the partials into the next start window.
// Tree-ordered jump-ahead: level k advances starts[m] by 2^k * C words into
// starts[m + 2^k] for every m < min(2^k, K - 2^k) at once, so K chunk starts
// cost ceil(log2 K) levels of three batched launches instead of K - 1
// sequential jumps. grid.z (or .y) = job m; branch b = blockIdx.y (or .x).
__global__ void __launch_bounds__(320) k_mt_wseq(const uint64_t* __restrict__ starts, uint32_t K,
                                                 uint64_t* __restrict__ wseq, uint32_t wlen) {
  __shared__ uint64_t buf[2][312];
  const uint32_t b = blockIdx.x, m = blockIdx.y, t = threadIdx.x;
  const uint64_t* st = starts + ((uint64_t)b * K + m) * 313;
  uint64_t* W = wseq + ((uint64_t)m * 2 + b) * wlen;
  for (uint32_t i = t; i < 312; i += blockDim.x) {
    buf[0][i] = st[i];
    W[i] = st[i];
  }
  __syncthreads();
  int c = 0;
  for (uint32_t blk = 1; 312 * blk < wlen; ++blk) {
    const uint64_t* A = buf[c];
    uint64_t* B = buf[c ^ 1];
    if (t < 156) {
      const uint64_t y = (A[t] & kMtUM) | (A[t + 1] & kMtLM);
      B[t] = A[t + 156] ^ (y >> 1) ^ ((y & 1) ? kMtA : 0);
      W[312 * blk + t] = B[t];
    }
    __syncthreads();
    if (t >= 156 && t < 312) {
      const uint64_t y = (A[t] & kMtUM) | ((t == 311 ? B[0] : A[t + 1]) & kMtLM);
      B[t] = B[t - 156] ^ (y >> 1) ^ ((y & 1) ? kMtA : 0);
      W[312 * blk + t] = B[t];
    }
    __syncthreads();
    c ^= 1;
  }
}

// partial[m][b][s][k] = XOR over set bits i of poly words [s*ws, (s+1)*ws) of W[k+i]
__global__ void __launch_bounds__(320) k_mt_xor(const uint64_t* __restrict__ wseq, uint32_t wlen,
                                                const uint64_t* __restrict__ poly, uint32_t ws,
                                                uint64_t* __restrict__ partial) {
  const uint32_t s = blockIdx.x, b = blockIdx.y, m = blockIdx.z, t = threadIdx.x;
  const uint32_t nw = (kMtDeg + 63) / 64;
  const uint64_t* W = wseq + ((uint64_t)m * 2 + b) * wlen;
  uint64_t acc = 0;
  if (t < 312)
    for (uint32_t wi = s * ws; wi < min(nw, (s + 1) * ws); ++wi) {
      uint64_t bits = __ldg(&poly[wi]);
      while (bits) {
        const uint32_t i = wi * 64 + __ffsll((long long)bits) - 1;
        acc ^= __ldg(&W[t + i]);
        bits &= bits - 1;
      }
    }
  if (t < 312) partial[(((uint64_t)m * 2 + b) * gridDim.x + s) * 312 + t] = acc;
}

__global__ void k_mt_xor_reduce(const uint64_t* __restrict__ partial, uint32_t S, uint64_t* __restrict__ starts,
                                uint32_t K, uint32_t step) {
  const uint32_t b = blockIdx.x, m = blockIdx.y, t = threadIdx.x;
  if (t >= 312) return;
  uint64_t acc = 0;
  for (uint32_t s = 0; s < S; ++s) acc ^= partial[(((uint64_t)m * 2 + b) * S + s) * 312 + t];
  uint64_t* dst = starts + ((uint64_t)b * K + m + step) * 313;
  dst[t] = acc;
  if (t == 0) dst[312] = 312;
}

// Chunk m of branch b generates draws [m*C, min((m+1)*C, total)) from its
// start window; the last chunk's final state is written back to `state`.
__global__ void __launch_bounds__(320) k_mt_chunks(uint64_t* __restrict__ starts, uint32_t K, uint64_t C,
                                                   uint64_t total, uint64_t* __restrict__ out,
                                                   uint64_t* __restrict__ state) {
  __shared__ uint64_t buf[2][312];
  const uint32_t m = blockIdx.x, b = blockIdx.y, t = threadIdx.x;
  const uint64_t* st = starts + ((uint64_t)b * K + m) * 313;
  const uint64_t begin = (uint64_t)m * C;
  const uint64_t count = min(C, total - begin);
  uint64_t* o = out + (uint64_t)b * total + begin;
  for (uint32_t i = t; i < 312; i += blockDim.x) buf[0][i] = st[i];
  __syncthreads();
  uint64_t pos = 0;
  uint32_t mti = 312;
  int cur = 0;
  while (pos < count) {
    const uint64_t* A = buf[cur];
    uint64_t* B = buf[cur ^ 1];
    if (t < 156) {
      const uint64_t y = (A[t] & kMtUM) | (A[t + 1] & kMtLM);
      const uint64_t v = A[t + 156] ^ (y >> 1) ^ ((y & 1) ? kMtA : 0);
      B[t] = v;
      if (pos + t < count) o[pos + t] = mt_temper(v);
    }
    __syncthreads();
    if (t >= 156 && t < 312) {
      const uint64_t y = (A[t] & kMtUM) | ((t == 311 ? B[0] : A[t + 1]) & kMtLM);
      const uint64_t v = B[t - 156] ^ (y >> 1) ^ ((y & 1) ? kMtA : 0);
      B[t] = v;
      if (pos + t < count) o[pos + t] = mt_temper(v);
    }
    __syncthreads();
    cur ^= 1;
    const uint64_t nw = min((uint64_t)312, count - pos);
    pos += nw;
    mti = (uint32_t)nw;
  }
  if (m + 1 == K) {
    uint64_t* fs = state + (uint64_t)b * 313;
    for (uint32_t i = t; i < 312; i += blockDim.x) fs[i] = buf[cur][i];
    if (t == 0) fs[312] = mti;
  }
}

}  // namespace heb_baseline
