// Client-side decryption and CRT unpacking on the device.
//
// Textually included by heinfer_b200.cu inside its kernel namespace (uses Geo,
// PrimeInfo, BranchInfo and the shared-memory NTTs). Follows
//   BfvContext::decrypt_core   proj/src/bfv/context.cpp:316-370
//   BfvContext::decode_slots   proj/src/bfv/context.cpp:95-102
//   TwinBackend::decode_signed proj/src/fpcrt/twin.cpp:113-121
//   fpcrt::crt_recombine       proj/src/fpcrt/fixed_point.cpp:89-106
// The reference does the CRT with a Boost cpp_int per coefficient; here every
// coefficient is one thread with fixed 8 x 32-bit limbs (Q < 2^218 for every
// parameter set validate() admits at N <= 16384, params.cpp:27-66), so the
// message, the rounding and the noise residual are exact and equal.
#pragma once

constexpr int kLimbs = 8;  // 256-bit fixed-width integers
constexpr int kMaxBranchPrimes = 8;

struct CrtBranch {
  uint32_t L, t;
  int q_msb;                                  // msb(Q)
  double Qd;                                  // Q as a double (quotient estimate)
  uint32_t q[kMaxBranchPrimes], y[kMaxBranchPrimes];  // y_i = (Q/q_i)^-1 mod q_i
  uint32_t Qp[kMaxBranchPrimes][kLimbs];      // Q/q_i
  uint32_t Q[kLimbs], Qh[kLimbs];             // Q, floor(Q/2)
};
struct CrtInfo {
  CrtBranch b[2];
};

__device__ __forceinline__ void mw_mul_add(uint32_t (&acc)[kLimbs], const uint32_t (&a)[kLimbs], uint32_t m) {
  uint64_t carry = 0;
#pragma unroll
  for (int k = 0; k < kLimbs; ++k) {
    const uint64_t v = (uint64_t)a[k] * m + acc[k] + carry;
    acc[k] = (uint32_t)v;
    carry = v >> 32;
  }
}
__device__ __forceinline__ bool mw_geq(const uint32_t (&a)[kLimbs], const uint32_t (&b)[kLimbs]) {
#pragma unroll
  for (int k = kLimbs - 1; k >= 0; --k)
    if (a[k] != b[k]) return a[k] > b[k];
  return true;
}
__device__ __forceinline__ void mw_sub(uint32_t (&a)[kLimbs], const uint32_t (&b)[kLimbs]) {  // a -= b, a >= b
  int64_t br = 0;
#pragma unroll
  for (int k = 0; k < kLimbs; ++k) {
    const int64_t v = (int64_t)a[k] - b[k] + br;
    a[k] = (uint32_t)v;
    br = v >> 32;
  }
}
__device__ __forceinline__ void mw_add(uint32_t (&a)[kLimbs], const uint32_t (&b)[kLimbs]) {
  uint64_t c = 0;
#pragma unroll
  for (int k = 0; k < kLimbs; ++k) {
    const uint64_t v = (uint64_t)a[k] + b[k] + c;
    a[k] = (uint32_t)v;
    c = v >> 32;
  }
}
__device__ __forceinline__ int mw_msb(const uint32_t (&a)[kLimbs]) {
#pragma unroll
  for (int k = kLimbs - 1; k >= 0; --k)
    if (a[k]) return 32 * k + 31 - __clz(a[k]);
  return -1;
}
__device__ __forceinline__ double mw_double(const uint32_t (&a)[kLimbs]) {
  double d = 0.0;
#pragma unroll
  for (int k = kLimbs - 1; k >= 0; --k) d = d * 4294967296.0 + (double)a[k];
  return d;
}

// Phase c0 + c1*s per (ct, prime), then the inverse NTT: w [ct][P][n]
// (decrypt_core, context.cpp:322-339; the coeff-form branch is the same value
// by linearity and is served by NTT-ing coeff inputs first).
__global__ void k_dec_phase(Geo g, const uint32_t* __restrict__ cts, const uint32_t* __restrict__ s_hat,
                            uint32_t* __restrict__ w) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n, gp = blockIdx.x % g.P;
  const uint64_t ct = blockIdx.x / g.P;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t* c0 = cts + ct * g.ct_words + (uint64_t)pr.poly0 * n;
  const uint32_t* c1 = cts + ct * g.ct_words + (uint64_t)pr.poly1 * n;
  const uint32_t* s = s_hat + (uint64_t)gp * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x)
    sm[x] = add_mod(mul_barrett(c1[x], s[x], pr.q, pr.mu), c0[x], pr.q);
  __syncthreads();
  ntt_inv_smem(sm, g.inv + (size_t)gp * n, pr.q, n, g.logn, pr.last, pr.ninv);
  uint32_t* o = w + (ct * g.P + gp) * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) o[x] = sm[x];
}

// Exact CRT + rounding per coefficient (context.cpp:341-361): m [ct][2][n]
// mod t_b, and msb(|r|) maxed into rmsb[ct][2] (max_r's msb; the budget only
// needs msb(2 max_r) = msb(max_r) + 1).
__global__ void k_dec_crt(Geo g, CrtInfo ci, const uint32_t* __restrict__ w, uint64_t count,
                          uint32_t* __restrict__ m, int* __restrict__ rmsb) {
  const uint64_t total = count * 2 * g.n;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t j = (uint32_t)(x % g.n);
    const uint32_t b = (uint32_t)((x / g.n) % 2);
    const uint64_t ct = x / (2ull * g.n);
    const CrtBranch& cb = ci.b[b];
    const uint32_t first = b ? g.L[0] : 0;
    uint32_t acc[kLimbs] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint32_t i = 0; i < cb.L; ++i) {
      const uint32_t wi = w[(ct * g.P + first + i) * g.n + j];
      const uint32_t c = (uint32_t)(((uint64_t)wi * cb.y[i]) % cb.q[i]);
      mw_mul_add(acc, cb.Qp[i], c);
    }
    while (mw_geq(acc, cb.Q)) mw_sub(acc, cb.Q);
    uint32_t z[kLimbs] = {0, 0, 0, 0, 0, 0, 0, 0};
    mw_mul_add(z, acc, cb.t);  // z = acc * t
    uint32_t num[kLimbs];
#pragma unroll
    for (int k = 0; k < kLimbs; ++k) num[k] = z[k];
    mw_add(num, cb.Qh);  // num = z + Q_half
    // quot = floor(num / Q) <= t: double estimate, then exact correction
    uint32_t quot = (uint32_t)fmin(floor(mw_double(num) / cb.Qd), (double)cb.t);
    uint32_t prod[kLimbs] = {0, 0, 0, 0, 0, 0, 0, 0};
    mw_mul_add(prod, cb.Q, quot);
    while (!mw_geq(num, prod)) {  // estimate too high
      --quot;
      mw_sub(prod, cb.Q);
    }
    uint32_t rem[kLimbs];
#pragma unroll
    for (int k = 0; k < kLimbs; ++k) rem[k] = num[k];
    mw_sub(rem, prod);
    while (mw_geq(rem, cb.Q)) {  // estimate too low
      ++quot;
      mw_sub(rem, cb.Q);
    }
    m[(ct * 2 + b) * g.n + j] = quot % cb.t;
    // r = z - quot*Q = rem - Q_half; |r|
    uint32_t r[kLimbs];
    if (mw_geq(rem, cb.Qh)) {
#pragma unroll
      for (int k = 0; k < kLimbs; ++k) r[k] = rem[k];
      mw_sub(r, cb.Qh);
    } else {
#pragma unroll
      for (int k = 0; k < kLimbs; ++k) r[k] = cb.Qh[k];
      mw_sub(r, rem);
    }
    const int mb = mw_msb(r);
    if (mb >= 0) atomicMax(&rmsb[ct * 2 + b], mb);
  }
}

// decode_slots (context.cpp:95-102): forward NTT mod t_b, then the slot
// gather through the generator-3 index map. slots [ct][2][n].
__global__ void k_dec_decode(Geo g, const uint32_t* __restrict__ m, uint32_t* __restrict__ slots) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n, b = blockIdx.x % 2;
  const uint64_t ct = blockIdx.x / 2;
  const BranchInfo& br = g.br[b];
  const uint32_t* src = m + (ct * 2 + b) * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) sm[x] = src[x];
  __syncthreads();
  ntt_fwd_smem(sm, g.fwd + (size_t)(g.P + b) * n, br.t, n, g.logn);
  uint32_t* o = slots + (ct * 2 + b) * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) o[x] = sm[g.index_map[x]];
}

// crt_recombine (fixed_point.cpp:89-106), Garner + centering, scattered to the
// caller's layout: mode 0 = packed results (out[g] for g < rows*cols, g = c*n +
// s, matmul.cpp:257-271), mode 1 = baseline blocks (ct = blk*cols + j, slot s
// -> out[(blk*n + s)*cols + j], matmul.cpp:346-358), mode 2 = raw [ct][n].
__global__ void k_dec_recombine(Geo g, const uint32_t* __restrict__ slots, uint64_t count, uint64_t rows,
                                uint64_t cols, int mode, uint32_t t0inv, int64_t* __restrict__ out) {
  const uint64_t total = count * g.n;
  const uint64_t t0 = g.br[0].t, t1 = g.br[1].t, prod = t0 * t1;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t ct = x / g.n;
    const uint32_t s = (uint32_t)(x % g.n);
    const uint64_t r0 = slots[(ct * 2) * g.n + s], r1 = slots[(ct * 2 + 1) * g.n + s];
    const uint64_t diff = (r1 + t1 - r0 % t1) % t1;
    const uint64_t k = diff * t0inv % t1;
    const uint64_t v = t0 * k + r0;  // < t0 * t1 < 2^63
    const int64_t sv = v > (prod - 1) / 2 ? (int64_t)v - (int64_t)prod : (int64_t)v;
    if (mode == 0) {
      if (x < rows * cols) out[x] = sv;
    } else if (mode == 1) {
      const uint64_t blk = ct / cols, j = ct % cols, row = blk * g.n + s;
      if (row < rows) out[row * cols + j] = sv;
    } else {
      out[x] = sv;
    }
  }
}

// lift_signed(s) mod q_i then NTT (prepared_secret, context.cpp:139-150).
__global__ void k_prepare_sk(Geo g, uint32_t b, const int8_t* __restrict__ s, uint32_t* __restrict__ s_hat) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n, gp = (b ? g.L[0] : 0) + blockIdx.x;
  const PrimeInfo& pr = g.pr[gp];
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) sm[x] = s[x] < 0 ? pr.q - 1 : (uint32_t)s[x];
  __syncthreads();
  ntt_fwd_smem(sm, g.fwd + (size_t)gp * n, pr.q, n, g.logn);
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) s_hat[(uint64_t)gp * n + x] = sm[x];
}
