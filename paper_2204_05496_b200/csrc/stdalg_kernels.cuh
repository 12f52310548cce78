// Standard-algorithm and client-encryption kernels (baseline_matmul,
// matmul.cpp:415-486; encrypt_parts, context.cpp:262-303). The mt19937_64
// replay and the noise sampler live in baseline.cuh. Textually included by
// heinfer_b200.cu inside its kernel namespace.
#pragma once

// ---------------------------------------------------------------------------
// Standard algorithm (baseline_matmul) kernels; see baseline.cuh.
// ---------------------------------------------------------------------------
// m = INTT_t(scatter(centered residues of x[base + s][k])) per (encryption,
// branch); encryption e = kk * B + blk (matmul.cpp:444-452 loop order).
template <int LOGN>
__global__ void __launch_bounds__(Ntt<LOGN>::T) k_bl_encode(Geo g, const int64_t* __restrict__ x, uint64_t R,
                                                           uint64_t f, uint64_t k0, uint32_t B,
                                                           uint32_t* __restrict__ m_out, int row_mode = 0) {
  using NT = Ntt<LOGN>;
  constexpr uint32_t N = NT::N;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  const uint32_t e = blockIdx.x, b = blockIdx.y;
  // column mode (baseline): slot s = row base + s of feature k.
  // row mode (encode_inputs, matmul.cpp:201-211): encryption k0 + e is chunk
  // (k0 + e) % B of row (k0 + e) / B (B = chunks per row), slot s = feature.
  const uint64_t eg = k0 + e;
  const uint64_t k = row_mode ? 0 : k0 + e / B;
  const uint64_t base = row_mode ? (eg / B) * f + (eg % B) * N : (uint64_t)(e % B) * N;
  const uint64_t lim = row_mode ? min((uint64_t)N, f - (eg % B) * N) : min((uint64_t)N, R - base);
  const BranchInfo& br = g.br[b];
  const int64_t t = br.t;
  for (uint32_t s = threadIdx.x; s < N; s += blockDim.x) {
    int64_t r = 0;
    if (s < lim) {
      r = (row_mode ? x[base + s] : x[(base + s) * f + k]) % t;
      if (r < 0) r += t;
    }
    sm[swz(g.index_map[s])] = (uint32_t)r;
  }
  __syncthreads();
  uint32_t v[16];
  NT::loadC(sm, threadIdx.x, v);
  NT::inv(v, sm, g.inv + (size_t)(g.P + b) * N, g.itwc + (size_t)(g.P + b) * g.twc_stride, br.t, br.last, br.ninv);
  uint32_t* o = m_out + ((uint64_t)e * 2 + b) * N;
#pragma unroll
  for (int r = 0; r < 16; ++r) o[NT::posA(threadIdx.x, r)] = v[r];
}

__device__ __forceinline__ uint32_t lift_small(int32_t v, uint32_t q) { return v >= 0 ? (uint32_t)v : q - (uint32_t)(-v); }

// Public-key encryption in eval form, block per (encryption, gp)
// (context.cpp:270-301): c0 = NTT(u) pk0 + NTT(e0 + Delta m),
// c1 = NTT(u) pk1 + NTT(e1). pk is prepared [gp][part] in the pass-C
// transposed layout.
template <int LOGN, bool PTW, int MINB = (LOGN <= 13 ? 2 : 1)>
__global__ void __launch_bounds__(Ntt<LOGN>::T, MINB) k_bl_encrypt(Geo g, const int8_t* __restrict__ noise,
                                                            const uint32_t* __restrict__ m,
                                                            const uint2* __restrict__ pkd,
                                                            uint32_t* __restrict__ cts,
                                                            const __grid_constant__ TwArg<PTW> tab) {
  // c0 = NTT(u) pk0 + NTT(e0 + Delta m), c1 = NTT(u) pk1 + NTT(e1)
  // (encrypt_parts, context.cpp:262-303); one transform live at a time.
  using NT = Ntt<LOGN>;
  constexpr uint32_t N = NT::N, T = NT::T;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  const uint32_t e = blockIdx.x / g.P, gp = blockIdx.x % g.P;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, b = pr.b, j = threadIdx.x, x0 = NT::posC0(j);
  const int8_t* nz = noise + ((uint64_t)e * 2 + b) * 3 * N;
  const uint32_t* mm = m + ((uint64_t)e * 2 + b) * N;
  const uint2* tw = g.fwd + (size_t)gp * N;
  const uint4* twc = g.twc + (size_t)gp * g.twc_stride;
  uint32_t* ct = cts + (uint64_t)e * g.ct_words;
  uint4* c0 = reinterpret_cast<uint4*>(ct + (uint64_t)pr.poly0 * N + x0);
  uint4* c1 = reinterpret_cast<uint4*>(ct + (uint64_t)pr.poly1 * N + x0);
  const uint4* p0 = reinterpret_cast<const uint4*>(pkd + (uint64_t)(2 * gp) * N) + j;
  const uint4* p1 = reinterpret_cast<const uint4*>(pkd + (uint64_t)(2 * gp + 1) * N) + j;
  uint32_t v[16];
  // one transform instance (a rolled phase loop keeps the compiler from
  // hoisting the shared twiddles of three inlined NTTs into registers)
#pragma unroll 1
  for (int ph = 0; ph < 3; ++ph) {
    if (ph == 1) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint32_t pa = NT::posA(j, r);
        v[r] = add_mod(lift_small(nz[N + pa], q), mul_shoup(mm[pa], pr.delta.x, pr.delta.y, q), q);
      }
    } else {
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = lift_small(nz[(uint32_t)ph * N + NT::posA(j, r)], q);
    }
    if constexpr (PTW)
      NT::fwd(v, sm, ParamTw{tab.w[gp]}, twc, q);
    else
      NT::fwd(v, sm, tw, twc, q);
    if (ph == 0) {  // NTT(u) pk0 -> c0, NTT(u) pk1 -> c1
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint4 a0 = __ldg(p0 + (2 * c) * T), a1 = __ldg(p0 + (2 * c + 1) * T);
        const uint4 b0 = __ldg(p1 + (2 * c) * T), b1 = __ldg(p1 + (2 * c + 1) * T);
        c1[c] = make_uint4(mul_shoup(v[4 * c], b0.x, b0.y, q), mul_shoup(v[4 * c + 1], b0.z, b0.w, q),
                           mul_shoup(v[4 * c + 2], b1.x, b1.y, q), mul_shoup(v[4 * c + 3], b1.z, b1.w, q));
        c0[c] = make_uint4(mul_shoup(v[4 * c], a0.x, a0.y, q), mul_shoup(v[4 * c + 1], a0.z, a0.w, q),
                           mul_shoup(v[4 * c + 2], a1.x, a1.y, q), mul_shoup(v[4 * c + 3], a1.z, a1.w, q));
      }
    } else {  // c0 += NTT(e0 + Delta m), c1 += NTT(e1)
      uint4* cp = ph == 1 ? c0 : c1;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint4 u = cp[c];
        cp[c] = make_uint4(add_mod(u.x, v[4 * c], q), add_mod(u.y, v[4 * c + 1], q), add_mod(u.z, v[4 * c + 2], q),
                           add_mod(u.w, v[4 * c + 3], q));
      }
    }
  }
}

// acc[blk][j] += sum_k ct[k, blk] * w(k, j) mod q, lazily in u64
// (mul_plain + add_inplace of matmul.cpp:453-459). Thread per slot x of one
// poly; weights of the batch for this branch sit in shared memory. The
// feature loop is unrolled so several coalesced loads are in flight.
constexpr int kBlJ = 12;
__global__ void k_bl_accum(Geo g, const uint32_t* __restrict__ cts, uint32_t F, uint32_t B, uint32_t cols,
                           uint32_t j0, const uint2* __restrict__ wc, unsigned long long* __restrict__ acc) {
  extern __shared__ uint2 wsm[];  // [F][kBlJ]
  const uint32_t n = g.n, polys = 2 * g.P;
  const uint32_t tiles = n / blockDim.x;
  const uint32_t tile = blockIdx.x % tiles;
  const uint32_t poly = (blockIdx.x / tiles) % polys;
  const uint32_t blk = blockIdx.x / (tiles * polys);
  const uint32_t gp = poly_prime(g, poly);
  const uint32_t q = g.pr[gp].q;
  const uint32_t jn = min((uint32_t)kBlJ, cols - j0);
  for (uint32_t x = threadIdx.x; x < F * kBlJ; x += blockDim.x) {
    const uint32_t kk = x / kBlJ, jj = x % kBlJ;
    wsm[x] = jj < jn ? wc[((uint64_t)kk * cols + j0 + jj) * g.P + gp] : make_uint2(0, 0);
  }
  __syncthreads();
  const uint32_t xs = tile * blockDim.x + threadIdx.x;
  const uint32_t* src = cts + (uint64_t)blk * g.ct_words + (uint64_t)poly * n + xs;
  const uint64_t stride = (uint64_t)B * g.ct_words;
  unsigned long long a[kBlJ];
#pragma unroll
  for (int jj = 0; jj < kBlJ; ++jj) a[jj] = 0;
  if (g.br[g.pr[gp].b].t < (1u << 20)) {
    // small plaintext modulus: the weight residues are < 2^20, so the exact
    // products (< 2^51) accumulate with one IMAD.WIDE each; this batch's
    // sums (< 2^59) are reduced mod q before they reach the accumulator
#pragma unroll 8
    for (uint32_t kk = 0; kk < F; ++kk) {
      const uint64_t v = src[kk * stride];
#pragma unroll
      for (int jj = 0; jj < kBlJ; ++jj) a[jj] += v * wsm[kk * kBlJ + jj].x;
    }
#pragma unroll
    for (int jj = 0; jj < kBlJ; ++jj) a[jj] %= q;
  } else {
#pragma unroll 8
    for (uint32_t kk = 0; kk < F; ++kk) {
      const uint32_t v = src[kk * stride];
#pragma unroll
      for (int jj = 0; jj < kBlJ; ++jj) {
        const uint2 w = wsm[kk * kBlJ + jj];
        const uint32_t qh = __umulhi(v, w.y);
        a[jj] += (uint32_t)(v * w.x - qh * q);  // in [0, 2q): reduced at the end
      }
    }
  }
#pragma unroll
  for (uint32_t jj = 0; jj < kBlJ; ++jj) {
    if (jj < jn) {
      unsigned long long* d = acc + (((uint64_t)blk * cols + j0 + jj) * g.ct_words) + (uint64_t)poly * n + xs;
      *d += a[jj];
    }
  }
}

// Same sums with exact 64-bit products and no Shoup step: every weight
// residue is < t < 2^31 and every ct residue < q < 2^31, so v * w < 2^62 and
// one IMAD.WIDE.U32 accumulates it. The accumulator is folded every 3
// features (a -> hi(a) * (2^32 mod q) + lo(a), congruent mod q): with k = 3
// products of < 2^61 (t0 < 2^30) between folds the bound stays below
// 3 * 2^62 + 2^33 < 2^64. For t < 2^20 (products < 2^51) no fold is needed
// within a batch. The batch sum is reduced mod q before it reaches `acc`, so
// the result equals k_bl_accum's mod q exactly. Weights (values only) are
// read from shared memory as 3 x 128-bit per feature.
//
// The batch's features are split over S block slices (blockIdx.y); slice s
// sums its feature range into its own accumulator copy acc + s * slice_words
// (k_bl_finish adds the copies), so a launch has S times the blocks.
__global__ void k_bl_accum_w(Geo g, const uint32_t* __restrict__ cts, uint32_t F, uint32_t B, uint32_t cols,
                             uint32_t j0, const uint2* __restrict__ wc, unsigned long long* __restrict__ acc,
                             uint64_t slice_words) {
  static_assert(kBlJ == 12, "3 x uint4 of weights per feature");
  extern __shared__ uint4 wsm4[];  // [F][3] = [F][kBlJ] u32
  uint32_t* wsm = reinterpret_cast<uint32_t*>(wsm4);
  const uint32_t n = g.n, polys = 2 * g.P;
  const uint32_t tiles = n / blockDim.x;
  const uint32_t tile = blockIdx.x % tiles;
  const uint32_t poly = (blockIdx.x / tiles) % polys;
  const uint32_t blk = blockIdx.x / (tiles * polys);
  const uint32_t gp = poly_prime(g, poly);
  const uint32_t q = g.pr[gp].q;
  const uint32_t jn = min((uint32_t)kBlJ, cols - j0);
  const uint32_t k_lo = (uint32_t)((uint64_t)F * blockIdx.y / gridDim.y);
  F = (uint32_t)((uint64_t)F * (blockIdx.y + 1) / gridDim.y) - k_lo;
  acc += blockIdx.y * slice_words;
  for (uint32_t x = threadIdx.x; x < F * kBlJ; x += blockDim.x) {
    const uint32_t kk = x / kBlJ, jj = x % kBlJ;
    wsm[x] = jj < jn ? wc[((uint64_t)(k_lo + kk) * cols + j0 + jj) * g.P + gp].x : 0u;
  }
  __syncthreads();
  const uint32_t xs = tile * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)B * g.ct_words;
  const uint32_t* src = cts + (uint64_t)blk * g.ct_words + (uint64_t)poly * n + xs + k_lo * stride;
  unsigned long long a[kBlJ];
#pragma unroll
  for (int jj = 0; jj < kBlJ; ++jj) a[jj] = 0;
  auto mac = [&](uint32_t kk) {
    const uint64_t v = src[kk * stride];
    const uint4 w0 = wsm4[3 * kk], w1 = wsm4[3 * kk + 1], w2 = wsm4[3 * kk + 2];
    const uint32_t w[kBlJ] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w, w2.x, w2.y, w2.z, w2.w};
#pragma unroll
    for (int jj = 0; jj < kBlJ; ++jj) a[jj] += v * w[jj];
  };
  if (g.br[g.pr[gp].b].t < (1u << 20)) {
#pragma unroll 8
    for (uint32_t kk = 0; kk < F; ++kk) mac(kk);
  } else {
    const uint64_t R = (uint64_t)((1ull << 32) % q);
    uint32_t kk = 0;
#pragma unroll 2
    for (; kk + 3 <= F; kk += 3) {
      mac(kk);
      mac(kk + 1);
      mac(kk + 2);
#pragma unroll
      for (int jj = 0; jj < kBlJ; ++jj) a[jj] = (a[jj] >> 32) * R + (a[jj] & 0xffffffffull);
    }
    for (; kk < F; ++kk) mac(kk);
  }
#pragma unroll
  for (uint32_t jj = 0; jj < kBlJ; ++jj) {
    if (jj < jn) {
      unsigned long long* d = acc + (((uint64_t)blk * cols + j0 + jj) * g.ct_words) + (uint64_t)poly * n + xs;
      *d += a[jj] % q;
    }
  }
}

// finish of the baseline (matmul.cpp:464-476): reduce, then part0 +=
// NTT(Delta * INTT_t(all slots = bias[j])). Block per ((blk, j), gp).
__global__ void k_bl_finish(Geo g, const unsigned long long* __restrict__ acc, const int64_t* __restrict__ bias,
                            uint32_t cols, uint32_t* __restrict__ out, uint32_t S = 1, uint64_t slice_words = 0) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n;
  const uint64_t c = blockIdx.x / g.P;  // (blk * cols + j)
  const uint32_t gp = blockIdx.x % g.P;
  const PrimeInfo& pr = g.pr[gp];
  const BranchInfo& br = g.br[pr.b];
  const int64_t t = br.t;
  int64_t r = bias[c % cols] % t;
  if (r < 0) r += t;
  for (uint32_t s = threadIdx.x; s < n; s += blockDim.x) sm[g.index_map[s]] = (uint32_t)r;
  __syncthreads();
  ntt_inv_smem(sm, g.inv + (size_t)(g.P + pr.b) * n, br.t, n, g.logn, br.last, br.ninv);
  const uint32_t q = pr.q;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) sm[x] = mul_shoup(sm[x], pr.delta.x, pr.delta.y, q);
  __syncthreads();
  ntt_fwd_smem(sm, g.fwd + (size_t)gp * n, q, n, g.logn);
  const unsigned long long* a0 = acc + c * g.ct_words + (uint64_t)pr.poly0 * n;
  const unsigned long long* a1 = acc + c * g.ct_words + (uint64_t)pr.poly1 * n;
  uint32_t* o0 = out + c * g.ct_words + (uint64_t)pr.poly0 * n;
  uint32_t* o1 = out + c * g.ct_words + (uint64_t)pr.poly1 * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
    unsigned long long s0 = a0[x], s1 = a1[x];  // each copy < 2^40: the sum cannot wrap
    for (uint32_t k = 1; k < S; ++k) {
      s0 += a0[x + k * slice_words];
      s1 += a1[x + k * slice_words];
    }
    o0[x] = add_mod((uint32_t)(s0 % q), sm[x], q);
    o1[x] = (uint32_t)(s1 % q);
  }
}

// Public key coeff [b][2][L][n] u64 -> eval-form prepared [gp][part] in the
// pass-C transposed layout (prepare_public, context.cpp:175-187).
template <int LOGN>
__global__ void __launch_bounds__(Ntt<LOGN>::T) k_prepare_pk(Geo g, const uint64_t* __restrict__ pk0,
                                                            const uint64_t* __restrict__ pk1, uint2* __restrict__ out,
                                                            uint32_t* err) {
  using NT = Ntt<LOGN>;
  constexpr uint32_t N = NT::N, T = NT::T;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  const uint32_t gp = blockIdx.x / 2, part = blockIdx.x % 2;
  const PrimeInfo& pr = g.pr[gp];
  const uint64_t* src = (pr.b ? pk1 : pk0) + ((uint64_t)part * pr.L + pr.i) * N;
  const uint32_t j = threadIdx.x;
  uint32_t v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint64_t a = src[NT::posA(j, r)];
    if (a >= pr.q) *err = 1;
    v[r] = (uint32_t)a;
  }
  NT::fwd(v, sm, g.fwd + (size_t)gp * N, g.twc + (size_t)gp * g.twc_stride, pr.q);
  uint4* o = reinterpret_cast<uint4*>(out + (uint64_t)(2 * gp + part) * N) + j;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint32_t a = v[2 * c], bb = v[2 * c + 1];
    o[c * T] = make_uint4(a, (uint32_t)(((uint64_t)a << 32) / pr.q), bb, (uint32_t)(((uint64_t)bb << 32) / pr.q));
  }
}

// Generic (small-ring) versions of the baseline encoders, natural layouts.
__global__ void k_bl_encode_g(Geo g, const int64_t* __restrict__ x, uint64_t R, uint64_t f, uint64_t k0, uint32_t B,
                              uint32_t* __restrict__ m_out, int row_mode = 0) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n, e = blockIdx.x, b = blockIdx.y;
  const uint64_t eg = k0 + e;
  const uint64_t k = row_mode ? 0 : k0 + e / B;
  const uint64_t base = row_mode ? (eg / B) * f + (eg % B) * n : (uint64_t)(e % B) * n;
  const uint64_t lim = row_mode ? min((uint64_t)n, f - (eg % B) * n) : min((uint64_t)n, R - base);
  const BranchInfo& br = g.br[b];
  const int64_t t = br.t;
  for (uint32_t s = threadIdx.x; s < n; s += blockDim.x) {
    int64_t r = 0;
    if (s < lim) {
      r = (row_mode ? x[base + s] : x[(base + s) * f + k]) % t;
      if (r < 0) r += t;
    }
    sm[g.index_map[s]] = (uint32_t)r;
  }
  __syncthreads();
  ntt_inv_smem(sm, g.inv + (size_t)(g.P + b) * n, br.t, n, g.logn, br.last, br.ninv);
  uint32_t* o = m_out + ((uint64_t)e * 2 + b) * n;
  for (uint32_t s = threadIdx.x; s < n; s += blockDim.x) o[s] = sm[s];
}

__global__ void k_bl_encrypt_g(Geo g, const int8_t* __restrict__ noise, const uint32_t* __restrict__ m,
                               const uint2* __restrict__ pkd, uint32_t* __restrict__ cts) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n, e = blockIdx.x / g.P, gp = blockIdx.x % g.P;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, b = pr.b;
  const int8_t* nz = noise + ((uint64_t)e * 2 + b) * 3 * n;
  const uint32_t* mm = m + ((uint64_t)e * 2 + b) * n;
  const uint2* tw = g.fwd + (size_t)gp * n;
  uint32_t* c0 = cts + (uint64_t)e * g.ct_words + (uint64_t)pr.poly0 * n;
  uint32_t* c1 = cts + (uint64_t)e * g.ct_words + (uint64_t)pr.poly1 * n;
  const uint2* p0 = pkd + (uint64_t)(2 * gp) * n;
  const uint2* p1 = pkd + (uint64_t)(2 * gp + 1) * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) sm[x] = lift_small(nz[x], q);
  __syncthreads();
  ntt_fwd_smem(sm, tw, q, n, g.logn);
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
    c0[x] = mul_shoup(sm[x], p0[x].x, p0[x].y, q);
    c1[x] = mul_shoup(sm[x], p1[x].x, p1[x].y, q);
  }
  __syncthreads();
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x)
    sm[x] = add_mod(lift_small(nz[n + x], q), mul_shoup(mm[x], pr.delta.x, pr.delta.y, q), q);
  __syncthreads();
  ntt_fwd_smem(sm, tw, q, n, g.logn);
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) c0[x] = add_mod(c0[x], sm[x], q);
  __syncthreads();
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) sm[x] = lift_small(nz[2 * n + x], q);
  __syncthreads();
  ntt_fwd_smem(sm, tw, q, n, g.logn);
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) c1[x] = add_mod(c1[x], sm[x], q);
}

__global__ void k_prepare_pk_g(Geo g, const uint64_t* __restrict__ pk0, const uint64_t* __restrict__ pk1,
                               uint2* __restrict__ out, uint32_t* err) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n, gp = blockIdx.x / 2, part = blockIdx.x % 2;
  const PrimeInfo& pr = g.pr[gp];
  const uint64_t* src = (pr.b ? pk1 : pk0) + ((uint64_t)part * pr.L + pr.i) * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
    if (src[x] >= pr.q) *err = 1;
    sm[x] = (uint32_t)src[x];
  }
  __syncthreads();
  ntt_fwd_smem(sm, g.fwd + (size_t)gp * n, pr.q, n, g.logn);
  uint2* o = out + (uint64_t)(2 * gp + part) * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x)
    o[x] = make_uint2(sm[x], (uint32_t)(((uint64_t)sm[x] << 32) / pr.q));
}

// prepare_constant_signed (twin.cpp:424-436, context.cpp:120-137) for every
// (feature, class): centered residue mod t_b with its Shoup constant mod q_i.
__global__ void k_bl_weights(Geo g, const int64_t* __restrict__ w, uint64_t count, uint2* __restrict__ out) {
  const uint64_t total = count * g.P;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t gp = (uint32_t)(x % g.P);
    const PrimeInfo& pr = g.pr[gp];
    const int64_t t = g.br[pr.b].t;
    int64_t r = w[x / g.P] % t;
    if (r < 0) r += t;
    out[x] = make_uint2((uint32_t)r, (uint32_t)(((uint64_t)r << 32) / pr.q));
  }
}
