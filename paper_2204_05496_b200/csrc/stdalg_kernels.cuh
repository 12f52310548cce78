// Standard-algorithm and client-encryption kernels (baseline_matmul,
// matmul.cpp:273-344; encrypt_parts, context.cpp:262-303). The mt19937_64
// replay and the noise sampler live in baseline.cuh. Textually included by
// heinfer_b200.cu inside its kernel namespace.
#pragma once

// ---------------------------------------------------------------------------
// Standard algorithm (baseline_matmul) kernels; see baseline.cuh.
// ---------------------------------------------------------------------------
// m = INTT_t(scatter(centered residues of x[base + s][k])) per (encryption,
// branch); encryption e = kk * B + blk (matmul.cpp:302-310 loop order).
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
  // row mode (encode_inputs, matmul.cpp:59-69): encryption k0 + e is chunk
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

// ---------------------------------------------------------------------------
// Standard algorithm by linearity (the path hei_gpu_baseline_matmul runs).
//
// The reference accumulates, per output (row block blk, class j) and prime
// q_i, acc = sum_k ct_k (x) w'_kj with ct_k = Enc(m_k; u_k, e0_k, e1_k) and
// w'_kj = [w_kj]_t the constant plaintext (prepare_constant_signed,
// twin.cpp:131-143; context.cpp:120-137), i.e. in eval form
//   acc.c0 = sum_k w'_kj (NTT(u_k) pk0 + NTT(e0_k + Delta m_k))
//   acc.c1 = sum_k w'_kj (NTT(u_k) pk1 + NTT(e1_k))          mod q_i
// (encrypt_parts, context.cpp:262-303; mul_plain + add_inplace,
// matmul.cpp:303-320). Every step is exact arithmetic mod q_i and the NTT is
// linear, so the same residues are
//   acc.c0 = NTT([sum_k w' u_k]) pk0 + NTT([sum_k w' e0_k] + Delta [sum_k w' m_k])
//   acc.c1 = NTT([sum_k w' u_k]) pk1 + NTT([sum_k w' e1_k])
// -- three transforms per (blk, j, prime) instead of 3 + 2 per (feature,
// prime). The sums over features are exact integer sums of the SAME sampled
// noise (the full util::Prng stream is still drawn and consumed in order) and
// the same encoded columns m_k = INTT_t(column k), reduced mod q_i at the end.
// ---------------------------------------------------------------------------

// Noise of one encryption per (e, branch), packed: raw draws [3][N] ->
// u32 [N] with byte 0 = u + 1, byte 1 = e0, byte 2 = e1 (sample_ternary,
// sample_gaussian twice; sampling.cpp:16-34). A thread takes coefficient pair
// (2k, 2k+1): the Box-Muller pair of Prng::gaussian (cos first, sin as the
// cached spare, rng.hpp:47-62). A rejection would shift the stream: flagged.
__global__ void k_bl_noise_p(const uint64_t* __restrict__ raw, uint64_t count, uint32_t n,
                             uint32_t* __restrict__ noisep, uint32_t* err) {
  const uint32_t e = blockIdx.x, b = blockIdx.y;
  const uint64_t* d = raw + (uint64_t)b * count + (uint64_t)e * 3 * n;
  uint2* o = reinterpret_cast<uint2*>(noisep + ((uint64_t)e * 2 + b) * n);
  for (uint32_t k = threadIdx.x; k < n / 2; k += blockDim.x) {
    const uint64_t v0 = d[2 * k], v1 = d[2 * k + 1];
    if (v0 == ~0ull || v1 == ~0ull) *err = 1;
    int8_t a0, a1, c0, c1;
    bool ok = heb_baseline::box_muller_pair(d[n + 2 * k], d[n + 2 * k + 1], a0, a1);
    ok &= heb_baseline::box_muller_pair(d[2 * n + 2 * k], d[2 * n + 2 * k + 1], c0, c1);
    if (!ok) *err = 1;
    const uint32_t u0 = (uint32_t)(v0 % 3), u1 = (uint32_t)(v1 % 3);  // u + 1
    o[k] = make_uint2(u0 | ((uint32_t)(uint8_t)a0 << 8) | ((uint32_t)(uint8_t)c0 << 16),
                      u1 | ((uint32_t)(uint8_t)a1 << 8) | ((uint32_t)(uint8_t)c1 << 16));
  }
}

// Feature sums of one batch: thread per coefficient x, block per (x tile,
// class group of J, feature slice s, row block, branch). Five exact int64
// sums per class: su = sum w' u, se0 = sum w' e0, se1 = sum w' e1 and the
// column sum sum w' m split as w' = wh 2^15 + wl (m < t < 2^31, so every
// product is < 2^46 and 2^17 features stay below 2^63). sums layout
// [s][blk][j][b][5][n]; each element has one owner per launch (plain RMW).
constexpr int kBlSumJ = 4;
__global__ void __launch_bounds__(128) k_bl_sums(Geo g, const uint32_t* __restrict__ noisep,
                                                 const uint32_t* __restrict__ m, uint32_t Fb, uint32_t B,
                                                 uint32_t cols, const uint2* __restrict__ wc,
                                                 long long* __restrict__ sums) {
  constexpr int J = kBlSumJ;
  __shared__ uint32_t wsm[1024 * J];
  const uint32_t n = g.n, G = (cols + J - 1) / J;
  const uint32_t tile = blockIdx.x / G, grp = blockIdx.x - tile * G;
  const uint32_t x = tile * blockDim.x + threadIdx.x;
  const uint32_t blk = blockIdx.z >> 1, b = blockIdx.z & 1, S = gridDim.y, s = blockIdx.y;
  const uint32_t k_lo = (uint32_t)((uint64_t)Fb * s / S), k_hi = (uint32_t)((uint64_t)Fb * (s + 1) / S);
  const uint32_t j0 = grp * J, jn = min((uint32_t)J, cols - j0);
  const uint32_t gp0 = b ? g.L[0] : 0;  // w' = [w]_t is the same value for every prime of the branch
  for (uint32_t i = threadIdx.x; i < (k_hi - k_lo) * J; i += blockDim.x) {
    const uint32_t kk = i / J, jj = i - kk * J;
    wsm[i] = jj < jn ? wc[((uint64_t)(k_lo + kk) * cols + j0 + jj) * g.P + gp0].x : 0u;
  }
  __syncthreads();
  long long su[J], s0[J], s1[J];
  unsigned long long ml[J], mh[J];
#pragma unroll
  for (int jj = 0; jj < J; ++jj) su[jj] = s0[jj] = s1[jj] = 0, ml[jj] = mh[jj] = 0;
  const uint64_t estride = (uint64_t)B * 2 * n;
  const uint32_t* np = noisep + ((uint64_t)(k_lo * B + blk) * 2 + b) * n + x;
  const uint32_t* mp = m + ((uint64_t)(k_lo * B + blk) * 2 + b) * n + x;
#pragma unroll 4
  for (uint32_t kk = 0; kk < k_hi - k_lo; ++kk) {
    const uint32_t pk = __ldg(np + kk * estride);
    const uint32_t mv = __ldg(mp + kk * estride);
    const int u = (int)(pk & 0xff) - 1, e0 = (int8_t)(pk >> 8), e1 = (int8_t)(pk >> 16);
    const uint4 w4 = *reinterpret_cast<const uint4*>(wsm + kk * J);
    const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
      const int wi = (int)w[jj];  // w' < t < 2^31
      su[jj] += (long long)wi * u;
      s0[jj] += (long long)wi * e0;
      s1[jj] += (long long)wi * e1;
      ml[jj] += (unsigned long long)mv * (w[jj] & 0x7fffu);
      mh[jj] += (unsigned long long)mv * (w[jj] >> 15);
    }
  }
  if (x >= n) return;
#pragma unroll
  for (int jj = 0; jj < J; ++jj) {
    if ((uint32_t)jj >= jn) break;
    long long* o = sums + ((((uint64_t)s * B + blk) * cols + j0 + jj) * 2 + b) * 5 * n + x;
    o[0] += su[jj];
    o[n] += s0[jj];
    o[2 * (uint64_t)n] += s1[jj];
    o[3 * (uint64_t)n] += (long long)ml[jj];
    o[4 * (uint64_t)n] += (long long)mh[jj];
  }
}

// Fold the int64 feature sums (all S slices) into residues mod every prime
// of the branch: res [blk*cols + j][gp][3][n] u32, accumulated mod q:
// [su], [se0 + Delta (ml + mh 2^15)], [se1]. Run at least every 2^17
// features and at the end; the caller zeroes `sums` afterwards.
__global__ void k_bl_fold_sums(Geo g, const long long* __restrict__ sums, uint32_t S, uint32_t B, uint32_t cols,
                               uint32_t* __restrict__ res) {
  const uint32_t n = g.n;
  const uint64_t total = (uint64_t)B * cols * g.P * n;
  for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = (uint32_t)(idx % n);
    const uint64_t cg = idx / n;
    const uint32_t gp = (uint32_t)(cg % g.P);
    const uint64_t c = cg / g.P;  // blk * cols + j
    const PrimeInfo& pr = g.pr[gp];
    const uint32_t q = pr.q;
    long long a[5] = {0, 0, 0, 0, 0};
    for (uint32_t s = 0; s < S; ++s) {
      const long long* p = sums + (((uint64_t)s * B * cols + c) * 2 + pr.b) * 5 * n + x;
#pragma unroll
      for (int k = 0; k < 5; ++k) a[k] += p[(uint64_t)k * n];
    }
    auto smod = [q](long long v) -> uint32_t {
      long long r = v % (long long)q;
      return (uint32_t)(r < 0 ? r + q : r);
    };
    const uint32_t ml = (uint32_t)((unsigned long long)a[3] % q), mh = (uint32_t)((unsigned long long)a[4] % q);
    const uint32_t mm = (uint32_t)(((uint64_t)mh << 15) % q);
    const uint32_t msum = add_mod(ml, mm, q);
    uint32_t* r = res + (c * g.P + gp) * 3 * n + x;
    r[0] = add_mod(r[0], smod(a[0]), q);
    r[n] = add_mod(r[n], add_mod(smod(a[1]), mul_shoup(msum, pr.delta.x, pr.delta.y, q), q), q);
    r[2 * n] = add_mod(r[2 * n], smod(a[2]), q);
  }
}

// Finish per ((blk, j), prime): c0 = NTT(A) NTT(pk0) + NTT(Bv) + [Delta r_j],
// c1 = NTT(A) NTT(pk1) + NTT(Cv), with (A, Bv, Cv) the folded residues and
// r_j = [bias_j]_t: the bias plaintext (all slots r_j) is the constant
// polynomial r_j, so NTT(Delta r_j) is Delta r_j in every slot
// (add_plain_inplace, context.cpp:393-402; matmul.cpp:327-334).
// pk is the coefficient-form public key [b][part][prime][n] u64.
__global__ void k_bl_finish_lin(Geo g, const uint32_t* __restrict__ res, const uint64_t* __restrict__ pk0,
                                const uint64_t* __restrict__ pk1, const int64_t* __restrict__ bias, uint32_t cols,
                                uint32_t* __restrict__ out) {
  extern __shared__ uint32_t smf[];
  const uint32_t n = g.n;
  uint32_t *S1 = smf, *S2 = smf + n, *S3 = smf + 2 * n;
  const uint64_t c = blockIdx.x / g.P;
  const uint32_t gp = blockIdx.x % g.P;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q;
  const uint2* tw = g.fwd + (size_t)gp * n;
  const uint32_t* r = res + (c * g.P + gp) * 3 * n;
  const uint64_t* pk = (pr.b ? pk1 : pk0);
  int64_t bt = bias[c % cols] % (int64_t)g.br[pr.b].t;
  if (bt < 0) bt += g.br[pr.b].t;
  const uint32_t bd = mul_shoup((uint32_t)bt, pr.delta.x, pr.delta.y, q);
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) S1[x] = r[x];
  __syncthreads();
  ntt_fwd_smem(S1, tw, q, n, g.logn);
  for (int part = 0; part < 2; ++part) {
    for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
      S2[x] = (uint32_t)pk[((uint64_t)part * pr.L + pr.i) * n + x];
      S3[x] = r[(uint64_t)(1 + part) * n + x];
    }
    __syncthreads();
    ntt_fwd_smem(S2, tw, q, n, g.logn);
    ntt_fwd_smem(S3, tw, q, n, g.logn);
    uint32_t* o = out + c * g.ct_words + (uint64_t)(part ? pr.poly1 : pr.poly0) * n;
    for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
      uint32_t v = add_mod(mul_barrett(S1[x], S2[x], q, pr.mu), S3[x], q);
      o[x] = part ? v : add_mod(v, bd, q);
    }
    __syncthreads();
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

// prepare_constant_signed (twin.cpp:131-143, context.cpp:120-137) for every
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
