// Kernels on the 32-residue-per-thread NTT (ntt32.cuh): polynomial NTT (test
// seam), digit INTT and the TMEM key switch. Same arithmetic as the
// 16-residue kernels (BfvContext::apply_galois, proj/src/bfv/context.cpp:
// 428-507), bit-identical outputs; the point is the transform shape: no
// warp-shuffle stages (N = 16384 has two in ntt_fast.cuh) and twice the
// independent butterflies per thread.
//
// Key layout for these kernels (k_prepare_keys with V = 32): for slot
// x = 32 j + rr, the (value, Shoup) pair sits at uint2 index
// ((rr >> 1) * T + j) * 2 + (rr & 1), so thread j reads its 32 slots as 16
// coalesced uint4. TMEM: thread (warp w, lane t) owns lane 32*(w%4)+t and
// 64 columns at (w/4)*64: acc0 slots 0..31, then acc1.
// Textually included by heinfer_b200.cu after tmem_ks.cuh.
#pragma once

template <int LOGN>
__global__ void __launch_bounds__(Ntt32<LOGN>::T) k_poly_ntt32(Geo g, uint32_t gp, uint32_t* __restrict__ polys,
                                                              int inverse) {
  using NT = Ntt32<LOGN>;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  const uint32_t j = threadIdx.x, x0 = NT::posC0(j);
  uint32_t* p = polys + (uint64_t)blockIdx.x * NT::N;
  const PrimeInfo& pr = g.pr[gp];
  const uint2* tw = (inverse ? g.inv : g.fwd) + (size_t)gp * NT::N;
  uint32_t e[32];
  if (inverse) {
#pragma unroll
    for (int r = 0; r < 32; ++r) e[r] = p[x0 + r];
    NT::inv(e, sm, tw, tw, g.itwc32 + (size_t)gp * g.twc32_stride, pr.q, pr.last, pr.ninv);
#pragma unroll
    for (int r = 0; r < 32; ++r) p[NT::posA(j, r)] = e[r];
  } else {
#pragma unroll
    for (int r = 0; r < 32; ++r) e[r] = p[NT::posA(j, r)];
    NT::fwd(e, sm, tw, tw, g.twc32 + (size_t)gp * g.twc32_stride, pr.q);
#pragma unroll
    for (int r = 0; r < 32; ++r) p[x0 + r] = e[r];
  }
}

// digit_l = INTT_l(sigma(c1)_l) (context.cpp:445-470): c1 lands in shared
// memory by one TMA bulk copy, is gathered through the Galois permutation
// into registers, and the same buffer then serves the transform's exchanges.
template <int LOGN, bool PTW>
__global__ void __launch_bounds__(Ntt32<LOGN>::T) k_rot_digits32(Geo g, const uint32_t* __restrict__ dot,
                                                                const uint32_t* __restrict__ perm,
                                                                uint32_t* __restrict__ digits,
                                                                const __grid_constant__ TwArg<PTW> itab) {
  using NT = Ntt32<LOGN>;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  __shared__ uint64_t bar;
  const uint32_t pair = blockIdx.x / g.P, gp = blockIdx.x % g.P;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t* c1 = dot + (uint64_t)pair * g.ct_words + (uint64_t)pr.poly1 * NT::N;
  const uint32_t j = threadIdx.x, x0 = NT::posC0(j);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    bulk_load(sm, c1, NT::N * 4, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  uint32_t e[32];
  const uint4* pp = reinterpret_cast<const uint4*>(perm + x0);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint4 pm = __ldg(pp + c);
    e[4 * c] = sm[pm.x];
    e[4 * c + 1] = sm[pm.y];
    e[4 * c + 2] = sm[pm.z];
    e[4 * c + 3] = sm[pm.w];
  }
  const uint2* itg = g.inv + (size_t)gp * NT::N;
  // NT::inv starts with register stages and a barrier before its first store
  if constexpr (PTW)
    NT::inv(e, sm, ParamTw{itab.w[gp]}, itg, g.itwc32 + (size_t)gp * g.twc32_stride, pr.q, pr.last, pr.ninv);
  else
    NT::inv(e, sm, itg, itg, g.itwc32 + (size_t)gp * g.twc32_stride, pr.q, pr.last, pr.ninv);
  uint32_t* d = digits + ((uint64_t)pair * g.P + gp) * NT::N;
#pragma unroll
  for (int r = 0; r < 32; ++r) d[NT::posA(j, r)] = e[r];
}

template <int LOGN>
struct Tm32 {
  static constexpr uint32_t WARPS = Ntt32<LOGN>::T / 32;
  static constexpr uint32_t COLS = (WARPS / 4) * 64;  // 128 (N = 8192) or 256 (N = 16384)
};

template <int LOGN, bool PTW, int MINB>
__global__ void __launch_bounds__(Ntt32<LOGN>::T, MINB) k_rot_keyswitch_t32(Geo g, const uint32_t* __restrict__ dot,
                                                                          const uint32_t* __restrict__ digits,
                                                                          const uint32_t* __restrict__ perm,
                                                                          const uint2* __restrict__ key0,
                                                                          const uint2* __restrict__ key1,
                                                                          uint32_t* __restrict__ out, int fold,
                                                                          const __grid_constant__ TwArg<PTW> tab) {
  using NT = Ntt32<LOGN>;
  constexpr uint32_t N = NT::N, T = NT::T, COLS = Tm32<LOGN>::COLS;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  __shared__ uint64_t gbar;
  __shared__ uint32_t tbase;
  const uint32_t pair = blockIdx.x / g.P, gp = blockIdx.x % g.P;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, L = pr.L, i = pr.i;
  const uint32_t j = threadIdx.x, x0 = NT::posC0(j), warp = j >> 5;
  const uint32_t* ct = dot + (uint64_t)pair * g.ct_words;
  const uint32_t* c0 = ct + (uint64_t)pr.poly0 * N;
  const uint32_t* c1 = ct + (uint64_t)pr.poly1 * N;
  const uint2* key = (pr.b ? key1 : key0) + (uint64_t)i * L * 2 * N;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tbase)),
                 "n"(COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 32) {
    mbar_init(&gbar, 1);
    bulk_load(sm, c1, N * 4, &gbar);
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t ta = tbase + ((32u * (warp & 3u)) << 16) + 64u * (warp >> 2);  // acc0; acc1 at +32
  mbar_wait(&gbar, 0);
  const uint4* pp = reinterpret_cast<const uint4*>(perm + x0);
  {
    // l == i term: NTT_i(INTT_i(x)) = x, so sigma(c1)_i multiplies the key directly
    const uint4* k0 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * i) * N) + j;
    const uint4* k1 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * i + 1) * N) + j;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint32_t A[4], B[4];
      const uint4 pm = __ldg(pp + c);
      const uint32_t d0 = sm[pm.x], d1 = sm[pm.y], d2 = sm[pm.z], d3 = sm[pm.w];
      const uint4 a = __ldg(k0 + (2 * c) * T), b = __ldg(k0 + (2 * c + 1) * T);
      const uint4 u = __ldg(k1 + (2 * c) * T), v = __ldg(k1 + (2 * c + 1) * T);
      A[0] = mul_shoup(d0, a.x, a.y, q);
      A[1] = mul_shoup(d1, a.z, a.w, q);
      A[2] = mul_shoup(d2, b.x, b.y, q);
      A[3] = mul_shoup(d3, b.z, b.w, q);
      B[0] = mul_shoup(d0, u.x, u.y, q);
      B[1] = mul_shoup(d1, u.z, u.w, q);
      B[2] = mul_shoup(d2, v.x, v.y, q);
      B[3] = mul_shoup(d3, v.z, v.w, q);
      tm_st(ta + 4 * c, A);
      tm_st(ta + 32 + 4 * c, B);
    }
  }
  const uint32_t* dig = digits + ((uint64_t)pair * g.P + pr.first) * N;
  const uint4* tc = g.twc32 + (size_t)gp * g.twc32_stride;
  const uint2* twg = g.fwd + (size_t)gp * N;
  uint32_t e[32];
  for (uint32_t l = 0; l < L; ++l) {
    if (l == i) continue;
    {
      const uint32_t* src = dig + (uint64_t)l * N;
      if (pr.fast_reduce) {
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const uint32_t v = src[NT::posA(j, r)];
          e[r] = min(v, v - q);
        }
      } else {
#pragma unroll
        for (int r = 0; r < 32; ++r) e[r] = src[NT::posA(j, r)] % q;
      }
    }
    if constexpr (PTW)
      NT::template fwd<true>(e, sm, ParamTw{tab.w[gp]}, twg, tc, q);
    else
      NT::template fwd<true>(e, sm, twg, twg, tc, q);
    const uint4* k0 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * l) * N) + j;
    const uint4* k1 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * l + 1) * N) + j;
    tm_wait_st();  // the previous digit's accumulator stores have landed
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint32_t A[4], B[4];
      tm_ld(ta + 4 * c, A);
      tm_ld(ta + 32 + 4 * c, B);
      tm_wait_ld(A, B);
      const uint4 a = __ldg(k0 + (2 * c) * T), b = __ldg(k0 + (2 * c + 1) * T);
      A[0] = add_mod(A[0], mul_shoup(e[4 * c], a.x, a.y, q), q);
      A[1] = add_mod(A[1], mul_shoup(e[4 * c + 1], a.z, a.w, q), q);
      A[2] = add_mod(A[2], mul_shoup(e[4 * c + 2], b.x, b.y, q), q);
      A[3] = add_mod(A[3], mul_shoup(e[4 * c + 3], b.z, b.w, q), q);
      const uint4 u = __ldg(k1 + (2 * c) * T), v = __ldg(k1 + (2 * c + 1) * T);
      B[0] = add_mod(B[0], mul_shoup(e[4 * c], u.x, u.y, q), q);
      B[1] = add_mod(B[1], mul_shoup(e[4 * c + 1], u.z, u.w, q), q);
      B[2] = add_mod(B[2], mul_shoup(e[4 * c + 2], v.x, v.y, q), q);
      B[3] = add_mod(B[3], mul_shoup(e[4 * c + 3], v.z, v.w, q), q);
      tm_st(ta + 4 * c, A);
      tm_st(ta + 32 + 4 * c, B);
    }
  }
  uint32_t* o = out + (uint64_t)pair * g.ct_words;
  __syncthreads();  // the last NTT's exchange reads of sm are done
  if (threadIdx.x == 0) {
    fence_proxy_async_smem();
    bulk_load(sm, c0, N * 4, &gbar);
  }
  tm_wait_st();
  mbar_wait(&gbar, 1);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    uint32_t A[4], B[4];
    tm_ld(ta + 4 * c, A);
    tm_ld(ta + 32 + 4 * c, B);
    tm_wait_ld(A, B);
    const uint4 pm = __ldg(pp + c);
    A[0] = add_mod(A[0], sm[pm.x], q);
    A[1] = add_mod(A[1], sm[pm.y], q);
    A[2] = add_mod(A[2], sm[pm.z], q);
    A[3] = add_mod(A[3], sm[pm.w], q);
    if (fold) {
      const uint4 u = *reinterpret_cast<const uint4*>(sm + x0 + 4 * c);
      const uint4 v = *reinterpret_cast<const uint4*>(c1 + x0 + 4 * c);
      A[0] = add_mod(A[0], u.x, q);
      A[1] = add_mod(A[1], u.y, q);
      A[2] = add_mod(A[2], u.z, q);
      A[3] = add_mod(A[3], u.w, q);
      B[0] = add_mod(B[0], v.x, q);
      B[1] = add_mod(B[1], v.y, q);
      B[2] = add_mod(B[2], v.z, q);
      B[3] = add_mod(B[3], v.w, q);
    }
    *reinterpret_cast<uint4*>(o + (uint64_t)pr.poly0 * N + x0 + 4 * c) = make_uint4(A[0], A[1], A[2], A[3]);
    *reinterpret_cast<uint4*>(o + (uint64_t)pr.poly1 * N + x0 + 4 * c) = make_uint4(B[0], B[1], B[2], B[3]);
  }
  tm_fence_before();
  __syncthreads();
  if (warp == 0) {
    tm_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(COLS) : "memory");
  }
}
