// Key switch with the two accumulator polynomials in tensor memory (TMEM).
//
// Same arithmetic as k_rot_keyswitch_s (BfvContext::apply_galois,
// proj/src/bfv/context.cpp:428-507; every sum exact mod q_i, so the output is
// bit-identical), but acc0/acc1 (2 x N u32 per (pair, prime) block) live in
// TMEM instead of shared memory. TMEM is otherwise idle in this integer
// kernel; moving the accumulators there removes 16 128-bit shared-memory
// accesses per thread per digit from the L1/shared pipe and leaves shared
// memory with just the NTT exchange buffer (N words) and the c1/c0 staging.
//
// Layout: the CTA allocates 128 columns. Warp w may only touch TMEM lanes
// 32*(w%4) .. +31 (its lane quarter), so the four warps sharing a quarter take
// 32-column blocks (w/4)*32: thread t of warp w owns lane 32*(w%4)+t, columns
// [ (w/4)*32, +16 ) for acc0's 16 slots and [ +16, +32 ) for acc1's.
// Textually included by heinfer_b200.cu after fold_kernels.cuh.
#pragma once

template <int X>
__device__ __forceinline__ void tm_ld(uint32_t taddr, uint32_t (&v)[X]) {
  if constexpr (X == 8)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
  else
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
}
template <int X>
__device__ __forceinline__ void tm_st(uint32_t taddr, const uint32_t (&v)[X]) {
  if constexpr (X == 8)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
  else
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3])
                 : "memory");
}
// wait::ld, threading the loaded registers through so no use is scheduled
// before the wait.
template <int X>
__device__ __forceinline__ void tm_wait_ld(uint32_t (&a)[X], uint32_t (&b)[X]) {
  if constexpr (X == 8)
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
                   "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]), "+r"(b[7])
                 :
                 : "memory");
  else
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3])
                 :
                 : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }


// N = 8192 full batches: 512 threads, 40 registers, 3 CTAs per SM (the
// launch bound), accumulators exchanged with TMEM in rounds of GS = 4 slots
// (tcgen05.ld/st 32x32b.x4). c1 (for the l == i term) and c0 (for the
// epilogue) are staged in the exchange buffer by TMA bulk copies so the
// Galois gathers read shared memory.
__global__ void __launch_bounds__(512, 3) k_rot_keyswitch_t(Geo g, const uint32_t* __restrict__ dot,
                                                          const uint32_t* __restrict__ digits,
                                                          const uint32_t* __restrict__ perm,
                                                          const uint2* __restrict__ key0,
                                                          const uint2* __restrict__ key1,
                                                          uint32_t* __restrict__ out, int fold,
                                                          const __grid_constant__ TwAB tab) {
  using NT = Ntt<13>;
  constexpr int GS = 4;
  constexpr uint32_t kTmemCols = NT::T / 4;  // 32 columns per warp, warps of a lane quarter side by side
  constexpr uint32_t N = NT::N, T = NT::T;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  __shared__ uint64_t gbar;
  __shared__ uint32_t tbase;
  uint32_t pair, gp;
  block_pair_prime(g, pair, gp);
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, L = pr.L, i = pr.i;
  const uint32_t j = threadIdx.x, x0 = NT::posC0(j), warp = j >> 5;
  const uint32_t* dig = digits + ((uint64_t)pair * g.P + pr.first) * N;
  const uint32_t* ct = dot + (uint64_t)pair * g.ct_words;
  const uint32_t* c0 = ct + (uint64_t)pr.poly0 * N;
  const uint32_t* c1 = ct + (uint64_t)pr.poly1 * N;
  const uint2* key = (pr.b ? key1 : key0) + (uint64_t)i * L * 2 * N;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tbase)),
                 "n"(kTmemCols)
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
  const uint32_t ta = tbase + ((32u * (warp & 3u)) << 16) + 32u * (warp >> 2);  // acc0 cols; acc1 at +16
  mbar_wait(&gbar, 0);
  const uint4* pp = reinterpret_cast<const uint4*>(perm + x0);
  {
    // l == i term: NTT_i(INTT_i(x)) = x, so sigma(c1)_i multiplies the key directly
    const uint4* k0 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * i) * N) + j;
    const uint4* k1 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * i + 1) * N) + j;
#pragma unroll
    for (int h = 0; h < 16 / GS; ++h) {
      uint32_t A[GS], B[GS];
#pragma unroll
      for (int c = h * GS / 4; c < (h + 1) * GS / 4; ++c) {
        const uint4 pm = __ldg(pp + c);
        const uint32_t d0 = sm[pm.x], d1 = sm[pm.y], d2 = sm[pm.z], d3 = sm[pm.w];
        const uint4 a = __ldg(k0 + (2 * c) * T), b = __ldg(k0 + (2 * c + 1) * T);
        const uint4 u = __ldg(k1 + (2 * c) * T), v = __ldg(k1 + (2 * c + 1) * T);
        const int o = 4 * c - GS * h;
        A[o] = mul_shoup(d0, a.x, a.y, q);
        A[o + 1] = mul_shoup(d1, a.z, a.w, q);
        A[o + 2] = mul_shoup(d2, b.x, b.y, q);
        A[o + 3] = mul_shoup(d3, b.z, b.w, q);
        B[o] = mul_shoup(d0, u.x, u.y, q);
        B[o + 1] = mul_shoup(d1, u.z, u.w, q);
        B[o + 2] = mul_shoup(d2, v.x, v.y, q);
        B[o + 3] = mul_shoup(d3, v.z, v.w, q);
      }
      tm_st(ta + GS * h, A);
      tm_st(ta + 16 + GS * h, B);
    }
  }
  const uint4* twc = g.twc + (size_t)gp * g.twc_stride;
  uint32_t e[16];
  const uint32_t lastl = i == L - 1 ? L - 2 : L - 1;  // the last digit besides l == i
  if (L == 1) {  // no other digit: stage c0 right away
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_proxy_async_smem();
      bulk_load(sm, c0, N * 4, &gbar);
    }
  }
  for (uint32_t l = 0; l < L; ++l) {
    if (l == i) continue;
    const uint32_t* src = dig + (uint64_t)l * N;
    // A digit enters the transform unreduced: its residues are < q_l < 2^31, and
    // with u < max(q_i, q_l) every butterfly sum stays below q_l + q_i < 2^32, each
    // conditional subtraction brings it back under max(q_i, q_l), and the lazy
    // outputs only feed Shoup products (exact for any 32-bit input): congruent
    // throughout, so the reduced key products are the reference's values.
#pragma unroll
    for (int r = 0; r < 16; ++r) e[r] = src[NT::posA(j, r)];
    NT::template fwd<true, ParamTw, true, true>(e, sm, ParamTw{tab.w[gp]}, twc, q);
    if (l == lastl) {
      // the last transform's exchange reads are done: stage c0 for the
      // epilogue now, under this digit's key products
      __syncthreads();
      if (threadIdx.x == 0) {
        fence_proxy_async_smem();
        bulk_load(sm, c0, N * 4, &gbar);
      }
    }
    const uint4* k0 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * l) * N) + j;
    const uint4* k1 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * l + 1) * N) + j;
    tm_wait_st();  // the previous digit's accumulator stores have landed
#pragma unroll
    for (int h = 0; h < 16 / GS; ++h) {
      uint32_t A[GS], B[GS];
      tm_ld(ta + GS * h, A);
      tm_ld(ta + 16 + GS * h, B);
      tm_wait_ld(A, B);
#pragma unroll
      for (int c = h * GS / 4; c < (h + 1) * GS / 4; ++c) {
        const uint4 a = __ldg(k0 + (2 * c) * T), b = __ldg(k0 + (2 * c + 1) * T);
        const int o = 4 * c - GS * h;
        A[o] = add_mod(A[o], mul_shoup(e[4 * c], a.x, a.y, q), q);
        A[o + 1] = add_mod(A[o + 1], mul_shoup(e[4 * c + 1], a.z, a.w, q), q);
        A[o + 2] = add_mod(A[o + 2], mul_shoup(e[4 * c + 2], b.x, b.y, q), q);
        A[o + 3] = add_mod(A[o + 3], mul_shoup(e[4 * c + 3], b.z, b.w, q), q);
        const uint4 u = __ldg(k1 + (2 * c) * T), v = __ldg(k1 + (2 * c + 1) * T);
        B[o] = add_mod(B[o], mul_shoup(e[4 * c], u.x, u.y, q), q);
        B[o + 1] = add_mod(B[o + 1], mul_shoup(e[4 * c + 1], u.z, u.w, q), q);
        B[o + 2] = add_mod(B[o + 2], mul_shoup(e[4 * c + 2], v.x, v.y, q), q);
        B[o + 3] = add_mod(B[o + 3], mul_shoup(e[4 * c + 3], v.z, v.w, q), q);
      }
      tm_st(ta + GS * h, A);
      tm_st(ta + 16 + GS * h, B);
    }
  }
  uint32_t* o = out + (uint64_t)pair * g.ct_words;
  // the fold's c1 slots (e is dead: 16 free registers), issued ahead of the
  // waits on the accumulator stores and the c0 copy
  uint4 fv[4];
  if (fold) {
#pragma unroll
    for (int c = 0; c < 4; ++c) fv[c] = *reinterpret_cast<const uint4*>(c1 + x0 + 4 * c);
  }
  tm_wait_st();
  mbar_wait(&gbar, 1);
#pragma unroll
  for (int h = 0; h < 16 / GS; ++h) {
    uint32_t A[GS], B[GS];
    tm_ld(ta + GS * h, A);
    tm_ld(ta + 16 + GS * h, B);
    tm_wait_ld(A, B);
#pragma unroll
    for (int c = h * GS / 4; c < (h + 1) * GS / 4; ++c) {
      const uint4 pm = __ldg(pp + c);
      const int k = 4 * c - GS * h;
      A[k] = add_mod(A[k], sm[pm.x], q);
      A[k + 1] = add_mod(A[k + 1], sm[pm.y], q);
      A[k + 2] = add_mod(A[k + 2], sm[pm.z], q);
      A[k + 3] = add_mod(A[k + 3], sm[pm.w], q);
      if (fold) {
        const uint4 u = *reinterpret_cast<const uint4*>(sm + x0 + 4 * c);
        const uint4 v = fv[c];
        A[k] = add_mod(A[k], u.x, q);
        A[k + 1] = add_mod(A[k + 1], u.y, q);
        A[k + 2] = add_mod(A[k + 2], u.z, q);
        A[k + 3] = add_mod(A[k + 3], u.w, q);
        B[k] = add_mod(B[k], v.x, q);
        B[k + 1] = add_mod(B[k + 1], v.y, q);
        B[k + 2] = add_mod(B[k + 2], v.z, q);
        B[k + 3] = add_mod(B[k + 3], v.w, q);
      }
      *reinterpret_cast<uint4*>(o + (uint64_t)pr.poly0 * N + x0 + 4 * c) = make_uint4(A[k], A[k + 1], A[k + 2], A[k + 3]);
      *reinterpret_cast<uint4*>(o + (uint64_t)pr.poly1 * N + x0 + 4 * c) = make_uint4(B[k], B[k + 1], B[k + 2], B[k + 3]);
    }
  }
  tm_fence_before();
  __syncthreads();
  if (warp == 0) {
    tm_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmemCols) : "memory");
  }
  if (gp == 0) count_ops(g, 0, 1, fold ? 1 : 0);  // one rotation (+ the fold add) per pair (backend.cpp:63-73)
}


// Fused digit INTT + key switch over a thread-block cluster (one cluster of
// L CTAs per (pair, branch); CTA i owns output prime i). CTA i gathers
// sigma(c1)_i, does the l == i key products from it, inverse-transforms it
// into digit_i and keeps the digit in its own shared memory; after a cluster
// barrier every CTA reads the other L - 1 digits from its peers through
// distributed shared memory (no digit polynomial in HBM), then proceeds as
// k_rot_keyswitch_t (TMEM accumulators, same arithmetic: bit-identical).
// Measured against the two-kernel path in DESIGN.md §6.3 (HEI_KS_CLUSTER=1).
template <int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(512, 3)
    k_rot_keyswitch_c(Geo g, const uint32_t* __restrict__ dot, const uint32_t* __restrict__ perm,
                      const uint2* __restrict__ keyb, uint32_t* __restrict__ out, int fold, uint32_t gp0,
                      const __grid_constant__ TwAB tab) {
  using NT = Ntt<13>;
  constexpr int GS = 4;
  constexpr uint32_t kTmemCols = NT::T / 4;
  constexpr uint32_t N = NT::N, T = NT::T;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);  // exchange buffer (N words)
  uint4* dbuf = smem4 + N / 4;                         // this CTA's digit, [c][T] uint4 (N words)
  __shared__ uint64_t gbar;
  __shared__ uint32_t tbase;
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t i = cl.block_rank(), pair = blockIdx.x / CL, gp = gp0 + i;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, L = pr.L;
  const uint32_t j = threadIdx.x, x0 = NT::posC0(j), warp = j >> 5;
  const uint32_t* ct = dot + (uint64_t)pair * g.ct_words;
  const uint32_t* c0 = ct + (uint64_t)pr.poly0 * N;
  const uint32_t* c1 = ct + (uint64_t)pr.poly1 * N;
  const uint2* key = keyb + (uint64_t)i * L * 2 * N;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tbase)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 32) mbar_init(&gbar, 1);
  uint32_t e[16];
  {
    // sigma(c1)_i: the thread's one aligned 16-slot source group, permuted
    // through its own column of the exchange buffer (no barrier)
    uint32_t pm[16];
    load16_ro(perm + x0, pm);
    const uint4* gs4 = reinterpret_cast<const uint4*>(c1 + (pm[0] & ~15u));
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 v = __ldg(gs4 + c);
      sm[(4 * c) * T + j] = v.x;
      sm[(4 * c + 1) * T + j] = v.y;
      sm[(4 * c + 2) * T + j] = v.z;
      sm[(4 * c + 3) * T + j] = v.w;
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) e[r] = sm[(pm[r] & 15u) * T + j];
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t ta = tbase + ((32u * (warp & 3u)) << 16) + 32u * (warp >> 2);  // acc0 cols; acc1 at +16
  {
    // l == i term: NTT_i(INTT_i(x)) = x, so sigma(c1)_i multiplies the key directly
    const uint4* k0 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * i) * N) + j;
    const uint4* k1 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * i + 1) * N) + j;
#pragma unroll
    for (int h = 0; h < 16 / GS; ++h) {
      uint32_t A[GS], B[GS];
      const uint4 a = __ldg(k0 + (2 * h) * T), b = __ldg(k0 + (2 * h + 1) * T);
      const uint4 u = __ldg(k1 + (2 * h) * T), v = __ldg(k1 + (2 * h + 1) * T);
      A[0] = mul_shoup(e[4 * h], a.x, a.y, q);
      A[1] = mul_shoup(e[4 * h + 1], a.z, a.w, q);
      A[2] = mul_shoup(e[4 * h + 2], b.x, b.y, q);
      A[3] = mul_shoup(e[4 * h + 3], b.z, b.w, q);
      B[0] = mul_shoup(e[4 * h], u.x, u.y, q);
      B[1] = mul_shoup(e[4 * h + 1], u.z, u.w, q);
      B[2] = mul_shoup(e[4 * h + 2], v.x, v.y, q);
      B[3] = mul_shoup(e[4 * h + 3], v.z, v.w, q);
      tm_st(ta + GS * h, A);
      tm_st(ta + 16 + GS * h, B);
    }
  }
  // digit_i = INTT_i(sigma(c1)_i), kept in this CTA's shared memory
  NT::inv(e, sm, g.inv + (size_t)gp * N, g.itwc + (size_t)gp * g.twc_stride, q, pr.last, pr.ninv);
#pragma unroll
  for (int c = 0; c < 4; ++c) dbuf[c * T + j] = make_uint4(e[4 * c], e[4 * c + 1], e[4 * c + 2], e[4 * c + 3]);
  cl.sync();  // every digit of the (pair, branch) is published
  const uint4* twc = g.twc + (size_t)gp * g.twc_stride;
  for (uint32_t l = 0; l < L; ++l) {
    if (l == i) continue;
    const uint4* pd = cl.map_shared_rank(dbuf, l);
    // only the first stage's u operands (r < 8) must be reduced mod q_i
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 v = pd[c * T + j];
      e[4 * c] = v.x;
      e[4 * c + 1] = v.y;
      e[4 * c + 2] = v.z;
      e[4 * c + 3] = v.w;
    }
    // (the digit enters unreduced, as in k_rot_keyswitch_t)
    NT::template fwd<true>(e, sm, ParamTw{tab.w[gp]}, twc, q);
    const uint4* k0 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * l) * N) + j;
    const uint4* k1 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * l + 1) * N) + j;
    tm_wait_st();
#pragma unroll
    for (int h = 0; h < 16 / GS; ++h) {
      uint32_t A[GS], B[GS];
      tm_ld(ta + GS * h, A);
      tm_ld(ta + 16 + GS * h, B);
      tm_wait_ld(A, B);
      const uint4 a = __ldg(k0 + (2 * h) * T), b = __ldg(k0 + (2 * h + 1) * T);
      A[0] = add_mod(A[0], mul_shoup(e[4 * h], a.x, a.y, q), q);
      A[1] = add_mod(A[1], mul_shoup(e[4 * h + 1], a.z, a.w, q), q);
      A[2] = add_mod(A[2], mul_shoup(e[4 * h + 2], b.x, b.y, q), q);
      A[3] = add_mod(A[3], mul_shoup(e[4 * h + 3], b.z, b.w, q), q);
      const uint4 u = __ldg(k1 + (2 * h) * T), v = __ldg(k1 + (2 * h + 1) * T);
      B[0] = add_mod(B[0], mul_shoup(e[4 * h], u.x, u.y, q), q);
      B[1] = add_mod(B[1], mul_shoup(e[4 * h + 1], u.z, u.w, q), q);
      B[2] = add_mod(B[2], mul_shoup(e[4 * h + 2], v.x, v.y, q), q);
      B[3] = add_mod(B[3], mul_shoup(e[4 * h + 3], v.z, v.w, q), q);
      tm_st(ta + GS * h, A);
      tm_st(ta + 16 + GS * h, B);
    }
  }
  uint32_t* o = out + (uint64_t)pair * g.ct_words;
  __syncthreads();  // the last NTT's exchange reads of sm are done
  if (threadIdx.x == 0) {
    fence_proxy_async_smem();
    bulk_load(sm, c0, N * 4, &gbar);
  }
  tm_wait_st();
  mbar_wait(&gbar, 0);
  const uint4* pp = reinterpret_cast<const uint4*>(perm + x0);
#pragma unroll
  for (int h = 0; h < 16 / GS; ++h) {
    uint32_t A[GS], B[GS];
    tm_ld(ta + GS * h, A);
    tm_ld(ta + 16 + GS * h, B);
    tm_wait_ld(A, B);
    const uint4 pm = __ldg(pp + h);
    A[0] = add_mod(A[0], sm[pm.x], q);
    A[1] = add_mod(A[1], sm[pm.y], q);
    A[2] = add_mod(A[2], sm[pm.z], q);
    A[3] = add_mod(A[3], sm[pm.w], q);
    if (fold) {
      const uint4 u = *reinterpret_cast<const uint4*>(sm + x0 + 4 * h);
      const uint4 v = *reinterpret_cast<const uint4*>(c1 + x0 + 4 * h);
      A[0] = add_mod(A[0], u.x, q);
      A[1] = add_mod(A[1], u.y, q);
      A[2] = add_mod(A[2], u.z, q);
      A[3] = add_mod(A[3], u.w, q);
      B[0] = add_mod(B[0], v.x, q);
      B[1] = add_mod(B[1], v.y, q);
      B[2] = add_mod(B[2], v.z, q);
      B[3] = add_mod(B[3], v.w, q);
    }
    *reinterpret_cast<uint4*>(o + (uint64_t)pr.poly0 * N + x0 + 4 * h) = make_uint4(A[0], A[1], A[2], A[3]);
    *reinterpret_cast<uint4*>(o + (uint64_t)pr.poly1 * N + x0 + 4 * h) = make_uint4(B[0], B[1], B[2], B[3]);
  }
  tm_fence_before();
  __syncthreads();
  if (warp == 0) {
    tm_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmemCols) : "memory");
  }
  if (gp == 0) count_ops(g, 0, 1, fold ? 1 : 0);  // one rotation (+ the fold add) per pair (backend.cpp:63-73)
  cl.sync();  // the peers have read this CTA's digit
}
