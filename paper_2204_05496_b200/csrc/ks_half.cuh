// N = 16384 key switch as two independent half-ring blocks of 512 threads.
//
// Same arithmetic as k_rot_keyswitch_t (BfvContext::apply_galois,
// proj/src/bfv/context.cpp:428-507; every sum exact mod q_i, so the output is
// bit-identical), but each (pair, prime) runs as two CTAs, one per half of
// the eval slots, so the N = 16384 fold gets the N = 8192 kernel's shape:
// 512 threads, 40 registers, 128 TMEM columns, 3 CTAs per SM (the 1024-thread
// kernel runs 1 CTA per SM).
//
// Why the halves are independent: the forward transform's first stage pairs
// coefficient x with x + N/2 (one twiddle, zetas[1]); after it, half h of the
// array only ever meets itself, and its stages 1..13 are an N/2-point
// transform whose stage-s' block i' uses zetas[2^(s'+1) + h 2^s' + i'] — a
// per-half twiddle table in Ntt<13>'s own layout (built on the host, `twh`).
// Its outputs are eval slots [h N/2, (h+1) N/2): exactly the slots this CTA
// accumulates. So each CTA reads both halves of the digit, does the first
// stage for its half only, and runs Ntt<13> with the half tables. Slot s is
// held by thread s / 16 in both the N = 16384 and the half layout, so the
// Galois keys keep their N = 16384 pass-C layout (stride 1024, offset
// 512 h). The Galois gathers read c1 / c0 through L1/L2 (a 64 KB polynomial
// does not fit next to the exchange buffer at 3 CTAs/SM; staging each
// thread's source group through shared memory as k_rot_digits_h does
// measured 0.8 % slower here).
// Textually included by heinfer_b200.cu after tmem_ks.cuh.
#pragma once

// Galois gather of a thread's 16 slots: their sources form one aligned
// 16-slot group (the automorphism maps groups onto groups), so the group is
// read with 4 x 128-bit loads and permuted through a per-thread column of
// shared memory (word k of thread j at scr[k * T + j]: conflict-free for any
// permutation, and only the writing thread reads it, so no barrier).
template <uint32_t T>
__device__ __forceinline__ void gather_group(const uint32_t* __restrict__ src, const uint32_t (&pm)[16],
                                             uint32_t* scr, uint32_t (&e)[16]) {
  const uint4* gs = reinterpret_cast<const uint4*>(src + (pm[0] & ~15u));
  const uint32_t j = threadIdx.x % T;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 v = __ldg(gs + c);
    scr[(4 * c) * T + j] = v.x;
    scr[(4 * c + 1) * T + j] = v.y;
    scr[(4 * c + 2) * T + j] = v.z;
    scr[(4 * c + 3) * T + j] = v.w;
  }
#pragma unroll
  for (int r = 0; r < 16; ++r) e[r] = scr[(pm[r] & 15u) * T + j];
}

// One launch per branch: both halves of primes [gp0, gp0 + np) with
// blockIdx = (pair * np + prime - gp0) * 2 + h, so the two halves of a
// (pair, prime) run side by side and the second read of each digit hits L2;
// the parameter-space twiddle rows are [prime - gp0][h].
__global__ void __launch_bounds__(512, 3) k_rot_keyswitch_h(Geo g, const uint32_t* __restrict__ dot,
                                                           const uint32_t* __restrict__ digits,
                                                           const uint32_t* __restrict__ perm,
                                                           const uint2* __restrict__ key0,
                                                           const uint2* __restrict__ key1,
                                                           uint32_t* __restrict__ out, int fold, uint32_t gp0,
                                                           uint32_t np, const __grid_constant__ TwAB tab) {
  constexpr int LOGF = 14;
  using NT = Ntt<LOGF - 1>;
  constexpr uint32_t NF = 1u << LOGF, NH = NF / 2, T = NH / 16, TF = NF / 16;
  constexpr uint32_t kTmemCols = T / 4;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  __shared__ uint32_t tbase;
  const uint32_t loc = blockIdx.x >> 1, h = blockIdx.x & 1u;
  const uint32_t pair = loc / np, gp = gp0 + loc % np, row = (loc % np) * 2 + h;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, L = pr.L, i = pr.i;
  const uint32_t j = threadIdx.x, warp = j >> 5;
  const uint32_t x0 = h * NH + NT::posC0(j);  // first of this thread's 16 eval slots
  const uint32_t jf = h * T + j;              // the same slots' thread in the N = 16384 layout
  const uint32_t* dig = digits + ((uint64_t)pair * g.P + pr.first) * NF;
  const uint32_t* ct = dot + (uint64_t)pair * g.ct_words;
  const uint32_t* c0 = ct + (uint64_t)pr.poly0 * NF;
  const uint32_t* c1 = ct + (uint64_t)pr.poly1 * NF;
  const uint2* key = (pr.b ? key1 : key0) + (uint64_t)i * L * 2 * NF;
  const uint2 z1 = __ldg(g.fwd + (size_t)gp * NF + 1);  // first-stage twiddle zetas[1]
  const uint4* twc = g.twch + ((size_t)gp * 2 + h) * g.twch_stride;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tbase)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t ta = tbase + ((32u * (warp & 3u)) << 16) + 32u * (warp >> 2);  // acc0 cols; acc1 at +16
  const uint4* pp = reinterpret_cast<const uint4*>(perm + x0);
  {
    // l == i term: NTT_i(INTT_i(x)) = x, so sigma(c1)_i multiplies the key directly
    const uint4* k0 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * i) * NF) + jf;
    const uint4* k1 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * i + 1) * NF) + jf;
#pragma unroll
    for (int hh = 0; hh < 4; ++hh) {
      uint32_t A[4], B[4];
      const uint4 pm = __ldg(pp + hh);
      const uint32_t d0 = __ldg(c1 + pm.x), d1 = __ldg(c1 + pm.y), d2 = __ldg(c1 + pm.z), d3 = __ldg(c1 + pm.w);
      const uint4 a = __ldg(k0 + (2 * hh) * TF), b = __ldg(k0 + (2 * hh + 1) * TF);
      const uint4 u = __ldg(k1 + (2 * hh) * TF), v = __ldg(k1 + (2 * hh + 1) * TF);
      A[0] = mul_shoup(d0, a.x, a.y, q);
      A[1] = mul_shoup(d1, a.z, a.w, q);
      A[2] = mul_shoup(d2, b.x, b.y, q);
      A[3] = mul_shoup(d3, b.z, b.w, q);
      B[0] = mul_shoup(d0, u.x, u.y, q);
      B[1] = mul_shoup(d1, u.z, u.w, q);
      B[2] = mul_shoup(d2, v.x, v.y, q);
      B[3] = mul_shoup(d3, v.z, v.w, q);
      tm_st(ta + 4 * hh, A);
      tm_st(ta + 16 + 4 * hh, B);
    }
  }
  uint32_t e[16];
  for (uint32_t l = 0; l < L; ++l) {
    if (l == i) continue;
    const uint32_t* src = dig + (uint64_t)l * NF;
    // first stage (t = N/2) for this half: x < N/2 gets u + z v, x + N/2 gets u - z v
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t x = NT::posA(j, r);
      // unreduced digit residues (< q_l < 2^31): v feeds a Shoup product, and
      // u + t, u - t + q stay below q_l + q_i < 2^32 (see k_rot_keyswitch_t)
      const uint32_t u = src[x], v = src[x + NH];
      const uint32_t t = mul_shoup(v, z1.x, z1.y, q);
      e[r] = h ? sub_mod(u, t, q) : add_mod(u, t, q);
    }
    NT::template fwd<true, ParamTw, true, true>(e, sm, ParamTw{tab.w[row]}, twc, q);
    const uint4* k0 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * l) * NF) + jf;
    const uint4* k1 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * l + 1) * NF) + jf;
    tm_wait_st();  // the previous digit's accumulator stores have landed
#pragma unroll
    for (int hh = 0; hh < 4; ++hh) {
      uint32_t A[4], B[4];
      tm_ld(ta + 4 * hh, A);
      tm_ld(ta + 16 + 4 * hh, B);
      tm_wait_ld(A, B);
      const uint4 a = __ldg(k0 + (2 * hh) * TF), b = __ldg(k0 + (2 * hh + 1) * TF);
      A[0] = add_mod(A[0], mul_shoup(e[4 * hh], a.x, a.y, q), q);
      A[1] = add_mod(A[1], mul_shoup(e[4 * hh + 1], a.z, a.w, q), q);
      A[2] = add_mod(A[2], mul_shoup(e[4 * hh + 2], b.x, b.y, q), q);
      A[3] = add_mod(A[3], mul_shoup(e[4 * hh + 3], b.z, b.w, q), q);
      const uint4 u = __ldg(k1 + (2 * hh) * TF), v = __ldg(k1 + (2 * hh + 1) * TF);
      B[0] = add_mod(B[0], mul_shoup(e[4 * hh], u.x, u.y, q), q);
      B[1] = add_mod(B[1], mul_shoup(e[4 * hh + 1], u.z, u.w, q), q);
      B[2] = add_mod(B[2], mul_shoup(e[4 * hh + 2], v.x, v.y, q), q);
      B[3] = add_mod(B[3], mul_shoup(e[4 * hh + 3], v.z, v.w, q), q);
      tm_st(ta + 4 * hh, A);
      tm_st(ta + 16 + 4 * hh, B);
    }
  }
  uint32_t* o = out + (uint64_t)pair * g.ct_words;
  tm_wait_st();
#pragma unroll
  for (int hh = 0; hh < 4; ++hh) {
    uint32_t A[4], B[4];
    tm_ld(ta + 4 * hh, A);
    tm_ld(ta + 16 + 4 * hh, B);
    tm_wait_ld(A, B);
    const uint4 pm = __ldg(pp + hh);
    A[0] = add_mod(A[0], __ldg(c0 + pm.x), q);
    A[1] = add_mod(A[1], __ldg(c0 + pm.y), q);
    A[2] = add_mod(A[2], __ldg(c0 + pm.z), q);
    A[3] = add_mod(A[3], __ldg(c0 + pm.w), q);
    if (fold) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(c0 + x0) + hh);
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(c1 + x0) + hh);
      A[0] = add_mod(A[0], u.x, q);
      A[1] = add_mod(A[1], u.y, q);
      A[2] = add_mod(A[2], u.z, q);
      A[3] = add_mod(A[3], u.w, q);
      B[0] = add_mod(B[0], v.x, q);
      B[1] = add_mod(B[1], v.y, q);
      B[2] = add_mod(B[2], v.z, q);
      B[3] = add_mod(B[3], v.w, q);
    }
    *reinterpret_cast<uint4*>(o + (uint64_t)pr.poly0 * NF + x0 + 4 * hh) = make_uint4(A[0], A[1], A[2], A[3]);
    *reinterpret_cast<uint4*>(o + (uint64_t)pr.poly1 * NF + x0 + 4 * hh) = make_uint4(B[0], B[1], B[2], B[3]);
  }
  tm_fence_before();
  __syncthreads();
  if (warp == 0) {
    tm_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmemCols) : "memory");
  }
  if (gp == 0 && h == 0) count_ops(g, 0, 1, fold ? 1 : 0);  // one rotation (+ the fold add) per pair
}

// N = 16384 digit INTT as a 2-CTA cluster, one CTA per half of the eval
// slots (the counterpart of k_rot_keyswitch_h; same arithmetic as
// k_rot_digits_f, context.cpp:445-470). The inverse transform's stages with
// m >= 2 blocks stay inside a half, with inv_zetas[2^(s'+1) + h 2^s' + i']
// at local index 2^s' + i' (the half tables `itwh`); Ntt<13>::inv runs them
// with its n^-1 fold replaced by 1. The last stage (m = 1) pairs local
// coefficient x of both halves: each CTA publishes its half in shared
// memory, reads its partner's through distributed shared memory, and writes
// its own output half: (U + V) n^-1 for half 0, (U - V) inv_zetas[1] n^-1 for
// half 1 — the digit comes out finished, exactly as k_rot_digits_f<14>'s.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 3)
    k_rot_digits_h(Geo g, const uint32_t* __restrict__ dot, const uint32_t* __restrict__ perm,
                   uint32_t* __restrict__ digits) {
  constexpr int LOGF = 14;
  using NT = Ntt<LOGF - 1>;
  constexpr uint32_t NF = 1u << LOGF, NH = NF / 2;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t h = cl.block_rank();
  const uint32_t blk = blockIdx.x >> 1, pair = blk / g.P, gp = blk % g.P;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, j = threadIdx.x;
  const uint32_t* c1 = dot + (uint64_t)pair * g.ct_words + (uint64_t)pr.poly1 * NF;
  const uint32_t x0 = h * NH + NT::posC0(j);
  uint32_t pm[16], e[16];
  load16_ro(perm + x0, pm);
  gather_group<NT::T>(c1, pm, sm, e);  // sm is free until the transform's first barrier
  const uint2* itn = g.invh + ((size_t)gp * 2 + h) * NH;
  const uint4* itc = g.itwch + ((size_t)gp * 2 + h) * g.twch_stride;
  const uint2 lastH = __ldg(itn + 1);                               // local last stage: inv_zetas[2 + h]
  const uint2 one = make_uint2(1u, (uint32_t)(0x100000000ull / q));  // Shoup constant of 1: a plain reduction
  NT::inv(e, sm, itn, itc, q, lastH, one);
  __syncthreads();  // the transform's last shared reads are done
#pragma unroll
  for (int r = 0; r < 16; ++r) sm[NT::posA(j, r)] = e[r];
  cl.sync();
  const uint32_t* peer = cl.map_shared_rank(sm, h ^ 1u);
  uint32_t* d = digits + ((uint64_t)pair * g.P + gp) * NF + h * NH;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint32_t x = NT::posA(j, r);
    const uint32_t o = peer[x];
    // U = half 0's value, V = half 1's at local coefficient x
    d[x] = h ? mul_shoup(o - e[r] + q, pr.last.x, pr.last.y, q) : mul_shoup(e[r] + o, pr.ninv.x, pr.ninv.y, q);
  }
  cl.sync();  // the partner has finished reading this CTA's shared memory
}
