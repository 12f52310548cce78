// Latency path (N = 8192, small batches): the whole rotate-and-sum fold
// (HeBackend::sum_all_slots, backend.cpp:63-73; apply_galois,
// context.cpp:428-507) as ONE persistent dataflow kernel of half-ring tasks.
//
// With one individual there are only 11 pairs x 10 primes = 110 (pair,
// prime) key switches per rotation, fewer than the 148 SMs, and each runs its
// L - 1 digit transforms back to back; the 13 rotations are a chain. The
// chain's length is set by how long one transform takes, so here every
// transform is split in two half-ring transforms (the ks_half.cuh
// decomposition at N = 8192): the forward transform's first stage pairs x
// with x + N/2, after which eval half h only meets itself (an N/2-point
// transform with the per-half tables fwdh/twch); the inverse's stages stay
// inside a half until its last one, which pairs local coefficient x of both
// halves. Each task is a 256-thread CTA doing one half:
//
//   D0(p, i, h)      half-digit a_h = INTT-half_h(sigma_0(c1)_i) of the input
//   K(s, p, i, l, h) l != i: the digit d_l = last stage(a_0, a_1) of (s, p, l)
//                    (mod q_l), reduced mod q_i, first forward stage for half h,
//                    NTT-half_h, times K_s[l][i] (both parts) -> product part_{i,l,h}
//   RI(s, p, i, h)   eval half h of prime i after rotation s (fold: c + rot(c)):
//                      c0' = c0 + sigma(c0)_i + sigma(c1)_i K[i][i]_0 + sum_l part_{i,l,0}
//                      c1' = c1 +               sigma(c1)_i K[i][i]_1 + sum_l part_{i,l,1}
//                    then (s + 1 < S) the next rotation's half-digit of the
//                    half that sigma_{s+1} fills from half h (the Galois
//                    automorphism maps each eval half onto one half: onto
//                    itself for g = 1 mod 4, onto the other for g = 3 mod 4),
//                    from c1' already on chip.
//
// So the per-rotation critical path is one half NTT and one half INTT, and
// the ~600 transforms of a C3 rotation spread over 4 CTAs per SM.
//
// Scheduling is a device-side ready queue: a CTA only ever takes a task whose
// inputs are complete. The host seeds D0(., ., .). Dependencies (per-parity
// counters, monotonic over the call: rotation s + 2's bumps can only start
// once rotation s's are all in):
//   dg(s, p, l)     2 half-digits; the second enqueues the 2 (L - 1) tasks K(s, p, ., l, .)
//   cr(s, p, i, h)  L + 1 inputs of RI(s, p, i, h): the L - 1 products
//                   K(s, p, i, ., h) and both halves of prime i entering the
//                   rotation (RI(s - 1, p, i, 0/1); D0(p, i, 0/1) at s = 0)
// Every write-after-read on the parity buffers is ordered transitively
// through the same dependencies. Each CTA claims its next queue slot while it
// runs the current task (the claim's L2 round trip is off the critical path);
// a CTA never waits on a claimed slot before finishing its current task, so
// some CTA always progresses. Arithmetic is exactly k_rot_keyswitch_s's and
// k_rot_digits_h's (every sum exact mod q_i, the split transforms equal to
// the whole ones), so the output is bit-identical to the reference.
// Cross-CTA data is read with ld.global.cg (L2); producers publish with
// __syncthreads + a gpu-scope fence before the counter update and a release
// store of the queue entry; consumers poll the entry with a gpu-scope acquire.
// Textually included by heinfer_b200.cu after fold_kernels.cuh.
#pragma once

constexpr int kDfLmax = 6;  // primes per branch on this path (the production L = 6 / 4)

struct DfParams {
  uint32_t pairs, S;  // pairs, rotations
  uint32_t KP;        // K tasks per pair, rotation and half = sum_b L_b (L_b - 1)
  uint32_t swapmask;  // bit s: sigma_s maps each eval half onto the other (g_s = 3 mod 4)
  const uint32_t* perm[kMaxElts];     // eval permutation of rotation s
  const uint2* key[2][kMaxElts];      // branch key set of rotation s: [i][l][part][N] (val, shoup), pass-C layout
  uint32_t* ct[2];                    // ciphertexts by parity: [pairs][ct_words]; ct[0] holds the input
  uint32_t* hd[2];                    // half-digits by parity: [pairs][P][2][N/2] (local coefficient order)
  uint32_t* part[2];                  // products by parity: [pairs][P][kDfLmax - 1][2][N] (per half: [c][j] uint4)
  uint32_t* count;                    // dg [2][pairs][P], then cr [2][pairs][P][2]
  uint32_t* queue;                    // [tasks] task ids, 0xffffffff = not yet enqueued
  uint32_t* head;                     // next queue slot to claim
  uint32_t* tail;                     // next queue slot to fill
  unsigned long long* trace;          // optional (HEI_DF_TRACE): [slot][4] claim, start, end ns, id << 32 | smid
};

// task id: bits 30..31 type (0 D0, 1 RI, 2 K), 26..29 rotation, 14..25 pair,
// 10..13 prime, 6..9 digit l (K), 5 half
constexpr uint32_t kDfD = 0u, kDfR = 1u, kDfK = 2u;
__host__ __device__ __forceinline__ uint32_t df_id(uint32_t type, uint32_t s, uint32_t p, uint32_t gp, uint32_t l,
                                                   uint32_t h) {
  return (type << 30) | (s << 26) | (p << 14) | (gp << 10) | (l << 6) | (h << 5);
}
__host__ __device__ __forceinline__ uint64_t df_tasks(uint32_t S, uint32_t pairs, uint32_t P, uint32_t KP) {
  return 2ull * ((uint64_t)pairs * P + (uint64_t)S * pairs * (P + KP));  // D0, then RI and K every rotation, per half
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint4 ldcg4(const uint32_t* p) { return __ldcg(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Resets the counters and seeds the queue with D0(p, i, h) for every (pair, prime, half).
__global__ void k_df_seed(DfParams d, uint32_t P, uint32_t total) {
  const uint32_t A = d.pairs * P;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
    d.queue[x] = x < 2 * A ? df_id(kDfD, 0, x / (2 * P), (x / 2) % P, 0, x & 1u) : 0xffffffffu;
    if (x < 6 * A) d.count[x] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *d.head = 0;
    *d.tail = 2 * A;
  }
}

// ---- thread-0 dependency updates (after the CTA's writes are published)
__device__ __forceinline__ void df_cr_bump(const Geo& g, const DfParams& d, const PrimeInfo& pr, uint32_t s,
                                           uint32_t p, uint32_t gp, uint32_t h) {
  uint32_t* c = d.count + 2 * d.pairs * g.P + (((uint64_t)(s & 1u) * d.pairs + p) * g.P + gp) * 2 + h;
  if (atomicAdd(c, 1u) + 1 == (pr.L + 1) * (s / 2 + 1))
    st_release(d.queue + atomicAdd(d.tail, 1u), df_id(kDfR, s, p, gp, 0, h));
}
// half-digit of (s, p, prime gp) done; the second enqueues the products that transform the digit
__device__ __forceinline__ void df_dg_bump(const Geo& g, const DfParams& d, const PrimeInfo& pr, uint32_t s,
                                           uint32_t p, uint32_t gp) {
  uint32_t* c = d.count + ((uint64_t)(s & 1u) * d.pairs + p) * g.P + gp;
  if (atomicAdd(c, 1u) + 1 == 2 * (s / 2 + 1)) {
    const uint32_t k = atomicAdd(d.tail, 2 * (pr.L - 1));
    for (uint32_t m = 0, o = 0; m < pr.L; ++m)
      if (m != pr.i)
        for (uint32_t h = 0; h < 2; ++h) st_release(d.queue + k + o++, df_id(kDfK, s, p, pr.first + m, pr.i, h));
  }
}

// Half-INTT of e (pass-C order of eval half h: thread j holds the half's
// local slots 16j..16j+15) into the half-digit buffer, local coefficient
// order; the last stage (pairing the halves) runs in the consumer.
__device__ __forceinline__ void df_half_inv(const Geo& g, uint32_t gp, uint32_t h, uint32_t (&e)[16], uint32_t* sm,
                                            uint32_t* dst) {
  using NT = Ntt<12>;
  const PrimeInfo& pr = g.pr[gp];
  const uint2* itn = g.invh + ((size_t)gp * 2 + h) * NT::N;
  const uint4* itc = g.itwch + ((size_t)gp * 2 + h) * g.twch_stride;
  const uint2 lastH = __ldg(itn + 1);                                  // local last stage: inv_zetas[2 + h]
  const uint2 one = make_uint2(1u, (uint32_t)(0x100000000ull / pr.q));  // Shoup constant of 1: a plain reduction
  NT::inv(e, sm, itn, itc, pr.q, lastH, one);
#pragma unroll
  for (int r = 0; r < 16; ++r) dst[NT::posA(threadIdx.x, r)] = e[r];
}

// D0(p, gp, h): half-digit of sigma_0(c1)_i on eval half h  (context.cpp:445-459)
__device__ __forceinline__ void df_task_D(const Geo& g, const DfParams& d, uint32_t p, uint32_t gp, uint32_t h,
                                          uint32_t* sm) {
  using NT = Ntt<12>;
  constexpr uint32_t NH = NT::N, T = NT::T;
  const uint32_t j = threadIdx.x;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t* c1 = d.ct[0] + (uint64_t)p * g.ct_words + (uint64_t)pr.poly1 * 2 * NH;
  uint32_t pm[16], e[16];
  load16_ro(d.perm[0] + h * NH + NT::posC0(j), pm);
  {
    // the 16 sources form one aligned group: 4 x 128-bit L2 loads, permuted
    // through this thread's shared-memory column (no barrier)
    const uint32_t* gs = c1 + (pm[0] & ~15u);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 v = ldcg4(gs + 4 * c);
      sm[(4 * c) * T + j] = v.x;
      sm[(4 * c + 1) * T + j] = v.y;
      sm[(4 * c + 2) * T + j] = v.z;
      sm[(4 * c + 3) * T + j] = v.w;
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) e[r] = sm[(pm[r] & 15u) * T + j];
  }
  df_half_inv(g, gp, h, e, sm, d.hd[0] + (((uint64_t)p * g.P + gp) * 2 + h) * NH);
  __syncthreads();
  if (j == 0) {
    __threadfence();
    df_dg_bump(g, d, pr, 0, p, gp);
    df_cr_bump(g, d, pr, 0, p, gp, 0);  // RI(0, p, gp, .) reads the input: ready; one bump per D0 half
    df_cr_bump(g, d, pr, 0, p, gp, 1);
  }
}

// K(s, p, gp, l, h): the digit of prime l from its two half-digits, mod q_i,
// first forward stage for half h, NTT-half, times K_s[l][i] (both parts).
__device__ __forceinline__ void df_task_K(const Geo& g, const DfParams& d, uint32_t s, uint32_t p, uint32_t gp,
                                          uint32_t l, uint32_t h, uint32_t* sm) {
  using NT = Ntt<12>;
  constexpr uint32_t NH = NT::N, T = NT::T, N = 2 * NH, TF = N / 16;
  const uint32_t j = threadIdx.x;
  const PrimeInfo& pr = g.pr[gp];
  const PrimeInfo& pl = g.pr[pr.first + l];
  const uint32_t q = pr.q, L = pr.L, i = pr.i, ql = pl.q;
  const uint32_t par = s & 1u;
  const uint32_t* a0 = d.hd[par] + (((uint64_t)p * g.P + pr.first + l) * 2) * NH;
  const uint32_t* a1 = a0 + NH;
  const uint2 z1 = __ldg(g.fwd + (size_t)gp * N + 1);  // first-stage twiddle zetas[1]
  uint32_t e[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint32_t x = NT::posA(j, r);
    const uint32_t U = __ldcg(a0 + x), V = __ldcg(a1 + x);
    // the digit's last inverse stage (k_rot_digits_h): d[x] = (U + V) n^-1, d[x + N/2] = (U - V) inv_zetas[1] n^-1
    uint32_t u = mul_shoup(U + V, pl.ninv.x, pl.ninv.y, ql), v = mul_shoup(U - V + ql, pl.last.x, pl.last.y, ql);
    if (pr.fast_reduce) {
      u = min(u, u - q);
      v = min(v, v - q);
    } else {
      u %= q;
      v %= q;
    }
    // first forward stage (t = N/2) for this half: x gets u + z v, x + N/2 gets u - z v
    const uint32_t t = mul_shoup(v, z1.x, z1.y, q);
    e[r] = h ? sub_mod(u, t, q) : add_mod(u, t, q);
  }
  NT::template fwd<true>(e, sm, g.fwdh + ((size_t)gp * 2 + h) * NH, g.twch + ((size_t)gp * 2 + h) * g.twch_stride, q);
  const uint2* key = d.key[pr.b][s] + ((uint64_t)i * L + l) * 2 * N;
  const uint4* k0 = reinterpret_cast<const uint4*>(key) + h * T + j;  // slot 16 (hT + j) + ... in the N layout
  const uint4* k1 = reinterpret_cast<const uint4*>(key + N) + h * T + j;
  const uint32_t sl = l < i ? l : l - 1;
  uint4* o = reinterpret_cast<uint4*>(d.part[par] + (((uint64_t)p * g.P + gp) * (kDfLmax - 1) + sl) * 2 * N + h * NH) + j;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 a = __ldg(k0 + (2 * c) * TF), b = __ldg(k0 + (2 * c + 1) * TF);
    o[c * T] = make_uint4(mul_shoup(e[4 * c], a.x, a.y, q), mul_shoup(e[4 * c + 1], a.z, a.w, q),
                          mul_shoup(e[4 * c + 2], b.x, b.y, q), mul_shoup(e[4 * c + 3], b.z, b.w, q));
    const uint4 u = __ldg(k1 + (2 * c) * TF), v = __ldg(k1 + (2 * c + 1) * TF);
    o[N / 4 + c * T] = make_uint4(mul_shoup(e[4 * c], u.x, u.y, q), mul_shoup(e[4 * c + 1], u.z, u.w, q),
                                  mul_shoup(e[4 * c + 2], v.x, v.y, q), mul_shoup(e[4 * c + 3], v.z, v.w, q));
  }
  __syncthreads();
  if (j == 0) {
    __threadfence();
    df_cr_bump(g, d, pr, s, p, gp, h);
  }
}

// RI(s, p, gp, h): thread j finishes the slots hN/2 + 16j .. +15 of prime i,
// then (s + 1 < S) the next rotation's half-digit of the half sigma_{s+1}
// fills from this one.
__device__ __forceinline__ void df_task_RI(const Geo& g, const DfParams& d, uint32_t s, uint32_t p, uint32_t gp,
                                           uint32_t h, uint32_t* sm) {
  using NT = Ntt<12>;
  constexpr uint32_t NH = NT::N, T = NT::T, N = 2 * NH, TF = N / 16;
  const uint32_t j = threadIdx.x;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, L = pr.L, i = pr.i;
  const uint32_t par = s & 1u;
  const uint32_t x0 = h * NH + NT::posC0(j);  // this thread's first slot
  const uint32_t* cin = d.ct[par] + (uint64_t)p * g.ct_words;
  const uint32_t* c0 = cin + (uint64_t)pr.poly0 * N;
  const uint32_t* c1 = cin + (uint64_t)pr.poly1 * N;
  uint32_t* out = d.ct[par ^ 1u] + (uint64_t)p * g.ct_words;
  // sigma(c1)_i and sigma(c0)_i of this thread's slots: one aligned 16-slot
  // source group each, 4 x 128-bit loads permuted through this thread's
  // shared-memory columns (thread-private, no barrier; sm holds 3 N/2 words:
  // columns 0..15 for c1, 16..31 for c0, then c1' of this half)
  {
    const uint32_t gsrc = __ldg(d.perm[s] + x0) & ~15u;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 v = ldcg4(c1 + gsrc + 4 * c), w = ldcg4(c0 + gsrc + 4 * c);
      sm[(4 * c) * T + j] = v.x;
      sm[(4 * c + 1) * T + j] = v.y;
      sm[(4 * c + 2) * T + j] = v.z;
      sm[(4 * c + 3) * T + j] = v.w;
      sm[(16 + 4 * c) * T + j] = w.x;
      sm[(16 + 4 * c + 1) * T + j] = w.y;
      sm[(16 + 4 * c + 2) * T + j] = w.z;
      sm[(16 + 4 * c + 3) * T + j] = w.w;
    }
  }
  const uint2* key = d.key[pr.b][s] + ((uint64_t)i * L + i) * 2 * N;
  const uint4* k0 = reinterpret_cast<const uint4*>(key) + h * T + j;
  const uint4* k1 = reinterpret_cast<const uint4*>(key + N) + h * T + j;
  const uint4* pp = reinterpret_cast<const uint4*>(d.perm[s] + x0);
  const uint4* pb =
      reinterpret_cast<const uint4*>(d.part[par] + ((uint64_t)p * g.P + gp) * (kDfLmax - 1) * 2 * N + h * NH) + j;
  uint32_t* nx = sm + 2 * NH;  // c1' of this half (local slot order), for the next half-digit
  // four slots at a time, part 0 then part 1 (each with all of its L - 1
  // product loads in flight at once)
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {
    const uint4 pm = __ldg(pp + c);
    const uint32_t r0 = (pm.x & 15u) * T + j, r1 = (pm.y & 15u) * T + j, r2 = (pm.z & 15u) * T + j,
                   r3 = (pm.w & 15u) * T + j;
    const uint32_t s0 = sm[r0], s1 = sm[r1], s2 = sm[r2], s3 = sm[r3];
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      uint4 U[kDfLmax - 1];
#pragma unroll
      for (int sl = 0; sl < kDfLmax - 1; ++sl)
        if ((uint32_t)sl + 1 < L) U[sl] = __ldcg(pb + (uint64_t)(2 * sl + part) * (N / 4) + c * T);
      const uint4* kp = part ? k1 : k0;
      const uint4 ka = __ldg(kp + (2 * c) * TF), kb = __ldg(kp + (2 * c + 1) * TF);
      const uint32_t* cp = part ? c1 : c0;
      const uint4 f = ldcg4(cp + x0 + 4 * c);
      // l == i term: NTT_i(INTT_i(x)) = x, so sigma(c1)_i multiplies K[i][i] directly
      uint4 A = make_uint4(mul_shoup(s0, ka.x, ka.y, q), mul_shoup(s1, ka.z, ka.w, q), mul_shoup(s2, kb.x, kb.y, q),
                           mul_shoup(s3, kb.z, kb.w, q));
      if (part == 0)  // + sigma(c0)_i
        A = make_uint4(add_mod(A.x, sm[16 * T + r0], q), add_mod(A.y, sm[16 * T + r1], q),
                       add_mod(A.z, sm[16 * T + r2], q), add_mod(A.w, sm[16 * T + r3], q));
#pragma unroll
      for (int sl = 0; sl < kDfLmax - 1; ++sl)
        if ((uint32_t)sl + 1 < L) {
          const uint4 u = U[sl];
          A = make_uint4(add_mod(A.x, u.x, q), add_mod(A.y, u.y, q), add_mod(A.z, u.z, q), add_mod(A.w, u.w, q));
        }
      // fold: c' = c + rot(c)   (sum_all_slots, backend.cpp:67-68)
      A = make_uint4(add_mod(A.x, f.x, q), add_mod(A.y, f.y, q), add_mod(A.z, f.z, q), add_mod(A.w, f.w, q));
      *reinterpret_cast<uint4*>(out + (uint64_t)(part ? pr.poly1 : pr.poly0) * N + x0 + 4 * c) = A;
      if (part == 1) *reinterpret_cast<uint4*>(nx + NT::posC0(j) + 4 * c) = A;
    }
  }
  const bool next = s + 1 < d.S;
  if (next) {
    // next rotation's half-digit: sigma_{s+1} fills half ht entirely from this half
    const uint32_t ht = h ^ ((d.swapmask >> (s + 1)) & 1u);
    __syncthreads();
    uint32_t pm[16], e[16];
    load16_ro(d.perm[s + 1] + ht * NH + NT::posC0(j), pm);
#pragma unroll
    for (int r = 0; r < 16; ++r) e[r] = nx[pm[r] - h * NH];
    df_half_inv(g, gp, ht, e, sm, d.hd[par ^ 1u] + (((uint64_t)p * g.P + gp) * 2 + ht) * NH);
  }
  __syncthreads();
  if (j == 0 && next) {
    __threadfence();
    df_dg_bump(g, d, pr, s + 1, p, gp);
    df_cr_bump(g, d, pr, s + 1, p, gp, 0);  // RI(s + 1, p, gp, .) reads this half
    df_cr_bump(g, d, pr, s + 1, p, gp, 1);
  }
}

__global__ void __launch_bounds__(256, 4) k_fold_dataflow(const __grid_constant__ Geo g,
                                                          const __grid_constant__ DfParams d) {
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  __shared__ uint32_t task_s;
  const uint32_t j = threadIdx.x;
  const uint32_t total = (uint32_t)df_tasks(d.S, d.pairs, g.P, d.KP);
  uint32_t claim = 0, slot = 0;  // thread 0: the queue slot claimed ahead
  if (j == 0) claim = atomicAdd(d.head, 1u);
  for (;;) {
    __syncthreads();  // the previous task's shared-memory reads are done
    if (j == 0) {
      uint32_t t = 0xffffffffu;
      slot = claim;
      const unsigned long long t0 = d.trace ? gtimer() : 0;
      if (slot < total) {
        uint32_t ns = 32;
        while ((t = ld_acquire(d.queue + slot)) == 0xffffffffu) {
          __nanosleep(ns);
          ns = min(ns * 2, 128u);
        }
        claim = atomicAdd(d.head, 1u);  // the next slot, resolved while this task runs
        if (d.trace) {
          uint32_t smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          d.trace[4 * slot] = t0;
          d.trace[4 * slot + 1] = gtimer();
          d.trace[4 * slot + 3] = ((unsigned long long)t << 32) | smid;
        }
      }
      task_s = t;
    }
    __syncthreads();
    const uint32_t t = task_s;
    if (t == 0xffffffffu) return;
    const uint32_t type = t >> 30, s = (t >> 26) & 15u, p = (t >> 14) & 0xfffu, gp = (t >> 10) & 15u,
                   l = (t >> 6) & 15u, h = (t >> 5) & 1u;
    if (type == kDfK)
      df_task_K(g, d, s, p, gp, l, h, sm);
    else if (type == kDfR)
      df_task_RI(g, d, s, p, gp, h, sm);
    else
      df_task_D(g, d, p, gp, h, sm);
    if (j == 0 && d.trace) d.trace[4 * slot + 2] = gtimer();
  }
}
