// Latency path (N = 8192, small batches): the whole rotate-and-sum fold
// (HeBackend::sum_all_slots, backend.cpp:63-73; apply_galois,
// context.cpp:428-507) as ONE persistent dataflow kernel.
//
// With one individual there are only 11 pairs x 10 primes = 110 (pair,
// prime) key switches per rotation, fewer than the 148 SMs, and each runs
// its L - 1 digit transforms back to back; the 13 rotations are a chain.
// Here every transform is its own task, so the per-rotation critical path is
// one NTT (+ key products) and one INTT (+ the element-wise finish):
//
//   D0(p, i)       digit_i = INTT_i(sigma_0(c1)_i) of the input ciphertext
//   K(s, p, i, l)  l != i: part_{i,l} = NTT_i(digit_l mod q_i) (.) K_s[l][i]  (both parts)
//   RD(s, p, i)    prime i after rotation s (fold: c + rot(c)):
//                    c0' = c0 + sigma(c0)_i + sigma(c1)_i K[i][i]_0 + sum_l part_{i,l,0}
//                    c1' = c1 +               sigma(c1)_i K[i][i]_1 + sum_l part_{i,l,1}
//                  then (s + 1 < S) the next rotation's digit_i = INTT_i(sigma_{s+1}(c1')_i)
//                  from c1' already on chip.
//
// Scheduling is a device-side ready queue: a CTA only ever takes a task
// whose inputs are complete. The host seeds D0(., .). A finished digit
// (D0(p, l) or RD(s - 1, p, l)) enqueues the L - 1 tasks K(s, p, i, l) that
// transform it. RD(s, p, i) has L inputs, each bumping the counter of (p, i)
// for the rotation's parity: the L - 1 products K(s, p, i, .) and the
// ciphertext of prime i entering the rotation (RD(s - 1, p, i); D0(p, i) at
// s = 0); the bump completing them enqueues RD(s, p, i) (per-parity counters:
// rotation s + 2's bumps can only start once rotation s's are all in). Each CTA claims its next queue slot while it runs the current task,
// so the claim's L2 round trip is off the critical path; a CTA never waits on
// a claimed slot before finishing its current task, so some CTA always
// progresses.
//
// Digits, key-switch products and the ciphertext are double-buffered by
// rotation parity; every write-after-read is ordered transitively through
// the same dependencies (RD(s + 1, p, l) follows RD(s, p, l) and every
// K(s, p, ., l) through RD(s, p, .) and K(s + 1, p, l, .)). Arithmetic is exactly
// k_rot_keyswitch_s's (every sum exact mod q_i), so the output is
// bit-identical to the reference. Cross-CTA data is read with ld.global.cg
// (L2); producers publish with __syncthreads + a gpu-scope fence before the
// counter update and a release store of the queue entry; consumers poll the
// entry with a gpu-scope acquire.
// Textually included by heinfer_b200.cu after fold_kernels.cuh.
#pragma once

constexpr int kDfLmax = 6;  // primes per branch on this path (the production L = 6 / 4)

struct DfParams {
  uint32_t pairs, S;  // pairs, rotations
  uint32_t KP;        // K tasks per pair and rotation = sum_b L_b (L_b - 1)
  const uint32_t* perm[kMaxElts];     // eval permutation of rotation s
  const uint2* key[2][kMaxElts];      // branch key set of rotation s: [i][l][part][N] (val, shoup), pass-C layout
  uint32_t* ct[2];                    // ciphertexts by parity: [pairs][ct_words]; ct[0] holds the input
  uint32_t* dig[2];                   // digits by parity: [pairs][P][N] (natural coefficient order)
  uint32_t* part[2];                  // key-switch products by parity: [pairs][P][kDfLmax - 1][2][N] (slot order)
  uint32_t* count;                    // [2 (parity)][pairs][P]: K completions (monotonic over the call)
  uint32_t* queue;                    // [tasks] task ids, 0xffffffff = not yet enqueued
  uint32_t* head;                     // next queue slot to claim
  uint32_t* tail;                     // next queue slot to fill
  unsigned long long* trace;          // optional (HEI_DF_TRACE): [slot][4] claim, start, end ns, id << 32 | smid
};

// task id: bits 30..31 type (0 D0, 1 RD, 2 K), 26..29 rotation, 14..25 pair,
// 10..13 prime, 6..9 digit l (K)
constexpr uint32_t kDfD = 0u, kDfR = 1u, kDfK = 2u;
__host__ __device__ __forceinline__ uint32_t df_id(uint32_t type, uint32_t s, uint32_t p, uint32_t gp, uint32_t x = 0) {
  return (type << 30) | (s << 26) | (p << 14) | (gp << 10) | (x << 6);
}
__host__ __device__ __forceinline__ uint64_t df_tasks(uint32_t S, uint32_t pairs, uint32_t P, uint32_t KP) {
  return (uint64_t)pairs * P + (uint64_t)S * pairs * (P + KP);  // D0, then RD per (pair, prime) and K per pair, every rotation
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

// Resets the counters and seeds the queue with D0(p, i) for every (pair, prime).
__global__ void k_df_seed(DfParams d, uint32_t P, uint32_t total) {
  const uint32_t A = d.pairs * P;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
    d.queue[x] = x < A ? df_id(kDfD, 0, x / P, x % P) : 0xffffffffu;
    if (x < 2 * A) d.count[x] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *d.head = 0;
    *d.tail = A;
  }
}

// Thread 0, after the CTA's writes are published: digit l of (p, rotation s)
// is ready, so the L - 1 products that transform it can run.
__device__ __forceinline__ void df_enqueue_K(const DfParams& d, const PrimeInfo& pr, uint32_t s, uint32_t p) {
  const uint32_t k = atomicAdd(d.tail, pr.L - 1);
  for (uint32_t m = 0, o = 0; m < pr.L; ++m)
    if (m != pr.i) st_release(d.queue + k + o++, df_id(kDfK, s, p, pr.first + m, pr.i));
}

// Thread 0: one of the L inputs of RD(s, p, gp) is complete — the L - 1
// products K(s, p, gp, .) and the ciphertext of prime gp entering rotation s
// (written by RD(s - 1, p, gp); D0 stands in at s = 0). The bump completing
// them enqueues RD(s, p, gp).
__device__ __forceinline__ void df_bump(const Geo& g, const DfParams& d, const PrimeInfo& pr, uint32_t s, uint32_t p,
                                        uint32_t gp) {
  uint32_t* cnt = d.count + ((uint64_t)(s & 1u) * d.pairs + p) * g.P + gp;
  if (atomicAdd(cnt, 1u) + 1 == pr.L * (s / 2 + 1)) st_release(d.queue + atomicAdd(d.tail, 1u), df_id(kDfR, s, p, gp));
}

// INTT of e (pass-C order: thread j holds slots 16j..16j+15) into the digit
// buffer in natural coefficient order.
__device__ __forceinline__ void df_digit_out(const Geo& g, uint32_t gp, uint32_t (&e)[16], uint32_t* sm,
                                             uint32_t* dst) {
  using NT = Ntt<13>;
  const PrimeInfo& pr = g.pr[gp];
  NT::inv(e, sm, g.inv + (size_t)gp * NT::N, g.itwc + (size_t)gp * g.twc_stride, pr.q, pr.last, pr.ninv);
#pragma unroll
  for (int r = 0; r < 16; ++r) dst[NT::posA(threadIdx.x, r)] = e[r];
}

// D0(p, gp): digit_i = INTT_i(sigma_0(c1)_i)   (context.cpp:445-459)
__device__ __forceinline__ void df_task_D(const Geo& g, const DfParams& d, uint32_t p, uint32_t gp, uint32_t* sm) {
  using NT = Ntt<13>;
  constexpr uint32_t N = NT::N, T = NT::T;
  const uint32_t j = threadIdx.x;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t x0 = NT::posC0(j);
  const uint32_t* c1 = d.ct[0] + (uint64_t)p * g.ct_words + (uint64_t)pr.poly1 * N;
  uint32_t pm[16], e[16];
  load16_ro(d.perm[0] + x0, pm);
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
  df_digit_out(g, gp, e, sm, d.dig[0] + ((uint64_t)p * g.P + gp) * N);
  __syncthreads();
  if (j == 0) {
    __threadfence();
    df_enqueue_K(d, pr, 0, p);
    df_bump(g, d, pr, 0, p, gp);
  }
}

// K(s, p, gp, l): NTT_i(digit_l mod q_i) (.) K_s[l][i], both parts, to the
// product buffer; the product completing the L - 1 of (s, p, gp) enqueues RD.
__device__ __forceinline__ void df_task_K(const Geo& g, const DfParams& d, uint32_t s, uint32_t p, uint32_t gp,
                                          uint32_t l, uint32_t* sm) {
  using NT = Ntt<13>;
  constexpr uint32_t N = NT::N, T = NT::T;
  const uint32_t j = threadIdx.x;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, L = pr.L, i = pr.i;
  const uint32_t par = s & 1u;
  const uint32_t x0 = NT::posC0(j), sl = l < i ? l : l - 1;
  const uint32_t* src = d.dig[par] + ((uint64_t)p * g.P + pr.first + l) * N;
  uint32_t e[16];
  if (pr.fast_reduce) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t v = __ldcg(src + NT::posA(j, r));
      e[r] = min(v, v - q);
    }
  } else {
#pragma unroll
    for (int r = 0; r < 16; ++r) e[r] = __ldcg(src + NT::posA(j, r)) % q;
  }
  NT::template fwd<true>(e, sm, g.fwd + (size_t)gp * N, g.twc + (size_t)gp * g.twc_stride, q);
  const uint2* key = d.key[pr.b][s] + ((uint64_t)i * L + l) * 2 * N;
  const uint4* k0 = reinterpret_cast<const uint4*>(key) + j;
  const uint4* k1 = reinterpret_cast<const uint4*>(key + N) + j;
  uint32_t* o = d.part[par] + (((uint64_t)p * g.P + gp) * (kDfLmax - 1) + sl) * 2 * N + x0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 a = __ldg(k0 + (2 * c) * T), b = __ldg(k0 + (2 * c + 1) * T);
    *reinterpret_cast<uint4*>(o + 4 * c) =
        make_uint4(mul_shoup(e[4 * c], a.x, a.y, q), mul_shoup(e[4 * c + 1], a.z, a.w, q),
                   mul_shoup(e[4 * c + 2], b.x, b.y, q), mul_shoup(e[4 * c + 3], b.z, b.w, q));
    const uint4 u = __ldg(k1 + (2 * c) * T), v = __ldg(k1 + (2 * c + 1) * T);
    *reinterpret_cast<uint4*>(o + N + 4 * c) =
        make_uint4(mul_shoup(e[4 * c], u.x, u.y, q), mul_shoup(e[4 * c + 1], u.z, u.w, q),
                   mul_shoup(e[4 * c + 2], v.x, v.y, q), mul_shoup(e[4 * c + 3], v.z, v.w, q));
  }
  __syncthreads();
  if (j == 0) {
    __threadfence();
    df_bump(g, d, pr, s, p, gp);
  }
}

// RD(s, p, gp): thread j finishes its 16 slots 16j..16j+15 of prime i, then
// (s + 1 < S) the next rotation's digit from c1' through shared memory.
__device__ __forceinline__ void df_task_RD(const Geo& g, const DfParams& d, uint32_t s, uint32_t p, uint32_t gp,
                                           uint32_t* sm) {
  using NT = Ntt<13>;
  constexpr uint32_t N = NT::N, T = NT::T;
  const uint32_t j = threadIdx.x;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, L = pr.L, i = pr.i;
  const uint32_t par = s & 1u;
  const uint32_t x0 = NT::posC0(j);
  const uint32_t* cin = d.ct[par] + (uint64_t)p * g.ct_words;
  const uint32_t* c0 = cin + (uint64_t)pr.poly0 * N;
  const uint32_t* c1 = cin + (uint64_t)pr.poly1 * N;
  uint32_t* out = d.ct[par ^ 1u] + (uint64_t)p * g.ct_words;
  // sigma(c1)_i and sigma(c0)_i of this thread's slots: one aligned 16-slot
  // source group each, 4 x 128-bit loads permuted through this thread's
  // shared-memory columns (thread-private, no barrier; sm holds 3 N words:
  // columns 0..15 for c1, 16..31 for c0, then c1' for the next digit)
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
  const uint4* k0 = reinterpret_cast<const uint4*>(key) + j;
  const uint4* k1 = reinterpret_cast<const uint4*>(key + N) + j;
  const uint4* pp = reinterpret_cast<const uint4*>(d.perm[s] + x0);
  const uint32_t* pb = d.part[par] + ((uint64_t)p * g.P + gp) * (kDfLmax - 1) * 2 * N + x0;
  uint32_t* nx = sm + 2 * N;  // c1' (slot order), for the next digit
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
        if ((uint32_t)sl + 1 < L) U[sl] = ldcg4(pb + (uint64_t)(2 * sl + part) * N + 4 * c);
      const uint4* kp = part ? k1 : k0;
      const uint4 ka = __ldg(kp + (2 * c) * T), kb = __ldg(kp + (2 * c + 1) * T);
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
      if (part == 1) *reinterpret_cast<uint4*>(nx + x0 + 4 * c) = A;
    }
  }
  if (s + 1 < d.S) {
    // next rotation's digit: INTT_i(sigma_{s+1}(c1')_i) from the c1' just written
    __syncthreads();
    uint32_t pm[16], e[16];
    load16_ro(d.perm[s + 1] + x0, pm);
#pragma unroll
    for (int r = 0; r < 16; ++r) e[r] = nx[pm[r]];
    df_digit_out(g, gp, e, sm, d.dig[par ^ 1u] + ((uint64_t)p * g.P + gp) * N);
  }
  __syncthreads();
  if (j == 0 && s + 1 < d.S) {
    __threadfence();
    df_enqueue_K(d, pr, s + 1, p);
    df_bump(g, d, pr, s + 1, p, gp);  // RD(s + 1, p, i) reads what this task wrote
  }
}

template <int MINB>
__global__ void __launch_bounds__(512, MINB) k_fold_dataflow(const __grid_constant__ Geo g,
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
                   xarg = (t >> 6) & 15u;
    if (type == kDfK)
      df_task_K(g, d, s, p, gp, xarg, sm);
    else if (type == kDfR)
      df_task_RD(g, d, s, p, gp, sm);
    else
      df_task_D(g, d, p, gp, sm);
    if (j == 0 && d.trace) d.trace[4 * slot + 2] = gtimer();
  }
}
