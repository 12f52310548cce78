// Latency path (N = 8192, small batches): the whole rotate-and-sum fold
// (HeBackend::sum_all_slots, backend.cpp:63-73; apply_galois,
// context.cpp:428-507) as ONE persistent dataflow kernel.
//
// With one individual there are only 11 pairs x 10 primes = 110 (pair,
// prime) key switches per rotation, fewer than the 148 SMs, and each runs
// its L - 1 digit transforms back to back; the 13 rotations are a chain.
// Here every transform is its own task, and the element-wise finish of a
// rotation is split four ways, so the per-rotation critical path is one
// INTT, one NTT and a quarter of the finish:
//
//   D(s, p, i)        digit_i = INTT_i(sigma_s(c1)_i) of the ciphertext entering rotation s
//   K(s, p, i, l)     l != i: part_{i,l} = NTT_i(digit_l mod q_i) (.) K_s[l][i]  (both parts)
//   R(s, p, i, h)     slots [h N/4, (h+1) N/4) of prime i after rotation s (fold: c + rot(c)):
//                       c0' = c0 + sigma(c0)_i + sigma(c1)_i K[i][i]_0 + sum_l part_{i,l,0}
//                       c1' = c1 +               sigma(c1)_i K[i][i]_1 + sum_l part_{i,l,1}
//
// Scheduling is a device-side ready queue: a CTA only ever takes a task
// whose inputs are complete. The host seeds D(0, ., .). A finished D(s, p, l)
// enqueues the L - 1 tasks K(s, p, i, l) that transform its digit. The L - 1
// K(s, p, i, .) and D(s, p, i) each bump counter A of (p, i) for the
// rotation's parity; the task completing the rotation's L bumps enqueues the
// four R(s, p, i, .). Those bump counter B; the last enqueues D(s+1, p, i).
// (Per-parity counters: rotation s+2's bumps can only start once rotation
// s's are all in.) A CTA whose claimed queue slot is still empty waits for
// it, which happens only when no task is ready.
//
// Digits, partials and the ciphertext are double-buffered by rotation
// parity; every write-after-read is ordered transitively through the same
// dependencies. Arithmetic is exactly k_rot_keyswitch_s's
// (every sum exact mod q_i), so the output is bit-identical to the
// reference. Cross-CTA data is read with ld.global.cg (L2); producers publish
// with __syncthreads + a gpu-scope fence before the counter update and a
// release store of the queue entry; consumers poll the entry with a
// gpu-scope acquire.
// Textually included by heinfer_b200.cu after fold_kernels.cuh.
#pragma once

constexpr int kDfLmax = 6;  // primes per branch on this path (the production L = 6 / 4)
constexpr uint32_t kDfRParts = 4;  // R tasks per (pair, prime, rotation): slot ranges of N / kDfRParts

struct DfParams {
  uint32_t pairs, S;  // pairs, rotations
  uint32_t KP;        // K tasks per pair and rotation = sum_b L_b (L_b - 1)
  const uint32_t* perm[kMaxElts];     // eval permutation of rotation s
  const uint2* key[2][kMaxElts];      // branch key set of rotation s: [i][l][part][N] (val, shoup), pass-C layout
  uint32_t* ct[2];                    // ciphertexts by parity: [pairs][ct_words]; ct[0] holds the input
  uint32_t* dig[2];                   // digits by parity: [pairs][P][N] (natural coefficient order)
  uint32_t* part[2];                  // key-switch products by parity: [pairs][P][kDfLmax - 1][2][N] (slot order)
  uint32_t* count;                    // [2 (A, B)][2 (parity)][pairs][P]: completions (monotonic over the call)
  uint32_t* queue;                    // [tasks] task ids, 0xffffffff = not yet enqueued
  uint32_t* head;                     // next queue slot to claim
  uint32_t* tail;                     // next queue slot to fill
  unsigned long long* trace;          // optional (HEI_DF_TRACE): [slot][4] claim, start, end ns, id << 32 | smid
};

// task id: bits 30..31 type (0 D, 1 R, 2 K), 26..29 rotation, 14..25 pair,
// 10..13 prime, 6..9 digit l (K) or slot range (R)
constexpr uint32_t kDfD = 0u, kDfR = 1u, kDfK = 2u;
__host__ __device__ __forceinline__ uint32_t df_id(uint32_t type, uint32_t s, uint32_t p, uint32_t gp, uint32_t x = 0) {
  return (type << 30) | (s << 26) | (p << 14) | (gp << 10) | (x << 6);
}
__host__ __device__ __forceinline__ uint64_t df_tasks(uint32_t S, uint32_t pairs, uint32_t P, uint32_t KP) {
  return (uint64_t)S * pairs * ((1 + kDfRParts) * P + KP);  // D + R parts per (pair, prime), K per pair, every rotation
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

// Resets the counters and seeds the queue with D(0, p, i) for every (pair, prime).
__global__ void k_df_seed(DfParams d, uint32_t P, uint32_t total) {
  const uint32_t A = d.pairs * P;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
    d.queue[x] = x < A ? df_id(kDfD, 0, x / P, x % P) : 0xffffffffu;
    if (x < 4 * A) d.count[x] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *d.head = 0;
    *d.tail = A;
  }
}

__device__ __forceinline__ uint32_t df_task_D(const Geo& g, const DfParams& d, uint32_t s, uint32_t p, uint32_t gp,
                                           uint32_t xarg) {
  using NT = Ntt<13>;
  constexpr uint32_t N = NT::N, T = NT::T, QP = N / kDfRParts, SPT = QP / 512;  // slots per thread in R
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  const uint32_t j = threadIdx.x, P = g.P;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, L = pr.L, i = pr.i;
  const uint32_t par = s & 1u;
  uint32_t* cntA = d.count + ((uint64_t)(0 * 2 + par) * d.pairs + p) * P + gp;
  uint32_t* cntB = d.count + ((uint64_t)(1 * 2 + par) * d.pairs + p) * P + gp;
  uint32_t enq_r = 0;
    // ---------------- D(s, p, gp): digit_i = INTT_i(sigma_s(c1)_i)   (context.cpp:445-459)
    const uint32_t x0 = NT::posC0(j);
    const uint32_t* c1 = d.ct[par] + (uint64_t)p * g.ct_words + (uint64_t)pr.poly1 * N;
    uint32_t pm[16], e[16];
    load16_ro(d.perm[s] + x0, pm);
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
    NT::inv(e, sm, g.inv + (size_t)gp * N, g.itwc + (size_t)gp * g.twc_stride, q, pr.last, pr.ninv);
    uint32_t* dd = d.dig[par] + ((uint64_t)p * P + gp) * N;
#pragma unroll
    for (int r = 0; r < 16; ++r) dd[NT::posA(j, r)] = e[r];
    __syncthreads();
    if (j == 0) {
      __threadfence();
      // the digit is ready: enqueue its L - 1 key-switch products
      const uint32_t k = atomicAdd(d.tail, L - 1);
      for (uint32_t m = 0, o = 0; m < L; ++m)
        if (m != i) st_release(d.queue + k + o++, df_id(kDfK, s, p, pr.first + m, i));
      enq_r = atomicAdd(cntA, 1u) + 1 == L * (s / 2 + 1);
    }
  return enq_r;
}

__device__ __forceinline__ uint32_t df_task_K(const Geo& g, const DfParams& d, uint32_t s, uint32_t p, uint32_t gp,
                                           uint32_t xarg) {
  using NT = Ntt<13>;
  constexpr uint32_t N = NT::N, T = NT::T, QP = N / kDfRParts, SPT = QP / 512;  // slots per thread in R
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  const uint32_t j = threadIdx.x, P = g.P;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, L = pr.L, i = pr.i;
  const uint32_t par = s & 1u;
  uint32_t* cntA = d.count + ((uint64_t)(0 * 2 + par) * d.pairs + p) * P + gp;
  uint32_t* cntB = d.count + ((uint64_t)(1 * 2 + par) * d.pairs + p) * P + gp;
  uint32_t enq_r = 0;
    // ---------------- K(s, p, gp, l)
    const uint32_t x0 = NT::posC0(j), l = xarg, sl = l < i ? l : l - 1;
    const uint32_t* src = d.dig[par] + ((uint64_t)p * P + pr.first + l) * N;
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
    uint32_t* o = d.part[par] + (((uint64_t)p * P + gp) * (kDfLmax - 1) + sl) * 2 * N + x0;
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
      enq_r = atomicAdd(cntA, 1u) + 1 == L * (s / 2 + 1);
    }
  return enq_r;
}

__device__ __forceinline__ uint32_t df_task_R(const Geo& g, const DfParams& d, uint32_t s, uint32_t p, uint32_t gp,
                                           uint32_t xarg) {
  using NT = Ntt<13>;
  constexpr uint32_t N = NT::N, T = NT::T, QP = N / kDfRParts, SPT = QP / 512;  // slots per thread in R
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  const uint32_t j = threadIdx.x, P = g.P;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, L = pr.L, i = pr.i;
  const uint32_t par = s & 1u;
  uint32_t* cntA = d.count + ((uint64_t)(0 * 2 + par) * d.pairs + p) * P + gp;
  uint32_t* cntB = d.count + ((uint64_t)(1 * 2 + par) * d.pairs + p) * P + gp;
  uint32_t enq_r = 0;
    // ---------------- R(s, p, gp, part): thread j owns slots x .. x + SPT - 1, 4 at a time
    const uint32_t* cin = d.ct[par] + (uint64_t)p * g.ct_words;
    const uint32_t* c0 = cin + (uint64_t)pr.poly0 * N;
    const uint32_t* c1 = cin + (uint64_t)pr.poly1 * N;
    uint32_t* out = d.ct[par ^ 1u] + (uint64_t)p * g.ct_words;
    const uint2* key = d.key[pr.b][s] + ((uint64_t)i * L + i) * 2 * N;
    const uint4* kq = reinterpret_cast<const uint4*>(key);
    const uint32_t* pbase = d.part[par] + ((uint64_t)p * P + gp) * (kDfLmax - 1) * 2 * N;
#pragma unroll 1
    for (uint32_t h = 0; h < SPT / 4; ++h) {
      const uint32_t x = xarg * QP + (h * 512 + j) * 4;
      const uint4 pm = __ldg(reinterpret_cast<const uint4*>(d.perm[s] + x));
      const uint32_t g1[4] = {__ldcg(c1 + pm.x), __ldcg(c1 + pm.y), __ldcg(c1 + pm.z), __ldcg(c1 + pm.w)};
      const uint32_t g0[4] = {__ldcg(c0 + pm.x), __ldcg(c0 + pm.y), __ldcg(c0 + pm.z), __ldcg(c0 + pm.w)};
      // key K[i][i] of the 4 slots: pass-C layout, slot 16 jj + k at uint2 ((k >> 1) T + jj) * 2 + (k & 1)
      const uint32_t jj = x >> 4, kk = x & 15u;
      const uint4 ka = __ldg(kq + (kk >> 1) * T + jj), kb = __ldg(kq + ((kk >> 1) + 1) * T + jj);
      const uint4 ku = __ldg(kq + N / 2 + (kk >> 1) * T + jj), kv = __ldg(kq + N / 2 + ((kk >> 1) + 1) * T + jj);
      uint32_t a0[4], a1[4];
      a0[0] = add_mod(mul_shoup(g1[0], ka.x, ka.y, q), g0[0], q);
      a0[1] = add_mod(mul_shoup(g1[1], ka.z, ka.w, q), g0[1], q);
      a0[2] = add_mod(mul_shoup(g1[2], kb.x, kb.y, q), g0[2], q);
      a0[3] = add_mod(mul_shoup(g1[3], kb.z, kb.w, q), g0[3], q);
      a1[0] = mul_shoup(g1[0], ku.x, ku.y, q);
      a1[1] = mul_shoup(g1[1], ku.z, ku.w, q);
      a1[2] = mul_shoup(g1[2], kv.x, kv.y, q);
      a1[3] = mul_shoup(g1[3], kv.z, kv.w, q);
      const uint32_t* pb = pbase + x;
      uint4 v[2 * (kDfLmax - 1)];
#pragma unroll
      for (int sl = 0; sl < kDfLmax - 1; ++sl)
        if ((uint32_t)sl + 1 < L) {
          v[2 * sl] = ldcg4(pb + (uint64_t)(2 * sl) * N);
          v[2 * sl + 1] = ldcg4(pb + (uint64_t)(2 * sl + 1) * N);
        }
#pragma unroll
      for (int sl = 0; sl < kDfLmax - 1; ++sl)
        if ((uint32_t)sl + 1 < L) {
          a0[0] = add_mod(a0[0], v[2 * sl].x, q);
          a0[1] = add_mod(a0[1], v[2 * sl].y, q);
          a0[2] = add_mod(a0[2], v[2 * sl].z, q);
          a0[3] = add_mod(a0[3], v[2 * sl].w, q);
          a1[0] = add_mod(a1[0], v[2 * sl + 1].x, q);
          a1[1] = add_mod(a1[1], v[2 * sl + 1].y, q);
          a1[2] = add_mod(a1[2], v[2 * sl + 1].z, q);
          a1[3] = add_mod(a1[3], v[2 * sl + 1].w, q);
        }
      // fold: c' = c + rot(c)   (sum_all_slots, backend.cpp:67-68)
      const uint4 u = ldcg4(c0 + x), w = ldcg4(c1 + x);
      *reinterpret_cast<uint4*>(out + (uint64_t)pr.poly0 * N + x) =
          make_uint4(add_mod(a0[0], u.x, q), add_mod(a0[1], u.y, q), add_mod(a0[2], u.z, q), add_mod(a0[3], u.w, q));
      *reinterpret_cast<uint4*>(out + (uint64_t)pr.poly1 * N + x) =
          make_uint4(add_mod(a1[0], w.x, q), add_mod(a1[1], w.y, q), add_mod(a1[2], w.z, q), add_mod(a1[3], w.w, q));
    }
    __syncthreads();
    if (j == 0) {
      __threadfence();
      // the last R part enqueues the next rotation's digit
      if (atomicAdd(cntB, 1u) + 1 == kDfRParts * (s / 2 + 1) && s + 1 < d.S)
        st_release(d.queue + atomicAdd(d.tail, 1u), df_id(kDfD, s + 1, p, gp));
    }
  return enq_r;
}

__global__ void __launch_bounds__(512, 2) k_fold_dataflow(const __grid_constant__ Geo g,
                                                          const __grid_constant__ DfParams d) {
  __shared__ uint32_t task_s, slot_s;
  const uint32_t j = threadIdx.x;
  const uint32_t P = g.P;
  const uint32_t total = (uint32_t)df_tasks(d.S, d.pairs, P, d.KP);
  for (;;) {
    __syncthreads();  // the previous task's shared-memory reads are done
    if (j == 0) {
      const uint32_t k = atomicAdd(d.head, 1u);
      uint32_t t = 0xffffffffu;
      const unsigned long long t0 = d.trace ? gtimer() : 0;
      if (k < total) {
        uint32_t ns = 32;
        while ((t = ld_acquire(d.queue + k)) == 0xffffffffu) {
          __nanosleep(ns);
          ns = min(ns * 2, 128u);
        }
        if (d.trace) {
          uint32_t smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          d.trace[4 * k] = t0;
          d.trace[4 * k + 1] = gtimer();
          d.trace[4 * k + 3] = ((unsigned long long)t << 32) | smid;
        }
      }
      task_s = t;
      slot_s = k;
    }
    __syncthreads();
    const uint32_t t = task_s;
    if (t == 0xffffffffu) return;
    const uint32_t type = t >> 30, s = (t >> 26) & 15u, p = (t >> 14) & 0xfffu, gp = (t >> 10) & 15u,
                   xarg = (t >> 6) & 15u;
    uint32_t enq_r;  // thread 0: enqueue this (p, gp)'s R tasks after the publish
    if (type == kDfD)
      enq_r = df_task_D(g, d, s, p, gp, xarg);
    else if (type == kDfK)
      enq_r = df_task_K(g, d, s, p, gp, xarg);
    else
      enq_r = df_task_R(g, d, s, p, gp, xarg);
    if (j == 0) {
      if (enq_r) {  // the rotation's key-switch products and digit are all in
        const uint32_t k = atomicAdd(d.tail, kDfRParts);
        for (uint32_t qq = 0; qq < kDfRParts; ++qq) st_release(d.queue + k + qq, df_id(kDfR, s, p, gp, qq));
      }
      if (d.trace) d.trace[4 * slot_s + 2] = gtimer();
    }
  }
}
