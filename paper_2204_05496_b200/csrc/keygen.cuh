// Key generation on the device: TwinContext::keygen
// (proj/src/fpcrt/twin.cpp:41-48) = per branch BfvContext::keygen
// (proj/src/bfv/context.cpp:152-172) then make_galois_keys (:201-251), all
// drawing from ONE util::Prng stream (rng.hpp:19-68) in that order.
//
// Textually included by heinfer_b200.cu inside its kernel namespace.
//
// The stream is replayed on the device (k_mt_generate), then k_kg_plan walks
// the draw plan in order with one 1024-thread block: uniform_u64 rejection
// sampling (ternary bound 3, uniform bound q_i) is resolved exactly with a
// block-wide ballot scan, so a rejected draw shifts every later segment just
// as it does in the reference. Gaussian segments record their start; their
// only rejection (u1 == 0, probability 2^-53 per pair) is flagged.
#pragma once

struct KgSeg {
  uint32_t kind;   // 0 uniform (u32 out), 1 ternary (i8 out), 2 gaussian (i8 out)
  uint32_t n;      // values
  uint64_t bound;  // uniform_u64 bound
  uint64_t limit;  // bound * floor(UINT64_MAX / bound): draws >= limit are rejected
  uint64_t out;    // offset into out32 (uniform) or out8 (ternary / gaussian)
};

// err bits: 2 gaussian u1 == 0 rejection, 4 raw stream too short (retry).
__global__ void __launch_bounds__(1024) k_kg_plan(const uint64_t* __restrict__ raw, uint64_t avail,
                                                  const KgSeg* __restrict__ segs, uint32_t nseg,
                                                  uint32_t* __restrict__ out32, int8_t* __restrict__ out8,
                                                  uint64_t* __restrict__ gpos, uint64_t* __restrict__ used,
                                                  uint32_t* err) {
  __shared__ uint32_t wcount[32];
  __shared__ uint32_t s_last;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  uint64_t p = 0;
  bool fail = false;
  for (uint32_t si = 0; si < nseg && !fail; ++si) {
    const KgSeg sg = segs[si];
    if (sg.kind == 2) {
      if (p + sg.n > avail) {
        fail = true;
        break;
      }
      if (tid == 0) gpos[si] = p;
      for (uint32_t k = tid; k < sg.n / 2; k += blockDim.x)
        if ((raw[p + 2 * k] >> 11) == 0) atomicOr(err, 2u);
      p += sg.n;
      continue;
    }
    uint32_t got = 0;
    while (got < sg.n) {
      const uint64_t pos = p + tid;
      uint64_t v = 0;
      bool acc = false;
      if (pos < avail) {
        v = raw[pos];
        acc = v < sg.limit;
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, acc);
      if (lane == 0) wcount[wid] = __popc(bal);
      __syncthreads();
      uint32_t woff = 0, total = 0;
      for (uint32_t w = 0; w < nw; ++w) {
        const uint32_t cw = wcount[w];
        total += cw;
        woff += w < wid ? cw : 0u;
      }
      const uint32_t idx = got + woff + __popc(bal & ((1u << lane) - 1u));
      if (acc && idx < sg.n) {
        if (sg.kind == 0) out32[sg.out + idx] = (uint32_t)(v % sg.bound);
        else out8[sg.out + idx] = (int8_t)((int)(v % 3) - 1);
        if (idx == sg.n - 1) s_last = tid;
      }
      __syncthreads();
      if (got + total >= sg.n) {
        p += s_last + 1;
        got = sg.n;
      } else {
        p += blockDim.x;
        got += total;
        if (p >= avail) fail = true;
      }
      __syncthreads();  // wcount / s_last reuse
      if (fail) break;
    }
  }
  if (tid == 0) {
    if (fail) atomicOr(err, 4u);
    used[0] = p;
  }
}

__global__ void k_kg_gauss(const uint64_t* __restrict__ raw, const KgSeg* __restrict__ segs,
                           const uint64_t* __restrict__ gpos, int8_t* __restrict__ out8) {
  const KgSeg sg = segs[blockIdx.x];
  if (sg.kind != 2) return;
  const uint64_t p = gpos[blockIdx.x];
  for (uint32_t k = threadIdx.x; k < sg.n / 2; k += blockDim.x)
    heb_baseline::box_muller_pair(raw[p + 2 * k], raw[p + 2 * k + 1], out8[sg.out + 2 * k], out8[sg.out + 2 * k + 1]);
}

__device__ __forceinline__ uint32_t lift_i8(int v, uint32_t q) { return v < 0 ? q - (uint32_t)(-v) : (uint32_t)v; }

// Public key of branch b (context.cpp:152-172), block per prime i:
// p1 = a (coeff form), p0 = -(INTT(NTT(a) * NTT(s)) + e). pk [part][L][n] u64.
__global__ void k_kg_pk(Geo g, uint32_t b, const int8_t* __restrict__ e, const uint32_t* __restrict__ a,
                        const uint32_t* __restrict__ s_hat, uint64_t* __restrict__ pk) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n, i = blockIdx.x, gp = (b ? g.L[0] : 0) + i, L = g.L[b];
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t* ai = a + (uint64_t)i * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) sm[x] = ai[x];
  __syncthreads();
  ntt_fwd_smem(sm, g.fwd + (size_t)gp * n, pr.q, n, g.logn);
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x)
    sm[x] = mul_barrett(sm[x], s_hat[(uint64_t)gp * n + x], pr.q, pr.mu);
  __syncthreads();
  ntt_inv_smem(sm, g.inv + (size_t)gp * n, pr.q, n, g.logn, pr.last, pr.ninv);
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
    const uint32_t as = add_mod(sm[x], lift_i8(e[x], pr.q), pr.q);
    pk[(uint64_t)i * n + x] = as ? pr.q - as : 0u;
    pk[((uint64_t)L + i) * n + x] = ai[x];
  }
}

// Galois key rows of branch b (context.cpp:201-251), block per (gen e, l, i):
// a = uniform (taken as eval form), b = NTT([i == l] sigma_g(s) - e_l) - a * NTT(s)
// (= -(a s + NTT(e_l)) + [i == l] NTT(sigma_g(s)), exact mod q_i).
// gk [slot(e)][l][part][i][n] u64, slot = ascending-element position.
__global__ void k_kg_gk(Geo g, uint32_t b, const uint64_t* __restrict__ elts, const uint32_t* __restrict__ slot,
                        const int8_t* __restrict__ s, const int8_t* __restrict__ e, const uint32_t* __restrict__ a,
                        const uint32_t* __restrict__ s_hat, uint64_t* __restrict__ gk) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n, L = g.L[b];
  const uint32_t i = blockIdx.x % L, l = (blockIdx.x / L) % L, ge = blockIdx.x / (L * L);
  const uint32_t gp = (b ? g.L[0] : 0) + i;
  const PrimeInfo& pr = g.pr[gp];
  const int8_t* el = e + ((uint64_t)ge * L + l) * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) sm[x] = lift_i8(-(int)el[x], pr.q);
  __syncthreads();
  if (i == l) {  // sigma_g(s) over the integers (context.cpp:215-224); a permutation, no write races
    const uint64_t elt = elts[ge], two_n = 2ull * n;
    for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) {
      const uint64_t tgt = ((uint64_t)j * elt) % two_n;
      const int v = tgt < n ? (int)s[j] : -(int)s[j];
      const uint32_t t = (uint32_t)(tgt < n ? tgt : tgt - n);
      sm[t] = add_mod(sm[t], lift_i8(v, pr.q), pr.q);
    }
    __syncthreads();
  }
  ntt_fwd_smem(sm, g.fwd + (size_t)gp * n, pr.q, n, g.logn);
  const uint32_t* ar = a + (((uint64_t)ge * L + l) * L + i) * n;
  uint64_t* row = gk + (((uint64_t)slot[ge] * L + l) * 2 * L) * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
    const uint32_t av = ar[x];
    const uint32_t as = mul_barrett(av, s_hat[(uint64_t)gp * n + x], pr.q, pr.mu);
    row[(uint64_t)i * n + x] = sub_mod(sm[x], as, pr.q);
    row[((uint64_t)L + i) * n + x] = av;
  }
}
