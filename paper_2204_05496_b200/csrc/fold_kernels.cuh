// Fast-algorithm kernels (MatmulStream::push_row / finish, matmul.cpp:165-232):
// ciphertext NTTs, chunk products, digit INTTs, key switching (small-batch
// and latency kernels), mask + packed accumulation, bias and finish,
// weight/key preparation. Textually included by heinfer_b200.cu inside its
// kernel namespace (uses Geo, PrimeInfo, BranchInfo, Ntt, modmath).
#pragma once

// Forward (or inverse) NTT of whole twin ciphertexts in place: block per poly.
__global__ void k_ct_ntt(Geo g, uint32_t* __restrict__ cts, int inverse) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n, polys = 2 * g.P;
  const uint64_t poly_g = blockIdx.x;
  const uint32_t poly = (uint32_t)(poly_g % polys);
  const uint32_t gp = poly_prime(g, poly);
  uint32_t* p = cts + poly_g * n;
  const PrimeInfo& pr = g.pr[gp];
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) sm[x] = p[x];
  __syncthreads();
  if (inverse) ntt_inv_smem(sm, g.inv + (size_t)gp * n, pr.q, n, g.logn, pr.last, pr.ninv);
  else ntt_fwd_smem(sm, g.fwd + (size_t)gp * n, pr.q, n, g.logn);
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) p[x] = sm[x];
}

// Batched NTT of `count` polys of one flat prime (kernel-level seam).
__global__ void k_poly_ntt(Geo g, uint32_t gp, uint32_t* __restrict__ polys, int inverse) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n;
  uint32_t* p = polys + (uint64_t)blockIdx.x * n;
  const PrimeInfo& pr = g.pr[gp];
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) sm[x] = p[x];
  __syncthreads();
  if (inverse) ntt_inv_smem(sm, g.inv + (size_t)gp * n, pr.q, n, g.logn, pr.last, pr.ninv);
  else ntt_fwd_smem(sm, g.fwd + (size_t)gp * n, pr.q, n, g.logn);
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) p[x] = sm[x];
}

// dot[pair] = sum_k in[row][k] (.) W[j][k]   (push_row, matmul.cpp:176-184)
// One block per (pair, poly); pairs of the batch map to (slot s = pair / cols,
// j = pair % cols) and input rows are stored per batch slot.
__global__ void k_chunk_dot(Geo g, const uint32_t* __restrict__ in, const uint2* __restrict__ W, uint32_t cols,
                            uint32_t kc, uint32_t* __restrict__ dot) {
  const uint32_t n = g.n, polys = 2 * g.P;
  const uint32_t pair = blockIdx.x / polys, poly = blockIdx.x % polys;
  const uint32_t s = pair / cols, j = pair % cols;
  if (poly == 0) count_ops(g, kc, 0, kc - 1);  // push_row: kc products, kc - 1 merges (add_many)
  const uint32_t gp = poly_prime(g, poly);
  const uint32_t q = g.pr[gp].q;
  const uint32_t* src = in + ((uint64_t)s * kc * g.ct_words) + (uint64_t)poly * n;
  const uint2* wj = W + ((uint64_t)j * kc * g.pt_words) + (uint64_t)gp * n;
  uint32_t* dst = dot + (uint64_t)pair * g.ct_words + (uint64_t)poly * n;
  for (uint32_t x = threadIdx.x * 4; x < n; x += blockDim.x * 4) {
    uint32_t acc[4] = {0, 0, 0, 0};
    for (uint32_t k = 0; k < kc; ++k) {
      const uint4 a = *reinterpret_cast<const uint4*>(src + (uint64_t)k * g.ct_words + x);
      const uint4 w01 = *reinterpret_cast<const uint4*>(wj + (uint64_t)k * g.pt_words + x);
      const uint4 w23 = *reinterpret_cast<const uint4*>(wj + (uint64_t)k * g.pt_words + x + 2);
      acc[0] = add_mod(acc[0], mul_shoup(a.x, w01.x, w01.y, q), q);
      acc[1] = add_mod(acc[1], mul_shoup(a.y, w01.z, w01.w, q), q);
      acc[2] = add_mod(acc[2], mul_shoup(a.z, w23.x, w23.y, q), q);
      acc[3] = add_mod(acc[3], mul_shoup(a.w, w23.z, w23.w, q), q);
    }
    *reinterpret_cast<uint4*>(dst + x) = make_uint4(acc[0], acc[1], acc[2], acc[3]);
  }
}

// Same products for a batch of rows, organised so the weights are read once
// per block instead of once per pair: block = (poly, 256-slot tile, group of
// up to CG classes); each thread keeps its slot's weights for those classes
// (CG x kc (value, Shoup) pairs) in registers and streams the rows. The
// chunk sum is exact mod q, so the order of the adds does not matter.
template <int CG, int KC>
__global__ void __launch_bounds__(256) k_chunk_dot_rows(Geo g, const uint32_t* __restrict__ in,
                                                       const uint2* __restrict__ W, uint32_t cols, uint32_t rows,
                                                       uint32_t* __restrict__ dot) {
  const uint32_t n = g.n, polys = 2 * g.P, tiles = n / 256, groups = (cols + CG - 1) / CG;
  // class groups vary fastest: the blocks that stream the same input slots for
  // different class groups run side by side, so the rows are read from HBM
  // once and from L2 by the other groups
  const uint32_t cg = blockIdx.x % groups, tp = blockIdx.x / groups;
  if (tp >= tiles * polys) return;
  const uint32_t tile = tp % tiles, poly = tp / tiles;
  const uint32_t x = tile * 256 + threadIdx.x;
  const uint32_t gp = poly_prime(g, poly);
  const uint32_t q = g.pr[gp].q;
  const uint32_t j0 = cg * CG, nj = min((uint32_t)CG, cols - j0);
  if (poly == 0 && tile == 0) count_ops(g, (uint64_t)rows * nj * KC, 0, (uint64_t)rows * nj * (KC - 1));
  uint2 w[CG][KC];
#pragma unroll
  for (int jj = 0; jj < CG; ++jj)
#pragma unroll
    for (int k = 0; k < KC; ++k)
      w[jj][k] = jj < (int)nj ? __ldg(W + ((uint64_t)(j0 + jj) * KC + k) * g.pt_words + (uint64_t)gp * n + x)
                              : make_uint2(0, 0);
  // the next row's chunks are in flight while this row's products are formed
  // (the loop is bound by load latency x rows, not by bandwidth)
  const uint32_t* src0 = in + (uint64_t)poly * n + x;
  const uint64_t rstride = (uint64_t)KC * g.ct_words;
  uint32_t a[KC], an[KC];
#pragma unroll
  for (int k = 0; k < KC; ++k) an[k] = __ldg(src0 + (uint64_t)k * g.ct_words);
  for (uint32_t s = 0; s < rows; ++s) {
#pragma unroll
    for (int k = 0; k < KC; ++k) a[k] = an[k];
    if (s + 1 < rows) {
      const uint32_t* src = src0 + (uint64_t)(s + 1) * rstride;
#pragma unroll
      for (int k = 0; k < KC; ++k) an[k] = __ldg(src + (uint64_t)k * g.ct_words);
    }
#pragma unroll
    for (int jj = 0; jj < CG; ++jj) {
      if (jj >= (int)nj) break;
      uint32_t acc = 0;
#pragma unroll
      for (int k = 0; k < KC; ++k) acc = add_mod(acc, mul_shoup(a[k], w[jj][k].x, w[jj][k].y, q), q);
      dot[((uint64_t)s * cols + j0 + jj) * g.ct_words + (uint64_t)poly * n + x] = acc;
    }
  }
}

// Feature-block sharding: the chunk products of chunks
// [k0, k0 + kn) of every pair, each reduced mod q, added into an unreduced
// u64 dot accumulator (ranks' partials sum exactly; reduced by k_dot_reduce).
__global__ void k_chunk_dot_part(Geo g, const uint32_t* __restrict__ in, const uint2* __restrict__ W, uint32_t cols,
                                 uint32_t kc, uint32_t k0, uint32_t kn, unsigned long long* __restrict__ dot) {
  const uint32_t n = g.n, polys = 2 * g.P;
  const uint32_t pair = blockIdx.x / polys, poly = blockIdx.x % polys;
  const uint32_t s = pair / cols, j = pair % cols;
  const uint32_t gp = poly_prime(g, poly);
  const uint32_t q = g.pr[gp].q;
  const uint32_t* src = in + ((uint64_t)s * kn * g.ct_words) + (uint64_t)poly * n;
  const uint2* wj = W + ((uint64_t)j * kc * g.pt_words) + (uint64_t)gp * n;
  unsigned long long* dst = dot + (uint64_t)pair * g.ct_words + (uint64_t)poly * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
    uint32_t acc = 0;
    for (uint32_t k = 0; k < kn; ++k) {
      const uint2 wv = wj[(uint64_t)(k0 + k) * g.pt_words + x];
      acc = add_mod(acc, mul_shoup(src[(uint64_t)k * g.ct_words + x], wv.x, wv.y, q), q);
    }
    dst[x] += acc;
  }
}

__global__ void k_dot_reduce(Geo g, const unsigned long long* __restrict__ in, uint64_t cts, uint32_t* __restrict__ out) {
  const uint64_t total = cts * g.ct_words;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t poly = (uint32_t)((x % g.ct_words) / g.n);
    out[x] = (uint32_t)(in[x] % g.pr[poly_prime(g, poly)].q);
  }
}

// digit_l = INTT_l(sigma(c1)_l), block per (pair, gp)  (context.cpp:455-459)
__global__ void k_rot_digits(Geo g, const uint32_t* __restrict__ dot, const uint32_t* __restrict__ perm,
                             uint32_t* __restrict__ digits) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n;
  const uint32_t pair = blockIdx.x / g.P, gp = blockIdx.x % g.P;
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t* c1 = dot + (uint64_t)pair * g.ct_words + (uint64_t)pr.poly1 * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) sm[x] = c1[__ldg(&perm[x])];
  __syncthreads();
  ntt_inv_smem(sm, g.inv + (size_t)gp * n, pr.q, n, g.logn, pr.last, pr.ninv);
  uint32_t* d = digits + ((uint64_t)pair * g.P + gp) * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) d[x] = sm[x];
}

// Key switch for output prime i of branch b plus the fold add
// (context.cpp:467-506, backend.cpp:65-68):
//   acc_{0,1} = sum_l NTT_i(digit_l mod q_i) (.) K[l][{0,1}][i]
//   fold: out0 = c0 + sigma(c0) + acc0, out1 = c1 + acc1
//   else: out0 = sigma(c0) + acc0,      out1 = acc1
// The l == i term needs no transform: NTT_i(INTT_i(x)) = x exactly.
// Keys: K[e] laid out [i][l][part][n] (val, shoup).
__global__ void k_rot_keyswitch(Geo g, const uint32_t* __restrict__ dot, const uint32_t* __restrict__ digits,
                                const uint32_t* __restrict__ perm, const uint2* __restrict__ key0,
                                const uint2* __restrict__ key1, uint32_t* __restrict__ out, int fold) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n;
  uint32_t* work = sm;
  uint32_t* acc0 = sm + n;
  uint32_t* acc1 = sm + 2 * n;
  const uint32_t pair = blockIdx.x / g.P, gp = blockIdx.x % g.P;
  if (gp == 0) count_ops(g, 0, 1, fold ? 1 : 0);  // one rotation (+ the fold add) per pair (backend.cpp:63-73)
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, L = pr.L, i = pr.i;
  const uint32_t* ct = dot + (uint64_t)pair * g.ct_words;
  const uint32_t* c0 = ct + (uint64_t)pr.poly0 * n;
  const uint32_t* c1 = ct + (uint64_t)pr.poly1 * n;
  const uint2* key = (pr.b ? key1 : key0) + (uint64_t)i * L * 2 * n;
  {
    const uint2* k0 = key + (uint64_t)(i * 2 + 0) * n;
    const uint2* k1 = key + (uint64_t)(i * 2 + 1) * n;
    for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
      const uint32_t d = c1[__ldg(&perm[x])];
      const uint2 a = __ldg(&k0[x]), b = __ldg(&k1[x]);
      acc0[x] = mul_shoup(d, a.x, a.y, q);
      acc1[x] = mul_shoup(d, b.x, b.y, q);
    }
  }
  const uint32_t* dig = digits + ((uint64_t)pair * g.P + pr.first) * n;
  for (uint32_t l = 0; l < L; ++l) {
    if (l == i) continue;
    const uint32_t* src = dig + (uint64_t)l * n;
    if (pr.fast_reduce) {
      for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
        const uint32_t v = src[x];
        work[x] = min(v, v - q);
      }
    } else {
      for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) work[x] = src[x] % q;
    }
    __syncthreads();
    ntt_fwd_smem(work, g.fwd + (size_t)gp * n, q, n, g.logn);
    const uint2* k0 = key + (uint64_t)(l * 2 + 0) * n;
    const uint2* k1 = key + (uint64_t)(l * 2 + 1) * n;
    for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
      const uint32_t d = work[x];
      const uint2 a = __ldg(&k0[x]), b = __ldg(&k1[x]);
      acc0[x] = add_mod(acc0[x], mul_shoup(d, a.x, a.y, q), q);
      acc1[x] = add_mod(acc1[x], mul_shoup(d, b.x, b.y, q), q);
    }
    __syncthreads();
  }
  uint32_t* o = out + (uint64_t)pair * g.ct_words;
  uint32_t* o0 = o + (uint64_t)pr.poly0 * n;
  uint32_t* o1 = o + (uint64_t)pr.poly1 * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
    uint32_t r0 = add_mod(acc0[x], c0[__ldg(&perm[x])], q);
    uint32_t r1 = acc1[x];
    if (fold) {
      r0 = add_mod(r0, c0[x], q);
      r1 = add_mod(r1, c1[x], q);
    }
    o0[x] = r0;
    o1[x] = r1;
  }
}

// packed[g / N] += mask_{g mod N} (.) dot   (matmul.cpp:187-196, mask :288-305)
// mask = NTT_q(lift(INTT_t(onehot at index_map[slot]))), regenerated per pair
// exactly as the reference does for N > 4096. u64 atomics make the packed
// accumulation order-free (mod-q addition is exact; reduced in k_finish_add).
__global__ void k_mask_acc(Geo g, const uint32_t* __restrict__ dot, const uint64_t* __restrict__ rows,
                           uint32_t cols, unsigned long long* __restrict__ acc64) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n;
  const uint32_t pair = blockIdx.x / g.P, gp = blockIdx.x % g.P;
  if (gp == 0) count_ops(g, 1, 0, 1);  // mask product + packed accumulation per pair (matmul.cpp:187-196)
  const PrimeInfo& pr = g.pr[gp];
  const BranchInfo& br = g.br[pr.b];
  const uint64_t gidx = rows[pair / cols] * cols + pair % cols;
  const uint32_t slot = (uint32_t)(gidx % n);
  const uint64_t c = gidx / n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) sm[x] = 0;
  __syncthreads();
  if (threadIdx.x == 0) sm[g.index_map[slot]] = 1;
  __syncthreads();
  ntt_inv_smem(sm, g.inv + (size_t)(g.P + pr.b) * n, br.t, n, g.logn, br.last, br.ninv);
  const uint32_t q = pr.q;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) sm[x] = sm[x] % q;
  __syncthreads();
  ntt_fwd_smem(sm, g.fwd + (size_t)gp * n, q, n, g.logn);
  const uint32_t* d0 = dot + (uint64_t)pair * g.ct_words + (uint64_t)pr.poly0 * n;
  const uint32_t* d1 = dot + (uint64_t)pair * g.ct_words + (uint64_t)pr.poly1 * n;
  unsigned long long* a0 = acc64 + (c * g.ct_words) + (uint64_t)pr.poly0 * n;
  unsigned long long* a1 = acc64 + (c * g.ct_words) + (uint64_t)pr.poly1 * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
    const uint32_t m = sm[x];
    atomicAdd(&a0[x], (unsigned long long)mul_barrett(d0[x], m, q, pr.mu));
    atomicAdd(&a1[x], (unsigned long long)mul_barrett(d1[x], m, q, pr.mu));
  }
}

// finish (matmul.cpp:200-232): reduce the u64 packed sums mod q and add the
// bias pattern: part0 += NTT_q(Delta * INTT_t(scatter(pattern)))
// (context.cpp:393-402). Block per (packed ct c, gp).
// Bias plaintext of every packed ciphertext (MatmulStream::finish,
// matmul.cpp:200-232): slot s of ct c carries bias[(cN + s) mod |Y|] while
// cN + s < R|Y|; encode_slots -> INTT_t -> Delta * lift -> NTT_q. One block
// per (c, prime); independent of the fold, so it runs on a side stream.
__global__ void k_bias_plain(Geo g, const int64_t* __restrict__ bias, uint32_t cols, uint64_t total,
                             uint32_t* __restrict__ biasp) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n;
  const uint64_t c = blockIdx.x / g.P;
  const uint32_t gp = blockIdx.x % g.P;
  const PrimeInfo& pr = g.pr[gp];
  const BranchInfo& br = g.br[pr.b];
  const int64_t t = br.t;
  for (uint32_t s = threadIdx.x; s < n; s += blockDim.x) {
    const uint64_t gi = c * n + s;
    int64_t v = gi < total ? bias[gi % cols] : 0;
    int64_t r = v % t;
    if (r < 0) r += t;
    sm[g.index_map[s]] = (uint32_t)r;
  }
  __syncthreads();
  ntt_inv_smem(sm, g.inv + (size_t)(g.P + pr.b) * n, br.t, n, g.logn, br.last, br.ninv);
  const uint32_t q = pr.q;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) sm[x] = mul_shoup(sm[x], pr.delta.x, pr.delta.y, q);
  __syncthreads();
  ntt_fwd_smem(sm, g.fwd + (size_t)gp * n, q, n, g.logn);
  uint32_t* o = biasp + blockIdx.x * (uint64_t)n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) o[x] = sm[x];
}

// Packed accumulators mod q plus the bias plaintext on part 0.
__global__ void k_finish_add(Geo g, const unsigned long long* __restrict__ acc64, const uint32_t* __restrict__ biasp,
                             uint64_t C, uint32_t* __restrict__ out, const unsigned long long* __restrict__ ops0,
                             unsigned long long* ops_out) {
  // the call's op counters: start snapshot and current values (every
  // counting kernel of the call precedes this one on the stream)
  if (ops_out && blockIdx.x == 0 && threadIdx.x < 3) {
    ops_out[threadIdx.x] = __ldcg(ops0 + threadIdx.x);
    ops_out[3 + threadIdx.x] = __ldcg(g.ops + threadIdx.x);
  }
  const uint64_t total = C * g.ct_words;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = x / g.ct_words;
    const uint32_t w = (uint32_t)(x % g.ct_words), poly = w / g.n, k = w % g.n;
    const uint32_t gp = poly_prime(g, poly);
    const PrimeInfo& pr = g.pr[gp];
    uint32_t v = (uint32_t)(acc64[x] % pr.q);
    if (poly == pr.poly0) v = add_mod(v, biasp[(c * g.P + gp) * g.n + k], pr.q);
    out[x] = v;
  }
}

// encode_weights on the device (matmul.cpp:83-104): block per (j, k, gp):
// slots -> centered residues mod t_b -> scatter -> INTT_t -> lift -> NTT_q.
__global__ void k_encode_weights(Geo g, const int64_t* __restrict__ w, uint64_t f, uint32_t cols, uint32_t kc,
                                 uint2* __restrict__ W) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = g.n;
  const uint32_t gp = blockIdx.x % g.P;
  const uint32_t jk = blockIdx.x / g.P;
  const uint32_t j = jk / kc, k = jk % kc;
  const PrimeInfo& pr = g.pr[gp];
  const BranchInfo& br = g.br[pr.b];
  const int64_t t = br.t;
  for (uint32_t s = threadIdx.x; s < n; s += blockDim.x) {
    const uint64_t feat = (uint64_t)k * n + s;
    int64_t v = feat < f ? w[feat * cols + j] : 0;
    int64_t r = v % t;
    if (r < 0) r += t;
    sm[g.index_map[s]] = (uint32_t)r;
  }
  __syncthreads();
  ntt_inv_smem(sm, g.inv + (size_t)(g.P + pr.b) * n, br.t, n, g.logn, br.last, br.ninv);
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) sm[x] = sm[x] % pr.q;
  __syncthreads();
  ntt_fwd_smem(sm, g.fwd + (size_t)gp * n, pr.q, n, g.logn);
  uint2* dst = W + ((uint64_t)jk * g.pt_words) + (uint64_t)gp * n;
  for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
    const uint32_t v = sm[x];
    dst[x] = make_uint2(v, (uint32_t)(((uint64_t)v << 32) / pr.q));
  }
}

// Prepared u64 values -> (val, shoup) with a range check.
__global__ void k_prepare_plain(Geo g, const uint64_t* __restrict__ vals, uint64_t count, uint2* __restrict__ out,
                                uint32_t* err) {
  const uint64_t total = count * g.pt_words;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t gp = (uint32_t)((x % g.pt_words) / g.n);
    const uint32_t q = g.pr[gp].q;
    const uint64_t v = vals[x];
    if (v >= q) *err = 1;
    out[x] = make_uint2((uint32_t)v, (uint32_t)((v << 32) / q));
  }
}

// Galois keys of one branch: host [e][l][part][i][n] u64 -> device
// [e][i][l][part][n] (val, shoup), the order k_rot_keyswitch streams them.
__global__ void k_prepare_keys(Geo g, uint32_t b, uint32_t elts, const uint64_t* __restrict__ rows,
                               uint2* __restrict__ out, uint32_t* err) {
  constexpr uint32_t V = 16;  // slots per thread of the register-blocked transforms
  const uint32_t n = g.n, L = g.L[b], first = b ? g.L[0] : 0;
  const uint64_t total = (uint64_t)elts * L * 2 * L * n;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total;
       x += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t r = x;
    const uint32_t c = (uint32_t)(r % n);
    r /= n;
    const uint32_t i = (uint32_t)(r % L);
    r /= L;
    const uint32_t part = (uint32_t)(r % 2);
    r /= 2;
    const uint32_t l = (uint32_t)(r % L);
    const uint64_t e = r / L;
    const uint32_t q = g.pr[first + i].q;
    const uint64_t v = rows[x];
    if (v >= q) *err = 1;
    // register-blocked rings (n >= 8192): pass-C transposed layout for V slots
    // per thread, slot x = V j + 2 c' + h stored at uint2 index
    // (c' * (n / V) + j) * 2 + h
    uint32_t cpos = c;
    if (n >= 8192) {
      const uint32_t jj = c / V, rr = c % V;
      cpos = ((rr >> 1) * (n / V) + jj) * 2 + (rr & 1);
    }
    const uint64_t dst = ((((e * L + i) * L + l) * 2 + part) * n) + cpos;
    out[dst] = make_uint2((uint32_t)v, (uint32_t)((v << 32) / q));
  }
}


// ---------------------------------------------------------------------------
// Register-blocked kernels (N = 2^LOGN, LOGN in 13..14, T = N/16 threads).
// ---------------------------------------------------------------------------
template <int LOGN>
__global__ void __launch_bounds__(Ntt<LOGN>::T) k_poly_ntt_f(Geo g, uint32_t gp, uint32_t* __restrict__ polys,
                                                            int inverse) {
  using NT = Ntt<LOGN>;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  const uint32_t j = threadIdx.x, x0 = NT::posC0(j);
  uint32_t* p = polys + (uint64_t)blockIdx.x * NT::N;
  const PrimeInfo& pr = g.pr[gp];
  uint32_t e[16];
  if (inverse) {
#pragma unroll
    for (int r = 0; r < 16; ++r) e[r] = p[x0 + r];
    NT::inv(e, sm, g.inv + (size_t)gp * NT::N, g.itwc + (size_t)gp * g.twc_stride, pr.q, pr.last, pr.ninv);
#pragma unroll
    for (int r = 0; r < 16; ++r) p[NT::posA(j, r)] = e[r];
  } else {
#pragma unroll
    for (int r = 0; r < 16; ++r) e[r] = p[NT::posA(j, r)];
    NT::fwd(e, sm, g.fwd + (size_t)gp * NT::N, g.twc + (size_t)gp * g.twc_stride, pr.q);
#pragma unroll
    for (int r = 0; r < 16; ++r) p[x0 + r] = e[r];
  }
}

template <int LOGN>
__global__ void __launch_bounds__(Ntt<LOGN>::T) k_ct_ntt_f(Geo g, uint32_t* __restrict__ cts) {
  using NT = Ntt<LOGN>;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  const uint32_t polys = 2 * g.P;
  const uint32_t poly = (uint32_t)(blockIdx.x % polys);
  const uint32_t gp = poly_prime(g, poly);
  uint32_t* p = cts + (uint64_t)blockIdx.x * NT::N;
  const uint32_t j = threadIdx.x, x0 = NT::posC0(j);
  uint32_t e[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) e[r] = p[NT::posA(j, r)];
  NT::fwd(e, sm, g.fwd + (size_t)gp * NT::N, g.twc + (size_t)gp * g.twc_stride, g.pr[gp].q);
#pragma unroll
  for (int r = 0; r < 16; ++r) p[x0 + r] = e[r];
}

// to_coeff of whole twin ciphertexts (context.cpp to_coeff / serialize.cpp:67-71).
template <int LOGN>
__global__ void __launch_bounds__(Ntt<LOGN>::T) k_ct_intt_f(Geo g, uint32_t* __restrict__ cts) {
  using NT = Ntt<LOGN>;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  const uint32_t polys = 2 * g.P;
  const uint32_t poly = (uint32_t)(blockIdx.x % polys);
  const uint32_t gp = poly_prime(g, poly);
  const PrimeInfo& pr = g.pr[gp];
  uint32_t* p = cts + (uint64_t)blockIdx.x * NT::N;
  const uint32_t j = threadIdx.x, x0 = NT::posC0(j);
  uint32_t e[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) e[r] = p[x0 + r];
  NT::inv(e, sm, g.inv + (size_t)gp * NT::N, g.itwc + (size_t)gp * g.twc_stride, pr.q, pr.last, pr.ninv);
#pragma unroll
  for (int r = 0; r < 16; ++r) p[NT::posA(j, r)] = e[r];
}

__device__ __forceinline__ void load16(const uint32_t* __restrict__ p, uint32_t (&v)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 a = *reinterpret_cast<const uint4*>(p + 4 * c);
    v[4 * c] = a.x;
    v[4 * c + 1] = a.y;
    v[4 * c + 2] = a.z;
    v[4 * c + 3] = a.w;
  }
}
__device__ __forceinline__ void load16_ro(const uint32_t* __restrict__ p, uint32_t (&v)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(p + 4 * c));
    v[4 * c] = a.x;
    v[4 * c + 1] = a.y;
    v[4 * c + 2] = a.z;
    v[4 * c + 3] = a.w;
  }
}
__device__ __forceinline__ void store16(uint32_t* __restrict__ p, const uint32_t (&v)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c)
    *reinterpret_cast<uint4*>(p + 4 * c) = make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
}

// digit_l = INTT_l(sigma(c1)_l), block per (pair, gp) (context.cpp:455-459).
// A thread's 16 sources form one aligned 16-slot group (the automorphism maps
// groups onto groups): 4 x 128-bit loads, permuted through a per-thread
// shared-memory column (conflict-free, no barrier before the transform's own).
template <int LOGN, bool PTW>
__global__ void __launch_bounds__(Ntt<LOGN>::T, (LOGN <= 13 ? 3 : 1)) k_rot_digits_f(Geo g, const uint32_t* __restrict__ dot,
                                                              const uint32_t* __restrict__ perm,
                                                              uint32_t* __restrict__ digits,
                                                              const __grid_constant__ TwArg<PTW> itab) {
  using NT = Ntt<LOGN>;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  uint32_t pair, gp;
  block_pair_prime(g, pair, gp);
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t* c1 = dot + (uint64_t)pair * g.ct_words + (uint64_t)pr.poly1 * NT::N;
  const uint32_t j = threadIdx.x, x0 = NT::posC0(j);
  uint32_t pm[16], e[16];
  load16_ro(perm + x0, pm);
  {
    const uint4* gs = reinterpret_cast<const uint4*>(c1 + (pm[0] & ~15u));
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 v = __ldg(gs + c);
      sm[(4 * c) * NT::T + j] = v.x;
      sm[(4 * c + 1) * NT::T + j] = v.y;
      sm[(4 * c + 2) * NT::T + j] = v.z;
      sm[(4 * c + 3) * NT::T + j] = v.w;
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) e[r] = sm[(pm[r] & 15u) * NT::T + j];
  }
  if constexpr (PTW)
    NT::inv(e, sm, ParamTw{itab.w[gp]}, g.itwc + (size_t)gp * g.twc_stride, pr.q, pr.last, pr.ninv);
  else
    NT::inv(e, sm, g.inv + (size_t)gp * NT::N, g.itwc + (size_t)gp * g.twc_stride, pr.q, pr.last, pr.ninv);
  uint32_t* d = digits + ((uint64_t)pair * g.P + gp) * NT::N;
#pragma unroll
  for (int r = 0; r < 16; ++r) d[NT::posA(j, r)] = e[r];
}

// Key switch with the two accumulators in shared memory
// (transposed [c][T] uint4, conflict-free), which keeps the kernel under 64
// registers so two 512-thread CTAs share an SM (32 warps for latency hiding).
template <int LOGN, bool PTW, bool NEXT>
__global__ void __launch_bounds__(Ntt<LOGN>::T, (LOGN <= 13 ? 2 : 1)) k_rot_keyswitch_s(Geo g, const uint32_t* __restrict__ dot,
                                                                    const uint32_t* __restrict__ digits,
                                                                    const uint32_t* __restrict__ perm,
                                                                    const uint2* __restrict__ key0,
                                                                    const uint2* __restrict__ key1,
                                                                    uint32_t* __restrict__ out, int fold,
                                                                    const uint32_t* __restrict__ perm_next,
                                                                    uint32_t* __restrict__ dig_next,
                                                                    const __grid_constant__ TwArg<PTW> tab) {
  using NT = Ntt<LOGN>;
  constexpr uint32_t N = NT::N, T = NT::T;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  uint4* a0s = smem4 + N / 4;
  uint4* a1s = a0s + 4 * T;
  const uint32_t pair = blockIdx.x / g.P, gp = blockIdx.x % g.P;
  if (gp == 0) count_ops(g, 0, 1, fold ? 1 : 0);  // one rotation (+ the fold add) per pair (backend.cpp:63-73)
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, L = pr.L, i = pr.i;
  const uint32_t j = threadIdx.x, x0 = NT::posC0(j);
  const uint32_t* ct = dot + (uint64_t)pair * g.ct_words;
  const uint32_t* c0 = ct + (uint64_t)pr.poly0 * N;
  const uint32_t* c1 = ct + (uint64_t)pr.poly1 * N;
  const uint2* key = (pr.b ? key1 : key0) + (uint64_t)i * L * 2 * N;
  // c1 (and, for the epilogue, c0) arrive in `sm` by one TMA bulk copy each;
  // the Galois gathers then read shared memory instead of scattering 4-byte
  // loads over L1/L2
  __shared__ uint64_t gbar;
  if (threadIdx.x == 0) {
    mbar_init(&gbar, 1);
    bulk_load(sm, c1, N * 4, &gbar);
  }
  __syncthreads();  // the barrier is initialised before anyone waits on it
  mbar_wait(&gbar, 0);
  {
    const uint4* k0 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * i) * N) + j;
    const uint4* k1 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * i + 1) * N) + j;
    const uint4* pp = reinterpret_cast<const uint4*>(perm + x0);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 pm = __ldg(pp + c);
      const uint32_t d0 = sm[pm.x], d1 = sm[pm.y], d2 = sm[pm.z], d3 = sm[pm.w];
      const uint4 a = __ldg(k0 + (2 * c) * T), b = __ldg(k0 + (2 * c + 1) * T);
      const uint4 u = __ldg(k1 + (2 * c) * T), v = __ldg(k1 + (2 * c + 1) * T);
      a0s[c * T + j] = make_uint4(mul_shoup(d0, a.x, a.y, q), mul_shoup(d1, a.z, a.w, q), mul_shoup(d2, b.x, b.y, q),
                                  mul_shoup(d3, b.z, b.w, q));
      a1s[c * T + j] = make_uint4(mul_shoup(d0, u.x, u.y, q), mul_shoup(d1, u.z, u.w, q), mul_shoup(d2, v.x, v.y, q),
                                  mul_shoup(d3, v.z, v.w, q));
    }
  }
  const uint32_t* dig = digits + ((uint64_t)pair * g.P + pr.first) * N;
  const uint4* twc = g.twc + (size_t)gp * g.twc_stride;
  uint32_t e[16];
  for (uint32_t l = 0; l < L; ++l) {
    if (l == i) continue;
    {
      const uint32_t* src = dig + (uint64_t)l * N;
      // (the digit enters unreduced: see k_rot_keyswitch_t)
#pragma unroll
      for (int r = 0; r < 16; ++r) e[r] = src[NT::posA(j, r)];
    }
    if constexpr (PTW)
      NT::template fwd<true>(e, sm, ParamTw{tab.w[gp]}, twc, q);
    else
      NT::template fwd<true>(e, sm, g.fwd + (size_t)gp * N, twc, q);
    const uint4* k0 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * l) * N) + j;
    const uint4* k1 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * l + 1) * N) + j;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 a = __ldg(k0 + (2 * c) * T), b = __ldg(k0 + (2 * c + 1) * T);
      uint4 A = a0s[c * T + j];
      A.x = add_mod(A.x, mul_shoup(e[4 * c], a.x, a.y, q), q);
      A.y = add_mod(A.y, mul_shoup(e[4 * c + 1], a.z, a.w, q), q);
      A.z = add_mod(A.z, mul_shoup(e[4 * c + 2], b.x, b.y, q), q);
      A.w = add_mod(A.w, mul_shoup(e[4 * c + 3], b.z, b.w, q), q);
      a0s[c * T + j] = A;
      const uint4 u = __ldg(k1 + (2 * c) * T), v = __ldg(k1 + (2 * c + 1) * T);
      uint4 B = a1s[c * T + j];
      B.x = add_mod(B.x, mul_shoup(e[4 * c], u.x, u.y, q), q);
      B.y = add_mod(B.y, mul_shoup(e[4 * c + 1], u.z, u.w, q), q);
      B.z = add_mod(B.z, mul_shoup(e[4 * c + 2], v.x, v.y, q), q);
      B.w = add_mod(B.w, mul_shoup(e[4 * c + 3], v.z, v.w, q), q);
      a1s[c * T + j] = B;
    }
  }
  uint32_t* o = out + (uint64_t)pair * g.ct_words;
  const uint4* pp = reinterpret_cast<const uint4*>(perm + x0);
  __syncthreads();  // the last NTT's exchange reads of sm are done
  if constexpr (!NEXT) {
    if (threadIdx.x == 0) {
      fence_proxy_async_smem();
      bulk_load(sm, c0, N * 4, &gbar);
    }
    mbar_wait(&gbar, 1);
  }
  const uint32_t* g0 = NEXT ? c0 : sm;  // NEXT reuses sm for the next digit
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 pm = __ldg(pp + c);
    uint4 A = a0s[c * T + j], B = a1s[c * T + j];
    A.x = add_mod(A.x, g0[pm.x], q);
    A.y = add_mod(A.y, g0[pm.y], q);
    A.z = add_mod(A.z, g0[pm.z], q);
    A.w = add_mod(A.w, g0[pm.w], q);
    if (fold) {
      const uint4 u = *reinterpret_cast<const uint4*>(g0 + x0 + 4 * c);
      const uint4 v = *reinterpret_cast<const uint4*>(c1 + x0 + 4 * c);
      A.x = add_mod(A.x, u.x, q);
      A.y = add_mod(A.y, u.y, q);
      A.z = add_mod(A.z, u.z, q);
      A.w = add_mod(A.w, u.w, q);
      B.x = add_mod(B.x, v.x, q);
      B.y = add_mod(B.y, v.y, q);
      B.z = add_mod(B.z, v.z, q);
      B.w = add_mod(B.w, v.w, q);
    }
    *reinterpret_cast<uint4*>(o + (uint64_t)pr.poly0 * N + x0 + 4 * c) = A;
    *reinterpret_cast<uint4*>(o + (uint64_t)pr.poly1 * N + x0 + 4 * c) = B;
    if constexpr (NEXT) *reinterpret_cast<uint4*>(sm + x0 + 4 * c) = B;
  }
  if constexpr (NEXT) {
    // Fused digit INTT of the NEXT rotation (apply_galois, context.cpp:445-470):
    // this block owns prime i of the new c1, so it permutes it from shared
    // memory and inverse-transforms it here instead of in k_rot_digits_f.
    __syncthreads();
    uint32_t pm[16];
    load16_ro(perm_next + x0, pm);
#pragma unroll
    for (int r = 0; r < 16; ++r) e[r] = sm[pm[r]];
    __syncthreads();
    NT::inv(e, sm, g.inv + (size_t)gp * N, g.itwc + (size_t)gp * g.twc_stride, q, pr.last, pr.ninv);
    uint32_t* d = dig_next + ((uint64_t)pair * g.P + gp) * N;
#pragma unroll
    for (int r = 0; r < 16; ++r) d[NT::posA(j, r)] = e[r];
  }
}


// Latency path, one CTA per (pair, prime i) with TWO 512-thread groups:
// group 0 takes the l == i term and the first floor(L/2) digits, group 1 the
// rest, each into its own shared accumulators (group barriers, 32 warps per
// SM instead of 16); the groups then finalise half of the slots each and
// group 1 runs the next rotation's digit INTT. Same arithmetic as
// k_rot_keyswitch_s.
#ifdef HEI_W2_TRACE  // debug builds only: per-(block, group) phase timestamps of the latency kernel
__device__ unsigned long long g_w2_trace[256][2][8];
#define W2T(k)                                                                                       \
  do {                                                                                               \
    if (threadIdx.x % T == 0 && blockIdx.x < 256) {                                                  \
      unsigned long long t_;                                                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                       \
      g_w2_trace[blockIdx.x][grp][k] = t_;                                                           \
    }                                                                                                \
  } while (0)
#else
#define W2T(k) \
  do {         \
  } while (0)
#endif
template <int LOGN, bool NEXT>
__global__ void __launch_bounds__(2 * Ntt<LOGN>::T, 1) k_rot_keyswitch_w2(
    Geo g, const uint32_t* __restrict__ dot, const uint32_t* __restrict__ digits, const uint32_t* __restrict__ perm,
    const uint2* __restrict__ key0, const uint2* __restrict__ key1, uint32_t* __restrict__ out, int fold,
    const uint32_t* __restrict__ perm_next, uint32_t* __restrict__ dig_next, const uint2* __restrict__ knext0,
    const uint2* __restrict__ knext1) {
  using NT = Ntt<LOGN, 2>;
  constexpr uint32_t N = NT::N, T = NT::T;
  extern __shared__ uint4 smem4[];
  const uint32_t grp = threadIdx.x / T;
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4 + grp * (3 * N / 4));
  uint4* a0s = smem4 + grp * (3 * N / 4) + N / 4;
  uint4* a1s = a0s + 4 * T;
  uint4* o0s = smem4 + (grp ^ 1u) * (3 * N / 4) + N / 4;  // the other group's accumulators
  uint4* o1s = o0s + 4 * T;
  uint32_t* sm1 = reinterpret_cast<uint32_t*>(smem4 + 3 * N / 4);  // group 1's buffer
  // programmatic dependent launch: the next rotation's grid may be scheduled
  // now (onto the idle SMs); this grid's inputs are the previous one's outputs
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t pair = blockIdx.x / g.P, gp = blockIdx.x % g.P;
  if (gp == 0) count_ops(g, 0, 1, fold ? 1 : 0);  // one rotation (+ the fold add) per pair (backend.cpp:63-73)
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, L = pr.L, i = pr.i;
  const uint32_t j = threadIdx.x % T, x0 = NT::posC0(j);
  const uint32_t* ct = dot + (uint64_t)pair * g.ct_words;
  const uint32_t* c0 = ct + (uint64_t)pr.poly0 * N;
  const uint32_t* c1 = ct + (uint64_t)pr.poly1 * N;
  const uint2* key = (pr.b ? key1 : key0) + (uint64_t)i * L * 2 * N;
  if (knext0 && pair == 0 && threadIdx.x < 2 * L) {
    // pull the next rotation's key rows of prime i into L2 (the pairs of an
    // individual read them ~40 us from now; they would come from HBM)
    const uint2* kn = (pr.b ? knext1 : knext0) + (uint64_t)i * L * 2 * N + (uint64_t)threadIdx.x * N;
    bulk_prefetch_l2(kn, N * 8);
  }
  W2T(0);
  if (grp == 1) {  // the l == i term needs no transform (group 1 has the fewer digits)
    const uint4* k0 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * i) * N) + j;
    const uint4* k1 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * i + 1) * N) + j;
    const uint4* pp = reinterpret_cast<const uint4*>(perm + x0);
    {
      // sigma(c1)_i of the thread's slots: its one aligned 16-slot source
      // group, 4 x 128-bit loads into its column of the group's buffer
      const uint4* gs4 = reinterpret_cast<const uint4*>(c1 + (__ldg(perm + x0) & ~15u));
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint4 v = __ldg(gs4 + c);
        sm[(4 * c) * T + j] = v.x;
        sm[(4 * c + 1) * T + j] = v.y;
        sm[(4 * c + 2) * T + j] = v.z;
        sm[(4 * c + 3) * T + j] = v.w;
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 pm = __ldg(pp + c);
      const uint32_t d0 = sm[(pm.x & 15u) * T + j], d1 = sm[(pm.y & 15u) * T + j], d2 = sm[(pm.z & 15u) * T + j],
                     d3 = sm[(pm.w & 15u) * T + j];
      const uint4 a = __ldg(k0 + (2 * c) * T), b = __ldg(k0 + (2 * c + 1) * T);
      const uint4 u = __ldg(k1 + (2 * c) * T), v = __ldg(k1 + (2 * c + 1) * T);
      a0s[c * T + j] = make_uint4(mul_shoup(d0, a.x, a.y, q), mul_shoup(d1, a.z, a.w, q), mul_shoup(d2, b.x, b.y, q),
                                  mul_shoup(d3, b.z, b.w, q));
      a1s[c * T + j] = make_uint4(mul_shoup(d0, u.x, u.y, q), mul_shoup(d1, u.z, u.w, q), mul_shoup(d2, v.x, v.y, q),
                                  mul_shoup(d3, v.z, v.w, q));
    }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      a0s[c * T + j] = make_uint4(0, 0, 0, 0);
      a1s[c * T + j] = make_uint4(0, 0, 0, 0);
    }
  }
  W2T(1);
  const uint32_t* dig = digits + ((uint64_t)pair * g.P + pr.first) * N;
  const uint4* twc = g.twc + (size_t)gp * g.twc_stride;
  const uint32_t half = L / 2;  // digits (l != i) with index < half go to group 0
  uint32_t e[16];
  // this group's digits, in order
  uint32_t mine[8], cnt = 0;
  for (uint32_t l = 0, k = 0; l < L; ++l) {
    if (l == i) continue;
    if (((k++ < half) ? 0u : 1u) == grp) mine[cnt++] = l;
  }
  for (uint32_t u = 0; u < cnt; ++u) {
    const uint32_t l = mine[u];
    const uint32_t* src = dig + (uint64_t)l * N;
    // (the digit enters unreduced: see k_rot_keyswitch_t)
#pragma unroll
    for (int r = 0; r < 16; ++r) e[r] = src[NT::posA(j, r)];
    NT::template fwd<true>(e, sm, g.fwd + (size_t)gp * N, twc, q);
    const uint4* k0 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * l) * N) + j;
    const uint4* k1 = reinterpret_cast<const uint4*>(key + (uint64_t)(2 * l + 1) * N) + j;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 a = __ldg(k0 + (2 * c) * T), b = __ldg(k0 + (2 * c + 1) * T);
      uint4 A = a0s[c * T + j];
      A.x = add_mod(A.x, mul_shoup(e[4 * c], a.x, a.y, q), q);
      A.y = add_mod(A.y, mul_shoup(e[4 * c + 1], a.z, a.w, q), q);
      A.z = add_mod(A.z, mul_shoup(e[4 * c + 2], b.x, b.y, q), q);
      A.w = add_mod(A.w, mul_shoup(e[4 * c + 3], b.z, b.w, q), q);
      a0s[c * T + j] = A;
      const uint4 u = __ldg(k1 + (2 * c) * T), v = __ldg(k1 + (2 * c + 1) * T);
      uint4 B = a1s[c * T + j];
      B.x = add_mod(B.x, mul_shoup(e[4 * c], u.x, u.y, q), q);
      B.y = add_mod(B.y, mul_shoup(e[4 * c + 1], u.z, u.w, q), q);
      B.z = add_mod(B.z, mul_shoup(e[4 * c + 2], v.x, v.y, q), q);
      B.w = add_mod(B.w, mul_shoup(e[4 * c + 3], v.z, v.w, q), q);
      a1s[c * T + j] = B;
    }
    W2T(2 + u);
  }
  // sigma(c0) of thread j's slots: one aligned 16-slot source group, loaded
  // with 4 x 128-bit loads by group 0's thread j into its column of group
  // 0's exchange buffer (free once group 0's last transform is done); both
  // groups' thread j read it after the CTA barrier
  if (grp == 0) {
    const uint4* gs4 = reinterpret_cast<const uint4*>(c0 + (__ldg(perm + x0) & ~15u));
    uint4 g0v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) g0v[c] = __ldg(gs4 + c);
    NT::sync();  // group 0's transforms no longer read its buffer
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      sm[(4 * c) * T + j] = g0v[c].x;
      sm[(4 * c + 1) * T + j] = g0v[c].y;
      sm[(4 * c + 2) * T + j] = g0v[c].z;
      sm[(4 * c + 3) * T + j] = g0v[c].w;
    }
  }
  // the finish's independent loads, issued before the barrier
  uint4 pmf[2], uf[2], vf[2];
#pragma unroll
  for (int cc = 0; cc < 2; ++cc) {
    const uint32_t xc = x0 + 4 * (2 * grp + cc);
    pmf[cc] = __ldg(reinterpret_cast<const uint4*>(perm + xc));
    uf[cc] = *reinterpret_cast<const uint4*>(c0 + xc);
    vf[cc] = *reinterpret_cast<const uint4*>(c1 + xc);
  }
  W2T(5);
  __syncthreads();  // both groups' accumulators complete; all transforms done
  const uint32_t* col = reinterpret_cast<const uint32_t*>(smem4);  // group 0's exchange buffer
  uint32_t* o = out + (uint64_t)pair * g.ct_words;
#pragma unroll
  for (int cc = 0; cc < 2; ++cc) {  // group r finalises chunks {2r, 2r + 1}
    const int c = 2 * (int)grp + cc;
    const uint32_t xc = x0 + 4 * c;
    const uint4 pm = pmf[cc];
    uint4 A = a0s[c * T + j], B = a1s[c * T + j];
    const uint4 RA = o0s[c * T + j], RB = o1s[c * T + j];
    A.x = add_mod(A.x, RA.x, q);
    A.y = add_mod(A.y, RA.y, q);
    A.z = add_mod(A.z, RA.z, q);
    A.w = add_mod(A.w, RA.w, q);
    B.x = add_mod(B.x, RB.x, q);
    B.y = add_mod(B.y, RB.y, q);
    B.z = add_mod(B.z, RB.z, q);
    B.w = add_mod(B.w, RB.w, q);
    A.x = add_mod(A.x, col[(pm.x & 15u) * T + j], q);
    A.y = add_mod(A.y, col[(pm.y & 15u) * T + j], q);
    A.z = add_mod(A.z, col[(pm.z & 15u) * T + j], q);
    A.w = add_mod(A.w, col[(pm.w & 15u) * T + j], q);
    if (fold) {
      const uint4 u = uf[cc], v = vf[cc];
      A.x = add_mod(A.x, u.x, q);
      A.y = add_mod(A.y, u.y, q);
      A.z = add_mod(A.z, u.z, q);
      A.w = add_mod(A.w, u.w, q);
      B.x = add_mod(B.x, v.x, q);
      B.y = add_mod(B.y, v.y, q);
      B.z = add_mod(B.z, v.z, q);
      B.w = add_mod(B.w, v.w, q);
    }
    *reinterpret_cast<uint4*>(o + (uint64_t)pr.poly0 * N + xc) = A;
    *reinterpret_cast<uint4*>(o + (uint64_t)pr.poly1 * N + xc) = B;
    if constexpr (NEXT) *reinterpret_cast<uint4*>(sm1 + xc) = B;
  }
  W2T(6);
  if constexpr (NEXT) {
    __syncthreads();  // c1' complete in group 1's buffer
    if (grp == 1) {   // next rotation's digit: INTT of sigma'(c1') mod q_i
      uint32_t pm[16];
      load16_ro(perm_next + x0, pm);
#pragma unroll
      for (int r = 0; r < 16; ++r) e[r] = sm[pm[r]];
      NT::sync();
      NT::inv(e, sm, g.inv + (size_t)gp * N, g.itwc + (size_t)gp * g.twc_stride, q, pr.last, pr.ninv);
      uint32_t* d = dig_next + ((uint64_t)pair * g.P + gp) * N;
#pragma unroll
      for (int r = 0; r < 16; ++r) d[NT::posA(j, r)] = e[r];
      W2T(7);
    }
  }
}

// Mask multiply + packed accumulation, G pairs per block (matmul.cpp:187-196).
// The one-hot's INTT_t has a closed form: slot s sits at eval position
// p = index_map[s], i.e. at psi^(2 brv(p) + 1), so its coefficients are
// m_j = n^-1 * w^j (mod t) with w = psi^-(2 brv(p) + 1) — identical values to
// the reference's INTT. Products accumulate mod q in shared memory across
// the block's pairs and leave through one u64 atomic per slot and flush.
__device__ __forceinline__ uint32_t pow_barrett(uint32_t b, uint32_t e, uint32_t t, uint64_t mu) {
  uint32_t r = 1;
  while (e) {
    if (e & 1) r = mul_barrett(r, b, t, mu);
    b = mul_barrett(b, b, t, mu);
    e >>= 1;
  }
  return r;
}


// Latency path, split in two: the one-hot mask plaintexts (same closed form
// as k_mask_acc_g) depend only on the slot, so k_mask_prep computes them on a
// side stream while the fold runs; k_mask_apply then multiplies and adds.
// masks [pair][P][N] in eval order.
template <int LOGN>
__global__ void __launch_bounds__(Ntt<LOGN>::T) k_mask_prep(Geo g, const uint64_t* __restrict__ rows, uint32_t cols,
                                                           uint32_t* __restrict__ masks) {
  using NT = Ntt<LOGN>;
  constexpr uint32_t N = NT::N, T = NT::T;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  const uint32_t gp = blockIdx.x % g.P, pair = blockIdx.x / g.P;
  const PrimeInfo& pr = g.pr[gp];
  const BranchInfo& br = g.br[pr.b];
  const uint32_t q = pr.q, t = br.t, j = threadIdx.x, x0 = NT::posC0(j);
  const uint64_t gidx = rows[pair / cols] * cols + pair % cols;
  const uint32_t slot = (uint32_t)(gidx % N);
  const uint32_t pe = __brev(__ldg(&g.index_map[slot])) >> (32 - LOGN);
  const uint32_t w = pow_barrett(br.psi_inv, 2 * pe + 1, t, br.mu);
  const uint32_t wT = pow_barrett(w, T, t, br.mu);
  uint32_t m = mul_barrett(br.ninv.x, pow_barrett(w, j, t, br.mu), t, br.mu);
  uint32_t e[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    e[r] = m % q;
    m = mul_barrett(m, wT, t, br.mu);
  }
  NT::fwd(e, sm, g.fwd + (size_t)gp * N, g.twc + (size_t)gp * g.twc_stride, q);
  uint4* o = reinterpret_cast<uint4*>(masks + (uint64_t)blockIdx.x * N + x0);
#pragma unroll
  for (int c = 0; c < 4; ++c) o[c] = make_uint4(e[4 * c], e[4 * c + 1], e[4 * c + 2], e[4 * c + 3]);
}

__global__ void k_mask_apply(Geo g, const uint32_t* __restrict__ dot, const uint32_t* __restrict__ masks,
                             const uint64_t* __restrict__ rows, uint32_t cols, uint64_t npairs,
                             unsigned long long* __restrict__ acc64) {
  const uint64_t per = (uint64_t)g.P * g.n, total = npairs * per;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t pair = x / per;
    const uint32_t gp = (uint32_t)((x % per) / g.n), k = (uint32_t)(x % g.n);
    const PrimeInfo& pr = g.pr[gp];
    const uint64_t gidx = rows[pair / cols] * cols + pair % cols, c = gidx / g.n;
    if (gp == 0 && k == 0 && g.ops) {  // mask product + packed accumulation per pair
      atomicAdd(g.ops, 1ull);
      atomicAdd(g.ops + 2, 1ull);
    }
    const uint32_t m = masks[x];
    const uint32_t* base = dot + pair * g.ct_words;
    const uint32_t a = mul_barrett(base[(uint64_t)pr.poly0 * g.n + k], m, pr.q, pr.mu);
    const uint32_t b = mul_barrett(base[(uint64_t)pr.poly1 * g.n + k], m, pr.q, pr.mu);
    atomicAdd(&acc64[c * g.ct_words + (uint64_t)pr.poly0 * g.n + k], (unsigned long long)a);
    atomicAdd(&acc64[c * g.ct_words + (uint64_t)pr.poly1 * g.n + k], (unsigned long long)b);
  }
}

template <int LOGN>
__global__ void __launch_bounds__(Ntt<LOGN>::T, (LOGN <= 13 ? 2 : 1)) k_mask_acc_g(Geo g, const uint32_t* __restrict__ dot,
                                                               const uint64_t* __restrict__ rows, uint32_t cols,
                                                               uint32_t npairs, uint32_t G,
                                                               unsigned long long* __restrict__ acc64) {
  using NT = Ntt<LOGN>;
  constexpr uint32_t N = NT::N, T = NT::T;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  uint4* a0s = smem4 + N / 4;
  uint4* a1s = a0s + 4 * T;
  const uint32_t gp = blockIdx.x % g.P;
  const uint32_t p0 = (blockIdx.x / g.P) * G, p1 = min(npairs, p0 + G);
  if (gp == 0) count_ops(g, p1 - p0, 0, p1 - p0);  // mask product + packed accumulation per pair
  const PrimeInfo& pr = g.pr[gp];
  const BranchInfo& br = g.br[pr.b];
  const uint32_t q = pr.q, t = br.t, j = threadIdx.x, x0 = NT::posC0(j);
#pragma unroll
  for (int c = 0; c < 4; ++c) a0s[c * T + j] = a1s[c * T + j] = make_uint4(0, 0, 0, 0);
  uint64_t c_cur = ~0ull;
  auto flush = [&](uint64_t cc) {
    unsigned long long* d0 = acc64 + cc * g.ct_words + (uint64_t)pr.poly0 * N + x0;
    unsigned long long* d1 = acc64 + cc * g.ct_words + (uint64_t)pr.poly1 * N + x0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint4 A = a0s[c * T + j], B = a1s[c * T + j];
      atomicAdd(&d0[4 * c], (unsigned long long)A.x);
      atomicAdd(&d0[4 * c + 1], (unsigned long long)A.y);
      atomicAdd(&d0[4 * c + 2], (unsigned long long)A.z);
      atomicAdd(&d0[4 * c + 3], (unsigned long long)A.w);
      atomicAdd(&d1[4 * c], (unsigned long long)B.x);
      atomicAdd(&d1[4 * c + 1], (unsigned long long)B.y);
      atomicAdd(&d1[4 * c + 2], (unsigned long long)B.z);
      atomicAdd(&d1[4 * c + 3], (unsigned long long)B.w);
      a0s[c * T + j] = a1s[c * T + j] = make_uint4(0, 0, 0, 0);
    }
  };
  for (uint32_t pair = p0; pair < p1; ++pair) {
    const uint64_t gidx = rows[pair / cols] * cols + pair % cols;
    const uint32_t slot = (uint32_t)(gidx % N);
    const uint64_t c = gidx / N;
    if (c != c_cur) {
      if (c_cur != ~0ull) flush(c_cur);
      c_cur = c;
    }
    // m at pass-A coefficient positions x = j + T r
    const uint32_t pe = __brev(__ldg(&g.index_map[slot])) >> (32 - LOGN);
    const uint32_t w = pow_barrett(br.psi_inv, 2 * pe + 1, t, br.mu);
    const uint32_t wT = pow_barrett(w, T, t, br.mu);
    uint32_t m = mul_barrett(br.ninv.x, pow_barrett(w, j, t, br.mu), t, br.mu);
    uint32_t e[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      e[r] = m % q;
      m = mul_barrett(m, wT, t, br.mu);
    }
    NT::fwd(e, sm, g.fwd + (size_t)gp * N, g.twc + (size_t)gp * g.twc_stride, q);
    const uint32_t* base = dot + (uint64_t)pair * g.ct_words;
    const uint4* d0 = reinterpret_cast<const uint4*>(base + (uint64_t)pr.poly0 * N + x0);
    const uint4* d1 = reinterpret_cast<const uint4*>(base + (uint64_t)pr.poly1 * N + x0);
#pragma unroll
    for (int c4 = 0; c4 < 4; ++c4) {
      const uint4 u = d0[c4], v = d1[c4];
      uint4 A = a0s[c4 * T + j], B = a1s[c4 * T + j];
      A.x = add_mod(A.x, mul_barrett(u.x, e[4 * c4], q, pr.mu), q);
      A.y = add_mod(A.y, mul_barrett(u.y, e[4 * c4 + 1], q, pr.mu), q);
      A.z = add_mod(A.z, mul_barrett(u.z, e[4 * c4 + 2], q, pr.mu), q);
      A.w = add_mod(A.w, mul_barrett(u.w, e[4 * c4 + 3], q, pr.mu), q);
      B.x = add_mod(B.x, mul_barrett(v.x, e[4 * c4], q, pr.mu), q);
      B.y = add_mod(B.y, mul_barrett(v.y, e[4 * c4 + 1], q, pr.mu), q);
      B.z = add_mod(B.z, mul_barrett(v.z, e[4 * c4 + 2], q, pr.mu), q);
      B.w = add_mod(B.w, mul_barrett(v.w, e[4 * c4 + 3], q, pr.mu), q);
      a0s[c4 * T + j] = A;
      a1s[c4 * T + j] = B;
    }
  }
  if (c_cur != ~0ull) flush(c_cur);
}

// Mask plaintexts of every slot, once per context (MatmulStream::mask_for_slot,
// matmul.cpp:146-163: one-hot slot -> INTT_t -> lift -> NTT_q). The reference
// caches them only for N <= 4096 (host memory); with 180 GB of HBM the device
// keeps all N of them (N = 8192: 2.7 GB, N = 16384: 10.7 GB), so the
// per-pair mask step becomes a streaming multiply-accumulate.
// masks [slot][P][N] in eval order; block = (slot, prime).
template <int LOGN>
__global__ void __launch_bounds__(Ntt<LOGN>::T) k_mask_table(Geo g, uint32_t slot0, uint32_t* __restrict__ masks) {
  using NT = Ntt<LOGN>;
  constexpr uint32_t N = NT::N, T = NT::T;
  extern __shared__ uint4 smem4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  const uint32_t gp = blockIdx.x % g.P, slot = slot0 + blockIdx.x / g.P;
  const PrimeInfo& pr = g.pr[gp];
  const BranchInfo& br = g.br[pr.b];
  const uint32_t q = pr.q, t = br.t, j = threadIdx.x, x0 = NT::posC0(j);
  const uint32_t pe = __brev(__ldg(&g.index_map[slot])) >> (32 - LOGN);
  const uint32_t w = pow_barrett(br.psi_inv, 2 * pe + 1, t, br.mu);
  const uint32_t wT = pow_barrett(w, T, t, br.mu);
  uint32_t m = mul_barrett(br.ninv.x, pow_barrett(w, j, t, br.mu), t, br.mu);
  uint32_t e[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    e[r] = m % q;
    m = mul_barrett(m, wT, t, br.mu);
  }
  NT::fwd(e, sm, g.fwd + (size_t)gp * N, g.twc + (size_t)gp * g.twc_stride, q);
  uint4* o = reinterpret_cast<uint4*>(masks + ((uint64_t)slot * g.P + gp) * N + x0);
#pragma unroll
  for (int c = 0; c < 4; ++c) o[c] = make_uint4(e[4 * c], e[4 * c + 1], e[4 * c + 2], e[4 * c + 3]);
}

// Same accumulation as k_mask_acc_g with the masks read from the table:
// block = (group of G consecutive pairs, prime, 1024-slot slice), 256 threads
// x 4 slots, sums in registers, one u64 RED per slot and packed ciphertext.
__global__ void __launch_bounds__(256) k_mask_acc_c(Geo g, const uint32_t* __restrict__ dot,
                                                    const uint64_t* __restrict__ rows, uint32_t cols, uint32_t npairs,
                                                    uint32_t G, const uint32_t* __restrict__ masks,
                                                    unsigned long long* __restrict__ acc64) {
  const uint32_t N = g.n, slices = N / 1024;
  const uint32_t sl = blockIdx.x % slices, gp = (blockIdx.x / slices) % g.P;
  const uint32_t p0 = (blockIdx.x / (slices * g.P)) * G, p1 = min(npairs, p0 + G);
  if (gp == 0 && sl == 0) count_ops(g, p1 - p0, 0, p1 - p0);  // mask product + packed accumulation per pair
  const PrimeInfo& pr = g.pr[gp];
  const uint32_t q = pr.q, x0 = sl * 1024 + 4 * threadIdx.x;
  uint32_t A[4] = {0, 0, 0, 0}, B[4] = {0, 0, 0, 0};
  uint64_t c_cur = ~0ull;
  auto flush = [&](uint64_t cc) {
    unsigned long long* d0 = acc64 + cc * g.ct_words + (uint64_t)pr.poly0 * N + x0;
    unsigned long long* d1 = acc64 + cc * g.ct_words + (uint64_t)pr.poly1 * N + x0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      atomicAdd(&d0[r], (unsigned long long)A[r]);
      atomicAdd(&d1[r], (unsigned long long)B[r]);
      A[r] = B[r] = 0;
    }
  };
  for (uint32_t pair = p0; pair < p1; ++pair) {
    const uint64_t gidx = rows[pair / cols] * cols + pair % cols;
    const uint32_t slot = (uint32_t)(gidx % N);
    const uint64_t c = gidx / N;
    if (c != c_cur) {
      if (c_cur != ~0ull) flush(c_cur);
      c_cur = c;
    }
    const uint32_t* base = dot + (uint64_t)pair * g.ct_words;
    const uint4 m = __ldg(reinterpret_cast<const uint4*>(masks + ((uint64_t)slot * g.P + gp) * N + x0));
    const uint4 u = *reinterpret_cast<const uint4*>(base + (uint64_t)pr.poly0 * N + x0);
    const uint4 v = *reinterpret_cast<const uint4*>(base + (uint64_t)pr.poly1 * N + x0);
    A[0] = add_mod(A[0], mul_barrett(u.x, m.x, q, pr.mu), q);
    A[1] = add_mod(A[1], mul_barrett(u.y, m.y, q, pr.mu), q);
    A[2] = add_mod(A[2], mul_barrett(u.z, m.z, q, pr.mu), q);
    A[3] = add_mod(A[3], mul_barrett(u.w, m.w, q, pr.mu), q);
    B[0] = add_mod(B[0], mul_barrett(v.x, m.x, q, pr.mu), q);
    B[1] = add_mod(B[1], mul_barrett(v.y, m.y, q, pr.mu), q);
    B[2] = add_mod(B[2], mul_barrett(v.z, m.z, q, pr.mu), q);
    B[3] = add_mod(B[3], mul_barrett(v.w, m.w, q, pr.mu), q);
  }
  if (c_cur != ~0ull) flush(c_cur);
}
