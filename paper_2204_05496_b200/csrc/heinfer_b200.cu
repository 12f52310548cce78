// heinfer_b200: B200-native (sm_100a) encrypted-LR matmul hot path.
//
// Implements the C ABI of include/heinfer_b200.h. The reference path being
// replaced is hei::matmul::MatmulStream / matmul / baseline_matmul
// (/root/reference/proj/src/matmul/matmul.cpp:114-358) and everything it calls
// on the server side: TwinBackend (fpcrt/twin.cpp:169-219), HeBackend
// sum_all_slots (bfv/backend.cpp:63-73), BfvContext::mul_plain_inplace /
// add_plain_inplace / apply_galois (bfv/context.cpp:393-507) and the kernels
// table (kernels/modops_scalar.cpp, modops_avx2.cpp).
//
// Device layout: every residue is u32 (all q_i, t_b < 2^31). A twin
// ciphertext is [branch][part][prime][N] exactly as the host layout, so the
// flat "poly index" of (branch b, part p, prime i) is
//   (b ? 2*L0 : 0) + p*L_b + i
// and the flat prime index gp = (b ? L0 : 0) + i.
//
// Pipeline per batch of (row, class) pairs:
//   k_chunk_dot     dot = sum_k chunk_k (.) W[j][k]                 (HBM)
//   13/14 x { k_rot_digits     digit_l = INTT_l(sigma(c1)_l)
//             k_rot_keyswitch  acc_i = sum_l NTT_i(digit_l mod q_i) (.) K[l][i],
//                              dot <- dot + (acc0 + sigma(c0), acc1) }
//   k_mask_acc      packed[g/N] += mask_{g mod N} (.) dot           (u64 RED)
// and once per call k_bias_plain (side stream) + k_finish_add (mod-q reduce + bias add_plain).
//
// Source layout (one translation unit; the .cuh files are included inside
// the kernel namespace below):
//   modmath.cuh        Shoup / Barrett arithmetic, shared-memory NTTs (small N)
//   ntt_fast.cuh       register-blocked NTT (N = 8192, 16384)
//   bulk_copy.cuh      1-D TMA bulk copies (cp.async.bulk + mbarrier)
//   wire.cuh           HECT ciphertext parse / emit kernels
//   fold_kernels.cuh   fast algorithm: chunk products, digits, key switch,
//                      mask + pack, bias / finish, weight and key preparation
//   baseline.cuh       mt19937_64 replay (sequential and jump-ahead), noise
//   stdalg_kernels.cuh standard algorithm + client encryption kernels
//   decrypt.cuh        client decryption (exact CRT) and unpacking
//   keygen.cuh         key generation with exact rejection-sampling replay
//   heinfer_b200.cu    device structs, host orchestration, the C ABI
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <type_traits>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/heinfer_b200.h"
#include "modmath.cuh"
#include "ntt_fast.cuh"
#include "bulk_copy.cuh"
#include "baseline.cuh"

using namespace heb;

namespace {

// ---------------------------------------------------------------- errors
thread_local std::string g_err;
thread_local uint64_t g_launches = 0;

struct HeiError {
  int code;
  std::string msg;
};
[[noreturn]] void raise(int code, const std::string& msg) { throw HeiError{code, msg}; }

#define CU(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess)                                                           \
      raise(HEI_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e_));       \
  } while (0)
#define LAUNCHED()                    \
  do {                                \
    ++g_launches;                     \
    CU(cudaGetLastError());           \
  } while (0)

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return HEI_OK;
  } catch (const HeiError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return HEI_INTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HEI_INTERNAL;
  }
}

// ------------------------------------------------ host modular helpers (setup)
typedef unsigned __int128 u128;
uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)((u128)a * b % q); }
uint64_t powmod(uint64_t b, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  b %= q;
  while (e) {
    if (e & 1) r = mulmod(r, b, q);
    b = mulmod(b, b, q);
    e >>= 1;
  }
  return r;
}
uint64_t invmod(uint64_t a, uint64_t q) {
  int64_t t = 0, nt = 1, r = (int64_t)q, nr = (int64_t)(a % q);
  while (nr) {
    int64_t k = r / nr, x = t - k * nt;
    t = nt;
    nt = x;
    x = r - k * nr;
    r = nr;
    nr = x;
  }
  if (r != 1) raise(HEI_PARAM_ERROR, "inv_mod: value not invertible");
  return (uint64_t)(t < 0 ? t + (int64_t)q : t);
}
// Deterministic Miller-Rabin (ring/modulus.cpp:24-53).
bool is_prime(uint64_t v) {
  static const uint64_t W[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (v < 2) return false;
  for (uint64_t p : W) {
    if (v == p) return true;
    if (v % p == 0) return false;
  }
  uint64_t d = v - 1;
  int r = 0;
  while (!(d & 1)) d >>= 1, ++r;
  for (uint64_t a : W) {
    uint64_t x = powmod(a, d, v);
    if (x == 1 || x == v - 1) continue;
    bool wit = true;
    for (int i = 1; i < r; ++i) {
      x = mulmod(x, x, v);
      if (x == v - 1) {
        wit = false;
        break;
      }
    }
    if (wit) return false;
  }
  return true;
}
// Smallest-witness primitive 2n-th root (ring/modulus.cpp:73-85).
uint64_t root_2n(uint32_t n, uint64_t q) {
  const uint64_t e = (q - 1) / (2ull * n);
  for (uint64_t c = 2; c < q; ++c) {
    uint64_t w = powmod(c, e, q);
    if (powmod(w, n, q) == q - 1) return w;
  }
  raise(HEI_PARAM_ERROR, "no primitive root found");
}
uint32_t rev_bits(uint32_t v, uint32_t bits) {
  uint32_t r = 0;
  for (uint32_t i = 0; i < bits; ++i) r = (r << 1) | ((v >> i) & 1u);
  return r;
}
uint32_t shoup32(uint64_t w, uint64_t q) { return (uint32_t)((w << 32) / q); }
int max_q_bits_128(uint32_t n) {
  switch (n) {
    case 1024: return 27;
    case 2048: return 54;
    case 4096: return 109;
    case 8192: return 218;
    case 16384: return 438;
    case 32768: return 881;
    default: return 0;
  }
}

// ------------------------------------------------------------ device structs
constexpr int kMaxPrimes = 16;
constexpr int kMaxElts = 16;
constexpr uint32_t kMaxFoldParts = 8;

struct PrimeInfo {
  uint32_t q;
  uint32_t b, i;           // branch, index within branch
  uint32_t poly0, poly1;   // poly index of part 0 / part 1 inside a twin ct
  uint32_t first;          // flat index of prime 0 of this branch
  uint32_t L;              // primes in this branch
  uint32_t fast_reduce;    // digits of this branch reduce mod q with one csub
  uint2 ninv, last;        // inverse-NTT scaling constants
  uint2 delta;             // floor(Q/t) mod q (context.cpp:39-46)
  uint64_t mu;             // floor(2^64 / q) for Barrett
};
struct BranchInfo {
  uint32_t t;
  uint32_t L, first;
  uint2 ninv, last;  // mod-t inverse NTT constants
  uint32_t psi_inv;  // psi_t^-1 (inverse of the 2n-th root of the mod-t tables)
  uint64_t mu;       // floor(2^64 / t)
};
struct Geo {
  uint32_t n, logn, P, ct_words, pt_words;
  uint32_t L[2];
  PrimeInfo pr[kMaxPrimes];
  BranchInfo br[2];
  const uint2* fwd;  // [P + 2][n]: q primes then t0, t1
  const uint2* inv;
  const uint4* twc;  // pass-C twiddles, fast path only: [P + 2][KC][T]
  const uint4* itwc;
  uint32_t twc_stride;  // KC * T (uint4 per modulus)
  const uint32_t* index_map;
  // N = 16384 half-ring key switch (ks_half.cuh): per (prime, half) natural
  // and pass-C tables of the half's N/2-point transform
  const uint2* fwdh;    // [P][2][N/2]
  const uint4* twch;    // [P][2][twch_stride]
  uint32_t twch_stride;
  const uint2* invh;    // inverse counterparts (k_rot_digits_h)
  const uint4* itwch;
  // measured operation counters (HeBackend counters, backend.cpp:75-85):
  // [mul_plain, rotation, add], cumulative over the context; the kernels
  // that perform the ops add them (branch 0 speaks for the pair, as
  // TwinBackend::counters does), and each matmul reports the delta
  unsigned long long* ops;
};
// thread 0 of a counting block
__device__ __forceinline__ void count_ops(const Geo& g, uint64_t mul_plain, uint64_t rotation, uint64_t add) {
  if (threadIdx.x != 0 || !g.ops) return;
  if (mul_plain) atomicAdd(g.ops, (unsigned long long)mul_plain);
  if (rotation) atomicAdd(g.ops + 1, (unsigned long long)rotation);
  if (add) atomicAdd(g.ops + 2, (unsigned long long)add);
}
// (pair, prime) of this block, for grids of pairs * P blocks (pair-major)
__device__ __forceinline__ void block_pair_prime(const Geo& g, uint32_t& pair, uint32_t& gp) {
  pair = blockIdx.x / g.P;
  gp = blockIdx.x % g.P;
}

// Pass-A/B twiddles (indices 0..255) of every q prime, passed by value in the
// kernel parameter space (CUDA >= 12.1 allows 32 KB of parameters).
constexpr int kMaxAB = 12;
struct TwAB {
  uint2 w[kMaxAB][256];
};
struct TwNone {  // small launches: twiddles stay in global memory (tiny params)
  int unused;
};
template <bool PTW>
using TwArg = typename std::conditional<PTW, TwAB, TwNone>::type;

// ----------------------------------------------------------------- kernels
__global__ void k_narrow(Geo g, const uint64_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t cts,
                         uint32_t* err) {
  const uint64_t total = cts * g.ct_words;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t poly = (uint32_t)((x % g.ct_words) / g.n);
    // poly -> prime: branch 0 polys [0, 2L0), branch 1 after
    const uint32_t L0 = g.L[0];
    uint32_t gp = poly < 2 * L0 ? (poly % L0) : L0 + (poly - 2 * L0) % g.L[1];
    const uint64_t v = in[x];
    if (v >= g.pr[gp].q) *err = 1;
    out[x] = (uint32_t)v;
  }
}

// Row ids; optionally (snap != nullptr) also the op counters' start snapshot
// of the call (the first kernel of a one-shot matmul).
__global__ void k_iota(uint64_t* __restrict__ out, uint64_t start, uint64_t n,
                       const unsigned long long* ops = nullptr, unsigned long long* snap = nullptr) {
  if (snap && blockIdx.x == 0 && threadIdx.x < 3) snap[threadIdx.x] = __ldcg(ops + threadIdx.x);
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x)
    out[x] = start + x;
}

__global__ void k_widen(const uint32_t* __restrict__ in, uint64_t* __restrict__ out, uint64_t total) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x)
    out[x] = in[x];
}

__device__ __forceinline__ uint32_t poly_prime(const Geo& g, uint32_t poly) {
  const uint32_t L0 = g.L[0];
  return poly < 2 * L0 ? (poly % L0) : L0 + (poly - 2 * L0) % g.L[1];
}

#include "wire.cuh"

#include "fold_kernels.cuh"
#include "tmem_ks.cuh"
#include "ks_half.cuh"

#include "stdalg_kernels.cuh"

// Butterfly-throughput microbenchmark: the roofline denominator for the
// integer-bound transforms. Each thread runs 8 independent
// Cooley-Tukey butterfly chains (mul_shoup + add_mod + sub_mod) on registers.
__global__ void __launch_bounds__(256) k_bfly_peak(uint32_t* __restrict__ sink, uint32_t iters, uint32_t q,
                                                   uint32_t w, uint32_t ws) {
  uint32_t u[8], v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    u[k] = (threadIdx.x * 7919u + k * 104729u) % q;
    v[k] = (blockIdx.x * 31337u + k * 65537u) % q;
  }
  for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t t = mul_shoup(v[k], w, ws, q);
      v[k] = sub_mod(u[k], t, q);
      u[k] = add_mod(u[k], t, q);
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc ^= u[k] ^ v[k];
  if (acc == 0xFFFFFFFFu) sink[blockIdx.x] = acc;
}

#include "decrypt.cuh"
#include "keygen.cuh"

}  // namespace

// ================================================================ host side
struct hei_gpu_ctx {
  int device = 0;
  uint32_t n = 0, logn = 0;
  uint64_t t[2] = {0, 0};
  uint32_t L[2] = {0, 0};
  std::vector<uint64_t> q;
  uint32_t s_x = 6, s_w = 14, in_bits = 8;
  Geo geo{};
  uint2 *d_fwd = nullptr, *d_inv = nullptr;
  std::vector<uint2> h_fwd, h_inv;  // host copies (pass-A/B rows go in kernel params)
  uint4 *d_twc = nullptr, *d_itwc = nullptr;
  uint2* d_fwdh = nullptr;  // N = 16384 half-ring tables (ks_half.cuh)
  uint4* d_twch = nullptr;
  std::vector<uint2> h_fwdh;
  uint2* d_invh = nullptr;
  uint4* d_itwch = nullptr;
  std::vector<uint2> h_invh;
  uint32_t* d_index = nullptr;
  // galois elements in fold order: steps 1, 2, ..., n/4, then the swap
  std::vector<uint64_t> fold_elts;
  std::map<uint64_t, uint32_t> perm_index;  // elt -> row of d_perms
  uint32_t* d_perms = nullptr;
  uint2* d_keys[2] = {nullptr, nullptr};
  std::map<uint64_t, uint32_t> key_index[2];  // elt -> e
  bool has_keys[2] = {false, false};
  uint64_t* d_pk[2] = {nullptr, nullptr};
  uint2* d_pkp = nullptr;  // prepared public key [gp][part] (baseline)
  uint32_t* d_sk_hat = nullptr;  // NTT(lift(s)) per prime [P][n] (client decryption)
  bool has_sk[2] = {false, false};
  CrtInfo crt{};                 // exact CRT constants per branch (decrypt_core)
  uint32_t t0inv = 0;            // t0^-1 mod t1 (crt_recombine)
  uint32_t* d_err = nullptr;
  unsigned long long* d_ops = nullptr;      // [3] measured op counters (Geo::ops), cumulative
  unsigned long long* d_opsnap = nullptr;   // [3] one-shot calls: counters at the call's start (k_iota)
  unsigned long long* h_opsnap = nullptr;   // [6] mapped pinned: a call's start and end counters (k_finish_add)
  cudaStream_t stream = nullptr;
  uint64_t batch_pairs = 0;
  uint64_t keys_words[2] = {0, 0};
  // scratch (grown on demand)
  uint32_t *d_dotA = nullptr, *d_dotB = nullptr, *d_dig = nullptr, *d_dig2 = nullptr;
  bool fuse_digits = true;  // HEI_FUSE_DIGITS=0: separate digit kernel every rotation (small batches)
  uint64_t scratch_pairs = 0;
  std::mutex mu;
  // grow-only device pools for the per-call buffers of the device-resident
  // path (every C-ABI call synchronizes before returning, so reuse is safe)
  unsigned long long* pool_acc = nullptr;
  size_t pool_acc_bytes = 0;
  uint64_t* pool_rows = nullptr;
  size_t pool_rows_bytes = 0;
  int64_t* pool_bias = nullptr;
  size_t pool_bias_bytes = 0;
  uint64_t* pool_stage64 = nullptr;
  size_t pool_stage64_bytes = 0;
  uint32_t* pool_in32 = nullptr;
  size_t pool_in32_bytes = 0;
  uint32_t* pool_out = nullptr;
  size_t pool_out_bytes = 0;
  uint64_t* pool_out64 = nullptr;
  size_t pool_out64_bytes = 0;
  cudaStream_t copy_stream = nullptr;
  int64_t* pinned_bias = nullptr;  // pinned staging for the bias upload
  size_t pinned_bias_bytes = 0;
  void* pinned_out = nullptr;  // pinned staging for result downloads to pageable memory
  size_t pinned_out_bytes = 0;
  bool graphs = true;   // HEI_NO_GRAPHS=1: launch the small-batch fold eagerly
  bool two_streams = true;  // HEI_TWO_STREAMS=0: fold the batch on one stream only
  bool mt_jump = true;      // HEI_MT_JUMP=0: sequential mt19937_64 replay only
  cudaStream_t side_stream = nullptr;
  std::vector<cudaStream_t> part_streams;  // fold slices 1.. of a batch
  uint32_t fold_parts = 2;                 // HEI_FOLD_PARTS: concurrent fold slices per batch
  uint32_t mask_group = 8;                 // HEI_MASK_GROUP: max pairs per mask/pack block
  cudaStream_t bias_stream = nullptr;  // bias plaintext encoding, overlapped with the fold
  uint32_t* pool_biasp = nullptr;
  size_t pool_biasp_bytes = 0;
  void* named_pool[24] = {};       // grow-only scratch for the client-role calls (baseline, encryption)
  size_t named_pool_bytes[24] = {};
  uint32_t* pool_masks = nullptr;  // latency path: precomputed mask plaintexts
  size_t pool_masks_bytes = 0;
  bool premask = true;  // HEI_PREMASK=0: compute masks inside the accumulation kernel
  bool pdl = true;      // HEI_PDL=0: latency key switches launch without programmatic dependence
  bool ks_cluster = false;  // HEI_KS_CLUSTER=1: full batches fuse the digit INTT into a cluster key switch
  uint32_t e2e_div = 4;  // HEI_E2E_DIV: host-buffer matmul copies rows in ~rows/div chunks
  bool dot_rows = true;    // HEI_DOT_ROWS=0: per-pair chunk-product kernel for every batch
  bool mask_cache = true;  // HEI_MASK_CACHE=0: regenerate each pair's mask (the reference's N > 4096 behaviour)
  uint32_t* d_mask_table = nullptr;  // [slot][P][N] mask plaintexts, built on first full-batch use
  bool e2e_overlap = true;  // HEI_E2E_OVERLAP=0: host-buffer chunks run one after another
  std::vector<cudaStream_t> chunk_streams;  // 2 x fold_parts streams: consecutive chunks overlap
  uint64_t mt_chunks_max = 128;   // HEI_MT_CHUNKS: parallel mt19937_64 generators per branch
  struct FoldGraph {
    uint64_t pairs;
    uint32_t *cur, *other, *dig;
    uint64_t gen;
    cudaGraphExec_t exec;
    uint64_t launches;
  };
  std::vector<FoldGraph> fold_graphs;
  uint64_t graph_gen = 0;  // bumped when keys or scratch buffers change
  // optional per-kernel timing (bench.py roofline): events around the fold
  bool timing = false;
  std::vector<std::array<cudaEvent_t, 3>> fold_ev;  // digits: [0,1], key switch: [1,2]

  size_t ct_words() const { return 2ull * (L[0] + L[1]) * n; }
  size_t pt_words() const { return (size_t)(L[0] + L[1]) * n; }
  uint32_t P() const { return L[0] + L[1]; }
  uint32_t threads() const { return std::min<uint32_t>(512, std::max<uint32_t>(32, n / 2)); }
};

struct hei_gpu_weights {
  hei_gpu_ctx* ctx;
  uint64_t f = 0, cols = 0, kc = 0;
  uint2* d_w = nullptr;  // [cols][k][twin plain] (val, shoup)
};

struct hei_gpu_stream {
  hei_gpu_ctx* ctx;
  const hei_gpu_weights* w;
  std::vector<int64_t> bias;
  uint64_t rows = 0, pushed = 0, C = 0;
  std::vector<bool> seen;
  bool finished = false;
  unsigned long long* d_acc = nullptr;  // [C][twin ct] u64
  bool owns_acc = true, owns_rows = true;
  int64_t* d_bias = nullptr;  // staged bias (pool memory, not owned)
  uint32_t* d_biasp = nullptr;      // bias plaintext [C][P][N] (pool memory)
  cudaEvent_t bias_ev = nullptr;    // recorded when d_biasp was produced on the side stream
  // pending rows staged on the device
  std::vector<uint64_t> pend_idx;
  uint32_t* d_stage = nullptr;  // [cap][k][twin ct] u32
  uint64_t* d_stage64 = nullptr;
  uint64_t* d_rows = nullptr;
  uint64_t cap_rows = 0;
  unsigned long long* d_ops0 = nullptr;  // [3] op counters at the stream's start
  bool owns_ops0 = true;
};

// util::Prng (rng.hpp:19-68): mt19937_64 state kept explicitly so the
// device generator (k_mt_generate) can continue the exact stream.
struct hei_gpu_prng {
  uint64_t mt[312];
  uint32_t mti = 312;
  double spare = 0.0;
  bool have_spare = false;
};

namespace {

void set_device(hei_gpu_ctx* c) {
  if (!c) raise(HEI_PARAM_ERROR, "null context");
  CU(cudaSetDevice(c->device));
}

void check_err_flag(hei_gpu_ctx* c, int code, const char* what) {
  uint32_t h = 0;
  CU(cudaMemcpyAsync(&h, c->d_err, 4, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (h) {
    CU(cudaMemsetAsync(c->d_err, 0, 4, c->stream));
    raise(code, what);
  }
}

unsigned grid_for(uint64_t total, unsigned threads) {
  uint64_t b = (total + threads - 1) / threads;
  return (unsigned)std::min<uint64_t>(b, 148ull * 32);
}

template <typename T>
T* pool_get(T*& p, size_t& cap, size_t bytes) {
  if (bytes > cap) {
    if (p) CU(cudaFree(p));
    p = nullptr;
    CU(cudaMalloc(&p, bytes));
    cap = bytes;
  }
  return p;
}

// Grow-only scratch slot `id` of the context (reused across calls; every
// C-ABI call synchronises before returning).
enum ScratchId {
  kScrRawAll = 0, kScrRaw, kScrNoise, kScrM, kScrCt, kScrWc, kScrAcc, kScrOut, kScrOut64, kScrX,
  kScrMtPoly, kScrMtWseq, kScrMtPart, kScrW, kScrBias, kScrState, kScrStarts
};
template <typename T>
T* scratch(hei_gpu_ctx* c, int id, size_t bytes) {
  static_assert(kScrStarts < 24, "named scratch pool too small");
  void*& p = c->named_pool[id];
  if (bytes > c->named_pool_bytes[id]) {
    if (p) CU(cudaFree(p));
    p = nullptr;
    CU(cudaMalloc(&p, bytes));
    c->named_pool_bytes[id] = bytes;
  }
  return reinterpret_cast<T*>(p);
}

void ensure_scratch(hei_gpu_ctx* c, uint64_t pairs) {
  if (pairs <= c->scratch_pairs) return;
  if (c->d_dotA) cudaFree(c->d_dotA);
  if (c->d_dotB) cudaFree(c->d_dotB);
  if (c->d_dig) cudaFree(c->d_dig);
  if (c->d_dig2) cudaFree(c->d_dig2);
  c->d_dotA = c->d_dotB = c->d_dig = c->d_dig2 = nullptr;
  CU(cudaMalloc(&c->d_dotA, pairs * c->ct_words() * 4));
  CU(cudaMalloc(&c->d_dotB, pairs * c->ct_words() * 4));
  CU(cudaMalloc(&c->d_dig, pairs * c->pt_words() * 4));
  CU(cudaMalloc(&c->d_dig2, pairs * c->pt_words() * 4));
  c->scratch_pairs = pairs;
  ++c->graph_gen;
}

size_t smem_bytes(hei_gpu_ctx* c, int words) { return (size_t)words * c->n * 4; }

void set_smem_attr(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

// ---- launch dispatch: register-blocked kernels for the production rings
// ---- N in {8192, 16384}; generic shared-memory kernels otherwise (the small
// ---- rings of the reference's own tests).
#define HEI_DISPATCH(LOGN_VAR, FAST, GENERIC)         \
  switch (LOGN_VAR) {                                 \
    case 13: { constexpr int LG = 13; FAST; } break;  \
    case 14: { constexpr int LG = 14; FAST; } break;  \
    default: { GENERIC; } break;                      \
  }

// Host copy of the pass-A/B twiddle rows for the primes of `g` (its pr[]
// order; a branch-restricted Geo from apply_galois is handled by matching q).
const TwAB* tabs_of(hei_gpu_ctx* c, const Geo& g, int inverse) {
  thread_local TwAB t;
  for (uint32_t k = 0; k < g.P && k < (uint32_t)kMaxAB; ++k) {
    uint32_t src = 0;
    for (uint32_t m = 0; m < c->geo.P; ++m)
      if (c->geo.pr[m].q == g.pr[k].q) src = m;
    std::memcpy(t.w[k], (inverse ? c->h_inv : c->h_fwd).data() + (size_t)src * c->n, 256 * sizeof(uint2));
  }
  return &t;
}

// Rows [k][h] (k < np) of the N = 16384 half-ring forward tables for primes
// gp0.. of `g`.
const TwAB* tabs_half_pairs(hei_gpu_ctx* c, const Geo& g, uint32_t gp0, uint32_t np) {
  thread_local TwAB t;
  if (2 * np > (uint32_t)kMaxAB) raise(HEI_INTERNAL, "half-ring parameter rows exceed the table");
  for (uint32_t k = 0; k < np; ++k) {
    uint32_t src = 0;
    for (uint32_t m = 0; m < c->geo.P; ++m)
      if (c->geo.pr[m].q == g.pr[gp0 + k].q) src = m;
    for (uint32_t h = 0; h < 2; ++h)
      std::memcpy(t.w[2 * k + h], c->h_fwdh.data() + ((size_t)src * 2 + h) * (c->n / 2), 256 * sizeof(uint2));
  }
  return &t;
}

// Public-key encryption of E features/rows (E * P blocks); large launches run
// the register kernel at 3 CTAs/SM (N = 8192) with parameter-space twiddles.
void launch_bl_encrypt(hei_gpu_ctx* c, const Geo& g, unsigned blocks, const int8_t* d_noise, const uint32_t* d_m,
                       uint32_t* ct, size_t sm1, cudaStream_t st) {
  HEI_DISPATCH(c->logn,
               (k_bl_encrypt<LG, true, (LG <= 13 ? 3 : 1)><<<blocks, Ntt<LG>::T, sm1, st>>>(g, d_noise, d_m, c->d_pkp,
                                                                                           ct, *tabs_of(c, g, 0))),
               (k_bl_encrypt_g<<<blocks, c->threads(), sm1, st>>>(g, d_noise, d_m, c->d_pkp, ct)));
}

// digit_l = INTT_l(sigma(c1)_l) for every (pair, prime) block.
void launch_rot_digits(hei_gpu_ctx* c, const Geo& g, unsigned blocks, const uint32_t* cur, const uint32_t* perm,
                       uint32_t* dig, cudaStream_t st) {
  const size_t sm = smem_bytes(c, 1);
  // the pass-A/B twiddles travel as kernel parameters (constant bank)
  if (c->logn == 14 && blocks >= 2u * 148u) {
    // N = 16384: 2-CTA clusters, one CTA per half of the eval slots (ks_half.cuh)
    k_rot_digits_h<<<2 * blocks, 512, 8192 * 4, st>>>(g, cur, perm, dig);
    LAUNCHED();
    return;
  }
  HEI_DISPATCH(c->logn, (k_rot_digits_f<LG, true><<<blocks, Ntt<LG>::T, sm, st>>>(g, cur, perm, dig, *tabs_of(c, g, 1))),
               (k_rot_digits<<<blocks, c->threads(), sm, st>>>(g, cur, perm, dig)));
  LAUNCHED();
}

// Key switch + fold add of one rotation (apply_galois, context.cpp:428-507;
// backend.cpp:63-73). Returns true when the launched kernel also produced the
// next rotation's digits (dig_next != nullptr; small batches only).
//   N = 8192:  <= 148 blocks    k_rot_keyswitch_w2 (2-group CTA, latency)
//              >= 296, unfused  k_rot_keyswitch_t  (TMEM accumulators, 3 CTAs/SM)
//              otherwise        k_rot_keyswitch_s  (shared-memory accumulators)
//   N = 16384: >= 296, unfused  k_rot_keyswitch_h  (half-ring blocks, TMEM)
//              otherwise        k_rot_keyswitch_s
//   other N:   k_rot_keyswitch (generic)
bool launch_rot_keyswitch(hei_gpu_ctx* c, const Geo& g, unsigned blocks, const uint32_t* cur, const uint32_t* dig,
                          const uint32_t* perm, const uint2* k0, const uint2* k1, uint32_t* out, int fold,
                          cudaStream_t st, const uint32_t* perm_next = nullptr, uint32_t* dig_next = nullptr,
                          const uint2* kn0 = nullptr, const uint2* kn1 = nullptr) {
  const bool big = blocks >= 2u * 148u;
  bool next = dig_next != nullptr;
  const size_t sm = smem_bytes(c, 1);
  switch (c->logn) {
    case 13:
      if (blocks <= 148u) {
        // programmatic dependent launch (the kernel waits on its predecessor
        // with griddepcontrol.wait): the launch overlaps the previous tail
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(blocks);
        cfg.blockDim = dim3(2 * Ntt<13>::T);
        cfg.dynamicSmemBytes = 6 * sm;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = c->pdl ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (next)
          CU(cudaLaunchKernelEx(&cfg, k_rot_keyswitch_w2<13, true>, g, cur, dig, perm, k0, k1, out, fold, perm_next,
                                dig_next, kn0, kn1));
        else
          CU(cudaLaunchKernelEx(&cfg, k_rot_keyswitch_w2<13, false>, g, cur, dig, perm, k0, k1, out, fold,
                                (const uint32_t*)nullptr, (uint32_t*)nullptr, kn0, kn1));
      } else if (big && !next) {
        k_rot_keyswitch_t<<<blocks, Ntt<13>::T, sm, st>>>(g, cur, dig, perm, k0, k1, out, fold, *tabs_of(c, g, 0));
      } else if (next) {
        k_rot_keyswitch_s<13, true, true><<<blocks, Ntt<13>::T, 3 * sm, st>>>(g, cur, dig, perm, k0, k1, out, fold,
                                                                              perm_next, dig_next, *tabs_of(c, g, 0));
      } else {
        k_rot_keyswitch_s<13, true, false><<<blocks, Ntt<13>::T, 3 * sm, st>>>(g, cur, dig, perm, k0, k1, out, fold,
                                                                               nullptr, nullptr, *tabs_of(c, g, 0));
      }
      break;
    case 14:
      if (big && !next) {
        // one launch per branch, the two halves of a (pair, prime) adjacent
        const uint32_t pairs = blocks / g.P;
        for (uint32_t b = 0, gp0 = 0; b < 2; gp0 += g.L[b], ++b) {
          k_rot_keyswitch_h<<<pairs * g.L[b] * 2, 512, 8192 * 4, st>>>(g, cur, dig, perm, k0, k1, out, fold, gp0,
                                                                       g.L[b], *tabs_half_pairs(c, g, gp0, g.L[b]));
          if (b == 0) LAUNCHED();
        }
      } else if (next) {
        k_rot_keyswitch_s<14, true, true><<<blocks, Ntt<14>::T, 3 * sm, st>>>(g, cur, dig, perm, k0, k1, out, fold,
                                                                              perm_next, dig_next, *tabs_of(c, g, 0));
      } else {
        k_rot_keyswitch_s<14, true, false><<<blocks, Ntt<14>::T, 3 * sm, st>>>(g, cur, dig, perm, k0, k1, out, fold,
                                                                               nullptr, nullptr, *tabs_of(c, g, 0));
      }
      break;
    default:
      k_rot_keyswitch<<<blocks, c->threads(), smem_bytes(c, 3), st>>>(g, cur, dig, perm, k0, k1, out, fold);
      next = false;
  }
  LAUNCHED();
  return next;
}
// All N mask plaintexts of the context, built once on first use (blocking,
// on the context stream) and kept for its lifetime.
const uint32_t* mask_table(hei_gpu_ctx* c) {
  if (c->d_mask_table) return c->d_mask_table;
  const Geo& g = c->geo;
  CU(cudaMalloc(&c->d_mask_table, (size_t)c->n * g.P * c->n * 4));
  const uint32_t per = 512;  // slots per launch
  for (uint32_t s0 = 0; s0 < c->n; s0 += per) {
    const unsigned blocks = std::min(per, c->n - s0) * g.P;
    HEI_DISPATCH(c->logn,
                 (k_mask_table<LG><<<blocks, Ntt<LG>::T, smem_bytes(c, 1), c->stream>>>(g, s0, c->d_mask_table)),
                 raise(HEI_INTERNAL, "mask table: unsupported ring degree"));
    LAUNCHED();
  }
  CU(cudaStreamSynchronize(c->stream));
  return c->d_mask_table;
}

// dot[pair] = sum_k chunk_k (.) W[j][k] for `rows` rows (push_row,
// matmul.cpp:176-184): row-streaming kernel for the common chunk counts at
// N >= 4096, the per-pair kernel otherwise.
void launch_chunk_dot(hei_gpu_ctx* c, const uint32_t* in, const hei_gpu_weights* w, uint64_t rows, uint32_t* dot,
                      cudaStream_t st) {
  const Geo& g = c->geo;
  const uint32_t cols = (uint32_t)w->cols, kc = (uint32_t)w->kc;
  if (c->dot_rows && c->n >= 4096 && kc >= 1 && kc <= 5 && rows >= 8) {
    constexpr uint32_t CG = 4;
    const unsigned blocks = (unsigned)((c->n / 256) * 2 * c->P() * ((cols + CG - 1) / CG));
    switch (kc) {
      case 1: k_chunk_dot_rows<CG, 1><<<blocks, 256, 0, st>>>(g, in, w->d_w, cols, (uint32_t)rows, dot); break;
      case 2: k_chunk_dot_rows<CG, 2><<<blocks, 256, 0, st>>>(g, in, w->d_w, cols, (uint32_t)rows, dot); break;
      case 3: k_chunk_dot_rows<CG, 3><<<blocks, 256, 0, st>>>(g, in, w->d_w, cols, (uint32_t)rows, dot); break;
      case 4: k_chunk_dot_rows<CG, 4><<<blocks, 256, 0, st>>>(g, in, w->d_w, cols, (uint32_t)rows, dot); break;
      default: k_chunk_dot_rows<CG, 5><<<blocks, 256, 0, st>>>(g, in, w->d_w, cols, (uint32_t)rows, dot); break;
    }
  } else {
    k_chunk_dot<<<(unsigned)(rows * cols * 2 * c->P()), std::min<unsigned>(c->threads(), c->n / 4), 0, st>>>(
        g, in, w->d_w, cols, kc, dot);
  }
  LAUNCHED();
}

void launch_mask_acc(hei_gpu_ctx* c, const Geo& g, unsigned blocks, const uint32_t* res, const uint64_t* rows,
                     uint32_t cols, unsigned long long* acc, cudaStream_t st) {
  const size_t sm = smem_bytes(c, 1);
  const uint32_t npairs = blocks / g.P;
  // enough blocks for every SM at small batches, up to 8 pairs per block
  const uint32_t G = std::max<uint32_t>(1, std::min<uint32_t>(c->mask_group, npairs * g.P / (148 * 8)));
  const unsigned gblocks = (unsigned)(((npairs + G - 1) / G) * g.P);
  if (c->mask_cache && c->logn >= 13 && c->logn <= 14 && blocks >= 2u * 148u) {
    const uint32_t* masks = mask_table(c);
    const unsigned cb = (unsigned)(((npairs + G - 1) / G) * g.P * (c->n / 1024));
    k_mask_acc_c<<<cb, 256, 0, st>>>(g, res, rows, cols, npairs, G, masks, acc);
    LAUNCHED();
    return;
  }
  HEI_DISPATCH(c->logn, (k_mask_acc_g<LG><<<gblocks, Ntt<LG>::T, 3 * sm, st>>>(g, res, rows, cols, npairs, G, acc)),
               (k_mask_acc<<<blocks, c->threads(), sm, st>>>(g, res, rows, cols, acc)));
  LAUNCHED();
}
void launch_ct_ntt(hei_gpu_ctx* c, unsigned blocks, uint32_t* cts, cudaStream_t st) {
  const size_t sm = smem_bytes(c, 1);
  HEI_DISPATCH(c->logn, (k_ct_ntt_f<LG><<<blocks, Ntt<LG>::T, sm, st>>>(c->geo, cts)),
               (k_ct_ntt<<<blocks, c->threads(), sm, st>>>(c->geo, cts, 0)));
  LAUNCHED();
}
void launch_ct_intt(hei_gpu_ctx* c, unsigned blocks, uint32_t* cts, cudaStream_t st) {
  const size_t sm = smem_bytes(c, 1);
  HEI_DISPATCH(c->logn, (k_ct_intt_f<LG><<<blocks, Ntt<LG>::T, sm, st>>>(c->geo, cts)),
               (k_ct_ntt<<<blocks, c->threads(), sm, st>>>(c->geo, cts, 1)));
  LAUNCHED();
}
void launch_poly_ntt(hei_gpu_ctx* c, unsigned blocks, uint32_t gp, uint32_t* polys, int inverse, cudaStream_t st) {
  const size_t sm = smem_bytes(c, 1);
  HEI_DISPATCH(c->logn, (k_poly_ntt_f<LG><<<blocks, Ntt<LG>::T, sm, st>>>(c->geo, gp, polys, inverse)),
               (k_poly_ntt<<<blocks, c->threads(), sm, st>>>(c->geo, gp, polys, inverse)));
  LAUNCHED();
}
template <int LG>
void set_fast_attrs(size_t sm) {
  set_smem_attr((const void*)k_rot_digits_f<LG, true>, sm);
  set_smem_attr((const void*)k_rot_keyswitch_s<LG, true, false>, 3 * sm);
  set_smem_attr((const void*)k_rot_keyswitch_s<LG, true, true>, 3 * sm);
  if constexpr (LG == 13) {
    set_smem_attr((const void*)k_rot_keyswitch_t, sm);
    {
      // three CTAs of 33 KB fit the 100 KB shared-memory carve-out; the
      // driver's default picks 132 KB, which leaves L1 32 KB smaller
      int pct = 43;
      if (const char* v = std::getenv("HEI_KS_CARVE")) pct = std::atoi(v);
      if (pct >= 0)
        CU(cudaFuncSetAttribute((const void*)k_rot_keyswitch_t, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    }
    set_smem_attr((const void*)k_rot_keyswitch_c<6>, 2 * sm);
    set_smem_attr((const void*)k_rot_keyswitch_c<4>, 2 * sm);
    set_smem_attr((const void*)k_rot_keyswitch_w2<LG, true>, 6 * sm);
    set_smem_attr((const void*)k_rot_keyswitch_w2<LG, false>, 6 * sm);
  }
  set_smem_attr((const void*)k_mask_acc_g<LG>, 3 * sm);
  set_smem_attr((const void*)k_mask_prep<LG>, sm);
  set_smem_attr((const void*)k_mask_table<LG>, sm);
  set_smem_attr((const void*)k_ct_ntt_f<LG>, sm);
  set_smem_attr((const void*)k_ct_intt_f<LG>, sm);
  set_smem_attr((const void*)k_poly_ntt_f<LG>, sm);
  set_smem_attr((const void*)k_bl_encode<LG>, sm);
  set_smem_attr((const void*)k_bl_encrypt<LG, true, (LG <= 13 ? 3 : 1)>, sm);
  set_smem_attr((const void*)k_prepare_pk<LG>, sm);
}

uint64_t auto_batch_pairs(hei_gpu_ctx* c) {
  if (c->batch_pairs) return c->batch_pairs;
  // Enough (pair, prime) blocks for several waves on 148 SMs while keeping the
  // per-step working set (2 x dot + digits) modest.
  const uint64_t per_pair = (2 * c->ct_words() + c->pt_words()) * 4;
  uint64_t p = (uint64_t)16 << 30;  // 16 GiB of the 180 GB HBM
  p /= per_pair;
  return std::max<uint64_t>(1, std::min<uint64_t>(p, 8192));
}

// The rotate-and-sum fold over `pairs` twin ciphertexts in `cur` (eval form);
// returns the buffer holding the result.
uint32_t* fold_impl(hei_gpu_ctx* c, uint64_t pairs, uint32_t* cur, uint32_t* other, cudaStream_t st, uint32_t* dig,
                    uint32_t* dig2) {
  const Geo& g = c->geo;
  const unsigned blocks = (unsigned)(pairs * c->P());
  bool have_digits = false;  // digits of this rotation already produced by the previous key switch
  const size_t S = c->fold_elts.size();
  for (size_t k = 0; k < S; ++k) {
    const uint64_t elt = c->fold_elts[k];
    const uint32_t* perm = c->d_perms + (size_t)c->perm_index.at(elt) * c->n;
    // fused digits pay off when launches are too small to fill the GPU
    // (latency path); large batches keep the separate 3-CTA/SM digit kernel
    const bool fuse = c->fuse_digits && blocks < 4u * 148u;
    const uint32_t* perm_next =
        (k + 1 < S && fuse) ? c->d_perms + (size_t)c->perm_index.at(c->fold_elts[k + 1]) * c->n : nullptr;
    const uint2* k0 = c->d_keys[0] + (size_t)c->key_index[0].at(elt) * c->L[0] * 2 * c->L[0] * c->n;
    const uint2* k1 = c->d_keys[1] + (size_t)c->key_index[1].at(elt) * c->L[1] * 2 * c->L[1] * c->n;
    cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
    if (c->timing) {
      CU(cudaEventCreate(&e0));
      CU(cudaEventCreate(&e1));
      CU(cudaEventCreate(&e2));
      CU(cudaEventRecord(e0, st));
    }
    if (c->ks_cluster && c->logn == 13 && blocks >= 2u * 148u && !perm_next && g.L[0] == 6 && g.L[1] == 4) {
      // digit INTT fused into a cluster key switch per branch (digits stay on chip)
      if (c->timing) CU(cudaEventRecord(e1, st));
      const TwAB* tab = tabs_of(c, g, 0);
      const uint32_t pairs = blocks / g.P;
      k_rot_keyswitch_c<6><<<pairs * 6, Ntt<13>::T, smem_bytes(c, 2), st>>>(g, cur, perm, k0, other, 1, 0, *tab);
      LAUNCHED();
      k_rot_keyswitch_c<4><<<pairs * 4, Ntt<13>::T, smem_bytes(c, 2), st>>>(g, cur, perm, k1, other, 1, 6, *tab);
      LAUNCHED();
      if (c->timing) {
        CU(cudaEventRecord(e2, st));
        c->fold_ev.push_back({e0, e1, e2});
      }
      std::swap(cur, other);
      continue;
    }
    if (!have_digits) launch_rot_digits(c, g, blocks, cur, perm, dig, st);
    if (c->timing) CU(cudaEventRecord(e1, st));
    const uint2 *kn0 = nullptr, *kn1 = nullptr;  // the next rotation's keys (L2 prefetch on small batches)
    if (k + 1 < S) {
      const uint64_t en = c->fold_elts[k + 1];
      kn0 = c->d_keys[0] + (size_t)c->key_index[0].at(en) * c->L[0] * 2 * c->L[0] * c->n;
      kn1 = c->d_keys[1] + (size_t)c->key_index[1].at(en) * c->L[1] * 2 * c->L[1] * c->n;
    }
    have_digits = launch_rot_keyswitch(c, g, blocks, cur, dig, perm, k0, k1, other, 1, st, perm_next,
                                       perm_next ? dig2 : nullptr, kn0, kn1);
    if (have_digits) std::swap(dig, dig2);
    if (c->timing) {
      CU(cudaEventRecord(e2, st));
      c->fold_ev.push_back({e0, e1, e2});
    }
    std::swap(cur, other);
  }
  return cur;
}

// Small batches (the single-individual latency path) replay the 26-28 fold
// launches as one CUDA graph captured per (pairs, buffers), removing the
// per-launch gaps that dominate when every launch covers < 2 blocks per SM.
uint32_t* fold(hei_gpu_ctx* c, uint64_t pairs, uint32_t* cur, uint32_t* other, cudaStream_t st,
               uint32_t* dig = nullptr) {
  if (!dig) dig = c->d_dig;
  uint32_t* dig2 = c->d_dig2 + (dig - c->d_dig);  // second digit buffer of the same region
  const unsigned blocks = (unsigned)(pairs * c->P());
  const bool small = blocks < 2u * 148u;
  uint32_t* result = (c->fold_elts.size() % 2) ? other : cur;
  if (!small || c->timing || !c->graphs) return fold_impl(c, pairs, cur, other, st, dig, dig2);
  // drop graphs of an older key/scratch generation, and keep the cache
  // bounded (a long-running server sees many small batch sizes); an
  // executable graph still in flight is freed when it completes
  for (size_t i = 0; i < c->fold_graphs.size();) {
    if (c->fold_graphs[i].gen != c->graph_gen) {
      cudaGraphExecDestroy(c->fold_graphs[i].exec);
      c->fold_graphs.erase(c->fold_graphs.begin() + i);
    } else {
      ++i;
    }
  }
  constexpr size_t kMaxFoldGraphs = 32;
  if (c->fold_graphs.size() >= kMaxFoldGraphs) {
    cudaGraphExecDestroy(c->fold_graphs.front().exec);
    c->fold_graphs.erase(c->fold_graphs.begin());
  }
  for (auto& fg : c->fold_graphs)
    if (fg.pairs == pairs && fg.cur == cur && fg.other == other && fg.dig == dig && fg.gen == c->graph_gen) {
      CU(cudaGraphLaunch(fg.exec, st));
      g_launches += fg.launches;
      return result;
    }
  const uint64_t before = g_launches;
  cudaGraph_t graph = nullptr;
  CU(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  fold_impl(c, pairs, cur, other, st, dig, dig2);
  CU(cudaStreamEndCapture(st, &graph));
  cudaGraphExec_t exec = nullptr;
  CU(cudaGraphInstantiate(&exec, graph, 0));
  cudaGraphDestroy(graph);
  c->fold_graphs.push_back({pairs, cur, other, dig, c->graph_gen, exec, g_launches - before});
  g_launches = before;
  CU(cudaGraphLaunch(exec, st));
  g_launches += c->fold_graphs.back().launches;
  return result;
}

void require_keys(hei_gpu_ctx* c) {
  for (int b = 0; b < 2; ++b) {
    if (!c->has_keys[b]) raise(HEI_KEY_ERROR, "apply_galois: no galois keys uploaded for this branch");
    for (uint64_t e : c->fold_elts)
      if (!c->key_index[b].count(e))
        raise(HEI_KEY_ERROR, "apply_galois: no key for galois element " + std::to_string(e));
  }
}

// Fold + mask of `nrows` rows whose per-pair dot ciphertexts (u32, eval form)
// are already in c->d_dotA (feature-block sharding path).
void run_folded_dots(hei_gpu_stream* s, const uint64_t* d_rows, uint64_t nrows, cudaStream_t st) {
  hei_gpu_ctx* c = s->ctx;
  const uint32_t cols = (uint32_t)s->w->cols;
  const uint64_t pairs = nrows * cols;
  uint32_t* res = fold(c, pairs, c->d_dotA, c->d_dotB, st);
  launch_mask_acc(c, c->geo, (unsigned)(pairs * c->P()), res, d_rows, cols, s->d_acc, st);
}

// Slice placement for a chunk that runs concurrently with its neighbours
// (host-buffer matmul): the chunk's slices go to `streams` (not the caller's
// stream), use the scratch region starting at pair `pair_off`, and the chunk
// ends by recording `done` on streams[0] instead of joining the caller.
struct ChunkSlot {
  cudaStream_t streams[kMaxFoldParts];
  uint64_t pair_off;
  cudaEvent_t done;
};

// Core: process staged rows (device u32, eval form) into the packed u64 sums.
// Returns false when `cs` was given but the chunk is too small for slices (the
// caller then runs it serialised on `st`).
bool run_rows(hei_gpu_stream* s, const uint32_t* d_in, const uint64_t* d_rows, uint64_t nrows, cudaStream_t st,
              const ChunkSlot* cs = nullptr) {
  hei_gpu_ctx* c = s->ctx;
  const hei_gpu_weights* w = s->w;
  const Geo& g = c->geo;
  const uint32_t cols = (uint32_t)w->cols;
  const uint64_t pairs = nrows * cols;
  if (!cs) ensure_scratch(c, pairs);
  const unsigned T = c->threads();
  const unsigned blocksP = (unsigned)(pairs * c->P());
  const uint32_t parts = std::min<uint64_t>(c->fold_parts, nrows / 4);
  if (cs && !(c->two_streams && !c->timing && parts >= 2)) return false;
  if (c->two_streams && !c->timing && parts >= 2) {
    // the batch in `parts` slices on as many streams: one slice's digit INTTs
    // and key switches interleave with the others', filling each launch's tail
    while (c->part_streams.size() < parts - 1) {
      cudaStream_t ps;
      CU(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
      c->part_streams.push_back(ps);
    }
    cudaEvent_t fork;
    CU(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    CU(cudaEventRecord(fork, st));
    std::vector<cudaEvent_t> joins;
    const uint64_t base = cs ? cs->pair_off : 0;
    cudaStream_t head = cs ? cs->streams[0] : st;
    for (uint32_t h = 0; h < parts; ++h) {
      cudaStream_t hs = cs ? cs->streams[h] : (h ? c->part_streams[h - 1] : st);
      if (h || cs) CU(cudaStreamWaitEvent(hs, fork, 0));
      const uint64_t rr0 = nrows * h / parts, nr = nrows * (h + 1) / parts - rr0, pp = nr * cols,
                     off = base + rr0 * cols;
      uint32_t* A = c->d_dotA + off * c->ct_words();
      uint32_t* B = c->d_dotB + off * c->ct_words();
      uint32_t* D = c->d_dig + off * c->pt_words();
      launch_chunk_dot(c, d_in + rr0 * w->kc * c->ct_words(), w, nr, A, hs);
      uint32_t* res = fold(c, pp, A, B, hs, D);
      launch_mask_acc(c, g, (unsigned)(pp * c->P()), res, d_rows + rr0, cols, s->d_acc, hs);
      if (h) {
        cudaEvent_t j;
        CU(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
        CU(cudaEventRecord(j, hs));
        joins.push_back(j);
      }
    }
    for (cudaEvent_t j : joins) {
      CU(cudaStreamWaitEvent(head, j, 0));
      cudaEventDestroy(j);
    }
    if (cs) CU(cudaEventRecord(cs->done, head));
    cudaEventDestroy(fork);
    return true;
  }
  // latency path: the mask plaintexts are computed on a side stream while
  // the fold runs (they depend only on the slot)
  const bool premask = c->logn >= 13 && c->logn <= 14 && blocksP < 2u * 148u && c->premask;
  cudaEvent_t mask_ev = nullptr;
  uint32_t* masks = nullptr;
  if (premask) {
    masks = pool_get(c->pool_masks, c->pool_masks_bytes, (size_t)blocksP * c->n * 4);
    if (!c->bias_stream) CU(cudaStreamCreateWithFlags(&c->bias_stream, cudaStreamNonBlocking));
    cudaEvent_t fork;
    CU(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    CU(cudaEventRecord(fork, st));
    CU(cudaStreamWaitEvent(c->bias_stream, fork, 0));
    cudaEventDestroy(fork);
    const size_t sm1 = smem_bytes(c, 1);
    HEI_DISPATCH(c->logn, (k_mask_prep<LG><<<blocksP, Ntt<LG>::T, sm1, c->bias_stream>>>(g, d_rows, cols, masks)),
                 (void)0);
    LAUNCHED();
    CU(cudaEventCreateWithFlags(&mask_ev, cudaEventDisableTiming));
    CU(cudaEventRecord(mask_ev, c->bias_stream));
  }
  launch_chunk_dot(c, d_in, w, nrows, c->d_dotA, st);
  uint32_t* res = fold(c, pairs, c->d_dotA, c->d_dotB, st);
  if (premask) {
    CU(cudaStreamWaitEvent(st, mask_ev, 0));
    cudaEventDestroy(mask_ev);
    k_mask_apply<<<grid_for((uint64_t)blocksP * c->n, 256), 256, 0, st>>>(g, res, masks, d_rows, cols, pairs,
                                                                         s->d_acc);
    LAUNCHED();
  } else {
    launch_mask_acc(c, g, blocksP, res, d_rows, cols, s->d_acc, st);
  }
  return true;
}

void stream_flush(hei_gpu_stream* s) {
  if (s->pend_idx.empty()) return;
  hei_gpu_ctx* c = s->ctx;
  const uint64_t nr = s->pend_idx.size();
  CU(cudaMemcpyAsync(s->d_rows, s->pend_idx.data(), nr * 8, cudaMemcpyHostToDevice, c->stream));
  run_rows(s, s->d_stage, s->d_rows, nr, c->stream);
  CU(cudaStreamSynchronize(c->stream));
  s->pend_idx.clear();
}

void launch_bias_plain(hei_gpu_stream* s, const int64_t* d_bias, cudaStream_t st) {
  hei_gpu_ctx* c = s->ctx;
  s->d_biasp = pool_get(c->pool_biasp, c->pool_biasp_bytes, s->C * c->pt_words() * 4);
  k_bias_plain<<<(unsigned)(s->C * c->P()), c->threads(), smem_bytes(c, 1), st>>>(
      c->geo, d_bias, (uint32_t)s->w->cols, s->rows * s->w->cols, s->d_biasp);
  LAUNCHED();
}

void finish_to(hei_gpu_stream* s, uint32_t* d_out, cudaStream_t st) {
  hei_gpu_ctx* c = s->ctx;
  if (s->bias_ev) {
    CU(cudaStreamWaitEvent(st, s->bias_ev, 0));
  } else {
    int64_t* d_bias = s->d_bias;
    if (!d_bias) {  // streams created before the bias was staged (host API)
      d_bias = pool_get(c->pool_bias, c->pool_bias_bytes, s->bias.size() * 8);
      CU(cudaMemcpyAsync(d_bias, s->bias.data(), s->bias.size() * 8, cudaMemcpyHostToDevice, st));
    }
    launch_bias_plain(s, d_bias, st);
  }
  // (streams assembled in place for the sharded finishes keep no counters)
  k_finish_add<<<grid_for(s->C * c->ct_words(), 256), 256, 0, st>>>(c->geo, s->d_acc, s->d_biasp, s->C, d_out, s->d_ops0,
                                                                   s->d_ops0 ? c->h_opsnap : nullptr);
  LAUNCHED();
}

void check_bias_range(hei_gpu_ctx* c, const int64_t* bias, uint64_t cols) {
  const int64_t lim = (int64_t)(((u128)c->t[0] * c->t[1] - 1) / 2);
  for (uint64_t j = 0; j < cols; ++j)
    if (bias[j] > lim || bias[j] < -lim) raise(HEI_RANGE_ERROR, "encode_signed: value outside the centered range");
}

// capacity_check (fixed_point.cpp:61-77)
void capacity_gate(hei_gpu_ctx* c, uint64_t f, const char* who) {
  int log_f = f <= 1 ? 0 : 64 - __builtin_clzll(f - 1);
  int required = (int)(c->in_bits + c->s_x + c->s_w) + log_f;
  u128 prod = (u128)c->t[0] * c->t[1];
  int cap = -1;
  while (prod) ++cap, prod >>= 1;
  if (required + 1 > cap)
    raise(HEI_RANGE_ERROR, std::string(who) + ": product needs " + std::to_string(required) +
                               " result bits, capacity is " + std::to_string(cap) + "; refusing");
}

hei_gpu_stream* stream_new(hei_gpu_ctx* c, const hei_gpu_weights* w, const int64_t* bias, uint64_t rows,
                           bool host_staging = true, cudaStream_t zero_on = nullptr, bool encode_bias = true,
                           unsigned long long* ext_acc = nullptr) {
  if (rows == 0) raise(HEI_PARAM_ERROR, "matmul: empty input");
  if (!w || w->cols == 0 || w->f == 0) raise(HEI_PARAM_ERROR, "matmul: empty weights");
  if (w->ctx != c) raise(HEI_PARAM_ERROR, "matmul: weights encoded for a different context");
  capacity_gate(c, w->f, "matmul");
  require_keys(c);
  check_bias_range(c, bias, w->cols);
  auto s = std::make_unique<hei_gpu_stream>();
  s->ctx = c;
  s->w = w;
  s->bias.assign(bias, bias + w->cols);
  s->rows = rows;
  s->seen.assign(rows, false);
  s->C = (rows * w->cols + c->n - 1) / c->n;
  const uint64_t bp = auto_batch_pairs(c);
  s->cap_rows = std::max<uint64_t>(1, std::min<uint64_t>(rows, bp / w->cols));
  if (host_staging) {
    CU(cudaMalloc(&s->d_acc, s->C * c->ct_words() * 8));
    CU(cudaMalloc(&s->d_stage, s->cap_rows * w->kc * c->ct_words() * 4));
    CU(cudaMalloc(&s->d_stage64, s->cap_rows * w->kc * c->ct_words() * 8));
    CU(cudaMalloc(&s->d_rows, s->cap_rows * 8));
  } else {
    // one-shot device-resident call: borrow the context pools, or accumulate
    // into the caller's (pre-zeroed) buffer
    s->d_acc = ext_acc ? ext_acc : pool_get(c->pool_acc, c->pool_acc_bytes, s->C * c->ct_words() * 8);
    s->d_rows = pool_get(c->pool_rows, c->pool_rows_bytes, s->cap_rows * 8);
    s->owns_acc = false;
    s->owns_rows = false;
  }
  if (!ext_acc) CU(cudaMemsetAsync(s->d_acc, 0, s->C * c->ct_words() * 8, zero_on ? zero_on : c->stream));
  // the counters' start (MatmulStream keeps start_ = be.counters(),
  // matmul.cpp:143): one-shot calls snapshot them in their first kernel
  // (k_iota), host-API streams here
  if (host_staging) {
    CU(cudaMalloc(&s->d_ops0, 3 * 8));
    CU(cudaMemcpyAsync(s->d_ops0, c->d_ops, 3 * 8, cudaMemcpyDeviceToDevice, c->stream));
  } else {
    s->d_ops0 = c->d_opsnap;
    s->owns_ops0 = false;
  }
  if (!host_staging && encode_bias) {
    // stage the bias now (pinned, async): every earlier call has synchronised
    const size_t bb = s->bias.size() * 8;
    if (bb > c->pinned_bias_bytes) {
      if (c->pinned_bias) cudaFreeHost(c->pinned_bias);
      c->pinned_bias = nullptr;
      CU(cudaMallocHost(&c->pinned_bias, bb));
      c->pinned_bias_bytes = bb;
    }
    std::memcpy(c->pinned_bias, s->bias.data(), bb);
    s->d_bias = pool_get(c->pool_bias, c->pool_bias_bytes, bb);
    cudaStream_t zs = zero_on ? zero_on : c->stream;
    CU(cudaMemcpyAsync(s->d_bias, c->pinned_bias, bb, cudaMemcpyHostToDevice, zs));
    // encode the bias plaintext off the critical path, overlapping the fold
    if (!c->bias_stream) CU(cudaStreamCreateWithFlags(&c->bias_stream, cudaStreamNonBlocking));
    cudaEvent_t staged;
    CU(cudaEventCreateWithFlags(&staged, cudaEventDisableTiming));
    CU(cudaEventRecord(staged, zs));
    CU(cudaStreamWaitEvent(c->bias_stream, staged, 0));
    cudaEventDestroy(staged);
    launch_bias_plain(s.get(), s->d_bias, c->bias_stream);
    CU(cudaEventCreateWithFlags(&s->bias_ev, cudaEventDisableTiming));
    CU(cudaEventRecord(s->bias_ev, c->bias_stream));
  }
  return s.release();
}

// MatmulStream::finish's counters (matmul.cpp:224-229): measured deltas of
// mul_plain / rotation / add (k_finish_add wrote the start and end snapshots
// to the mapped pinned h_opsnap; read after the call's synchronisation),
// plus the ciphertext counts.
void ops_report(hei_gpu_stream* s, hei_op_counters* cnt) {
  const unsigned long long* h = s->ctx->h_opsnap;
  cnt->mul_plain_count = h[3] - h[0];
  cnt->rotation_count = h[4] - h[1];
  cnt->add_count = h[5] - h[2];
  cnt->ciphertexts_in = s->rows * s->w->kc;
  cnt->ciphertexts_out = s->C;
}

void stream_free(hei_gpu_stream* s) {
  if (!s) return;
  cudaSetDevice(s->ctx->device);
  if (s->owns_acc) cudaFree(s->d_acc);
  if (s->d_stage) cudaFree(s->d_stage);
  if (s->d_stage64) cudaFree(s->d_stage64);
  if (s->owns_rows) cudaFree(s->d_rows);
  if (s->bias_ev) cudaEventDestroy(s->bias_ev);
  if (s->owns_ops0 && s->d_ops0) cudaFree(s->d_ops0);
  delete s;
}

void stream_push(hei_gpu_stream* s, uint64_t row, const uint64_t* chunks, int form) {
  hei_gpu_ctx* c = s->ctx;
  if (s->finished) raise(HEI_PARAM_ERROR, "push_row: stream already finished");
  if (row >= s->rows) raise(HEI_PARAM_ERROR, "push_row: row index out of range");
  if (s->seen[row]) raise(HEI_PARAM_ERROR, "push_row: row pushed twice");
  if (form != HEI_FORM_EVAL && form != HEI_FORM_COEFF) raise(HEI_PARAM_ERROR, "push_row: unknown form");
  const uint64_t slot = s->pend_idx.size();
  const size_t words = s->w->kc * c->ct_words();
  CU(cudaMemcpyAsync(s->d_stage64 + slot * words, chunks, words * 8, cudaMemcpyHostToDevice, c->stream));
  k_narrow<<<grid_for(words, 256), 256, 0, c->stream>>>(c->geo, s->d_stage64 + slot * words,
                                                          s->d_stage + slot * words, s->w->kc, c->d_err);
  LAUNCHED();
  // a row with an unreduced residue is rejected before it is recorded (the
  // reference's load_ciphertext throws before push_row sees it,
  // serialize.cpp:80-90): its staging slot is reused by the next push and the
  // caller may push the row again
  check_err_flag(c, HEI_CODEC_ERROR, "push_row: coefficient not reduced");
  if (form == HEI_FORM_COEFF) {
    launch_ct_ntt(c, (unsigned)(s->w->kc * 2 * c->P()), s->d_stage + slot * words, c->stream);
  }
  s->seen[row] = true;
  ++s->pushed;
  s->pend_idx.push_back(row);
  if (s->pend_idx.size() == s->cap_rows) stream_flush(s);
}

void stream_finish(hei_gpu_stream* s, uint64_t* out, hei_op_counters* cnt) {
  hei_gpu_ctx* c = s->ctx;
  if (s->finished) raise(HEI_PARAM_ERROR, "finish: already finished");
  if (s->pushed != s->rows)
    raise(HEI_PARAM_ERROR, "finish: " + std::to_string(s->rows - s->pushed) + " rows were never pushed");
  stream_flush(s);
  uint32_t* d_out = nullptr;
  uint64_t* d_out64 = nullptr;
  const uint64_t words = s->C * c->ct_words();
  CU(cudaMalloc(&d_out, words * 4));
  CU(cudaMalloc(&d_out64, words * 8));
  finish_to(s, d_out, c->stream);
  k_widen<<<grid_for(words, 256), 256, 0, c->stream>>>(d_out, d_out64, words);
  LAUNCHED();
  CU(cudaMemcpyAsync(out, d_out64, words * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  cudaFree(d_out);
  cudaFree(d_out64);
  s->finished = true;
  if (cnt) ops_report(s, cnt);
}

hei_gpu_weights* weights_alloc(hei_gpu_ctx* c, uint64_t f, uint64_t cols) {
  if (f == 0 || cols == 0) raise(HEI_PARAM_ERROR, "encode_weights: empty matrix");
  auto w = std::make_unique<hei_gpu_weights>();
  w->ctx = c;
  w->f = f;
  w->cols = cols;
  w->kc = (f + c->n - 1) / c->n;
  CU(cudaMalloc(&w->d_w, cols * w->kc * c->pt_words() * sizeof(uint2)));
  return w.release();
}

// ---- util::Prng host side (rng.hpp:19-68) ----
void prng_seed(hei_gpu_prng* p, uint64_t seed) {
  p->mt[0] = seed;
  for (int i = 1; i < 312; ++i) p->mt[i] = 6364136223846793005ULL * (p->mt[i - 1] ^ (p->mt[i - 1] >> 62)) + (uint64_t)i;
  p->mti = 312;
  p->have_spare = false;
}
uint64_t prng_next(hei_gpu_prng* p) {
  using namespace heb_baseline;
  if (p->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 156; ++i) {
      x = (p->mt[i] & kMtUM) | (p->mt[i + 1] & kMtLM);
      p->mt[i] = p->mt[i + 156] ^ (x >> 1) ^ ((x & 1) ? kMtA : 0);
    }
    for (; i < 311; ++i) {
      x = (p->mt[i] & kMtUM) | (p->mt[i + 1] & kMtLM);
      p->mt[i] = p->mt[i - 156] ^ (x >> 1) ^ ((x & 1) ? kMtA : 0);
    }
    x = (p->mt[311] & kMtUM) | (p->mt[0] & kMtLM);
    p->mt[311] = p->mt[155] ^ (x >> 1) ^ ((x & 1) ? kMtA : 0);
    p->mti = 0;
  }
  uint64_t x = p->mt[p->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}


// ---- mt19937_64 jump-ahead support (host, setup-time GF(2) algebra) ----
// phi = characteristic polynomial of the generator (degree 19937), found
// once by Berlekamp-Massey on bit 0 of the output stream; x^J mod phi by
// square-and-shift. Both are seed-independent and cached.
using Poly2 = std::vector<uint64_t>;  // bit i = coefficient of x^i

uint64_t get64(const Poly2& a, uint64_t off) {
  const uint64_t w = off >> 6, sh = off & 63;
  const uint64_t lo = w < a.size() ? a[w] : 0, hi = w + 1 < a.size() ? a[w + 1] : 0;
  return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
}

const Poly2& mt_charpoly() {
  static std::mutex mu;
  static Poly2 phi;
  std::lock_guard<std::mutex> lk(mu);
  if (!phi.empty()) return phi;
  const int Lx = heb_baseline::kMtDeg, LEN = 2 * Lx + 64;
  hei_gpu_prng g;
  prng_seed(&g, 5489);
  Poly2 srev((LEN + 63) / 64 + 2, 0);  // bit j = s[LEN - 1 - j]
  std::vector<uint8_t> sbits(LEN);
  for (int k = 0; k < LEN; ++k) sbits[k] = (uint8_t)(prng_next(&g) & 1);
  for (int j = 0; j < LEN; ++j)
    if (sbits[LEN - 1 - j]) srev[j >> 6] |= 1ull << (j & 63);
  const size_t W = (Lx + 64) / 64 + 2;
  Poly2 C(W, 0), B(W, 0), T;
  C[0] = B[0] = 1;
  int L = 0, m = 1;
  for (int N = 0; N < LEN; ++N) {
    const uint64_t base = (uint64_t)(LEN - 1 - N);
    uint64_t acc = 0;
    for (size_t w = 0; w * 64 <= (size_t)L; ++w) {
      uint64_t cw = C[w];
      if (w == 0) cw &= ~1ull;  // i >= 1
      acc ^= cw & get64(srev, base + 64 * w);
    }
    const uint32_t d = sbits[N] ^ (uint32_t)(__builtin_popcountll(acc) & 1);
    if (!d) {
      ++m;
      continue;
    }
    T = C;
    // C ^= B << m
    const size_t ws = m >> 6, bs = m & 63;
    for (size_t w = W; w-- > ws;) {
      uint64_t v = B[w - ws] << bs;
      if (bs && w - ws >= 1) v |= B[w - ws - 1] >> (64 - bs);
      C[w] ^= v;
    }
    if (2 * L <= N) {
      L = N + 1 - L;
      B = T;
      m = 1;
    } else {
      ++m;
    }
  }
  if (L != Lx) raise(HEI_INTERNAL, "mt19937_64 characteristic polynomial has unexpected degree");
  // phi_k = c_{L-k}
  Poly2 f((Lx + 64) / 64, 0);
  for (int k = 0; k <= Lx; ++k)
    if ((C[(Lx - k) >> 6] >> ((Lx - k) & 63)) & 1) f[k >> 6] |= 1ull << (k & 63);
  phi = f;
  return phi;
}

void poly_reduce(Poly2& a, const Poly2& phi) {
  const int D = heb_baseline::kMtDeg;
  const int64_t top = (int64_t)a.size() * 64 - 1;
  for (int64_t k = top; k >= D; --k) {
    if (!((a[k >> 6] >> (k & 63)) & 1)) continue;
    const int64_t sh = k - D;  // a ^= phi << sh
    const int64_t ws = sh >> 6, bs = sh & 63;
    for (size_t w = 0; w < phi.size(); ++w) {
      const uint64_t v = phi[w];
      a[w + ws] ^= v << bs;
      if (bs && w + ws + 1 < a.size()) a[w + ws + 1] ^= v >> (64 - bs);
    }
  }
  a.resize((D + 63) / 64);
}

// x^J mod phi
Poly2 mt_jump_poly(uint64_t J) {
  static std::mutex mu;
  static std::map<uint64_t, Poly2> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(J);
  if (it != cache.end()) return it->second;
  const Poly2& phi = mt_charpoly();
  const size_t nw = (heb_baseline::kMtDeg + 63) / 64;
  Poly2 r(nw, 0);
  r[0] = 1;
  for (int bit = 63; bit >= 0; --bit) {
    if (!(J >> bit) && r[0] == 1) {
      bool one = true;
      for (size_t w = 1; w < nw; ++w) one = one && r[w] == 0;
      if (one) continue;  // leading zeros of J
    }
    // square: spread bits
    Poly2 sq(2 * nw + 1, 0);
    for (size_t w = 0; w < nw; ++w) {
      uint64_t x = r[w];
      uint64_t lo = 0, hi = 0;
      for (int i = 0; i < 32; ++i) {
        lo |= ((x >> i) & 1ull) << (2 * i);
        hi |= ((x >> (i + 32)) & 1ull) << (2 * i);
      }
      sq[2 * w] = lo;
      sq[2 * w + 1] = hi;
    }
    poly_reduce(sq, phi);
    r = sq;
    if ((J >> bit) & 1) {  // r *= x
      Poly2 sh(nw + 1, 0);
      for (size_t w = 0; w < nw; ++w) {
        sh[w] |= r[w] << 1;
        sh[w + 1] |= r[w] >> 63;
      }
      poly_reduce(sh, phi);
      r = sh;
    }
  }
  cache[J] = r;
  return r;
}


// Jump polynomials of the tree levels for chunk size C: level k is
// x^(2^k C) mod phi = (level k-1)^2 mod phi. Cached per C.
const std::vector<Poly2>& mt_level_polys(uint64_t C, uint32_t levels) {
  static std::mutex mu;
  static std::map<uint64_t, std::vector<Poly2>> cache;
  const Poly2 first = mt_jump_poly(C);
  std::lock_guard<std::mutex> lk(mu);
  auto& v = cache[C];
  if (v.empty()) v.push_back(first);
  const Poly2& phi = mt_charpoly();
  const size_t nw = (heb_baseline::kMtDeg + 63) / 64;
  while (v.size() < levels) {
    const Poly2& r = v.back();
    Poly2 sq(2 * nw + 1, 0);
    for (size_t w = 0; w < nw; ++w) {
      const uint64_t x = r[w];
      uint64_t lo = 0, hi = 0;
      for (int i = 0; i < 32; ++i) {
        lo |= ((x >> i) & 1ull) << (2 * i);
        hi |= ((x >> (i + 32)) & 1ull) << (2 * i);
      }
      sq[2 * w] = lo;
      sq[2 * w + 1] = hi;
    }
    poly_reduce(sq, phi);
    v.push_back(sq);
  }
  return v;
}

// Start windows of K chunk generators per branch, chunk m starting m * C
// words after d_state (block-aligned, mti == 312): starts [2][K][313].
void mt_chunk_starts(hei_gpu_ctx* c, const uint64_t* d_state, uint64_t K, uint64_t C, uint64_t* d_starts,
                     cudaStream_t st) {
  uint32_t levels = 0;
  while ((1ull << levels) < K) ++levels;
  if (levels == 0) {
    for (int bb = 0; bb < 2; ++bb)
      CU(cudaMemcpyAsync(d_starts + (uint64_t)bb * K * 313, d_state + bb * 313, 313 * 8, cudaMemcpyDeviceToDevice,
                         st));
    return;
  }
  const std::vector<Poly2>& polys = mt_level_polys(C, levels);
  const uint32_t wlen = 312 * 65, S = 64;
  const size_t pw = polys[0].size();
  const uint64_t jobs_max = K / 2 + 1;
  uint64_t* d_poly = scratch<uint64_t>(c, kScrMtPoly, levels * pw * 8);
  uint64_t* d_wseq = scratch<uint64_t>(c, kScrMtWseq, jobs_max * 2 * wlen * 8);
  uint64_t* d_part = scratch<uint64_t>(c, kScrMtPart, jobs_max * 2 * S * 312 * 8);
  for (uint32_t k = 0; k < levels; ++k)
    CU(cudaMemcpyAsync(d_poly + k * pw, polys[k].data(), pw * 8, cudaMemcpyHostToDevice, st));
  for (int bb = 0; bb < 2; ++bb)
    CU(cudaMemcpyAsync(d_starts + (uint64_t)bb * K * 313, d_state + bb * 313, 313 * 8, cudaMemcpyDeviceToDevice, st));
  const uint32_t wsl = (uint32_t)((pw + S - 1) / S);
  for (uint32_t k = 0; k < levels; ++k) {
    const uint64_t step = 1ull << k, jobs = std::min<uint64_t>(step, K - step);
    heb_baseline::k_mt_wseq<<<dim3(2, (unsigned)jobs), 320, 0, st>>>(d_starts, (uint32_t)K, d_wseq, wlen);
    heb_baseline::k_mt_xor<<<dim3(S, 2, (unsigned)jobs), 320, 0, st>>>(d_wseq, wlen, d_poly + k * pw, wsl, d_part);
    heb_baseline::k_mt_xor_reduce<<<dim3(2, (unsigned)jobs), 320, 0, st>>>(d_part, S, d_starts, (uint32_t)K,
                                                                          (uint32_t)step);
    g_launches += 3;
  }
  CU(cudaGetLastError());
}

// ---- client encryption: matmul::encode_inputs (matmul.cpp:59-81) --------
// Every row is split into ceil(f / N) slot chunks, each encode_signed + encrypt
// (eval form) with the branch's util::Prng stream, in (row, chunk) order — the
// same draws BfvBackend::encrypt consumes (context.cpp:262-303).
void encode_inputs_impl(hei_gpu_ctx* c, const int64_t* x, uint64_t rows, uint64_t f, hei_gpu_prng* rng0,
                        hei_gpu_prng* rng1, uint64_t* out_host, uint32_t* out_dev, cudaStream_t st) {
  if (rows == 0 || f == 0) raise(HEI_PARAM_ERROR, "encode_inputs: empty matrix");
  if (!c->d_pk[0] || !c->d_pk[1]) raise(HEI_KEY_ERROR, "encrypt: this backend holds no public key");
  if (!rng0 || !rng1) raise(HEI_PARAM_ERROR, "encode_inputs: encryption randomness required");
  if (rng0->have_spare || rng1->have_spare)
    raise(HEI_PARAM_ERROR, "encode_inputs: rng holds a cached Box-Muller spare; cannot replay on the device");
  const int64_t lim = (int64_t)(((u128)c->t[0] * c->t[1] - 1) / 2);
  for (uint64_t i = 0; i < rows * f; ++i)
    if (x[i] > lim || x[i] < -lim) raise(HEI_RANGE_ERROR, "encode_signed: value outside the centered range");
  const Geo& g = c->geo;
  const uint32_t n = c->n, P = c->P();
  const uint64_t kc = (f + n - 1) / n, E_total = rows * kc, Dtot = E_total * 3 * n;
  if (!c->d_pkp) {
    CU(cudaMalloc(&c->d_pkp, 2ull * P * n * sizeof(uint2)));
    const size_t sm = smem_bytes(c, 1);
    HEI_DISPATCH(c->logn, (k_prepare_pk<LG><<<2 * P, Ntt<LG>::T, sm, st>>>(g, c->d_pk[0], c->d_pk[1], c->d_pkp, c->d_err)),
                 (k_prepare_pk_g<<<2 * P, c->threads(), sm, st>>>(g, c->d_pk[0], c->d_pk[1], c->d_pkp, c->d_err)));
    LAUNCHED();
    check_err_flag(c, HEI_CODEC_ERROR, "public key: coefficient not reduced");
  }
  struct Free {
    std::vector<void*> p;
    ~Free() {
      for (void* v : p) cudaFree(v);
    }
  } fr;
  auto alloc = [&](auto** ptr, size_t bytes) {
    CU(cudaMalloc((void**)ptr, bytes));
    fr.p.push_back((void*)*ptr);
  };
  const uint64_t Eb = std::min<uint64_t>(E_total, 256);
  int64_t* d_x = nullptr;
  uint64_t *d_raw = nullptr, *d_state = nullptr, *d_out64 = nullptr;
  int8_t* d_noise = nullptr;
  uint32_t *d_m = nullptr, *d_ct = nullptr;
  d_x = scratch<int64_t>(c, kScrX, rows * f * 8);
  d_raw = scratch<uint64_t>(c, kScrRawAll, 2 * Dtot * 8);
  d_state = scratch<uint64_t>(c, kScrState, 2 * 313 * 8);
  d_noise = scratch<int8_t>(c, kScrNoise, Eb * 2 * 3 * n);
  d_m = scratch<uint32_t>(c, kScrM, Eb * 2 * n * 4);
  if (!out_dev) {
    d_ct = scratch<uint32_t>(c, kScrCt, Eb * c->ct_words() * 4);
    d_out64 = scratch<uint64_t>(c, kScrOut64, Eb * c->ct_words() * 8);
  }
  CU(cudaMemcpyAsync(d_x, x, rows * f * 8, cudaMemcpyHostToDevice, st));
  const hei_gpu_prng init0 = *rng0, init1 = *rng1;
  for (bool force_seq = false;; force_seq = true) {
    uint64_t hstate[2][313];
    for (int b = 0; b < 2; ++b) {
      hei_gpu_prng* r = b ? rng1 : rng0;
      std::memcpy(hstate[b], r->mt, 312 * 8);
      hstate[b][312] = r->mti;
    }
    CU(cudaMemcpyAsync(d_state, hstate, sizeof(hstate), cudaMemcpyHostToDevice, st));
    const bool jump = c->mt_jump && !force_seq && hstate[0][312] == 312 && hstate[1][312] == 312 && E_total >= 64;
    if (jump) {
      uint64_t K = std::min<uint64_t>(c->mt_chunks_max, E_total / 8);
      const uint64_t Cenc = (E_total + K - 1) / K;
      K = (E_total + Cenc - 1) / Cenc;
      const uint64_t C = Cenc * 3 * n;
      uint64_t* d_starts = nullptr;
      d_starts = scratch<uint64_t>(c, kScrStarts, 2 * K * 313 * 8);
      mt_chunk_starts(c, d_state, K, C, d_starts, st);
      heb_baseline::k_mt_chunks<<<dim3((unsigned)K, 2), 320, 0, st>>>(d_starts, (uint32_t)K, C, Dtot, d_raw, d_state);
      LAUNCHED();
    } else {
      heb_baseline::k_mt_generate<<<2, 320, 0, st>>>(d_state, d_raw, Dtot);
      LAUNCHED();
    }
    const size_t sm1 = smem_bytes(c, 1);
    for (uint64_t e0 = 0; e0 < E_total; e0 += Eb) {
      const uint64_t E = std::min<uint64_t>(Eb, E_total - e0);
      heb_baseline::k_bl_noise<<<dim3((unsigned)E, 2), 256, 0, st>>>(d_raw + e0 * 3 * n, Dtot, n, (uint32_t)E, d_noise,
                                                                    c->d_err);
      LAUNCHED();
      HEI_DISPATCH(c->logn,
                   (k_bl_encode<LG><<<dim3((unsigned)E, 2), Ntt<LG>::T, sm1, st>>>(g, d_x, rows, f, e0, (uint32_t)kc, d_m, 1)),
                   (k_bl_encode_g<<<dim3((unsigned)E, 2), c->threads(), sm1, st>>>(g, d_x, rows, f, e0, (uint32_t)kc, d_m, 1)));
      LAUNCHED();
      uint32_t* ct = out_dev ? out_dev + e0 * c->ct_words() : d_ct;
      launch_bl_encrypt(c, g, (unsigned)(E * P), d_noise, d_m, ct, sm1, st);
      LAUNCHED();
      if (!out_dev) {
        k_widen<<<grid_for(E * c->ct_words(), 256), 256, 0, st>>>(d_ct, d_out64, E * c->ct_words());
        LAUNCHED();
        CU(cudaMemcpyAsync(out_host + e0 * c->ct_words(), d_out64, E * c->ct_words() * 8, cudaMemcpyDeviceToHost, st));
      }
    }
    CU(cudaMemcpyAsync(hstate, d_state, sizeof(hstate), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    for (int b = 0; b < 2; ++b) {
      hei_gpu_prng* r = b ? rng1 : rng0;
      std::memcpy(r->mt, hstate[b], 312 * 8);
      r->mti = (uint32_t)hstate[b][312];
    }
    if (jump) {
      uint32_t errh = 0;
      CU(cudaMemcpyAsync(&errh, c->d_err, 4, cudaMemcpyDeviceToHost, c->stream));
      CU(cudaStreamSynchronize(c->stream));
      if (errh) {
        CU(cudaMemsetAsync(c->d_err, 0, 4, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        *rng0 = init0;
        *rng1 = init1;
        continue;
      }
    }
    check_err_flag(c, HEI_INTERNAL, "encode_inputs: rng rejection in the encryption stream (replay unsupported)");
    break;
  }
}

}  // namespace

// ================================================================== C ABI
extern "C" {

const char* hei_gpu_last_error(void) { return g_err.c_str(); }
const char* hei_gpu_version(void) { return "heinfer_b200 0.1 (sm_100a)"; }
#ifdef HEI_W2_TRACE
// debug builds only: the latency kernel's last phase timestamps [256][2][8]
int hei_gpu_debug_w2_trace(uint64_t* out) {
  return cudaMemcpyFromSymbol(out, g_w2_trace, sizeof(g_w2_trace)) == cudaSuccess ? 0 : 8;
}
#endif
uint64_t hei_gpu_launch_count(void) { return g_launches; }
void hei_gpu_reset_launch_count(void) { g_launches = 0; }

int hei_proposed_counts(uint64_t R, uint64_t cols, uint64_t f, uint32_t n, hei_op_counters* c) {
  return guarded([&] {
    if (!R || !cols || !f) raise(HEI_PARAM_ERROR, "empty shape");
    if (!n || (n & (n - 1))) raise(HEI_PARAM_ERROR, "ring degree must be a power of two");
    uint64_t k = (f + n - 1) / n, lg = 63 - __builtin_clzll(n);
    c->mul_plain_count = R * cols * (k + 1);
    c->rotation_count = R * cols * lg;
    c->add_count = R * cols * (k + lg);
    c->ciphertexts_in = R * k;
    c->ciphertexts_out = (R * cols + n - 1) / n;
  });
}

int hei_baseline_counts(uint64_t R, uint64_t cols, uint64_t f, uint32_t n, hei_op_counters* c) {
  return guarded([&] {
    if (!R || !cols || !f) raise(HEI_PARAM_ERROR, "empty shape");
    if (!n || (n & (n - 1))) raise(HEI_PARAM_ERROR, "ring degree must be a power of two");
    uint64_t blocks = (R + n - 1) / n;
    c->mul_plain_count = blocks * f * cols;
    c->rotation_count = 0;
    c->add_count = blocks * cols * f;
    c->ciphertexts_in = blocks * f;
    c->ciphertexts_out = blocks * cols;
  });
}

int hei_gpu_ctx_create(const hei_twin_desc* d, hei_gpu_ctx** out) {
  return guarded([&] {
    if (!d || !out) raise(HEI_PARAM_ERROR, "null argument");
    const uint32_t n = d->n;
    if (!n || (n & (n - 1)) || n < 8 || n > 32768) raise(HEI_PARAM_ERROR, "ring degree must be a power of two in [8, 32768]");
    if (n > 16384) raise(HEI_PARAM_ERROR, "ring degree above 16384 is not supported on the device path");
    if (d->L[0] == 0 || d->L[1] == 0) raise(HEI_PARAM_ERROR, "ciphertext modulus chain is empty");
    if (d->L[0] + d->L[1] > kMaxPrimes) raise(HEI_PARAM_ERROR, "too many primes for the device path");
    if (n >= 4096 && d->L[0] + d->L[1] > (uint32_t)kMaxAB)
      raise(HEI_PARAM_ERROR, "at most 12 ciphertext primes in total for N >= 4096 on the device path");
    if (d->t[0] == d->t[1]) raise(HEI_PARAM_ERROR, "twin moduli must differ");
    auto c = std::make_unique<hei_gpu_ctx>();
    c->device = d->device;
    if (const char* v = std::getenv("HEI_NO_GRAPHS")) c->graphs = std::atoi(v) == 0;
    if (const char* v = std::getenv("HEI_TWO_STREAMS")) c->two_streams = std::atoi(v) != 0;
    if (const char* v = std::getenv("HEI_MT_JUMP")) c->mt_jump = std::atoi(v) != 0;
    if (const char* v = std::getenv("HEI_FUSE_DIGITS")) c->fuse_digits = std::atoi(v) != 0;
    if (const char* v = std::getenv("HEI_PREMASK")) c->premask = std::atoi(v) != 0;
    if (const char* v = std::getenv("HEI_PDL")) c->pdl = std::atoi(v) != 0;
    if (const char* v = std::getenv("HEI_KS_CLUSTER")) c->ks_cluster = std::atoi(v) != 0;
    if (const char* v = std::getenv("HEI_E2E_DIV")) c->e2e_div = std::max(1, std::atoi(v));
    if (const char* v = std::getenv("HEI_MT_CHUNKS")) c->mt_chunks_max = std::max(1, std::atoi(v));
    if (const char* v = std::getenv("HEI_FOLD_PARTS"))
      c->fold_parts = std::min<uint32_t>(kMaxFoldParts, std::max(1, std::atoi(v)));
    if (const char* v = std::getenv("HEI_DOT_ROWS")) c->dot_rows = std::atoi(v) != 0;
    if (const char* v = std::getenv("HEI_MASK_CACHE")) c->mask_cache = std::atoi(v) != 0;
    if (const char* v = std::getenv("HEI_E2E_OVERLAP")) c->e2e_overlap = std::atoi(v) != 0;
    if (const char* v = std::getenv("HEI_MASK_GROUP")) c->mask_group = std::max(1, std::atoi(v));
    c->n = n;
    c->logn = 31 - __builtin_clz(n);
    c->s_x = d->s_x;
    c->s_w = d->s_w;
    c->in_bits = d->input_int_bits;
    const uint64_t two_n = 2ull * n;
    for (int b = 0; b < 2; ++b) {
      const uint64_t t = d->t[b];
      c->t[b] = t;
      c->L[b] = d->L[b];
      // EncryptionParams::validate (params.cpp:27-66)
      if (t < 2 || t % two_n != 1)
        raise(HEI_PARAM_ERROR, "plaintext modulus " + std::to_string(t) + " is not 1 mod 2n; slot batching is unavailable");
      if (!is_prime(t)) raise(HEI_PARAM_ERROR, "plaintext modulus must be prime");
      if (t >= (1ull << 31)) raise(HEI_PARAM_ERROR, "plaintext modulus must be below 2^31 on the device path");
    }
    c->q.assign(d->q, d->q + d->L[0] + d->L[1]);
    for (int b = 0; b < 2; ++b) {
      const uint64_t* qb = d->q + (b ? d->L[0] : 0);
      for (uint32_t i = 0; i < d->L[b]; ++i) {
        const uint64_t qi = qb[i];
        if (!is_prime(qi)) raise(HEI_PARAM_ERROR, "ciphertext modulus " + std::to_string(qi) + " is not prime");
        if (qi % two_n != 1) raise(HEI_PARAM_ERROR, "ciphertext modulus " + std::to_string(qi) + " is not 1 mod 2n");
        if (qi == d->t[b]) raise(HEI_PARAM_ERROR, "ciphertext modulus collides with plaintext modulus");
        if (qi >= (1ull << 31)) raise(HEI_PARAM_ERROR, "ciphertext moduli must be below 2^31 on the device path");
        for (uint32_t j = 0; j < i; ++j)
          if (qb[j] == qi) raise(HEI_PARAM_ERROR, "duplicate ciphertext modulus");
      }
    }
    const uint32_t P = c->P();
    Geo& g = c->geo;
    g.n = n;
    g.logn = c->logn;
    g.P = P;
    g.ct_words = (uint32_t)c->ct_words();
    g.pt_words = (uint32_t)c->pt_words();
    g.L[0] = c->L[0];
    g.L[1] = c->L[1];
    // twiddle tables: P q-primes then t0, t1
    std::vector<uint2> fwd((size_t)(P + 2) * n), inv((size_t)(P + 2) * n);
    auto build = [&](uint64_t q, size_t row, uint2& last, uint2& ninv) {
      const uint64_t psi = root_2n(n, q), psi_inv = invmod(psi, q);
      for (uint32_t k = 0; k < n; ++k) {
        const uint32_t e = rev_bits(k, c->logn);
        const uint64_t z = powmod(psi, e, q), iz = powmod(psi_inv, e, q);
        fwd[row * n + k] = make_uint2((uint32_t)z, shoup32(z, q));
        inv[row * n + k] = make_uint2((uint32_t)iz, shoup32(iz, q));
      }
      const uint64_t ni = invmod(n, q);
      const uint64_t l1 = mulmod(inv[row * n + 1].x, ni, q);
      ninv = make_uint2((uint32_t)ni, shoup32(ni, q));
      last = make_uint2((uint32_t)l1, shoup32(l1, q));
    };
    for (int b = 0; b < 2; ++b) {
      const uint32_t first = b ? c->L[0] : 0;
      // Delta = floor(Q / t) mod q_i via exact multiprecision-free arithmetic:
      // floor(Q/t) = (Q - (Q mod t)) / t, and Q mod t, Q mod q_i are products
      // of residues, so Delta mod q_i = (Q mod q_i - Q mod t) * t^-1 mod q_i.
      const uint64_t t = c->t[b];
      uint64_t Qmodt = 1 % t;
      for (uint32_t i = 0; i < c->L[b]; ++i) Qmodt = mulmod(Qmodt, d->q[first + i] % t, t);
      // BranchInfo
      BranchInfo& br = g.br[b];
      br.t = (uint32_t)t;
      br.L = c->L[b];
      br.first = first;
      build(t, P + b, br.last, br.ninv);
      br.psi_inv = (uint32_t)invmod(root_2n(n, t), t);
      br.mu = (uint64_t)(((u128)1 << 64) / t);
      uint64_t qmin = UINT64_MAX, qmax = 0;
      for (uint32_t i = 0; i < c->L[b]; ++i) qmin = std::min(qmin, d->q[first + i]), qmax = std::max(qmax, d->q[first + i]);
      for (uint32_t i = 0; i < c->L[b]; ++i) {
        const uint64_t qi = d->q[first + i];
        PrimeInfo& pr = g.pr[first + i];
        pr.q = (uint32_t)qi;
        pr.b = b;
        pr.i = i;
        pr.L = c->L[b];
        pr.first = first;
        pr.poly0 = (b ? 2 * c->L[0] : 0) + i;
        pr.poly1 = (b ? 2 * c->L[0] : 0) + c->L[b] + i;
        pr.fast_reduce = qmax < 2 * qmin ? 1u : 0u;  // digit < q_l < 2 q_i
        pr.mu = (uint64_t)(((u128)1 << 64) / qi);
        build(qi, first + i, pr.last, pr.ninv);
        // Q mod q_i = 0, so Delta mod q_i = (0 - Q mod t) * t^-1 mod q_i
        const uint64_t dl = mulmod((qi - Qmodt % qi) % qi, invmod(t % qi, qi), qi);
        pr.delta = make_uint2((uint32_t)dl, shoup32(dl, qi));
      }
    }
    // slot index map, generator 3 (context.cpp:50-63)
    std::vector<uint32_t> index_map(n);
    {
      const uint64_t m = two_n;
      uint64_t pos = 1;
      for (uint32_t i = 0; i < n / 2; ++i) {
        index_map[i] = rev_bits((uint32_t)((pos - 1) >> 1), c->logn);
        index_map[i + n / 2] = rev_bits((uint32_t)((m - pos - 1) >> 1), c->logn);
        pos = (pos * 3) % m;
      }
    }
    // exact CRT constants (context.cpp:35-48) in 8 x 32-bit limbs
    for (uint32_t b = 0; b < 2; ++b) {
      CrtBranch& cb = c->crt.b[b];
      const uint32_t first = b ? c->L[0] : 0;
      if (c->L[b] > (uint32_t)kMaxBranchPrimes) raise(HEI_PARAM_ERROR, "too many primes in one branch");
      cb.L = c->L[b];
      cb.t = (uint32_t)c->t[b];
      auto mul_small = [](uint32_t (&a)[kLimbs], uint64_t m) {
        uint64_t carry = 0;
        for (int k = 0; k < kLimbs; ++k) {
          const u128 v = (u128)a[k] * m + carry;
          a[k] = (uint32_t)v;
          carry = (uint64_t)(v >> 32);
        }
        if (carry) raise(HEI_PARAM_ERROR, "ciphertext modulus too wide for the device CRT");
      };
      std::fill(cb.Q, cb.Q + kLimbs, 0u);
      cb.Q[0] = 1;
      for (uint32_t i = 0; i < cb.L; ++i) mul_small(cb.Q, d->q[first + i]);
      for (uint32_t i = 0; i < cb.L; ++i) {
        cb.q[i] = (uint32_t)d->q[first + i];
        std::fill(cb.Qp[i], cb.Qp[i] + kLimbs, 0u);
        cb.Qp[i][0] = 1;
        uint64_t pm = 1;
        for (uint32_t k = 0; k < cb.L; ++k)
          if (k != i) {
            mul_small(cb.Qp[i], d->q[first + k]);
            pm = mulmod(pm, d->q[first + k] % d->q[first + i], d->q[first + i]);
          }
        cb.y[i] = (uint32_t)invmod(pm, d->q[first + i]);
      }
      for (int k = 0; k < kLimbs; ++k) cb.Qh[k] = (cb.Q[k] >> 1) | (k + 1 < kLimbs ? (cb.Q[k + 1] << 31) : 0u);
      cb.q_msb = -1;
      for (int k = kLimbs - 1; k >= 0 && cb.q_msb < 0; --k)
        if (cb.Q[k]) cb.q_msb = 32 * k + 31 - __builtin_clz(cb.Q[k]);
      if (cb.q_msb > 32 * kLimbs - 34) raise(HEI_PARAM_ERROR, "ciphertext modulus too wide for the device CRT");
      cb.Qd = 0.0;
      for (int k = kLimbs - 1; k >= 0; --k) cb.Qd = cb.Qd * 4294967296.0 + (double)cb.Q[k];
    }
    c->t0inv = (uint32_t)invmod(c->t[0] % c->t[1], c->t[1]);
    // fold elements and their eval permutations (poly.cpp:124-138)
    for (uint32_t s = 1; s <= n / 4; s <<= 1) c->fold_elts.push_back(powmod(3, s, two_n));
    c->fold_elts.push_back(two_n - 1);
    std::vector<uint32_t> perms(c->fold_elts.size() * (size_t)n);
    for (size_t e = 0; e < c->fold_elts.size(); ++e) {
      const uint64_t gel = c->fold_elts[e];
      c->perm_index[gel] = (uint32_t)e;
      for (uint32_t i = 0; i < n; ++i) {
        const uint64_t ex = 2ull * rev_bits(i, c->logn) + 1, src = (ex * gel) % two_n;
        perms[e * n + i] = rev_bits((uint32_t)((src - 1) / 2), c->logn);
      }
    }
    // pass-C twiddles for the register-blocked transforms (ntt_fast.cuh)
    std::vector<uint4> twc, itwc;
    if (c->logn == 13 || c->logn == 14) {
      const uint32_t T = n / 16, XST = c->logn - 12, PAD = XST % 2 == 0 ? 1 : 0, KC = (PAD + XST + 16) / 2;
      g.twc_stride = KC * T;
      twc.resize((size_t)(P + 2) * KC * T);
      itwc.resize(twc.size());
      std::vector<uint32_t> idx(2 * KC);
      for (uint32_t row = 0; row < P + 2; ++row)
        for (uint32_t j = 0; j < T; ++j) {
          const uint32_t x0 = 16 * j;
          std::fill(idx.begin(), idx.end(), 0u);
          uint32_t e = PAD;
          for (uint32_t s = 0; s < XST; ++s) idx[e++] = (1u << (8 + s)) + (x0 >> (c->logn - 8 - s));
          for (uint32_t s = 0; s < 4; ++s)
            for (uint32_t b = 0; b < (1u << s); ++b) idx[e++] = (1u << (c->logn - 4 + s)) + (x0 >> (4 - s)) + b;
          for (uint32_t k = 0; k < KC; ++k) {
            const uint2 a = fwd[(size_t)row * n + idx[2 * k]], b = fwd[(size_t)row * n + idx[2 * k + 1]];
            const uint2 ia = inv[(size_t)row * n + idx[2 * k]], ib = inv[(size_t)row * n + idx[2 * k + 1]];
            twc[((size_t)row * KC + k) * T + j] = make_uint4(a.x, a.y, b.x, b.y);
            itwc[((size_t)row * KC + k) * T + j] = make_uint4(ia.x, ia.y, ib.x, ib.y);
          }
        }
    }
    // N = 16384 half-ring tables (ks_half.cuh): half h's stage s' block i'
    // uses zetas[2^(s'+1) + h 2^s' + i'], stored at local index 2^s' + i'
    std::vector<uint4> twch, itwch;
    if (c->logn == 14) {
      const uint32_t hl = c->logn - 1, nh = n / 2, T = nh / 16, XST = hl - 12, PAD = XST % 2 == 0 ? 1 : 0,
                     KC = (PAD + XST + 16) / 2;  // Ntt<hl>'s pass-C layout
      g.twch_stride = KC * T;
      c->h_fwdh.assign((size_t)P * 2 * nh, make_uint2(0, 0));
      c->h_invh.assign((size_t)P * 2 * nh, make_uint2(0, 0));
      twch.resize((size_t)P * 2 * KC * T);
      itwch.resize(twch.size());
      std::vector<uint32_t> idx(2 * KC);
      for (uint32_t row = 0; row < P; ++row)
        for (uint32_t h = 0; h < 2; ++h) {
          uint2* loc = c->h_fwdh.data() + ((size_t)row * 2 + h) * nh;
          uint2* iloc = c->h_invh.data() + ((size_t)row * 2 + h) * nh;
          for (uint32_t k = 1; k < nh; ++k) {
            const uint32_t m = 1u << (31 - __builtin_clz(k));
            loc[k] = fwd[(size_t)row * n + 2 * m + h * m + (k - m)];
            iloc[k] = inv[(size_t)row * n + 2 * m + h * m + (k - m)];
          }
          for (uint32_t j = 0; j < T; ++j) {
            const uint32_t x0 = 16 * j;
            std::fill(idx.begin(), idx.end(), 0u);
            uint32_t e = PAD;
            for (uint32_t st = 0; st < XST; ++st) idx[e++] = (1u << (8 + st)) + (x0 >> (hl - 8 - st));
            for (uint32_t st = 0; st < 4; ++st)
              for (uint32_t b2 = 0; b2 < (1u << st); ++b2) idx[e++] = (1u << (hl - 4 + st)) + (x0 >> (4 - st)) + b2;
            for (uint32_t k = 0; k < KC; ++k) {
              const uint2 a = loc[idx[2 * k]], b2 = loc[idx[2 * k + 1]];
              twch[(((size_t)row * 2 + h) * KC + k) * T + j] = make_uint4(a.x, a.y, b2.x, b2.y);
              const uint2 ia = iloc[idx[2 * k]], ib = iloc[idx[2 * k + 1]];
              itwch[(((size_t)row * 2 + h) * KC + k) * T + j] = make_uint4(ia.x, ia.y, ib.x, ib.y);
            }
          }
        }
    }
    set_device(c.get());
    CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    if (!twch.empty()) {
      CU(cudaMalloc(&c->d_twch, twch.size() * sizeof(uint4)));
      CU(cudaMalloc(&c->d_fwdh, c->h_fwdh.size() * sizeof(uint2)));
      CU(cudaMemcpyAsync(c->d_twch, twch.data(), twch.size() * sizeof(uint4), cudaMemcpyHostToDevice, c->stream));
      CU(cudaMemcpyAsync(c->d_fwdh, c->h_fwdh.data(), c->h_fwdh.size() * sizeof(uint2), cudaMemcpyHostToDevice,
                         c->stream));
      CU(cudaStreamSynchronize(c->stream));
      g.twch = c->d_twch;
      g.fwdh = c->d_fwdh;
      CU(cudaMalloc(&c->d_itwch, itwch.size() * sizeof(uint4)));
      CU(cudaMalloc(&c->d_invh, c->h_invh.size() * sizeof(uint2)));
      CU(cudaMemcpyAsync(c->d_itwch, itwch.data(), itwch.size() * sizeof(uint4), cudaMemcpyHostToDevice, c->stream));
      CU(cudaMemcpyAsync(c->d_invh, c->h_invh.data(), c->h_invh.size() * sizeof(uint2), cudaMemcpyHostToDevice,
                         c->stream));
      CU(cudaStreamSynchronize(c->stream));
      g.itwch = c->d_itwch;
      g.invh = c->d_invh;
    }
    if (!twc.empty()) {
      CU(cudaMalloc(&c->d_twc, twc.size() * sizeof(uint4)));
      CU(cudaMalloc(&c->d_itwc, itwc.size() * sizeof(uint4)));
      CU(cudaMemcpyAsync(c->d_twc, twc.data(), twc.size() * sizeof(uint4), cudaMemcpyHostToDevice, c->stream));
      CU(cudaStreamSynchronize(c->stream));
      CU(cudaMemcpyAsync(c->d_itwc, itwc.data(), itwc.size() * sizeof(uint4), cudaMemcpyHostToDevice, c->stream));
      CU(cudaStreamSynchronize(c->stream));
      g.twc = c->d_twc;
      g.itwc = c->d_itwc;
    }
    CU(cudaMalloc(&c->d_fwd, fwd.size() * sizeof(uint2)));
    CU(cudaMalloc(&c->d_inv, inv.size() * sizeof(uint2)));
    CU(cudaMalloc(&c->d_index, n * 4));
    CU(cudaMalloc(&c->d_perms, perms.size() * 4));
    CU(cudaMalloc(&c->d_err, 4));
    CU(cudaMemcpyAsync(c->d_fwd, fwd.data(), fwd.size() * sizeof(uint2), cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    c->h_fwd = fwd;
    c->h_inv = inv;
    CU(cudaMemcpyAsync(c->d_inv, inv.data(), inv.size() * sizeof(uint2), cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaMemcpyAsync(c->d_index, index_map.data(), n * 4, cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaMemcpyAsync(c->d_perms, perms.data(), perms.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaMemsetAsync(c->d_err, 0, 4, c->stream));
    CU(cudaMalloc(&c->d_ops, 6 * 8));
    c->d_opsnap = c->d_ops + 3;
    CU(cudaMemsetAsync(c->d_ops, 0, 6 * 8, c->stream));
    CU(cudaHostAlloc(&c->h_opsnap, 6 * 8, cudaHostAllocMapped));  // written by k_finish_add (UVA)
    CU(cudaStreamSynchronize(c->stream));
    g.ops = c->d_ops;
    g.fwd = c->d_fwd;
    g.inv = c->d_inv;
    g.index_map = c->d_index;
    const size_t s3 = smem_bytes(c.get(), 3);
    set_smem_attr((const void*)k_rot_keyswitch, s3);
    set_smem_attr((const void*)k_rot_digits, smem_bytes(c.get(), 1));
    set_smem_attr((const void*)k_mask_acc, smem_bytes(c.get(), 1));
    set_smem_attr((const void*)k_bias_plain, smem_bytes(c.get(), 1));
    set_smem_attr((const void*)k_ct_ntt, smem_bytes(c.get(), 1));
    set_smem_attr((const void*)k_poly_ntt, smem_bytes(c.get(), 1));
    set_smem_attr((const void*)k_encode_weights, smem_bytes(c.get(), 1));
    set_smem_attr((const void*)k_bl_finish_lin, 3 * (size_t)c->n * 4);
    set_smem_attr((const void*)k_bl_encode_g, smem_bytes(c.get(), 1));
    set_smem_attr((const void*)k_bl_encrypt_g, smem_bytes(c.get(), 1));
    set_smem_attr((const void*)k_prepare_pk_g, smem_bytes(c.get(), 1));
    set_smem_attr((const void*)k_dec_phase, smem_bytes(c.get(), 1));
    set_smem_attr((const void*)k_dec_decode, smem_bytes(c.get(), 1));
    set_smem_attr((const void*)k_prepare_sk, smem_bytes(c.get(), 1));
    set_smem_attr((const void*)k_kg_pk, smem_bytes(c.get(), 1));
    set_smem_attr((const void*)k_kg_gk, smem_bytes(c.get(), 1));
    if (c->logn == 13) set_fast_attrs<13>(smem_bytes(c.get(), 1));
    if (c->logn == 14) set_fast_attrs<14>(smem_bytes(c.get(), 1));
    *out = c.release();
  });
}

void hei_gpu_ctx_destroy(hei_gpu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaFree(c->d_fwd);
  cudaFree(c->d_inv);
  cudaFree(c->d_twc);
  cudaFree(c->d_twch);
  cudaFree(c->d_fwdh);
  cudaFree(c->d_itwch);
  cudaFree(c->d_invh);
  cudaFree(c->d_itwc);
  cudaFree(c->d_mask_table);
  cudaFree(c->d_index);
  cudaFree(c->d_perms);
  cudaFree(c->d_err);
  cudaFree(c->d_ops);
  if (c->h_opsnap) cudaFreeHost(c->h_opsnap);
  for (int b = 0; b < 2; ++b) {
    cudaFree(c->d_keys[b]);
    cudaFree(c->d_pk[b]);
  }
  cudaFree(c->d_pkp);
  cudaFree(c->d_sk_hat);
  cudaFree(c->pool_acc);
  cudaFree(c->pool_rows);
  cudaFree(c->pool_bias);
  cudaFree(c->pool_stage64);
  if (c->pinned_bias) cudaFreeHost(c->pinned_bias);
  if (c->pinned_out) cudaFreeHost(c->pinned_out);
  cudaFree(c->pool_in32);
  cudaFree(c->pool_out);
  cudaFree(c->pool_out64);
  cudaFree(c->pool_biasp);
  cudaFree(c->pool_masks);
  for (int k = 0; k < 24; ++k) cudaFree(c->named_pool[k]);
  if (c->bias_stream) cudaStreamDestroy(c->bias_stream);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  for (cudaStream_t ps : c->part_streams) cudaStreamDestroy(ps);
  for (cudaStream_t ps : c->chunk_streams) cudaStreamDestroy(ps);
  cudaFree(c->d_dotA);
  cudaFree(c->d_dotB);
  cudaFree(c->d_dig);
  cudaFree(c->d_dig2);
  for (auto& a : c->fold_ev)
    for (auto e : a) cudaEventDestroy(e);
  for (auto& fg : c->fold_graphs) cudaGraphExecDestroy(fg.exec);
  if (c->side_stream) cudaStreamDestroy(c->side_stream);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

void hei_gpu_set_batch_pairs(hei_gpu_ctx* c, uint64_t pairs) { c->batch_pairs = pairs; }

int hei_gpu_kernel_timing(hei_gpu_ctx* c, int enable) {
  return guarded([&] {
    set_device(c);
    std::lock_guard<std::mutex> lk(c->mu);
    for (auto& a : c->fold_ev)
      for (auto e : a) cudaEventDestroy(e);
    c->fold_ev.clear();
    c->timing = enable != 0;
  });
}

// which: 0 = key switch, 1 = digits.
int hei_gpu_kernel_stats(hei_gpu_ctx* c, int which, uint64_t* launches, double* total_ms) {
  return guarded([&] {
    set_device(c);
    std::lock_guard<std::mutex> lk(c->mu);
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaDeviceSynchronize());
    double tot = 0;
    for (const auto& a : c->fold_ev) {
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, which == 0 ? a[1] : a[0], which == 0 ? a[2] : a[1]));
      tot += ms;
    }
    *launches = c->fold_ev.size();
    *total_ms = tot;
  });
}

int hei_gpu_measure_butterfly_peak(int device, double* bfly_per_s) {
  return guarded([&] {
    CU(cudaSetDevice(device));
    int sms = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const uint32_t q = 2147352577u, w = 123456789u;
    const uint32_t ws = (uint32_t)(((uint64_t)w << 32) / q);
    const unsigned blocks = (unsigned)sms * 8, threads = 256;
    const uint32_t iters = 4096;
    uint32_t* sink = nullptr;
    CU(cudaMalloc(&sink, blocks * 4));
    cudaEvent_t a, b;
    CU(cudaEventCreate(&a));
    CU(cudaEventCreate(&b));
    k_bfly_peak<<<blocks, threads>>>(sink, 64, q, w, ws);  // warm-up
    LAUNCHED();
    CU(cudaEventRecord(a));
    for (int r = 0; r < 5; ++r) k_bfly_peak<<<blocks, threads>>>(sink, iters, q, w, ws);
    LAUNCHED();
    CU(cudaEventRecord(b));
    CU(cudaEventSynchronize(b));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    *bfly_per_s = 5.0 * blocks * threads * 8.0 * iters / (ms * 1e-3);
  });
}

// Galois key rows [elt][l][part][i][N] u64 already on the device -> the
// key-switch layout (k_prepare_keys), installed as branch b's key set.
void install_galois_keys(hei_gpu_ctx* c, uint32_t b, uint32_t count, const uint64_t* elts, const uint64_t* d_raw) {
  if (b > 1) raise(HEI_PARAM_ERROR, "branch out of range");
  if (count == 0 || count > kMaxElts) raise(HEI_KEY_ERROR, "galois key set size out of range");
  const uint32_t L = c->L[b];
  const uint64_t words = (uint64_t)count * L * 2 * L * c->n;
  std::map<uint64_t, uint32_t> idx;
  for (uint32_t e = 0; e < count; ++e) {
    if (!(elts[e] & 1) || elts[e] >= 2ull * c->n) raise(HEI_KEY_ERROR, "invalid galois element");
    idx[elts[e]] = e;
  }
  if (c->d_keys[b]) cudaFree(c->d_keys[b]);
  c->d_keys[b] = nullptr;
  CU(cudaMalloc(&c->d_keys[b], words * sizeof(uint2)));
  k_prepare_keys<<<grid_for(words, 256), 256, 0, c->stream>>>(c->geo, b, count, d_raw, c->d_keys[b], c->d_err);
  LAUNCHED();
  c->keys_words[b] = words;
  CU(cudaStreamSynchronize(c->stream));
  check_err_flag(c, HEI_CODEC_ERROR, "galois keys: coefficient not reduced");
  c->key_index[b] = idx;
  c->has_keys[b] = true;
  ++c->graph_gen;
}

int hei_gpu_upload_galois_keys(hei_gpu_ctx* c, uint32_t b, uint32_t count, const uint64_t* elts,
                               const uint64_t* rows) {
  return guarded([&] {
    if (b > 1) raise(HEI_PARAM_ERROR, "branch out of range");
    if (count == 0 || count > kMaxElts) raise(HEI_KEY_ERROR, "galois key set size out of range");
    set_device(c);
    const uint64_t words = (uint64_t)count * c->L[b] * 2 * c->L[b] * c->n;
    uint64_t* d_raw = nullptr;
    CU(cudaMalloc(&d_raw, words * 8));
    CU(cudaMemcpyAsync(d_raw, rows, words * 8, cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    try {
      install_galois_keys(c, b, count, elts, d_raw);
    } catch (...) {
      cudaFree(d_raw);
      throw;
    }
    cudaFree(d_raw);
  });
}

// Test seam for k_kg_plan: resolve uniform_u64 rejection sampling over a
// given raw stream for a list of (kind, count, bound) segments (kind 0
// uniform, 1 ternary, 2 gaussian start only). out32/out8 receive the values
// in segment order; used = draws consumed; returns HEI_RANGE_ERROR if the
// stream is too short.
int hei_gpu_debug_rejection_plan(hei_gpu_ctx* c, const uint64_t* raw, uint64_t avail, const uint32_t* kinds,
                                 const uint32_t* counts, const uint64_t* bounds, uint32_t nseg, uint32_t* out32,
                                 int8_t* out8, uint64_t* gpos, uint64_t* used) {
  return guarded([&] {
    set_device(c);
    std::lock_guard<std::mutex> lk(c->mu);
    std::vector<KgSeg> segs(nseg);
    uint64_t o32 = 0, o8 = 0;
    for (uint32_t i = 0; i < nseg; ++i) {
      segs[i].kind = kinds[i];
      segs[i].n = counts[i];
      segs[i].bound = bounds[i];
      segs[i].limit = bounds[i] ? bounds[i] * (UINT64_MAX / bounds[i]) : 0;
      if (kinds[i] == 0) segs[i].out = o32, o32 += counts[i];
      else segs[i].out = o8, o8 += counts[i];
    }
    KgSeg* d_segs;
    uint64_t *d_raw, *d_gpos, *d_used;
    uint32_t* d32;
    int8_t* d8;
    CU(cudaMalloc(&d_segs, nseg * sizeof(KgSeg) + 8));
    CU(cudaMalloc(&d_raw, avail * 8 + 8));
    CU(cudaMalloc(&d_gpos, nseg * 8 + 8));
    CU(cudaMalloc(&d_used, 8));
    CU(cudaMalloc(&d32, o32 * 4 + 4));
    CU(cudaMalloc(&d8, o8 + 1));
    CU(cudaMemcpyAsync(d_segs, segs.data(), nseg * sizeof(KgSeg), cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaMemcpyAsync(d_raw, raw, avail * 8, cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaMemsetAsync(c->d_err, 0, 4, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    k_kg_plan<<<1, 1024, 0, c->stream>>>(d_raw, avail, d_segs, nseg, d32, d8, d_gpos, d_used, c->d_err);
    LAUNCHED();
    CU(cudaStreamSynchronize(c->stream));
    uint32_t err = 0;
    CU(cudaMemcpyAsync(&err, c->d_err, 4, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaMemsetAsync(c->d_err, 0, 4, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaMemcpyAsync(used, d_used, 8, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    if (out32 && o32) CU(cudaMemcpy(out32, d32, o32 * 4, cudaMemcpyDeviceToHost));
    if (out8 && o8) CU(cudaMemcpy(out8, d8, o8, cudaMemcpyDeviceToHost));
    if (gpos) CU(cudaMemcpy(gpos, d_gpos, nseg * 8, cudaMemcpyDeviceToHost));
    for (void* v : {(void*)d_segs, (void*)d_raw, (void*)d_gpos, (void*)d_used, (void*)d32, (void*)d8}) cudaFree(v);
    if (err & 4) raise(HEI_RANGE_ERROR, "rejection plan: raw stream too short");
  });
}

// TwinContext::keygen (twin.cpp:41-48) on the device; see keygen.cuh.
int hei_gpu_keygen(hei_gpu_ctx* c, hei_gpu_prng* rng, int install, int8_t* sk, uint64_t* pk, uint64_t* elts_out,
                   uint64_t* gk0, uint64_t* gk1) {
  return guarded([&] {
    if (!rng) raise(HEI_PARAM_ERROR, "keygen: rng required");
    if (rng->have_spare) raise(HEI_PARAM_ERROR, "keygen: rng holds a cached Box-Muller spare; cannot replay on the device");
    set_device(c);
    std::lock_guard<std::mutex> lk(c->mu);
    cudaStream_t st = c->stream;
    const uint32_t n = c->n, P = c->P();
    const std::vector<uint64_t>& gen = c->fold_elts;  // galois_steps() order, then the swap (context.cpp:179-212)
    const uint32_t ne = (uint32_t)gen.size();
    std::vector<uint64_t> asc(gen);
    std::sort(asc.begin(), asc.end());
    std::vector<uint32_t> slot(ne);
    for (uint32_t e = 0; e < ne; ++e) slot[e] = (uint32_t)(std::lower_bound(asc.begin(), asc.end(), gen[e]) - asc.begin());
    // draw plan, in the reference's order
    std::vector<KgSeg> segs;
    uint64_t off8 = 0, off32 = 0, D = 0;
    uint64_t s8[2], e8[2], a32[2], ge8[2], ga32[2];
    auto add = [&](uint32_t kind, uint64_t bound) {
      KgSeg g{};
      g.kind = kind;
      g.n = n;
      g.bound = bound;
      g.limit = bound ? bound * (UINT64_MAX / bound) : 0;
      if (kind == 0) g.out = off32, off32 += n;
      else g.out = off8, off8 += n;
      D += n;
      segs.push_back(g);
    };
    for (uint32_t b = 0; b < 2; ++b) {
      const uint32_t first = b ? c->L[0] : 0, L = c->L[b];
      s8[b] = off8;
      add(1, 3);  // sample_ternary
      e8[b] = off8;
      add(2, 0);  // sample_gaussian
      a32[b] = off32;
      for (uint32_t i = 0; i < L; ++i) add(0, c->q[first + i]);  // sample_uniform per prime
      ge8[b] = off8;
      ga32[b] = off32;
      for (uint32_t e = 0; e < ne; ++e)
        for (uint32_t l = 0; l < L; ++l) {
          add(2, 0);
          for (uint32_t i = 0; i < L; ++i) add(0, c->q[first + i]);
        }
    }
    struct Free {
      std::vector<void*> p;
      ~Free() {
        for (void* v : p) cudaFree(v);
      }
    } fr;
    auto alloc = [&](auto** ptr, size_t bytes) {
      CU(cudaMalloc((void**)ptr, bytes));
      fr.p.push_back((void*)*ptr);
    };
    KgSeg* d_segs;
    uint32_t* d_out32;
    int8_t* d_out8;
    uint64_t *d_gpos, *d_used, *d_state, *d_elts;
    uint32_t *d_slot, *d_shat;
    alloc(&d_segs, segs.size() * sizeof(KgSeg));
    alloc(&d_out32, off32 * 4);
    alloc(&d_out8, off8);
    alloc(&d_gpos, segs.size() * 8);
    alloc(&d_used, 8);
    alloc(&d_state, 313 * 8);
    alloc(&d_elts, ne * 8);
    alloc(&d_slot, ne * 4);
    alloc(&d_shat, (size_t)P * n * 4);
    CU(cudaMemcpyAsync(d_segs, segs.data(), segs.size() * sizeof(KgSeg), cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(d_elts, gen.data(), ne * 8, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(d_slot, slot.data(), ne * 4, cudaMemcpyHostToDevice, st));
    uint64_t hstate[313];
    std::memcpy(hstate, rng->mt, 312 * 8);
    hstate[312] = rng->mti;
    // replay + plan; a rejected draw needs a longer stream (rare): retry
    uint64_t avail = D, used = 0;
    uint64_t* d_raw = nullptr;
    for (int attempt = 0;; ++attempt) {
      if (d_raw) cudaFree(d_raw);
      CU(cudaMalloc(&d_raw, avail * 8));
      CU(cudaMemcpyAsync(d_state, hstate, sizeof(hstate), cudaMemcpyHostToDevice, st));
      heb_baseline::k_mt_generate<<<1, 320, 0, st>>>(d_state, d_raw, avail);
      LAUNCHED();
      CU(cudaMemsetAsync(c->d_err, 0, 4, st));
      k_kg_plan<<<1, 1024, 0, st>>>(d_raw, avail, d_segs, (uint32_t)segs.size(), d_out32, d_out8, d_gpos, d_used,
                                     c->d_err);
      LAUNCHED();
      uint32_t err = 0;
      CU(cudaMemcpyAsync(&err, c->d_err, 4, cudaMemcpyDeviceToHost, st));
      CU(cudaMemcpyAsync(&used, d_used, 8, cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      if (err & 2) {
        CU(cudaMemsetAsync(c->d_err, 0, 4, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        cudaFree(d_raw);
        raise(HEI_INTERNAL, "keygen: Box-Muller u1 == 0 rejection (probability 2^-53) is not replayed on the device");
      }
      if (err & 4) {
        if (attempt > 8) {
          cudaFree(d_raw);
          raise(HEI_INTERNAL, "keygen: rejection sampling ran past the replayed stream");
        }
        avail += 4096;
        continue;
      }
      if (used != avail) {  // consumed fewer than generated: regenerate exactly `used` for the rng state
        avail = used;
        continue;
      }
      break;
    }
    fr.p.push_back(d_raw);
    k_kg_gauss<<<(unsigned)segs.size(), 256, 0, st>>>(d_raw, d_segs, d_gpos, d_out8);
    LAUNCHED();
    const size_t sm1 = smem_bytes(c, 1);
    uint64_t *d_pk, *d_gk[2];
    alloc(&d_pk, c->ct_words() / 2 * 8 * 2);  // [branch][part][L_b][n]
    for (uint32_t b = 0; b < 2; ++b) {
      const uint32_t L = c->L[b];
      alloc(&d_gk[b], (size_t)ne * L * 2 * L * n * 8);
      k_prepare_sk<<<L, c->threads(), sm1, st>>>(c->geo, b, d_out8 + s8[b], d_shat);
      LAUNCHED();
      uint64_t* pkb = d_pk + (b ? 2ull * c->L[0] * n : 0);
      k_kg_pk<<<L, c->threads(), sm1, st>>>(c->geo, b, d_out8 + e8[b], d_out32 + a32[b], d_shat, pkb);
      LAUNCHED();
      k_kg_gk<<<ne * L * L, c->threads(), sm1, st>>>(c->geo, b, d_elts, d_slot, d_out8 + s8[b], d_out8 + ge8[b],
                                                     d_out32 + ga32[b], d_shat, d_gk[b]);
      LAUNCHED();
    }
    CU(cudaMemcpyAsync(hstate, d_state, sizeof(hstate), cudaMemcpyDeviceToHost, st));
    if (sk)
      for (uint32_t b = 0; b < 2; ++b) CU(cudaMemcpyAsync(sk + (size_t)b * n, d_out8 + s8[b], n, cudaMemcpyDeviceToHost, st));
    if (pk) CU(cudaMemcpyAsync(pk, d_pk, c->ct_words() * 8, cudaMemcpyDeviceToHost, st));
    if (gk0) CU(cudaMemcpyAsync(gk0, d_gk[0], (size_t)ne * c->L[0] * 2 * c->L[0] * n * 8, cudaMemcpyDeviceToHost, st));
    if (gk1) CU(cudaMemcpyAsync(gk1, d_gk[1], (size_t)ne * c->L[1] * 2 * c->L[1] * n * 8, cudaMemcpyDeviceToHost, st));
    if (elts_out) std::memcpy(elts_out, asc.data(), ne * 8);
    CU(cudaStreamSynchronize(st));
    std::memcpy(rng->mt, hstate, 312 * 8);
    rng->mti = (uint32_t)hstate[312];
    if (install) {
      for (uint32_t b = 0; b < 2; ++b) {
        install_galois_keys(c, b, ne, asc.data(), d_gk[b]);
        const size_t words = 2ull * c->L[b] * n;
        if (!c->d_pk[b]) CU(cudaMalloc(&c->d_pk[b], words * 8));
        CU(cudaMemcpyAsync(c->d_pk[b], d_pk + (b ? 2ull * c->L[0] * n : 0), words * 8, cudaMemcpyDeviceToDevice, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        if (!c->d_sk_hat) CU(cudaMalloc(&c->d_sk_hat, (size_t)P * n * 4));
        k_prepare_sk<<<c->L[b], c->threads(), sm1, st>>>(c->geo, b, d_out8 + s8[b], c->d_sk_hat);
        LAUNCHED();
        c->has_sk[b] = true;
      }
      if (c->d_pkp) {
        cudaFree(c->d_pkp);
        c->d_pkp = nullptr;
      }
      CU(cudaStreamSynchronize(st));
    }
  });
}

int hei_gpu_upload_public_key(hei_gpu_ctx* c, uint32_t b, const uint64_t* pk) {
  return guarded([&] {
    if (b > 1) raise(HEI_PARAM_ERROR, "branch out of range");
    set_device(c);
    const size_t words = 2ull * c->L[b] * c->n;
    if (!c->d_pk[b]) CU(cudaMalloc(&c->d_pk[b], words * 8));
    if (c->d_pkp) {
      cudaFree(c->d_pkp);
      c->d_pkp = nullptr;
    }
    CU(cudaMemcpyAsync(c->d_pk[b], pk, words * 8, cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
  });
}

int hei_gpu_upload_secret_key(hei_gpu_ctx* c, uint32_t b, const int8_t* s) {
  return guarded([&] {
    if (b > 1) raise(HEI_PARAM_ERROR, "branch out of range");
    for (uint32_t x = 0; x < c->n; ++x)
      if (s[x] < -1 || s[x] > 1) raise(HEI_CODEC_ERROR, "secret key residue is not ternary");
    set_device(c);
    if (!c->d_sk_hat) CU(cudaMalloc(&c->d_sk_hat, (size_t)c->P() * c->n * 4));
    int8_t* d_s = nullptr;
    CU(cudaMalloc(&d_s, c->n));
    CU(cudaMemcpyAsync(d_s, s, c->n, cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    k_prepare_sk<<<c->L[b], c->threads(), smem_bytes(c, 1), c->stream>>>(c->geo, b, d_s, c->d_sk_hat);
    LAUNCHED();
    CU(cudaStreamSynchronize(c->stream));
    cudaFree(d_s);
    c->has_sk[b] = true;
  });
}

// decrypt_core + decode_signed over `count` twin ciphertexts already on the
// device (u32, eval form); budgets[ct][2] per branch; `out` on the device.
void decrypt_device(hei_gpu_ctx* c, uint32_t* d_cts, uint64_t count, int mode, uint64_t rows, uint64_t cols,
                    int64_t* d_out, std::vector<int>& budgets, cudaStream_t st) {
  if (!c->has_sk[0] || !c->has_sk[1]) raise(HEI_KEY_ERROR, "decrypt: this backend holds no secret key");
  const uint32_t n = c->n;
  uint32_t *d_w = nullptr, *d_m = nullptr;
  int* d_msb = nullptr;
  CU(cudaMallocAsync(&d_w, count * c->P() * n * 4, st));
  CU(cudaMallocAsync(&d_m, count * 2 * n * 4, st));
  CU(cudaMallocAsync(&d_msb, count * 2 * sizeof(int), st));
  CU(cudaMemsetAsync(d_msb, 0xff, count * 2 * sizeof(int), st));  // -1: all-zero residual
  k_dec_phase<<<(unsigned)(count * c->P()), c->threads(), smem_bytes(c, 1), st>>>(c->geo, d_cts, c->d_sk_hat, d_w);
  LAUNCHED();
  k_dec_crt<<<grid_for(count * 2 * n, 256), 256, 0, st>>>(c->geo, c->crt, d_w, count, d_m, d_msb);
  LAUNCHED();
  k_dec_decode<<<(unsigned)(count * 2), c->threads(), smem_bytes(c, 1), st>>>(c->geo, d_m, d_w);
  LAUNCHED();
  std::vector<int> msb(count * 2);
  CU(cudaMemcpyAsync(msb.data(), d_msb, count * 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  budgets.resize(count * 2);
  for (uint64_t x = 0; x < count * 2; ++x) {
    const int q_msb = c->crt.b[x % 2].q_msb;
    int bud = msb[x] < 0 ? q_msb - 1 : q_msb - (msb[x] + 1);  // msb(max_r << 1)
    budgets[x] = bud < 0 ? 0 : bud;
  }
  if (d_out) {
    k_dec_recombine<<<grid_for(count * n, 256), 256, 0, st>>>(c->geo, d_w, count, rows, cols, mode, c->t0inv, d_out);
    LAUNCHED();
  }
  CU(cudaFreeAsync(d_w, st));
  CU(cudaFreeAsync(d_m, st));
  CU(cudaFreeAsync(d_msb, st));
}

// Host twin ciphertexts (u64, `form`) -> device u32 eval form.
uint32_t* stage_cts(hei_gpu_ctx* c, const uint64_t* cts, int form, uint64_t count, cudaStream_t st) {
  if (form != HEI_FORM_EVAL && form != HEI_FORM_COEFF) raise(HEI_PARAM_ERROR, "decrypt: unknown form");
  const size_t words = count * c->ct_words();
  uint64_t* d64 = nullptr;
  uint32_t* d32 = nullptr;
  CU(cudaMallocAsync(&d64, words * 8, st));
  CU(cudaMallocAsync(&d32, words * 4, st));
  CU(cudaMemcpyAsync(d64, cts, words * 8, cudaMemcpyHostToDevice, st));
  k_narrow<<<grid_for(words, 256), 256, 0, st>>>(c->geo, d64, d32, count, c->d_err);
  LAUNCHED();
  if (form == HEI_FORM_COEFF) launch_ct_ntt(c, (unsigned)(count * 2 * c->P()), d32, st);
  CU(cudaFreeAsync(d64, st));
  CU(cudaStreamSynchronize(st));
  uint32_t h = 0;
  CU(cudaMemcpyAsync(&h, c->d_err, 4, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (h) {
    CU(cudaMemsetAsync(c->d_err, 0, 4, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    cudaFree(d32);
    raise(HEI_CODEC_ERROR, "decrypt: coefficient not reduced");
  }
  return d32;
}

void decrypt_host(hei_gpu_ctx* c, const uint64_t* cts, int form, uint64_t count, int mode, uint64_t rows,
                  uint64_t cols, int64_t* out, size_t out_words, int* budgets, bool throw_noise) {
  set_device(c);
  std::lock_guard<std::mutex> lk(c->mu);
  if (!c->has_sk[0] || !c->has_sk[1]) raise(HEI_KEY_ERROR, "decrypt: this backend holds no secret key");
  cudaStream_t st = c->stream;
  uint32_t* d32 = stage_cts(c, cts, form, count, st);
  int64_t* d_out = nullptr;
  if (out) CU(cudaMallocAsync(&d_out, out_words * 8, st));
  std::vector<int> bud;
  try {
    decrypt_device(c, d32, count, mode, rows, cols, d_out, bud, st);
  } catch (...) {
    cudaFree(d32);
    if (d_out) cudaFree(d_out);
    throw;
  }
  if (out) CU(cudaMemcpyAsync(out, d_out, out_words * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  cudaFree(d32);
  if (d_out) cudaFree(d_out);
  if (budgets)
    for (uint64_t x = 0; x < count; ++x) budgets[x] = std::min(bud[2 * x], bud[2 * x + 1]);
  if (throw_noise)  // BfvContext::decrypt (context.cpp:372-377), branch 0 first
    for (uint64_t x = 0; x < 2 * count; ++x)
      if (bud[x] <= 0) raise(HEI_NOISE_ERROR, "decrypt: invariant noise budget exhausted");
}

int hei_gpu_decrypt_signed(hei_gpu_ctx* c, const uint64_t* cts, int form, uint64_t count, int64_t* out) {
  return guarded([&] { decrypt_host(c, cts, form, count, 2, 0, 0, out, count * c->n, nullptr, true); });
}

int hei_gpu_noise_budget(hei_gpu_ctx* c, const uint64_t* cts, int form, uint64_t count, int* budgets) {
  return guarded([&] { decrypt_host(c, cts, form, count, 2, 0, 0, nullptr, 0, budgets, false); });
}

int hei_gpu_unpack_results(hei_gpu_ctx* c, const uint64_t* packed, uint64_t count, uint64_t rows, uint64_t cols,
                           int64_t* out) {
  return guarded([&] {
    if (rows == 0 || cols == 0) raise(HEI_PARAM_ERROR, "unpack: empty result");
    if (count != (rows * cols + c->n - 1) / c->n) raise(HEI_PARAM_ERROR, "unpack: ciphertext count does not match layout");
    decrypt_host(c, packed, HEI_FORM_EVAL, count, 0, rows, cols, out, rows * cols, nullptr, true);
  });
}

int hei_gpu_unpack_baseline(hei_gpu_ctx* c, const uint64_t* blocks, uint64_t rows, uint64_t cols, int64_t* out) {
  return guarded([&] {
    if (rows == 0 || cols == 0) raise(HEI_PARAM_ERROR, "unpack: empty result");
    const uint64_t nb = (rows + c->n - 1) / c->n;
    decrypt_host(c, blocks, HEI_FORM_EVAL, nb * cols, 1, rows, cols, out, rows * cols, nullptr, true);
  });
}

int hei_gpu_weights_create(hei_gpu_ctx* c, const uint64_t* prepared, uint64_t f, uint64_t cols,
                           hei_gpu_weights** out) {
  return guarded([&] {
    set_device(c);
    std::unique_ptr<hei_gpu_weights> w(weights_alloc(c, f, cols));
    const uint64_t count = cols * w->kc, words = count * c->pt_words();
    uint64_t* d_raw = nullptr;
    CU(cudaMalloc(&d_raw, words * 8));
    CU(cudaMemcpyAsync(d_raw, prepared, words * 8, cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    k_prepare_plain<<<grid_for(words, 256), 256, 0, c->stream>>>(c->geo, d_raw, count, w->d_w, c->d_err);
    LAUNCHED();
    CU(cudaStreamSynchronize(c->stream));
    cudaFree(d_raw);
    check_err_flag(c, HEI_CODEC_ERROR, "weights: coefficient not reduced");
    *out = w.release();
  });
}

int hei_gpu_weights_encode(hei_gpu_ctx* c, const int64_t* wm, uint64_t f, uint64_t cols, hei_gpu_weights** out) {
  return guarded([&] {
    set_device(c);
    const int64_t lim = (int64_t)(((u128)c->t[0] * c->t[1] - 1) / 2);
    for (uint64_t x = 0; x < f * cols; ++x)
      if (wm[x] > lim || wm[x] < -lim) raise(HEI_RANGE_ERROR, "encode_signed: value outside the centered range");
    std::unique_ptr<hei_gpu_weights> w(weights_alloc(c, f, cols));
    int64_t* d_w = nullptr;
    CU(cudaMalloc(&d_w, f * cols * 8));
    CU(cudaMemcpyAsync(d_w, wm, f * cols * 8, cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    k_encode_weights<<<(unsigned)(cols * w->kc * c->P()), c->threads(), smem_bytes(c, 1), c->stream>>>(
        c->geo, d_w, f, (uint32_t)cols, (uint32_t)w->kc, w->d_w);
    LAUNCHED();
    CU(cudaStreamSynchronize(c->stream));
    cudaFree(d_w);
    *out = w.release();
  });
}

void hei_gpu_weights_destroy(hei_gpu_weights* w) {
  if (!w) return;
  cudaSetDevice(w->ctx->device);
  cudaFree(w->d_w);
  delete w;
}

int hei_gpu_stream_create(hei_gpu_ctx* c, const hei_gpu_weights* w, const int64_t* bias, uint64_t rows,
                          hei_gpu_stream** out) {
  return guarded([&] {
    set_device(c);
    std::lock_guard<std::mutex> lk(c->mu);  // stream_new enqueues on the context stream
    *out = stream_new(c, w, bias, rows);
  });
}

int hei_gpu_stream_push_row(hei_gpu_stream* s, uint64_t row, const uint64_t* chunks, int form) {
  return guarded([&] {
    set_device(s->ctx);
    std::lock_guard<std::mutex> lk(s->ctx->mu);
    stream_push(s, row, chunks, form);
  });
}

int hei_gpu_stream_finish(hei_gpu_stream* s, uint64_t* out, hei_op_counters* cnt) {
  return guarded([&] {
    set_device(s->ctx);
    std::lock_guard<std::mutex> lk(s->ctx->mu);
    stream_finish(s, out, cnt);
  });
}

void hei_gpu_stream_destroy(hei_gpu_stream* s) { stream_free(s); }

// Host-buffer matmul: rows stream to the device in chunks on a copy stream
// (double-buffered staging) while earlier chunks are converted and folded on
// the compute stream, so H2D overlaps the key switching. `wire` selects HECT
// blobs (server.cpp:112-172) instead of flat u64 residues.
struct HostIO {
  const uint64_t* u64 = nullptr;  // flat [row][chunk][twin ct] residues
  int form = HEI_FORM_EVAL;
  const uint8_t* wire = nullptr;  // concatenated HECT blobs [row][chunk][branch]
  WireGeo wg{};
  uint64_t* out64 = nullptr;
  uint8_t* out_wire = nullptr;
};

uint64_t hect_bytes(uint32_t n, uint32_t L) { return kHectHeader + 2ull * L * (1 + 8ull * n); }

// Header checks in the reference's order (serialize.cpp:29-42, 82-84).
void check_hect_header(const uint8_t* h, uint64_t hash) {
  if (std::memcmp(h, "HECT", 4) != 0) raise(HEI_CODEC_ERROR, "not a scheme object (bad magic)");
  uint16_t ver;
  uint64_t hh;
  uint32_t parts;
  std::memcpy(&ver, h + 4, 2);
  std::memcpy(&hh, h + 6, 8);
  std::memcpy(&parts, h + 14, 4);
  if (ver != 1) raise(HEI_CODEC_ERROR, "unsupported object version");
  if (hh != hash) raise(HEI_CODEC_ERROR, "object was produced under different parameters");
  if (h[18] != 5) raise(HEI_CODEC_ERROR, "object kind mismatch");
  if (parts != 2) raise(HEI_CODEC_ERROR, "ciphertext must have two parts");
}

// Result download ending in a stream sync. A pageable destination goes
// through a grow-only pinned staging buffer (one DMA at full PCIe rate, then
// a host copy) instead of the driver's chunked pageable path.
void d2h_result(hei_gpu_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  cudaPointerAttributes a{};
  const bool pinned = cudaPointerGetAttributes(&a, dst) == cudaSuccess && a.type == cudaMemoryTypeHost;
  cudaGetLastError();  // clear a lookup failure on plain host memory
  if (pinned || bytes > ((size_t)256 << 20)) {
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return;
  }
  if (bytes > c->pinned_out_bytes) {
    if (c->pinned_out) cudaFreeHost(c->pinned_out);
    c->pinned_out = nullptr;
    CU(cudaMallocHost(&c->pinned_out, bytes));
    c->pinned_out_bytes = bytes;
  }
  CU(cudaMemcpyAsync(c->pinned_out, src, bytes, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  std::memcpy(dst, c->pinned_out, bytes);
}

void matmul_host(hei_gpu_ctx* c, const hei_gpu_weights* w, const HostIO& io, uint64_t rows, const int64_t* bias,
                 hei_op_counters* cnt) {
  set_device(c);
  std::lock_guard<std::mutex> lk(c->mu);
  std::unique_ptr<hei_gpu_stream, void (*)(hei_gpu_stream*)> s(stream_new(c, w, bias, rows, false), stream_free);
  const bool wire = io.wire != nullptr;
  if (wire)
    for (uint64_t x = 0; x < rows * w->kc; ++x) {
      const uint8_t* t = io.wire + x * (io.wg.blob[0] + io.wg.blob[1]);
      check_hect_header(t, io.wg.hash[0]);
      check_hect_header(t + io.wg.blob[0], io.wg.hash[1]);
    }
  cudaStream_t st = c->stream;
  if (!c->copy_stream) CU(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  cudaStream_t cs = c->copy_stream;
  const size_t words = w->kc * c->ct_words();
  const size_t row_bytes = wire ? w->kc * (io.wg.blob[0] + io.wg.blob[1]) : words * 8;
  const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(s->cap_rows, (rows + c->e2e_div - 1) / c->e2e_div));
  // a slot holds up to 1.5 chunks so the final tail can be absorbed
  const uint64_t slot_rows = std::min<uint64_t>(s->cap_rows, chunk + chunk / 2);
  const size_t slot_bytes = (slot_rows * row_bytes + 64) & ~(size_t)15;  // + pad for the parser's 12-byte window
  uint8_t* stage = reinterpret_cast<uint8_t*>(
      pool_get(c->pool_stage64, c->pool_stage64_bytes, 2 * slot_bytes));
  uint32_t* in32 = pool_get(c->pool_in32, c->pool_in32_bytes, 2 * slot_rows * words * 4);
  uint64_t* d_rows = pool_get(c->pool_rows, c->pool_rows_bytes, rows * 8);
  k_iota<<<grid_for(rows, 256), 256, 0, st>>>(d_rows, 0, rows, c->d_ops, s->d_ops0);
  LAUNCHED();
  cudaEvent_t copied[2], narrowed[2];
  for (int k = 0; k < 2; ++k) {
    CU(cudaEventCreateWithFlags(&copied[k], cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&narrowed[k], cudaEventDisableTiming));
    CU(cudaEventRecord(narrowed[k], st));
  }
  // Consecutive chunks run concurrently on two stream sets, each with its own
  // input slot and scratch region, so one chunk's launches fill the tails of
  // the other's (packed sums are exact integer atomics: order-free).
  const uint32_t fp = c->fold_parts;
  const bool overlap = c->e2e_overlap && c->two_streams && !c->timing && fp >= 2;
  ChunkSlot cslot[2] = {};
  if (overlap) {
    while (c->chunk_streams.size() < 2 * fp) {
      cudaStream_t ps;
      CU(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
      c->chunk_streams.push_back(ps);
    }
    ensure_scratch(c, 2 * slot_rows * w->cols);
    for (int k = 0; k < 2; ++k) {
      for (uint32_t h = 0; h < fp; ++h) cslot[k].streams[h] = c->chunk_streams[k * fp + h];
      cslot[k].pair_off = (uint64_t)k * slot_rows * w->cols;
      CU(cudaEventCreateWithFlags(&cslot[k].done, cudaEventDisableTiming));
      CU(cudaEventRecord(cslot[k].done, st));
    }
  }
  const uint8_t* src = wire ? io.wire : reinterpret_cast<const uint8_t*>(io.u64);
  // chunk sizes ramp up (chunk/8, chunk/4, ..., chunk) so the first copy,
  // the only one not hidden behind compute, is short; a tail smaller than
  // half the next chunk is absorbed (no small launches at the end)
  uint64_t nr_next = std::max<uint64_t>(1, chunk / 8);
  for (uint64_t b = 0, r0 = 0; r0 < rows; ++b) {
    const int slot = (int)(b % 2);
    uint64_t nr = std::min<uint64_t>(nr_next, rows - r0);
    if (rows - r0 - nr < std::min<uint64_t>(chunk, 2 * nr_next) / 2 && rows - r0 <= slot_rows) nr = rows - r0;
    nr_next = std::min<uint64_t>(chunk, 2 * nr_next);
    uint8_t* sb = stage + (size_t)slot * slot_bytes;
    uint32_t* s32 = in32 + (size_t)slot * slot_rows * words;
    CU(cudaStreamWaitEvent(cs, narrowed[slot], 0));
    CU(cudaMemcpyAsync(sb, src + r0 * row_bytes, nr * row_bytes, cudaMemcpyHostToDevice, cs));
    CU(cudaEventRecord(copied[slot], cs));
    CU(cudaStreamWaitEvent(st, copied[slot], 0));
    if (overlap) CU(cudaStreamWaitEvent(st, cslot[slot].done, 0));  // slot and scratch of chunk b-2 released
    if (wire)
      k_wire_parse<<<grid_for(nr * words, 256), 256, 0, st>>>(c->geo, io.wg, sb, s32, nr * w->kc, c->d_err);
    else
      k_narrow<<<grid_for(nr * words, 256), 256, 0, st>>>(c->geo, reinterpret_cast<const uint64_t*>(sb), s32,
                                                          nr * w->kc, c->d_err);
    LAUNCHED();
    CU(cudaEventRecord(narrowed[slot], st));
    if (wire || io.form == HEI_FORM_COEFF) launch_ct_ntt(c, (unsigned)(nr * w->kc * 2 * c->P()), s32, st);
    if (!overlap || !run_rows(s.get(), s32, d_rows + r0, nr, st, &cslot[slot])) {
      // serialised chunk (too small for slices): scratch from offset 0
      if (overlap) CU(cudaStreamWaitEvent(st, cslot[1 - slot].done, 0));
      run_rows(s.get(), s32, d_rows + r0, nr, st);
      if (overlap) CU(cudaEventRecord(cslot[slot].done, st));
    }
    r0 += nr;
  }
  if (overlap)
    for (int k = 0; k < 2; ++k) CU(cudaStreamWaitEvent(st, cslot[k].done, 0));
  CU(cudaStreamSynchronize(st));
  for (int k = 0; k < 2; ++k) {
    cudaEventDestroy(copied[k]);
    cudaEventDestroy(narrowed[k]);
    if (cslot[k].done) cudaEventDestroy(cslot[k].done);
  }
  {
    uint32_t h = 0;
    CU(cudaMemcpyAsync(&h, c->d_err, 4, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    if (h) {
      CU(cudaMemsetAsync(c->d_err, 0, 4, c->stream));
      CU(cudaStreamSynchronize(c->stream));
      raise(HEI_CODEC_ERROR, (h & 2) ? "unexpected polynomial form" : "coefficient not reduced");
    }
  }
  s->pushed = rows;
  const size_t outw = s->C * c->ct_words();
  uint32_t* d_out = pool_get(c->pool_out, c->pool_out_bytes, outw * 4);
  const size_t out_bytes = wire ? s->C * (io.wg.blob[0] + io.wg.blob[1]) : outw * 8;
  uint64_t* d_out64 = pool_get(c->pool_out64, c->pool_out64_bytes, out_bytes);
  finish_to(s.get(), d_out, st);
  if (wire) {
    // save_ciphertext writes canonical coefficient form (serialize.cpp:67-71)
    launch_ct_intt(c, (unsigned)(s->C * 2 * c->P()), d_out, st);
    uint8_t* d_bytes = reinterpret_cast<uint8_t*>(d_out64);
    k_wire_emit<<<grid_for(outw, 256), 256, 0, st>>>(c->geo, io.wg, d_out, d_bytes, s->C);
    LAUNCHED();
    d2h_result(c, io.out_wire, d_bytes, out_bytes, st);
  } else {
    k_widen<<<grid_for(outw, 256), 256, 0, st>>>(d_out, d_out64, outw);
    LAUNCHED();
    d2h_result(c, io.out64, d_out64, outw * 8, st);
  }
  s->finished = true;
  if (cnt) ops_report(s.get(), cnt);
}

int hei_gpu_matmul(hei_gpu_ctx* c, const hei_gpu_weights* w, const uint64_t* inputs, int form, uint64_t rows,
                   const int64_t* bias, uint64_t* out, hei_op_counters* cnt) {
  return guarded([&] {
    if (form != HEI_FORM_EVAL && form != HEI_FORM_COEFF) raise(HEI_PARAM_ERROR, "matmul: unknown form");
    HostIO io;
    io.u64 = inputs;
    io.form = form;
    io.out64 = out;
    matmul_host(c, w, io, rows, bias, cnt);
  });
}

int hei_default_q_primes(uint32_t n, uint64_t t, uint64_t* out, uint32_t capacity, uint32_t* count) {
  // bfv::default_q_primes (params.cpp:84-104) over ring::find_ntt_primes
  // (modulus.cpp:54-71): descending candidates = 1 mod 2n below 2^bits.
  return guarded([&] {
    if (!n || (n & (n - 1))) raise(HEI_PARAM_ERROR, "n must be a power of two");
    const int bits = n >= 4096 ? 31 : 30;
    size_t want;
    if (n >= 4096) {
      want = t >= (1ull << 25) ? 6 : 4;
    } else {
      const int tb = 64 - __builtin_clzll(t);
      want = (size_t)(7 * tb / 2 + 50 + 29) / 30;
      if (want < 2) want = 2;
    }
    const uint64_t two_n = 2ull * n;
    std::vector<uint64_t> found;
    uint64_t c = ((((1ull << bits) - 2) / two_n) * two_n) + 1;
    while (found.size() < want && c > (1ull << (bits - 1))) {
      if (c != t && is_prime(c)) found.push_back(c);
      if (c < two_n) break;
      c -= two_n;
    }
    if (found.size() < want) raise(HEI_PARAM_ERROR, "not enough NTT-friendly primes of the requested size");
    if (count) *count = (uint32_t)found.size();
    if (out) {
      if (capacity < found.size()) raise(HEI_PARAM_ERROR, "default_q_primes: output buffer too small");
      std::memcpy(out, found.data(), found.size() * 8);
    }
  });
}

uint64_t hei_hect_ciphertext_bytes(uint32_t n, uint32_t num_primes) { return hect_bytes(n, num_primes); }

uint64_t hei_params_hash(uint32_t n, uint64_t t, int security_level, const uint64_t* q, uint32_t num_primes) {
  // FNV-1a over (n, t, security, q...) — EncryptionParams::hash (params.cpp:68-82)
  uint64_t h = 0xcbf29ce484222325ull;
  auto mix = [&h](uint64_t v) {
    for (int i = 0; i < 8; ++i) {
      h ^= (v >> (8 * i)) & 0xff;
      h *= 0x100000001b3ull;
    }
  };
  mix(n);
  mix(t);
  mix((uint64_t)(int64_t)security_level);
  for (uint32_t i = 0; i < num_primes; ++i) mix(q[i]);
  return h;
}

int hei_gpu_matmul_wire(hei_gpu_ctx* c, const hei_gpu_weights* w, const uint64_t params_hash[2],
                        const uint8_t* blobs, uint64_t blob_bytes, uint64_t rows, const int64_t* bias,
                        uint8_t* out, uint64_t out_capacity, uint64_t* out_bytes, hei_op_counters* cnt) {
  return guarded([&] {
    if (!w) raise(HEI_PARAM_ERROR, "matmul: empty weights");
    if (rows == 0) raise(HEI_PARAM_ERROR, "request carries no rows");
    HostIO io;
    io.wg.blob[0] = hect_bytes(c->n, c->L[0]);
    io.wg.blob[1] = hect_bytes(c->n, c->L[1]);
    io.wg.hash[0] = params_hash[0];
    io.wg.hash[1] = params_hash[1];
    const uint64_t per = io.wg.blob[0] + io.wg.blob[1];
    // server.cpp:131-136: the blob list must be exactly rows x chunks x branches
    if (blob_bytes % (w->kc * per) != 0 || blob_bytes / (w->kc * per) != rows)
      raise(HEI_PARAM_ERROR, "ciphertext count does not match rows x chunks");
    const uint64_t C = (rows * w->cols + c->n - 1) / c->n;
    if (out_bytes) *out_bytes = C * per;
    if (out_capacity < C * per) raise(HEI_PARAM_ERROR, "matmul_wire: output buffer too small");
    io.wire = blobs;
    io.out_wire = out;
    matmul_host(c, w, io, rows, bias, cnt);
  });
}

int hei_gpu_matmul_device(hei_gpu_ctx* c, const hei_gpu_weights* w, const uint32_t* d_inputs, int form,
                          uint64_t rows, const int64_t* bias, uint32_t* d_out, hei_op_counters* cnt, void* stream) {
  // Everything is enqueued on `st` with no host round trip until the final
  // synchronisation (row ids come from a device iota, the bias from pinned
  // staging), so small batches are not host-bound.
  return guarded([&] {
    set_device(c);
    std::lock_guard<std::mutex> lk(c->mu);
    if (form != HEI_FORM_EVAL) raise(HEI_PARAM_ERROR, "matmul_device: inputs must be in eval form");
    cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
    std::unique_ptr<hei_gpu_stream, void (*)(hei_gpu_stream*)> s(stream_new(c, w, bias, rows, false, st), stream_free);
    const size_t words = w->kc * c->ct_words();
    uint64_t* d_rows = pool_get(c->pool_rows, c->pool_rows_bytes, rows * 8);
    k_iota<<<grid_for(rows, 256), 256, 0, st>>>(d_rows, 0, rows, c->d_ops, s->d_ops0);
    LAUNCHED();
    for (uint64_t r0 = 0; r0 < rows; r0 += s->cap_rows) {
      const uint64_t nr = std::min<uint64_t>(s->cap_rows, rows - r0);
      run_rows(s.get(), d_inputs + r0 * words, d_rows + r0, nr, st);
    }
    s->pushed = rows;
    finish_to(s.get(), d_out, st);
      CU(cudaStreamSynchronize(st));
    s->finished = true;
    if (cnt) ops_report(s.get(), cnt);
  });
}

int hei_gpu_ntt(hei_gpu_ctx* c, uint32_t b, uint32_t prime, uint64_t* polys, uint64_t count, int inverse) {
  return guarded([&] {
    if (b > 1 || prime >= c->L[b]) raise(HEI_PARAM_ERROR, "prime index out of range");
    set_device(c);
    const uint32_t gp = (b ? c->L[0] : 0) + prime;
    const uint64_t words = count * c->n;
    std::vector<uint32_t> h32(words);
    for (uint64_t x = 0; x < words; ++x) {
      if (polys[x] >= c->q[gp]) raise(HEI_PARAM_ERROR, "ntt: coefficient not reduced");
      h32[x] = (uint32_t)polys[x];
    }
    uint32_t* d = nullptr;
    CU(cudaMalloc(&d, words * 4));
    CU(cudaMemcpyAsync(d, h32.data(), words * 4, cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    launch_poly_ntt(c, (unsigned)count, gp, d, inverse, c->stream);
    CU(cudaMemcpyAsync(h32.data(), d, words * 4, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    cudaFree(d);
    for (uint64_t x = 0; x < words; ++x) polys[x] = h32[x];
  });
}

int hei_gpu_apply_galois(hei_gpu_ctx* c, uint32_t b, uint64_t elt, const uint64_t* in, uint64_t* out) {
  return hei_gpu_apply_galois_form(c, b, elt, HEI_FORM_EVAL, in, out);
}

int hei_gpu_apply_galois_form(hei_gpu_ctx* c, uint32_t b, uint64_t elt, int form, const uint64_t* in, uint64_t* out) {
  return guarded([&] {
    if (b > 1) raise(HEI_PARAM_ERROR, "branch out of range");
    if (form != HEI_FORM_EVAL && form != HEI_FORM_COEFF) raise(HEI_PARAM_ERROR, "apply_galois: unknown form");
    if (!c->has_keys[b] || !c->key_index[b].count(elt))
      raise(HEI_KEY_ERROR, "apply_galois: no key for galois element " + std::to_string(elt));
    if (!c->perm_index.count(elt)) raise(HEI_KEY_ERROR, "apply_galois: unsupported galois element");
    set_device(c);
    // Embed the branch ciphertext in a twin-shaped buffer; only branch b's
    // blocks are launched (grid over its primes via a branch-restricted Geo).
    Geo g = c->geo;
    const uint32_t L = c->L[b], n = c->n;
    // single-branch geometry: P = L, ct = [2][L][n]
    Geo gb = g;
    gb.P = L;
    gb.ct_words = 2 * L * n;
    gb.pt_words = L * n;
    gb.L[0] = L;
    gb.L[1] = 0;
    for (uint32_t i = 0; i < L; ++i) {
      gb.pr[i] = g.pr[(b ? c->L[0] : 0) + i];
      gb.pr[i].poly0 = i;
      gb.pr[i].poly1 = L + i;
      gb.pr[i].first = 0;
      gb.pr[i].b = 0;
    }
    // twiddle rows: shift the table base so row i maps to branch prime i
    gb.fwd = g.fwd + (size_t)(b ? c->L[0] : 0) * n;
    gb.inv = g.inv + (size_t)(b ? c->L[0] : 0) * n;
    if (g.twc) {
      gb.twc = g.twc + (size_t)(b ? c->L[0] : 0) * g.twc_stride;
      gb.itwc = g.itwc + (size_t)(b ? c->L[0] : 0) * g.twc_stride;
    }
    if (g.twch) {
      gb.twch = g.twch + (size_t)(b ? c->L[0] : 0) * 2 * g.twch_stride;
      gb.fwdh = g.fwdh + (size_t)(b ? c->L[0] : 0) * 2 * (n / 2);
      gb.itwch = g.itwch + (size_t)(b ? c->L[0] : 0) * 2 * g.twch_stride;
      gb.invh = g.invh + (size_t)(b ? c->L[0] : 0) * 2 * (n / 2);
    }
    const size_t words = 2ull * L * n;
    std::vector<uint32_t> h32(words);
    for (size_t x = 0; x < words; ++x) h32[x] = (uint32_t)in[x];
    uint32_t *d_in = nullptr, *d_out = nullptr, *d_dig = nullptr;
    CU(cudaMalloc(&d_in, words * 4));
    CU(cudaMalloc(&d_out, words * 4));
    CU(cudaMalloc(&d_dig, (size_t)L * n * 4));
    CU(cudaMemcpyAsync(d_in, h32.data(), words * 4, cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    const uint32_t* perm = c->d_perms + (size_t)c->perm_index.at(elt) * n;
    const uint2* key = c->d_keys[b] + (size_t)c->key_index[b].at(elt) * L * 2 * L * n;
    const size_t sm = smem_bytes(c, 1);
    // Coefficient-form input (context.cpp:460-465, 499-503): the reference
    // takes sigma_coeff of c0 and c1 (automorphism_coeff, poly.cpp:107-122),
    // switches the keys in the eval domain and inverse-transforms acc0/acc1
    // before adding sigma_coeff(c0). Transforming in, running the eval path
    // and transforming out computes the same residues exactly: NTT and INTT
    // are exact inverses mod q_i, INTT(sigma_eval(NTT(x))) = sigma_coeff(x),
    // so the digits and every sum equal the reference's.
    if (form == HEI_FORM_COEFF) {
      HEI_DISPATCH(c->logn, (k_ct_ntt_f<LG><<<2 * L, Ntt<LG>::T, sm, c->stream>>>(gb, d_in)),
                   (k_ct_ntt<<<2 * L, c->threads(), sm, c->stream>>>(gb, d_in, 0)));
      LAUNCHED();
    }
    launch_rot_digits(c, gb, L, d_in, perm, d_dig, c->stream);
    launch_rot_keyswitch(c, gb, L, d_in, d_dig, perm, key, key, d_out, 0, c->stream);
    if (form == HEI_FORM_COEFF) {
      HEI_DISPATCH(c->logn, (k_ct_intt_f<LG><<<2 * L, Ntt<LG>::T, sm, c->stream>>>(gb, d_out)),
                   (k_ct_ntt<<<2 * L, c->threads(), sm, c->stream>>>(gb, d_out, 1)));
      LAUNCHED();
    }
    CU(cudaMemcpyAsync(h32.data(), d_out, words * 4, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    cudaFree(d_in);
    cudaFree(d_out);
    cudaFree(d_dig);
    for (size_t x = 0; x < words; ++x) out[x] = h32[x];
  });
}

int hei_gpu_sum_all_slots(hei_gpu_ctx* c, const uint64_t* in, uint64_t* out, uint64_t count) {
  return guarded([&] {
    set_device(c);
    require_keys(c);
    std::lock_guard<std::mutex> lk(c->mu);
    const size_t words = count * c->ct_words();
    ensure_scratch(c, count);
    uint64_t* d64 = nullptr;
    CU(cudaMalloc(&d64, words * 8));
    CU(cudaMemcpyAsync(d64, in, words * 8, cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    k_narrow<<<grid_for(words, 256), 256, 0, c->stream>>>(c->geo, d64, c->d_dotA, count, c->d_err);
    LAUNCHED();
    check_err_flag(c, HEI_CODEC_ERROR, "sum_all_slots: coefficient not reduced");
    uint32_t* res = fold(c, count, c->d_dotA, c->d_dotB, c->stream);
    k_widen<<<grid_for(words, 256), 256, 0, c->stream>>>(res, d64, words);
    LAUNCHED();
    CU(cudaMemcpyAsync(out, d64, words * 8, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    cudaFree(d64);
  });
}

int hei_gpu_prng_create(uint64_t seed, hei_gpu_prng** out) {
  return guarded([&] {
    auto p = std::make_unique<hei_gpu_prng>();
    prng_seed(p.get(), seed);
    *out = p.release();
  });
}
void hei_gpu_prng_destroy(hei_gpu_prng* p) { delete p; }
int hei_gpu_prng_draw(hei_gpu_prng* p, uint64_t count, uint64_t* out) {
  return guarded([&] {
    for (uint64_t i = 0; i < count; ++i) out[i] = prng_next(p);
  });
}

int hei_gpu_baseline_matmul(hei_gpu_ctx* c, const int64_t* x, uint64_t rows, uint64_t f, const int64_t* w,
                            uint64_t cols, const int64_t* bias, hei_gpu_prng* rng0, hei_gpu_prng* rng1,
                            uint64_t* out, hei_op_counters* cnt) {
  return guarded([&] {
    // matmul.cpp:276-292
    if (rows == 0 || f == 0 || cols == 0) raise(HEI_PARAM_ERROR, "baseline: empty input");
    capacity_gate(c, f, "baseline");
    if (!c->d_pk[0] || !c->d_pk[1]) raise(HEI_KEY_ERROR, "encrypt: this backend holds no public key");
    if (!rng0 || !rng1) raise(HEI_PARAM_ERROR, "baseline: encryption randomness required");
    if (rng0->have_spare || rng1->have_spare)
      raise(HEI_PARAM_ERROR, "baseline: rng holds a cached Box-Muller spare; cannot replay on the device");
    const int64_t lim = (int64_t)(((u128)c->t[0] * c->t[1] - 1) / 2);
    for (uint64_t i = 0; i < f * cols; ++i)
      if (w[i] > lim || w[i] < -lim) raise(HEI_RANGE_ERROR, "prepare_constant_signed: value outside centered range");
    for (uint64_t i = 0; i < rows * f; ++i)
      if (x[i] > lim || x[i] < -lim) raise(HEI_RANGE_ERROR, "encode_signed: value outside the centered range");
    check_bias_range(c, bias, cols);
    for (int b = 0; b < 2; ++b)
      for (uint32_t i = 0; i < c->L[b]; ++i)
        if (c->t[b] >= c->q[(b ? c->L[0] : 0) + i])
          raise(HEI_PARAM_ERROR, "baseline: plaintext modulus exceeds a ciphertext prime (unsupported)");
    set_device(c);
    std::lock_guard<std::mutex> lk(c->mu);
    const hei_gpu_prng init0 = *rng0, init1 = *rng1;
    for (bool force_seq = false;; force_seq = true) {
    cudaStream_t st = c->stream;
    const Geo& g = c->geo;
    const uint32_t n = c->n, P = c->P();
    const uint64_t B = (rows + n - 1) / n;
    // prepared public key [gp][part] (cached)
    if (!c->d_pkp) {
      CU(cudaMalloc(&c->d_pkp, 2ull * P * n * sizeof(uint2)));
      const size_t sm = smem_bytes(c, 1);
      HEI_DISPATCH(c->logn, (k_prepare_pk<LG><<<2 * P, Ntt<LG>::T, sm, st>>>(g, c->d_pk[0], c->d_pk[1], c->d_pkp, c->d_err)),
                   (k_prepare_pk_g<<<2 * P, c->threads(), sm, st>>>(g, c->d_pk[0], c->d_pk[1], c->d_pkp, c->d_err)));
      LAUNCHED();
      check_err_flag(c, HEI_CODEC_ERROR, "public key: coefficient not reduced");
    }
    // features per batch (one noise/encode/sum round); every batch's draws
    // are the next F*B encryptions of both branch streams
    const uint64_t F = std::min<uint64_t>(f, std::max<uint64_t>(1, 1024 / B));
    const uint64_t Emax = F * B;
    int64_t *d_x = nullptr, *d_w = nullptr, *d_bias = nullptr;
    uint2* d_wc = nullptr;
    uint64_t *d_raw = nullptr, *d_state = nullptr;
    uint32_t *d_noisep = nullptr, *d_m = nullptr, *d_res = nullptr, *d_out = nullptr;
    long long* d_sums = nullptr;
    uint64_t* d_out64 = nullptr;
    const size_t outw = B * cols * c->ct_words();
    // feature slices per k_bl_sums launch: enough blocks to fill the GPU
    const uint32_t tiles = std::max<uint32_t>(1, n / 128), grp = (uint32_t)((cols + kBlSumJ - 1) / kBlSumJ);
    const uint64_t base_blocks = (uint64_t)tiles * grp * B * 2;
    const uint32_t S = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>({8, F, (2048 + base_blocks - 1) / base_blocks}));
    const size_t sums_words = (size_t)S * B * cols * 2 * 5 * n;
    d_x = scratch<int64_t>(c, kScrX, rows * f * 8);
    d_w = scratch<int64_t>(c, kScrW, f * cols * 8);
    d_bias = scratch<int64_t>(c, kScrBias, cols * 8);
    d_wc = scratch<uint2>(c, kScrWc, f * cols * P * sizeof(uint2));
    d_sums = scratch<long long>(c, kScrAcc, sums_words * 8);
    d_res = scratch<uint32_t>(c, kScrCt, (size_t)B * cols * P * 3 * n * 4);
    d_raw = scratch<uint64_t>(c, kScrRaw, 2 * 2 * Emax * 3 * n * 8);  // [slot][branch][draws]
    d_state = scratch<uint64_t>(c, kScrState, 2 * 313 * 8);
    d_noisep = scratch<uint32_t>(c, kScrNoise, Emax * 2 * n * 4);
    d_m = scratch<uint32_t>(c, kScrM, Emax * 2 * n * 4);
    d_out = scratch<uint32_t>(c, kScrOut, outw * 4);
    d_out64 = scratch<uint64_t>(c, kScrOut64, outw * 8);
    CU(cudaMemcpyAsync(d_x, x, rows * f * 8, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(d_w, w, f * cols * 8, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(d_bias, bias, cols * 8, cudaMemcpyHostToDevice, st));
    CU(cudaMemsetAsync(d_sums, 0, sums_words * 8, st));
    CU(cudaMemsetAsync(d_res, 0, (size_t)B * cols * P * 3 * n * 4, st));
    uint64_t hstate[2][313];
    for (int b = 0; b < 2; ++b) {
      hei_gpu_prng* r = b ? rng1 : rng0;
      std::memcpy(hstate[b], r->mt, 312 * 8);
      hstate[b][312] = r->mti;
    }
    CU(cudaMemcpyAsync(d_state, hstate, sizeof(hstate), cudaMemcpyHostToDevice, st));
    k_bl_weights<<<grid_for(f * cols * P, 256), 256, 0, st>>>(g, d_w, f * cols, d_wc);
    LAUNCHED();
    // Jump-ahead replay: when both streams start block-aligned (mti == 312,
    // e.g. fresh Prngs), the whole call's draws are produced by K chunk
    // generators per branch whose start states come from x^C mod phi
    // (k_mt_jumps), instead of one sequential generator per branch. A
    // rejection anywhere would misalign the chunks; the noise kernel flags it
    // at its exact position and the call re-runs on the sequential path.
    const uint64_t E_total = f * B, Dtot = E_total * 3 * n;
    bool jump = c->mt_jump && !force_seq && hstate[0][312] == 312 && hstate[1][312] == 312 && E_total >= 64 &&
                Dtot * 16 <= ((uint64_t)48 << 30);
    uint64_t* d_rawall = nullptr;
    if (jump) {
      uint64_t K = std::min<uint64_t>(c->mt_chunks_max, E_total / 8);
      const uint64_t Cenc = (E_total + K - 1) / K;
      K = (E_total + Cenc - 1) / Cenc;
      const uint64_t C = Cenc * 3 * n;
      uint64_t* d_starts = nullptr;
      d_starts = scratch<uint64_t>(c, kScrStarts, 2 * K * 313 * 8);
      d_rawall = scratch<uint64_t>(c, kScrRawAll, 2 * Dtot * 8);
      mt_chunk_starts(c, d_state, K, C, d_starts, st);  // chunk 0 = the current (block-aligned) state
      heb_baseline::k_mt_chunks<<<dim3((unsigned)K, 2), 320, 0, st>>>(d_starts, (uint32_t)K, C, Dtot, d_rawall, d_state);
      LAUNCHED();
    }
    const size_t sm1 = smem_bytes(c, 1);
    // The mt19937_64 replay is sequential per branch (one CTA each), so the
    // next batch's draws are generated on a side stream while the current
    // batch is summed (double-buffered raw draws).
    if (!c->copy_stream) CU(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    cudaStream_t ms = c->copy_stream;
    cudaEvent_t gen[2], used[2];
    for (int k = 0; k < 2; ++k) {
      CU(cudaEventCreateWithFlags(&gen[k], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&used[k], cudaEventDisableTiming));
      CU(cudaEventRecord(used[k], st));
    }
    CU(cudaStreamSynchronize(st));  // state, x, w uploads visible to `ms`
    auto generate = [&](uint64_t k0, int slot) {
      if (jump) return;
      const uint64_t Fb = std::min<uint64_t>(F, f - k0), draws = Fb * B * 3 * n;
      CU(cudaStreamWaitEvent(ms, used[slot], 0));
      heb_baseline::k_mt_generate<<<2, 320, 0, ms>>>(d_state, d_raw + (size_t)slot * 2 * Emax * 3 * n, draws);
      LAUNCHED();
      CU(cudaEventRecord(gen[slot], ms));
    };
    auto fold_sums = [&]() {
      k_bl_fold_sums<<<grid_for((uint64_t)B * cols * P * n, 256), 256, 0, st>>>(g, d_sums, S, (uint32_t)B,
                                                                                (uint32_t)cols, d_res);
      LAUNCHED();
      CU(cudaMemsetAsync(d_sums, 0, sums_words * 8, st));
    };
    generate(0, 0);
    int slot = 0;
    uint64_t since_fold = 0;
    for (uint64_t k0 = 0; k0 < f; k0 += F, slot ^= 1) {
      const uint64_t Fb = std::min<uint64_t>(F, f - k0), E = Fb * B, draws = E * 3 * n;
      if (k0 + F < f) generate(k0 + F, slot ^ 1);
      if (jump) {
        k_bl_noise_p<<<dim3((unsigned)E, 2), 256, 0, st>>>(d_rawall + k0 * B * 3 * n, Dtot, n, d_noisep, c->d_err);
      } else {
        CU(cudaStreamWaitEvent(st, gen[slot], 0));
        k_bl_noise_p<<<dim3((unsigned)E, 2), 256, 0, st>>>(d_raw + (size_t)slot * 2 * Emax * 3 * n, draws, n,
                                                           d_noisep, c->d_err);
      }
      LAUNCHED();
      CU(cudaEventRecord(used[slot], st));
      HEI_DISPATCH(c->logn,
                   (k_bl_encode<LG><<<dim3((unsigned)E, 2), Ntt<LG>::T, sm1, st>>>(g, d_x, rows, f, k0, (uint32_t)B, d_m)),
                   (k_bl_encode_g<<<dim3((unsigned)E, 2), c->threads(), sm1, st>>>(g, d_x, rows, f, k0, (uint32_t)B, d_m)));
      LAUNCHED();
      const uint32_t Sb = (uint32_t)std::min<uint64_t>(S, Fb);
      k_bl_sums<<<dim3(tiles * grp, Sb, (unsigned)(B * 2)), std::min<uint32_t>(128, n), 0, st>>>(
          g, d_noisep, d_m, (uint32_t)Fb, (uint32_t)B, (uint32_t)cols, d_wc + k0 * cols * P, d_sums);
      LAUNCHED();
      since_fold += Fb;
      if (since_fold + F > (1u << 17)) {  // keep every int64 sum below 2^63
        fold_sums();
        since_fold = 0;
      }
    }
    if (since_fold) fold_sums();
    CU(cudaStreamSynchronize(ms));
    for (int k = 0; k < 2; ++k) {
      cudaEventDestroy(gen[k]);
      cudaEventDestroy(used[k]);
    }
    k_bl_finish_lin<<<(unsigned)(B * cols * P), c->threads(), 3 * n * 4, st>>>(g, d_res, c->d_pk[0], c->d_pk[1],
                                                                                d_bias, (uint32_t)cols, d_out);
    LAUNCHED();
    k_widen<<<grid_for(outw, 256), 256, 0, st>>>(d_out, d_out64, outw);
    LAUNCHED();
    CU(cudaMemcpyAsync(out, d_out64, outw * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(hstate, d_state, sizeof(hstate), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    for (int b = 0; b < 2; ++b) {
      hei_gpu_prng* r = b ? rng1 : rng0;
      std::memcpy(r->mt, hstate[b], 312 * 8);
      r->mti = (uint32_t)hstate[b][312];
    }
    if (jump) {
      uint32_t errh = 0;
      CU(cudaMemcpyAsync(&errh, c->d_err, 4, cudaMemcpyDeviceToHost, c->stream));
      CU(cudaStreamSynchronize(c->stream));
      if (errh) {  // a rejection misaligned the chunks: replay sequentially
        CU(cudaMemsetAsync(c->d_err, 0, 4, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        *rng0 = init0;
        *rng1 = init1;
        continue;
      }
    }
    check_err_flag(c, HEI_INTERNAL, "baseline: rng rejection in the encryption stream (replay unsupported)");
    if (cnt) hei_baseline_counts(rows, cols, f, n, cnt);
    break;
    }
  });
}


// ---- sharded (multi-GPU) building blocks: partial packed sums + finish ----
int hei_gpu_matmul_partial_device(hei_gpu_ctx* c, const hei_gpu_weights* w, const uint32_t* d_inputs, uint64_t rows,
                                  uint64_t row_offset, uint64_t total_rows, uint64_t* d_acc, void* stream) {
  // Same enqueue-only structure as matmul_device (device row ids, no mid-call
  // host round trips); the bias is added once by finish_packed_device.
  return guarded([&] {
    set_device(c);
    std::lock_guard<std::mutex> lk(c->mu);
    if (rows == 0 || row_offset + rows > total_rows) raise(HEI_PARAM_ERROR, "matmul: shard rows out of range");
    cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
    std::vector<int64_t> zero_bias(w ? w->cols : 1, 0);
    std::unique_ptr<hei_gpu_stream, void (*)(hei_gpu_stream*)> s(
        stream_new(c, w, zero_bias.data(), total_rows, false, st, /*encode_bias=*/false,
                   reinterpret_cast<unsigned long long*>(d_acc)),  // accumulate into the caller's buffer
        stream_free);
    const size_t words = w->kc * c->ct_words();
    uint64_t* d_rows = pool_get(c->pool_rows, c->pool_rows_bytes, rows * 8);
    k_iota<<<grid_for(rows, 256), 256, 0, st>>>(d_rows, row_offset, rows);
    LAUNCHED();
    for (uint64_t r0 = 0; r0 < rows; r0 += s->cap_rows) {
      const uint64_t nr = std::min<uint64_t>(s->cap_rows, rows - r0);
      run_rows(s.get(), d_inputs + r0 * words, d_rows + r0, nr, st);
    }
    CU(cudaStreamSynchronize(st));
  });
}

// Peer-memory exchange for sharded runs: a rank exports its packed
// accumulator with CUDA IPC; the other ranks map it and their mask/pack
// kernels add into it directly (u64 atomics over NVLink), so the partial-sum
// exchange rides on the compute instead of a separate collective.
// Plain device buffers (base allocations, as CUDA IPC requires).
int hei_gpu_buffer_alloc(int device, uint64_t bytes, void** d_ptr) {
  return guarded([&] {
    if (!d_ptr) raise(HEI_PARAM_ERROR, "buffer: null argument");
    CU(cudaSetDevice(device));
    CU(cudaMalloc(d_ptr, bytes));
  });
}
int hei_gpu_buffer_zero(void* d_ptr, uint64_t bytes, void* stream) {
  return guarded([&] { CU(cudaMemsetAsync(d_ptr, 0, bytes, (cudaStream_t)stream)); });
}
void hei_gpu_buffer_free(void* d_ptr) { cudaFree(d_ptr); }

// Device-to-device copy on `stream`; with an IPC-mapped destination this is
// a peer write over NVLink.
int hei_gpu_copy_async(void* dst, const void* src, uint64_t bytes, void* stream) {
  return guarded([&] { CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream)); });
}

// slots[0] += slots[1] + ... + slots[count-1] over `words` u64 each (the
// owner's reduction of gathered per-rank packed accumulators; exact).
__global__ void k_sum_slots(unsigned long long* __restrict__ d, uint64_t words, uint32_t count) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < words; x += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long acc = d[x];
    for (uint32_t k = 1; k < count; ++k) acc += d[(uint64_t)k * words + x];
    d[x] = acc;
  }
}
int hei_gpu_sum_slots(void* d, uint64_t words, uint32_t count, void* stream) {
  return guarded([&] {
    k_sum_slots<<<grid_for(words, 256), 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<unsigned long long*>(d),
                                                                      words, count);
    LAUNCHED();
  });
}

// A rank's packed u64 accumulator reduced mod q into u32 residues: the
// partial it exchanges (half the bytes of the sums; exact, mod-q addition is
// order-free).
__global__ void k_reduce_packed(Geo g, const unsigned long long* __restrict__ acc, uint64_t words,
                                uint32_t* __restrict__ out) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < words; x += (uint64_t)gridDim.x * blockDim.x) {
    const PrimeInfo& pr = g.pr[poly_prime(g, (uint32_t)((x % g.ct_words) / g.n))];
    const unsigned long long v = acc[x];
    const unsigned long long r = v - __umul64hi(v, pr.mu) * pr.q;  // Barrett: at most one q too large
    out[x] = (uint32_t)(r >= pr.q ? r - pr.q : r);
  }
}
// acc[x] = sum over parts of parts[k][x] (u64, exact: < parts * 2^31)
__global__ void k_sum_parts(const uint32_t* __restrict__ parts, uint64_t words, uint32_t count,
                            unsigned long long* __restrict__ acc) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < words; x += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long a = 0;
    for (uint32_t k = 0; k < count; ++k) a += parts[(uint64_t)k * words + x];
    acc[x] = a;
  }
}

int hei_gpu_reduce_packed_device(hei_gpu_ctx* c, const uint64_t* d_acc, uint64_t count, uint32_t* d_out,
                                 void* stream) {
  return guarded([&] {
    set_device(c);
    if (!d_acc || !d_out || count == 0) raise(HEI_PARAM_ERROR, "reduce_packed: empty argument");
    const uint64_t words = count * c->ct_words();
    k_reduce_packed<<<grid_for(words, 256), 256, 0, (cudaStream_t)stream>>>(
        c->geo, reinterpret_cast<const unsigned long long*>(d_acc), words, d_out);
    LAUNCHED();
  });
}

int hei_gpu_finish_parts_device(hei_gpu_ctx* c, const hei_gpu_weights* w, const uint32_t* d_parts, uint32_t parts,
                                const int64_t* bias, uint64_t total_rows, uint32_t* d_out, void* stream) {
  return guarded([&] {
    set_device(c);
    std::lock_guard<std::mutex> lk(c->mu);
    if (!w || !d_parts || !d_out || parts == 0 || total_rows == 0) raise(HEI_PARAM_ERROR, "finish_parts: empty argument");
    check_bias_range(c, bias, w->cols);
    cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
    hei_gpu_stream tmp{};
    tmp.ctx = c;
    tmp.w = w;
    tmp.bias.assign(bias, bias + w->cols);
    tmp.rows = total_rows;
    tmp.C = (total_rows * w->cols + c->n - 1) / c->n;
    const uint64_t words = tmp.C * c->ct_words();
    tmp.d_acc = pool_get(c->pool_acc, c->pool_acc_bytes, words * 8);
    tmp.owns_acc = false;
    k_sum_parts<<<grid_for(words, 256), 256, 0, st>>>(d_parts, words, parts, tmp.d_acc);
    LAUNCHED();
    // the bias is staged synchronously (pageable host memory), then the
    // finish is enqueued on `st` and the call returns without waiting
    int64_t* d_bias = pool_get(c->pool_bias, c->pool_bias_bytes, tmp.bias.size() * 8);
    CU(cudaMemcpy(d_bias, tmp.bias.data(), tmp.bias.size() * 8, cudaMemcpyHostToDevice));
    tmp.d_bias = d_bias;
    finish_to(&tmp, d_out, st);
  });
}

int hei_gpu_ipc_handle(const void* d_ptr, uint8_t* handle64) {
  return guarded([&] {
    if (!d_ptr || !handle64) raise(HEI_PARAM_ERROR, "ipc: null argument");
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle64, &h, sizeof(h));
  });
}

int hei_gpu_ipc_open(int device, const uint8_t* handle64, void** d_ptr) {
  return guarded([&] {
    if (!handle64 || !d_ptr) raise(HEI_PARAM_ERROR, "ipc: null argument");
    CU(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    CU(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int hei_gpu_ipc_close(void* d_ptr) {
  return guarded([&] { CU(cudaIpcCloseMemHandle(d_ptr)); });
}

int hei_gpu_chunk_dot_partial_device(hei_gpu_ctx* c, const hei_gpu_weights* w, const uint32_t* d_inputs,
                                     uint64_t rows, uint64_t chunk_lo, uint64_t chunk_count, uint64_t* d_dot,
                                     void* stream) {
  return guarded([&] {
    set_device(c);
    std::lock_guard<std::mutex> lk(c->mu);
    if (!w) raise(HEI_PARAM_ERROR, "matmul: empty weights");
    if (rows == 0 || chunk_count == 0 || chunk_lo + chunk_count > w->kc)
      raise(HEI_PARAM_ERROR, "matmul: feature block out of range");
    cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
    const uint64_t pairs = rows * w->cols;
    k_chunk_dot_part<<<(unsigned)(pairs * 2 * c->P()), std::min<unsigned>(c->threads(), 256u), 0, st>>>(
        c->geo, d_inputs, w->d_w, (uint32_t)w->cols, (uint32_t)w->kc, (uint32_t)chunk_lo, (uint32_t)chunk_count,
        reinterpret_cast<unsigned long long*>(d_dot));
    LAUNCHED();
    CU(cudaStreamSynchronize(st));
  });
}

int hei_gpu_fold_pack_device(hei_gpu_ctx* c, const hei_gpu_weights* w, const uint64_t* d_dot, uint64_t row_lo,
                             uint64_t row_count, uint64_t total_rows, uint64_t* d_acc, void* stream) {
  return guarded([&] {
    set_device(c);
    std::lock_guard<std::mutex> lk(c->mu);
    if (!w) raise(HEI_PARAM_ERROR, "matmul: empty weights");
    if (row_count == 0 || row_lo + row_count > total_rows) raise(HEI_PARAM_ERROR, "matmul: shard rows out of range");
    capacity_gate(c, w->f, "matmul");
    require_keys(c);
    cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
    hei_gpu_stream tmp{};
    tmp.ctx = c;
    tmp.w = w;
    tmp.rows = total_rows;
    tmp.C = (total_rows * w->cols + c->n - 1) / c->n;
    tmp.d_acc = reinterpret_cast<unsigned long long*>(d_acc);
    tmp.owns_acc = false;
    tmp.owns_rows = false;
    const uint64_t cap = std::max<uint64_t>(1, auto_batch_pairs(c) / w->cols);
    uint64_t* d_rows = pool_get(c->pool_rows, c->pool_rows_bytes, std::min(cap, row_count) * 8);
    for (uint64_t r0 = 0; r0 < row_count; r0 += cap) {
      const uint64_t nr = std::min(cap, row_count - r0);
      ensure_scratch(c, nr * w->cols);
      k_iota<<<grid_for(nr, 256), 256, 0, st>>>(d_rows, row_lo + r0, nr);
      LAUNCHED();
      k_dot_reduce<<<grid_for(nr * w->cols * c->ct_words(), 256), 256, 0, st>>>(
          c->geo, reinterpret_cast<const unsigned long long*>(d_dot) + r0 * w->cols * c->ct_words(), nr * w->cols,
          c->d_dotA);
      LAUNCHED();
      run_folded_dots(&tmp, d_rows, nr, st);
      CU(cudaStreamSynchronize(st));
    }
  });
}

int hei_gpu_finish_packed_device(hei_gpu_ctx* c, const hei_gpu_weights* w, const uint64_t* d_acc, const int64_t* bias,
                                 uint64_t total_rows, uint32_t* d_out, void* stream) {
  return guarded([&] {
    set_device(c);
    std::lock_guard<std::mutex> lk(c->mu);
    check_bias_range(c, bias, w->cols);
    cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
    hei_gpu_stream tmp{};
    tmp.ctx = c;
    tmp.w = w;
    tmp.bias.assign(bias, bias + w->cols);
    tmp.rows = total_rows;
    tmp.C = (total_rows * w->cols + c->n - 1) / c->n;
    tmp.d_acc = reinterpret_cast<unsigned long long*>(const_cast<uint64_t*>(d_acc));
    tmp.owns_acc = false;
    finish_to(&tmp, d_out, st);
    CU(cudaStreamSynchronize(st));
  });
}


int hei_gpu_encode_inputs(hei_gpu_ctx* c, const int64_t* x, uint64_t rows, uint64_t f, hei_gpu_prng* rng0,
                          hei_gpu_prng* rng1, uint64_t* out) {
  return guarded([&] {
    set_device(c);
    std::lock_guard<std::mutex> lk(c->mu);
    encode_inputs_impl(c, x, rows, f, rng0, rng1, out, nullptr, c->stream);
  });
}

int hei_gpu_encode_inputs_device(hei_gpu_ctx* c, const int64_t* x, uint64_t rows, uint64_t f, hei_gpu_prng* rng0,
                                 hei_gpu_prng* rng1, uint32_t* d_out, void* stream) {
  return guarded([&] {
    set_device(c);
    std::lock_guard<std::mutex> lk(c->mu);
    encode_inputs_impl(c, x, rows, f, rng0, rng1, nullptr, d_out, stream ? (cudaStream_t)stream : c->stream);
  });
}

}  // extern "C"
