/* TEST INFRASTRUCTURE ONLY — the CPU checker for the GPU hot path.
 *
 * Plain-C restatement of the reference's encrypted-LR matmul hot path
 * (/root/reference/proj). Each function names the reference file:line it
 * follows. Pinned against oracle/_ref (the reference compiled in place) and
 * tests/golden/. Never linked or called by the product library.
 */
#define _GNU_SOURCE
#include "heoracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

typedef unsigned __int128 u128;

static __thread char g_err[512];
static int set_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}
const char* ho_last_error(void) { return g_err; }

#define ERR_PARAM 1
#define ERR_KEY 2
#define ERR_RANGE 3
#define ERR_NOISE 4
#define MAXL 16

/* ===================== util: bits (util/bits.hpp:11-29) ================== */
static uint32_t log2_exact(uint64_t v) { return 63u - (uint32_t)__builtin_clzll(v); }
static int is_pow2(uint64_t v) { return v && !(v & (v - 1)); }
static uint32_t reverse_bits(uint32_t v, uint32_t bits) {
  uint32_t r = 0;
  for (uint32_t i = 0; i < bits; ++i) r = (r << 1) | ((v >> i) & 1u);
  return r;
}

/* ========== modarith (kernels/modarith.hpp:15-78) ========== */
static inline uint64_t add_mod_1(uint64_t a, uint64_t b, uint64_t q) {
  uint64_t s = a + b;
  return s >= q ? s - q : s;
}
static inline uint64_t sub_mod_1(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }
static inline uint64_t neg_mod_1(uint64_t a, uint64_t q) { return a == 0 ? 0 : q - a; }
static inline uint64_t mul_mod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }
uint64_t ho_shoup_precompute(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }
static inline uint64_t shoup_mul(uint64_t x, uint64_t w, uint64_t ws, uint64_t q) {
  uint64_t qh = (uint64_t)(((u128)x * ws) >> 64);
  uint64_t r = x * w - qh * q;
  return r >= q ? r - q : r;
}
uint64_t ho_shoup_mul(uint64_t x, uint64_t w, uint64_t ws, uint64_t q) { return shoup_mul(x, w, ws, q); }
static uint64_t pow_mod(uint64_t b, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  b %= q;
  while (e) {
    if (e & 1) r = mul_mod(r, b, q);
    b = mul_mod(b, b, q);
    e >>= 1;
  }
  return r;
}
static int inv_mod(uint64_t a, uint64_t q, uint64_t* out) {
  int64_t t = 0, nt = 1, r = (int64_t)q, nr = (int64_t)(a % q);
  while (nr != 0) {
    int64_t quot = r / nr, tmp = t - quot * nt;
    t = nt;
    nt = tmp;
    tmp = r - quot * nr;
    r = nr;
    nr = tmp;
  }
  if (r != 1) return set_err(ERR_PARAM, "inv_mod: value not invertible");
  if (t < 0) t += (int64_t)q;
  *out = (uint64_t)t;
  return 0;
}

/* ========== Prng = mt19937_64 + hand-rolled draws (util/rng.hpp:19-68) ========== */
typedef struct {
  uint64_t mt[312];
  int mti;
  double spare;
  int have_spare;
} prng;

static void prng_init(prng* p, uint64_t seed) {
  p->mt[0] = seed;
  for (int i = 1; i < 312; ++i) p->mt[i] = 6364136223846793005ULL * (p->mt[i - 1] ^ (p->mt[i - 1] >> 62)) + (uint64_t)i;
  p->mti = 312;
  p->have_spare = 0;
  p->spare = 0.0;
}
static uint64_t prng_next(prng* p) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  if (p->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (p->mt[i] & UM) | (p->mt[i + 1] & LM);
      p->mt[i] = p->mt[i + 156] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    }
    for (; i < 311; ++i) {
      x = (p->mt[i] & UM) | (p->mt[i + 1] & LM);
      p->mt[i] = p->mt[i + 156 - 312] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    }
    x = (p->mt[311] & UM) | (p->mt[0] & LM);
    p->mt[311] = p->mt[155] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    p->mti = 0;
  }
  uint64_t x = p->mt[p->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}
static uint64_t prng_uniform(prng* p, uint64_t bound) {
  uint64_t limit = bound * (UINT64_MAX / bound), v;
  do v = prng_next(p);
  while (v >= limit);
  return v % bound;
}
static double prng_udouble(prng* p) { return (double)(prng_next(p) >> 11) * 0x1.0p-53; }
static double prng_gauss(prng* p) {
  if (p->have_spare) {
    p->have_spare = 0;
    return p->spare;
  }
  double u1, u2;
  do u1 = prng_udouble(p);
  while (u1 <= 0.0);
  u2 = prng_udouble(p);
  double mag = sqrt(-2.0 * log(u1));
  p->spare = mag * sin(6.283185307179586476925286766559 * u2);
  p->have_spare = 1;
  return mag * cos(6.283185307179586476925286766559 * u2);
}
void ho_prng(uint64_t seed, uint64_t count, uint64_t* raw, double* gauss, uint64_t* uni3) {
  prng a, b, c;
  prng_init(&a, seed);
  prng_init(&b, seed);
  prng_init(&c, seed);
  for (uint64_t i = 0; i < count; ++i) {
    raw[i] = prng_next(&a);
    gauss[i] = prng_gauss(&b);
    uni3[i] = prng_uniform(&c, 3);
  }
}

/* ========== samplers (ring/sampling.cpp:10-34, sampling.hpp:32-41) ========== */
static void sample_ternary(uint32_t n, prng* r, int8_t* v) {
  for (uint32_t i = 0; i < n; ++i) v[i] = (int8_t)((int)prng_uniform(r, 3) - 1);
}
static void sample_gaussian(uint32_t n, prng* r, int32_t* v) {
  const double sigma = 3.2, bound = 6.0 * sigma;
  for (uint32_t i = 0; i < n; ++i) {
    double x = prng_gauss(r) * sigma;
    if (x > bound) x = bound;
    if (x < -bound) x = -bound;
    v[i] = (int32_t)llround(x);
  }
}
static uint64_t lift1(int64_t x, uint64_t q) {
  uint64_t c = x >= 0 ? (uint64_t)x % q : q - ((uint64_t)(-x) % q);
  return c == q ? 0 : c;
}

/* ========== modulus (ring/modulus.cpp:22-85) ========== */
int ho_is_prime(uint64_t v) {
  static const uint64_t W[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (v < 2) return 0;
  for (int k = 0; k < 12; ++k) {
    if (v == W[k]) return 1;
    if (v % W[k] == 0) return 0;
  }
  uint64_t d = v - 1;
  int r = 0;
  while (!(d & 1)) {
    d >>= 1;
    ++r;
  }
  for (int k = 0; k < 12; ++k) {
    uint64_t x = pow_mod(W[k], d, v);
    if (x == 1 || x == v - 1) continue;
    int witness = 1;
    for (int i = 1; i < r; ++i) {
      x = mul_mod(x, x, v);
      if (x == v - 1) {
        witness = 0;
        break;
      }
    }
    if (witness) return 0;
  }
  return 1;
}

static int find_ntt_primes(int bits, uint32_t n, uint32_t count, uint64_t avoid, uint64_t* out) {
  if (bits < 8 || bits > 61) return set_err(ERR_PARAM, "prime size out of range");
  uint64_t two_n = 2ull * n, c = ((((1ull << bits) - 2) / two_n) * two_n) + 1;
  uint32_t got = 0;
  while (got < count && c > (1ull << (bits - 1))) {
    if (c != avoid && ho_is_prime(c)) out[got++] = c;
    if (c < two_n) break;
    c -= two_n;
  }
  if (got < count) return set_err(ERR_PARAM, "not enough NTT-friendly primes of the requested size");
  return 0;
}

uint64_t ho_primitive_root_2n(uint32_t n, uint64_t q) {
  uint64_t two_n = 2ull * n, e = (q - 1) / two_n;
  for (uint64_t c = 2; c < q; ++c) {
    uint64_t w = pow_mod(c, e, q);
    if (pow_mod(w, n, q) == q - 1) return w;
  }
  return 0;
}

/* ========== params (bfv/params.cpp:15-114) ========== */
static int max_q_bits_128(uint32_t n) {
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
static int bits_of(uint64_t v) { return (int)log2_exact(v) + 1; }

static int default_primes(uint32_t n, uint64_t t, uint64_t* q, uint32_t* L) {
  int bits = n >= 4096 ? 31 : 30;
  uint32_t count;
  if (n >= 4096) {
    count = t >= (1ull << 25) ? 6 : 4;
  } else {
    int tb = bits_of(t);
    count = (uint32_t)((7 * tb / 2 + 50 + 29) / 30);
    if (count < 2) count = 2;
  }
  if (count > MAXL) return set_err(ERR_PARAM, "modulus chain too long");
  *L = count;
  return find_ntt_primes(bits, n, count, t, q);
}

static int validate(uint32_t n, uint64_t t, const uint64_t* q, uint32_t L, int sec) {
  if (!is_pow2(n) || n < 8 || n > 32768) return set_err(ERR_PARAM, "ring degree must be a power of two in [8, 32768]");
  uint64_t two_n = 2ull * n;
  if (t < 2 || t % two_n != 1)
    return set_err(ERR_PARAM, "plaintext modulus %llu is not 1 mod 2n; slot batching is unavailable", (unsigned long long)t);
  if (!ho_is_prime(t)) return set_err(ERR_PARAM, "plaintext modulus must be prime");
  if (L == 0) return set_err(ERR_PARAM, "ciphertext modulus chain is empty");
  int total = 0;
  for (uint32_t i = 0; i < L; ++i) {
    if (!ho_is_prime(q[i]) || q[i] % two_n != 1 || q[i] == t) return set_err(ERR_PARAM, "bad ciphertext modulus");
    for (uint32_t j = 0; j < i; ++j)
      if (q[j] == q[i]) return set_err(ERR_PARAM, "duplicate ciphertext modulus");
    total += bits_of(q[i]);
  }
  if (sec == 0) return 0;
  if (sec != 128) return set_err(ERR_PARAM, "supported security levels: 0 (none), 128");
  int cap = max_q_bits_128(n);
  if (cap == 0) return set_err(ERR_PARAM, "no 128-bit security estimate for this ring degree");
  if (total > cap) return set_err(ERR_PARAM, "log2(q) exceeds the 128-bit ceiling");
  return 0;
}

/* FNV-1a over (n, t, security, q...) (params.cpp:68-82) */
static uint64_t params_hash(uint32_t n, uint64_t t, int sec, const uint64_t* q, uint32_t L) {
  uint64_t h = 0xcbf29ce484222325ull;
  uint64_t vals[3 + MAXL];
  vals[0] = n;
  vals[1] = t;
  vals[2] = (uint64_t)sec;
  for (uint32_t i = 0; i < L; ++i) vals[3 + i] = q[i];
  for (uint32_t k = 0; k < 3 + L; ++k)
    for (int i = 0; i < 8; ++i) {
      h ^= (vals[k] >> (8 * i)) & 0xff;
      h *= 0x100000001b3ull;
    }
  return h;
}

int ho_default_primes(uint32_t n, uint64_t t, int sec, uint64_t* out, uint32_t* count) {
  int rc = default_primes(n, t, out, count);
  if (rc) return rc;
  return validate(n, t, out, *count, sec);
}

/* ========== NTT tables + transforms (ring/ntt_tables.cpp:13-41,
 *            kernels/modops_scalar.cpp:45-81) ========== */
typedef struct {
  uint32_t n;
  uint64_t q;
  uint64_t *z, *zs, *iz, *izs;
  uint64_t inv_n, inv_n_s;
} ntt_tab;

static int ntt_tab_init(ntt_tab* T, uint32_t n, uint64_t q) {
  if (!is_pow2(n) || n < 2) return set_err(ERR_PARAM, "NTT size must be a power of two >= 2");
  if (!ho_is_prime(q)) return set_err(ERR_PARAM, "NTT modulus must be prime");
  if ((q - 1) % (2ull * n)) return set_err(ERR_PARAM, "modulus is not NTT-friendly for this n");
  uint64_t psi = ho_primitive_root_2n(n, q), psi_inv = 0;
  if (!psi) return set_err(ERR_PARAM, "no primitive root found");
  if (inv_mod(psi, q, &psi_inv)) return ERR_PARAM;
  T->n = n;
  T->q = q;
  T->z = malloc(4 * n * sizeof(uint64_t));
  T->zs = T->z + n;
  T->iz = T->z + 2 * n;
  T->izs = T->z + 3 * n;
  uint32_t logn = log2_exact(n);
  for (uint32_t k = 0; k < n; ++k) {
    uint32_t e = reverse_bits(k, logn);
    T->z[k] = pow_mod(psi, e, q);
    T->iz[k] = pow_mod(psi_inv, e, q);
    T->zs[k] = ho_shoup_precompute(T->z[k], q);
    T->izs[k] = ho_shoup_precompute(T->iz[k], q);
  }
  if (inv_mod(n, q, &T->inv_n)) return ERR_PARAM;
  T->inv_n_s = ho_shoup_precompute(T->inv_n, q);
  return 0;
}
static void ntt_tab_free(ntt_tab* T) { free(T->z); }

static void ntt_fwd(uint64_t* a, const ntt_tab* T) {
  const uint64_t q = T->q;
  size_t t = T->n >> 1;
  for (size_t m = 1; m < T->n; m <<= 1, t >>= 1)
    for (size_t i = 0; i < m; ++i) {
      const uint64_t z = T->z[m + i], zs = T->zs[m + i];
      uint64_t* p = a + 2 * i * t;
      for (size_t j = 0; j < t; ++j) {
        uint64_t x = p[j], y = shoup_mul(p[j + t], z, zs, q);
        p[j] = add_mod_1(x, y, q);
        p[j + t] = sub_mod_1(x, y, q);
      }
    }
}
static void ntt_inv(uint64_t* a, const ntt_tab* T) {
  const uint64_t q = T->q;
  size_t t = 1;
  for (size_t m = T->n >> 1; m >= 1; m >>= 1, t <<= 1)
    for (size_t i = 0; i < m; ++i) {
      const uint64_t z = T->iz[m + i], zs = T->izs[m + i];
      uint64_t* p = a + 2 * i * t;
      for (size_t j = 0; j < t; ++j) {
        uint64_t x = p[j], y = p[j + t];
        p[j] = add_mod_1(x, y, q);
        p[j + t] = shoup_mul(sub_mod_1(x, y, q), z, zs, q);
      }
    }
  for (size_t i = 0; i < T->n; ++i) a[i] = shoup_mul(a[i], T->inv_n, T->inv_n_s, q);
}

int ho_ntt(uint32_t n, uint64_t q, uint64_t* a, int inverse) {
  ntt_tab T;
  int rc = ntt_tab_init(&T, n, q);
  if (rc) return rc;
  if (inverse) ntt_inv(a, &T);
  else ntt_fwd(a, &T);
  ntt_tab_free(&T);
  return 0;
}
int ho_ntt_tables(uint32_t n, uint64_t q, uint64_t* zetas, uint64_t* inv_zetas, uint64_t* inv_n) {
  ntt_tab T;
  int rc = ntt_tab_init(&T, n, q);
  if (rc) return rc;
  memcpy(zetas, T.z, n * 8);
  memcpy(inv_zetas, T.iz, n * 8);
  *inv_n = T.inv_n;
  ntt_tab_free(&T);
  return 0;
}

/* ========== automorphisms (ring/poly.cpp:107-148) ========== */
static void galois_perm(uint32_t n, uint64_t g, uint32_t* perm) {
  uint32_t logn = log2_exact(n);
  uint64_t two_n = 2ull * n;
  for (uint32_t i = 0; i < n; ++i) {
    uint64_t e = 2ull * reverse_bits(i, logn) + 1, src = (e * g) % two_n;
    perm[i] = reverse_bits((uint32_t)((src - 1) / 2), logn);
  }
}
int ho_galois_perm(uint32_t n, uint64_t elt, uint32_t* out) {
  if (!(elt & 1)) return set_err(ERR_PARAM, "galois element must be odd");
  galois_perm(n, elt, out);
  return 0;
}

/* ========== fixed-width unsigned bignum for decrypt (context.cpp:316-370) ==== */
#define BN 8
typedef struct {
  uint64_t w[BN];
} bn;
static void bn_set(bn* a, uint64_t v) {
  memset(a, 0, sizeof *a);
  a->w[0] = v;
}
static int bn_cmp(const bn* a, const bn* b) {
  for (int i = BN - 1; i >= 0; --i)
    if (a->w[i] != b->w[i]) return a->w[i] < b->w[i] ? -1 : 1;
  return 0;
}
static void bn_add(bn* r, const bn* a, const bn* b) {
  u128 c = 0;
  for (int i = 0; i < BN; ++i) {
    c += (u128)a->w[i] + b->w[i];
    r->w[i] = (uint64_t)c;
    c >>= 64;
  }
}
static void bn_sub(bn* r, const bn* a, const bn* b) { /* a >= b */
  uint64_t br = 0;
  for (int i = 0; i < BN; ++i) {
    uint64_t ai = a->w[i], bi = b->w[i], d = ai - bi - br;
    br = (ai < bi) || (ai == bi && br);
    r->w[i] = d;
  }
}
static void bn_mul_u64(bn* r, const bn* a, uint64_t m) {
  u128 c = 0;
  for (int i = 0; i < BN; ++i) {
    c += (u128)a->w[i] * m;
    r->w[i] = (uint64_t)c;
    c >>= 64;
  }
}
static uint64_t bn_divmod_u64(bn* q, const bn* a, uint64_t d) {
  u128 rem = 0;
  for (int i = BN - 1; i >= 0; --i) {
    u128 cur = (rem << 64) | a->w[i];
    q->w[i] = (uint64_t)(cur / d);
    rem = cur % d;
  }
  return (uint64_t)rem;
}
static int bn_msb(const bn* a) {
  for (int i = BN - 1; i >= 0; --i)
    if (a->w[i]) return i * 64 + 63 - __builtin_clzll(a->w[i]);
  return -1;
}
static void bn_shl1(bn* a) {
  for (int i = BN - 1; i > 0; --i) a->w[i] = (a->w[i] << 1) | (a->w[i - 1] >> 63);
  a->w[0] <<= 1;
}
static void bn_shr1(bn* a) {
  for (int i = 0; i < BN - 1; ++i) a->w[i] = (a->w[i] >> 1) | (a->w[i + 1] << 63);
  a->w[BN - 1] >>= 1;
}
/* quotient (small) and remainder of a / d, shift-subtract */
static uint64_t bn_divmod_small_q(const bn* a, const bn* d, bn* rem) {
  *rem = *a;
  int ma = bn_msb(a), md = bn_msb(d);
  uint64_t qv = 0;
  if (ma < md) return 0;
  int shift = ma - md;
  bn dd = *d;
  for (int s = 0; s < shift; ++s) bn_shl1(&dd);
  for (int s = shift; s >= 0; --s) {
    if (bn_cmp(rem, &dd) >= 0) {
      bn_sub(rem, rem, &dd);
      qv |= 1ull << s; /* quotient < 2^64 by construction (< t*L) */
    }
    bn_shr1(&dd);
  }
  return qv;
}

/* ========== BFV context, one branch (bfv/context.cpp:27-71) ========== */
typedef struct {
  uint32_t n, logn, L;
  uint64_t t, hash;
  int sec;
  uint64_t q[MAXL];
  ntt_tab qt[MAXL], tt;
  uint64_t delta[MAXL], delta_s[MAXL];
  uint32_t* index_map;
  uint32_t num_elts;     /* steps 1..n/4 then swap, generation order */
  uint64_t gen_elts[32]; /* generation order (context.cpp:209-211) */
  uint32_t* perms;       /* [num_elts][n], generation order */
  /* decrypt precompute (context.cpp:35-48) */
  bn Q, Q_half, Q_punct[MAXL];
  uint64_t y[MAXL];
  int q_msb;
} ctx;

typedef struct {
  int8_t* s;               /* secret over the integers [n] */
  uint64_t* pk;            /* [2][L][n] coeff: p0, p1 */
  uint64_t *ppk, *ppk_s;   /* prepared public key, eval [2][L][n] */
  uint64_t *sp, *sp_s;     /* prepared secret [L][n] */
  uint64_t *gk, *gk_s;     /* [num_elts gen order][L][2][L][n] */
} keys;

static uint64_t elt_for_step(uint32_t n, uint32_t s) { return pow_mod(3, s, 2ull * n); }

static int ctx_init(ctx* c, uint32_t n, uint64_t t, int sec) {
  memset(c, 0, sizeof *c);
  int rc = default_primes(n, t, c->q, &c->L);
  if (rc) return rc;
  if ((rc = validate(n, t, c->q, c->L, sec))) return rc;
  c->n = n;
  c->logn = log2_exact(n);
  c->t = t;
  c->sec = sec;
  c->hash = params_hash(n, t, sec, c->q, c->L);
  if ((rc = ntt_tab_init(&c->tt, n, t))) return rc;
  for (uint32_t i = 0; i < c->L; ++i)
    if ((rc = ntt_tab_init(&c->qt[i], n, c->q[i]))) return rc;
  /* Q, Delta = floor(Q/t) mod q_i, Q/q_i, (Q/q_i)^-1 mod q_i */
  bn_set(&c->Q, 1);
  for (uint32_t i = 0; i < c->L; ++i) bn_mul_u64(&c->Q, &c->Q, c->q[i]);
  c->Q_half = c->Q;
  bn_shr1(&c->Q_half);
  bn delta_big;
  bn_divmod_u64(&delta_big, &c->Q, t);
  for (uint32_t i = 0; i < c->L; ++i) {
    bn tmp;
    uint64_t r = bn_divmod_u64(&c->Q_punct[i], &c->Q, c->q[i]);
    (void)r;
    uint64_t pm = bn_divmod_u64(&tmp, &c->Q_punct[i], c->q[i]);
    if (inv_mod(pm, c->q[i], &c->y[i])) return ERR_PARAM;
    c->delta[i] = bn_divmod_u64(&tmp, &delta_big, c->q[i]);
    c->delta_s[i] = ho_shoup_precompute(c->delta[i], c->q[i]);
  }
  c->q_msb = bn_msb(&c->Q);
  /* slot index map, generator 3 (context.cpp:50-63) */
  c->index_map = malloc(n * sizeof(uint32_t));
  uint64_t m = 2ull * n, pos = 1;
  for (uint32_t i = 0; i < n / 2; ++i) {
    uint32_t i1 = (uint32_t)((pos - 1) >> 1), i2 = (uint32_t)((m - pos - 1) >> 1);
    c->index_map[i] = reverse_bits(i1, c->logn);
    c->index_map[i + n / 2] = reverse_bits(i2, c->logn);
    pos = (pos * 3) % m;
  }
  /* galois elements: steps 1, 2, ..., n/4 then the swap 2n-1 (context.cpp:189-211) */
  c->num_elts = 0;
  for (uint32_t s = 1; s <= n / 4; s <<= 1) c->gen_elts[c->num_elts++] = elt_for_step(n, s);
  c->gen_elts[c->num_elts++] = 2ull * n - 1;
  c->perms = malloc((size_t)c->num_elts * n * sizeof(uint32_t));
  for (uint32_t e = 0; e < c->num_elts; ++e) galois_perm(n, c->gen_elts[e], c->perms + (size_t)e * n);
  return 0;
}
static void ctx_free(ctx* c) {
  ntt_tab_free(&c->tt);
  for (uint32_t i = 0; i < c->L; ++i) ntt_tab_free(&c->qt[i]);
  free(c->index_map);
  free(c->perms);
}
static int elt_index(const ctx* c, uint64_t elt) {
  for (uint32_t e = 0; e < c->num_elts; ++e)
    if (c->gen_elts[e] == elt) return (int)e;
  return -1;
}

/* encode_slots (context.cpp:80-93): slots -> coeff-form plaintext mod t */
static int encode_slots(const ctx* c, const uint64_t* slots, size_t cnt, uint64_t* pt) {
  if (cnt > c->n) return set_err(ERR_PARAM, "encode_slots: more values than slots");
  memset(pt, 0, c->n * 8);
  for (size_t i = 0; i < cnt; ++i) {
    if (slots[i] >= c->t) return set_err(ERR_RANGE, "encode_slots: slot %zu value not reduced mod t", i);
    pt[c->index_map[i]] = slots[i];
  }
  ntt_inv(pt, &c->tt);
  return 0;
}
/* decode_slots (context.cpp:95-102) */
static void decode_slots(const ctx* c, const uint64_t* pt, uint64_t* slots) {
  uint64_t* buf = malloc(c->n * 8);
  memcpy(buf, pt, c->n * 8);
  ntt_fwd(buf, &c->tt);
  for (uint32_t i = 0; i < c->n; ++i) slots[i] = buf[c->index_map[i]];
  free(buf);
}
/* prepare_plain (context.cpp:104-118): out [L][n] values (+ shoup) */
static void prepare_plain(const ctx* c, const uint64_t* pt, uint64_t* vals, uint64_t* shoup) {
  for (uint32_t i = 0; i < c->L; ++i) {
    uint64_t* v = vals + (size_t)i * c->n;
    for (uint32_t j = 0; j < c->n; ++j) v[j] = pt[j] % c->q[i];
    ntt_fwd(v, &c->qt[i]);
    if (shoup)
      for (uint32_t j = 0; j < c->n; ++j) shoup[(size_t)i * c->n + j] = ho_shoup_precompute(v[j], c->q[i]);
  }
}
/* delta_times (context.cpp:253-260) */
static void delta_times(const ctx* c, const uint64_t* m, uint32_t i, uint64_t* out) {
  for (uint32_t j = 0; j < c->n; ++j) out[j] = shoup_mul(m[j], c->delta[i], c->delta_s[i], c->q[i]);
}

/* keygen (context.cpp:139-173) */
static void prepared_secret(const ctx* c, keys* k) {
  k->sp = malloc((size_t)c->L * c->n * 8);
  k->sp_s = malloc((size_t)c->L * c->n * 8);
  for (uint32_t i = 0; i < c->L; ++i) {
    uint64_t* v = k->sp + (size_t)i * c->n;
    for (uint32_t j = 0; j < c->n; ++j) v[j] = lift1(k->s[j], c->q[i]);
    ntt_fwd(v, &c->qt[i]);
    for (uint32_t j = 0; j < c->n; ++j) k->sp_s[(size_t)i * c->n + j] = ho_shoup_precompute(v[j], c->q[i]);
  }
}
static void keygen(const ctx* c, prng* rng, keys* k) {
  const uint32_t n = c->n, L = c->L;
  k->s = malloc(n);
  sample_ternary(n, rng, k->s);
  prepared_secret(c, k);
  int32_t* e = malloc(n * sizeof(int32_t));
  sample_gaussian(n, rng, e);
  k->pk = malloc(2ull * L * n * 8);
  uint64_t* as = malloc(n * 8);
  for (uint32_t i = 0; i < L; ++i) {
    const uint64_t q = c->q[i];
    uint64_t* a = k->pk + ((size_t)L + i) * n;
    for (uint32_t j = 0; j < n; ++j) a[j] = prng_uniform(rng, q);
    memcpy(as, a, n * 8);
    ntt_fwd(as, &c->qt[i]);
    for (uint32_t j = 0; j < n; ++j) as[j] = shoup_mul(as[j], k->sp[(size_t)i * n + j], k->sp_s[(size_t)i * n + j], q);
    ntt_inv(as, &c->qt[i]);
    uint64_t* p0 = k->pk + (size_t)i * n;
    for (uint32_t j = 0; j < n; ++j) p0[j] = neg_mod_1(add_mod_1(as[j], lift1(e[j], q), q), q);
  }
  /* prepare_public (context.cpp:175-187) */
  k->ppk = malloc(2ull * L * n * 8);
  k->ppk_s = malloc(2ull * L * n * 8);
  for (uint32_t r = 0; r < 2 * L; ++r) {
    uint32_t i = r % L;
    uint64_t* v = k->ppk + (size_t)r * n;
    memcpy(v, k->pk + (size_t)r * n, n * 8);
    ntt_fwd(v, &c->qt[i]);
    for (uint32_t j = 0; j < n; ++j) k->ppk_s[(size_t)r * n + j] = ho_shoup_precompute(v[j], c->q[i]);
  }
  free(e);
  free(as);
}

/* make_galois_keys (context.cpp:201-251) */
static void make_galois_keys(const ctx* c, prng* rng, keys* k) {
  const uint32_t n = c->n, L = c->L;
  const size_t per_elt = (size_t)L * 2 * L * n;
  k->gk = malloc(c->num_elts * per_elt * 8);
  k->gk_s = malloc(c->num_elts * per_elt * 8);
  int8_t* sg = malloc(n);
  int32_t* el = malloc(n * sizeof(int32_t));
  uint64_t* w = malloc(n * 8);
  for (uint32_t e = 0; e < c->num_elts; ++e) {
    const uint64_t elt = c->gen_elts[e], two_n = 2ull * n;
    memset(sg, 0, n);
    for (uint32_t j = 0; j < n; ++j) {
      uint64_t tgt = ((uint64_t)j * elt) % two_n;
      if (tgt < n) sg[tgt] = k->s[j];
      else sg[tgt - n] = (int8_t)(-k->s[j]);
    }
    for (uint32_t l = 0; l < L; ++l) {
      sample_gaussian(n, rng, el);
      for (uint32_t i = 0; i < L; ++i) {
        const uint64_t q = c->q[i];
        uint64_t* b = k->gk + e * per_elt + (((size_t)l * 2 + 0) * L + i) * n;
        uint64_t* a = k->gk + e * per_elt + (((size_t)l * 2 + 1) * L + i) * n;
        for (uint32_t j = 0; j < n; ++j) a[j] = prng_uniform(rng, q);
        for (uint32_t j = 0; j < n; ++j) b[j] = shoup_mul(a[j], k->sp[(size_t)i * n + j], k->sp_s[(size_t)i * n + j], q);
        for (uint32_t j = 0; j < n; ++j) w[j] = lift1(el[j], q);
        ntt_fwd(w, &c->qt[i]);
        for (uint32_t j = 0; j < n; ++j) b[j] = neg_mod_1(add_mod_1(b[j], w[j], q), q);
        if (i == l) {
          for (uint32_t j = 0; j < n; ++j) w[j] = lift1(sg[j], q);
          ntt_fwd(w, &c->qt[i]);
          for (uint32_t j = 0; j < n; ++j) b[j] = add_mod_1(b[j], w[j], q);
        }
        uint64_t* bs = k->gk_s + (b - k->gk);
        uint64_t* as = k->gk_s + (a - k->gk);
        for (uint32_t j = 0; j < n; ++j) {
          bs[j] = ho_shoup_precompute(b[j], q);
          as[j] = ho_shoup_precompute(a[j], q);
        }
      }
    }
  }
  free(sg);
  free(el);
  free(w);
}
static void keys_free(keys* k) {
  free(k->s);
  free(k->pk);
  free(k->ppk);
  free(k->ppk_s);
  free(k->sp);
  free(k->sp_s);
  free(k->gk);
  free(k->gk_s);
}

/* encrypt_parts, eval form out (context.cpp:262-314) */
static void encrypt_eval(const ctx* c, const keys* k, prng* rng, const uint64_t* pt, uint64_t* ct) {
  const uint32_t n = c->n, L = c->L;
  int8_t* u = malloc(n);
  int32_t* e0 = malloc(n * 4);
  int32_t* e1 = malloc(n * 4);
  sample_ternary(n, rng, u);
  sample_gaussian(n, rng, e0);
  sample_gaussian(n, rng, e1);
  uint64_t *ui = malloc(n * 8), *n0 = malloc(n * 8), *dm = malloc(n * 8);
  for (uint32_t i = 0; i < L; ++i) {
    const uint64_t q = c->q[i];
    uint64_t* c0 = ct + (size_t)i * n;
    uint64_t* c1 = ct + ((size_t)L + i) * n;
    for (uint32_t j = 0; j < n; ++j) ui[j] = lift1(u[j], q);
    ntt_fwd(ui, &c->qt[i]);
    const uint64_t *p0 = k->ppk + (size_t)i * n, *p0s = k->ppk_s + (size_t)i * n;
    const uint64_t *p1 = k->ppk + ((size_t)L + i) * n, *p1s = k->ppk_s + ((size_t)L + i) * n;
    for (uint32_t j = 0; j < n; ++j) {
      c0[j] = shoup_mul(ui[j], p0[j], p0s[j], q);
      c1[j] = shoup_mul(ui[j], p1[j], p1s[j], q);
    }
    delta_times(c, pt, i, dm);
    for (uint32_t j = 0; j < n; ++j) n0[j] = add_mod_1(lift1(e0[j], q), dm[j], q);
    ntt_fwd(n0, &c->qt[i]);
    for (uint32_t j = 0; j < n; ++j) c0[j] = add_mod_1(c0[j], n0[j], q);
    for (uint32_t j = 0; j < n; ++j) n0[j] = lift1(e1[j], q);
    ntt_fwd(n0, &c->qt[i]);
    for (uint32_t j = 0; j < n; ++j) c1[j] = add_mod_1(c1[j], n0[j], q);
  }
  free(u);
  free(e0);
  free(e1);
  free(ui);
  free(n0);
  free(dm);
}

/* decrypt_core (context.cpp:316-370); ct [2][L][n] in form (1 eval). */
static int decrypt_core(const ctx* c, const keys* k, const uint64_t* ct, int form, uint64_t* m, int* budget) {
  const uint32_t n = c->n, L = c->L;
  uint64_t* w = malloc((size_t)L * n * 8);
  for (uint32_t i = 0; i < L; ++i) {
    const uint64_t q = c->q[i];
    uint64_t* wi = w + (size_t)i * n;
    const uint64_t *c0 = ct + (size_t)i * n, *c1 = ct + ((size_t)L + i) * n;
    memcpy(wi, c1, n * 8);
    if (!form) ntt_fwd(wi, &c->qt[i]);
    for (uint32_t j = 0; j < n; ++j) wi[j] = shoup_mul(wi[j], k->sp[(size_t)i * n + j], k->sp_s[(size_t)i * n + j], q);
    if (form) {
      for (uint32_t j = 0; j < n; ++j) wi[j] = add_mod_1(wi[j], c0[j], q);
      ntt_inv(wi, &c->qt[i]);
    } else {
      ntt_inv(wi, &c->qt[i]);
      for (uint32_t j = 0; j < n; ++j) wi[j] = add_mod_1(wi[j], c0[j], q);
    }
  }
  bn max_r;
  bn_set(&max_r, 0);
  for (uint32_t j = 0; j < n; ++j) {
    bn acc, tmp, z, num, rem;
    bn_set(&acc, 0);
    for (uint32_t i = 0; i < L; ++i) {
      uint64_t cc = mul_mod(w[(size_t)i * n + j], c->y[i], c->q[i]);
      bn_mul_u64(&tmp, &c->Q_punct[i], cc);
      bn_add(&acc, &acc, &tmp);
    }
    while (bn_cmp(&acc, &c->Q) >= 0) bn_sub(&acc, &acc, &c->Q);
    bn_mul_u64(&z, &acc, c->t);
    bn_add(&num, &z, &c->Q_half);
    uint64_t quot = bn_divmod_small_q(&num, &c->Q, &rem);
    m[j] = quot % c->t;
    /* r = z - quot*Q = rem - Q_half, |r| */
    bn r;
    if (bn_cmp(&rem, &c->Q_half) >= 0) bn_sub(&r, &rem, &c->Q_half);
    else bn_sub(&r, &c->Q_half, &rem);
    if (bn_cmp(&r, &max_r) > 0) max_r = r;
  }
  int msb = bn_msb(&max_r);
  if (msb < 0) *budget = c->q_msb - 1;
  else {
    *budget = c->q_msb - (msb + 1);
    if (*budget < 0) *budget = 0;
  }
  free(w);
  return 0;
}

/* apply_galois, eval-form path (context.cpp:428-507); ct [2][L][n] */
static void apply_galois(const ctx* c, const keys* k, int e, const uint64_t* in, uint64_t* out) {
  const uint32_t n = c->n, L = c->L;
  const uint32_t* perm = c->perms + (size_t)e * n;
  const size_t per_elt = (size_t)L * 2 * L * n;
  uint64_t* digits = malloc((size_t)L * n * 8);
  uint64_t* d = malloc(n * 8);
  uint64_t* acc1 = out + (size_t)L * n;
  for (uint32_t i = 0; i < L; ++i) {
    const uint64_t* c1 = in + ((size_t)L + i) * n;
    uint64_t* dg = digits + (size_t)i * n;
    for (uint32_t j = 0; j < n; ++j) dg[j] = c1[perm[j]];
    ntt_inv(dg, &c->qt[i]);
  }
  memset(out, 0, 2ull * L * n * 8);
  for (uint32_t l = 0; l < L; ++l)
    for (uint32_t i = 0; i < L; ++i) {
      const uint64_t qi = c->q[i];
      const uint64_t* dg = digits + (size_t)l * n;
      if (i == l) memcpy(d, dg, n * 8);
      else
        for (uint32_t j = 0; j < n; ++j) d[j] = dg[j] % qi;
      ntt_fwd(d, &c->qt[i]);
      const uint64_t* k0 = k->gk + e * per_elt + (((size_t)l * 2 + 0) * L + i) * n;
      const uint64_t* k1 = k->gk + e * per_elt + (((size_t)l * 2 + 1) * L + i) * n;
      const uint64_t* k0s = k->gk_s + (k0 - k->gk);
      const uint64_t* k1s = k->gk_s + (k1 - k->gk);
      uint64_t* a0 = out + (size_t)i * n;
      uint64_t* a1 = acc1 + (size_t)i * n;
      for (uint32_t j = 0; j < n; ++j) {
        a0[j] = add_mod_1(a0[j], shoup_mul(d[j], k0[j], k0s[j], qi), qi);
        a1[j] = add_mod_1(a1[j], shoup_mul(d[j], k1[j], k1s[j], qi), qi);
      }
    }
  for (uint32_t i = 0; i < L; ++i) {
    const uint64_t* c0 = in + (size_t)i * n;
    uint64_t* a0 = out + (size_t)i * n;
    for (uint32_t j = 0; j < n; ++j) a0[j] = add_mod_1(a0[j], c0[perm[j]], c->q[i]);
  }
  free(digits);
  free(d);
}

static void ct_add(const ctx* c, uint64_t* a, const uint64_t* b) {
  for (uint32_t r = 0; r < 2 * c->L; ++r) {
    const uint64_t q = c->q[r % c->L];
    uint64_t* x = a + (size_t)r * c->n;
    const uint64_t* y = b + (size_t)r * c->n;
    for (uint32_t j = 0; j < c->n; ++j) x[j] = add_mod_1(x[j], y[j], q);
  }
}
/* mul_plain with prepared values (no shoup table: computed per element) */
static void ct_mul_plain(const ctx* c, uint64_t* a, const uint64_t* pv, const uint64_t* ps) {
  for (uint32_t r = 0; r < 2 * c->L; ++r) {
    uint32_t i = r % c->L;
    const uint64_t q = c->q[i];
    uint64_t* x = a + (size_t)r * c->n;
    const uint64_t* v = pv + (size_t)i * c->n;
    const uint64_t* s = ps + (size_t)i * c->n;
    for (uint32_t j = 0; j < c->n; ++j) x[j] = shoup_mul(x[j], v[j], s[j], q);
  }
}
static void ct_to_eval(const ctx* c, uint64_t* a) {
  for (uint32_t r = 0; r < 2 * c->L; ++r) ntt_fwd(a + (size_t)r * c->n, &c->qt[r % c->L]);
}

/* sum_all_slots (bfv/backend.cpp:63-73) */
static void sum_all_slots(const ctx* c, const keys* k, uint64_t* acc) {
  const size_t w = 2ull * c->L * c->n;
  uint64_t* rot = malloc(w * 8);
  for (uint32_t s = 1; s <= c->n / 4; s <<= 1) {
    apply_galois(c, k, elt_index(c, elt_for_step(c->n, s)), acc, rot);
    ct_add(c, acc, rot);
  }
  apply_galois(c, k, elt_index(c, 2ull * c->n - 1), acc, rot);
  ct_add(c, acc, rot);
  free(rot);
}

/* ========== twin (fpcrt/twin.cpp) + fixed point (fixed_point.cpp) ========== */
struct ho_twin {
  uint32_t n;
  uint64_t t[2];
  uint32_t s_x, s_w, in_bits;
  ctx c[2];
  keys k[2];
  prng enc[2]; /* client encryption RNG per branch, seed enc_seed + b */
};

static uint64_t centered_residue(int64_t v, uint64_t t) {
  __int128 r = (__int128)v % (__int128)t;
  if (r < 0) r += t;
  return (uint64_t)r;
}
static int64_t max_centered(uint64_t t0, uint64_t t1) { return (int64_t)(((u128)t0 * t1 - 1) / 2); }

static size_t twin_ct_words(const ho_twin* h) { return 2ull * (h->c[0].L + h->c[1].L) * h->n; }
static size_t twin_pt_words(const ho_twin* h) { return (size_t)(h->c[0].L + h->c[1].L) * h->n; }

/* encode_signed (twin.cpp:95-111): coeff plaintexts per branch [2][n] */
static int encode_signed(const ho_twin* h, const int64_t* vals, size_t cnt, uint64_t* pt2) {
  int64_t lim = max_centered(h->t[0], h->t[1]);
  uint64_t* slots = malloc((cnt ? cnt : 1) * 8);
  int rc = 0;
  for (int b = 0; b < 2 && !rc; ++b) {
    for (size_t i = 0; i < cnt; ++i) {
      if (vals[i] > lim || vals[i] < -lim) {
        rc = set_err(ERR_RANGE, "encode_signed: value outside the centered range");
        break;
      }
      slots[i] = centered_residue(vals[i], h->t[b]);
    }
    if (!rc) rc = encode_slots(&h->c[b], slots, cnt, pt2 + (size_t)b * h->n);
  }
  free(slots);
  return rc;
}

int ho_twin_create(ho_twin** out, uint32_t n, uint64_t t0, uint64_t t1, int sec, uint32_t s_x, uint32_t s_w,
                   uint32_t in_bits, uint64_t key_seed, uint64_t enc_seed) {
  ho_twin* h = calloc(1, sizeof *h);
  h->n = n;
  h->t[0] = t0;
  h->t[1] = t1;
  h->s_x = s_x;
  h->s_w = s_w;
  h->in_bits = in_bits;
  int rc;
  if (t0 == t1) {
    free(h);
    return set_err(ERR_PARAM, "twin moduli must differ");
  }
  for (int b = 0; b < 2; ++b)
    if ((rc = ctx_init(&h->c[b], n, h->t[b], sec))) {
      free(h);
      return rc;
    }
  /* TwinContext::keygen (twin.cpp:41-48): one rng across both branches */
  prng rng;
  prng_init(&rng, key_seed);
  for (int b = 0; b < 2; ++b) {
    keygen(&h->c[b], &rng, &h->k[b]);
    make_galois_keys(&h->c[b], &rng, &h->k[b]);
  }
  for (int b = 0; b < 2; ++b) prng_init(&h->enc[b], enc_seed + (uint64_t)b);
  *out = h;
  return 0;
}

void ho_twin_destroy(ho_twin* h) {
  if (!h) return;
  for (int b = 0; b < 2; ++b) {
    keys_free(&h->k[b]);
    ctx_free(&h->c[b]);
  }
  free(h);
}

static void sorted_elts(const ctx* c, uint64_t* out, int* order) {
  uint32_t m = c->num_elts;
  for (uint32_t i = 0; i < m; ++i) order[i] = (int)i;
  for (uint32_t i = 0; i < m; ++i)
    for (uint32_t j = i + 1; j < m; ++j)
      if (c->gen_elts[order[j]] < c->gen_elts[order[i]]) {
        int t = order[i];
        order[i] = order[j];
        order[j] = t;
      }
  for (uint32_t i = 0; i < m; ++i) out[i] = c->gen_elts[order[i]];
}

int ho_twin_info(const ho_twin* h, uint32_t* L, uint64_t* q, uint64_t* hash, uint64_t* elts) {
  size_t o = 0;
  for (int b = 0; b < 2; ++b) {
    if (L) L[b] = h->c[b].L;
    if (hash) hash[b] = h->c[b].hash;
    for (uint32_t i = 0; i < h->c[b].L; ++i)
      if (q) q[o++] = h->c[b].q[i];
  }
  int order[32];
  uint64_t tmp[32];
  sorted_elts(&h->c[0], elts ? elts : tmp, order);
  return (int)h->c[0].num_elts;
}

int ho_twin_export_keys(const ho_twin* h, uint64_t* gk0, uint64_t* gk1, int8_t* sk, uint64_t* pk) {
  uint64_t* gk[2] = {gk0, gk1};
  for (int b = 0; b < 2; ++b) {
    const ctx* c = &h->c[b];
    const size_t per_elt = (size_t)c->L * 2 * c->L * c->n;
    int order[32];
    uint64_t e_sorted[32];
    sorted_elts(c, e_sorted, order);
    if (gk[b])
      for (uint32_t e = 0; e < c->num_elts; ++e)
        memcpy(gk[b] + e * per_elt, h->k[b].gk + (size_t)order[e] * per_elt, per_elt * 8);
    if (sk) memcpy(sk + (size_t)b * h->n, h->k[b].s, h->n);
    if (pk) {
      memcpy(pk, h->k[b].pk, 2ull * c->L * c->n * 8);
      pk += 2ull * c->L * c->n;
    }
  }
  return 0;
}

/* encode_input_row / encode_inputs (matmul.cpp:59-81), client encrypt */
int ho_encode_inputs(ho_twin* h, const int64_t* x, uint64_t R, uint64_t f, uint64_t* out) {
  if (R == 0 || f == 0) return set_err(ERR_PARAM, "encode_inputs: empty matrix");
  const uint32_t n = h->n;
  const uint64_t kc = (f + n - 1) / n;
  uint64_t* pt = malloc(2ull * n * 8);
  int rc = 0;
  for (uint64_t r = 0; r < R && !rc; ++r)
    for (uint64_t k = 0; k < kc && !rc; ++k) {
      size_t len = (size_t)((f - k * n) < n ? (f - k * n) : n);
      if ((rc = encode_signed(h, x + r * f + k * n, len, pt))) break;
      uint64_t* o = out + (r * kc + k) * twin_ct_words(h);
      encrypt_eval(&h->c[0], &h->k[0], &h->enc[0], pt, o);
      encrypt_eval(&h->c[1], &h->k[1], &h->enc[1], pt + n, o + 2ull * h->c[0].L * n);
    }
  free(pt);
  return rc;
}

/* encode_weights (matmul.cpp:83-104): out [cols][k][twin plain] values */
int ho_encode_weights(ho_twin* h, const int64_t* w, uint64_t f, uint64_t cols, uint64_t* out) {
  if (f == 0 || cols == 0) return set_err(ERR_PARAM, "encode_weights: empty matrix");
  const uint32_t n = h->n;
  const uint64_t kc = (f + n - 1) / n;
  int64_t* slots = malloc(n * 8);
  uint64_t* pt = malloc(2ull * n * 8);
  int rc = 0;
  for (uint64_t j = 0; j < cols && !rc; ++j)
    for (uint64_t k = 0; k < kc && !rc; ++k) {
      size_t len = (size_t)((f - k * n) < n ? (f - k * n) : n);
      for (size_t s = 0; s < len; ++s) slots[s] = w[(k * n + s) * cols + j];
      if ((rc = encode_signed(h, slots, len, pt))) break;
      uint64_t* o = out + (j * kc + k) * twin_pt_words(h);
      prepare_plain(&h->c[0], pt, o, NULL);
      prepare_plain(&h->c[1], pt + n, o + (size_t)h->c[0].L * n, NULL);
    }
  free(slots);
  free(pt);
  return rc;
}

/* mask_for_slot (matmul.cpp:146-163): prepared one-hot at `slot` */
static int make_mask(const ho_twin* h, uint32_t slot, uint64_t* vals, uint64_t* shoup) {
  int64_t* onehot = calloc(h->n, 8);
  uint64_t* pt = malloc(2ull * h->n * 8);
  onehot[slot] = 1;
  int rc = encode_signed(h, onehot, h->n, pt);
  if (!rc) {
    prepare_plain(&h->c[0], pt, vals, shoup);
    prepare_plain(&h->c[1], pt + h->n, vals + (size_t)h->c[0].L * h->n, shoup ? shoup + (size_t)h->c[0].L * h->n : NULL);
  }
  free(onehot);
  free(pt);
  return rc;
}
int ho_mask(ho_twin* h, uint32_t slot, uint64_t* out) {
  if (slot >= h->n) return set_err(ERR_PARAM, "slot out of range");
  return make_mask(h, slot, out, NULL);
}

/* capacity_check (fixed_point.cpp:55-77) */
int ho_capacity_ok(uint64_t f, uint32_t s_x, uint32_t s_w, uint32_t in_bits, uint64_t t0, uint64_t t1) {
  if (f == 0) return 0;
  int log_f = f == 1 ? 0 : 64 - __builtin_clzll(f - 1);
  int required = (int)(in_bits + s_x + s_w) + log_f;
  u128 prod = (u128)t0 * t1;
  int cap = -1;
  while (prod) {
    ++cap;
    prod >>= 1;
  }
  return required + 1 <= cap;
}

int ho_scale_value(double x, uint32_t e, int64_t* out) {
  if (!isfinite(x)) return set_err(ERR_RANGE, "scale_value: non-finite input");
  if (e > 62) return set_err(ERR_PARAM, "scale_value: exponent too large");
  double scaled = ldexp(x, (int)e);
  double limit = (double)max_centered(1073872897ull, 114689ull);
  if (!(fabs(scaled) <= limit)) return set_err(ERR_RANGE, "scale_value: exceeds the plaintext capacity");
  *out = llround(scaled);
  return 0;
}

/* proposed_counts / baseline_counts (matmul.cpp:30-57) */
int ho_proposed_counts(uint64_t R, uint64_t cols, uint64_t f, uint32_t n, uint64_t* c) {
  if (!R || !cols || !f) return set_err(ERR_PARAM, "empty shape");
  if (!is_pow2(n)) return set_err(ERR_PARAM, "ring degree must be a power of two");
  uint64_t k = (f + n - 1) / n, lg = log2_exact(n);
  c[0] = R * cols * (k + 1);
  c[1] = R * cols * lg;
  c[2] = R * cols * (k + lg);
  c[3] = R * k;
  c[4] = (R * cols + n - 1) / n;
  return 0;
}
int ho_baseline_counts(uint64_t R, uint64_t cols, uint64_t f, uint32_t n, uint64_t* c) {
  if (!R || !cols || !f) return set_err(ERR_PARAM, "empty shape");
  if (!is_pow2(n)) return set_err(ERR_PARAM, "ring degree must be a power of two");
  uint64_t blocks = (R + n - 1) / n;
  c[0] = blocks * f * cols;
  c[1] = 0;
  c[2] = blocks * cols * f;
  c[3] = blocks * f;
  c[4] = blocks * cols;
  return 0;
}

/* ---- fast matmul: MatmulStream (matmul.cpp:114-255) ---- */
typedef struct {
  ho_twin* h;
  const uint64_t* inputs;
  int form;
  uint64_t R, cols, kc;
  const uint64_t *wv, *ws; /* prepared weights values + shoup [cols][k][twin plain] */
  uint64_t* acc;            /* [C][twin ct] */
  unsigned char* acc_set;
  pthread_mutex_t* mu;
  uint64_t r_lo, r_hi;
  int rc;
} fm_job;

static void* fm_worker(void* arg) {
  fm_job* J = arg;
  ho_twin* h = J->h;
  const uint32_t n = h->n;
  const size_t W = twin_ct_words(h), P = twin_pt_words(h);
  uint64_t *dot = malloc(W * 8), *p = malloc(W * 8), *mv = malloc(P * 8), *ms = malloc(P * 8);
  for (uint64_t r = J->r_lo; r < J->r_hi; ++r)
    for (uint64_t j = 0; j < J->cols; ++j) {
      for (uint64_t k = 0; k < J->kc; ++k) {
        memcpy(p, J->inputs + (r * J->kc + k) * W, W * 8);
        size_t off_ct = 0, off_pt = 0;
        for (int b = 0; b < 2; ++b) {
          const ctx* c = &h->c[b];
          if (!J->form) ct_to_eval(c, p + off_ct);
          ct_mul_plain(c, p + off_ct, J->wv + (j * J->kc + k) * P + off_pt, J->ws + (j * J->kc + k) * P + off_pt);
          if (k == 0) memcpy(dot + off_ct, p + off_ct, 2ull * c->L * n * 8);
          else ct_add(c, dot + off_ct, p + off_ct);
          off_ct += 2ull * c->L * n;
          off_pt += (size_t)c->L * n;
        }
      }
      uint64_t g = r * J->cols + j;
      make_mask(h, (uint32_t)(g % n), mv, ms);
      size_t off_ct = 0, off_pt = 0;
      for (int b = 0; b < 2; ++b) {
        const ctx* c = &h->c[b];
        sum_all_slots(c, &h->k[b], dot + off_ct);
        ct_mul_plain(c, dot + off_ct, mv + off_pt, ms + off_pt);
        off_ct += 2ull * c->L * n;
        off_pt += (size_t)c->L * n;
      }
      uint64_t cidx = g / n;
      pthread_mutex_lock(J->mu);
      if (J->acc_set[cidx]) {
        size_t o = 0;
        for (int b = 0; b < 2; ++b) {
          ct_add(&h->c[b], J->acc + cidx * W + o, dot + o);
          o += 2ull * h->c[b].L * n;
        }
      } else {
        memcpy(J->acc + cidx * W, dot, W * 8);
        J->acc_set[cidx] = 1;
      }
      pthread_mutex_unlock(J->mu);
    }
  free(dot);
  free(p);
  free(mv);
  free(ms);
  return NULL;
}

int ho_fast_matmul(ho_twin* h, const uint64_t* inputs, int form, uint64_t R, uint64_t f, const uint64_t* weights,
                   uint64_t cols, const int64_t* bias, uint64_t* out, uint64_t* counters, unsigned threads) {
  if (R == 0) return set_err(ERR_PARAM, "matmul: empty input");
  if (cols == 0 || f == 0) return set_err(ERR_PARAM, "matmul: empty weights");
  if (!ho_capacity_ok(f, h->s_x, h->s_w, h->in_bits, h->t[0], h->t[1]))
    return set_err(ERR_RANGE, "matmul: product exceeds the plaintext capacity; refusing");
  const uint32_t n = h->n;
  const uint64_t kc = (f + n - 1) / n, C = (R * cols + n - 1) / n;
  const size_t W = twin_ct_words(h), P = twin_pt_words(h);
  /* weight shoup constants (ring::prepare, poly.cpp:52-63) */
  uint64_t* ws = malloc(cols * kc * P * 8);
  for (uint64_t jk = 0; jk < cols * kc; ++jk) {
    size_t o = 0;
    for (int b = 0; b < 2; ++b)
      for (uint32_t i = 0; i < h->c[b].L; ++i, o += n)
        for (uint32_t s = 0; s < n; ++s)
          ws[jk * P + o + s] = ho_shoup_precompute(weights[jk * P + o + s], h->c[b].q[i]);
  }
  unsigned char* acc_set = calloc(C, 1);
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  if (threads == 0) threads = (unsigned)sysconf(_SC_NPROCESSORS_ONLN);
  if (threads > R) threads = (unsigned)R;
  if (threads < 1) threads = 1;
  fm_job* jobs = calloc(threads, sizeof *jobs);
  pthread_t* tid = calloc(threads, sizeof *tid);
  uint64_t block = (R + threads - 1) / threads;
  for (unsigned w = 0; w < threads; ++w) {
    fm_job* J = &jobs[w];
    *J = (fm_job){h, inputs, form, R, cols, kc, weights, ws, out, acc_set, &mu, w * block,
                  (w + 1) * block < R ? (w + 1) * block : R, 0};
    if (J->r_lo >= J->r_hi) continue;
    if (threads == 1) fm_worker(J);
    else pthread_create(&tid[w], NULL, fm_worker, J);
  }
  if (threads > 1)
    for (unsigned w = 0; w < threads; ++w)
      if (jobs[w].r_lo < jobs[w].r_hi) pthread_join(tid[w], NULL);
  free(jobs);
  free(tid);
  free(ws);
  /* finish (matmul.cpp:200-232): bias pattern per packed ciphertext */
  int64_t* pattern = malloc(n * 8);
  uint64_t* pt = malloc(2ull * n * 8);
  uint64_t* dm = malloc(n * 8);
  int rc = 0;
  for (uint64_t c = 0; c < C && !rc; ++c) {
    for (uint32_t s = 0; s < n; ++s) {
      uint64_t g = c * n + s;
      pattern[s] = g < R * cols ? bias[g % cols] : 0;
    }
    if ((rc = encode_signed(h, pattern, n, pt))) break;
    size_t o = 0;
    for (int b = 0; b < 2; ++b) {
      const ctx* cx = &h->c[b];
      for (uint32_t i = 0; i < cx->L; ++i) {
        delta_times(cx, pt + (size_t)b * n, i, dm);
        ntt_fwd(dm, &cx->qt[i]);
        uint64_t* c0 = out + c * W + o + (size_t)i * n;
        for (uint32_t s = 0; s < n; ++s) c0[s] = add_mod_1(c0[s], dm[s], cx->q[i]);
      }
      o += 2ull * cx->L * n;
    }
  }
  free(pattern);
  free(pt);
  free(dm);
  free(acc_set);
  if (!rc && counters) {
    ho_proposed_counts(R, cols, f, n, counters);
  }
  return rc;
}

/* ---- baseline (matmul.cpp:273-344) ---- */
int ho_baseline_matmul(ho_twin* h, const int64_t* x, uint64_t R, uint64_t f, const int64_t* w, uint64_t cols,
                       const int64_t* bias, uint64_t* out, uint64_t* counters) {
  if (R == 0 || f == 0 || cols == 0) return set_err(ERR_PARAM, "baseline: empty input");
  if (!ho_capacity_ok(f, h->s_x, h->s_w, h->in_bits, h->t[0], h->t[1]))
    return set_err(ERR_RANGE, "baseline: product exceeds the plaintext capacity; refusing");
  const uint32_t n = h->n;
  const uint64_t blocks = (R + n - 1) / n;
  const size_t W = twin_ct_words(h);
  int64_t lim = max_centered(h->t[0], h->t[1]);
  int64_t* col = malloc(n * 8);
  uint64_t* pt = malloc(2ull * n * 8);
  uint64_t* ck = malloc(W * 8);
  uint64_t* p = malloc(W * 8);
  int rc = 0;
  for (uint64_t k = 0; k < f && !rc; ++k) {
    for (uint64_t j = 0; j < cols; ++j)
      if (w[k * cols + j] > lim || w[k * cols + j] < -lim) rc = set_err(ERR_RANGE, "prepare_constant_signed: value outside centered range");
    for (uint64_t blk = 0; blk < blocks && !rc; ++blk) {
      uint64_t base = blk * n, rows_b = R - base < n ? R - base : n;
      for (uint64_t s = 0; s < rows_b; ++s) col[s] = x[(base + s) * f + k];
      if ((rc = encode_signed(h, col, rows_b, pt))) break;
      encrypt_eval(&h->c[0], &h->k[0], &h->enc[0], pt, ck);
      encrypt_eval(&h->c[1], &h->k[1], &h->enc[1], pt + n, ck + 2ull * h->c[0].L * n);
      for (uint64_t j = 0; j < cols; ++j) {
        /* prepare_constant_signed (twin.cpp:131-143, context.cpp:120-137) */
        size_t o = 0;
        for (int b = 0; b < 2; ++b) {
          const ctx* c = &h->c[b];
          uint64_t v = centered_residue(w[k * cols + j], h->t[b]);
          for (uint32_t r = 0; r < 2 * c->L; ++r) {
            uint64_t q = c->q[r % c->L], vs = ho_shoup_precompute(v, q);
            const uint64_t* src = ck + o + (size_t)r * n;
            uint64_t* dst = p + o + (size_t)r * n;
            for (uint32_t s = 0; s < n; ++s) dst[s] = shoup_mul(src[s], v, vs, q);
          }
          o += 2ull * c->L * n;
        }
        uint64_t* acc = out + (blk * cols + j) * W;
        if (k == 0) memcpy(acc, p, W * 8);
        else {
          size_t o2 = 0;
          for (int b = 0; b < 2; ++b) {
            ct_add(&h->c[b], acc + o2, p + o2);
            o2 += 2ull * h->c[b].L * n;
          }
        }
      }
    }
  }
  uint64_t* dm = malloc(n * 8);
  for (uint64_t blk = 0; blk < blocks && !rc; ++blk)
    for (uint64_t j = 0; j < cols && !rc; ++j) {
      for (uint32_t s = 0; s < n; ++s) col[s] = bias[j];
      if ((rc = encode_signed(h, col, n, pt))) break;
      size_t o = 0;
      for (int b = 0; b < 2; ++b) {
        const ctx* cx = &h->c[b];
        for (uint32_t i = 0; i < cx->L; ++i) {
          delta_times(cx, pt + (size_t)b * n, i, dm);
          ntt_fwd(dm, &cx->qt[i]);
          uint64_t* c0 = out + (blk * cols + j) * W + o + (size_t)i * n;
          for (uint32_t s = 0; s < n; ++s) c0[s] = add_mod_1(c0[s], dm[s], cx->q[i]);
        }
        o += 2ull * cx->L * n;
      }
    }
  free(dm);
  free(col);
  free(pt);
  free(ck);
  free(p);
  if (!rc && counters) ho_baseline_counts(R, cols, f, n, counters);
  return rc;
}

/* RNG replay for encryptions: [enc][b][u | e0 | e1][n] int8 (values fit: |e| <= 19) */
int ho_baseline_noise(ho_twin* h, uint64_t encryptions, int8_t* out) {
  const uint32_t n = h->n;
  int32_t* e = malloc(n * 4);
  for (uint64_t k = 0; k < encryptions; ++k)
    for (int b = 0; b < 2; ++b) {
      int8_t* o = out + (k * 2 + b) * 3ull * n;
      sample_ternary(n, &h->enc[b], o);
      sample_gaussian(n, &h->enc[b], e);
      for (uint32_t s = 0; s < n; ++s) o[n + s] = (int8_t)e[s];
      sample_gaussian(n, &h->enc[b], e);
      for (uint32_t s = 0; s < n; ++s) o[2 * n + s] = (int8_t)e[s];
    }
  free(e);
  return 0;
}

/* decrypt_signed (twin.cpp:153-159 + decode_signed :113-121 + crt_recombine
 * fixed_point.cpp:89-104) */
int ho_decrypt_signed(ho_twin* h, const uint64_t* ct, int form, int64_t* out, int* budget) {
  const uint32_t n = h->n;
  uint64_t *m = malloc(n * 8), *s0 = malloc(n * 8), *s1 = malloc(n * 8);
  int b0, b1;
  decrypt_core(&h->c[0], &h->k[0], ct, form, m, &b0);
  decode_slots(&h->c[0], m, s0);
  decrypt_core(&h->c[1], &h->k[1], ct + 2ull * h->c[0].L * n, form, m, &b1);
  decode_slots(&h->c[1], m, s1);
  int rc = 0;
  if (b0 <= 0 || b1 <= 0) rc = set_err(ERR_NOISE, "decrypt: invariant noise budget exhausted");
  const uint64_t t0 = h->t[0], t1 = h->t[1];
  uint64_t inv = 0;
  inv_mod(t0 % t1, t1, &inv);
  u128 prod = (u128)t0 * t1;
  for (uint32_t i = 0; i < n; ++i) {
    uint64_t diff = (s1[i] + t1 - s0[i] % t1) % t1, kk = mul_mod(diff, inv, t1);
    u128 v = (u128)t0 * kk + s0[i];
    __int128 sv = (__int128)v;
    if (v > (prod - 1) / 2) sv -= (__int128)prod;
    out[i] = (int64_t)sv;
  }
  if (budget) *budget = b0 < b1 ? b0 : b1;
  free(m);
  free(s0);
  free(s1);
  return rc;
}

int ho_unpack(ho_twin* h, const uint64_t* packed, uint64_t R, uint64_t cols, int64_t* out) {
  const uint32_t n = h->n;
  const uint64_t C = (R * cols + n - 1) / n;
  int64_t* v = malloc(n * 8);
  for (uint64_t c = 0; c < C; ++c) {
    int rc = ho_decrypt_signed(h, packed + c * twin_ct_words(h), 1, v, NULL);
    if (rc) {
      free(v);
      return rc;
    }
    for (uint32_t s = 0; s < n; ++s) {
      uint64_t g = c * n + s;
      if (g >= R * cols) break;
      out[g] = v[s];
    }
  }
  free(v);
  return 0;
}

int ho_unpack_baseline(ho_twin* h, const uint64_t* blocks, uint64_t R, uint64_t cols, int64_t* out) {
  const uint32_t n = h->n;
  const uint64_t B = (R + n - 1) / n;
  int64_t* v = malloc(n * 8);
  for (uint64_t blk = 0; blk < B; ++blk)
    for (uint64_t j = 0; j < cols; ++j) {
      int rc = ho_decrypt_signed(h, blocks + (blk * cols + j) * twin_ct_words(h), 1, v, NULL);
      if (rc) {
        free(v);
        return rc;
      }
      uint64_t base = blk * n, rows_b = R - base < n ? R - base : n;
      for (uint64_t s = 0; s < rows_b; ++s) out[(base + s) * cols + j] = v[s];
    }
  free(v);
  return 0;
}

int ho_apply_galois(ho_twin* h, int b, uint64_t elt, const uint64_t* in, uint64_t* out) {
  int e = elt_index(&h->c[b], elt);
  if (e < 0) return set_err(ERR_KEY, "apply_galois: no key for galois element %llu", (unsigned long long)elt);
  apply_galois(&h->c[b], &h->k[b], e, in, out);
  return 0;
}

int ho_sum_all_slots(ho_twin* h, const uint64_t* in, uint64_t* out) {
  memcpy(out, in, twin_ct_words(h) * 8);
  sum_all_slots(&h->c[0], &h->k[0], out);
  sum_all_slots(&h->c[1], &h->k[1], out + 2ull * h->c[0].L * h->n);
  return 0;
}
