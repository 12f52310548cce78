/* TEST INFRASTRUCTURE ONLY — the CPU checker for the GPU hot path.
 *
 * heoracle: a plain-C restatement of the reference's encrypted-LR matmul hot
 * path (arXiv 2204.05496 reference, /root/reference/proj, C++20 "heinfer").
 * Every function cites the reference file:line it restates. It is pinned
 * against the reference itself (oracle/_ref/libheiref.so, built in place from
 * the reference sources) and against the golden fixtures in tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library. The product (libheinfer_b200.so) never links or calls it.
 *
 * Flat layouts (shared with include/heinfer_b200.h):
 *   single-branch ciphertext  [part 2][prime L][N] u64
 *   twin ciphertext           [branch 2][part 2][prime L_b][N] u64
 *   twin plain (prepared)     [branch 2][prime L_b][N] u64 (values only)
 *   galois keys (branch b)    [elt ascending][l][part][i][N] u64 (eval form)
 */
#ifndef HEORACLE_H
#define HEORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes: 0 ok, 1 ParamError, 2 KeyError, 3 RangeError, 4 NoiseError. */
const char* ho_last_error(void);

/* ---- single-value / kernel layer ---- */
uint64_t ho_shoup_precompute(uint64_t w, uint64_t q);
uint64_t ho_shoup_mul(uint64_t x, uint64_t w, uint64_t ws, uint64_t q);
int ho_is_prime(uint64_t v);
int ho_default_primes(uint32_t n, uint64_t t, int sec, uint64_t* out, uint32_t* count);
uint64_t ho_primitive_root_2n(uint32_t n, uint64_t q);
int ho_ntt(uint32_t n, uint64_t q, uint64_t* a, int inverse);
int ho_ntt_tables(uint32_t n, uint64_t q, uint64_t* zetas, uint64_t* inv_zetas, uint64_t* inv_n);
int ho_galois_perm(uint32_t n, uint64_t elt, uint32_t* out);
void ho_prng(uint64_t seed, uint64_t count, uint64_t* raw, double* gauss, uint64_t* uni3);

/* ---- twin session (two BFV branches, t0 / t1) ---- */
typedef struct ho_twin ho_twin;

int ho_twin_create(ho_twin** out, uint32_t n, uint64_t t0, uint64_t t1, int sec,
                   uint32_t s_x, uint32_t s_w, uint32_t in_bits,
                   uint64_t key_seed, uint64_t enc_seed);
void ho_twin_destroy(ho_twin* h);
/* L[2], q[L0+L1], hash[2], elts[num_elts] (ascending); returns num_elts. */
int ho_twin_info(const ho_twin* h, uint32_t* L, uint64_t* q, uint64_t* hash, uint64_t* elts);
int ho_twin_export_keys(const ho_twin* h, uint64_t* gk0, uint64_t* gk1, int8_t* sk, uint64_t* pk);

/* encode_inputs + encrypt (eval form) with the client RNG: out [R][k][twin ct] */
int ho_encode_inputs(ho_twin* h, const int64_t* x, uint64_t R, uint64_t f, uint64_t* out);
/* encode_weights prepared values: out [cols][k][twin plain] */
int ho_encode_weights(ho_twin* h, const int64_t* w, uint64_t f, uint64_t cols, uint64_t* out);
/* Fast slot-packed matmul (MatmulStream): inputs [R][k][twin ct] in `form`
 * (1 eval, 0 coeff), weights as from ho_encode_weights, bias scaled [cols].
 * out [ceil(R*cols/N)][twin ct] eval form; counters[5]. threads 0 = nproc. */
int ho_fast_matmul(ho_twin* h, const uint64_t* inputs, int form, uint64_t R, uint64_t f,
                   const uint64_t* weights, uint64_t cols, const int64_t* bias,
                   uint64_t* out, uint64_t* counters, unsigned threads);
/* Standard sample-batched matmul; encrypts with the client RNG.
 * out [ceil(R/N)][cols][twin ct] eval form. */
int ho_baseline_matmul(ho_twin* h, const int64_t* x, uint64_t R, uint64_t f,
                       const int64_t* w, uint64_t cols, const int64_t* bias,
                       uint64_t* out, uint64_t* counters);
/* Encryption noise of baseline feature columns, as the RNG replay produces it
 * (u ternary, e0, e1 gaussian), per encryption per branch: [enc][b][3][N] i8. */
int ho_baseline_noise(ho_twin* h, uint64_t encryptions, int8_t* out);
int ho_decrypt_signed(ho_twin* h, const uint64_t* ct, int form, int64_t* out, int* budget);
int ho_unpack(ho_twin* h, const uint64_t* packed, uint64_t R, uint64_t cols, int64_t* out);
int ho_unpack_baseline(ho_twin* h, const uint64_t* blocks, uint64_t R, uint64_t cols, int64_t* out);
/* Single ops (branch b ciphertext [2][L_b][N] eval form). */
int ho_apply_galois(ho_twin* h, int b, uint64_t elt, const uint64_t* in, uint64_t* out);
int ho_sum_all_slots(ho_twin* h, const uint64_t* in, uint64_t* out);
/* Slot mask for slot s, prepared values [twin plain] (matmul.cpp:146-163). */
int ho_mask(ho_twin* h, uint32_t slot, uint64_t* out);
/* Closed forms (matmul.cpp:30-57): counters[5]. */
int ho_proposed_counts(uint64_t R, uint64_t cols, uint64_t f, uint32_t n, uint64_t* c);
int ho_baseline_counts(uint64_t R, uint64_t cols, uint64_t f, uint32_t n, uint64_t* c);
/* fixed point (fixed_point.cpp:37-106) */
int ho_scale_value(double x, uint32_t e, int64_t* out);
int ho_capacity_ok(uint64_t f, uint32_t s_x, uint32_t s_w, uint32_t in_bits, uint64_t t0, uint64_t t1);

#ifdef __cplusplus
}
#endif
#endif
