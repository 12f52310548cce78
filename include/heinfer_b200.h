/* heinfer_b200 — C ABI of the B200-native encrypted-LR matmul hot path.
 *
 * Drop-in boundary for the reference's hei::matmul entry points
 * (/root/reference/proj/include/hei/matmul/matmul.hpp). Plain pointers and
 * sizes only; every residue array uses the reference's own u64 values and the
 * flat layouts below, so the C++ adapter only flattens
 * std::vector<uint64_t> polynomials.
 *
 * Layouts (N = ring degree, L_b = primes of branch b, branch 0 = t0):
 *   twin ciphertext   [branch 2][part 2][prime L_b][N] u64
 *   twin plain        [branch 2][prime L_b][N] u64
 *   inputs            [row][chunk k][twin ciphertext]
 *   prepared weights  [col j][chunk k][twin plain]   (EncodedWeights values)
 *   packed output     [ct c][twin ciphertext], eval form
 *   galois keys (b)   [elt, ascending][l][part][i][N] u64, eval form
 *                     (GaloisKey::rows[l][part][i].vals, keys.hpp:37-43)
 *
 * Errors: every entry point returns HEI_OK or the code of the reference
 * exception it replaces (hei/util/errors.hpp:13-53); hei_gpu_last_error()
 * returns the message of the last failure on the calling thread.
 */
#ifndef HEINFER_B200_H
#define HEINFER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HEI_OK 0
#define HEI_PARAM_ERROR 1 /* hei::ParamError */
#define HEI_KEY_ERROR 2   /* hei::KeyError   */
#define HEI_RANGE_ERROR 3 /* hei::RangeError */
#define HEI_NOISE_ERROR 4 /* hei::NoiseError */
#define HEI_CODEC_ERROR 5 /* hei::CodecError */
#define HEI_CUDA_ERROR 6  /* device failure (no reference counterpart) */
#define HEI_INTERNAL 9

#define HEI_FORM_COEFF 0 /* ring::PolyForm::coeff (poly.hpp:13) */
#define HEI_FORM_EVAL 1  /* ring::PolyForm::eval */

typedef struct hei_gpu_ctx hei_gpu_ctx;         /* TwinContext + server keys on one device */
typedef struct hei_gpu_weights hei_gpu_weights; /* EncodedWeights resident in HBM */
typedef struct hei_gpu_stream hei_gpu_stream;   /* MatmulStream */
typedef struct hei_gpu_prng hei_gpu_prng;       /* util::Prng replay (rng.hpp:19-68) */

/* matmul::OpCounters (matmul.hpp:21-27). The matmul entry points report
 * MEASURED deltas, as MatmulStream::finish does (matmul.cpp:224-229): the
 * kernels that perform the chunk products, rotations, fold adds, mask
 * products and packed accumulations add them to context counters (branch 0
 * speaks for the pair, as TwinBackend::counters does), and each call
 * reports end minus start. ciphertexts_in/out are the call's shapes. */
typedef struct {
  uint64_t mul_plain_count;
  uint64_t rotation_count;
  uint64_t add_count;
  uint64_t ciphertexts_in;
  uint64_t ciphertexts_out;
} hei_op_counters;

/* fpcrt::TwinParams (twin.hpp:20-25) + the derived q chains
 * (bfv::default_q_primes, params.cpp:84-104). */
typedef struct {
  uint32_t n;
  uint64_t t[2];
  uint32_t L[2];
  const uint64_t* q; /* [L0 + L1] */
  uint32_t s_x, s_w, input_int_bits;
  int device;
} hei_twin_desc;

/* bfv::default_q_primes (params.cpp:84-104): the ciphertext modulus chain
 * make_params derives for (n, t) — the q[] a hei_twin_desc expects per
 * branch. Host only. */
int hei_default_q_primes(uint32_t n, uint64_t t, uint64_t* out, uint32_t capacity, uint32_t* count);

const char* hei_gpu_last_error(void);
const char* hei_gpu_version(void);

/* Context + keys. Replaces TwinContext / server_backend (twin.hpp:49-115).
 * Validates like EncryptionParams::validate (params.cpp:27-66). */
int hei_gpu_ctx_create(const hei_twin_desc* desc, hei_gpu_ctx** out);
void hei_gpu_ctx_destroy(hei_gpu_ctx* ctx);
/* GaloisKeySet of one branch (keys.hpp:44-49); elts ascending. */
int hei_gpu_upload_galois_keys(hei_gpu_ctx* ctx, uint32_t branch, uint32_t count,
                               const uint64_t* elts, const uint64_t* rows);
/* PublicKey of one branch, coeff form [2][L][N] (keys.hpp:28-32); needed by
 * the encrypting calls only: the standard (baseline) algorithm and client
 * encryption (hei_gpu_encode_inputs). */
int hei_gpu_upload_public_key(hei_gpu_ctx* ctx, uint32_t branch, const uint64_t* pk);

/* Weights. hei_gpu_weights_create uploads EncodedWeights values as produced by
 * matmul::encode_weights (matmul.cpp:83-104); hei_gpu_weights_encode runs
 * encode_weights itself on the device from the scaled f x cols matrix. */
int hei_gpu_weights_create(hei_gpu_ctx* ctx, const uint64_t* prepared, uint64_t f,
                           uint64_t cols, hei_gpu_weights** out);
int hei_gpu_weights_encode(hei_gpu_ctx* ctx, const int64_t* w, uint64_t f, uint64_t cols,
                           hei_gpu_weights** out);
void hei_gpu_weights_destroy(hei_gpu_weights* w);

/* matmul::matmul (matmul.cpp:239-255). Host buffers; inputs in `form`;
 * bias = EncodedBias::scaled [cols]; out = PackedResult cts (eval form). */
int hei_gpu_matmul(hei_gpu_ctx* ctx, const hei_gpu_weights* w, const uint64_t* inputs,
                   int form, uint64_t rows, const int64_t* bias, uint64_t* out,
                   hei_op_counters* counters);

/* Client-side decryption on the device. The secret key
 * of branch b is SecretKey::s (ternary int8 [N], keys.hpp). decrypt_core
 * (context.cpp:316-370) with an exact multi-limb CRT per coefficient,
 * decode_slots (context.cpp:95-102) and crt_recombine (fixed_point.cpp:89-106).
 *   decrypt_signed: out [count][N] = TwinBackend::decrypt_signed per ct;
 *                   HEI_NOISE_ERROR when a branch budget is exhausted.
 *   noise_budget:   budgets [count] = TwinBackend::noise_budget (min of branches).
 *   unpack_results: matmul::unpack_results (matmul.cpp:257-271), packed eval
 *                   cts [count][twin ct] -> out [rows][cols].
 *   unpack_baseline: matmul::unpack_baseline (matmul.cpp:346-358), blocks
 *                   [ceil(rows/N)][cols][twin ct] -> out [rows][cols]. */
int hei_gpu_upload_secret_key(hei_gpu_ctx* ctx, uint32_t branch, const int8_t* s);
int hei_gpu_decrypt_signed(hei_gpu_ctx* ctx, const uint64_t* cts, int form, uint64_t count, int64_t* out);
int hei_gpu_noise_budget(hei_gpu_ctx* ctx, const uint64_t* cts, int form, uint64_t count, int* budgets);
int hei_gpu_unpack_results(hei_gpu_ctx* ctx, const uint64_t* packed, uint64_t count, uint64_t rows,
                           uint64_t cols, int64_t* out);
int hei_gpu_unpack_baseline(hei_gpu_ctx* ctx, const uint64_t* blocks, uint64_t rows, uint64_t cols,
                            int64_t* out);

/* TwinContext::keygen (twin.cpp:41-48; BfvContext::keygen context.cpp:152-172
 * and make_galois_keys :201-251 per branch) on the device, drawing from `rng`
 * exactly as the reference draws from its util::Prng (the stream is replayed
 * and rejection sampling resolved on the device; rng is advanced past every
 * draw the reference would consume). Outputs (each may be NULL):
 *   sk       [2][N] int8 (SecretKey::s per branch)
 *   pk       [branch][part][prime][N] u64 coeff form (PublicKey p0, p1)
 *   elts_out [log2(N)] galois elements, ascending
 *   gk0/gk1  [elt ascending][l][part][i][N] u64 eval form (GaloisKey::rows)
 * install != 0 also installs them in ctx (Galois keys for the server role,
 * public and secret keys for the client role). */
int hei_gpu_keygen(hei_gpu_ctx* ctx, hei_gpu_prng* rng, int install, int8_t* sk, uint64_t* pk,
                   uint64_t* elts_out, uint64_t* gk0, uint64_t* gk1);

/* Test seam (not a reference interface): the keygen draw planner on a given
 * raw mt19937_64 stream; kinds 0 uniform_u64(bound) -> out32 (low 32 bits),
 * 1 ternary -> out8, 2 gaussian (records the start in gpos). */
int hei_gpu_debug_rejection_plan(hei_gpu_ctx* ctx, const uint64_t* raw, uint64_t avail, const uint32_t* kinds,
                                 const uint32_t* counts, const uint64_t* bounds, uint32_t nseg,
                                 uint32_t* out32, int8_t* out8, uint64_t* gpos, uint64_t* used);

/* Server wire path (InferenceServer::do_infer, server.cpp:112-172): the
 * request's HECT ciphertext blobs (bfv::load_ciphertext, serialize.cpp:80-91;
 * coeff form) concatenated in request order [row][chunk][branch], each branch-b
 * blob exactly hei_hect_ciphertext_bytes(N, L_b) bytes; the response blobs
 * (bfv::save_ciphertext, serialize.cpp:63-78) are written to `out` in order
 * [packed ct][branch]. Parsing, range checks, to_eval, the matmul, to_coeff
 * and serialization all run on the device. params_hash[b] =
 * BfvContext::hash() of branch b (hei_params_hash). Header errors raise
 * HEI_CODEC_ERROR with the reference's messages. */
uint64_t hei_hect_ciphertext_bytes(uint32_t n, uint32_t num_primes);
uint64_t hei_params_hash(uint32_t n, uint64_t t, int security_level, const uint64_t* q,
                         uint32_t num_primes);
int hei_gpu_matmul_wire(hei_gpu_ctx* ctx, const hei_gpu_weights* w, const uint64_t params_hash[2],
                        const uint8_t* blobs, uint64_t blob_bytes, uint64_t rows, const int64_t* bias,
                        uint8_t* out, uint64_t out_capacity, uint64_t* out_bytes,
                        hei_op_counters* counters);

/* Same call on device-resident u32 residues (the HBM-resident bench path):
 * d_inputs [row][k][twin ct] u32, d_out [C][twin ct] u32, both device
 * pointers; `stream` is a cudaStream_t (NULL = legacy default). */
int hei_gpu_matmul_device(hei_gpu_ctx* ctx, const hei_gpu_weights* w, const uint32_t* d_inputs,
                          int form, uint64_t rows, const int64_t* bias, uint32_t* d_out,
                          hei_op_counters* counters, void* stream);

/* Sharded execution (one process per GPU). Each rank adds the
 * masked class results of its rows [row_offset, row_offset + rows) of a
 * total_rows batch into d_acc, an unreduced u64 packed accumulator
 * [C][twin ct] (C = ceil(total_rows * cols / N)): the call ACCUMULATES into
 * the caller's buffer, which must be zeroed before the first call (it is not
 * cleared here). Partial accumulators of all ranks sum exactly (no wrap
 * below 2^63), so the exchange is one integer reduction; finish_packed then
 * reduces mod q and adds the bias once (MatmulStream::finish,
 * matmul.cpp:200-232). */
int hei_gpu_matmul_partial_device(hei_gpu_ctx* ctx, const hei_gpu_weights* w, const uint32_t* d_inputs,
                                  uint64_t rows, uint64_t row_offset, uint64_t total_rows, uint64_t* d_acc,
                                  void* stream);
int hei_gpu_finish_packed_device(hei_gpu_ctx* ctx, const hei_gpu_weights* w, const uint64_t* d_acc,
                                 const int64_t* bias, uint64_t total_rows, uint32_t* d_out, void* stream);

/* Stream-ordered exchange (no host synchronisation): reduce_packed turns a
 * rank's u64 accumulator of `count` packed twin ciphertexts into u32
 * residues mod q (its partial: half the bytes, exact); after the ranks'
 * partials are gathered (an NCCL all-gather of `count` x twin-ct u32 words
 * per rank), finish_parts sums the `parts` partials [parts][count][twin ct]
 * mod q and adds the bias plaintext once (MatmulStream::finish,
 * matmul.cpp:200-232). Both are enqueued on `stream` and return without
 * waiting. */
int hei_gpu_reduce_packed_device(hei_gpu_ctx* ctx, const uint64_t* d_acc, uint64_t count, uint32_t* d_out,
                                 void* stream);
int hei_gpu_finish_parts_device(hei_gpu_ctx* ctx, const hei_gpu_weights* w, const uint32_t* d_parts, uint32_t parts,
                                const int64_t* bias, uint64_t total_rows, uint32_t* d_out, void* stream);

/* Peer-memory exchange: the owner rank exports a receive buffer
 * (one slot per rank) as a 64-byte CUDA IPC handle; every rank maps it and
 * writes its packed accumulator into its slot with a device-to-device copy
 * (an NVLink peer write); the owner sums the slots (exact u64) and finishes. */
int hei_gpu_buffer_alloc(int device, uint64_t bytes, void** d_ptr);
int hei_gpu_buffer_zero(void* d_ptr, uint64_t bytes, void* stream);
void hei_gpu_buffer_free(void* d_ptr);
int hei_gpu_copy_async(void* dst, const void* src, uint64_t bytes, void* stream);
int hei_gpu_sum_slots(void* d, uint64_t words, uint32_t count, void* stream);
int hei_gpu_ipc_handle(const void* d_ptr, uint8_t* handle64);
int hei_gpu_ipc_open(int device, const uint8_t* handle64, void** d_ptr);
int hei_gpu_ipc_close(void* d_ptr);

/* Feature-block sharding (C5 "shard by feature block"): rank r
 * holds chunks [chunk_lo, chunk_lo + chunk_count) of every row
 * (d_inputs [rows][chunk_count][twin ct] u32) and adds its chunk products,
 * each reduced mod q, into d_dot [rows * cols][twin ct] u64 (zeroed by the
 * caller). The ranks' d_dot partials sum exactly (reduce-scatter by rows);
 * fold_pack then reduces the summed dots of rows [row_lo, row_lo + row_count)
 * mod q, runs sum_all_slots and the mask into the packed accumulator d_acc
 * (as matmul_partial_device does), and finish_packed_device completes it.
 * Bit-exact with the single-GPU result: the chunk sum is reduced before
 * sum_all_slots, as MatmulStream::push_row does (matmul.cpp:176-184). */
int hei_gpu_chunk_dot_partial_device(hei_gpu_ctx* ctx, const hei_gpu_weights* w, const uint32_t* d_inputs,
                                     uint64_t rows, uint64_t chunk_lo, uint64_t chunk_count, uint64_t* d_dot,
                                     void* stream);
int hei_gpu_fold_pack_device(hei_gpu_ctx* ctx, const hei_gpu_weights* w, const uint64_t* d_dot, uint64_t row_lo,
                             uint64_t row_count, uint64_t total_rows, uint64_t* d_acc, void* stream);

/* MatmulStream (matmul.hpp:83-114): rows in any order, each once. */
int hei_gpu_stream_create(hei_gpu_ctx* ctx, const hei_gpu_weights* w, const int64_t* bias,
                          uint64_t total_rows, hei_gpu_stream** out);
int hei_gpu_stream_push_row(hei_gpu_stream* s, uint64_t row_index, const uint64_t* chunks,
                            int form);
int hei_gpu_stream_finish(hei_gpu_stream* s, uint64_t* out, hei_op_counters* counters);
void hei_gpu_stream_destroy(hei_gpu_stream* s);

/* matmul::baseline_matmul (matmul.cpp:273-344). Encrypts every feature column
 * with the public key; encryption randomness is replayed from one util::Prng
 * per branch, exactly as BfvBackend::encrypt draws it (context.cpp:262-303).
 * out [ceil(rows/N)][cols][twin ct] eval form. */
int hei_gpu_prng_create(uint64_t seed, hei_gpu_prng** out);
void hei_gpu_prng_destroy(hei_gpu_prng* p);
/* Draw raw mt19937_64 outputs (test seam: Prng::next, rng.hpp:37). */
int hei_gpu_prng_draw(hei_gpu_prng* p, uint64_t count, uint64_t* out);
int hei_gpu_baseline_matmul(hei_gpu_ctx* ctx, const int64_t* x, uint64_t rows, uint64_t f,
                            const int64_t* w, uint64_t cols, const int64_t* bias,
                            hei_gpu_prng* rng0, hei_gpu_prng* rng1, uint64_t* out,
                            hei_op_counters* counters);

/* Client-side encryption of inputs: matmul::encode_inputs
 * (matmul.cpp:59-81) — ceil(f/N) slot chunks per row, encode_signed +
 * encrypt in eval form, randomness replayed from the two branch Prngs exactly
 * as BfvBackend::encrypt draws it. x is rows x f (scaled, row-major);
 * out [row][k][twin ct] u64 (host) or u32 (device variant). */
int hei_gpu_encode_inputs(hei_gpu_ctx* ctx, const int64_t* x, uint64_t rows, uint64_t f,
                          hei_gpu_prng* rng0, hei_gpu_prng* rng1, uint64_t* out);
int hei_gpu_encode_inputs_device(hei_gpu_ctx* ctx, const int64_t* x, uint64_t rows, uint64_t f,
                                 hei_gpu_prng* rng0, hei_gpu_prng* rng1, uint32_t* d_out,
                                 void* stream);

/* Closed forms (matmul.cpp:30-57). */
int hei_proposed_counts(uint64_t rows, uint64_t cols, uint64_t f, uint32_t n, hei_op_counters* c);
int hei_baseline_counts(uint64_t rows, uint64_t cols, uint64_t f, uint32_t n, hei_op_counters* c);

/* ---- kernel-level seam (the reference's kernels::Kernels table,
 *      modops.hpp:29-51), batched over `count` polynomials of one prime. ---- */
int hei_gpu_ntt(hei_gpu_ctx* ctx, uint32_t branch, uint32_t prime, uint64_t* polys,
                uint64_t count, int inverse);
/* One keyed automorphism on a single-branch eval-form ciphertext [2][L][N]
 * (BfvContext::apply_galois, context.cpp:428-507). */
int hei_gpu_apply_galois(hei_gpu_ctx* ctx, uint32_t branch, uint64_t elt, const uint64_t* in,
                         uint64_t* out);
/* The same on a ciphertext in either form (HEI_FORM_EVAL / HEI_FORM_COEFF):
 * BfvContext::apply_galois's coefficient-form path (context.cpp:460-465,
 * 499-503; automorphism_coeff, poly.cpp:107-122) returns coefficient form. */
int hei_gpu_apply_galois_form(hei_gpu_ctx* ctx, uint32_t branch, uint64_t elt, int form,
                              const uint64_t* in, uint64_t* out);
/* HeBackend::sum_all_slots on twin ciphertexts (backend.cpp:63-73). */
int hei_gpu_sum_all_slots(hei_gpu_ctx* ctx, const uint64_t* in, uint64_t* out, uint64_t count);
/* Kernel launches issued by this thread since the last reset. */
uint64_t hei_gpu_launch_count(void);
void hei_gpu_reset_launch_count(void);
/* Tuning: pairs per device batch (0 = automatic). */
void hei_gpu_set_batch_pairs(hei_gpu_ctx* ctx, uint64_t pairs);
/* Measurement hooks for bench.py: CUDA events around every fold kernel
 * (which = 0 key switch, 1 digit INTT), and a register-only butterfly
 * throughput microbenchmark (the integer roofline denominator). */
int hei_gpu_kernel_timing(hei_gpu_ctx* ctx, int enable);
int hei_gpu_kernel_stats(hei_gpu_ctx* ctx, int which, uint64_t* launches, double* total_ms);
int hei_gpu_measure_butterfly_peak(int device, double* butterflies_per_s);

#ifdef __cplusplus
}
#endif
#endif
