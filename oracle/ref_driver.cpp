// TEST INFRASTRUCTURE ONLY — the checker, never the product.
//
// extern "C" driver over the UNMODIFIED reference implementation
// (/root/reference/proj, compiled in place by oracle/Makefile into
// oracle/_ref/libheiref.so). Used by tests/ to pin the C restatement
// (oracle/heoracle.c) and the GPU path against the reference itself, to write
// the golden fixtures under tests/golden/, and by bench.py's reference arm /
// cpu_baseline leg to time the reference CPU path on the host cores.
//
// The reference's own `heinfer bench` does not compile (tools/heinfer.cpp:611-612
// passes a 1-argument lambda to parallel_for), so this driver times
// hei::matmul::matmul (proj/src/matmul/matmul.cpp:239-255) and
// hei::matmul::baseline_matmul (:415-486) directly, exactly as the bench's
// "computation" phase would (tools/heinfer.cpp:596-628).
//
// Flat layouts shared with the C-ABI (include/heinfer_b200.h):
//   twin ciphertext  = [branch][part][prime][N] u64  (L0 + L1 primes)
//   twin plain       = [branch][prime][N] u64
//   galois keys (b)  = [elt (ascending)][l][part][i][N] u64, eval form
#include <chrono>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "hei/bfv/backend.hpp"
#include "hei/bfv/context.hpp"
#include "hei/bfv/params.hpp"
#include "hei/bfv/serialize.hpp"
#include "hei/fpcrt/twin.hpp"
#include "hei/kernels/modops.hpp"
#include "hei/matmul/matmul.hpp"
#include "hei/ring/ntt_tables.hpp"
#include "hei/ring/poly.hpp"
#include "hei/util/errors.hpp"
#include "hei/util/parallel.hpp"
#include "hei/util/rng.hpp"

using namespace hei;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

#define GUARD_BEGIN try {
#define GUARD_END                                           \
  }                                                         \
  catch (const ParamError& e) { return fail(e, 1); }        \
  catch (const KeyError& e) { return fail(e, 2); }          \
  catch (const RangeError& e) { return fail(e, 3); }        \
  catch (const NoiseError& e) { return fail(e, 4); }        \
  catch (const CodecError& e) { return fail(e, 5); }        \
  catch (const std::exception& e) { return fail(e, 9); }

struct Session {
  fpcrt::TwinParams params;
  std::unique_ptr<fpcrt::TwinContext> ctx;
  fpcrt::TwinKeys keys;
  std::unique_ptr<fpcrt::TwinBackend> client;
  std::unique_ptr<fpcrt::TwinBackend> server;
  matmul::EncodedInputs inputs;
  matmul::EncodedWeights weights;
  matmul::EncodedBias bias;
  uint32_t L[2] = {0, 0};
};

const bfv::BfvBackend& bfv_branch(fpcrt::TwinBackend& be, size_t b) {
  return dynamic_cast<const bfv::BfvBackend&>(be.branch(b));
}

size_t twin_ct_words(const Session& s) {
  return 2ull * (s.L[0] + s.L[1]) * s.params.n;
}

void write_ct(const bfv::Ciphertext& ct, uint64_t* out, size_t L, uint32_t n) {
  for (int p = 0; p < 2; ++p)
    for (size_t i = 0; i < L; ++i)
      std::memcpy(out + (p * L + i) * n, ct.parts[p][i].c.data(), n * 8);
}

void write_twin(const Session& s, const fpcrt::TwinCipher& tc, uint64_t* out) {
  const uint32_t n = s.params.n;
  for (size_t b = 0; b < 2; ++b) {
    const auto& ct = std::get<bfv::Ciphertext>(tc.b[b].v);
    write_ct(ct, out, s.L[b], n);
    out += 2ull * s.L[b] * n;
  }
}

bfv::Ciphertext read_ct(const uint64_t* in, const bfv::BfvContext& ctx,
                        ring::PolyForm form) {
  bfv::Ciphertext ct;
  ct.params_hash = ctx.hash();
  const size_t L = ctx.num_primes();
  const uint32_t n = ctx.n();
  for (int p = 0; p < 2; ++p)
    for (size_t i = 0; i < L; ++i) {
      ring::RingPoly poly = ring::RingPoly::zero(n, ctx.params().q[i], form);
      std::memcpy(poly.c.data(), in + (p * L + i) * n, n * 8);
      ct.parts[p].push_back(std::move(poly));
    }
  return ct;
}

fpcrt::TwinCipher read_twin(const Session& s, const uint64_t* in,
                            ring::PolyForm form) {
  fpcrt::TwinCipher tc;
  for (size_t b = 0; b < 2; ++b) {
    tc.b.push_back(bfv::HeCipher{read_ct(in, *s.ctx->branch(b), form)});
    in += 2ull * s.L[b] * s.params.n;
  }
  return tc;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Default modulus chain (proj/src/bfv/params.cpp:84-114).
int ref_default_primes(uint32_t n, uint64_t t, int sec, uint64_t* out,
                       uint32_t* count) {
  GUARD_BEGIN
  auto p = bfv::make_params(n, t, sec);
  *count = static_cast<uint32_t>(p.q.size());
  for (size_t i = 0; i < p.q.size(); ++i) out[i] = p.q[i];
  return 0;
  GUARD_END
}

// One kernels::scalar NTT (proj/src/kernels/modops_scalar.cpp:45-81) or the
// dispatched (AVX2) one when use_dispatch != 0.
int ref_ntt(uint32_t n, uint64_t q, uint64_t* a, int inverse, int use_dispatch) {
  GUARD_BEGIN
  ring::NttTables tab(n, q);
  const kernels::Kernels& k =
      use_dispatch ? kernels::select(q) : kernels::scalar::kTable;
  if (inverse)
    k.ntt_inverse(a, tab.view());
  else
    k.ntt_forward(a, tab.view());
  return 0;
  GUARD_END
}

int ref_ntt_tables(uint32_t n, uint64_t q, uint64_t* psi, uint64_t* zetas,
                   uint64_t* inv_zetas, uint64_t* inv_n) {
  GUARD_BEGIN
  ring::NttTables tab(n, q);
  *psi = tab.psi();
  std::memcpy(zetas, tab.view().zetas, n * 8);
  std::memcpy(inv_zetas, tab.view().inv_zetas, n * 8);
  *inv_n = tab.view().inv_n;
  return 0;
  GUARD_END
}

int ref_galois_perm(uint32_t n, uint64_t elt, uint32_t* out) {
  GUARD_BEGIN
  auto p = ring::galois_eval_permutation(n, elt);
  std::memcpy(out, p.data(), n * 4);
  return 0;
  GUARD_END
}

// Seeded twin session: keys from Prng(key_seed) (twin.cpp:41-48), client
// encryption seeds enc_seed + b (twin.cpp:58), server = evaluate-only.
int ref_create(void** out, uint32_t n, uint64_t t0, uint64_t t1, int sec,
               uint32_t s_x, uint32_t s_w, uint32_t in_bits, uint64_t key_seed,
               uint64_t enc_seed) {
  GUARD_BEGIN
  auto s = std::make_unique<Session>();
  s->params = fpcrt::TwinParams{n, {t0, t1}, sec, fpcrt::ScalingConfig{s_x, s_w, in_bits}};
  s->ctx = std::make_unique<fpcrt::TwinContext>(s->params);
  util::Prng rng(key_seed);
  s->keys = s->ctx->keygen(rng);
  s->client = s->ctx->client_backend(s->keys, enc_seed);
  s->server = s->ctx->server_backend(s->keys.gks);
  for (size_t b = 0; b < 2; ++b)
    s->L[b] = static_cast<uint32_t>(s->ctx->branch(b)->num_primes());
  *out = s.release();
  return 0;
  GUARD_END
}

void ref_destroy(void* h) { delete static_cast<Session*>(h); }

int ref_params(void* h, uint32_t* L, uint64_t* q, uint64_t* hash) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  size_t o = 0;
  for (size_t b = 0; b < 2; ++b) {
    L[b] = s.L[b];
    hash[b] = s.ctx->branch(b)->hash();
    for (uint64_t qi : s.ctx->branch(b)->params().q) q[o++] = qi;
  }
  return 0;
  GUARD_END
}

// Galois elements (ascending, the GaloisKeySet map order) and key rows.
int ref_export_keys(void* h, uint64_t* elts, uint64_t* gk0, uint64_t* gk1,
                    int8_t* sk, uint64_t* pk) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  const uint32_t n = s.params.n;
  uint64_t* gk[2] = {gk0, gk1};
  for (size_t b = 0; b < 2; ++b) {
    const size_t L = s.L[b];
    size_t e = 0;
    uint64_t* o = gk[b];
    for (const auto& [elt, key] : s.keys.gks[b].keys) {
      if (b == 0) elts[e] = elt;
      ++e;
      for (size_t l = 0; l < L; ++l)
        for (int p = 0; p < 2; ++p)
          for (size_t i = 0; i < L; ++i) {
            if (o) std::memcpy(o, key.rows[l][p][i].vals.data(), n * 8);
            if (o) o += n;
          }
    }
    if (sk) std::memcpy(sk + b * n, s.keys.kp[b].secret.s.data(), n);
    if (pk) {
      for (size_t i = 0; i < L; ++i) std::memcpy(pk + i * n, s.keys.kp[b].pub.p0[i].c.data(), n * 8);
      for (size_t i = 0; i < L; ++i) std::memcpy(pk + (L + i) * n, s.keys.kp[b].pub.p1[i].c.data(), n * 8);
      pk += 2ull * L * n;
    }
  }
  return 0;
  GUARD_END
}

int ref_num_galois(void* h) {
  auto& s = *static_cast<Session*>(h);
  return static_cast<int>(s.keys.gks[0].keys.size());
}

// encode_inputs with the client backend (matmul.cpp:59-81); optional export.
int ref_encode_inputs(void* h, const int64_t* x, uint64_t R, uint64_t f,
                      uint64_t* out) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  util::IntMat m(R, f);
  std::memcpy(m.a.data(), x, R * f * 8);
  s.inputs = matmul::encode_inputs(*s.client, m);
  if (out) {
    const size_t w = twin_ct_words(s);
    for (const auto& row : s.inputs.rows)
      for (const auto& ch : row.chunks) {
        write_twin(s, ch, out);
        out += w;
      }
  }
  return 0;
  GUARD_END
}

// Inputs supplied as flat twin ciphertexts (form 1 = eval, 0 = coeff).
int ref_load_inputs(void* h, const uint64_t* in, uint64_t R, uint64_t f, int form) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  const uint32_t n = s.params.n;
  const uint64_t k = (f + n - 1) / n;
  s.inputs = {};
  s.inputs.f = f;
  s.inputs.n = n;
  const size_t w = twin_ct_words(s);
  for (uint64_t r = 0; r < R; ++r) {
    matmul::EncodedInputRow row;
    for (uint64_t c = 0; c < k; ++c) {
      row.chunks.push_back(read_twin(s, in, form ? ring::PolyForm::eval : ring::PolyForm::coeff));
      in += w;
    }
    s.inputs.rows.push_back(std::move(row));
  }
  return 0;
  GUARD_END
}

// encode_weights (matmul.cpp:83-104): export the prepared values
// [j][k][branch][prime][N].
int ref_encode_weights(void* h, const int64_t* w, uint64_t f, uint64_t cols,
                       uint64_t* out) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  util::IntMat m(f, cols);
  std::memcpy(m.a.data(), w, f * cols * 8);
  s.weights = matmul::encode_weights(*s.server, m);
  if (out) {
    const uint32_t n = s.params.n;
    for (const auto& row : s.weights.outputs)
      for (const auto& tp : row)
        for (size_t b = 0; b < 2; ++b) {
          const auto& ep = std::get<bfv::EvalPlain>(tp.b[b].v);
          for (const auto& pp : ep.primes) {
            std::memcpy(out, pp.vals.data(), n * 8);
            out += n;
          }
        }
  }
  return 0;
  GUARD_END
}

int ref_set_bias(void* h, const int64_t* bias, uint64_t cols) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  s.bias.scaled.assign(bias, bias + cols);
  return 0;
  GUARD_END
}

// hei::matmul::matmul on the server backend; *secs = wall time of the call.
int ref_matmul(void* h, unsigned threads, uint64_t* out_packed,
               uint64_t* counters, double* secs) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  matmul::OpCounters ops;
  auto t0 = std::chrono::steady_clock::now();
  auto packed = matmul::matmul(*s.server, s.inputs, s.weights, s.bias, &ops, threads);
  auto t1 = std::chrono::steady_clock::now();
  if (secs) *secs = std::chrono::duration<double>(t1 - t0).count();
  if (out_packed) {
    const size_t w = twin_ct_words(s);
    for (const auto& ct : packed.cts) {
      write_twin(s, ct, out_packed);
      out_packed += w;
    }
  }
  if (counters) {
    counters[0] = ops.mul_plain_count;
    counters[1] = ops.rotation_count;
    counters[2] = ops.add_count;
    counters[3] = ops.ciphertexts_in;
    counters[4] = ops.ciphertexts_out;
  }
  return 0;
  GUARD_END
}

// The reference bench's streaming shape (tools/heinfer.cpp:589-620): encrypt
// `block` rows at a time with the client backend (encode_input_row, in row
// order, so the Prng stream is the one encode_inputs would consume), push
// them into one MatmulStream on the server backend with parallel_for, then
// finish. Keeps paper-scale batches (C5: 4096 x 40000 at N = 16384, 32 GB of
// u64 inputs) out of host memory. The weights and bias must be set.
// *secs = the push_row + finish time only (the bench's "computation" phase).
int ref_stream_matmul(void* h, const int64_t* x, uint64_t R, uint64_t f,
                      uint64_t block, unsigned threads, uint64_t* out_packed,
                      uint64_t* counters, double* secs) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  if (R == 0 || f != s.weights.f) throw ParamError("ref_stream_matmul: shape");
  if (block == 0) block = 64;
  matmul::MatmulStream stream(*s.server, s.weights, s.bias, R);
  std::vector<matmul::EncodedInputRow> enc;
  double comp = 0;
  for (uint64_t base = 0; base < R; base += block) {
    const uint64_t count = std::min<uint64_t>(block, R - base);
    enc.clear();
    for (uint64_t i = 0; i < count; ++i)
      enc.push_back(matmul::encode_input_row(
          *s.client, std::span<const int64_t>(x + (base + i) * f, f)));
    auto t0 = std::chrono::steady_clock::now();
    util::parallel_for(
        count,
        [&](size_t lo, size_t hi) {
          for (size_t i = lo; i < hi; ++i) stream.push_row(base + i, enc[i]);
        },
        threads);
    comp += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  auto t0 = std::chrono::steady_clock::now();
  auto packed = stream.finish();
  comp += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (secs) *secs = comp;
  if (out_packed) {
    const size_t w = twin_ct_words(s);
    for (const auto& ct : packed.cts) {
      write_twin(s, ct, out_packed);
      out_packed += w;
    }
  }
  if (counters) {
    const auto& ops = stream.counters();
    counters[0] = ops.mul_plain_count;
    counters[1] = ops.rotation_count;
    counters[2] = ops.add_count;
    counters[3] = ops.ciphertexts_in;
    counters[4] = ops.ciphertexts_out;
  }
  return 0;
  GUARD_END
}

// unpack_results (matmul.cpp:257-271) on flat packed ciphertexts (eval form).
int ref_unpack(void* h, const uint64_t* packed, uint64_t R, uint64_t cols,
               int64_t* out) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  const uint32_t n = s.params.n;
  matmul::PackedResult pr;
  pr.rows = R;
  pr.cols = cols;
  pr.n = n;
  const uint64_t c = (R * cols + n - 1) / n;
  for (uint64_t i = 0; i < c; ++i)
    pr.cts.push_back(read_twin(s, packed + i * twin_ct_words(s), ring::PolyForm::eval));
  auto m = matmul::unpack_results(*s.client, pr);
  std::memcpy(out, m.a.data(), R * cols * 8);
  return 0;
  GUARD_END
}

// baseline_matmul (matmul.cpp:273-344) with the client backend (it encrypts).
int ref_baseline(void* h, const int64_t* x, uint64_t R, uint64_t f,
                 const int64_t* w, uint64_t cols, uint64_t* out_blocks,
                 uint64_t* counters, double* secs) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  util::IntMat xm(R, f), wm(f, cols);
  std::memcpy(xm.a.data(), x, R * f * 8);
  std::memcpy(wm.a.data(), w, f * cols * 8);
  matmul::OpCounters ops;
  auto t0 = std::chrono::steady_clock::now();
  auto res = matmul::baseline_matmul(*s.client, xm, wm, s.bias, &ops);
  auto t1 = std::chrono::steady_clock::now();
  if (secs) *secs = std::chrono::duration<double>(t1 - t0).count();
  if (out_blocks) {
    const size_t wd = twin_ct_words(s);
    for (const auto& blk : res.blocks)
      for (const auto& ct : blk) {
        write_twin(s, ct, out_blocks);
        out_blocks += wd;
      }
  }
  if (counters) {
    counters[0] = ops.mul_plain_count;
    counters[1] = ops.rotation_count;
    counters[2] = ops.add_count;
    counters[3] = ops.ciphertexts_in;
    counters[4] = ops.ciphertexts_out;
  }
  return 0;
  GUARD_END
}

// Decrypt one twin ciphertext (form 1 = eval) to signed slot values
// (twin.cpp:153-159) and report the min noise budget.
int ref_decrypt_signed(void* h, const uint64_t* ct, int form, int64_t* out,
                       int* budget) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  auto tc = read_twin(s, ct, form ? ring::PolyForm::eval : ring::PolyForm::coeff);
  auto v = s.client->decrypt_signed(tc);
  std::memcpy(out, v.data(), v.size() * 8);
  if (budget) *budget = s.client->noise_budget(tc);
  return 0;
  GUARD_END
}

// One keyed automorphism on a single-branch ciphertext [part][prime][N]
// (context.cpp:428-507).
int ref_apply_galois(void* h, int branch, uint64_t elt, const uint64_t* in,
                     int form, uint64_t* out) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  const auto& ctx = *s.ctx->branch(branch);
  auto ct = read_ct(in, ctx, form ? ring::PolyForm::eval : ring::PolyForm::coeff);
  auto r = ctx.apply_galois(ct, elt, s.keys.gks[branch]);
  write_ct(r, out, ctx.num_primes(), ctx.n());
  return 0;
  GUARD_END
}

// sum_all_slots on one twin ciphertext (backend.cpp:63-73).
int ref_sum_all_slots(void* h, const uint64_t* in, uint64_t* out) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  auto tc = read_twin(s, in, ring::PolyForm::eval);
  auto r = s.server->sum_all_slots(tc);
  write_twin(s, r, out);
  return 0;
  GUARD_END
}

// The session's inputs as the client sends them: one HECT blob per
// (row, chunk, branch) from bfv::save_ciphertext (serialize.cpp:63-78),
// concatenated in request order (client.cpp / server.cpp:145-147).
int ref_inputs_wire(void* h, uint8_t* out, uint64_t cap, uint64_t* len) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  std::string all;
  for (const auto& row : s.inputs.rows)
    for (const auto& ch : row.chunks)
      for (size_t b = 0; b < 2; ++b) {
        std::ostringstream os(std::ios::binary);
        bfv::save_ciphertext(os, std::get<bfv::Ciphertext>(ch.b[b].v), *s.ctx->branch(b));
        all += os.str();
      }
  if (len) *len = all.size();
  if (out) {
    if (cap < all.size()) throw ParamError("ref_inputs_wire: buffer too small");
    std::memcpy(out, all.data(), all.size());
  }
  return 0;
  GUARD_END
}

// The computation of InferenceServer::do_infer (server.cpp:112-172) on a
// concatenated blob list: load_ciphertext per blob, MatmulStream over rows
// with parallel_for, finish, save_ciphertext per packed twin branch.
int ref_server_wire(void* h, const uint8_t* blobs, uint64_t blob_bytes, uint64_t rows,
                    unsigned threads, uint8_t* out, uint64_t cap, uint64_t* len,
                    double* secs) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  const uint32_t n = s.params.n;
  const uint64_t chunks = (s.weights.f + n - 1) / n;
  uint64_t bsz[2];
  for (size_t b = 0; b < 2; ++b) bsz[b] = 19 + 2ull * s.L[b] * (1 + 8ull * n);
  const uint64_t per_row = chunks * (bsz[0] + bsz[1]);
  if (rows == 0 || blob_bytes != rows * per_row)
    throw ParamError("ciphertext count does not match rows x chunks");
  auto t0 = std::chrono::steady_clock::now();
  matmul::MatmulStream stream(*s.server, s.weights, s.bias, rows);
  util::parallel_for(
      rows,
      [&](size_t lo, size_t hi) {
        for (size_t i = lo; i < hi; ++i) {
          matmul::EncodedInputRow row;
          const uint8_t* p = blobs + i * per_row;
          for (uint64_t c = 0; c < chunks; ++c) {
            fpcrt::TwinCipher ct;
            for (size_t b = 0; b < 2; ++b) {
              std::istringstream is(std::string(reinterpret_cast<const char*>(p), bsz[b]),
                                    std::ios::binary);
              ct.b.push_back(bfv::HeCipher{bfv::load_ciphertext(is, *s.ctx->branch(b))});
              p += bsz[b];
            }
            row.chunks.push_back(std::move(ct));
          }
          stream.push_row(i, row);
        }
      },
      threads);
  auto packed = stream.finish();
  std::string all;
  for (const auto& ct : packed.cts)
    for (size_t b = 0; b < 2; ++b) {
      std::ostringstream os(std::ios::binary);
      bfv::save_ciphertext(os, std::get<bfv::Ciphertext>(ct.b[b].v), *s.ctx->branch(b));
      all += os.str();
    }
  auto t1 = std::chrono::steady_clock::now();
  if (secs) *secs = std::chrono::duration<double>(t1 - t0).count();
  if (len) *len = all.size();
  if (out) {
    if (cap < all.size()) throw ParamError("ref_server_wire: buffer too small");
    std::memcpy(out, all.data(), all.size());
  }
  return 0;
  GUARD_END
}

// The draws that follow TwinContext::keygen(Prng(seed)) (twin.cpp:41-48):
// pins where a keygen replay must leave the stream.
int ref_keygen_next(void* h, uint64_t seed, uint64_t count, uint64_t* out) {
  GUARD_BEGIN
  auto& s = *static_cast<Session*>(h);
  util::Prng rng(seed);
  auto keys = s.ctx->keygen(rng);
  for (uint64_t k = 0; k < count; ++k) out[k] = rng.next();
  return 0;
  GUARD_END
}

// Prng stream check (proj/include/hei/util/rng.hpp:19-68).
int ref_prng(uint64_t seed, uint64_t count, uint64_t* raw, double* gauss,
             uint64_t* uni3) {
  util::Prng a(seed), b(seed), c(seed);
  for (uint64_t i = 0; i < count; ++i) {
    raw[i] = a.next();
    gauss[i] = b.gaussian();
    uni3[i] = c.uniform_u64(3);
  }
  return 0;
}

}  // extern "C"
