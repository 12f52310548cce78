// TEST INFRASTRUCTURE ONLY.
//
// Drop-in parity: the UNMODIFIED reference (hei::matmul::matmul,
// MatmulStream, baseline_matmul; /root/reference/proj/src/matmul/matmul.cpp)
// against the product's C++ adapter (paper_2204_05496_b200/dropin, which runs
// the B200 path through libheinfer_b200.so) on the same TwinBackend, keys and
// input ciphertexts. Compares every output residue and the decrypted scores.
// Built by oracle/Makefile (target dropin) into oracle/_ref/dropin_test.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "hei/bfv/serialize.hpp"
#include "hei/matmul/matmul.hpp"
#include "hei/util/errors.hpp"
#include "hei/util/rng.hpp"
#include "hei_matmul_gpu.hpp"

using namespace hei;

static int failures = 0;
#define CHECK(c)                                                     \
  do {                                                               \
    if (!(c)) {                                                      \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);       \
      ++failures;                                                    \
    }                                                                \
  } while (0)

static bool same_ct(const fpcrt::TwinCipher& a, const fpcrt::TwinCipher& b) {
  for (size_t br = 0; br < 2; ++br) {
    const auto& x = std::get<bfv::Ciphertext>(a.b[br].v);
    const auto& y = std::get<bfv::Ciphertext>(b.b[br].v);
    if (x.form() != y.form()) return false;
    for (int p = 0; p < 2; ++p)
      for (size_t i = 0; i < x.parts[p].size(); ++i)
        if (x.parts[p][i].c != y.parts[p][i].c) return false;
  }
  return true;
}

static util::IntMat rmat(std::mt19937_64& g, size_t r, size_t c, int64_t mag) {
  util::IntMat m(r, c);
  for (auto& v : m.a) v = static_cast<int64_t>(g() % (2 * mag + 1)) - mag;
  return m;
}

static void run(const fpcrt::TwinParams& p, size_t R, size_t f, size_t cols, const char* name) {
  fpcrt::TwinContext ctx(p);
  util::Prng rng(1);
  auto keys = ctx.keygen(rng);
  auto client = ctx.client_backend(keys, 2);
  auto server = ctx.server_backend(keys.gks);
  std::mt19937_64 g(R * 131 + f);
  util::IntMat x = rmat(g, R, f, 40), w = rmat(g, f, cols, 300);
  matmul::EncodedBias bias;
  for (size_t j = 0; j < cols; ++j) bias.scaled.push_back(static_cast<int64_t>(g() % 20001) - 10000);
  auto ex = matmul::encode_inputs(*client, x);
  auto ew = matmul::encode_weights(*server, w);

  matmul::OpCounters rc, gc;
  auto ref = matmul::matmul(*server, ex, ew, bias, &rc);
  auto gpu = matmul::gpu::matmul(*server, ex, ew, bias, &gc);
  CHECK(ref.cts.size() == gpu.cts.size());
  bool same = ref.cts.size() == gpu.cts.size();
  for (size_t c = 0; same && c < ref.cts.size(); ++c) same = same_ct(ref.cts[c], gpu.cts[c]);
  CHECK(same);
  CHECK(rc.mul_plain_count == gc.mul_plain_count && rc.rotation_count == gc.rotation_count &&
        rc.add_count == gc.add_count && rc.ciphertexts_in == gc.ciphertexts_in &&
        rc.ciphertexts_out == gc.ciphertexts_out);
  auto ru = matmul::unpack_results(*client, ref), gu = matmul::unpack_results(*client, gpu);
  CHECK(ru == gu);
  std::printf("DROPIN %s matmul %s (%zu ct)\n", name, same && ru == gu ? "bit-exact" : "MISMATCH", ref.cts.size());

  // MatmulStream, rows in shuffled order
  std::vector<size_t> order(R);
  for (size_t i = 0; i < R; ++i) order[i] = i;
  std::shuffle(order.begin(), order.end(), g);
  matmul::gpu::MatmulStream st(*server, ew, bias, R);
  for (size_t i : order) st.push_row(i, ex.rows[i]);
  auto sres = st.finish();
  bool s2 = true;
  for (size_t c = 0; c < ref.cts.size(); ++c) s2 = s2 && same_ct(ref.cts[c], sres.cts[c]);
  CHECK(s2);
  bool threw = false;
  try {
    st.finish();
  } catch (const ParamError&) {
    threw = true;
  }
  CHECK(threw);
  std::printf("DROPIN %s stream %s\n", name, s2 ? "bit-exact" : "MISMATCH");

  // baseline with a fresh client seeded like client_backend(keys, 9)
  size_t fb = std::min<size_t>(f, 16);
  util::IntMat xb(R, fb), wb(fb, cols);
  for (size_t i = 0; i < R; ++i)
    for (size_t k = 0; k < fb; ++k) xb(i, k) = x(i, k);
  for (size_t k = 0; k < fb; ++k)
    for (size_t j = 0; j < cols; ++j) wb(k, j) = w(k, j);
  auto client9 = ctx.client_backend(keys, 9);
  auto bref = matmul::baseline_matmul(*client9, xb, wb, bias);
  std::vector<bfv::PublicKey> pub = {keys.kp[0].pub, keys.kp[1].pub};
  auto bgpu = matmul::gpu::baseline_matmul(*server, pub, 9, xb, wb, bias);
  bool s3 = bref.blocks.size() == bgpu.blocks.size();
  for (size_t blk = 0; s3 && blk < bref.blocks.size(); ++blk)
    for (size_t j = 0; j < cols; ++j) s3 = s3 && same_ct(bref.blocks[blk][j], bgpu.blocks[blk][j]);
  CHECK(s3);
  std::printf("DROPIN %s baseline %s\n", name, s3 ? "bit-exact" : "MISMATCH");

  // server wire path: client blobs (save_ciphertext) -> infer_wire -> blobs,
  // against the reference's load_ciphertext -> MatmulStream -> save_ciphertext
  {
    std::vector<std::string> blobs;
    for (const auto& row : ex.rows)
      for (const auto& ch : row.chunks)
        for (size_t b = 0; b < 2; ++b)
          blobs.push_back(bfv::to_bytes(std::get<bfv::Ciphertext>(ch.b[b].v), *ctx.branch(b),
                                        [](std::ostream& os, const bfv::Ciphertext& c, const bfv::BfvContext& cx) {
                                          bfv::save_ciphertext(os, c, cx);
                                        }));
    matmul::MatmulStream rs(*server, ew, bias, R);
    const size_t k = ex.rows[0].chunks.size();
    for (size_t i = 0; i < R; ++i) {
      matmul::EncodedInputRow row;
      for (size_t c = 0; c < k; ++c) {
        fpcrt::TwinCipher tc;
        for (size_t b = 0; b < 2; ++b) {
          std::istringstream is(blobs[(i * k + c) * 2 + b], std::ios::binary);
          tc.b.push_back(bfv::HeCipher{bfv::load_ciphertext(is, *ctx.branch(b))});
        }
        row.chunks.push_back(std::move(tc));
      }
      rs.push_row(i, row);
    }
    auto rp = rs.finish();
    std::vector<std::string> want;
    for (const auto& ct : rp.cts)
      for (size_t b = 0; b < 2; ++b) {
        std::ostringstream os(std::ios::binary);
        bfv::save_ciphertext(os, std::get<bfv::Ciphertext>(ct.b[b].v), *ctx.branch(b));
        want.push_back(os.str());
      }
    auto got = matmul::gpu::infer_wire(*server, blobs, R, ew, bias);
    CHECK(got == want);
    blobs[1][0] = 'X';
    bool codec = false;
    try {
      matmul::gpu::infer_wire(*server, blobs, R, ew, bias);
    } catch (const CodecError&) {
      codec = true;
    }
    CHECK(codec);
    std::printf("DROPIN %s wire %s\n", name, got == want ? "byte-identical" : "MISMATCH");
  }

  // error contract: no rotation keys -> KeyError (test_matmul.cpp:410-414)
  auto norot = ctx.client_backend(keys, 3, false);
  bool key_err = false;
  try {
    matmul::gpu::matmul(*norot, ex, ew, bias);
  } catch (const KeyError&) {
    key_err = true;
  }
  CHECK(key_err);
}

int main(int argc, char** argv) {
  bool prod = argc > 1 && std::string(argv[1]) == "--production";
  run(fpcrt::TwinParams{32, {7681, 12289}, 0, fpcrt::ScalingConfig{2, 3, 3}}, 9, 70, 3, "n=32");
  if (prod) run(fpcrt::production_params(), 2, 9000, 3, "n=8192");
  std::printf("DROPIN %s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
