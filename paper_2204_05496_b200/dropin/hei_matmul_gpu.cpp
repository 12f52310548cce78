// Drop-in adapter implementation: flattens the reference's value types into
// the C ABI's layouts and rethrows C-ABI error codes as the reference's
// exception types (hei/util/errors.hpp:13-53).
#include "hei_matmul_gpu.hpp"

#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "../../include/heinfer_b200.h"
#include "hei/bfv/backend.hpp"
#include "hei/util/errors.hpp"

namespace hei::matmul::gpu {

namespace {

void check(int rc) {
  if (rc == HEI_OK) return;
  const std::string msg = hei_gpu_last_error();
  switch (rc) {
    case HEI_PARAM_ERROR: throw ParamError(msg);
    case HEI_KEY_ERROR: throw KeyError(msg);
    case HEI_RANGE_ERROR: throw RangeError(msg);
    case HEI_NOISE_ERROR: throw NoiseError(msg);
    case HEI_CODEC_ERROR: throw CodecError(msg);
    default: throw std::runtime_error("heinfer_b200: " + msg);
  }
}

const bfv::BfvBackend& bfv_branch(fpcrt::TwinBackend& be, size_t b) {
  const auto* p = dynamic_cast<const bfv::BfvBackend*>(&be.branch(b));
  if (!p) throw ParamError("gpu matmul: backend is not a BFV backend");
  return *p;
}

size_t twin_words(fpcrt::TwinBackend& be) {
  size_t L = 0;
  for (size_t b = 0; b < 2; ++b) L += bfv_branch(be, b).context().num_primes();
  return 2 * L * be.slot_count();
}

// TwinCipher -> flat [branch][part][prime][N]; returns the form.
int flatten_ct(const fpcrt::TwinCipher& tc, uint64_t* out) {
  int form = -1;
  for (size_t b = 0; b < tc.b.size(); ++b) {
    const auto& ct = std::get<bfv::Ciphertext>(tc.b[b].v);
    const int f = ct.form() == ring::PolyForm::eval ? HEI_FORM_EVAL : HEI_FORM_COEFF;
    if (form >= 0 && f != form) throw ParamError("gpu matmul: branch forms differ");
    form = f;
    for (int p = 0; p < 2; ++p)
      for (const auto& poly : ct.parts[p]) {
        std::memcpy(out, poly.c.data(), poly.c.size() * 8);
        out += poly.c.size();
      }
  }
  return form;
}

fpcrt::TwinCipher unflatten_ct(fpcrt::TwinBackend& be, const uint64_t* in) {
  fpcrt::TwinCipher tc;
  const uint32_t n = be.slot_count();
  for (size_t b = 0; b < 2; ++b) {
    const auto& ctx = bfv_branch(be, b).context();
    bfv::Ciphertext ct;
    ct.params_hash = ctx.hash();
    for (int p = 0; p < 2; ++p)
      for (size_t i = 0; i < ctx.num_primes(); ++i) {
        ring::RingPoly poly = ring::RingPoly::zero(n, ctx.params().q[i], ring::PolyForm::eval);
        std::memcpy(poly.c.data(), in, n * 8);
        in += n;
        ct.parts[p].push_back(std::move(poly));
      }
    tc.b.push_back(bfv::HeCipher{std::move(ct)});
  }
  return tc;
}

std::mutex g_mu;
std::map<std::pair<const fpcrt::TwinBackend*, int>, std::unique_ptr<DeviceSession>> g_sessions;

}  // namespace

DeviceSession& DeviceSession::for_backend(fpcrt::TwinBackend& be, int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(static_cast<const fpcrt::TwinBackend*>(&be), device);
  auto it = g_sessions.find(key);
  if (it == g_sessions.end())
    it = g_sessions.emplace(key, std::unique_ptr<DeviceSession>(new DeviceSession(be, device))).first;
  return *it->second;
}

DeviceSession::DeviceSession(fpcrt::TwinBackend& be, int device) {
  const auto& tp = be.params();
  std::vector<uint64_t> q;
  for (size_t b = 0; b < 2; ++b) {
    const auto& ctx = bfv_branch(be, b).context();
    L_[b] = static_cast<uint32_t>(ctx.num_primes());
    for (uint64_t qi : ctx.params().q) q.push_back(qi);
  }
  n_ = tp.n;
  hei_twin_desc d{};
  d.n = tp.n;
  d.t[0] = tp.t.t0;
  d.t[1] = tp.t.t1;
  d.L[0] = L_[0];
  d.L[1] = L_[1];
  d.q = q.data();
  d.s_x = tp.scaling.s_x;
  d.s_w = tp.scaling.s_w;
  d.input_int_bits = tp.scaling.input_int_bits;
  d.device = device;
  check(hei_gpu_ctx_create(&d, &ctx_));
  for (size_t b = 0; b < 2; ++b) {
    const auto& gks = bfv_branch(be, b).galois_keys();
    if (gks.keys.empty()) continue;  // fold then raises KeyError like the reference
    std::vector<uint64_t> elts, rows;
    const size_t L = L_[b];
    for (const auto& [elt, key] : gks.keys) {  // std::map: ascending elements
      elts.push_back(elt);
      for (size_t l = 0; l < L; ++l)
        for (int p = 0; p < 2; ++p)
          for (size_t i = 0; i < L; ++i) rows.insert(rows.end(), key.rows[l][p][i].vals.begin(), key.rows[l][p][i].vals.end());
    }
    check(hei_gpu_upload_galois_keys(ctx_, static_cast<uint32_t>(b), static_cast<uint32_t>(elts.size()), elts.data(),
                                     rows.data()));
  }
}

DeviceSession::~DeviceSession() {
  for (auto& e : wcache_) hei_gpu_weights_destroy(e.second);
  hei_gpu_ctx_destroy(ctx_);
}

hei_gpu_weights* DeviceSession::weights(const EncodedWeights& w) {
  for (auto& e : wcache_)
    if (e.first.p == &w && e.first.f == w.f && e.first.cols == w.outputs.size()) return e.second;
  const uint64_t cols = w.outputs.size();
  if (cols == 0 || w.f == 0) throw ParamError("matmul: empty weights");
  const uint64_t k = (w.f + n_ - 1) / n_;
  std::vector<uint64_t> flat;
  flat.reserve(cols * k * (L_[0] + L_[1]) * n_);
  for (const auto& row : w.outputs) {
    if (row.size() != k) throw ParamError("matmul: ragged weight encoding");
    for (const auto& tp : row)
      for (size_t b = 0; b < 2; ++b)
        for (const auto& pp : std::get<bfv::EvalPlain>(tp.b[b].v).primes) flat.insert(flat.end(), pp.vals.begin(), pp.vals.end());
  }
  hei_gpu_weights* h = nullptr;
  check(hei_gpu_weights_create(ctx_, flat.data(), w.f, cols, &h));
  wcache_.push_back({{&w, w.f, cols}, h});
  return h;
}

void DeviceSession::upload_public_keys(const std::vector<bfv::PublicKey>& pub) {
  if (pub.size() != 2) throw KeyError("baseline: need one public key per branch");
  for (size_t b = 0; b < 2; ++b) {
    std::vector<uint64_t> flat;
    for (const auto& p : pub[b].p0) flat.insert(flat.end(), p.c.begin(), p.c.end());
    for (const auto& p : pub[b].p1) flat.insert(flat.end(), p.c.begin(), p.c.end());
    check(hei_gpu_upload_public_key(ctx_, static_cast<uint32_t>(b), flat.data()));
  }
}

static OpCounters to_counters(const hei_op_counters& c) {
  OpCounters o;
  o.mul_plain_count = c.mul_plain_count;
  o.rotation_count = c.rotation_count;
  o.add_count = c.add_count;
  o.ciphertexts_in = c.ciphertexts_in;
  o.ciphertexts_out = c.ciphertexts_out;
  return o;
}

PackedResult matmul(fpcrt::TwinBackend& be, const EncodedInputs& x, const EncodedWeights& w, const EncodedBias& b,
                    OpCounters* counters, unsigned /*threads: the device path is batch-parallel*/) {
  if (x.rows.empty()) throw ParamError("matmul: empty input");
  if (x.f != w.f || x.n != w.n) throw ParamError("matmul: input and weight shapes do not match");
  auto& sess = DeviceSession::for_backend(be);
  hei_gpu_weights* hw = sess.weights(w);
  const size_t words = twin_words(be);
  const uint64_t k = (w.f + w.n - 1) / w.n;
  std::vector<uint64_t> in(x.rows.size() * k * words);
  int form = -1;
  for (size_t r = 0; r < x.rows.size(); ++r) {
    if (x.rows[r].chunks.size() != k) throw ParamError("push_row: row has the wrong chunk count");
    for (size_t c = 0; c < k; ++c) {
      const int f = flatten_ct(x.rows[r].chunks[c], in.data() + (r * k + c) * words);
      if (form >= 0 && f != form) throw ParamError("gpu matmul: mixed input forms");
      form = f;
    }
  }
  const uint64_t cols = w.outputs.size();
  if (b.scaled.size() != cols) throw ParamError("matmul: bias length does not match output count");
  const uint64_t C = (x.rows.size() * cols + w.n - 1) / w.n;
  std::vector<uint64_t> out(C * words);
  hei_op_counters hc{};
  check(hei_gpu_matmul(sess.ctx(), hw, in.data(), form, x.rows.size(), b.scaled.data(), out.data(), &hc));
  PackedResult pr;
  pr.rows = x.rows.size();
  pr.cols = cols;
  pr.n = w.n;
  for (uint64_t c = 0; c < C; ++c) pr.cts.push_back(unflatten_ct(be, out.data() + c * words));
  if (counters) *counters = to_counters(hc);
  return pr;
}

MatmulStream::MatmulStream(fpcrt::TwinBackend& be, const EncodedWeights& w, const EncodedBias& b, uint64_t total_rows)
    : be_(be), rows_(total_rows), cols_(w.outputs.size()), f_(w.f), n_(w.n) {
  if (total_rows == 0) throw ParamError("matmul: empty input");
  if (b.scaled.size() != cols_) throw ParamError("matmul: bias length does not match output count");
  auto& sess = DeviceSession::for_backend(be);
  check(hei_gpu_stream_create(sess.ctx(), sess.weights(w), b.scaled.data(), total_rows, &s_));
}

MatmulStream::~MatmulStream() { hei_gpu_stream_destroy(s_); }

void MatmulStream::push_row(uint64_t row_index, const EncodedInputRow& row) {
  const uint64_t k = (f_ + n_ - 1) / n_;
  if (row.chunks.size() != k) throw ParamError("push_row: row has the wrong chunk count");
  const size_t words = twin_words(be_);
  std::vector<uint64_t> buf(k * words);
  int form = -1;
  for (size_t c = 0; c < k; ++c) form = flatten_ct(row.chunks[c], buf.data() + c * words);
  check(hei_gpu_stream_push_row(s_, row_index, buf.data(), form));
}

PackedResult MatmulStream::finish() {
  const size_t words = twin_words(be_);
  const uint64_t C = (rows_ * cols_ + n_ - 1) / n_;
  std::vector<uint64_t> out(C * words);
  hei_op_counters hc{};
  check(hei_gpu_stream_finish(s_, out.data(), &hc));
  PackedResult pr;
  pr.rows = rows_;
  pr.cols = cols_;
  pr.n = n_;
  for (uint64_t c = 0; c < C; ++c) pr.cts.push_back(unflatten_ct(be_, out.data() + c * words));
  counters_ = to_counters(hc);
  finished_ = true;
  return pr;
}

const OpCounters& MatmulStream::counters() const {
  if (!finished_) throw ParamError("counters: stream not finished");
  return counters_;
}

BaselineResult baseline_matmul(fpcrt::TwinBackend& be, const std::vector<bfv::PublicKey>& pub, uint64_t rng_seed,
                               const util::IntMat& x, const util::IntMat& w, const EncodedBias& b,
                               OpCounters* counters) {
  if (x.rows == 0 || x.cols == 0 || w.cols == 0) throw ParamError("baseline: empty input");
  if (w.rows != x.cols) throw ParamError("baseline: input and weight shapes do not match");
  if (b.scaled.size() != w.cols) throw ParamError("baseline: bias length does not match output count");
  auto& sess = DeviceSession::for_backend(be);
  sess.upload_public_keys(pub);
  hei_gpu_prng *r0 = nullptr, *r1 = nullptr;
  check(hei_gpu_prng_create(rng_seed, &r0));
  check(hei_gpu_prng_create(rng_seed + 1, &r1));
  std::unique_ptr<hei_gpu_prng, void (*)(hei_gpu_prng*)> g0(r0, hei_gpu_prng_destroy), g1(r1, hei_gpu_prng_destroy);
  const uint32_t n = be.slot_count();
  const size_t words = twin_words(be);
  const uint64_t blocks = x.rows ? (x.rows + n - 1) / n : 0;
  std::vector<uint64_t> out(blocks * w.cols * words);
  hei_op_counters hc{};
  check(hei_gpu_baseline_matmul(sess.ctx(), x.a.data(), x.rows, x.cols, w.a.data(), w.cols, b.scaled.data(), r0, r1,
                                out.data(), &hc));
  BaselineResult res;
  res.rows = x.rows;
  res.cols = w.cols;
  res.n = n;
  res.blocks.resize(blocks);
  for (uint64_t blk = 0; blk < blocks; ++blk)
    for (uint64_t j = 0; j < w.cols; ++j) res.blocks[blk].push_back(unflatten_ct(be, out.data() + (blk * w.cols + j) * words));
  if (counters) *counters = to_counters(hc);
  return res;
}

}  // namespace hei::matmul::gpu

namespace hei::matmul::gpu {

std::vector<std::string> infer_wire(fpcrt::TwinBackend& be, const std::vector<std::string>& ct_blobs, uint64_t rows,
                                    const EncodedWeights& w, const EncodedBias& b, OpCounters* counters) {
  auto& sess = DeviceSession::for_backend(be);
  hei_gpu_weights* hw = sess.weights(w);
  uint64_t hash[2], bytes[2];
  for (size_t br = 0; br < 2; ++br) {
    const auto& cx = bfv_branch(be, br).context();
    hash[br] = cx.hash();
    bytes[br] = hei_hect_ciphertext_bytes(cx.n(), (uint32_t)cx.num_primes());
  }
  // Concatenate. load_ciphertext reads exactly one object from each blob:
  // a short blob fails with util::read_bytes's CodecError (io.hpp:26-30),
  // trailing bytes are ignored.
  std::string all;
  all.reserve(ct_blobs.size() * (bytes[0] + bytes[1]) / 2);
  for (size_t i = 0; i < ct_blobs.size(); ++i) {
    if (ct_blobs[i].size() < bytes[i % 2]) throw CodecError("unexpected end of stream");
    all.append(ct_blobs[i], 0, bytes[i % 2]);
  }
  const uint64_t cols = w.outputs.size();
  const uint64_t C = rows ? (rows * cols + w.n - 1) / w.n : 0;
  std::vector<uint8_t> out(std::max<uint64_t>(C, 1) * (bytes[0] + bytes[1]));
  uint64_t out_len = 0;
  hei_op_counters hc{};
  check(hei_gpu_matmul_wire(sess.ctx(), hw, hash, reinterpret_cast<const uint8_t*>(all.data()), all.size(), rows,
                            b.scaled.data(), out.data(), out.size(), &out_len, &hc));
  std::vector<std::string> res;
  const uint8_t* p = out.data();
  for (uint64_t c = 0; c < C; ++c)
    for (size_t br = 0; br < 2; ++br) {
      res.emplace_back(reinterpret_cast<const char*>(p), bytes[br]);
      p += bytes[br];
    }
  if (counters) *counters = to_counters(hc);
  return res;
}

}  // namespace hei::matmul::gpu
