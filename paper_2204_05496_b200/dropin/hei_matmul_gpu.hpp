// Drop-in C++ adapter: the reference's hei::matmul entry points
// (/root/reference/proj/include/hei/matmul/matmul.hpp:71-140) executed by the
// B200 path through the C ABI (include/heinfer_b200.h).
//
// Compile this header + hei_matmul_gpu.cpp inside the reference's build (it
// uses the reference's own types) and link libheinfer_b200.so. Same
// signatures, argument meaning and exception types as the reference; the
// functions live in hei::matmul::gpu so a maintainer can switch call sites
// (InferenceServer::do_infer, server.cpp:137-158) with a using-declaration,
// or define HEI_GPU_DROPIN to have hei_matmul_gpu.cpp provide
// hei::matmul::matmul itself in place of proj/src/matmul/matmul.cpp.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "hei/bfv/keys.hpp"
#include "hei/matmul/matmul.hpp"

struct hei_gpu_ctx;
struct hei_gpu_weights;
struct hei_gpu_stream;

namespace hei::matmul::gpu {

// Device-resident state for one evaluation backend: context tables and the
// Galois keys of both branches, uploaded once and keyed by backend identity
// and the branch parameter hashes (SURVEY §8b "Ownership").
class DeviceSession {
 public:
  static DeviceSession& for_backend(fpcrt::TwinBackend& be, int device = 0);
  hei_gpu_ctx* ctx() const { return ctx_; }
  // Weights are cached by address (the caller keeps EncodedWeights alive,
  // matmul.hpp:100) and shape.
  hei_gpu_weights* weights(const EncodedWeights& w);
  void upload_public_keys(const std::vector<bfv::PublicKey>& pk);
  ~DeviceSession();

 private:
  DeviceSession(fpcrt::TwinBackend& be, int device);
  hei_gpu_ctx* ctx_ = nullptr;
  struct WKey {
    const EncodedWeights* p;
    uint64_t f, cols;
  };
  std::vector<std::pair<WKey, hei_gpu_weights*>> wcache_;
  uint32_t n_ = 0, L_[2] = {0, 0};
};

PackedResult matmul(fpcrt::TwinBackend& be, const EncodedInputs& x, const EncodedWeights& w, const EncodedBias& b,
                    OpCounters* counters = nullptr, unsigned threads = 0);

class MatmulStream {
 public:
  MatmulStream(fpcrt::TwinBackend& be, const EncodedWeights& w, const EncodedBias& b, uint64_t total_rows);
  ~MatmulStream();
  void push_row(uint64_t row_index, const EncodedInputRow& row);
  PackedResult finish();
  const OpCounters& counters() const;

 private:
  fpcrt::TwinBackend& be_;
  hei_gpu_stream* s_ = nullptr;
  uint64_t rows_, cols_, f_;
  uint32_t n_;
  bool finished_ = false;
  OpCounters counters_;
};

// baseline_matmul (matmul.cpp:273-344). The reference draws encryption
// randomness from BfvBackend's private rng_; the device replays the same
// util::Prng stream from `rng_seed` (branch b uses rng_seed + b, exactly as
// TwinContext::client_backend seeds it, twin.cpp:58). Public keys come from
// TwinKeys::kp[b].pub.
BaselineResult baseline_matmul(fpcrt::TwinBackend& be, const std::vector<bfv::PublicKey>& pub, uint64_t rng_seed,
                               const util::IntMat& x, const util::IntMat& w, const EncodedBias& b,
                               OpCounters* counters = nullptr);

// The computation of InferenceServer::do_infer (server.cpp:137-170) on wire
// objects: `ct_blobs` = the request's HECT ciphertext blobs in request order
// [row][chunk][branch] (InferRequestPayload::ct_blobs); returns the response
// blobs [packed ct][branch] as bfv::save_ciphertext would write them.
// load_ciphertext's CodecErrors and the blob-count check are preserved.
std::vector<std::string> infer_wire(fpcrt::TwinBackend& be, const std::vector<std::string>& ct_blobs, uint64_t rows,
                                    const EncodedWeights& w, const EncodedBias& b, OpCounters* counters = nullptr);

}  // namespace hei::matmul::gpu
