// HECT ciphertext (de)serialisation kernels. Textually included by
// heinfer_b200.cu inside its kernel namespace (uses Geo, poly_prime).
#pragma once

// ---------------------------------------------------------------------------
// HECT wire format (proj/include/hei/bfv/serialize.hpp:18-24,
// proj/src/bfv/serialize.cpp:19-27,44-48,63-78): a ciphertext blob is
//   "HECT" | version u16 | params_hash u64 | parts u32 (=2) | kind u8 (=5)
// followed by 2·L polys [part][prime], each [form u8 | n x u64 LE], coeff form.
// The 19-byte header makes every u64 unaligned, so the device reads/writes
// them through aligned 32-bit words and funnel shifts.
// ---------------------------------------------------------------------------
constexpr uint32_t kHectHeader = 19;

struct WireGeo {
  uint64_t blob[2];  // bytes of one branch blob
  uint64_t hash[2];  // params_hash per branch
};

__device__ __forceinline__ uint64_t wire_offset(const Geo& g, const WireGeo& wg, uint64_t x, uint32_t& poly,
                                                uint32_t& j) {
  const uint64_t ct = x / g.ct_words;
  const uint32_t w = (uint32_t)(x % g.ct_words);
  poly = w / g.n;
  j = w % g.n;
  const uint32_t b = poly >= 2 * g.L[0];
  const uint32_t lp = b ? poly - 2 * g.L[0] : poly;
  return ct * (wg.blob[0] + wg.blob[1]) + (b ? wg.blob[0] : 0) + kHectHeader + (uint64_t)lp * (1 + 8ull * g.n) + 1 +
         8ull * j;
}

// bytes (rows·kc twin blobs, padded by >= 8 bytes) -> u32 coeff residues.
// err bit 1: coefficient >= q; bit 2: a poly's form byte is not coeff.
__global__ void k_wire_parse(Geo g, WireGeo wg, const uint8_t* __restrict__ in, uint32_t* __restrict__ out,
                             uint64_t cts, uint32_t* err) {
  const uint64_t total = cts * g.ct_words;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t poly, j;
    const uint64_t off = wire_offset(g, wg, x, poly, j);
    const uint32_t* a = reinterpret_cast<const uint32_t*>(in + (off & ~3ull));
    const uint32_t sh = (uint32_t)(off & 3) * 8;
    const uint32_t w0 = __ldg(a), w1 = __ldg(a + 1), w2 = __ldg(a + 2);
    const uint32_t lo = __funnelshift_r(w0, w1, sh), hi = __funnelshift_r(w1, w2, sh);
    if (hi != 0 || lo >= g.pr[poly_prime(g, poly)].q) atomicOr(err, 1u);
    if (j == 0 && in[off - 1] != 0) atomicOr(err, 2u);
    out[x] = lo;
  }
}

// u32 coeff residues (cts twin ciphertexts) -> HECT bytes, headers included.
__global__ void k_wire_emit(Geo g, WireGeo wg, const uint32_t* __restrict__ in, uint8_t* __restrict__ out,
                            uint64_t cts) {
  const uint64_t total = cts * g.ct_words;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t poly, j;
    const uint64_t off = wire_offset(g, wg, x, poly, j);
    const uint32_t v = in[x];
    uint8_t* o = out + off;
#pragma unroll
    for (int k = 0; k < 4; ++k) o[k] = (uint8_t)(v >> (8 * k));
#pragma unroll
    for (int k = 4; k < 8; ++k) o[k] = 0;
    if (j == 0) {
      o[-1] = 0;  // PolyForm::coeff
      const uint32_t b = poly >= 2 * g.L[0];
      if (poly == (b ? 2 * g.L[0] : 0)) {  // first poly of a blob writes the header
        uint8_t* h = o - 1 - kHectHeader;
        h[0] = 'H'; h[1] = 'E'; h[2] = 'C'; h[3] = 'T';
        h[4] = 1; h[5] = 0;  // version
        for (int k = 0; k < 8; ++k) h[6 + k] = (uint8_t)(wg.hash[b] >> (8 * k));
        h[14] = 2; h[15] = 0; h[16] = 0; h[17] = 0;  // parts
        h[18] = 5;                                   // ObjectKind::ciphertext
      }
    }
  }
}
