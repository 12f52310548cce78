// TEST INFRASTRUCTURE ONLY — not product code.
//
// Minimal stand-in for boost::multiprecision::cpp_int, written for this repo so
// the unmodified reference sources under /root/reference/proj can be compiled
// into the CPU oracle (oracle/_ref). Boost is not installed in this image.
//
// The reference uses cpp_int only for exact integer constants and the decrypt
// rounding (proj/src/bfv/context.cpp:19-48, :341-368): construction from
// integers, + - * with u64 and bignums, / and % by u64 and bignum, shifts,
// comparisons, unary minus, msb() and an explicit uint64_t conversion. Any
// correct bignum reproduces those values exactly, which is all parity needs.
//
// Representation: sign + magnitude, fixed 8 x 64-bit limbs (512 bits), far
// above the ~340 bits the largest parameter sets reach.
#pragma once

#include <cstdint>
#include <stdexcept>

namespace boost {
namespace multiprecision {

class cpp_int {
 public:
  static constexpr int kLimbs = 8;

  cpp_int() { clear(); }
  cpp_int(int v) { set_signed(v); }
  cpp_int(long v) { set_signed(v); }
  cpp_int(long long v) { set_signed(v); }
  cpp_int(unsigned v) { set_u64(v); }
  cpp_int(unsigned long v) { set_u64(v); }
  cpp_int(unsigned long long v) { set_u64(v); }

  explicit operator uint64_t() const {
    // Boost semantics for negative values are not needed by the reference.
    return neg_ ? static_cast<uint64_t>(-static_cast<int64_t>(m_[0])) : m_[0];
  }

  unsigned msb_bit() const {
    int b = msb_mag(m_);
    if (b < 0) throw std::domain_error("msb of zero");
    return static_cast<unsigned>(b);
  }

  cpp_int operator-() const {
    cpp_int r = *this;
    if (!r.is_zero()) r.neg_ = !r.neg_;
    return r;
  }

  // ---- arithmetic ----
  friend cpp_int operator+(const cpp_int& a, const cpp_int& b) {
    cpp_int r;
    if (a.neg_ == b.neg_) {
      add_mag(r.m_, a.m_, b.m_);
      r.neg_ = a.neg_;
    } else if (cmp_mag(a.m_, b.m_) >= 0) {
      sub_mag(r.m_, a.m_, b.m_);
      r.neg_ = a.neg_;
    } else {
      sub_mag(r.m_, b.m_, a.m_);
      r.neg_ = b.neg_;
    }
    r.normalize();
    return r;
  }
  friend cpp_int operator-(const cpp_int& a, const cpp_int& b) { return a + (-b); }
  friend cpp_int operator*(const cpp_int& a, const cpp_int& b) {
    cpp_int r;
    for (int i = 0; i < kLimbs; ++i) {
      if (!a.m_[i]) continue;
      unsigned __int128 carry = 0;
      for (int j = 0; i + j < kLimbs; ++j) {
        unsigned __int128 cur = static_cast<unsigned __int128>(a.m_[i]) * b.m_[j] +
                                r.m_[i + j] + carry;
        r.m_[i + j] = static_cast<uint64_t>(cur);
        carry = cur >> 64;
      }
      if (carry) throw std::overflow_error("cpp_int stand-in overflow");
    }
    r.neg_ = a.neg_ != b.neg_;
    r.normalize();
    return r;
  }
  friend cpp_int operator/(const cpp_int& a, const cpp_int& b) {
    cpp_int q, r;
    divmod(a, b, q, r);
    return q;
  }
  friend cpp_int operator%(const cpp_int& a, const cpp_int& b) {
    cpp_int q, r;
    divmod(a, b, q, r);
    return r;
  }
  friend cpp_int operator<<(const cpp_int& a, unsigned s) {
    cpp_int r = a;
    shl_mag(r.m_, s);
    return r;
  }
  friend cpp_int operator>>(const cpp_int& a, unsigned s) {
    cpp_int r = a;
    shr_mag(r.m_, s);
    r.normalize();
    return r;
  }

  cpp_int& operator+=(const cpp_int& b) { return *this = *this + b; }
  cpp_int& operator-=(const cpp_int& b) { return *this = *this - b; }
  cpp_int& operator*=(const cpp_int& b) { return *this = *this * b; }

  // ---- comparison ----
  friend int compare(const cpp_int& a, const cpp_int& b) {
    if (a.neg_ != b.neg_) return a.neg_ ? -1 : 1;
    int c = cmp_mag(a.m_, b.m_);
    return a.neg_ ? -c : c;
  }
  friend bool operator<(const cpp_int& a, const cpp_int& b) { return compare(a, b) < 0; }
  friend bool operator>(const cpp_int& a, const cpp_int& b) { return compare(a, b) > 0; }
  friend bool operator<=(const cpp_int& a, const cpp_int& b) { return compare(a, b) <= 0; }
  friend bool operator>=(const cpp_int& a, const cpp_int& b) { return compare(a, b) >= 0; }
  friend bool operator==(const cpp_int& a, const cpp_int& b) { return compare(a, b) == 0; }
  friend bool operator!=(const cpp_int& a, const cpp_int& b) { return compare(a, b) != 0; }

 private:
  uint64_t m_[kLimbs];
  bool neg_ = false;

  void clear() {
    for (auto& x : m_) x = 0;
    neg_ = false;
  }
  void set_u64(uint64_t v) {
    clear();
    m_[0] = v;
  }
  void set_signed(long long v) {
    clear();
    if (v < 0) {
      m_[0] = static_cast<uint64_t>(-(v + 1)) + 1;
      neg_ = true;
    } else {
      m_[0] = static_cast<uint64_t>(v);
    }
  }
  bool is_zero() const {
    for (auto x : m_)
      if (x) return false;
    return true;
  }
  void normalize() {
    if (is_zero()) neg_ = false;
  }
  static int cmp_mag(const uint64_t* a, const uint64_t* b) {
    for (int i = kLimbs - 1; i >= 0; --i)
      if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
  }
  static void add_mag(uint64_t* r, const uint64_t* a, const uint64_t* b) {
    unsigned __int128 c = 0;
    for (int i = 0; i < kLimbs; ++i) {
      c += static_cast<unsigned __int128>(a[i]) + b[i];
      r[i] = static_cast<uint64_t>(c);
      c >>= 64;
    }
    if (c) throw std::overflow_error("cpp_int stand-in overflow");
  }
  // r = a - b, requires |a| >= |b|
  static void sub_mag(uint64_t* r, const uint64_t* a, const uint64_t* b) {
    uint64_t borrow = 0;
    for (int i = 0; i < kLimbs; ++i) {
      uint64_t ai = a[i], bi = b[i];
      uint64_t d = ai - bi - borrow;
      borrow = (ai < bi) || (ai == bi && borrow) ? 1 : 0;
      r[i] = d;
    }
  }
  static void shl_mag(uint64_t* a, unsigned s) {
    unsigned limbs = s / 64, bits = s % 64;
    for (int i = kLimbs - 1; i >= 0; --i) {
      uint64_t v = 0;
      int src = i - static_cast<int>(limbs);
      if (src >= 0) {
        v = a[src] << bits;
        if (bits && src - 1 >= 0) v |= a[src - 1] >> (64 - bits);
      }
      a[i] = v;
    }
  }
  static void shr_mag(uint64_t* a, unsigned s) {
    unsigned limbs = s / 64, bits = s % 64;
    for (int i = 0; i < kLimbs; ++i) {
      uint64_t v = 0;
      unsigned src = i + limbs;
      if (src < kLimbs) {
        v = a[src] >> bits;
        if (bits && src + 1 < kLimbs) v |= a[src + 1] << (64 - bits);
      }
      a[i] = v;
    }
  }
  static int msb_mag(const uint64_t* a) {
    for (int i = kLimbs - 1; i >= 0; --i)
      if (a[i]) return i * 64 + 63 - __builtin_clzll(a[i]);
    return -1;
  }
  // Truncating division (C++ / and % semantics: quotient toward zero,
  // remainder takes the dividend's sign), shift-subtract on magnitudes.
  static void divmod(const cpp_int& a, const cpp_int& b, cpp_int& q, cpp_int& r) {
    int mb = msb_mag(b.m_);
    if (mb < 0) throw std::domain_error("cpp_int division by zero");
    q.clear();
    r.clear();
    for (int i = 0; i < kLimbs; ++i) r.m_[i] = a.m_[i];
    int ma = msb_mag(a.m_);
    if (ma >= mb) {
      int shift = ma - mb;
      uint64_t d[kLimbs];
      for (int i = 0; i < kLimbs; ++i) d[i] = b.m_[i];
      shl_mag(d, static_cast<unsigned>(shift));
      for (int s = shift; s >= 0; --s) {
        if (cmp_mag(r.m_, d) >= 0) {
          sub_mag(r.m_, r.m_, d);
          q.m_[s / 64] |= uint64_t(1) << (s % 64);
        }
        shr_mag(d, 1);
      }
    }
    q.neg_ = a.neg_ != b.neg_;
    r.neg_ = a.neg_;
    q.normalize();
    r.normalize();
  }
};

inline unsigned msb(const cpp_int& a) { return a.msb_bit(); }

}  // namespace multiprecision
}  // namespace boost
