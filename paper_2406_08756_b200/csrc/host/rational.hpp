// Exact rational arithmetic for the host planner.
//
// The reference computes every time and byte quantity of the planner,
// schedulers and ledger exactly (`proj/include/lynx/rational.hpp:22-54`, on
// Boost cpp_rational). Plans, peak memory and liveness must be bit-exact, so
// this restatement is exact too: an int64 numerator/denominator fast path
// (all profile quantities fit, and int64 x int64 products are formed in
// __int128) that falls back to an arbitrary-precision BigInt pair when a
// result leaves int64 — e.g. the 2^-(i+1) retention tie-break weights of
// heusched.cpp:227-232 on long templates.
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <string>
#include <string_view>
#include <vector>

namespace lynx::host {

// Sign-magnitude arbitrary-precision integer (base 2^32 limbs).
class BigInt {
 public:
  BigInt() = default;
  BigInt(long long v);  // NOLINT
  BigInt(long v) : BigInt(static_cast<long long>(v)) {}  // NOLINT
  BigInt(int v) : BigInt(static_cast<long long>(v)) {}   // NOLINT
  static BigInt from_i128(__int128 v);

  bool is_zero() const { return mag_.empty(); }
  bool negative() const { return neg_; }
  int sign() const { return mag_.empty() ? 0 : (neg_ ? -1 : 1); }
  bool fits_i64() const;
  long long to_i64() const;  // requires fits_i64()
  double to_double() const;
  std::string str() const;
  unsigned bit_length() const;

  friend BigInt operator+(const BigInt& a, const BigInt& b);
  friend BigInt operator-(const BigInt& a, const BigInt& b);
  friend BigInt operator*(const BigInt& a, const BigInt& b);
  // Truncating division / remainder (C++ semantics).
  static void divmod(const BigInt& a, const BigInt& b, BigInt& q, BigInt& r);
  friend BigInt operator/(const BigInt& a, const BigInt& b);
  friend BigInt operator%(const BigInt& a, const BigInt& b);
  BigInt operator-() const;
  BigInt shl(unsigned bits) const;
  friend int cmp(const BigInt& a, const BigInt& b);
  friend bool operator==(const BigInt& a, const BigInt& b) { return cmp(a, b) == 0; }
  friend bool operator!=(const BigInt& a, const BigInt& b) { return cmp(a, b) != 0; }
  friend bool operator<(const BigInt& a, const BigInt& b) { return cmp(a, b) < 0; }
  static BigInt gcd(BigInt a, BigInt b);
  static BigInt pow10(unsigned n);

 private:
  bool neg_ = false;
  std::vector<uint32_t> mag_;
  void trim();
};

class Rat {
 public:
  Rat() = default;
  Rat(long long v) : n_(v), d_(1) {}  // NOLINT: implicit like the reference's Rat
  Rat(int v) : n_(v), d_(1) {}        // NOLINT
  Rat(long v) : n_(v), d_(1) {}       // NOLINT (int64_t)
  static Rat frac(long long n, long long d);
  static Rat from_big(BigInt n, BigInt d);
  static Rat from_double(double v);  // exact (doubles are dyadic)

  BigInt num() const;
  BigInt den() const;
  bool is_small() const { return !big_; }
  bool is_integer() const;
  int sign() const;
  double to_double() const;

  friend Rat operator+(const Rat& a, const Rat& b);
  friend Rat operator-(const Rat& a, const Rat& b);
  friend Rat operator*(const Rat& a, const Rat& b);
  friend Rat operator/(const Rat& a, const Rat& b);
  Rat operator-() const;
  Rat& operator+=(const Rat& o) { return *this = *this + o; }
  Rat& operator-=(const Rat& o) { return *this = *this - o; }
  Rat& operator*=(const Rat& o) { return *this = *this * o; }
  Rat& operator/=(const Rat& o) { return *this = *this / o; }

  friend int cmp(const Rat& a, const Rat& b);
  friend bool operator==(const Rat& a, const Rat& b);
  friend bool operator!=(const Rat& a, const Rat& b) { return !(a == b); }
  friend bool operator<(const Rat& a, const Rat& b) { return cmp(a, b) < 0; }
  friend bool operator<=(const Rat& a, const Rat& b) { return cmp(a, b) <= 0; }
  friend bool operator>(const Rat& a, const Rat& b) { return cmp(a, b) > 0; }
  friend bool operator>=(const Rat& a, const Rat& b) { return cmp(a, b) >= 0; }

 private:
  struct Big {
    BigInt n, d;
  };
  long long n_ = 0, d_ = 1;        // valid when big_ == nullptr
  std::shared_ptr<const Big> big_;  // immutable; shared on copy
  static Rat make_small_or_big(__int128 n, __int128 d);
  static Rat normalize_big(BigInt n, BigInt d);
};

inline Rat rmin(const Rat& a, const Rat& b) { return a < b ? a : b; }
inline Rat rmax(const Rat& a, const Rat& b) { return a < b ? b : a; }

// Parsers / printers with the reference's exact text semantics
// (proj/src/rational.cpp:84-137).
std::optional<Rat> parse_rat(std::string_view text);
std::string to_canonical(const Rat& r);          // integer | terminating decimal | num/den
std::string to_fixed(const Rat& r, int digits);  // round half away from zero
BigInt ceil_nonneg(const Rat& r);                // ceil for r >= 0

}  // namespace lynx::host
