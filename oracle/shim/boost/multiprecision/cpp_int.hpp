// TEST INFRASTRUCTURE ONLY — part of the parity oracle under oracle/.
//
// A minimal, header-only stand-in for the slice of Boost.Multiprecision that
// the Lynx reference (`/root/reference/proj`) uses, so that the reference's
// own, unmodified `proj/src/*.cpp` compile into `oracle/_ref/` as the CPU
// ground truth. Boost is not installed in this image and its version is
// unpinned by the reference (`proj/src/CMakeLists.txt:1`), so this shim
// restates the published semantics of the API surface actually used:
//
//   cpp_int       arbitrary-precision signed integer; / and % truncate toward
//                 zero (C++ semantics), str() is base-10.
//   cpp_rational  normalized fraction (gcd(num,den)=1, den>0); exact
//                 construction from integers and from finite doubles.
//   numerator / denominator / abs / gcd / lcm, explicit conversions to
//   int64 and double.
//
// Call sites: proj/include/lynx/rational.hpp:22,29-33; proj/src/rational.cpp:25-139;
// proj/src/ilp_exhaustive.cpp:32-58; proj/src/optsched.cpp:199-203;
// proj/src/partition.cpp:69-70; proj/tools/lynx_main.cpp:129-131.
//
// Representation: an int64 fast path (no heap) that promotes to a
// sign-magnitude base-2^32 limb vector on overflow and demotes back when the
// value fits again. The product code under paper_2406_08756_b200/ never
// includes this file.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace boost {
namespace multiprecision {

class cpp_int {
 public:
  cpp_int() = default;
  template <class T, typename std::enable_if<std::is_integral<T>::value, int>::type = 0>
  cpp_int(T v) {  // NOLINT: implicit like Boost
    if constexpr (std::is_signed<T>::value) {
      small_ = static_cast<std::int64_t>(v);
    } else {
      if (static_cast<unsigned long long>(v) <=
          static_cast<unsigned long long>(std::numeric_limits<std::int64_t>::max())) {
        small_ = static_cast<std::int64_t>(v);
      } else {
        big_ = true;
        neg_ = false;
        unsigned long long u = v;
        while (u) {
          mag_.push_back(static_cast<std::uint32_t>(u));
          u >>= 32;
        }
      }
    }
  }
  explicit cpp_int(const std::string& s) { *this = from_string(s); }

  // ---- observers -------------------------------------------------------
  int sign() const {
    if (!big_) return small_ < 0 ? -1 : (small_ > 0 ? 1 : 0);
    return mag_.empty() ? 0 : (neg_ ? -1 : 1);
  }
  bool is_zero() const { return sign() == 0; }

  explicit operator std::int64_t() const {
    if (!big_) return small_;
    // Boost saturates out-of-range conversions; keep the low bits otherwise.
    unsigned long long u = 0;
    for (std::size_t i = 0; i < mag_.size() && i < 2; ++i)
      u |= static_cast<unsigned long long>(mag_[i]) << (32 * i);
    return neg_ ? -static_cast<std::int64_t>(u) : static_cast<std::int64_t>(u);
  }
  explicit operator int() const { return static_cast<int>(static_cast<std::int64_t>(*this)); }
  explicit operator double() const {
    if (!big_) return static_cast<double>(small_);
    double r = 0;
    for (std::size_t i = mag_.size(); i-- > 0;) r = r * 4294967296.0 + mag_[i];
    return neg_ ? -r : r;
  }
  explicit operator bool() const { return !is_zero(); }

  std::string str() const {
    if (!big_) return std::to_string(small_);
    std::vector<std::uint32_t> m = mag_;
    std::string digits;
    while (!m.empty()) {
      std::uint32_t rem = divmod_small(m, 1000000000u);
      for (int k = 0; k < 9; ++k) {
        digits.push_back(static_cast<char>('0' + rem % 10));
        rem /= 10;
        if (m.empty() && rem == 0) break;
      }
    }
    while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
    if (digits.empty()) digits = "0";
    if (neg_) digits.push_back('-');
    std::reverse(digits.begin(), digits.end());
    return digits;
  }

  // ---- arithmetic --------------------------------------------------------
  friend cpp_int operator+(const cpp_int& a, const cpp_int& b) {
    if (!a.big_ && !b.big_) {
      std::int64_t r;
      if (!__builtin_add_overflow(a.small_, b.small_, &r)) return cpp_int(r);
    }
    return add_signed(a.to_sm(), b.to_sm(), false);
  }
  friend cpp_int operator-(const cpp_int& a, const cpp_int& b) {
    if (!a.big_ && !b.big_) {
      std::int64_t r;
      if (!__builtin_sub_overflow(a.small_, b.small_, &r)) return cpp_int(r);
    }
    return add_signed(a.to_sm(), b.to_sm(), true);
  }
  friend cpp_int operator*(const cpp_int& a, const cpp_int& b) {
    if (!a.big_ && !b.big_) {
      std::int64_t r;
      if (!__builtin_mul_overflow(a.small_, b.small_, &r)) return cpp_int(r);
    }
    SM x = a.to_sm(), y = b.to_sm();
    SM z{x.neg != y.neg, mul_mag(x.mag, y.mag)};
    return from_sm(std::move(z));
  }
  friend cpp_int operator/(const cpp_int& a, const cpp_int& b) {
    if (b.is_zero()) throw std::domain_error("cpp_int: division by zero");
    if (!a.big_ && !b.big_ && !(a.small_ == std::numeric_limits<std::int64_t>::min() && b.small_ == -1))
      return cpp_int(a.small_ / b.small_);
    SM x = a.to_sm(), y = b.to_sm();
    std::vector<std::uint32_t> q, r;
    divmod_mag(x.mag, y.mag, q, r);
    return from_sm(SM{x.neg != y.neg, std::move(q)});
  }
  friend cpp_int operator%(const cpp_int& a, const cpp_int& b) {
    if (b.is_zero()) throw std::domain_error("cpp_int: division by zero");
    if (!a.big_ && !b.big_ && !(a.small_ == std::numeric_limits<std::int64_t>::min() && b.small_ == -1))
      return cpp_int(a.small_ % b.small_);
    SM x = a.to_sm(), y = b.to_sm();
    std::vector<std::uint32_t> q, r;
    divmod_mag(x.mag, y.mag, q, r);
    return from_sm(SM{x.neg, std::move(r)});  // remainder takes the dividend's sign
  }
  cpp_int operator-() const { return cpp_int(0) - *this; }
  cpp_int operator+() const { return *this; }

  cpp_int& operator+=(const cpp_int& o) { return *this = *this + o; }
  cpp_int& operator-=(const cpp_int& o) { return *this = *this - o; }
  cpp_int& operator*=(const cpp_int& o) { return *this = *this * o; }
  cpp_int& operator/=(const cpp_int& o) { return *this = *this / o; }
  cpp_int& operator%=(const cpp_int& o) { return *this = *this % o; }
  cpp_int& operator++() { return *this += 1; }
  cpp_int& operator--() { return *this -= 1; }

  friend int compare(const cpp_int& a, const cpp_int& b) {
    if (!a.big_ && !b.big_) return a.small_ < b.small_ ? -1 : (a.small_ > b.small_ ? 1 : 0);
    SM x = a.to_sm(), y = b.to_sm();
    int sx = x.mag.empty() ? 0 : (x.neg ? -1 : 1);
    int sy = y.mag.empty() ? 0 : (y.neg ? -1 : 1);
    if (sx != sy) return sx < sy ? -1 : 1;
    int c = cmp_mag(x.mag, y.mag);
    return sx < 0 ? -c : c;
  }
  friend bool operator==(const cpp_int& a, const cpp_int& b) { return compare(a, b) == 0; }
  friend bool operator!=(const cpp_int& a, const cpp_int& b) { return compare(a, b) != 0; }
  friend bool operator<(const cpp_int& a, const cpp_int& b) { return compare(a, b) < 0; }
  friend bool operator<=(const cpp_int& a, const cpp_int& b) { return compare(a, b) <= 0; }
  friend bool operator>(const cpp_int& a, const cpp_int& b) { return compare(a, b) > 0; }
  friend bool operator>=(const cpp_int& a, const cpp_int& b) { return compare(a, b) >= 0; }

  friend std::ostream& operator<<(std::ostream& os, const cpp_int& v) { return os << v.str(); }

  // Used by cpp_rational's exact double constructor.
  cpp_int shifted_left(unsigned bits) const {
    SM x = to_sm();
    if (x.mag.empty()) return *this;
    std::vector<std::uint32_t> r(bits / 32, 0);
    unsigned sh = bits % 32;
    std::uint32_t carry = 0;
    for (std::uint32_t limb : x.mag) {
      r.push_back(sh ? ((limb << sh) | carry) : limb);
      carry = sh ? (limb >> (32 - sh)) : 0;
    }
    if (carry) r.push_back(carry);
    return from_sm(SM{x.neg, std::move(r)});
  }
  unsigned bit_length() const {
    SM x = to_sm();
    if (x.mag.empty()) return 0;
    return 32 * static_cast<unsigned>(x.mag.size() - 1) + (32 - __builtin_clz(x.mag.back()));
  }

 private:
  struct SM {
    bool neg = false;
    std::vector<std::uint32_t> mag;
  };

  static cpp_int from_string(const std::string& s) {
    cpp_int r = 0;
    std::size_t i = 0;
    bool neg = false;
    if (i < s.size() && (s[i] == '-' || s[i] == '+')) neg = s[i++] == '-';
    for (; i < s.size(); ++i) {
      if (s[i] < '0' || s[i] > '9') throw std::invalid_argument("cpp_int: bad digit");
      r = r * 10 + (s[i] - '0');
    }
    return neg ? -r : r;
  }

  SM to_sm() const {
    if (big_) return SM{neg_, mag_};
    SM r;
    r.neg = small_ < 0;
    unsigned long long u = r.neg ? (0ull - static_cast<unsigned long long>(small_))
                                 : static_cast<unsigned long long>(small_);
    while (u) {
      r.mag.push_back(static_cast<std::uint32_t>(u));
      u >>= 32;
    }
    return r;
  }

  static cpp_int from_sm(SM s) {
    trim(s.mag);
    cpp_int r;
    if (s.mag.size() <= 2) {
      unsigned long long u = 0;
      for (std::size_t i = 0; i < s.mag.size(); ++i)
        u |= static_cast<unsigned long long>(s.mag[i]) << (32 * i);
      const unsigned long long lim = static_cast<unsigned long long>(std::numeric_limits<std::int64_t>::max());
      if (u <= lim) {
        r.small_ = s.neg ? -static_cast<std::int64_t>(u) : static_cast<std::int64_t>(u);
        return r;
      }
      if (s.neg && u == lim + 1) {
        r.small_ = std::numeric_limits<std::int64_t>::min();
        return r;
      }
    }
    r.big_ = true;
    r.neg_ = s.neg;
    r.mag_ = std::move(s.mag);
    return r;
  }

  static void trim(std::vector<std::uint32_t>& m) {
    while (!m.empty() && m.back() == 0) m.pop_back();
  }
  static int cmp_mag(const std::vector<std::uint32_t>& a, const std::vector<std::uint32_t>& b) {
    if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
    for (std::size_t i = a.size(); i-- > 0;)
      if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
  }
  static std::vector<std::uint32_t> add_mag(const std::vector<std::uint32_t>& a,
                                            const std::vector<std::uint32_t>& b) {
    std::vector<std::uint32_t> r;
    std::uint64_t carry = 0;
    for (std::size_t i = 0; i < std::max(a.size(), b.size()); ++i) {
      std::uint64_t s = carry;
      if (i < a.size()) s += a[i];
      if (i < b.size()) s += b[i];
      r.push_back(static_cast<std::uint32_t>(s));
      carry = s >> 32;
    }
    if (carry) r.push_back(static_cast<std::uint32_t>(carry));
    return r;
  }
  // requires a >= b
  static std::vector<std::uint32_t> sub_mag(const std::vector<std::uint32_t>& a,
                                            const std::vector<std::uint32_t>& b) {
    std::vector<std::uint32_t> r(a.size());
    std::int64_t borrow = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
      std::int64_t d = static_cast<std::int64_t>(a[i]) - borrow - (i < b.size() ? b[i] : 0);
      borrow = d < 0;
      if (d < 0) d += (1ll << 32);
      r[i] = static_cast<std::uint32_t>(d);
    }
    trim(r);
    return r;
  }
  static std::vector<std::uint32_t> mul_mag(const std::vector<std::uint32_t>& a,
                                            const std::vector<std::uint32_t>& b) {
    if (a.empty() || b.empty()) return {};
    std::vector<std::uint32_t> r(a.size() + b.size(), 0);
    for (std::size_t i = 0; i < a.size(); ++i) {
      std::uint64_t carry = 0;
      for (std::size_t j = 0; j < b.size(); ++j) {
        std::uint64_t t = static_cast<std::uint64_t>(a[i]) * b[j] + r[i + j] + carry;
        r[i + j] = static_cast<std::uint32_t>(t);
        carry = t >> 32;
      }
      std::size_t k = i + b.size();
      while (carry) {
        std::uint64_t t = static_cast<std::uint64_t>(r[k]) + carry;
        r[k++] = static_cast<std::uint32_t>(t);
        carry = t >> 32;
      }
    }
    trim(r);
    return r;
  }
  static std::uint32_t divmod_small(std::vector<std::uint32_t>& m, std::uint32_t d) {
    std::uint64_t rem = 0;
    for (std::size_t i = m.size(); i-- > 0;) {
      std::uint64_t cur = (rem << 32) | m[i];
      m[i] = static_cast<std::uint32_t>(cur / d);
      rem = cur % d;
    }
    trim(m);
    return static_cast<std::uint32_t>(rem);
  }
  // Schoolbook binary long division (the oracle rarely leaves the int64 path).
  static void divmod_mag(const std::vector<std::uint32_t>& a, const std::vector<std::uint32_t>& b,
                         std::vector<std::uint32_t>& q, std::vector<std::uint32_t>& r) {
    q.clear();
    r.clear();
    if (cmp_mag(a, b) < 0) {
      r = a;
      return;
    }
    if (b.size() == 1) {
      q = a;
      std::uint32_t rem = divmod_small(q, b[0]);
      if (rem) r.push_back(rem);
      return;
    }
    q.assign(a.size(), 0);
    for (std::size_t i = a.size(); i-- > 0;) {
      for (int bit = 31; bit >= 0; --bit) {
        // r = r*2 + bit
        std::uint32_t carry = (a[i] >> bit) & 1u;
        for (auto& limb : r) {
          std::uint32_t nc = limb >> 31;
          limb = (limb << 1) | carry;
          carry = nc;
        }
        if (carry) r.push_back(carry);
        if (cmp_mag(r, b) >= 0) {
          r = sub_mag(r, b);
          q[i] |= (1u << bit);
        }
      }
    }
    trim(q);
    trim(r);
  }
  static cpp_int add_signed(SM x, SM y, bool subtract) {
    if (subtract) y.neg = !y.neg;
    if (x.neg == y.neg) return from_sm(SM{x.neg, add_mag(x.mag, y.mag)});
    int c = cmp_mag(x.mag, y.mag);
    if (c == 0) return cpp_int(0);
    if (c > 0) return from_sm(SM{x.neg, sub_mag(x.mag, y.mag)});
    return from_sm(SM{y.neg, sub_mag(y.mag, x.mag)});
  }

  bool big_ = false;
  std::int64_t small_ = 0;
  bool neg_ = false;
  std::vector<std::uint32_t> mag_;
};

inline cpp_int abs(const cpp_int& v) { return v.sign() < 0 ? -v : v; }
inline cpp_int gcd(cpp_int a, cpp_int b) {
  a = abs(a);
  b = abs(b);
  while (!b.is_zero()) {
    cpp_int t = a % b;
    a = std::move(b);
    b = std::move(t);
  }
  return a;
}
inline cpp_int lcm(const cpp_int& a, const cpp_int& b) {
  if (a.is_zero() || b.is_zero()) return cpp_int(0);
  return abs(a / gcd(a, b) * b);
}

class cpp_rational {
 public:
  cpp_rational() : num_(0), den_(1) {}
  template <class T, typename std::enable_if<std::is_integral<T>::value, int>::type = 0>
  cpp_rational(T v) : num_(v), den_(1) {}  // NOLINT: implicit like Boost
  cpp_rational(const cpp_int& v) : num_(v), den_(1) {}  // NOLINT
  cpp_rational(double d) : num_(0), den_(1) {            // NOLINT: exact, like Boost
    if (!std::isfinite(d)) throw std::domain_error("cpp_rational: non-finite double");
    if (d == 0) return;
    int exp = 0;
    double m = std::frexp(d, &exp);  // d = m * 2^exp, 0.5 <= |m| < 1
    // 53 significant bits -> integer mantissa
    long long mant = static_cast<long long>(std::ldexp(m, 53));
    exp -= 53;
    num_ = cpp_int(mant);
    if (exp >= 0) {
      num_ = num_.shifted_left(static_cast<unsigned>(exp));
    } else {
      den_ = cpp_int(1).shifted_left(static_cast<unsigned>(-exp));
    }
    normalize();
  }
  cpp_rational(const cpp_int& n, const cpp_int& d) : num_(n), den_(d) {
    if (den_.is_zero()) throw std::domain_error("cpp_rational: zero denominator");
    normalize();
  }

  friend const cpp_int& numerator_ref(const cpp_rational& r) { return r.num_; }
  friend const cpp_int& denominator_ref(const cpp_rational& r) { return r.den_; }

  friend cpp_rational operator+(const cpp_rational& a, const cpp_rational& b) {
    if (a.den_ == b.den_) return cpp_rational(a.num_ + b.num_, a.den_);
    return cpp_rational(a.num_ * b.den_ + b.num_ * a.den_, a.den_ * b.den_);
  }
  friend cpp_rational operator-(const cpp_rational& a, const cpp_rational& b) {
    if (a.den_ == b.den_) return cpp_rational(a.num_ - b.num_, a.den_);
    return cpp_rational(a.num_ * b.den_ - b.num_ * a.den_, a.den_ * b.den_);
  }
  friend cpp_rational operator*(const cpp_rational& a, const cpp_rational& b) {
    return cpp_rational(a.num_ * b.num_, a.den_ * b.den_);
  }
  friend cpp_rational operator/(const cpp_rational& a, const cpp_rational& b) {
    if (b.num_.is_zero()) throw std::domain_error("cpp_rational: division by zero");
    return cpp_rational(a.num_ * b.den_, a.den_ * b.num_);
  }
  cpp_rational operator-() const {
    cpp_rational r = *this;
    r.num_ = -r.num_;
    return r;
  }
  cpp_rational operator+() const { return *this; }
  cpp_rational& operator+=(const cpp_rational& o) { return *this = *this + o; }
  cpp_rational& operator-=(const cpp_rational& o) { return *this = *this - o; }
  cpp_rational& operator*=(const cpp_rational& o) { return *this = *this * o; }
  cpp_rational& operator/=(const cpp_rational& o) { return *this = *this / o; }

  friend int compare(const cpp_rational& a, const cpp_rational& b) {
    if (a.den_ == b.den_) return compare(a.num_, b.num_);
    return compare(a.num_ * b.den_, b.num_ * a.den_);
  }
  friend bool operator==(const cpp_rational& a, const cpp_rational& b) {
    return a.num_ == b.num_ && a.den_ == b.den_;
  }
  friend bool operator!=(const cpp_rational& a, const cpp_rational& b) { return !(a == b); }
  friend bool operator<(const cpp_rational& a, const cpp_rational& b) { return compare(a, b) < 0; }
  friend bool operator<=(const cpp_rational& a, const cpp_rational& b) { return compare(a, b) <= 0; }
  friend bool operator>(const cpp_rational& a, const cpp_rational& b) { return compare(a, b) > 0; }
  friend bool operator>=(const cpp_rational& a, const cpp_rational& b) { return compare(a, b) >= 0; }

  explicit operator double() const {
    // Scale the quotient to >= 64 significant bits, then round once.
    if (num_.is_zero()) return 0.0;
    cpp_int n = abs(num_);
    int nb = static_cast<int>(n.bit_length()), db = static_cast<int>(den_.bit_length());
    int shift = 65 - (nb - db);
    cpp_int q = shift > 0 ? n.shifted_left(static_cast<unsigned>(shift)) / den_
                          : n / den_.shifted_left(static_cast<unsigned>(-shift));
    double r = std::ldexp(static_cast<double>(q), -shift);
    return num_.sign() < 0 ? -r : r;
  }

  friend std::ostream& operator<<(std::ostream& os, const cpp_rational& r) {
    os << r.num_;
    if (r.den_ != 1) os << "/" << r.den_;
    return os;
  }

 private:
  void normalize() {
    if (den_.sign() < 0) {
      num_ = -num_;
      den_ = -den_;
    }
    if (num_.is_zero()) {
      den_ = 1;
      return;
    }
    if (den_ == 1) return;
    cpp_int g = gcd(num_, den_);
    if (g != 1) {
      num_ /= g;
      den_ /= g;
    }
  }

  cpp_int num_;
  cpp_int den_;
};

inline cpp_int numerator(const cpp_rational& r) { return numerator_ref(r); }
inline cpp_int denominator(const cpp_rational& r) { return denominator_ref(r); }
inline cpp_rational abs(const cpp_rational& r) { return r < 0 ? -r : r; }

}  // namespace multiprecision
}  // namespace boost
