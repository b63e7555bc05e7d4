#include "host/rational.hpp"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <limits>
#include <stdexcept>

namespace lynx::host {

// ============================================================== BigInt
BigInt::BigInt(long long v) {
  neg_ = v < 0;
  unsigned long long u = neg_ ? 0ull - static_cast<unsigned long long>(v) : static_cast<unsigned long long>(v);
  while (u) {
    mag_.push_back(static_cast<uint32_t>(u));
    u >>= 32;
  }
}

BigInt BigInt::from_i128(__int128 v) {
  BigInt r;
  r.neg_ = v < 0;
  unsigned __int128 u = r.neg_ ? static_cast<unsigned __int128>(0) - static_cast<unsigned __int128>(v)
                               : static_cast<unsigned __int128>(v);
  while (u) {
    r.mag_.push_back(static_cast<uint32_t>(u));
    u >>= 32;
  }
  return r;
}

void BigInt::trim() {
  while (!mag_.empty() && mag_.back() == 0) mag_.pop_back();
  if (mag_.empty()) neg_ = false;
}

bool BigInt::fits_i64() const {
  if (mag_.size() > 2) return false;
  unsigned long long u = 0;
  for (size_t i = 0; i < mag_.size(); ++i) u |= static_cast<unsigned long long>(mag_[i]) << (32 * i);
  const unsigned long long lim = static_cast<unsigned long long>(std::numeric_limits<long long>::max());
  return u <= lim || (neg_ && u == lim + 1);
}

long long BigInt::to_i64() const {
  unsigned long long u = 0;
  for (size_t i = 0; i < mag_.size() && i < 2; ++i) u |= static_cast<unsigned long long>(mag_[i]) << (32 * i);
  return neg_ ? static_cast<long long>(0ull - u) : static_cast<long long>(u);
}

double BigInt::to_double() const {
  double r = 0;
  for (size_t i = mag_.size(); i-- > 0;) r = r * 4294967296.0 + mag_[i];
  return neg_ ? -r : r;
}

unsigned BigInt::bit_length() const {
  if (mag_.empty()) return 0;
  return 32u * static_cast<unsigned>(mag_.size() - 1) + (32u - static_cast<unsigned>(__builtin_clz(mag_.back())));
}

namespace {
int cmp_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
  if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
  for (size_t i = a.size(); i-- > 0;)
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  return 0;
}
std::vector<uint32_t> add_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
  std::vector<uint32_t> r(std::max(a.size(), b.size()) + 1, 0);
  uint64_t c = 0;
  for (size_t i = 0; i + 1 < r.size(); ++i) {
    uint64_t s = c + (i < a.size() ? a[i] : 0) + (i < b.size() ? b[i] : 0);
    r[i] = static_cast<uint32_t>(s);
    c = s >> 32;
  }
  r.back() = static_cast<uint32_t>(c);
  return r;
}
// |a| >= |b|
std::vector<uint32_t> sub_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
  std::vector<uint32_t> r(a.size(), 0);
  int64_t br = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    int64_t d = static_cast<int64_t>(a[i]) - br - (i < b.size() ? static_cast<int64_t>(b[i]) : 0);
    br = d < 0 ? 1 : 0;
    r[i] = static_cast<uint32_t>(d + (br << 32));
  }
  return r;
}
}  // namespace

BigInt operator+(const BigInt& a, const BigInt& b) {
  BigInt r;
  if (a.neg_ == b.neg_) {
    r.mag_ = add_mag(a.mag_, b.mag_);
    r.neg_ = a.neg_;
  } else if (cmp_mag(a.mag_, b.mag_) >= 0) {
    r.mag_ = sub_mag(a.mag_, b.mag_);
    r.neg_ = a.neg_;
  } else {
    r.mag_ = sub_mag(b.mag_, a.mag_);
    r.neg_ = b.neg_;
  }
  r.trim();
  return r;
}

BigInt BigInt::operator-() const {
  BigInt r = *this;
  if (!r.mag_.empty()) r.neg_ = !r.neg_;
  return r;
}

BigInt operator-(const BigInt& a, const BigInt& b) { return a + (-b); }

BigInt operator*(const BigInt& a, const BigInt& b) {
  BigInt r;
  if (a.mag_.empty() || b.mag_.empty()) return r;
  r.mag_.assign(a.mag_.size() + b.mag_.size(), 0);
  for (size_t i = 0; i < a.mag_.size(); ++i) {
    uint64_t c = 0;
    for (size_t j = 0; j < b.mag_.size(); ++j) {
      uint64_t t = static_cast<uint64_t>(a.mag_[i]) * b.mag_[j] + r.mag_[i + j] + c;
      r.mag_[i + j] = static_cast<uint32_t>(t);
      c = t >> 32;
    }
    size_t k = i + b.mag_.size();
    while (c) {
      uint64_t t = static_cast<uint64_t>(r.mag_[k]) + c;
      r.mag_[k++] = static_cast<uint32_t>(t);
      c = t >> 32;
    }
  }
  r.neg_ = a.neg_ != b.neg_;
  r.trim();
  return r;
}

BigInt BigInt::shl(unsigned bits) const {
  if (mag_.empty()) return *this;
  BigInt r;
  r.neg_ = neg_;
  r.mag_.assign(bits / 32, 0);
  const unsigned s = bits % 32;
  uint32_t carry = 0;
  for (uint32_t limb : mag_) {
    r.mag_.push_back(s ? ((limb << s) | carry) : limb);
    carry = s ? (limb >> (32 - s)) : 0;
  }
  if (carry) r.mag_.push_back(carry);
  r.trim();
  return r;
}

void BigInt::divmod(const BigInt& a, const BigInt& b, BigInt& q, BigInt& r) {
  if (b.is_zero()) throw std::domain_error("BigInt division by zero");
  q = BigInt();
  r = BigInt();
  if (cmp_mag(a.mag_, b.mag_) < 0) {
    r = a;
    return;
  }
  if (b.mag_.size() == 1) {  // single-limb divisor
    const uint64_t d = b.mag_[0];
    q.mag_.assign(a.mag_.size(), 0);
    uint64_t rem = 0;
    for (size_t i = a.mag_.size(); i-- > 0;) {
      const uint64_t cur = (rem << 32) | a.mag_[i];
      q.mag_[i] = static_cast<uint32_t>(cur / d);
      rem = cur % d;
    }
    if (rem) r.mag_.push_back(static_cast<uint32_t>(rem));
  } else {  // restoring binary long division on magnitudes
    q.mag_.assign(a.mag_.size(), 0);
    for (size_t i = a.mag_.size(); i-- > 0;) {
      for (int bit = 31; bit >= 0; --bit) {
        uint32_t carry = (a.mag_[i] >> bit) & 1u;
        for (auto& limb : r.mag_) {
          const uint32_t nc = limb >> 31;
          limb = (limb << 1) | carry;
          carry = nc;
        }
        if (carry) r.mag_.push_back(carry);
        if (cmp_mag(r.mag_, b.mag_) >= 0) {
          r.mag_ = sub_mag(r.mag_, b.mag_);
          while (!r.mag_.empty() && r.mag_.back() == 0) r.mag_.pop_back();
          q.mag_[i] |= 1u << bit;
        }
      }
    }
  }
  q.neg_ = a.neg_ != b.neg_;
  r.neg_ = a.neg_;
  q.trim();
  r.trim();
}

BigInt operator/(const BigInt& a, const BigInt& b) {
  BigInt q, r;
  BigInt::divmod(a, b, q, r);
  return q;
}
BigInt operator%(const BigInt& a, const BigInt& b) {
  BigInt q, r;
  BigInt::divmod(a, b, q, r);
  return r;
}

int cmp(const BigInt& a, const BigInt& b) {
  const int sa = a.sign(), sb = b.sign();
  if (sa != sb) return sa < sb ? -1 : 1;
  const int c = cmp_mag(a.mag_, b.mag_);
  return sa < 0 ? -c : c;
}

BigInt BigInt::gcd(BigInt a, BigInt b) {
  if (a.negative()) a = -a;
  if (b.negative()) b = -b;
  while (!b.is_zero()) {
    BigInt t = a % b;
    a = std::move(b);
    b = std::move(t);
  }
  return a;
}

BigInt BigInt::pow10(unsigned n) {
  BigInt r(1);
  const BigInt ten(10);
  for (unsigned i = 0; i < n; ++i) r = r * ten;
  return r;
}

std::string BigInt::str() const {
  if (mag_.empty()) return "0";
  std::vector<uint32_t> m = mag_;
  std::string out;
  while (!m.empty()) {
    uint64_t rem = 0;
    for (size_t i = m.size(); i-- > 0;) {
      const uint64_t cur = (rem << 32) | m[i];
      m[i] = static_cast<uint32_t>(cur / 1000000000u);
      rem = cur % 1000000000u;
    }
    while (!m.empty() && m.back() == 0) m.pop_back();
    for (int k = 0; k < 9; ++k) {
      out.push_back(static_cast<char>('0' + rem % 10));
      rem /= 10;
      if (m.empty() && rem == 0) break;
    }
  }
  if (neg_) out.push_back('-');
  std::reverse(out.begin(), out.end());
  return out;
}

// ============================================================== Rat
namespace {
__int128 gcd128(__int128 a, __int128 b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b) {
    __int128 t = a % b;
    a = b;
    b = t;
  }
  return a;
}
constexpr long long kSafe = 1ll << 62;
inline bool safe(long long v) { return v > -kSafe && v < kSafe; }
}  // namespace

Rat Rat::make_small_or_big(__int128 n, __int128 d) {
  if (d < 0) {
    n = -n;
    d = -d;
  }
  if (n == 0) return Rat(0);
  const __int128 g = gcd128(n, d);
  if (g > 1) {
    n /= g;
    d /= g;
  }
  const __int128 lo = std::numeric_limits<long long>::min(), hi = std::numeric_limits<long long>::max();
  if (n >= lo && n <= hi && d <= hi) {
    Rat r;
    r.n_ = static_cast<long long>(n);
    r.d_ = static_cast<long long>(d);
    return r;
  }
  Rat r;
  r.big_ = std::make_shared<const Big>(Big{BigInt::from_i128(n), BigInt::from_i128(d)});
  return r;
}

Rat Rat::normalize_big(BigInt n, BigInt d) {
  if (d.is_zero()) throw std::domain_error("rational with zero denominator");
  if (d.negative()) {
    n = -n;
    d = -d;
  }
  if (n.is_zero()) return Rat(0);
  BigInt g = BigInt::gcd(n, d);
  if (g != BigInt(1)) {
    n = n / g;
    d = d / g;
  }
  if (n.fits_i64() && d.fits_i64()) {
    Rat r;
    r.n_ = n.to_i64();
    r.d_ = d.to_i64();
    return r;
  }
  Rat r;
  r.big_ = std::make_shared<const Big>(Big{std::move(n), std::move(d)});
  return r;
}

Rat Rat::frac(long long n, long long d) {
  if (d == 0) throw std::domain_error("rational with zero denominator");
  return make_small_or_big(n, d);
}

Rat Rat::from_big(BigInt n, BigInt d) { return normalize_big(std::move(n), std::move(d)); }

Rat Rat::from_double(double v) {
  if (!std::isfinite(v) || v == 0.0) return Rat(0);
  int e = 0;
  const double m = std::frexp(v, &e);
  const long long mant = static_cast<long long>(std::ldexp(m, 53));
  e -= 53;
  if (e >= 0) return normalize_big(BigInt(mant).shl(static_cast<unsigned>(e)), BigInt(1));
  if (-e <= 62) return make_small_or_big(mant, static_cast<__int128>(1) << (-e));
  return normalize_big(BigInt(mant), BigInt(1).shl(static_cast<unsigned>(-e)));
}

BigInt Rat::num() const { return big_ ? big_->n : BigInt(n_); }
BigInt Rat::den() const { return big_ ? big_->d : BigInt(d_); }
bool Rat::is_integer() const { return big_ ? big_->d == BigInt(1) : d_ == 1; }
int Rat::sign() const { return big_ ? big_->n.sign() : (n_ > 0) - (n_ < 0); }

double Rat::to_double() const {
  if (!big_ && n_ > -(1ll << 53) && n_ < (1ll << 53) && (d_ <= (1ll << 53) || (d_ & (d_ - 1)) == 0))
    return static_cast<double>(n_) / static_cast<double>(d_);
  BigInt n = num(), d = den();
  if (n.is_zero()) return 0.0;
  const bool neg = n.negative();
  if (neg) n = -n;
  const int shift = 65 - (static_cast<int>(n.bit_length()) - static_cast<int>(d.bit_length()));
  BigInt q = shift > 0 ? n.shl(static_cast<unsigned>(shift)) / d : n / d.shl(static_cast<unsigned>(-shift));
  const double r = std::ldexp(q.to_double(), -shift);
  return neg ? -r : r;
}

Rat operator+(const Rat& a, const Rat& b) {
  if (!a.big_ && !b.big_ && safe(a.n_) && safe(b.n_) && safe(a.d_) && safe(b.d_)) {
    if (a.d_ == b.d_) return Rat::make_small_or_big(static_cast<__int128>(a.n_) + b.n_, a.d_);
    return Rat::make_small_or_big(static_cast<__int128>(a.n_) * b.d_ + static_cast<__int128>(b.n_) * a.d_,
                                  static_cast<__int128>(a.d_) * b.d_);
  }
  return Rat::normalize_big(a.num() * b.den() + b.num() * a.den(), a.den() * b.den());
}

Rat Rat::operator-() const {
  if (!big_ && n_ != std::numeric_limits<long long>::min()) {
    Rat r = *this;
    r.n_ = -n_;
    return r;
  }
  return normalize_big(-num(), den());
}

Rat operator-(const Rat& a, const Rat& b) { return a + (-b); }

Rat operator*(const Rat& a, const Rat& b) {
  if (!a.big_ && !b.big_ && safe(a.n_) && safe(b.n_) && safe(a.d_) && safe(b.d_))
    return Rat::make_small_or_big(static_cast<__int128>(a.n_) * b.n_, static_cast<__int128>(a.d_) * b.d_);
  return Rat::normalize_big(a.num() * b.num(), a.den() * b.den());
}

Rat operator/(const Rat& a, const Rat& b) {
  if (b.sign() == 0) throw std::domain_error("rational division by zero");
  if (!a.big_ && !b.big_ && safe(a.n_) && safe(b.n_) && safe(a.d_) && safe(b.d_))
    return Rat::make_small_or_big(static_cast<__int128>(a.n_) * b.d_, static_cast<__int128>(a.d_) * b.n_);
  return Rat::normalize_big(a.num() * b.den(), a.den() * b.num());
}

int cmp(const Rat& a, const Rat& b) {
  if (!a.big_ && !b.big_) {
    if (a.d_ == b.d_) return (a.n_ > b.n_) - (a.n_ < b.n_);
    const __int128 l = static_cast<__int128>(a.n_) * b.d_, r = static_cast<__int128>(b.n_) * a.d_;
    return (l > r) - (l < r);
  }
  return cmp(a.num() * b.den(), b.num() * a.den());
}

bool operator==(const Rat& a, const Rat& b) {
  if (!a.big_ && !b.big_) return a.n_ == b.n_ && a.d_ == b.d_;
  return cmp(a, b) == 0;
}

// ============================================================== text
namespace {
std::optional<Rat> parse_decimal(std::string_view s) {
  size_t i = 0;
  bool neg = false;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  BigInt mant(0);
  const BigInt ten(10);
  int frac_digits = 0;
  bool any = false;
  auto digit = [&](char c) { mant = mant * ten + BigInt(c - '0'); };
  for (; i < s.size() && std::isdigit(static_cast<unsigned char>(s[i])); ++i, any = true) digit(s[i]);
  if (i < s.size() && s[i] == '.') {
    ++i;
    for (; i < s.size() && std::isdigit(static_cast<unsigned char>(s[i])); ++i, any = true, ++frac_digits)
      digit(s[i]);
  }
  if (!any) return std::nullopt;
  long exp10 = 0;
  if (i < s.size() && (s[i] == 'e' || s[i] == 'E')) {
    ++i;
    bool eneg = false;
    if (i < s.size() && (s[i] == '+' || s[i] == '-')) eneg = s[i++] == '-';
    if (i >= s.size()) return std::nullopt;
    long e = 0;
    for (; i < s.size() && std::isdigit(static_cast<unsigned char>(s[i])); ++i) {
      e = e * 10 + (s[i] - '0');
      if (e > 100000) return std::nullopt;
    }
    exp10 = eneg ? -e : e;
  }
  if (i != s.size()) return std::nullopt;
  const long net = exp10 - frac_digits;
  BigInt n = mant, d(1);
  if (net > 0) n = n * BigInt::pow10(static_cast<unsigned>(net));
  if (net < 0) d = BigInt::pow10(static_cast<unsigned>(-net));
  if (neg) n = -n;
  return Rat::from_big(n, d);
}
}  // namespace

std::optional<Rat> parse_rat(std::string_view text) {
  const size_t slash = text.find('/');
  if (slash != std::string_view::npos) {
    auto n = parse_decimal(text.substr(0, slash));
    auto d = parse_decimal(text.substr(slash + 1));
    if (!n || !d || d->sign() == 0) return std::nullopt;
    if (!n->is_integer() || !d->is_integer()) return std::nullopt;
    return *n / *d;
  }
  return parse_decimal(text);
}

std::string to_canonical(const Rat& r) {
  BigInt n = r.num(), d = r.den();
  if (d == BigInt(1)) return n.str();
  unsigned a = 0, b = 0;
  BigInt rest = d;
  const BigInt two(2), five(5);
  while ((rest % two).is_zero()) {
    rest = rest / two;
    ++a;
  }
  while ((rest % five).is_zero()) {
    rest = rest / five;
    ++b;
  }
  if (rest != BigInt(1)) return n.str() + "/" + d.str();
  const unsigned digits = std::max(a, b);
  BigInt scaled = n * BigInt::pow10(digits) / d;
  const bool neg = scaled.negative();
  if (neg) scaled = -scaled;
  std::string s = scaled.str();
  if (s.size() <= digits) s.insert(0, digits + 1 - s.size(), '0');
  s.insert(s.size() - digits, ".");
  return (neg ? "-" : "") + s;
}

std::string to_fixed(const Rat& r, int digits) {
  BigInt n = r.num() * BigInt::pow10(static_cast<unsigned>(digits)) * BigInt(2);
  const bool neg = n.negative();
  if (neg) n = -n;
  BigInt scaled = (n / r.den() + BigInt(1)) / BigInt(2);
  std::string s = scaled.str();
  if (digits > 0) {
    if (s.size() <= static_cast<size_t>(digits)) s.insert(0, static_cast<size_t>(digits) + 1 - s.size(), '0');
    s.insert(s.size() - static_cast<size_t>(digits), ".");
  }
  return (neg && !scaled.is_zero() ? "-" : "") + s;
}

BigInt ceil_nonneg(const Rat& r) {
  const BigInt n = r.num(), d = r.den();
  return (n + d - BigInt(1)) / d;
}

}  // namespace lynx::host
