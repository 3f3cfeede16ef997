// TEST INFRASTRUCTURE ONLY — minimal stand-in for boost::rational, which the
// reference's store.hpp includes (store.hpp:4, 17) for its analytical
// memory_model.  Boost is not vendored with the reference and not installed
// in this image; nothing on the SAMO hot path uses it.  Normalised
// numerator/denominator with a positive denominator, as boost's contract.
#pragma once

#include <numeric>
#include <stdexcept>

namespace boost {

template <typename I>
class rational {
 public:
  rational() : n_(0), d_(1) {}
  rational(I n) : n_(n), d_(1) {}  // NOLINT: implicit like boost
  rational(I n, I d) : n_(n), d_(d) { norm(); }

  I numerator() const { return n_; }
  I denominator() const { return d_; }

  friend rational operator+(const rational& a, const rational& b) {
    return rational(a.n_ * b.d_ + b.n_ * a.d_, a.d_ * b.d_);
  }
  friend rational operator-(const rational& a, const rational& b) {
    return rational(a.n_ * b.d_ - b.n_ * a.d_, a.d_ * b.d_);
  }
  friend rational operator*(const rational& a, const rational& b) {
    return rational(a.n_ * b.n_, a.d_ * b.d_);
  }
  friend rational operator/(const rational& a, const rational& b) {
    return rational(a.n_ * b.d_, a.d_ * b.n_);
  }
  friend rational operator*(const rational& a, I b) { return a * rational(b); }
  friend rational operator*(I a, const rational& b) { return rational(a) * b; }
  friend bool operator==(const rational& a, const rational& b) {
    return a.n_ == b.n_ && a.d_ == b.d_;
  }
  friend bool operator!=(const rational& a, const rational& b) { return !(a == b); }
  friend bool operator<(const rational& a, const rational& b) {
    return a.n_ * b.d_ < b.n_ * a.d_;
  }
  friend bool operator>(const rational& a, const rational& b) { return b < a; }
  friend bool operator<=(const rational& a, const rational& b) { return !(b < a); }
  friend bool operator>=(const rational& a, const rational& b) { return !(a < b); }

 private:
  void norm() {
    if (d_ == 0) throw std::domain_error("zero denominator");
    if (d_ < 0) { n_ = -n_; d_ = -d_; }
    const I g = std::gcd(n_ < 0 ? -n_ : n_, d_);
    if (g > 1) { n_ /= g; d_ /= g; }
  }
  I n_, d_;
};

}  // namespace boost
