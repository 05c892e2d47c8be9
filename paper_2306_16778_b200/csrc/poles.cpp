// Pole/residue tables of R_n(z) = 1/exp_n(-z) on the host.
//
// Same numbers as reference roots.default_table(n) (roots.py:143-226,315-318):
//   * theta_k: the n roots of exp_n(z) = sum_{j<=n} z^j/j!, refined to
//     double-double accuracy, conjugate pairs stored as one Im>0 representative,
//     representatives sorted by (Re, Im) ascending (roots.py:148-170);
//   * a_k = -n! / prod_{j != k} (theta_k - theta_j) in double-double
//     (product formula, roots.py:182-209);
//   * binary64 values = the leading limb of the double-double
//     (DoubleDoubleComplex.to_complex, ddreal.py:196-197).
// The pipeline differs from the reference only in how it obtains starting
// points (Aberth iteration here instead of LAPACK companion eigenvalues): both
// converge to the same double-double roots, whose leading limbs are
// then identical (checked for every even n in [2, 64] against the
// reference-generated golden tables, tests/test_poles.py).
#include <algorithm>
#include <cmath>
#include <complex>
#include <string>
#include <vector>

#include "../../include/pfx.h"

namespace pfx {

int fail(int status, const std::string& msg);

namespace {

struct dd {
  double hi, lo;
};

inline dd two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  double err = (a - (s - bb)) + (b - bb);
  return {s, err};
}
inline dd quick_two_sum(double a, double b) {
  double s = a + b;
  return {s, b - (s - a)};
}
inline dd two_prod(double a, double b) {
  double p = a * b;
  return {p, std::fma(a, b, -p)};
}
inline dd dd_from(double a) { return {a, 0.0}; }
inline dd operator+(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
inline dd operator-(dd a) { return {-a.hi, -a.lo}; }
inline dd operator-(dd a, dd b) { return a + (-b); }
inline dd operator*(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}
inline dd operator*(dd a, double b) { return a * dd_from(b); }
inline dd operator/(dd a, dd b) {
  double q1 = a.hi / b.hi;
  dd r = a - b * q1;
  double q2 = r.hi / b.hi;
  r = r - b * q2;
  double q3 = r.hi / b.hi;
  dd q = quick_two_sum(q1, q2);
  return q + dd_from(q3);
}

struct ddc {
  dd re, im;
};
inline ddc operator+(ddc a, ddc b) { return {a.re + b.re, a.im + b.im}; }
inline ddc operator-(ddc a, ddc b) { return {a.re - b.re, a.im - b.im}; }
inline ddc operator*(ddc a, ddc b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
inline ddc operator/(ddc a, ddc b) {
  dd den = b.re * b.re + b.im * b.im;
  ddc num = a * ddc{b.re, -b.im};
  return {num.re / den, num.im / den};
}
inline double abs2hi(ddc a) { return (a.re * a.re + a.im * a.im).hi; }

// 1/k! in double-double, k = 0..n
std::vector<dd> inv_fact(int n) {
  std::vector<dd> v(n + 1);
  v[0] = dd_from(1.0);
  for (int k = 1; k <= n; ++k) v[k] = v[k - 1] / dd_from((double)k);
  return v;
}

ddc eval_trunc(const std::vector<dd>& inv, int n, ddc z) {
  ddc p{inv[n], dd_from(0.0)};
  for (int k = n - 1; k >= 0; --k) p = p * z + ddc{inv[k], dd_from(0.0)};
  return p;
}

using cd = std::complex<double>;

// All n roots of exp_n in binary64 by Aberth-Ehrlich iteration.
std::vector<cd> aberth_roots(int n) {
  std::vector<double> c(n + 1);  // c[k] = 1/k!
  c[0] = 1.0;
  for (int k = 1; k <= n; ++k) c[k] = c[k - 1] / k;
  std::vector<cd> z(n);
  const double R = 0.7 * n + 1.0;
  for (int k = 0; k < n; ++k) z[k] = std::polar(R, 2.0 * M_PI * (k + 0.25) / n);
  for (int it = 0; it < 500; ++it) {
    double maxstep = 0.0;
    for (int k = 0; k < n; ++k) {
      cd p = c[n], dp = 0.0;
      for (int j = n - 1; j >= 0; --j) {
        dp = dp * z[k] + p;
        p = p * z[k] + c[j];
      }
      cd ratio = p / dp;
      cd s = 0.0;
      for (int j = 0; j < n; ++j)
        if (j != k) s += 1.0 / (z[k] - z[j]);
      cd step = ratio / (1.0 - ratio * s);
      z[k] -= step;
      maxstep = std::max(maxstep, std::abs(step) / std::max(1.0, std::abs(z[k])));
    }
    if (maxstep < 1e-15) break;
  }
  // binary64 Newton polish
  for (int it = 0; it < 4; ++it)
    for (int k = 0; k < n; ++k) {
      cd p = c[n], dp = 0.0;
      for (int j = n - 1; j >= 0; --j) {
        dp = dp * z[k] + p;
        p = p * z[k] + c[j];
      }
      if (dp != 0.0) z[k] -= p / dp;
    }
  return z;
}

// Newton in double-double: exp_n' = exp_{n-1}; keeps the iterate of smallest residual.
ddc refine_dd(const std::vector<dd>& inv, int n, cd z0) {
  ddc z{dd_from(z0.real()), dd_from(z0.imag())};
  ddc best = z;
  double best_res = INFINITY;
  for (int it = 0; it < 8; ++it) {
    ddc p = eval_trunc(inv, n, z);
    ddc dp = eval_trunc(inv, n - 1, z);
    double res = abs2hi(p);
    if (res < best_res) {
      best = z;
      best_res = res;
    }
    if (abs2hi(dp) == 0.0) break;
    z = z - p / dp;
  }
  ddc p = eval_trunc(inv, n, z);
  if (abs2hi(p) < best_res) best = z;
  return best;
}

}  // namespace

int pole_table_host(int n, double* theta2, double* coef2) {
  const std::vector<dd> inv = inv_fact(n);
  std::vector<cd> guess = aberth_roots(n);
  std::vector<ddc> reps;
  for (const cd& g : guess) {
    if (g.imag() > 0.0) reps.push_back(refine_dd(inv, n, g));
  }
  if ((int)reps.size() != n / 2) return fail(PFX_CUDA, "pole refinement lost the conjugate split");
  std::sort(reps.begin(), reps.end(), [](const ddc& a, const ddc& b) {
    if (a.re.hi != b.re.hi) return a.re.hi < b.re.hi;
    return a.im.hi < b.im.hi;
  });
  std::vector<ddc> all;
  for (const ddc& r : reps) {
    all.push_back(r);
    all.push_back(ddc{r.re, -r.im});
  }
  dd fact = dd_from(1.0);
  for (int k = 2; k <= n; ++k) fact = fact * dd_from((double)k);
  for (int k = 0; k < n / 2; ++k) {
    const ddc& rep = all[2 * k];
    ddc prod{dd_from(1.0), dd_from(0.0)};
    for (int j = 0; j < n; ++j)
      if (j != 2 * k) prod = prod * (rep - all[j]);
    ddc a = ddc{fact, dd_from(0.0)} / prod;
    a = ddc{-a.re, -a.im};
    theta2[2 * k] = rep.re.hi;
    theta2[2 * k + 1] = rep.im.hi;
    coef2[2 * k] = a.re.hi;
    coef2[2 * k + 1] = a.im.hi;
  }
  return PFX_OK;
}

}  // namespace pfx
