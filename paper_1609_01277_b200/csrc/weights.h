// Central-difference weights of the CUDA path, in closed form (the test
// reference solves the moment conditions instead).  Internal header.
#pragma once
#include <vector>

namespace osbli {

struct Frac64 {
  long long n, d;
};

inline long long gcdll(long long a, long long b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b) {
    long long t = a % b;
    a = b;
    b = t;
  }
  return a;
}

inline long long fact(int n) {
  long long r = 1;
  for (int i = 2; i <= n; ++i) r *= i;
  return r;
}

// Explicit Lagrange-derivative formula, exact in int64 for m <= 6:
//   a_k = (-1)^(k+1) (m!)^2 / (k (m-k)! (m+k)!)
//   b_k = 2 (-1)^(k+1) (m!)^2 / (k^2 (m-k)! (m+k)!),  b_0 = -2 sum_k b_k
inline void central_weights(int m, double *a, double *b) {
  const long long mf2 = fact(m) * fact(m);
  std::vector<Frac64> bk;
  for (int k = 1; k <= m; ++k) {
    const long long sgn = (k % 2 == 1) ? 1 : -1;
    long long n = sgn * mf2, d = (long long)k * fact(m - k) * fact(m + k);
    long long g = gcdll(n, d);
    a[k - 1] = (double)(n / g) / (double)(d / g);
    long long n2 = 2 * sgn * mf2, d2 = (long long)k * k * fact(m - k) * fact(m + k);
    g = gcdll(n2, d2);
    bk.push_back({n2 / g, d2 / g});
    b[k] = (double)(n2 / g) / (double)(d2 / g);
  }
  long long N = 0, D = 1;
  for (auto &f : bk) {
    const long long g = gcdll(D, f.d);
    const long long L = D / g * f.d;
    N = N * (L / D) + f.n * (L / f.d);
    D = L;
    const long long h = gcdll(N, D);
    if (h > 1) {
      N /= h;
      D /= h;
    }
  }
  b[0] = -2.0 * (double)N / (double)D;
}

}  // namespace osbli
