// kmeans.cpp -- exact host slow path (see kmeans.hpp for the reference lines followed).
#include "kmeans.hpp"

#include <algorithm>
#include <cmath>
#include <limits>

#include "kvc_core.hpp"

namespace kvc {

void mt64_first2(std::uint64_t seed, std::uint64_t out[2]) {
  constexpr std::uint64_t kF = 6364136223846793005ULL, kA = 0xB5026F5AA96619E9ULL;
  constexpr std::uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;
  std::uint64_t x[158];
  x[0] = seed;
  for (std::uint64_t i = 1; i < 158; ++i) x[i] = kF * (x[i - 1] ^ (x[i - 1] >> 62)) + i;
  for (int i = 0; i < 2; ++i) {
    const std::uint64_t y = (x[i] & kUpper) | (x[i + 1] & kLower);
    std::uint64_t z = x[i + 156] ^ (y >> 1) ^ ((y & 1ULL) ? kA : 0ULL);
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    out[i] = z;
  }
}

std::uint64_t mix_seed(std::uint64_t a, std::uint64_t b) {
  std::uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

double dot_fd(const float* a, const double* b, int d) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) s += static_cast<double>(a[i]) * b[i];
  return s;
}
double dot_dd(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) s += a[i] * b[i];
  return s;
}
double norm_f(const float* a, int d) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) s += static_cast<double>(a[i]) * static_cast<double>(a[i]);
  return std::sqrt(s);
}
double norm_d(const double* a, int d) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) s += a[i] * a[i];
  return std::sqrt(s);
}
double cosine_fd(const float* a, const double* b, int d) {
  const double na = norm_f(a, d), nb = norm_d(b, d);
  if (na < kDegenerate || nb < kDegenerate) fail(-2, "cosine of zero vector");
  return std::clamp(dot_fd(a, b, d) / (na * nb), -1.0, 1.0);
}

namespace {

// Unit-sphere copies of the points (clustering.cpp:14-22): row / norm(row), fp64.
std::vector<double> unit_rows(const float* pts, int n, int d) {
  std::vector<double> u(static_cast<std::size_t>(n) * d);
  for (int i = 0; i < n; ++i) {
    double* r = &u[static_cast<std::size_t>(i) * d];
    const float* p = pts + static_cast<std::size_t>(i) * d;
    for (int c = 0; c < d; ++c) r[c] = static_cast<double>(p[c]);
    const double nr = norm_d(r, d);
    if (nr < kDegenerate) fail(-2, "normalize of zero vector");
    for (int c = 0; c < d; ++c) r[c] = r[c] / nr;
  }
  return u;
}

// Cosine of a unit point to an unnormalised centroid; -2 for a degenerate centroid
// (clustering.cpp:72-76).
inline double unit_cos(const double* p, const double* c, int d) {
  const double nc = norm_d(c, d);
  if (nc < kDegenerate) return -2.0;
  return std::clamp(dot_dd(p, c, d) / nc, -1.0, 1.0);
}

// k-means++-style seeding with 1 - cosine weights (clustering.cpp:25-70).
std::vector<int> plus_plus(const std::vector<double>& u, int n, int d, int k, Rng64& rng) {
  std::vector<int> picks;
  std::vector<char> taken(static_cast<std::size_t>(n), 0);
  std::vector<double> near(static_cast<std::size_t>(n));
  const int first = static_cast<int>(rng.index(static_cast<std::size_t>(n)));
  picks.push_back(first);
  taken[first] = 1;
  for (int i = 0; i < n; ++i) near[i] = dot_dd(&u[static_cast<std::size_t>(i) * d], &u[static_cast<std::size_t>(first) * d], d);
  while (static_cast<int>(picks.size()) < k) {
    double mass = 0.0;
    for (int i = 0; i < n; ++i)
      if (!taken[i]) mass += std::max(0.0, 1.0 - near[i]);
    int pick = n;
    if (mass > 1e-15) {
      const double target = rng.uniform() * mass;
      double run = 0.0;
      for (int i = 0; i < n; ++i) {
        if (taken[i]) continue;
        run += std::max(0.0, 1.0 - near[i]);
        if (run >= target) {
          pick = i;
          break;
        }
      }
    }
    if (pick == n)
      for (int i = 0; i < n; ++i)
        if (!taken[i]) {
          pick = i;
          break;
        }
    picks.push_back(pick);
    taken[pick] = 1;
    const double* pp = &u[static_cast<std::size_t>(pick) * d];
    for (int i = 0; i < n; ++i) near[i] = std::max(near[i], dot_dd(&u[static_cast<std::size_t>(i) * d], pp, d));
  }
  return picks;
}

}  // namespace

KMeansOut spherical_kmeans(const float* pts, int n, int d, int k_req, int max_iters, double tol,
                           std::uint64_t seed) {
  if (n <= 0) fail(-4, "spherical_kmeans: no points");
  const int k = std::max(1, std::min(k_req, n));
  const std::vector<double> u = unit_rows(pts, n, d);
  Rng64 rng(seed);
  std::vector<double> cent(static_cast<std::size_t>(k) * d);
  {
    std::vector<int> seeds = plus_plus(u, n, d, k, rng);
    for (int j = 0; j < k; ++j)
      std::copy_n(&u[static_cast<std::size_t>(seeds[j]) * d], d, &cent[static_cast<std::size_t>(j) * d]);
  }
  auto row = [&](int i) { return &u[static_cast<std::size_t>(i) * d]; };
  auto ctr = [&](int j) { return &cent[static_cast<std::size_t>(j) * d]; };

  KMeansOut out;
  out.assign.assign(static_cast<std::size_t>(n), 0);
  std::vector<int>& a = out.assign;
  std::vector<std::int64_t> cnt(static_cast<std::size_t>(k));
  std::vector<double> acc(static_cast<std::size_t>(k) * d);
  double prev = -std::numeric_limits<double>::infinity();

  for (int it = 0; it < max_iters; ++it) {
    bool moved = false;
    for (int i = 0; i < n; ++i) {  // assignment, ties to the lowest index (99-112)
      int bj = 0;
      double bs = unit_cos(row(i), ctr(0), d);
      for (int j = 1; j < k; ++j) {
        const double s = unit_cos(row(i), ctr(j), d);
        if (s > bs) {
          bs = s;
          bj = j;
        }
      }
      if (a[i] != bj) moved = true;
      a[i] = bj;
    }
    std::fill(cnt.begin(), cnt.end(), 0);
    for (int i = 0; i < n; ++i) ++cnt[a[i]];
    for (int j = 0; j < k; ++j) {  // empty-cluster reseed (117-136)
      if (cnt[j] != 0) continue;
      int far = n;
      double far_s = std::numeric_limits<double>::infinity();
      for (int i = 0; i < n; ++i) {
        if (cnt[a[i]] <= 1) continue;
        const double s = unit_cos(row(i), ctr(a[i]), d);
        if (s < far_s) {
          far_s = s;
          far = i;
        }
      }
      if (far == n) continue;
      --cnt[a[far]];
      a[far] = j;
      ++cnt[j];
      moved = true;
    }
    std::fill(acc.begin(), acc.end(), 0.0);  // arithmetic means (138-150)
    for (int i = 0; i < n; ++i) {
      double* s = &acc[static_cast<std::size_t>(a[i]) * d];
      const double* p = row(i);
      for (int c = 0; c < d; ++c) s[c] += p[c];
    }
    for (int j = 0; j < k; ++j) {
      if (cnt[j] == 0) continue;
      const double inv = 1.0 / static_cast<double>(cnt[j]);
      double* s = &acc[static_cast<std::size_t>(j) * d];
      double* cj = ctr(j);
      for (int c = 0; c < d; ++c) cj[c] = s[c] * inv;
    }
    double obj = 0.0;  // mean cosine, convergence (152-163)
    for (int i = 0; i < n; ++i) obj += unit_cos(row(i), ctr(a[i]), d);
    obj /= static_cast<double>(n);
    out.iterations = it + 1;
    out.objective = obj;
    if (it > 0 && obj - prev < tol) break;
    prev = obj;
    if (!moved) break;
  }
  // compact ids (166-177)
  std::vector<int> remap(static_cast<std::size_t>(k), -1);
  std::fill(cnt.begin(), cnt.end(), 0);
  for (int v : a) ++cnt[v];
  int live = 0;
  for (int j = 0; j < k; ++j)
    if (cnt[j] != 0) remap[j] = live++;
  for (int& v : a) v = remap[v];
  out.k_live = live;
  return out;
}

KMeansOut split_two(const float* pts, int n, int d, std::uint64_t seed) {
  if (n < 2) fail(-6, "split_two: need at least 2 points");
  const std::vector<double> u = unit_rows(pts, n, d);
  bool same = true;
  for (int i = 1; i < n && same; ++i)
    if (dot_dd(&u[static_cast<std::size_t>(i) * d], &u[0], d) < 1.0 - 1e-12) same = false;
  if (same) {  // deterministic (n-1, 1) partition (clustering.cpp:190-200)
    KMeansOut o;
    o.degenerate = true;
    o.assign.assign(static_cast<std::size_t>(n), 0);
    o.assign[static_cast<std::size_t>(n - 1)] = 1;
    o.k_live = 2;
    o.objective = 1.0;
    return o;
  }
  return spherical_kmeans(pts, n, d, 2, 50, 1e-9, seed);
}

void representative(const float* pts, const int* rows, int n, int d, double* rep) {
  if (n <= 0) fail(-5, "cluster with no members");
  for (int c = 0; c < d; ++c) rep[c] = 0.0;
  for (int i = 0; i < n; ++i) {
    const float* p = pts + static_cast<std::size_t>(rows[i]) * d;
    for (int c = 0; c < d; ++c) rep[c] += p[c];
  }
  const double inv = 1.0 / static_cast<double>(n);
  for (int c = 0; c < d; ++c) rep[c] *= inv;
}

double variance(const float* pts, const int* rows, int n, int d, const double* rep) {
  if (n <= 0) fail(-5, "cluster with no members");
  double total = 0.0;
  for (int i = 0; i < n; ++i) {
    const float* p = pts + static_cast<std::size_t>(rows[i]) * d;
    double s = 0.0;
    for (int c = 0; c < d; ++c) {
      const double diff = static_cast<double>(p[c]) - rep[c];
      s += diff * diff;
    }
    total += s;
  }
  return total / static_cast<double>(n);
}

}  // namespace kvc
