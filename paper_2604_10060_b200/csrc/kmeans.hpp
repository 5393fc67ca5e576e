// kmeans.hpp -- host slow path of cluster maintenance: the exact (bit-reproducible)
// arithmetic the split / settle / batch-build paths share with the reference.
//
// Follows, operation for operation (fp64, sequential sums, no FMA contraction -- the library
// is built with -ffp-contract=off like the reference, CMakeLists.txt:11-13):
//   vecmath.hpp:27-99  dot / norm / sq_dist / cosine / dnormalize / dmean
//   rng.hpp:14-52      Rng (std::mt19937_64 + 53-bit uniform + modulo index), mix_seed
//   clustering.cpp     spherical_kmeans (80-178), split_two (180-208)
//   index.cpp:345-362  compute_representative / compute_variance
// Data is flat row-major: n rows of d floats.
#pragma once

#include <cstdint>
#include <random>
#include <vector>

namespace kvc {

inline constexpr double kDegenerate = 1e-12;  // vecmath.hpp:19

class Rng64 {  // rng.hpp:14-44 semantics
 public:
  explicit Rng64(std::uint64_t seed) : eng_(seed) {}
  std::uint64_t u64() { return eng_(); }
  double uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  std::size_t index(std::size_t n) { return static_cast<std::size_t>(eng_() % n); }

 private:
  std::mt19937_64 eng_;
};

std::uint64_t mix_seed(std::uint64_t a, std::uint64_t b);  // rng.hpp:47-52

// The first two outputs of std::mt19937_64(seed) without building the whole 312-word state: the
// first twist step of words 0 and 1 reads only words 0..2 and 156..157 of the seeded state. A
// split's k-means++ makes exactly two draws (the first centre's index, then the uniform), so the
// wave engine derives them from this (equal to Rng64's by construction; checked against
// std::mt19937_64 in tests/test_host_abi.py through kvc_host_rng_first2).
void mt64_first2(std::uint64_t seed, std::uint64_t out[2]);

// fp64 sequential kernels (vecmath.hpp:27-51)
double dot_fd(const float* a, const double* b, int d);
double dot_dd(const double* a, const double* b, int d);
double norm_f(const float* a, int d);
double norm_d(const double* a, int d);
// cosine_sim (vecmath.hpp:54-61); throws Error(KVC_E_DEGENERATE) on a zero vector
double cosine_fd(const float* a, const double* b, int d);

struct KMeansOut {
  std::vector<int> assign;  // dense cluster index per point
  int k_live = 0;
  double objective = 0.0;
  int iterations = 0;
  bool degenerate = false;
  // (device batch build only) Eq. 1 representative [k_live][d] and Eq. 2 variance [k_live] of
  // each output cluster, computed exactly as representative() / variance() below
  std::vector<double> reps, vars;
};

KMeansOut spherical_kmeans(const float* pts, int n, int d, int k, int max_iters, double tol,
                           std::uint64_t seed);
KMeansOut split_two(const float* pts, int n, int d, std::uint64_t seed);

// Eq. 1/2 exact statistics over selected rows (rows[i] indexes `pts`).
void representative(const float* pts, const int* rows, int n, int d, double* rep);
double variance(const float* pts, const int* rows, int n, int d, const double* rep);

}  // namespace kvc
