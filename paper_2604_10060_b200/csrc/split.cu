// split.cu -- split_two (clustering.cpp:180-208) on the GPU: 2-way spherical k-means of a
// cluster's members, bit-identical to the host restatement (kmeans.cpp), which follows the
// reference operation for operation.
//
// One CTA per split. Every fp64 quantity is formed with round-to-nearest intrinsics in the
// reference's order: per-point sums (norms, dots) run sequentially over the dimension in one
// thread; sums over points (k-means++ mass, centroid accumulators, the objective) run
// sequentially over the point index in one thread per output value. The two random draws of the
// seeding (mt19937_64: the first centre's index, then the uniform) are made on the host, which
// owns the generator (rng.hpp:14-44), and passed in.
#include "devmath.cuh"

namespace kvc {

namespace {

using namespace dm;

constexpr int SPT = 512;

__device__ __forceinline__ double dot_seq(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int c = 0; c < d; ++c) s = dadd(s, dmul(a[c], b[c]));
  return s;
}

__device__ __forceinline__ double unit_cos(const double* p, const double* c, double nc, int d) {
  if (nc < 1e-12) return -2.0;  // degenerate centroid (clustering.cpp:72-76)
  return clamp1(ddiv(dot_seq(p, c, d), nc));
}

struct SplitSmem {
  double cent[2][256];
  double cn[2];
  double prev;
  int cnt[2];
  int moved, same, pick, stop, degen, far_i;
  double far_s;
};

// rows: staged f32 rows; idx[n]: the points of this split (rows idx[i]); u: scratch [n][d].
// out: assign[n]; meta[4] = {k_live, iterations, degenerate, error}; obj[1].
__global__ void __launch_bounds__(SPT) k_split_two(const float* rows, const int32_t* idx, int n, int d, int first,
                                                    double uni, double* u, int32_t* assign, int32_t* meta,
                                                    double* objective) {
  __shared__ SplitSmem S;
  const int tid = threadIdx.x;
  if (tid == 0) {
    S.same = 1;
    S.degen = 0;
  }
  __syncthreads();
  // unit rows (clustering.cpp:14-22): r / norm(r)
  for (int i = tid; i < n; i += SPT) {
    const float* p = rows + static_cast<int64_t>(idx[i]) * d;
    double* r = u + static_cast<int64_t>(i) * d;
    double s = 0.0;
    for (int c = 0; c < d; ++c) {
      const double x = static_cast<double>(p[c]);
      s = dadd(s, dmul(x, x));
    }
    const double nr = __dsqrt_rn(s);
    if (nr < 1e-12) S.degen = 1;
    for (int c = 0; c < d; ++c) r[c] = ddiv(static_cast<double>(p[c]), nr);
  }
  __syncthreads();
  if (S.degen) {
    if (tid == 0) meta[3] = -2;  // zero vector (the host raises KVC_E_DEGENERATE)
    return;
  }
  // all points equal (within 1e-12 of the first): the deterministic (n-1, 1) partition
  for (int i = 1 + tid; i < n; i += SPT)
    if (dot_seq(u + static_cast<int64_t>(i) * d, u, d) < 1.0 - 1e-12) S.same = 0;
  __syncthreads();
  if (S.same) {
    for (int i = tid; i < n; i += SPT) assign[i] = i == n - 1 ? 1 : 0;
    if (tid == 0) {
      meta[0] = 2;
      meta[1] = 0;
      meta[2] = 1;
      meta[3] = 0;
      *objective = 1.0;
    }
    return;
  }
  // k-means++ seeding with 1 - cosine weights, k = 2 (clustering.cpp:25-70). near[] -> assign
  // (as doubles in u's tail would cost memory; the weights are recomputed by the sequential pass)
  double* nearv = u + static_cast<int64_t>(n) * d;  // [n] (scratch sized n * (d + 1))
  for (int i = tid; i < n; i += SPT) nearv[i] = dot_seq(u + static_cast<int64_t>(i) * d, u + static_cast<int64_t>(first) * d, d);
  __syncthreads();
  if (tid == 0) {
    double mass = 0.0;
    for (int i = 0; i < n; ++i)
      if (i != first) mass = dadd(mass, fmax(0.0, dsub(1.0, nearv[i])));
    int pick = n;
    if (mass > 1e-15) {
      const double target = dmul(uni, mass);
      double run = 0.0;
      for (int i = 0; i < n; ++i) {
        if (i == first) continue;
        run = dadd(run, fmax(0.0, dsub(1.0, nearv[i])));
        if (run >= target) {
          pick = i;
          break;
        }
      }
    }
    if (pick == n) pick = first == 0 ? 1 : 0;
    S.pick = pick;
    S.prev = -INFINITY;
    S.stop = 0;
  }
  __syncthreads();
  for (int c = tid; c < d; c += SPT) {
    S.cent[0][c] = u[static_cast<int64_t>(first) * d + c];
    S.cent[1][c] = u[static_cast<int64_t>(S.pick) * d + c];
  }
  for (int i = tid; i < n; i += SPT) assign[i] = 0;
  __syncthreads();
  for (int it = 0; it < 50; ++it) {
    // centroid norms (unit_cos recomputes them per call: the same value each time)
    if (tid < 2) {
      double s = 0.0;
      for (int c = 0; c < d; ++c) s = dadd(s, dmul(S.cent[tid][c], S.cent[tid][c]));
      S.cn[tid] = __dsqrt_rn(s);
    }
    if (tid == 0) {
      S.moved = 0;
      S.cnt[0] = 0;
      S.cnt[1] = 0;
    }
    __syncthreads();
    // assignment, ties to the lower index (clustering.cpp:99-112)
    int c0 = 0, c1 = 0, mv = 0;
    for (int i = tid; i < n; i += SPT) {
      const double* p = u + static_cast<int64_t>(i) * d;
      const double s0 = unit_cos(p, S.cent[0], S.cn[0], d);
      const double s1 = unit_cos(p, S.cent[1], S.cn[1], d);
      const int bj = s1 > s0 ? 1 : 0;
      if (assign[i] != bj) mv = 1;
      assign[i] = bj;
      c0 += bj == 0;
      c1 += bj == 1;
    }
    if (mv) S.moved = 1;
    atomicAdd(&S.cnt[0], c0);
    atomicAdd(&S.cnt[1], c1);
    __syncthreads();
    // empty-cluster reseed (clustering.cpp:117-136): the point farthest from its centroid among
    // clusters with more than one point (first minimum in index order)
    for (int j = 0; j < 2; ++j) {
      if (S.cnt[j] != 0) continue;  // block-uniform
      if (tid == 0) {
        S.far_i = n;
        S.far_s = INFINITY;
      }
      __syncthreads();
      if (tid == 0) {  // sequential scan: the strict < keeps the first minimum
        for (int i = 0; i < n; ++i) {
          const int ai = assign[i];
          if (S.cnt[ai] <= 1) continue;
          const double s = unit_cos(u + static_cast<int64_t>(i) * d, S.cent[ai], S.cn[ai], d);
          if (s < S.far_s) {
            S.far_s = s;
            S.far_i = i;
          }
        }
        if (S.far_i != n) {
          S.cnt[assign[S.far_i]] -= 1;
          assign[S.far_i] = j;
          S.cnt[j] += 1;
          S.moved = 1;
        }
      }
      __syncthreads();
    }
    // arithmetic means, sums in point order (clustering.cpp:138-150); one (cluster, dim) per thread
    double newc = 0.0;
    int wj = -1, wc = 0;
    if (tid < 2 * d) {
      wj = tid / d;
      wc = tid - wj * d;
      double acc = 0.0;
      for (int i = 0; i < n; ++i)
        if (assign[i] == wj) acc = dadd(acc, u[static_cast<int64_t>(i) * d + wc]);
      if (S.cnt[wj] != 0) newc = dmul(acc, ddiv(1.0, static_cast<double>(S.cnt[wj])));
      else wj = -1;  // an empty cluster keeps its centroid
    }
    __syncthreads();
    if (wj >= 0) S.cent[wj][wc] = newc;
    __syncthreads();
    if (tid < 2) {
      double s2 = 0.0;
      for (int c = 0; c < d; ++c) s2 = dadd(s2, dmul(S.cent[tid][c], S.cent[tid][c]));
      S.cn[tid] = __dsqrt_rn(s2);
    }
    __syncthreads();
    // mean cosine to the own centroid, summed in point order (clustering.cpp:152-163)
    for (int i = tid; i < n; i += SPT) {
      const int ai = assign[i];
      nearv[i] = unit_cos(u + static_cast<int64_t>(i) * d, S.cent[ai], S.cn[ai], d);
    }
    __syncthreads();
    if (tid == 0) {
      double obj = 0.0;
      for (int i = 0; i < n; ++i) obj = dadd(obj, nearv[i]);
      obj = ddiv(obj, static_cast<double>(n));
      *objective = obj;
      meta[1] = it + 1;
      S.stop = (it > 0 && dsub(obj, S.prev) < 1e-9) || !S.moved;
      S.prev = obj;
    }
    __syncthreads();
    if (S.stop) break;
  }
  // compact ids (clustering.cpp:166-177)
  if (tid == 0) {
    int c[2] = {0, 0};
    for (int i = 0; i < n; ++i) c[assign[i]] += 1;
    S.cnt[0] = c[0];
    S.cnt[1] = c[1];
  }
  __syncthreads();
  const int live0 = S.cnt[0] != 0, live1 = S.cnt[1] != 0;
  if (!live0)
    for (int i = tid; i < n; i += SPT) assign[i] = 0;  // cluster 1 becomes 0
  if (tid == 0) {
    meta[0] = live0 + live1;
    meta[2] = 0;
    meta[3] = 0;
  }
}

}  // namespace

int launch_split_two(const float* rows, const int32_t* idx, int n, int d, int first, double uni, double* scratch,
                     int32_t* assign, int32_t* meta, double* objective, cudaStream_t st) {
  if (n < 2 || d > 256) return 0;
  k_split_two<<<1, SPT, 0, st>>>(rows, idx, n, d, first, uni, scratch, assign, meta, objective);
  return 1;
}

}  // namespace kvc
