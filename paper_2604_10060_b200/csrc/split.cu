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
constexpr int OBJ_CHUNK = 4096;  // 32 KB of the objective's terms per shared-memory pass

// Sequential fp64 dot of point i (column-major unit rows ut[c * n + i]: coalesced across the
// threads of a warp, which take consecutive points) with a shared-memory vector.
__device__ __forceinline__ double dot_col(const double* __restrict__ ut, int n, int i, const double* v, int d) {
  double s = 0.0;
  int c = 0;
  for (; c + 16 <= d; c += 16) {  // the loads of 16 dimensions in flight ahead of the chain
    double x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = ut[static_cast<int64_t>(c + k) * n + i];
#pragma unroll
    for (int k = 0; k < 16; ++k) s = dadd(s, dmul(x[k], v[c + k]));
  }
  for (; c < d; ++c) s = dadd(s, dmul(ut[static_cast<int64_t>(c) * n + i], v[c]));
  return s;
}

// Both centroids in one pass (two independent chains; each is the reference's sequential dot).
__device__ __forceinline__ void dot2_col(const double* __restrict__ ut, int n, int i, const double* c0,
                                         const double* c1, int d, double& s0, double& s1) {
  double a = 0.0, b = 0.0;
  for (int c = 0; c < d; ++c) {
    const double x = ut[static_cast<int64_t>(c) * n + i];
    a = dadd(a, dmul(x, c0[c]));
    b = dadd(b, dmul(x, c1[c]));
  }
  s0 = a;
  s1 = b;
}

__device__ __forceinline__ double cos_of(double dot, double nc) {
  if (nc < 1e-12) return -2.0;  // degenerate centroid (clustering.cpp:72-76)
  return clamp1(ddiv(dot, nc));
}

// Phase clocks of the batched kernel (KVC_SPLIT_PROF, development): per job, cycles of
// [unit rows, same check, seeding, assign+reseed+lists, centroid update, norms, cosines,
// objective, compaction, child stats] and [10] iterations, [11] n.
__device__ long long* g_split_prof = nullptr;

struct SplitSmem {
  long long pc[12];
  long long pc_t;
  double cent[2][256];
  double cn[2];
  double prev;
  int cnt[2];
  int moved, same, pick, stop, degen, far_i;
  double far_s;
};

// Cosines of every point to both centroids (unit_cos, clustering.cpp:72-76) into sc[2][n]. The
// reference recomputes them in the objective of one iteration and the assignment of the next,
// with the same centroids: computing them once yields the identical values.
__device__ __forceinline__ void cosines(const double* __restrict__ ut, int n, int d, SplitSmem& S, double* sc) {
  if (n <= SPT) {
    // one point per thread: the loads of 16 dimensions in flight ahead of the two chains
    const int i0 = threadIdx.x;
    if (i0 < n) {
      double a0 = 0.0, b0 = 0.0;
      int c = 0;
      for (; c + 16 <= d; c += 16) {
        double x0[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) x0[k] = ut[static_cast<int64_t>(c + k) * n + i0];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          a0 = dadd(a0, dmul(x0[k], S.cent[0][c + k]));
          b0 = dadd(b0, dmul(x0[k], S.cent[1][c + k]));
        }
      }
      for (; c < d; ++c) {
        const double x0 = ut[static_cast<int64_t>(c) * n + i0];
        a0 = dadd(a0, dmul(x0, S.cent[0][c]));
        b0 = dadd(b0, dmul(x0, S.cent[1][c]));
      }
      sc[i0] = cos_of(a0, S.cn[0]);
      sc[n + i0] = cos_of(b0, S.cn[1]);
    }
    return;
  }
  // two points per thread (four independent chains) and the loads of 8 dimensions issued ahead
  // of their arithmetic: the chains are latency-bound, so memory-level parallelism is the lever
  for (int i0 = threadIdx.x; i0 < n; i0 += 2 * SPT) {
    const int i1 = i0 + SPT;
    const bool has1 = i1 < n;
    const int j1 = has1 ? i1 : i0;
    double a0 = 0.0, b0 = 0.0, a1 = 0.0, b1 = 0.0;
    int c = 0;
    for (; c + 8 <= d; c += 8) {
      double x0[8], x1[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        x0[k] = ut[static_cast<int64_t>(c + k) * n + i0];
        x1[k] = ut[static_cast<int64_t>(c + k) * n + j1];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double c0 = S.cent[0][c + k], c1 = S.cent[1][c + k];
        a0 = dadd(a0, dmul(x0[k], c0));
        b0 = dadd(b0, dmul(x0[k], c1));
        a1 = dadd(a1, dmul(x1[k], c0));
        b1 = dadd(b1, dmul(x1[k], c1));
      }
    }
    for (; c < d; ++c) {
      const double x0 = ut[static_cast<int64_t>(c) * n + i0], x1 = ut[static_cast<int64_t>(c) * n + j1];
      a0 = dadd(a0, dmul(x0, S.cent[0][c]));
      b0 = dadd(b0, dmul(x0, S.cent[1][c]));
      a1 = dadd(a1, dmul(x1, S.cent[0][c]));
      b1 = dadd(b1, dmul(x1, S.cent[1][c]));
    }
    sc[i0] = cos_of(a0, S.cn[0]);
    sc[n + i0] = cos_of(b0, S.cn[1]);
    if (has1) {
      sc[i1] = cos_of(a1, S.cn[0]);
      sc[n + i1] = cos_of(b1, S.cn[1]);
    }
  }
}

// Sequential sum s + x[0] + x[1] + ... (exact order) with the shared-memory loads issued 8 ahead.
__device__ __forceinline__ double seq_sum8(double s, const double* x, int m) {
  int k = 0;
  for (; k + 8 <= m; k += 8) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = x[k + j];
#pragma unroll
    for (int j = 0; j < 8; ++j) s = dadd(s, v[j]);
  }
  for (; k < m; ++k) s = dadd(s, x[k]);
  return s;
}

__device__ __forceinline__ void centroid_norms(SplitSmem& S, int d) {
  if (threadIdx.x < 2) {
    const double* c = S.cent[threadIdx.x];
    double s = 0.0;
    for (int k = 0; k < d; ++k) s = dadd(s, dmul(c[k], c[k]));
    S.cn[threadIdx.x] = __dsqrt_rn(s);
  }
}

// rows: staged f32 rows; idx[n]: the points of this split (rows idx[i]).
// scratch (doubles): u[n][d] | ut[d][n] | sc[2][n] | nearv[n]
// out: assign[n]; meta[4] = {k_live, iterations, degenerate, error}; objective[1].
__device__ __forceinline__ void split_two_body(const float* rows, const int32_t* idx, int n, int d, int first,
                                               double uni, double* scratch, int32_t* assign, int32_t* meta,
                                               double* objective, double* S_ob) {
  __shared__ SplitSmem S;
  __shared__ double S_mass;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* u = scratch;
  double* ut = u + static_cast<int64_t>(n) * d;
  double* sc = ut + static_cast<int64_t>(n) * d;
  double* nearv = sc + 2 * static_cast<int64_t>(n);
  const bool prof = g_split_prof != nullptr;
#define SPROF(k)                                   \
  if (prof && tid == 0) {                          \
    const long long c_ = clock64();                \
    S.pc[k] += c_ - S.pc_t;                        \
    S.pc_t = c_;                                   \
  }
  if (tid == 0) {
    S.same = 1;
    S.degen = 0;
    for (int k = 0; k < 12; ++k) S.pc[k] = 0;
    S.pc[11] = n;
    S.pc_t = clock64();
  }
  __syncthreads();
  // unit rows (clustering.cpp:14-22): r / norm(r), stored row- and column-major. One point per
  // thread (the norm is the reference's sequential sum); rows are read 16 bytes per load and the
  // row-major copy written 16 bytes per store (each warp instruction touches 32 rows: 4x fewer
  // of them than element-wise accesses)
  const bool vec = (d & 3) == 0;
  for (int i = tid; i < n; i += SPT) {
    const float* p = rows + static_cast<int64_t>(idx[i]) * d;
    double s = 0.0;
    for (int c0 = 0; c0 < d; c0 += 16) {  // 16 elements in flight ahead of the sequential sum
      float x[16];
      if (vec && c0 + 16 <= d) {
#pragma unroll
        for (int k = 0; k < 16; k += 4) {
          const float4 v = *reinterpret_cast<const float4*>(p + c0 + k);
          x[k] = v.x;
          x[k + 1] = v.y;
          x[k + 2] = v.z;
          x[k + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = c0 + k < d ? p[c0 + k] : 0.f;
      }
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (c0 + k < d) s = dadd(s, dmul(static_cast<double>(x[k]), static_cast<double>(x[k])));
    }
    const double nr = __dsqrt_rn(s);
    if (nr < 1e-12) S.degen = 1;
    // RN(x / nr) for every element from one reciprocal (div_rcp: Markstein's correctly rounded
    // step, bit-identical to __ddiv_rn; tests/test_kernels_gpu.py checks it on real divisors)
    const double y = ddiv(1.0, nr);
    double* ur = u + static_cast<int64_t>(i) * d;
    for (int c0 = 0; c0 < d; c0 += 16) {
      float x[16];
      if (vec && c0 + 16 <= d) {
#pragma unroll
        for (int k = 0; k < 16; k += 4) {
          const float4 v = *reinterpret_cast<const float4*>(p + c0 + k);
          x[k] = v.x;
          x[k + 1] = v.y;
          x[k + 2] = v.z;
          x[k + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = c0 + k < d ? p[c0 + k] : 0.f;
      }
      double r[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) r[k] = nr < 1e-12 || c0 + k >= d ? 0.0 : div_rcp(static_cast<double>(x[k]), nr, y);
      if (vec && c0 + 16 <= d) {
#pragma unroll
        for (int k = 0; k < 16; k += 2) *reinterpret_cast<double2*>(ur + c0 + k) = make_double2(r[k], r[k + 1]);
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (c0 + k < d) ur[c0 + k] = r[k];
      }
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (c0 + k < d) ut[static_cast<int64_t>(c0 + k) * n + i] = r[k];
    }
  }
  __syncthreads();
  SPROF(0)
  if (S.degen) {
    if (tid == 0) meta[3] = -2;  // zero vector (the host raises KVC_E_DEGENERATE)
    return;
  }
  for (int c = tid; c < d; c += SPT) S.cent[0][c] = u[c];
  __syncthreads();
  // all points equal (within 1e-12 of the first): the deterministic (n-1, 1) partition
  for (int i = 1 + tid; i < n; i += SPT)
    if (dot_col(ut, n, i, S.cent[0], d) < 1.0 - 1e-12) S.same = 0;
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
  // k-means++ seeding with 1 - cosine weights, k = 2 (clustering.cpp:25-70)
  __syncthreads();
  SPROF(1)
  for (int c = tid; c < d; c += SPT) S.cent[0][c] = u[static_cast<int64_t>(first) * d + c];
  __syncthreads();
  for (int i = tid; i < n; i += SPT) nearv[i] = dot_col(ut, n, i, S.cent[0], d);
  __syncthreads();
  // The seeding's two sequential sums over the points (the mass, then the weighted scan) run on
  // one thread; the weights are staged in shared memory (the chosen point's weight 0.0: adding
  // +0.0 to a sum of non-negative terms is exact, the same as skipping it) and read 8 at a time
  // ahead of the dependent adds.
  double mass = 0.0;
  for (int base = 0; base < n; base += OBJ_CHUNK) {
    const int m = min(OBJ_CHUNK, n - base);
    for (int k = tid; k < m; k += SPT) S_ob[k] = base + k == first ? 0.0 : fmax(0.0, dsub(1.0, nearv[base + k]));
    __syncthreads();
    if (tid == 0) mass = seq_sum8(mass, S_ob, m);
    __syncthreads();
  }
  if (tid == 0) {
    S.pick = n;
    S.prev = -INFINITY;
    S.stop = 0;
    S_mass = mass;
  }
  __syncthreads();
  if (S_mass > 1e-15) {
    const double target = dmul(uni, S_mass);
    double run = 0.0;
    int pick = n;  // thread 0's scan state; S.pick is written once, when the pick is found
    for (int base = 0; base < n; base += OBJ_CHUNK) {
      const int m = min(OBJ_CHUNK, n - base);
      for (int k = tid; k < m; k += SPT) S_ob[k] = base + k == first ? 0.0 : fmax(0.0, dsub(1.0, nearv[base + k]));
      __syncthreads();
      if (tid == 0) {
        for (int k = 0; k < m; ++k) {
          if (base + k == first) continue;
          run = dadd(run, S_ob[k]);
          if (run >= target) {
            pick = base + k;
            break;
          }
        }
        if (pick != n) S.pick = pick;
      }
      __syncthreads();
      if (S.pick != n) break;
    }
  }
  if (tid == 0 && S.pick == n) S.pick = first == 0 ? 1 : 0;
  __syncthreads();
  for (int c = tid; c < d; c += SPT) S.cent[1][c] = u[static_cast<int64_t>(S.pick) * d + c];
  for (int i = tid; i < n; i += SPT) assign[i] = 0;
  __syncthreads();
  centroid_norms(S, d);
  __syncthreads();
  cosines(ut, n, d, S, sc);
  __syncthreads();
  SPROF(2)
  for (int it = 0; it < 50; ++it) {
    if (tid == 0) {
      S.moved = 0;
      S.cnt[0] = 0;
      S.cnt[1] = 0;
    }
    __syncthreads();
    // assignment, ties to the lower index (clustering.cpp:99-112), from the cached cosines
    int c0 = 0, c1 = 0, mv = 0;
    for (int i = tid; i < n; i += SPT) {
      const int bj = sc[n + i] > sc[i] ? 1 : 0;
      if (assign[i] != bj) mv = 1;
      assign[i] = bj;
      c0 += 1 - bj;
      c1 += bj;
    }
    if (__syncthreads_or(mv) && tid == 0) S.moved = 1;
    if (c0) atomicAdd(&S.cnt[0], c0);
    if (c1) atomicAdd(&S.cnt[1], c1);
    __syncthreads();
    // empty-cluster reseed (clustering.cpp:117-136): the point farthest from its centroid among
    // clusters with more than one point (first minimum in index order), with this iteration's
    // centroids, i.e. the cached cosines
    for (int j = 0; j < 2; ++j) {
      if (S.cnt[j] != 0) continue;  // block-uniform
      if (tid == 0) {
        int far = n;
        double far_s = INFINITY;
        for (int i = 0; i < n; ++i) {
          const int ai = assign[i];
          if (S.cnt[ai] <= 1) continue;
          const double s = sc[static_cast<int64_t>(ai) * n + i];
          if (s < far_s) {
            far_s = s;
            far = i;
          }
        }
        if (far != n) {
          S.cnt[assign[far]] -= 1;
          assign[far] = j;
          S.cnt[j] += 1;
          S.moved = 1;
        }
      }
      __syncthreads();
    }
    // member lists in point order (warp j scans cluster j with ballots), in the k-means++ scratch
    // (nearv is dead after seeding): memb[0, cnt0) = cluster 0, memb[cnt0, n) = cluster 1
    // (in shared memory -- the objective's staging area, free until the objective -- when they fit:
    // the centroid sums below read them ahead of their dependent row loads)
    int* memb = n <= 2 * OBJ_CHUNK ? reinterpret_cast<int*>(S_ob) : reinterpret_cast<int*>(nearv);
    if (warp < 2) {
      int w = warp == 0 ? 0 : S.cnt[0];
      for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        const bool m = i < n && assign[i] == warp;
        const unsigned bal = __ballot_sync(0xffffffffu, m);
        if (m) memb[w + __popc(bal & ((1u << lane) - 1u))] = i;
        w += __popc(bal);
      }
    }
    __syncthreads();
    SPROF(3)
    // arithmetic means, sums in member (= point) order (clustering.cpp:138-150); one (cluster,
    // dim) chain per thread over that cluster's members only, rows read coalesced across the
    // dimension, the next 16 members' loads in flight while a group is summed
    double newc = 0.0;
    int wj = -1, wc = 0;
    if (tid < 2 * d) {
      wj = tid / d;
      wc = tid - wj * d;
      const int mb = wj == 0 ? 0 : S.cnt[0], me = wj == 0 ? S.cnt[0] : n;
      double acc = 0.0;
      const int m16 = mb + ((me - mb) & ~15);
      double x[16];
      auto load16 = [&](int m) {
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = u[static_cast<int64_t>(memb[m + k]) * d + wc];
      };
      if (m16 > mb) load16(mb);
      for (int m = mb; m < m16; m += 16) {
        double y[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) y[k] = x[k];
        if (m + 16 < m16) load16(m + 16);
#pragma unroll
        for (int k = 0; k < 16; ++k) acc = dadd(acc, y[k]);
      }
      for (int m = m16; m < me; ++m) acc = dadd(acc, u[static_cast<int64_t>(memb[m]) * d + wc]);
      if (S.cnt[wj] != 0) newc = dmul(acc, ddiv(1.0, static_cast<double>(S.cnt[wj])));
      else wj = -1;  // an empty cluster keeps its centroid
    }
    __syncthreads();
    if (wj >= 0) S.cent[wj][wc] = newc;
    __syncthreads();
    SPROF(4)
    if (n < SPT) {
      // an idle thread forms both centroid norms (two interleaved sequential chains) while the
      // point threads form their dots; the cosines divide once both are there
      double a0 = 0.0, b0 = 0.0;
      if (tid == SPT - 1) {
        double s0 = 0.0, s1 = 0.0;
        for (int k = 0; k < d; ++k) {
          s0 = dadd(s0, dmul(S.cent[0][k], S.cent[0][k]));
          s1 = dadd(s1, dmul(S.cent[1][k], S.cent[1][k]));
        }
        S.cn[0] = __dsqrt_rn(s0);
        S.cn[1] = __dsqrt_rn(s1);
      } else if (tid < n) {
        int c = 0;
        for (; c + 16 <= d; c += 16) {
          double x0[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) x0[k] = ut[static_cast<int64_t>(c + k) * n + tid];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            a0 = dadd(a0, dmul(x0[k], S.cent[0][c + k]));
            b0 = dadd(b0, dmul(x0[k], S.cent[1][c + k]));
          }
        }
        for (; c < d; ++c) {
          const double x0 = ut[static_cast<int64_t>(c) * n + tid];
          a0 = dadd(a0, dmul(x0, S.cent[0][c]));
          b0 = dadd(b0, dmul(x0, S.cent[1][c]));
        }
      }
      __syncthreads();
      SPROF(5)
      if (tid < n) {
        sc[tid] = cos_of(a0, S.cn[0]);
        sc[n + tid] = cos_of(b0, S.cn[1]);
      }
    } else {
      centroid_norms(S, d);
      __syncthreads();
      SPROF(5)
      cosines(ut, n, d, S, sc);
    }
    __syncthreads();
    SPROF(6)
    // mean cosine to the own centroid, summed in point order (clustering.cpp:152-163)
    // staged through shared memory in chunks so the one summing thread reads at smem latency
    double obj = 0.0;
    for (int base = 0; base < n; base += OBJ_CHUNK) {
      const int m = min(OBJ_CHUNK, n - base);
      for (int k = tid; k < m; k += SPT) S_ob[k] = sc[static_cast<int64_t>(assign[base + k]) * n + base + k];
      __syncthreads();
      if (tid == 0) obj = seq_sum8(obj, S_ob, m);
      __syncthreads();
    }
    if (tid == 0) {
      obj = ddiv(obj, static_cast<double>(n));
      *objective = obj;
      meta[1] = it + 1;
      S.stop = (it > 0 && dsub(obj, S.prev) < 1e-9) || !S.moved;
      S.prev = obj;
    }
    __syncthreads();
    SPROF(7)
    if (prof && tid == 0) S.pc[10] = it + 1;
    if (S.stop) break;
  }
  // compact ids (clustering.cpp:166-177)
  if (tid == 0) {
    S.cnt[0] = 0;
    S.cnt[1] = 0;
  }
  __syncthreads();
  {
    int c1 = 0;
    for (int i = tid; i < n; i += SPT) c1 += assign[i];
    if (c1) atomicAdd(&S.cnt[1], c1);
  }
  __syncthreads();
  if (tid == 0) S.cnt[0] = n - S.cnt[1];
  __syncthreads();
  const int live0 = S.cnt[0] != 0, live1 = S.cnt[1] != 0;
  if (!live0)
    for (int i = tid; i < n; i += SPT) assign[i] = 0;  // cluster 1 becomes 0
  if (tid == 0) {
    meta[0] = live0 + live1;
    meta[2] = 0;
    meta[3] = 0;
  }
  SPROF(8)
  if (prof && tid == 0)
    for (int k = 0; k < 12; ++k) g_split_prof[blockIdx.x * 16 + k] = S.pc[k];
#undef SPROF
}

__global__ void __launch_bounds__(SPT) k_split_two(const float* rows, const int32_t* idx, int n, int d, int first,
                                                    double uni, double* scratch, int32_t* assign, int32_t* meta,
                                                    double* objective) {
  __shared__ double S_ob[OBJ_CHUNK];
  split_two_body(rows, idx, n, d, first, uni, scratch, assign, meta, objective, S_ob);
}

// Eq. 1 / Eq. 2 statistics of the two groups of a split (compute_representative /
// compute_variance, index.cpp:345-362, exactly as k_exact_stats computes them: sums over the
// group's rows in pool order, fp64, round-to-nearest, uncontracted) into slots slot[0] / slot[1]
// (rep64, rep32, rnorm, var), and the variances to var_out (the host's Eq. 5 recursion test).
// memb: n ints of scratch.
__device__ void child_stats(const DevTables& t, const float* rows, const int32_t* idx, int n, const int32_t* assign,
                            const int32_t slot[2], double* var_out, int* memb, double* sq, double* sbuf) {
  __shared__ double srep[2][256];
  __shared__ int scnt[2];
  __shared__ double sinv[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, d = t.d;
  // member lists in pool order (warp g scans group g with ballots)
  if (warp < 2) {
    int w = 0;
    if (warp == 1) {  // group 1 starts after group 0's count
      for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        w += __popc(__ballot_sync(0xffffffffu, i < n && assign[i] == 0));
      }
    }
    const int start = w;
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      const bool m = i < n && assign[i] == warp;
      const unsigned bal = __ballot_sync(0xffffffffu, m);
      if (m) memb[w + __popc(bal & ((1u << lane) - 1u))] = i;
      w += __popc(bal);
    }
    if (lane == 0) scnt[warp] = w - start;
  }
  __syncthreads();
  const int c0 = scnt[0], c1 = scnt[1];
  if (tid < 2) sinv[tid] = (tid == 0 ? c0 : c1) > 0 ? ddiv(1.0, static_cast<double>(tid == 0 ? c0 : c1)) : 0.0;
  // the members' staged row indices (one dependent load less in the chains below), in shared
  // memory when they fit beside the squared distances (n ints + n doubles in the staging area)
  const bool in_smem = static_cast<int64_t>(n) * 12 <= static_cast<int64_t>(OBJ_CHUNK) * 8;
  int* mrow = in_smem ? reinterpret_cast<int*>(sbuf + n) : memb;
  for (int m = tid; m < n; m += blockDim.x) mrow[m] = idx[memb[m]];
  __syncthreads();
  // representatives: one (group, dim) chain per thread over the group's rows, 16 loads ahead
  if (tid < 2 * d) {
    const int g = tid / d, c = tid - g * d;
    const int mb = g == 0 ? 0 : c0, me = g == 0 ? c0 : c0 + c1;
    double acc = 0.0;
    const int m16 = mb + ((me - mb) & ~15);
    float x[16];
    auto load16 = [&](int m) {
#pragma unroll
      for (int k = 0; k < 16; ++k) x[k] = rows[static_cast<int64_t>(mrow[m + k]) * d + c];
    };
    if (m16 > mb) load16(mb);
    for (int m = mb; m < m16; m += 16) {
      float y[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) y[k] = x[k];
      if (m + 16 < m16) load16(m + 16);
#pragma unroll
      for (int k = 0; k < 16; ++k) acc = dadd(acc, static_cast<double>(y[k]));
    }
    for (int m = m16; m < me; ++m) acc = dadd(acc, static_cast<double>(rows[static_cast<int64_t>(mrow[m]) * d + c]));
    const double r = dmul(acc, sinv[g]);
    srep[g][c] = r;
    if (me > mb && slot[g] >= 0) {
      t.rep64[static_cast<int64_t>(slot[g]) * d + c] = r;
      t.rep32[static_cast<int64_t>(slot[g]) * d + c] = static_cast<float>(r);
    }
  }
  __syncthreads();
  // squared distances per row (sequential over the dimension), in member order; rows read 16
  // bytes per load (one row per thread)
  double* sqs = in_smem ? sbuf : sq;
  const bool vec = (d & 3) == 0;
  for (int m = tid; m < c0 + c1; m += blockDim.x) {
    const int g = m < c0 ? 0 : 1;
    const float* p = rows + static_cast<int64_t>(mrow[m]) * d;
    double a = 0.0;
    if (vec) {
      for (int c = 0; c < d; c += 16) {
        float4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = *reinterpret_cast<const float4*>(p + c + 4 * k);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float e[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (c + 4 * k + q >= d) break;
            const double df = dsub(static_cast<double>(e[q]), srep[g][c + 4 * k + q]);
            a = dadd(a, dmul(df, df));
          }
        }
      }
    } else {
      for (int c = 0; c < d; ++c) {
        const double df = dsub(static_cast<double>(p[c]), srep[g][c]);
        a = dadd(a, dmul(df, df));
      }
    }
    sqs[m] = a;
  }
  __syncthreads();
  // sequential sums over the rows (one thread per group, staged reads 8 ahead), and the norms of
  // the representatives on two other threads
  if (tid == 0 || tid == 32) {
    const int g = tid == 0 ? 0 : 1;
    const int mb = g == 0 ? 0 : c0, me = g == 0 ? c0 : c0 + c1;
    if (me > mb) {
      const double total = seq_sum8(0.0, sqs + mb, me - mb);
      const double var = ddiv(total, static_cast<double>(me - mb));
      if (slot[g] >= 0) t.var[slot[g]] = var;
      if (var_out) var_out[g] = var;
    } else if (var_out) {
      var_out[g] = 0.0;
    }
  }
  if (tid == 64 || tid == 96) {
    const int g = tid == 64 ? 0 : 1;
    const int mb = g == 0 ? 0 : c0, me = g == 0 ? c0 : c0 + c1;
    if (me > mb && slot[g] >= 0) {
      double nn = 0.0;
      for (int c = 0; c < d; ++c) nn = dadd(nn, dmul(srep[g][c], srep[g][c]));
      t.rnorm[slot[g]] = __dsqrt_rn(nn);
    }
  }
}

// Independent splits in one launch (one CTA each): the ingest wave engine settles the split
// events of many domains at once (context_waves.cpp). A job with slots also installs its two
// groups' statistics; a job with assign_in skips the k-means (a result already known).
__global__ void __launch_bounds__(SPT) k_split_two_batch(DevTables t, const SplitJob* jobs, int d) {
  __shared__ double S_ob[OBJ_CHUNK];  // staging shared by the k-means and the children statistics
  const SplitJob j = jobs[blockIdx.x];
  if (j.assign_in) {
    for (int i = threadIdx.x; i < j.n; i += SPT) j.assign[i] = j.assign_in[i];
    if (threadIdx.x == 0) {
      j.meta[0] = 2;
      j.meta[1] = 0;
      j.meta[2] = 0;
      j.meta[3] = 0;
    }
    __syncthreads();
  } else {
    split_two_body(j.rows, j.idx, j.n, d, j.first, j.uni, j.scratch, j.assign, j.meta, j.objective, S_ob);
    __syncthreads();
    if (j.meta[3] != 0) return;  // degenerate row: the host raises it
  }
  if (j.slot[0] < 0 && j.slot[1] < 0 && !j.var_out) return;
  int* memb = reinterpret_cast<int*>(j.scratch);
  double* sq = j.scratch + (static_cast<int64_t>(j.n) + 1) / 2 + 1;
  const long long c0 = clock64();
  child_stats(t, j.rows, j.idx, j.n, j.assign, j.slot, j.var_out, memb, sq, S_ob);
  if (g_split_prof && threadIdx.x == 0) g_split_prof[blockIdx.x * 16 + 9] = clock64() - c0;
}

}  // namespace

void split_prof_set(long long* p) { cudaMemcpyToSymbol(g_split_prof, &p, sizeof(p)); }

int launch_split_two_batch(const DevTables& t, const SplitJob* jobs, int n_jobs, int d, cudaStream_t st) {
  if (n_jobs <= 0 || d > 256) return 0;
  k_split_two_batch<<<n_jobs, SPT, 0, st>>>(t, jobs, d);
  return 1;
}

int launch_split_two(const float* rows, const int32_t* idx, int n, int d, int first, double uni, double* scratch,
                     int32_t* assign, int32_t* meta, double* objective, cudaStream_t st) {
  if (n < 2 || d > 256) return 0;
  k_split_two<<<1, SPT, 0, st>>>(rows, idx, n, d, first, uni, scratch, assign, meta, objective);
  return 1;
}

}  // namespace kvc
