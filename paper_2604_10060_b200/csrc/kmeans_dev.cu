// kmeans_dev.cu -- batch index build (index.cpp:364-450): spherical k-means (clustering.cpp:80-178)
// of every (partition, layer) pool on the GPU, one CTA per pool, bit-identical to the host
// restatement (kmeans.cpp) and so to the reference.
//
// Exactness follows split.cu: every fp64 quantity is formed with round-to-nearest intrinsics in
// the reference's order. Per-point dots run sequentially over the dimension in one thread (two
// points x eight centroids of independent chains per thread, column-major unit rows so a warp's
// loads coalesce); sums over points (k-means++ mass, centroid accumulators, objective) run
// sequentially over the point index in one thread per output value. The generator stays on the
// host: it draws the first centre's index and k - 1 uniforms in order, and the device consumes a
// uniform only where plus_plus draws one (mass > 1e-15), so the stream of draws is the same.
//
// The cosines of every point to every centroid are computed once per centroid set: right after
// the means update they give the objective (cosine to the own centroid) and the next iteration's
// assignment (best centroid, ties to the lower index) -- the reference recomputes the same values.
#include "devmath.cuh"

namespace kvc {

namespace {

using namespace dm;

constexpr int KT = 512;       // threads per pool
constexpr int JB = 8;         // centroids per register block in the cosine pass
constexpr int SEQ_CHUNK = 2048;  // doubles staged in shared memory for the sequential sums

__device__ __forceinline__ double cos_of(double dot, double nc) {
  if (nc < 1e-12) return -2.0;  // degenerate centroid (clustering.cpp:72-76)
  return clamp1(ddiv(dot, nc));
}

struct KmShared {
  double prev, mass, target, far_s;
  int stop, moved, pick, far_i, n_uni_used, degen;
};

// Sequential sum of f(i) over i in [0, n) by thread 0, the terms staged through shared memory by
// the whole block (so the one summing thread reads at shared-memory latency).
template <class F>
__device__ double seq_sum(int n, double* stage, F f) {
  double s = 0.0;
  for (int base = 0; base < n; base += SEQ_CHUNK) {
    const int m = min(SEQ_CHUNK, n - base);
    for (int q = threadIdx.x; q < m; q += KT) stage[q] = f(base + q);
    __syncthreads();
    if (threadIdx.x == 0)
      for (int q = 0; q < m; ++q) s = dadd(s, stage[q]);
    __syncthreads();
  }
  return s;  // valid in thread 0
}

// Cosines of every point to all k centroids: best (value, index; ties to the lower index) and the
// cosine to the point's own centroid a[i].
__device__ void all_cosines(const double* __restrict__ ut, int n, int d, int k, const double* cent,
                            const double* cn, const int32_t* a, double* bs, int32_t* bj, double* own) {
  for (int i0 = threadIdx.x; i0 < n; i0 += 2 * KT) {
    const int i1 = i0 + KT;
    const bool has1 = i1 < n;
    const int r1 = has1 ? i1 : i0;
    const int a0 = a[i0], a1 = a[r1];
    double b0 = -INFINITY, b1 = -INFINITY, o0 = 0.0, o1 = 0.0;
    int j0b = 0, j1b = 0;
    for (int jb = 0; jb < k; jb += JB) {
      const int nj = min(JB, k - jb);
      double s0[JB], s1[JB];
#pragma unroll
      for (int q = 0; q < JB; ++q) s0[q] = s1[q] = 0.0;
      for (int c = 0; c < d; c += 4) {
        double x0[4], x1[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          x0[e] = ut[static_cast<int64_t>(c + e) * n + i0];
          x1[e] = ut[static_cast<int64_t>(c + e) * n + r1];
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
          for (int q = 0; q < JB; ++q) {
            if (q < nj) {
              const double cv = cent[(jb + q) * d + c + e];
              s0[q] = dadd(s0[q], dmul(x0[e], cv));
              s1[q] = dadd(s1[q], dmul(x1[e], cv));
            }
          }
      }
#pragma unroll
      for (int q = 0; q < JB; ++q) {
        if (q < nj) {
          const int j = jb + q;
          const double c0 = cos_of(s0[q], cn[j]), c1 = cos_of(s1[q], cn[j]);
          if (c0 > b0) {
            b0 = c0;
            j0b = j;
          }
          if (c1 > b1) {
            b1 = c1;
            j1b = j;
          }
          if (j == a0) o0 = c0;
          if (j == a1) o1 = c1;
        }
      }
    }
    bs[i0] = b0;
    bj[i0] = j0b;
    own[i0] = o0;
    if (has1) {
      bs[i1] = b1;
      bj[i1] = j1b;
      own[i1] = o1;
    }
  }
}

__device__ void centroid_norms(const double* cent, double* cn, int k, int d) {
  for (int j = threadIdx.x; j < k; j += KT) {
    double s = 0.0;
    for (int c = 0; c < d; ++c) s = dadd(s, dmul(cent[j * d + c], cent[j * d + c]));
    cn[j] = __dsqrt_rn(s);
  }
}

// One pool per CTA. Dynamic shared memory: cent[k][d] doubles | cn[k] | stage[SEQ_CHUNK] |
// cnt[k] ints | off[k + 1] ints.
__global__ void __launch_bounds__(KT) k_kmeans(const float* rows, const KmJob* jobs, const double* uniforms,
                                                double* scratch, int32_t* assign_out, int32_t* meta,
                                                double* objective, double* reps, double* vars, int d,
                                                int max_iters, double tol) {
  const KmJob J = jobs[blockIdx.x];
  const int n = J.n, k = J.k, tid = threadIdx.x;
  extern __shared__ __align__(16) uint8_t km_smem[];
  double* cent = reinterpret_cast<double*>(km_smem);
  double* cn = cent + static_cast<int64_t>(k) * d;
  double* stage = cn + k;
  int* cnt = reinterpret_cast<int*>(stage + SEQ_CHUNK);
  int* off = cnt + k;
  __shared__ KmShared S;
  // per-pool scratch: u[n][d] | ut[d][n] | bs[n] | own[n] | near[n] (doubles) | bj[n] | memb[n] | taken[n]
  double* u = scratch + J.scratch0;
  double* ut = u + static_cast<int64_t>(n) * d;
  double* bs = ut + static_cast<int64_t>(n) * d;
  double* own = bs + n;
  double* nearv = own + n;
  int32_t* bj = reinterpret_cast<int32_t*>(nearv + n);
  int32_t* memb = bj + n;
  int32_t* taken = memb + n;
  int32_t* a = assign_out + J.out0;
  const float* P = rows + J.row0 * d;
  const double* uni = uniforms + J.uni0;
  if (tid == 0) S.degen = 0;
  __syncthreads();
  // unit rows (clustering.cpp:14-22)
  for (int i = tid; i < n; i += KT) {
    const float* p = P + static_cast<int64_t>(i) * d;
    double s = 0.0;
    for (int c = 0; c < d; ++c) {
      const double x = static_cast<double>(p[c]);
      s = dadd(s, dmul(x, x));
    }
    const double nr = __dsqrt_rn(s);
    if (nr < 1e-12) S.degen = 1;
    for (int c = 0; c < d; ++c) {
      const double r = ddiv(static_cast<double>(p[c]), nr);
      u[static_cast<int64_t>(i) * d + c] = r;
      ut[static_cast<int64_t>(c) * n + i] = r;
    }
    taken[i] = 0;
    a[i] = 0;
  }
  __syncthreads();
  if (S.degen) {
    if (tid == 0) meta[blockIdx.x * 4 + 3] = -2;
    return;
  }
  // k-means++ seeding with 1 - cosine weights (clustering.cpp:25-70)
  int pick = J.first;
  if (tid == 0) {
    S.n_uni_used = 0;
    taken[pick] = 1;
  }
  for (int c = tid; c < d; c += KT) cent[c] = u[static_cast<int64_t>(pick) * d + c];
  __syncthreads();
  for (int i = tid; i < n; i += KT) {
    double s = 0.0;
    for (int c = 0; c < d; ++c) s = dadd(s, dmul(ut[static_cast<int64_t>(c) * n + i], cent[c]));
    nearv[i] = s;
  }
  __syncthreads();
  for (int j = 1; j < k; ++j) {
    const double mass = seq_sum(n, stage, [&](int i) { return taken[i] ? 0.0 : fmax(0.0, dsub(1.0, nearv[i])); });
    // (adding +0.0 for taken points leaves the sequential sum unchanged: it is never -0.0)
    // the weighted pick: the first untaken point whose running weight reaches the target,
    // scanned by thread 0 over shared-memory chunks (taken points staged as -1: skipped)
    if (tid == 0) {
      S.pick = n;
      S.mass = mass;
      S.target = mass > 1e-15 ? dmul(uni[S.n_uni_used++], mass) : 0.0;
      S.far_s = 0.0;  // running weight
    }
    __syncthreads();
    if (S.mass > 1e-15) {
      for (int base = 0; base < n; base += SEQ_CHUNK) {
        const int m = min(SEQ_CHUNK, n - base);
        for (int q = tid; q < m; q += KT) stage[q] = taken[base + q] ? -1.0 : fmax(0.0, dsub(1.0, nearv[base + q]));
        __syncthreads();
        if (tid == 0) {
          double run = S.far_s;
          for (int q = 0; q < m; ++q) {
            if (stage[q] < 0.0) continue;
            run = dadd(run, stage[q]);
            if (run >= S.target) {
              S.pick = base + q;
              break;
            }
          }
          S.far_s = run;
        }
        __syncthreads();
        if (S.pick != n) break;
      }
    }
    if (tid == 0) {
      int pk = S.pick;
      if (pk == n)
        for (int i = 0; i < n; ++i)
          if (!taken[i]) {
            pk = i;
            break;
          }
      taken[pk] = 1;
      S.pick = pk;
    }
    __syncthreads();
    pick = S.pick;
    double* cj = cent + static_cast<int64_t>(j) * d;
    for (int c = tid; c < d; c += KT) cj[c] = u[static_cast<int64_t>(pick) * d + c];
    __syncthreads();
    if (j + 1 < k)
      for (int i = tid; i < n; i += KT) {
        double s = 0.0;
        for (int c = 0; c < d; ++c) s = dadd(s, dmul(ut[static_cast<int64_t>(c) * n + i], cj[c]));
        nearv[i] = fmax(nearv[i], s);
      }
    __syncthreads();
  }
  centroid_norms(cent, cn, k, d);
  if (tid == 0) {
    S.prev = -INFINITY;
    S.stop = 0;
  }
  __syncthreads();
  all_cosines(ut, n, d, k, cent, cn, a, bs, bj, own);
  __syncthreads();
  int iters = 0;
  double obj = 0.0;
  for (int it = 0; it < max_iters; ++it) {
    // assignment from the cached cosines (clustering.cpp:99-112)
    for (int j = tid; j < k; j += KT) cnt[j] = 0;
    if (tid == 0) S.moved = 0;
    __syncthreads();
    int mv = 0;
    for (int i = tid; i < n; i += KT) {
      const int b = bj[i];
      if (a[i] != b) mv = 1;
      a[i] = b;
      own[i] = bs[i];  // cosine to the own centroid, for the reseed scan
      atomicAdd(&cnt[b], 1);
    }
    if (__syncthreads_or(mv) && tid == 0) S.moved = 1;
    // empty-cluster reseed (clustering.cpp:117-136): for each empty cluster in order, the point
    // with the smallest cosine to its own centroid among clusters of more than one point -- the
    // first minimum in index order, i.e. the lexicographic (cosine, index) minimum
    for (int j = 0; j < k; ++j) {
      if (cnt[j] != 0) continue;  // block-uniform (cnt changes only between barriers)
      double bv = INFINITY;
      int bi = n;
      for (int i = tid; i < n; i += KT) {
        if (cnt[a[i]] <= 1) continue;
        const double s = own[i];
        if (s < bv) {  // i increases within a thread: strict < keeps the first
          bv = s;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov < bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if ((tid & 31) == 0) {
        stage[tid >> 5] = bv;
        reinterpret_cast<int*>(stage + 32)[tid >> 5] = bi;
      }
      __syncthreads();
      if (tid == 0) {
        double v = INFINITY;
        int far = n;
        for (int w = 0; w < KT / 32; ++w) {
          const double ov = stage[w];
          const int oi = reinterpret_cast<int*>(stage + 32)[w];
          if (ov < v || (ov == v && oi < far)) {
            v = ov;
            far = oi;
          }
        }
        if (far != n) {
          cnt[a[far]] -= 1;
          a[far] = j;
          cnt[j] += 1;
          double s = 0.0;  // its cosine to the new own centroid (for later scans of this pass)
          for (int c = 0; c < d; ++c) s = dadd(s, dmul(u[static_cast<int64_t>(far) * d + c], cent[j * d + c]));
          own[far] = cos_of(s, cn[j]);
          S.moved = 1;
        }
      }
      __syncthreads();
    }
    // member lists in point order (one warp per cluster, ballots keep the order)
    if (tid == 0) {
      int o = 0;
      for (int j = 0; j < k; ++j) {
        off[j] = o;
        o += cnt[j];
      }
      off[k] = o;
    }
    __syncthreads();
    {
      const int warp = tid >> 5, lane = tid & 31;
      for (int j = warp; j < k; j += KT / 32) {
        int w = off[j];
        for (int base = 0; base < n; base += 32) {
          const int i = base + lane;
          const bool m = i < n && a[i] == j;
          const unsigned bal = __ballot_sync(0xffffffffu, m);
          if (m) memb[w + __popc(bal & ((1u << lane) - 1u))] = i;
          w += __popc(bal);
        }
      }
    }
    __syncthreads();
    // arithmetic means, sums in point order (clustering.cpp:138-150); one (cluster, dim) chain
    // per thread, loads 8 members ahead
    for (int q = tid; q < k * d; q += KT) {
      const int j = q / d, c = q - j * d;
      if (cnt[j] == 0) continue;  // an empty cluster keeps its centroid
      const int b = off[j], e = off[j + 1];
      double acc = 0.0;
      int m = b;
      for (; m + 8 <= e; m += 8) {
        double x[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) x[r] = u[static_cast<int64_t>(memb[m + r]) * d + c];
#pragma unroll
        for (int r = 0; r < 8; ++r) acc = dadd(acc, x[r]);
      }
      for (; m < e; ++m) acc = dadd(acc, u[static_cast<int64_t>(memb[m]) * d + c]);
      const double inv = ddiv(1.0, static_cast<double>(cnt[j]));
      cent[q] = dmul(acc, inv);
    }
    __syncthreads();
    centroid_norms(cent, cn, k, d);
    __syncthreads();
    all_cosines(ut, n, d, k, cent, cn, a, bs, bj, own);
    __syncthreads();
    // mean cosine to the own centroid (clustering.cpp:152-163)
    const double tot = seq_sum(n, stage, [&](int i) { return own[i]; });
    if (tid == 0) {
      obj = ddiv(tot, static_cast<double>(n));
      S.stop = (it > 0 && dsub(obj, S.prev) < tol) || !S.moved;
      S.prev = obj;
      objective[blockIdx.x] = obj;
      meta[blockIdx.x * 4 + 1] = it + 1;
    }
    iters = it + 1;
    __syncthreads();
    if (S.stop) break;
  }
  (void)iters;
  // compact ids (clustering.cpp:166-177)
  for (int j = tid; j < k; j += KT) cnt[j] = 0;
  __syncthreads();
  for (int i = tid; i < n; i += KT) atomicAdd(&cnt[a[i]], 1);
  __syncthreads();
  if (tid == 0) {
    int live = 0;
    for (int j = 0; j < k; ++j) off[j] = cnt[j] != 0 ? live++ : -1;
    meta[blockIdx.x * 4 + 0] = live;
    meta[blockIdx.x * 4 + 2] = 0;
    meta[blockIdx.x * 4 + 3] = 0;
    if (max_iters <= 0) {
      meta[blockIdx.x * 4 + 1] = 0;
      objective[blockIdx.x] = 0.0;
    }
  }
  __syncthreads();
  for (int i = tid; i < n; i += KT) a[i] = off[a[i]];
  if (J.rep0 < 0) return;
  // Eq. 1 / Eq. 2 statistics of every output cluster (representative(), variance() in
  // kmeans.cpp: member sums in point order over the f32 rows, then the mean; per-member squared
  // distances sequential over the dimension, summed in member order)
  __syncthreads();
  const int live = meta[blockIdx.x * 4 + 0];
  for (int j = tid; j < live; j += KT) cnt[j] = 0;
  __syncthreads();
  for (int i = tid; i < n; i += KT) atomicAdd(&cnt[a[i]], 1);
  __syncthreads();
  if (tid == 0) {
    int o = 0;
    for (int j = 0; j < live; ++j) {
      off[j] = o;
      o += cnt[j];
    }
    off[live] = o;
  }
  __syncthreads();
  {
    const int warp = tid >> 5, lane = tid & 31;
    for (int j = warp; j < live; j += KT / 32) {
      int w = off[j];
      for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        const bool m = i < n && a[i] == j;
        const unsigned bal = __ballot_sync(0xffffffffu, m);
        if (m) memb[w + __popc(bal & ((1u << lane) - 1u))] = i;
        w += __popc(bal);
      }
    }
  }
  __syncthreads();
  double* R = reps + J.rep0;
  for (int q = tid; q < live * d; q += KT) {
    const int j = q / d, c = q - j * d;
    double acc = 0.0;
    for (int m = off[j]; m < off[j + 1]; ++m) acc = dadd(acc, static_cast<double>(P[static_cast<int64_t>(memb[m]) * d + c]));
    R[q] = dmul(acc, ddiv(1.0, static_cast<double>(cnt[j])));
  }
  __syncthreads();
  for (int pos = tid; pos < n; pos += KT) {  // per member, in cluster-major member order
    const int i = memb[pos];
    const int j = a[i];
    const float* p = P + static_cast<int64_t>(i) * d;
    const double* r = R + static_cast<int64_t>(j) * d;
    double sq = 0.0;
    for (int c = 0; c < d; ++c) {
      const double df = dsub(static_cast<double>(p[c]), r[c]);
      sq = dadd(sq, dmul(df, df));
    }
    bs[pos] = sq;
  }
  __syncthreads();
  for (int j = tid; j < live; j += KT) {
    double tot = 0.0;
    for (int m = off[j]; m < off[j + 1]; ++m) tot = dadd(tot, bs[m]);
    vars[J.var0 + j] = ddiv(tot, static_cast<double>(cnt[j]));
  }
}

}  // namespace

size_t kmeans_smem_bytes(int k, int d) {
  return (static_cast<size_t>(k) * d + k + SEQ_CHUNK) * 8 + (2 * static_cast<size_t>(k) + 1) * 4;
}

size_t kmeans_scratch_doubles(int n, int d) { return static_cast<size_t>(n) * (2 * d + 3) + 2 * static_cast<size_t>(n); }

int launch_kmeans(const float* rows, const KmJob* jobs, int n_jobs, const double* uniforms, double* scratch,
                  int32_t* assign, int32_t* meta, double* objective, double* reps, double* vars, int d, int k_max,
                  int max_iters, double tol, cudaStream_t st) {
  if (n_jobs <= 0) return 0;
  const size_t smem = kmeans_smem_bytes(k_max, d);
  if (!smem_optin(reinterpret_cast<const void*>(k_kmeans), smem)) return 0;
  k_kmeans<<<n_jobs, KT, smem, st>>>(rows, jobs, uniforms, scratch, assign, meta, objective, reps, vars, d,
                                     max_iters, tol);
  return 1;
}

}  // namespace kvc
