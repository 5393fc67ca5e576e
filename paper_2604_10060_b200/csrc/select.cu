// select.cu -- K4 v3: cluster scoring and selection for one decode step, one CTA per domain.
//
// Same contract as k_score_select2 (kernels.cu): visual_topk (index.cpp:192-208), semantic_topk
// over the chosen partitions' clusters + registered buffers (index.cpp:210-240), the optional
// prefetch ranking of layer l+1 (retrieval.cpp:117-128), the verified list (retrieval.cpp:20-26),
// the attended-set size, and the attention work list (page descriptors) for K6.
//
// The CTA is latency bound: every phase is one round of independent global loads followed by
// shared-memory work. The schedule is built around keeping that round count minimal:
//   R1  query, window-ring owners, visual representatives (+ norms)
//   R2  chosen partitions' list offsets
//   R3  the candidate slots
//   R4  per candidate: lazy flag, norm, id, and (warp-cooperative) the fp32 mirror row
//   R5  boundary set S: fp64 masters (warp-cooperative) + page counts / member counts
//   R6  verified clusters' page ids, R7 their fills
// Exactness: the boundary set S = {c : #{j : approx_j > approx_c + 2m} < take} (m bounds
// |fp32 mirror cosine - exact cosine|) contains every candidate that can reach the exact top-take;
// S is re-scored with the reference's sequential fp64 cosine (vecmath.hpp:54-61) and ranked by
// (sim desc, cluster id asc, live before buffer), so selections are bit-exact.
#include "devmath.cuh"

namespace kvc {

namespace {

using namespace dm;

constexpr int K5T = 512;
constexpr int K5W = K5T / 32;
constexpr int K5_SROWS = 32;   // fp64 rows staged per exact re-score chunk
constexpr int K5_SMAX = 256;   // boundary-set capacity
constexpr int K5_CB = 16;      // mirror rows per warp in flight
constexpr float kMargin3 = 1e-4f;  // |fp32 mirror cosine - exact cosine| bound (as kScoreMargin)

// rank(i) = #entries better than i under (sim desc, key asc) -> order[rank] = i for rank < take
__device__ void rank_select(const double* sim, const long long* key, int n, int take, int* order) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double si = sim[i];
    const long long ki = key[i];
    int r = 0;
    for (int j = 0; j < n; ++j) r += better(sim[j], key[j], si, ki) ? 1 : 0;
    if (r < take) order[r] = i;
  }
  __syncthreads();
}

struct Sel3Smem {
  // static part; the dynamic part holds stage / candidate arrays / owners
  double nq;
  float nq32;
  int nc, nb, ns, nver, degen, lazy_any;
  unsigned long long att;
  int chosen[64];
  int plo[64], plc[64], plpre[65];
  int spo[64], spc[64];  // pl_off / pl_cnt of partitions 0..63 at layer l (R1, speculative)
  int sset[K5_SMAX];
  double ssim[K5_SMAX];
  long long skey[K5_SMAX];
  int snp[K5_SMAX], snbp[K5_SMAX];
  long long snm[K5_SMAX];
  int snb[K5_SMAX];
  unsigned char slz[K5_SMAX];
  int order[64];
  int rank_si[64];  // rank -> S index
  int vers[64], vsi[64];
  int voff[65], ring_off[65], ring_count[64];
  unsigned long long ring_mask[64];  // per window page: tokens K6 attends (not owned by a verified cluster)
  unsigned ring_half[128];           // the same, 32 tokens per word as the ring pass writes them
  int vhash[128];
  int fr_base[64], fr_job[64];  // fetch-on-read: free-stack base / first copy of verified cluster v
  int fr_cnt, fr_jn;
  float red[K5W];
  int redi[32];
};

__host__ __device__ inline size_t sel3_dyn_bytes(int d, int cmax, int parts, int W, int tmax) {
  const int nsel = ((cmax > parts ? cmax : parts) + 1) & ~1;  // even: keeps the float4 arrays aligned
  const int c4 = (cmax + 3) & ~3;
  return static_cast<size_t>(K5_SROWS) * (d + 1) * 8  // stage
         + static_cast<size_t>(d) * 8 + static_cast<size_t>(d) * 4  // qd, qf
         + static_cast<size_t>(nsel) * 8 * 2                         // sim / ckey
         + static_cast<size_t>(nsel) * 8                             // cnr (norms)
         + static_cast<size_t>(c4) * 4                               // approx (float4-padded)
         + static_cast<size_t>(cmax) * 4 + static_cast<size_t>(cmax) // cslot, cbuf
         + static_cast<size_t>(W) * tmax * 4 + 64;                   // owners
}

__global__ void __launch_bounds__(K5T) k_select3(DevTables t, DecodeArgs a, int* work_ctr) {
  extern __shared__ __align__(16) uint8_t dyn[];
  __shared__ Sel3Smem S;
  const int l = blockIdx.x, d = t.d, L = t.L, DS = d + 1;
  const int P = a.n_parts_host;
  const int cmax = t.cmax;
  const int nsel = ((cmax > P ? cmax : P) + 1) & ~1;
  const int c4 = (cmax + 3) & ~3;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = t.W, rpp = t.rpp;
  uint8_t* p = dyn;
  double* stage = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(K5_SROWS) * DS * 8;
  double* qd = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(d) * 8;
  double* sim = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(nsel) * 8;
  long long* ckey = reinterpret_cast<long long*>(p);
  p += static_cast<size_t>(nsel) * 8;
  double* cnr = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(nsel) * 8;
  float* approx = reinterpret_cast<float*>(p);
  p += static_cast<size_t>(c4) * 4;
  float* qf = reinterpret_cast<float*>(p);
  p += static_cast<size_t>(d) * 4;
  int* cslot = reinterpret_cast<int*>(p);
  p += static_cast<size_t>(cmax) * 4;
  int* owners = reinterpret_cast<int*>(p);
  p += static_cast<size_t>(W) * t.tmax * 4;
  uint8_t* cbuf = p;

  // K6 (the attention kernel) may launch now: its prologue overlaps this kernel, and it waits for
  // this grid's completion (griddepcontrol.wait) before reading the work list
  asm volatile("griddepcontrol.launch_dependents;");
  long long kc0 = clock64();
  if (a.k4prof && threadIdx.x == 0) {  // block start on the global timer (launch skew, instrumentation)
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    a.k4prof[l * 16 + 13] = static_cast<long long>(gt);
  }
#define K5MARK(k) if (a.k4prof && tid == 0) { const long long kc1 = clock64(); a.k4prof[l * 16 + (k)] = kc1 - kc0; kc0 = kc1; }
  if (l == 0 && tid == 0) *work_ctr = 0;

  // ------------------------------------------------------------------ R1
  const float* q = (a.q_src ? a.q_src : a.q) + static_cast<int64_t>(l) * d;
  float qx = 0.f;
  if (tid < d) {
    qx = q[tid];
    if (a.q_src) const_cast<float*>(a.q)[static_cast<int64_t>(l) * d + tid] = qx;
    qd[tid] = static_cast<double>(qx);
    qf[tid] = qx;
  }
  {
    const int n_own = W * t.tmax;
    const int* src = t.ring_owner + static_cast<int64_t>(l) * n_own;
    int v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = tid + K5T * j;
      v[j] = i < n_own ? src[i] : -1;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = tid + K5T * j;
      if (i < n_own) owners[i] = v[j];
    }
    for (int i = tid + K5T * 4; i < n_own; i += K5T) owners[i] = src[i];
  }
  if (tid < W && tid < 64) S.ring_count[tid] = t.ring_count[tid];
  if (tid < P && tid < 64) {  // partition list offsets at layer l for the (likely few) partitions
    S.spo[tid] = t.pl_off[static_cast<int64_t>(tid) * L + l];
    S.spc[tid] = t.pl_cnt[static_cast<int64_t>(tid) * L + l];
  }
  if (tid < 128) S.vhash[tid] = -1;
  if (tid < 128) S.ring_half[tid] = 0u;
  if (tid == 0) {
    S.degen = 0;
    S.att = 0;
    S.lazy_any = 0;
    S.fr_cnt = 0;
    S.fr_jn = 0;
  }
  // first chunk of visual representatives (P <= 32 in one chunk) staged with the query loads
  const int p0rows = min(P, K5_SROWS);
  for (int r = warp; r < p0rows; r += K5W) {
    const double* src = t.vrep + static_cast<int64_t>(r) * d;
    for (int i = lane; i < d; i += 32) stage[r * DS + i] = __ldg(src + i);
  }
  {
    float sq = qx * qx;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(kFull, sq, o);
    if (lane == 0) S.red[warp] = sq;
  }
  __syncthreads();
  // exact |q| (vecmath.hpp:35-40) by the last thread while the visual chains run
  if (tid == K5T - 1) {
    double s = 0.0;
#pragma unroll 16
    for (int i = 0; i < d; ++i) s = dadd(s, dmul(qd[i], qd[i]));
    S.nq = __dsqrt_rn(s);
    float s32 = 0.f;
    for (int w = 0; w < K5W; ++w) s32 += S.red[w];
    S.nq32 = sqrtf(s32);
  }
  // ---- visual_topk: exact cosines (sim desc, partition id asc)
  double vdot = 0.0, vnr = 1.0;
  if (tid < p0rows) {
    const double* row = stage + tid * DS;
#pragma unroll 16
    for (int i = 0; i < d; ++i) vdot = dadd(vdot, dmul(qd[i], row[i]));
    vnr = t.vnorm[tid];
  }
  __syncthreads();
  const double nq = S.nq;
  const float nq32 = S.nq32;
  if (tid == 0 && nq < 1e-12) S.degen = 1;
  if (tid < p0rows) {
    if (vnr < 1e-12) S.degen = 1;
    sim[tid] = clamp1(ddiv(vdot, dmul(nq, vnr)));
    ckey[tid] = tid;
  }
  for (int p0 = K5_SROWS; p0 < P; p0 += K5_SROWS) {  // more partitions: further chunks
    const int rows = min(K5_SROWS, P - p0);
    __syncthreads();
    for (int r = warp; r < rows; r += K5W) {
      const double* src = t.vrep + static_cast<int64_t>(p0 + r) * d;
      for (int i = lane; i < d; i += 32) stage[r * DS + i] = __ldg(src + i);
    }
    __syncthreads();
    if (tid < rows) {
      double acc = 0.0;
      const double* row = stage + tid * DS;
#pragma unroll 16
      for (int i = 0; i < d; ++i) acc = dadd(acc, dmul(qd[i], row[i]));
      const double nr = t.vnorm[p0 + tid];
      if (nr < 1e-12) S.degen = 1;
      sim[p0 + tid] = clamp1(ddiv(acc, dmul(nq, nr)));
      ckey[p0 + tid] = p0 + tid;
    }
  }
  __syncthreads();
  const int kv = min(a.k_v, P);
  rank_select(sim, ckey, P, kv, S.chosen);
  if (tid < kv) a.parts[l * a.k_v + tid] = S.chosen[tid];
  if (tid == 0) a.n_parts_sel[l] = kv;
  K5MARK(0)

  // ------------------------------------------------------------------ semantic_topk (+ prefetch)
  const int passes = (a.prefetch && l + 1 < L) ? 2 : 1;
  for (int pass = 0; pass < passes; ++pass) {
    const int layer = l + pass;
    const int ktake = pass == 0 ? a.k_s : a.prefetch_k;
    if (tid == 0) S.nb = 0;
    // R2: list offsets of the chosen partitions at `layer` (pass 0: loaded speculatively in R1)
    if (tid < kv) {
      const int cp = S.chosen[tid];
      if (pass == 0 && cp < 64) {
        S.plo[tid] = S.spo[cp];
        S.plc[tid] = S.spc[cp];
      } else {
        const int64_t pk = static_cast<int64_t>(cp) * L + layer;
        S.plo[tid] = t.pl_off[pk];
        S.plc[tid] = t.pl_cnt[pk];
      }
    }
    __syncthreads();
    if (tid == 0) {
      int acc = 0;
      for (int i = 0; i < kv; ++i) {
        S.plpre[i] = acc;
        acc += S.plc[i];
      }
      S.plpre[kv] = acc;
    }
    __syncthreads();
    const int nlive = min(S.plpre[kv], cmax);
    if (S.plpre[kv] > cmax && tid == 0) set_err(t, DERR_CANDIDATES);
    if (pass == 0) K5MARK(1)
    // R3 + R4 fused per warp: a warp owns 16 candidates per round; lanes 0-15 load their slots,
    // then (in the same round) the slots' lazy flags / norms / ids and, warp-cooperatively, their
    // fp32 mirror rows; approximate cosines follow without a block barrier. Live entries take
    // indices [0, nlive); registered buffers of pending splits are appended after them (ranking
    // is by key, so the list order only has to be deterministic).
    const int nv4 = d >> 2;
    const float4 qv = lane < nv4 ? reinterpret_cast<const float4*>(qf)[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
    auto score16 = [&](int c0, int cend, int my_slot, bool my_buf) {
      float4 rv[K5_CB];
#pragma unroll
      for (int b = 0; b < K5_CB; ++b) {
        const int sb = __shfl_sync(kFull, my_slot, b);
        const bool bb = __shfl_sync(kFull, my_buf ? 1 : 0, b) != 0;
        rv[b] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c0 + b < cend && lane < nv4)
          rv[b] = __ldg(reinterpret_cast<const float4*>((bb ? t.brep32 : t.rep32) + static_cast<int64_t>(sb) * d) + lane);
      }
      float acc[K5_CB];
#pragma unroll
      for (int b = 0; b < K5_CB; ++b) {
        acc[b] = qv.x * rv[b].x;
        acc[b] = fmaf(qv.y, rv[b].y, acc[b]);
        acc[b] = fmaf(qv.z, rv[b].z, acc[b]);
        acc[b] = fmaf(qv.w, rv[b].w, acc[b]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int b = 0; b < K5_CB; ++b) acc[b] += __shfl_xor_sync(kFull, acc[b], o);
      float mine = acc[0];
#pragma unroll
      for (int b = 1; b < K5_CB; ++b)
        if (lane == b) mine = acc[b];
      return mine;
    };
    int my_lz = 0;
    for (int r0 = 0; r0 < nlive; r0 += K5W * K5_CB) {
      const int c0 = r0 + warp * K5_CB;
      const int j = c0 + lane;
      int s = 0;
      double nr = 1.0;
      if (lane < K5_CB && j < nlive) {
        int i = 0;
        while (i + 1 < kv && S.plpre[i + 1] <= j) ++i;
        s = t.pl_pool[S.plo[i] + (j - S.plpre[i])];
        const int lz = t.lazy[s];
        nr = t.rnorm[s];
        const long long cid = t.cid[s];
        cslot[j] = s;
        cbuf[j] = 0;
        cnr[j] = nr;
        ckey[j] = 2LL * cid;
        my_lz += lz;
      }
      if (c0 < nlive) {  // warp-uniform
        const float sc = score16(c0, nlive, s, false);
        if (lane < K5_CB && j < nlive) {
          if (nr < 1e-12) S.degen = 1;
          approx[j] = sc / (nq32 * static_cast<float>(nr));
        }
      }
    }
    int nb_total = 0;
    if (__syncthreads_or(my_lz)) {  // registered buffers of pending splits (rare)
      // buffer entries: positions by a block scan over the live list (order: live index)
      for (int j0 = 0; j0 < nlive; j0 += K5T) {
        const int j = j0 + tid;
        const int lz = j < nlive ? t.lazy[cslot[j]] : 0;
        int x = lz;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFull, x, o);
          if (lane >= o) x += y;
        }
        if (lane == 31) S.redi[warp] = x;
        __syncthreads();
        int before = 0, chunk = 0;
        for (int w = 0; w < K5W; ++w) {
          if (w < warp) before += S.redi[w];
          chunk += S.redi[w];
        }
        if (lz) {
          const int k = nlive + S.nb + before + x - 1;
          const int sl = cslot[j];
          if (k < cmax) {
            cslot[k] = sl;
            cbuf[k] = 1;
            cnr[k] = t.bnorm[sl];
            ckey[k] = 2LL * t.cid[sl] + 1;
          }
        }
        __syncthreads();
        if (tid == 0) S.nb += chunk;
        __syncthreads();
      }
      nb_total = S.nb;
      const int nce = min(nlive + nb_total, cmax);
      for (int c0 = nlive + warp * K5_CB; c0 < nce; c0 += K5W * K5_CB) {
        const int j = c0 + lane;
        const int sl = (lane < K5_CB && j < nce) ? cslot[j] : 0;
        const float sc = score16(c0, nce, sl, true);
        if (lane < K5_CB && j < nce) {
          const double nr = cnr[j];
          if (nr < 1e-12) S.degen = 1;
          approx[j] = sc / (nq32 * static_cast<float>(nr));
        }
      }
    }
    const int nc_all = nlive + nb_total;
    if (nc_all > cmax && tid == 0) set_err(t, DERR_CANDIDATES);
    const int nc = min(nc_all, cmax);
    if (pass == 0 && tid == 0) a.n_cand[l] = nc;
    const int take = min(ktake, nc);
    for (int c = nc + tid; c < c4; c += K5T) approx[c] = -INFINITY;
    if (tid == 0) S.ns = 0;
    __syncthreads();
    if (pass == 0) K5MARK(2)
    // boundary set S: candidates fewer than `take` of which beat approx_c by more than 2m
    auto in_boundary = [&](int c) -> bool {
      if (take >= nc) return true;
      const float thr = approx[c] + 2.f * kMargin3 + 1e-6f;
      const int n4 = (nc + 3) >> 2;
      int cnt = 0;
      const float4* a4 = reinterpret_cast<const float4*>(approx);
      int j = 0;
      for (; j + 4 <= n4 && cnt < take; j += 4) {
        const float4 x0 = a4[j], x1 = a4[j + 1], x2 = a4[j + 2], x3 = a4[j + 3];
        cnt += (x0.x > thr) + (x0.y > thr) + (x0.z > thr) + (x0.w > thr);
        cnt += (x1.x > thr) + (x1.y > thr) + (x1.z > thr) + (x1.w > thr);
        cnt += (x2.x > thr) + (x2.y > thr) + (x2.z > thr) + (x2.w > thr);
        cnt += (x3.x > thr) + (x3.y > thr) + (x3.z > thr) + (x3.w > thr);
      }
      for (; j < n4 && cnt < take; ++j) {
        const float4 x = a4[j];
        cnt += (x.x > thr) + (x.y > thr) + (x.z > thr) + (x.w > thr);
      }
      return cnt < take;
    };
    for (int c = tid; c < nc; c += K5T)
      if (in_boundary(c)) {
        const int k = atomicAdd(&S.ns, 1);
        if (k < K5_SMAX) S.sset[k] = c;
      }
    __syncthreads();
    const int ns_all = S.ns;
    if (pass == 0 && a.k4prof && tid == 0) a.k4prof[l * 16 + 7] = ns_all;
    // R5: exact cosines of S entries [lo, hi) (fp64 masters staged warp-cooperatively) + counts
    // for the tail
    auto rescore = [&](int lo, int hi) {
    for (int r0 = lo; r0 < hi; r0 += K5_SROWS) {
      const int rows = min(K5_SROWS, hi - r0);
      for (int r = warp; r < rows; r += K5W) {
        const int c = S.sset[r0 + r];
        const double* src = (cbuf[c] ? t.brep64 : t.rep64) + static_cast<int64_t>(cslot[c]) * d;
        for (int i = lane; i < d; i += 32) stage[r * DS + i] = __ldg(src + i);
      }
      if (pass == 0 && tid >= K5T - 32) {  // last warp: counts of this chunk's members
        const int r = tid - (K5T - 32);
        if (r < rows) {
          const int s = cslot[S.sset[r0 + r]];
          S.snp[r0 + r] = t.npages[s];
          S.snbp[r0 + r] = t.nbpages[s];
          S.snm[r0 + r] = t.nmem[s];
          S.snb[r0 + r] = t.nbuf[s];
          S.slz[r0 + r] = t.lazy[s];
        }
      }
      if (pass == 0 && r0 == 0 && a.l2pf_pages > 0 && warp == 8 && hi > 0) {
        // HBM is idle while this CTA is latency bound: pull the first pages of the likely
        // selection (S contains every cluster that can be ranked) into L2 for K6; a small
        // per-domain budget keeps the per-SM TMA issue short
        const int per = min(16, (a.l2pf_pages + hi - 1) / hi);
        for (int w = lane; w < hi * per; w += 32) {
          const int s = cslot[S.sset[w / per]];
          const int j = w % per;
          const int np = t.npages[s];
          const int pg = t.pages[static_cast<int64_t>(s) * t.maxp + j];
          if (j < np && pg >= 0 && pg < t.max_pages)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(page_k(t, pg)),
                         "r"(static_cast<uint32_t>(t.page_bytes)) : "memory");
        }
      }
      __syncthreads();
      if (tid < rows) {
        const int c = S.sset[r0 + tid];
        const double* row = stage + tid * DS;
        double acc = 0.0;
#pragma unroll 16
        for (int i = 0; i < d; ++i) acc = dadd(acc, dmul(qd[i], row[i]));  // exact_cos order
        S.ssim[r0 + tid] = clamp1(ddiv(acc, dmul(nq, cnr[c])));
        S.skey[r0 + tid] = ckey[c];
      }
      __syncthreads();
    }
    };
    int ns = min(ns_all, K5_SMAX);
    if (ns_all <= K5_SMAX) {
      rescore(0, ns);
    } else {
      // Near-tie-heavy query (rare): S exceeds its shared-memory capacity. Exact chunked
      // tournament instead of a failure -- the reference ranks any number of ties
      // (index.cpp:210-240): keep the exact top-`take` of the S members seen so far in entries
      // [0, kept), append the next chunk of S members (candidate order) after them, re-score the
      // chunk, rank the union and compact its top-`take` back to the front. The final ranking
      // below then sees exactly the top-`take` of all of S.
      int kept = 0;
      const int room = K5_SMAX - take;  // take <= 64
      for (int cb = 0; cb < nc; cb += room) {
        __syncthreads();
        if (tid == 0) S.ns = kept;
        __syncthreads();
        for (int c = cb + tid; c < min(cb + room, nc); c += K5T)
          if (in_boundary(c)) S.sset[atomicAdd(&S.ns, 1)] = c;
        __syncthreads();
        const int hi = S.ns;
        if (hi == kept) continue;
        rescore(kept, hi);
        rank_select(S.ssim, S.skey, hi, take, S.order);
        const int keep = min(take, hi);
        int csset = 0, csnp = 0, csnbp = 0, csnb = 0;
        double cssim = 0.0;
        long long cskey = 0, csnm = 0;
        unsigned char cslz = 0;
        if (tid < keep) {
          const int si = S.order[tid];
          csset = S.sset[si]; cssim = S.ssim[si]; cskey = S.skey[si];
          csnp = S.snp[si]; csnbp = S.snbp[si]; csnm = S.snm[si]; csnb = S.snb[si]; cslz = S.slz[si];
        }
        __syncthreads();
        if (tid < keep) {
          S.sset[tid] = csset; S.ssim[tid] = cssim; S.skey[tid] = cskey;
          S.snp[tid] = csnp; S.snbp[tid] = csnbp; S.snm[tid] = csnm; S.snb[tid] = csnb; S.slz[tid] = cslz;
        }
        kept = keep;
      }
      __syncthreads();
      ns = kept;
    }
    if (pass == 0) K5MARK(3)
    rank_select(S.ssim, S.skey, ns, take, S.order);
    if (tid < take) {
      const int si = S.order[tid];
      const int c = S.sset[si];
      if (pass == 0) {
        S.rank_si[tid] = si;
        a.ranked_slot[l * a.k_s + tid] = cslot[c];
        a.ranked_buf[l * a.k_s + tid] = cbuf[c];
      } else {
        a.pf_slot[l * a.prefetch_k + tid] = cslot[c];
        a.pf_buf[l * a.prefetch_k + tid] = cbuf[c];
      }
    }
    if (tid == 0) {
      if (pass == 0) a.n_ranked[l] = take;
      else a.n_pf[l] = take;
    }
    if (pass == 0) {  // verified: rank order, first occurrence of each slot (retrieval.cpp:20-26)
      __syncthreads();
      if (warp == 0) {
        const int s0 = lane < take ? cslot[S.sset[S.rank_si[lane]]] : -1;
        const int s1 = lane + 32 < take ? cslot[S.sset[S.rank_si[lane + 32]]] : -1;
        bool k0 = s0 >= 0, k1 = s1 >= 0;
        for (int j = 0; j < take; ++j) {
          const int sj = cslot[S.sset[S.rank_si[j]]];
          if (j < lane && sj == s0) k0 = false;
          if (j < lane + 32 && sj == s1) k1 = false;
        }
        const unsigned m0 = __ballot_sync(kFull, k0), m1 = __ballot_sync(kFull, k1);
        const unsigned lt = (1u << lane) - 1u;
        if (k0) {
          S.vers[__popc(m0 & lt)] = s0;
          S.vsi[__popc(m0 & lt)] = S.rank_si[lane];
        }
        if (k1) {
          S.vers[__popc(m0) + __popc(m1 & lt)] = s1;
          S.vsi[__popc(m0) + __popc(m1 & lt)] = S.rank_si[lane + 32];
        }
        if (lane == 0) {
          S.nver = __popc(m0) + __popc(m1);
          a.n_ver[l] = S.nver;
        }
      }
    }
    __syncthreads();
  }
  if (passes == 1 && tid == 0) a.n_pf[l] = 0;
  if (S.degen && tid == 0) set_err(t, DERR_DEGENERATE);

  // ------------------------------------------------------------------ attended set + work list
  const int nv = S.nver;
  if (tid < nv) {
    const int s = S.vers[tid];
    const int si = S.vsi[tid];
    a.ver_slot[l * a.k_s + tid] = s;
    atomicAdd(&S.att, static_cast<unsigned long long>(S.snm[si] + S.snb[si]));
    if (S.slz[si]) S.lazy_any = 1;  // a pending split: the host settles it before the next step
    int h = (s * 0x9E3779B1u) >> 25;
    while (atomicCAS(&S.vhash[h], -1, s) != -1) h = (h + 1) & 127;
  }
  __syncthreads();
  if (tid == 0) a.flags[l] = S.lazy_any;
  K5MARK(4)
  {  // window ring tokens whose owner is not a verified cluster (retrieval.cpp:107-108), page-major:
     // warp-sized runs of one ring page, so each warp's ballot IS 32 bits of that page's mask
    unsigned long long mine = 0;
    const int P = t.P;
    const int nv_tok = W * rpp * P;  // (P % 32 == 0: launch_select3)
    for (int v0 = 0; v0 < nv_tok; v0 += K5T) {
      const int v = v0 + tid;
      bool keep = false;
      if (v < nv_tok) {
        const int pg = v / P, k = v - pg * P;
        const int rs = pg / rpp, tt = (pg - rs * rpp) * P + k;
        if (tt < S.ring_count[rs]) {
          keep = true;
          const int own = owners[rs * t.tmax + tt];
          if (own >= 0) {
            int h = (own * 0x9E3779B1u) >> 25;
            for (;;) {
              const int x = S.vhash[h];
              if (x == own) {
                keep = false;
                break;
              }
              if (x < 0) break;
              h = (h + 1) & 127;
            }
          }
        }
      }
      const unsigned b = __ballot_sync(kFull, keep);
      if (lane == 0 && v < nv_tok) S.ring_half[v >> 5] = b;
      mine += lane == 0 ? __popc(b) : 0;
    }
    if (lane == 0) atomicAdd(&S.att, mine);
  }
  __syncthreads();
  if (warp == 0) {  // descriptor offsets: verified clusters' pages, then non-empty ring pages
    const int cnt0 = lane < nv ? S.snp[S.vsi[lane]] + S.snbp[S.vsi[lane]] : 0;
    const int cnt1 = lane + 32 < nv ? S.snp[S.vsi[lane + 32]] + S.snbp[S.vsi[lane + 32]] : 0;
    int x0 = cnt0, x1 = cnt1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y0 = __shfl_up_sync(kFull, x0, o), y1 = __shfl_up_sync(kFull, x1, o);
      if (lane >= o) {
        x0 += y0;
        x1 += y1;
      }
    }
    const int tot0 = __shfl_sync(kFull, x0, 31);
    if (lane < nv) S.voff[lane] = x0 - cnt0;
    if (lane + 32 < nv) S.voff[lane + 32] = tot0 + x1 - cnt1;
    const int vtot = tot0 + __shfl_sync(kFull, x1, 31);
    if (lane == 0) S.voff[nv] = vtot;
    const int nrp = min(W * rpp, 64);
    const int hp = t.P / 32;  // 32-bit halves per page
    auto page_mask = [&](int pg) -> unsigned long long {
      return hp == 2 ? (static_cast<unsigned long long>(S.ring_half[2 * pg + 1]) << 32) | S.ring_half[2 * pg]
                     : static_cast<unsigned long long>(S.ring_half[pg]);
    };
    if (lane < nrp) S.ring_mask[lane] = page_mask(lane);
    if (lane + 32 < nrp) S.ring_mask[lane + 32] = page_mask(lane + 32);
    const int r0 = lane < nrp && page_mask(lane) != 0ull ? 1 : 0;
    const int r1 = lane + 32 < nrp && page_mask(lane + 32) != 0ull ? 1 : 0;
    const unsigned rm0 = __ballot_sync(kFull, r0), rm1 = __ballot_sync(kFull, r1);
    const unsigned lt = (1u << lane) - 1u;
    if (lane < nrp) S.ring_off[lane] = vtot + __popc(rm0 & lt);
    if (lane + 32 < nrp) S.ring_off[lane + 32] = vtot + __popc(rm0) + __popc(rm1 & lt);
    int o = vtot + __popc(rm0) + __popc(rm1);
    if (lane == 0) {
      S.ring_off[nrp] = o;
      if (o > a.max_desc) {
        set_err(t, DERR_ITEMS);
        o = a.max_desc;
      }
      a.n_desc[l] = o;
      a.n_items[l] = (o + a.chunk_pages - 1) / a.chunk_pages;
      a.attended[l] = static_cast<int64_t>(S.att);
    }
  }
  __syncthreads();
  K5MARK(5)
  // fetch-on-read: a verified cluster whose member pages are in the host tier (its leading pages,
  // store.cpp:95-130 / context_tiers.cpp) takes fresh HBM pages for all of them (CAS on the free
  // stack, never below fr_reserve; none when that fails: K6 then reads them in place). The work
  // list below names the new pages and k_fetch_read fills them before K6 runs.
  if (a.fr_on) {
    for (int v = warp; v < nv; v += K5W) {
      const int s = S.vers[v];
      const int np = S.snp[S.vsi[v]];
      const int* list = t.pages + static_cast<int64_t>(s) * t.maxp;
      int nh = 0, last = -1;
      for (int k0 = 0; k0 < np; k0 += 32) {
        const unsigned m = __ballot_sync(kFull, k0 + lane < np && is_host_page(t, list[k0 + lane]));
        nh += __popc(m);
        if (m) last = k0 + 31 - __clz(static_cast<int>(m));
      }
      if (lane == 0) {
        int base = -1;
        if (nh > 0 && last + 1 == nh) {
          int top = *reinterpret_cast<volatile int*>(t.free_top);
          while (top - nh >= a.fr_reserve) {
            const int old = atomicCAS(t.free_top, top, top - nh);
            if (old == top) {
              base = top - nh;
              break;
            }
            top = old;
          }
        }
        if (base >= 0) {
          const int j = atomicAdd(&S.fr_cnt, 1);
          const long long cid = t.cid[s];
          a.fr_rec[l * a.fr_max + j] = make_int4(static_cast<int>(cid & 0xffffffffll), static_cast<int>(cid >> 32),
                                                 static_cast<int>(list[0] - t.max_pages), nh);
          S.fr_job[v] = atomicAdd(&S.fr_jn, nh);
        }
        S.fr_base[v] = base;
      }
    }
    __syncthreads();
  }
  // R6 + R7: page ids, then fills
  int4* desc = a.desc + static_cast<int64_t>(l) * a.max_desc;
  const int ndesc = min(S.voff[nv], a.max_desc);
  for (int i0 = 0; i0 < ndesc; i0 += K5T) {
    const int i = i0 + tid;
    int page = -1, isb = 0;
    if (i < ndesc) {
      int lo = 0, hi = nv - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (S.voff[mid] <= i) lo = mid; else hi = mid - 1;
      }
      const int s = S.vers[lo];
      const int k = i - S.voff[lo];
      const int np = S.snp[S.vsi[lo]];
      isb = k >= np;
      page = isb ? t.bpages[static_cast<int64_t>(s) * t.maxbp + (k - np)] : t.pages[static_cast<int64_t>(s) * t.maxp + k];
      if (a.fr_on && !isb && S.fr_base[lo] >= 0 && is_host_page(t, page)) {  // leading: k < its host page count
        const int dst = t.free_stack[S.fr_base[lo] + k];
        a.fr_jobs[static_cast<int64_t>(l) * a.max_desc + S.fr_job[lo] + k] = make_int4(page, dst, s, k);
        desc[i] = make_int4(dst, t.pg_fill[page], -1, -1);
        page = -1;
      }
    }
    if (page >= 0) desc[i] = make_int4(page, t.pg_fill[page] | (isb << 16), -1, -1);
  }
  for (int i = tid; i < W * rpp && i < 64; i += K5T)
    if (S.ring_mask[i] != 0ull && S.ring_off[i] < a.max_desc) {
      const int rs = i / rpp, j = i % rpp;
      const int page = t.ring_pages[(static_cast<int64_t>(l) * W + rs) * rpp + j];
      desc[S.ring_off[i]] = make_int4(page, t.pg_fill[page] | (2 << 16), static_cast<int>(S.ring_mask[i] & 0xffffffffu),
                                      static_cast<int>(S.ring_mask[i] >> 32));
    }
  __syncthreads();
  K5MARK(6)
#undef K5MARK
  if (tid == 0) {
    a.fr_n[l] = a.fr_on ? S.fr_cnt : 0;
    if (a.fr_on) a.fr_nj[l] = S.fr_jn;
    __threadfence();
    a.errw[l] = atomicOr(t.err, 0);
  }
  if (a.n_items[l] == 0)
    for (int i = tid; i < d; i += K5T) {
      a.out[static_cast<int64_t>(l) * d + i] = 0.f;
      for (int r = 0; r < a.peer.n; ++r) a.peer.out[r][static_cast<int64_t>(a.peer.dom_offset + l) * d + i] = 0.f;
    }
  if (a.k4prof && threadIdx.x == 0) {
    a.k4prof[l * 16 + 12] = clock64() - kc0;  // the tail after the last phase mark
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    a.k4prof[l * 16 + 14] = static_cast<long long>(gt);
  }
}

}  // namespace

// Launches K4 v3 when the shape fits (d % 4 == 0, d <= 128, take lists <= 64, W * rpp <= 64);
// returns false otherwise (the caller uses k_score_select2).
bool launch_select3(const DevTables& t, const DecodeArgs& a, cudaStream_t st) {
  if (t.d % 4 != 0 || t.d > 128 || t.W > 64 || t.W * t.rpp > 64 || a.k_s > 64 || a.prefetch_k > 64 || a.k_v > 64 ||
      t.P % 32 != 0)
    return false;
  const size_t smem = sel3_dyn_bytes(t.d, t.cmax, a.n_parts_host, t.W, t.tmax);
  if (smem + sizeof(Sel3Smem) > static_cast<size_t>(device_smem_optin())) return false;
  if (!smem_optin(reinterpret_cast<const void*>(k_select3), smem)) return false;
  k_select3<<<t.L, K5T, smem, st>>>(t, a, a.work_ctr);
  return true;
}

}  // namespace kvc
