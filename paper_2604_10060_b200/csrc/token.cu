// token.cu -- token-level top-k retrieval baseline (retrieve_token_baseline, retrieval.cpp:166-254)
// on the GPU: the ablation the cluster path is measured against (config 5).
//
// Per domain the token pool is every ingested (frame, token) entry in ingest order, stored
// row-major in HBM (keys and values in the kv dtype) with two key norms per row: the exact fp64
// sequential norm of vecmath.hpp:35-40 and an fp32 norm for the approximate scan.
//
//   KT1 k_tok_append   frame rows -> pool, norms
//   KT2 k_tok_approx   fp32 cosine of q with every pool key (HBM scan, one row per thread)
//   KT3 k_tok_select   one CTA per domain: radix-select the budget-th approximate score, classify
//                      rows as surely in / surely out / boundary (|approx - exact| <= m), exact
//                      fp64 cosines for the boundary rows, exact ranking (sim desc, frame asc,
//                      token asc; retrieval.cpp:198-204) of the boundary for the remaining slots,
//                      window rows (retrieval.cpp:240-242), attended list + ledger statistics
//   KT4 k_tok_gather   attended rows -> contiguous staging pages (16-byte vectorised) + the work
//                      list of the split-KV attention kernel (K6), which then runs unchanged.
#include <algorithm>

#include "devmath.cuh"
#include "token.hpp"

namespace kvc {

namespace {

using namespace dm;

constexpr int TT = 1024;         // KT3 threads
constexpr int TB_EQ = 1024;      // tie-group rows ranked in shared memory (more: a second radix select)
// |fp32 scan cosine - exact cosine| bound for d <= 256: the fp32 dot of bf16/fp32 rows with an fp32
// query errs by <= gamma_d * |q||k| (gamma_256 ~ 1.5e-5) and each fp32 norm by <= ~(d/2+2)u; 4e-5
// covers the sum with margin. Clustered keys put many rows near the threshold, so the margin is
// kept tight and the boundary is ranked exactly by a radix select, not by pairwise counting.
constexpr float kTokMargin = 4e-5f;
constexpr int kTokRowsPerBlock = 1024;  // KT2 (bf16, d = 128): rows per block

__device__ __forceinline__ float ldf(const uint8_t* row, int i, int bf16) {
  return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(row)[i]) : reinterpret_cast<const float*>(row)[i];
}

// KT1: grid (T, L), one warp per row
__global__ void k_tok_append(TokArgs a, const uint8_t* fk, const uint8_t* fv, int T, int tmax, int64_t n0) {
  const int t = blockIdx.x, l = blockIdx.y, lane = threadIdx.x;
  const int rb = a.d * a.es;
  const uint8_t* sk = fk + (static_cast<int64_t>(l) * tmax + t) * rb;
  const uint8_t* sv = fv + (static_cast<int64_t>(l) * tmax + t) * rb;
  const int64_t row = static_cast<int64_t>(l) * a.cap + n0 + t;
  uint8_t* dk = a.pk + row * rb;
  uint8_t* dv = a.pv + row * rb;
  for (int o = lane * 16; o < rb; o += 32 * 16) {
    *reinterpret_cast<uint4*>(dk + o) = *reinterpret_cast<const uint4*>(sk + o);
    *reinterpret_cast<uint4*>(dv + o) = *reinterpret_cast<const uint4*>(sv + o);
  }
  float s32 = 0.f;
  for (int i = lane; i < a.d; i += 32) {
    const float x = ldf(sk, i, a.es == 2);
    s32 = fmaf(x, x, s32);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s32 += __shfl_xor_sync(kFull, s32, o);
  if (lane == 0) {
    double s = 0.0;  // vecmath.hpp:35-40, sequential
    for (int i = 0; i < a.d; ++i) {
      const double x = static_cast<double>(ldf(sk, i, a.es == 2));
      s = dadd(s, dmul(x, x));
    }
    a.kn64[row] = __dsqrt_rn(s);
    a.kn32[row] = sqrtf(s32);
  }
}

// KT2: grid (ceil(n / 256), L), 256 threads, 256 rows per block. bf16 d = 128 (256-byte rows):
// a half-warp per row, each lane one 16-byte chunk, so a warp instruction reads two whole rows
// (coalesced 512 B) and every warp keeps 16 rows (8 loads per lane) in flight before the math.
// Other shapes: one row per thread.
__global__ void __launch_bounds__(256) k_tok_approx(TokArgs a, int64_t n) {
  extern __shared__ float qs[];
  const int l = blockIdx.y;
  const float* q = a.q + static_cast<int64_t>(l) * a.d;
  for (int i = threadIdx.x; i < a.d; i += blockDim.x) qs[i] = q[i];
  __shared__ float nq32;
  if (threadIdx.x < 32) {
    float s = 0.f;
    for (int i = threadIdx.x; i < a.d; i += 32) s = fmaf(q[i], q[i], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (threadIdx.x == 0) nq32 = sqrtf(s);
  }
  __syncthreads();
  const int rb = a.d * a.es;
  const uint8_t* base = a.pk + static_cast<int64_t>(l) * a.cap * rb;
  float* outp = a.approx + static_cast<int64_t>(l) * a.cap;
  const float* knp = a.kn32 + static_cast<int64_t>(l) * a.cap;
  if (rb == 256 && a.es == 2) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
    float qv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) qv[u] = qs[hl * 8 + u];
    // a block walks TOK_ROWS_PER_BLOCK / 256 tiles of 256 rows (amortises the query prologue)
    for (int64_t tile = static_cast<int64_t>(blockIdx.x) * (kTokRowsPerBlock / 256);
         tile < static_cast<int64_t>(blockIdx.x + 1) * (kTokRowsPerBlock / 256); ++tile) {
    const int64_t r0 = tile * 256 + warp * 32;  // this warp's 32 rows
    if (r0 >= n) break;  // warp-uniform
#pragma unroll
    for (int g = 0; g < 2; ++g) {  // two groups of 16 rows
      uint4 w[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int64_t i = r0 + g * 16 + p * 2 + half;
        w[p] = i < n ? *reinterpret_cast<const uint4*>(base + i * 256 + hl * 16) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const uint32_t ww[4] = {w[p].x, w[p].y, w[p].z, w[p].w};
        float acc = 0.f;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc = fmaf(__uint_as_float(ww[u] << 16), qv[2 * u], acc);
          acc = fmaf(__uint_as_float(ww[u] & 0xffff0000u), qv[2 * u + 1], acc);
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        const int64_t i = r0 + g * 16 + p * 2 + half;
        if (hl == 0 && i < n) outp[i] = acc / (nq32 * knp[i]);
      }
    }
    }
    return;
  }
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t* row = base + i * rb;
  float acc = 0.f;
  for (int o = 0; o < rb; o += 16) {
    const uint4 w = *reinterpret_cast<const uint4*>(row + o);
    if (a.es == 2) {
      const int e = o / 2;
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc = fmaf(__uint_as_float(ww[k] << 16), qs[e + 2 * k], acc);
        acc = fmaf(__uint_as_float(ww[k] & 0xffff0000u), qs[e + 2 * k + 1], acc);
      }
    } else {
      const int e = o / 4;
      acc = fmaf(__uint_as_float(w.x), qs[e], acc);
      acc = fmaf(__uint_as_float(w.y), qs[e + 1], acc);
      acc = fmaf(__uint_as_float(w.z), qs[e + 2], acc);
      acc = fmaf(__uint_as_float(w.w), qs[e + 3], acc);
    }
  }
  outp[i] = acc / (nq32 * knp[i]);
}

__device__ __forceinline__ uint32_t fkey(float f) {  // order-preserving float -> uint
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

struct SelSmem {
  uint32_t hist[2048];
  int esel[TB_EQ];
  int64_t efr[TB_EQ];
  int etk[TB_EQ];
  int wtot[32];
  double q64[256];
  double nq;
  uint32_t prefix, pmask;
  unsigned long long prefix64, pmask64;
  int kk, nb, nu, ncnt, nattd, ops, host_tok, degen, neq;
};

__device__ __forceinline__ unsigned long long dkey(double x) {  // order-preserving double -> u64
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// KT3: one CTA per domain.
__global__ void __launch_bounds__(TT) k_tok_select(TokArgs a, int64_t n, int budget, int64_t win_lo) {
  __shared__ SelSmem S;
  const int l = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (l == 0 && tid == 0) *a.work_ctr = 0;
  long long kc0 = clock64();
#define TKMARK(k) if (a.prof && tid == 0) { const long long kc1 = clock64(); a.prof[l * 8 + (k)] = kc1 - kc0; kc0 = kc1; }
  const float* ap = a.approx + static_cast<int64_t>(l) * a.cap;
  uint32_t* pick = a.pick + static_cast<int64_t>(l) * a.wcap;
  const int k = static_cast<int>(n < budget ? n : static_cast<int64_t>(budget));
  if (tid < a.d) S.q64[tid] = static_cast<double>(a.q[static_cast<int64_t>(l) * a.d + tid]);
  if (tid == 0) {
    S.prefix = 0;
    S.pmask = 0;
    S.kk = k;
    S.nb = 0;
    S.nu = 0;
    S.ncnt = 0;
    S.degen = 0;
  }
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int i = 0; i < a.d; ++i) s = dadd(s, dmul(S.q64[i], S.q64[i]));
    S.nq = __dsqrt_rn(s);
    if (S.nq < 1e-12) S.degen = 1;
  }
  // ---- radix select: the k-th largest key, 4 digits of 8 bits. Each warp counts into its own
  // shared sub-histogram (match_any aggregates a warp's equal bins; the leader adds without an
  // atomic), so clustered keys do not serialise every warp on one hot bin; the 32 sub-histograms
  // are then summed per bin.
  __shared__ uint16_t whist[TT / 32][256];
  uint32_t vk = 0;
  if (k > 0) {
    for (int p = 0; p < 4; ++p) {
      const int shift = 24 - 8 * p;
      constexpr int nbins = 256;
      const uint32_t pre = S.prefix, pm = S.pmask;
      const int64_t npad = (n + TT - 1) / TT * TT;
      // chunks of 2047 keys per thread keep a warp's 16-bit counts below 65535
      constexpr int64_t kChunk = static_cast<int64_t>(2047) * TT;
      for (int b = tid; b < nbins; b += TT) S.hist[b] = 0;
      for (int64_t c0 = 0; c0 < npad; c0 += kChunk) {
        for (int i = lane; i < nbins; i += 32) whist[warp][i] = 0;
        __syncwarp();
        const int64_t c1 = min(npad, c0 + kChunk);
        // eight keys per thread are loaded before any is counted: the warp-synchronous counting
        // would otherwise expose one memory latency per key
        constexpr int KB = 8;
        for (int64_t i0 = c0 + tid; i0 < c1; i0 += KB * TT) {
          int bins[KB];
#pragma unroll
          for (int j = 0; j < KB; ++j) {
            const int64_t i = i0 + static_cast<int64_t>(j) * TT;
            const bool in = i < c1 && i < n;
            const uint32_t key = in ? fkey(ap[i]) : 0u;
            bins[j] = (in && (key & pm) == pre) ? static_cast<int>((key >> shift) & (nbins - 1)) : -1;
          }
#pragma unroll
          for (int j = 0; j < KB; ++j) {
            if (i0 + static_cast<int64_t>(j) * TT - lane >= c1) break;  // warp-uniform (c1 is a multiple of 32)
            const int bin = bins[j];
            const unsigned same = __match_any_sync(kFull, bin);
            if (bin >= 0 && lane == __ffs(same) - 1) whist[warp][bin] = static_cast<uint16_t>(whist[warp][bin] + __popc(same));
            __syncwarp();
          }
        }
        __syncthreads();
        for (int b = tid; b < nbins; b += TT) {
          uint32_t c = 0;
#pragma unroll 8
          for (int w = 0; w < TT / 32; ++w) c += whist[w][b];
          S.hist[b] += c;
        }
        __syncthreads();
      }
      if (warp == 0) {  // find the bin holding the kk-th largest (scan from the top)
        const int per = nbins / 32;
        int cnt = 0;
        const int hi = nbins - 1 - lane * per;
        for (int b = 0; b < per; ++b) cnt += S.hist[hi - b];
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += y;
        }
        const int kk = S.kk;
        const unsigned hit = __ballot_sync(kFull, incl >= kk);
        const int src = __ffs(hit) - 1;
        if (lane == src) {
          int acc = incl - cnt;
          int b = 0;
          for (; b < per; ++b) {
            const int c = S.hist[hi - b];
            if (acc + c >= kk) break;
            acc += c;
          }
          const uint32_t bin = static_cast<uint32_t>(hi - b);
          S.prefix = pre | (bin << shift);
          S.pmask = pm | (static_cast<uint32_t>(nbins - 1) << shift);
          S.kk = kk - acc;
          S.ncnt = S.hist[bin];  // after the last digit: rows whose key equals v_k
        }
      }
      __syncthreads();
    }
    vk = S.prefix;
  }
  TKMARK(0)
  // v_k as a float (inverse of fkey)
  const float vkf = k > 0 ? __uint_as_float((vk & 0x80000000u) ? (vk & 0x7fffffffu) : ~vk) : INFINITY;
  // ---- classify (valid with ties at v_k too):
  //  * approx >= v_k + 2m (+slack): surely in -- only rows with approx > v_k (fewer than k of them)
  //    can have an exact score at least as high (rows tied at v_k score at most v_k + m exactly);
  //  * approx < v_k - 2m: surely out -- the >= k rows with approx >= v_k all score higher exactly;
  //  * the rest is the boundary, ranked exactly below.
  __syncthreads();
  const float hi_t = vkf + 2.f * kTokMargin + 1e-6f, lo_t = vkf - 2.f * kTokMargin - 1e-6f;
  const int64_t nw = (n + 31) / 32;
  // word-aligned passes: warp w handles words w, w + 32, ...; lane = bit
  // (eight words per warp are loaded before any is classified: one memory latency per batch)
  constexpr int WB = 8;
  for (int64_t wb = 0; wb < nw; wb += WB * (TT / 32)) {
    float xs[WB];
#pragma unroll
    for (int j = 0; j < WB; ++j) {
      const int64_t w = wb + static_cast<int64_t>(j) * (TT / 32) + warp;
      const int64_t i = w * 32 + lane;
      xs[j] = (w < nw && i < n && k > 0) ? ap[i] : -INFINITY;
    }
#pragma unroll
    for (int j = 0; j < WB; ++j) {
      const int64_t w = wb + static_cast<int64_t>(j) * (TT / 32) + warp;
      const int64_t i = w * 32 + lane;
      bool in = false, bd = false;
      if (w < nw && i < n && k > 0) {
        const float x = xs[j];
        if (x >= hi_t) in = true;
        else if (x >= lo_t) bd = true;
      }
      const unsigned bin = __ballot_sync(kFull, in);
      const unsigned bbd = __ballot_sync(kFull, bd);
      if (w < nw) {
        if (lane == 0) pick[w] = bin;
        if (lane == 0 && bin) atomicAdd(&S.nu, __popc(bin));
        if (bbd) {
          int base = 0;
          if (lane == 0) base = atomicAdd(&S.nb, __popc(bbd));
          base = __shfl_sync(kFull, base, 0);
          if (bd) a.bidx[static_cast<int64_t>(l) * a.cap + base + __popc(bbd & ((1u << lane) - 1u))] = static_cast<int>(i);
        }
      }
    }
  }
  for (int64_t w = nw + tid; w < a.wcap; w += TT) pick[w] = 0u;
  __syncthreads();
  TKMARK(1)
  const int nb = S.nb;
  const int r = k - S.nu;  // slots the boundary fills
  int32_t* bidx = a.bidx + static_cast<int64_t>(l) * a.cap;
  double* bsim = a.bsim + static_cast<int64_t>(l) * a.cap;
  long long* btie = a.btie + static_cast<int64_t>(l) * a.cap;  // (frame id, token) order key
  // ---- exact cosines of the boundary rows (vecmath.hpp:54-61, sequential fp64)
  const int rb = a.d * a.es;
  for (int j = tid; j < nb; j += TT) {
    const int i = bidx[j];
    const uint8_t* row = a.pk + (static_cast<int64_t>(l) * a.cap + i) * rb;
    double acc = 0.0;
    for (int e = 0; e < a.d; ++e) acc = dadd(acc, dmul(S.q64[e], static_cast<double>(ldf(row, e, a.es == 2))));
    const double kn = a.kn64[static_cast<int64_t>(l) * a.cap + i];
    if (kn < 1e-12) S.degen = 1;
    bsim[j] = clamp1(ddiv(acc, dmul(S.nq, kn)));
    const int ord = a.fidx[i];
    btie[j] = (static_cast<long long>(a.fid[ord]) << 24) | static_cast<long long>(i - a.fstart[ord]);
  }
  if (tid == 0) {
    S.prefix64 = 0ull;
    S.pmask64 = 0ull;
    S.kk = r;
    S.neq = 0;
  }
  __syncthreads();
  if (r >= nb) {  // every boundary row is in
    for (int j = tid; j < nb; j += TT) atomicOr(&pick[bidx[j] >> 5], 1u << (bidx[j] & 31));
  } else if (r > 0 && nb <= 4096) {
    // small boundary (the common case): rank counting under (sim desc, frame asc, token asc)
    for (int j = tid; j < nb; j += TT) {
      const double sj = bsim[j];
      const long long tj = btie[j];
      int rank = 0;
      for (int u = 0; u < nb && rank < r; ++u) {
        const double su = bsim[u];
        rank += (su > sj || (su == sj && btie[u] < tj)) ? 1 : 0;
      }
      if (rank < r) atomicOr(&pick[bidx[j] >> 5], 1u << (bidx[j] & 31));
    }
  } else if (r > 0) {
    // the r-th largest exact value: radix select over order-preserving 64-bit keys (6 x 11 bits)
    for (int p = 0; p < 6; ++p) {
      const int sh = p < 5 ? 53 - 11 * p : 0;
      const int width = p < 5 ? 11 : 9;
      const int nbins = 1 << width;
      for (int i = tid; i < nbins; i += TT) S.hist[i] = 0;
      __syncthreads();
      const unsigned long long pre = S.prefix64, pm = S.pmask64;
      const int nbp = (nb + TT - 1) / TT * TT;
      for (int j = tid; j < nbp; j += TT) {
        const unsigned long long key = j < nb ? dkey(bsim[j]) : 0ull;
        const int bin = (j < nb && (key & pm) == pre) ? static_cast<int>((key >> sh) & static_cast<unsigned long long>(nbins - 1)) : -1;
        const unsigned same = __match_any_sync(kFull, bin);
        if (bin >= 0 && lane == __ffs(same) - 1) atomicAdd(&S.hist[bin], static_cast<unsigned>(__popc(same)));
      }
      __syncthreads();
      if (warp == 0) {
        const int per = nbins / 32;
        int cnt = 0;
        const int hi = nbins - 1 - lane * per;
        for (int b = 0; b < per; ++b) cnt += S.hist[hi - b];
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += y;
        }
        const int kk = S.kk;
        const unsigned hit = __ballot_sync(kFull, incl >= kk);
        const int src = __ffs(hit) - 1;
        if (lane == src) {
          int acc = incl - cnt;
          int b = 0;
          for (; b < per; ++b) {
            const int c = S.hist[hi - b];
            if (acc + c >= kk) break;
            acc += c;
          }
          S.prefix64 = pre | (static_cast<unsigned long long>(hi - b) << sh);
          S.pmask64 = pm | (static_cast<unsigned long long>(nbins - 1) << sh);
          S.kk = kk - acc;
        }
      }
      __syncthreads();
    }
    // rows above the r-th value are in; of the rows equal to it, the S.kk first by (frame, token)
    const unsigned long long tau = S.prefix64;
    for (int j = tid; j < nb; j += TT) {
      const unsigned long long key = dkey(bsim[j]);
      const int i = bidx[j];
      if (key > tau) {
        atomicOr(&pick[i >> 5], 1u << (i & 31));
      } else if (key == tau) {
        const int e = atomicAdd(&S.neq, 1);
        if (e < TB_EQ) {
          const int ord = a.fidx[i];
          S.esel[e] = i;
          S.efr[e] = a.fid[ord];
          S.etk[e] = i - static_cast<int>(a.fstart[ord]);
        }
      }
    }
    __syncthreads();
    const int need = S.kk;
    if (S.neq <= TB_EQ) {  // rank the tie group in shared memory by (frame, token)
      const int neq = S.neq;
      for (int e = tid; e < neq; e += TT) {
        int rank = 0;
        for (int u = 0; u < neq; ++u)
          rank += (S.efr[u] < S.efr[e] || (S.efr[u] == S.efr[e] && S.etk[u] < S.etk[e])) ? 1 : 0;
        if (rank < need) atomicOr(&pick[S.esel[e] >> 5], 1u << (S.esel[e] & 31));
      }
    } else {
      // a larger tie group (repeated / static frames): the need-th smallest (frame, token) key of
      // the tied rows by a second radix select (keys inverted so the smallest rank first); the
      // keys are unique, so exactly the rows at or below it are taken
      __syncthreads();
      if (tid == 0) {
        S.prefix64 = 0ull;
        S.pmask64 = 0ull;
        S.kk = need;
      }
      __syncthreads();
      for (int p = 0; p < 6; ++p) {
        const int sh = p < 5 ? 53 - 11 * p : 0;
        const int width = p < 5 ? 11 : 9;
        const int nbins = 1 << width;
        for (int i = tid; i < nbins; i += TT) S.hist[i] = 0;
        __syncthreads();
        const unsigned long long pre = S.prefix64, pm = S.pmask64;
        const int nbp = (nb + TT - 1) / TT * TT;
        for (int j = tid; j < nbp; j += TT) {
          const bool tied = j < nb && dkey(bsim[j]) == tau;
          const unsigned long long key = tied ? ~static_cast<unsigned long long>(btie[j]) : 0ull;
          const int bin = (tied && (key & pm) == pre) ? static_cast<int>((key >> sh) & static_cast<unsigned long long>(nbins - 1)) : -1;
          const unsigned same = __match_any_sync(kFull, bin);
          if (bin >= 0 && lane == __ffs(same) - 1) atomicAdd(&S.hist[bin], static_cast<unsigned>(__popc(same)));
        }
        __syncthreads();
        if (warp == 0) {
          const int per = nbins / 32;
          int cnt = 0;
          const int hi = nbins - 1 - lane * per;
          for (int b = 0; b < per; ++b) cnt += S.hist[hi - b];
          int incl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
          }
          const int kk = S.kk;
          const unsigned hit = __ballot_sync(kFull, incl >= kk);
          const int src = __ffs(hit) - 1;
          if (lane == src) {
            int acc = incl - cnt;
            int b = 0;
            for (; b < per; ++b) {
              const int c = S.hist[hi - b];
              if (acc + c >= kk) break;
              acc += c;
            }
            S.prefix64 = pre | (static_cast<unsigned long long>(hi - b) << sh);
            S.pmask64 = pm | (static_cast<unsigned long long>(nbins - 1) << sh);
            S.kk = kk - acc;
          }
        }
        __syncthreads();
      }
      const unsigned long long tau2 = S.prefix64;
      for (int j = tid; j < nb; j += TT)
        if (dkey(bsim[j]) == tau && ~static_cast<unsigned long long>(btie[j]) >= tau2)
          atomicOr(&pick[bidx[j] >> 5], 1u << (bidx[j] & 31));
    }
  }
  __syncthreads();
  TKMARK(2)
  if (S.degen && tid == 0) atomicOr(a.err, 1);
  // ---- window rows + statistics: attended = picked | window; host-side runs over picked rows
  //      of non-window frames (retrieval.cpp:212-231)
  if (tid == 0) {
    S.nattd = 0;
    S.ops = 0;
    S.host_tok = 0;
  }
  __syncthreads();
  // warp per 32-row word, lane = row: coalesced frame ordinals, run starts by shuffles
  int att = 0, ops = 0, htok = 0;
  for (int64_t w = warp; w < nw; w += TT / 32) {
    const int64_t i = w * 32 + lane;
    const bool valid = i < n;
    const uint32_t pw = pick[w];
    const bool pk = valid && ((pw >> lane) & 1u);
    const bool win = valid && i >= win_lo;
    const int ord = valid ? a.fidx[i] : -1;
    const bool host = pk && !win;  // picked row of a non-window frame (retrieval.cpp:212-215)
    // previous row: lane - 1, or the last row of the previous word for lane 0
    int prev_ord = __shfl_up_sync(kFull, ord, 1);
    bool prev_host = __shfl_up_sync(kFull, host, 1);
    if (lane == 0) {
      prev_host = false;
      if (i > 0 && valid) {
        prev_ord = a.fidx[i - 1];
        prev_host = ((pick[w - 1] >> 31) & 1u) && (i - 1 < win_lo);
      }
    }
    const bool start = host && !(prev_host && prev_ord == ord);
    const bool at = pk || win;
    const unsigned bh = __ballot_sync(kFull, host), bs = __ballot_sync(kFull, start), ba = __ballot_sync(kFull, at);
    if (lane == 0) {
      htok += __popc(bh);
      ops += __popc(bs);
      att += __popc(ba);
      a.attw[static_cast<int64_t>(l) * a.wcap + w] = ba;
    }
    if (at) a.frame_hit[ord] = 1;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    att += __shfl_xor_sync(kFull, att, o);
    ops += __shfl_xor_sync(kFull, ops, o);
    htok += __shfl_xor_sync(kFull, htok, o);
  }
  if (lane == 0) {
    atomicAdd(&S.nattd, att);
    atomicAdd(&S.ops, ops);
    atomicAdd(&S.host_tok, htok);
  }
  __syncthreads();
  TKMARK(3)
  if (tid == 0) {
    a.stats[l * 4 + 0] = S.nattd;
    a.stats[l * 4 + 1] = S.ops;
    a.stats[l * 4 + 2] = S.host_tok;
    a.stats[l * 4 + 3] = nb;
  }
  // ---- attended row list in order (block scan over words)
  int base = 0;
  for (int64_t w0 = 0; w0 < nw; w0 += TT) {
    const int64_t w = w0 + tid;
    const uint32_t attw = w < nw ? a.attw[static_cast<int64_t>(l) * a.wcap + w] : 0u;
    const int c = __popc(attw);
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) S.wtot[warp] = x;
    __syncthreads();
    int before = 0, tot = 0;
    for (int u = 0; u < TT / 32; ++u) {
      if (u < warp) before += S.wtot[u];
      tot += S.wtot[u];
    }
    int pos = base + before + x - c;
    for (uint32_t m = attw; m; m &= m - 1) {
      if (pos < a.max_att) a.att_idx[static_cast<int64_t>(l) * a.max_att + pos] = static_cast<int>(w * 32 + __ffs(m) - 1);
      ++pos;
    }
    base += tot;
    __syncthreads();
  }
  TKMARK(4)
#undef TKMARK
}

// KT4: grid (ceil(max_att / 8), L), one warp per attended row; block (0, l) writes the work list.
__global__ void k_tok_gather(TokArgs a, DevTables st, DecodeArgs da) {
  const int l = blockIdx.y;
  const int natt = min(a.stats[l * 4 + 0], a.max_att);
  const int warps = blockDim.x / 32, warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int rb = a.d * a.es;
  const int P = st.P;
  const int pages = (natt + P - 1) / P;
  const int page0 = l * a.pages_per_dom;
  // a half-warp per row, 4 row pairs per warp in flight: 16-byte lane copies of K and V
  const int half = lane >> 4, hl = lane & 15;
  for (int j0 = (blockIdx.x * warps + warp) * 8; j0 < natt; j0 += gridDim.x * warps * 8) {
    uint4 kk[4][2], vv[4][2];
    int dst[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u * 2 + half;
      dst[u] = -1;
      if (j < natt) {
        const int i = a.att_idx[static_cast<int64_t>(l) * a.max_att + j];
        const int64_t row = static_cast<int64_t>(l) * a.cap + i;
        const uint8_t* sk = a.pk + row * rb;
        const uint8_t* sv = a.pv + row * rb;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int o = (hl + 16 * c) * 16;
          if (o < rb) {
            kk[u][c] = *reinterpret_cast<const uint4*>(sk + o);
            vv[u][c] = *reinterpret_cast<const uint4*>(sv + o);
          }
        }
        dst[u] = j;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (dst[u] < 0) continue;
      const int j = dst[u];
      const int pg = page0 + j / P, rr = j % P;
      uint8_t* dk = page_k(st, pg) + static_cast<int64_t>(rr) * rb;
      uint8_t* dv = page_v(st, pg) + static_cast<int64_t>(rr) * rb;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int o = (hl + 16 * c) * 16;
        if (o < rb) {
          *reinterpret_cast<uint4*>(dk + o) = kk[u][c];
          *reinterpret_cast<uint4*>(dv + o) = vv[u][c];
        }
      }
    }
  }
  if (blockIdx.x == 0) {
    int4* desc = da.desc + static_cast<int64_t>(l) * da.max_desc;
    for (int p = threadIdx.x; p < pages && p < da.max_desc; p += blockDim.x)
      desc[p] = make_int4(page0 + p, min(P, natt - p * P), -1, -1);
    if (threadIdx.x == 0) {
      const int nd = min(pages, da.max_desc);
      da.n_desc[l] = nd;
      da.n_items[l] = (nd + da.chunk_pages - 1) / da.chunk_pages;
    }
    if (natt == 0)
      for (int i = threadIdx.x; i < a.d; i += blockDim.x) da.out[static_cast<int64_t>(l) * a.d + i] = 0.f;
  }
}

}  // namespace

int launch_tok_append(const TokArgs& a, const void* fk, const void* fv, int T, int tmax, int64_t n0, cudaStream_t st) {
  k_tok_append<<<dim3(T, a.L), 32, 0, st>>>(a, static_cast<const uint8_t*>(fk), static_cast<const uint8_t*>(fv), T,
                                            tmax, n0);
  return 1;
}

int launch_tok_decode(const TokArgs& a, const DevTables& stage, const DecodeArgs& da, int64_t n, int budget,
                      int64_t win_lo, cudaStream_t st) {
  if (n <= 0) return 0;
  const int64_t per_block = (a.d * a.es == 256 && a.es == 2) ? kTokRowsPerBlock : 256;
  k_tok_approx<<<dim3(static_cast<unsigned>((n + per_block - 1) / per_block), a.L), 256, a.d * 4, st>>>(a, n);
  k_tok_select<<<a.L, TT, 0, st>>>(a, n, budget, win_lo);
  k_tok_gather<<<dim3(static_cast<unsigned>(max(1, (a.max_att + 63) / 64)), a.L), 256, 0, st>>>(a, stage, da);
  // (rows of more than 512 bytes -- d > 128 in fp32 -- are outside the gather's two 16-byte chunks per lane)
  return 3 + launch_attend(stage, da, st);
}

}  // namespace kvc
