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
#include "devmath.cuh"
#include "token.hpp"

namespace kvc {

namespace {

using namespace dm;

constexpr int TT = 1024;         // KT3 threads
constexpr int TB_MAX = 1024;     // boundary capacity per domain (static shared memory)
constexpr float kTokMargin = 1e-4f;  // |fp32 scan cosine - exact cosine| bound (d <= 256)

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

// KT2: grid (ceil(n / 256), L), one row per thread, 16-byte loads of the row
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
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int rb = a.d * a.es;
  const uint8_t* row = a.pk + (static_cast<int64_t>(l) * a.cap + i) * rb;
  float acc = 0.f;
  if (a.es == 2) {
    for (int o = 0; o < rb; o += 16) {
      const uint4 w = *reinterpret_cast<const uint4*>(row + o);
      const int e = o / 2;
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc = fmaf(__uint_as_float(ww[k] << 16), qs[e + 2 * k], acc);
        acc = fmaf(__uint_as_float(ww[k] & 0xffff0000u), qs[e + 2 * k + 1], acc);
      }
    }
  } else {
    for (int o = 0; o < rb; o += 16) {
      const float4 w = *reinterpret_cast<const float4*>(row + o);
      const int e = o / 4;
      acc = fmaf(w.x, qs[e], acc);
      acc = fmaf(w.y, qs[e + 1], acc);
      acc = fmaf(w.z, qs[e + 2], acc);
      acc = fmaf(w.w, qs[e + 3], acc);
    }
  }
  const float kn = a.kn32[static_cast<int64_t>(l) * a.cap + i];
  a.approx[static_cast<int64_t>(l) * a.cap + i] = acc / (nq32 * kn);
}

__device__ __forceinline__ uint32_t fkey(float f) {  // order-preserving float -> uint
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// (sim desc, frame asc, token asc): a better than b
__device__ __forceinline__ bool tok_better(double sa, int64_t fa, int ta, double sb, int64_t fb, int tb) {
  if (sa != sb) return sa > sb;
  if (fa != fb) return fa < fb;
  return ta < tb;
}

struct SelSmem {
  uint32_t hist[2048];
  int bsel[TB_MAX];
  double bsim[TB_MAX];
  int64_t bfr[TB_MAX];
  int btk[TB_MAX];
  int wtot[32];
  double q64[256];
  double nq;
  uint32_t prefix, pmask;
  int kk, nb, nu, ncnt, nattd, ops, host_tok, degen;
};

// KT3: one CTA per domain.
__global__ void __launch_bounds__(TT) k_tok_select(TokArgs a, int64_t n, int budget, int64_t win_lo) {
  __shared__ SelSmem S;
  const int l = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (l == 0 && tid == 0) *a.work_ctr = 0;
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
  // ---- radix select: the k-th largest key (3 digits: 11, 11, 10 bits)
  uint32_t vk = 0;
  if (k > 0) {
    const int shifts[3] = {21, 10, 0};
    const int widths[3] = {11, 11, 10};
    for (int p = 0; p < 3; ++p) {
      const int nbins = 1 << widths[p];
      for (int i = tid; i < nbins; i += TT) S.hist[i] = 0;
      __syncthreads();
      const uint32_t pre = S.prefix, pm = S.pmask;
      for (int64_t i = tid; i < n; i += TT) {
        const uint32_t key = fkey(ap[i]);
        if ((key & pm) == pre) atomicAdd(&S.hist[(key >> shifts[p]) & (nbins - 1)], 1u);
      }
      __syncthreads();
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
          S.prefix = pre | (bin << shifts[p]);
          S.pmask = pm | (static_cast<uint32_t>(nbins - 1) << shifts[p]);
          S.kk = kk - acc;
        }
      }
      __syncthreads();
    }
    vk = S.prefix;
  }
  // v_k as a float (inverse of fkey)
  const float vkf = k > 0 ? __uint_as_float((vk & 0x80000000u) ? (vk & 0x7fffffffu) : ~vk) : INFINITY;
  // ---- classify: A = #(approx >= v_k); ties at v_k put every near-threshold row in the boundary
  {
    int c = 0;
    for (int64_t i = tid; i < n; i += TT) c += ap[i] >= vkf ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
    if (lane == 0) atomicAdd(&S.ncnt, c);
  }
  __syncthreads();
  const bool ties = S.ncnt > k;
  const float hi_t = vkf + 2.f * kTokMargin + 1e-6f, lo_t = vkf - 2.f * kTokMargin - 1e-6f;
  const int64_t nw = (n + 31) / 32;
  // word-aligned passes: warp w handles words w, w + 32, ...; lane = bit
  for (int64_t w0 = 0; w0 < nw; w0 += TT / 32) {
    const int64_t w = w0 + warp;
    const int64_t i = w * 32 + lane;
    bool in = false, bd = false;
    if (w < nw && i < n && k > 0) {
      const float x = ap[i];
      if (!ties && x >= hi_t) in = true;
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
        if (bd) {
          const int pos = base + __popc(bbd & ((1u << lane) - 1u));
          if (pos < TB_MAX) S.bsel[pos] = static_cast<int>(i);
        }
      }
    }
  }
  for (int64_t w = nw + tid; w < a.wcap; w += TT) pick[w] = 0u;
  __syncthreads();
  const int nb = min(S.nb, TB_MAX);
  if (S.nb > TB_MAX && tid == 0) atomicOr(a.err, 1 << 6);
  const int r = k - S.nu;  // slots the boundary fills
  // ---- exact cosines of the boundary rows (vecmath.hpp:54-61, sequential fp64)
  const int rb = a.d * a.es;
  for (int j = tid; j < nb; j += TT) {
    const int i = S.bsel[j];
    const uint8_t* row = a.pk + (static_cast<int64_t>(l) * a.cap + i) * rb;
    double acc = 0.0;
    for (int e = 0; e < a.d; ++e) acc = dadd(acc, dmul(S.q64[e], static_cast<double>(ldf(row, e, a.es == 2))));
    const double kn = a.kn64[static_cast<int64_t>(l) * a.cap + i];
    if (kn < 1e-12) S.degen = 1;
    S.bsim[j] = clamp1(ddiv(acc, dmul(S.nq, kn)));
    const int ord = a.fidx[i];
    S.bfr[j] = a.fid[ord];
    S.btk[j] = i - static_cast<int>(a.fstart[ord]);
  }
  __syncthreads();
  for (int j = tid; j < nb; j += TT) {  // rank counting inside the boundary
    const double sj = S.bsim[j];
    const int64_t fj = S.bfr[j];
    const int tj = S.btk[j];
    int rank = 0;
    for (int u = 0; u < nb; ++u) rank += tok_better(S.bsim[u], S.bfr[u], S.btk[u], sj, fj, tj) ? 1 : 0;
    if (rank < r) {
      const int i = S.bsel[j];
      atomicOr(&pick[i >> 5], 1u << (i & 31));
    }
  }
  __syncthreads();
  if (S.degen && tid == 0) atomicOr(a.err, 1);
  // ---- window rows + statistics: attended = picked | window; host-side runs over picked rows
  //      of non-window frames (retrieval.cpp:212-231)
  if (tid == 0) {
    S.nattd = 0;
    S.ops = 0;
    S.host_tok = 0;
  }
  __syncthreads();
  int att = 0, ops = 0, htok = 0;
  for (int64_t w = tid; w < nw; w += TT) {
    const uint32_t pw = pick[w];
    uint32_t win = 0;
    const int64_t b0 = w * 32;
    if (b0 + 31 >= win_lo) {
      for (int b = 0; b < 32; ++b)
        if (b0 + b >= win_lo && b0 + b < n) win |= 1u << b;
    }
    const uint32_t hostw = pw & ~win;
    htok += __popc(hostw);
    // run starts: bit set and (previous row not host-side or in another frame)
    for (uint32_t m = hostw; m; m &= m - 1) {
      const int b = __ffs(m) - 1;
      const int64_t i = b0 + b;
      bool start = true;
      if (i > 0) {
        const bool prev = (b > 0) ? ((hostw >> (b - 1)) & 1u)
                                  : ((pick[w - 1] >> 31) & 1u) && (i - 1 < win_lo);
        start = !(prev && a.fidx[i - 1] == a.fidx[i]);
      }
      ops += start ? 1 : 0;
    }
    const uint32_t attw = pw | win;
    att += __popc(attw);
    a.attw[static_cast<int64_t>(l) * a.wcap + w] = attw;
    for (uint32_t m = attw; m; m &= m - 1) {
      const int64_t i = b0 + __ffs(m) - 1;
      a.frame_hit[a.fidx[i]] = 1;
    }
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
  for (int j = blockIdx.x * warps + warp; j < natt; j += gridDim.x * warps) {
    const int i = a.att_idx[static_cast<int64_t>(l) * a.max_att + j];
    const int64_t row = static_cast<int64_t>(l) * a.cap + i;
    const uint8_t* sk = a.pk + row * rb;
    const uint8_t* sv = a.pv + row * rb;
    const int pg = page0 + j / P, rr = j % P;
    uint8_t* dk = page_k(st, pg) + static_cast<int64_t>(rr) * rb;
    uint8_t* dv = page_v(st, pg) + static_cast<int64_t>(rr) * rb;
    for (int o = lane * 16; o < rb; o += 32 * 16) {
      *reinterpret_cast<uint4*>(dk + o) = *reinterpret_cast<const uint4*>(sk + o);
      *reinterpret_cast<uint4*>(dv + o) = *reinterpret_cast<const uint4*>(sv + o);
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
  k_tok_approx<<<dim3(static_cast<unsigned>((n + 255) / 256), a.L), 256, a.d * 4, st>>>(a, n);
  k_tok_select<<<a.L, TT, 0, st>>>(a, n, budget, win_lo);
  k_tok_gather<<<dim3(static_cast<unsigned>(max(1, (a.max_att + 63) / 64)), a.L), 256, 0, st>>>(a, stage, da);
  return 3 + launch_attend(stage, da, st);
}

}  // namespace kvc
