// kernels.cu -- sm_100a kernels of the cluster-level KV-cache hot path.
//
//   K0 build_cands     candidate list of the frame's partition per domain (maintainer.cpp:91-109)
//   K1 approx          approximate cosine tile S~[t][c] for every token x candidate (fp32)
//   K2 resolve         exact sequential on_insert per domain: fp64 re-score of the candidates the
//                      approximate tile cannot rule out, Eq. 3/4 update, Eq. 5 test, branch
//                      (maintainer.cpp:88-176); appends K/V into cluster-contiguous pages
//   K4 score_select    visual_topk + semantic_topk (+ prefetch ranking) per domain with exact fp64
//                      cosines and the reference tie-breaks (index.cpp:192-240); attended count and
//                      the attention work list
//   K6 attend          split-KV attention over the selected clusters' pages and the window ring,
//                      TMA bulk copies (cp.async.bulk) into a shared-memory page pipeline, online
//                      softmax, in-kernel combine by the last CTA of each domain
// plus store maintenance (append / gather / free / exact stats / mirrors).
//
// Exactness: every fp64 operation that must reproduce the reference bit-for-bit is written with
// explicit round-to-nearest intrinsics (__dmul_rn/__dadd_rn/__ddiv_rn/__dsqrt_rn) so no FMA
// contraction can occur (the reference builds with -ffp-contract=off, CMakeLists.txt:11-13),
// and every sum runs in the reference's sequential order.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <cstdlib>

#include "kvc_core.hpp"

namespace kvc {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
// RN(a / b) for b > 0 given y = RN(1 / b): a faithful quotient + Markstein's correctly rounded
// step, bit-identical to __ddiv_rn (devmath.cuh dm::div_rcp; kvc_debug_div_check)
__device__ __forceinline__ double div_rcp(double a, double b, double y) {
  const double q1 = __dmul_rn(a, y);
  const double r1 = __fma_rn(-q1, b, a);
  const double q2 = __fma_rn(r1, y, q1);
  const double r2 = __fma_rn(-q2, b, a);
  return __fma_rn(r2, y, q2);
}
__device__ __forceinline__ double clamp1(double x) { return x < -1.0 ? -1.0 : (x > 1.0 ? 1.0 : x); }

__device__ __forceinline__ float ld_kv(const void* base, int64_t i, int bf16) {
  if (bf16) return __bfloat162float(static_cast<const __nv_bfloat16*>(base)[i]);
  return static_cast<const float*>(base)[i];
}

__device__ __forceinline__ void set_err(const DevTables& t, int bit) { atomicOr(t.err, bit); }

// (sim desc, key asc) "a better than b"
__device__ __forceinline__ bool better(double sa, long long ka, double sb, long long kb) {
  return sa > sb || (sa == sb && ka < kb);
}

// Warp arg-best over (sim, key, payload).
__device__ __forceinline__ void warp_best(double& s, long long& k, int& p) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double so = __shfl_xor_sync(kFull, s, o);
    long long ko = __shfl_xor_sync(kFull, k, o);
    int po = __shfl_xor_sync(kFull, p, o);
    if (better(so, ko, s, k)) {
      s = so;
      k = ko;
      p = po;
    }
  }
}

// One warp appends one K/V row (kv dtype) to a slot's member or buffer page list.
__device__ bool warp_append(const DevTables& t, int slot, bool to_buf, const uint8_t* src_k,
                            const uint8_t* src_v) {
  const int lane = threadIdx.x & 31;
  int page = -1, row = -1;
  if (lane == 0) {
    int* np = to_buf ? &t.nbpages[slot] : &t.npages[slot];
    int* list = to_buf ? t.bpages + static_cast<int64_t>(slot) * t.maxbp
                       : t.pages + static_cast<int64_t>(slot) * t.maxp;
    const int cap = to_buf ? t.maxbp : t.maxp;
    const int n = *np;
    page = n > (to_buf ? 0 : t.seal[slot]) ? list[n - 1] : -1;  // sealed pages take no rows
    if (page < 0 || t.pg_fill[page] >= t.P) {
      if (n >= cap) {
        set_err(t, DERR_CLUSTER_PAGES);
        page = -1;
      } else {
        const int top = atomicSub(t.free_top, 1) - 1;
        if (top < 0) {
          atomicAdd(t.free_top, 1);
          set_err(t, DERR_PAGES);
          page = -1;
        } else {
          page = t.free_stack[top];
          list[n] = page;
          *np = n + 1;
          t.pg_fill[page] = 0;
        }
      }
    }
    if (page >= 0) row = t.pg_fill[page]++;
  }
  page = __shfl_sync(kFull, page, 0);
  row = __shfl_sync(kFull, row, 0);
  if (page < 0) return false;
  const int rb = t.d * t.es;
  uint8_t* dk = page_k(t, page) + static_cast<int64_t>(row) * rb;
  uint8_t* dv = page_v(t, page) + static_cast<int64_t>(row) * rb;
  for (int o = lane * 16; o < rb; o += 32 * 16) {
    *reinterpret_cast<uint4*>(dk + o) = *reinterpret_cast<const uint4*>(src_k + o);
    *reinterpret_cast<uint4*>(dv + o) = *reinterpret_cast<const uint4*>(src_v + o);
  }
  return true;
}

// ============================================================================ K0
__global__ void k_build_cands(DevTables t, IngestArgs a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (a dependent of the ring write)
  const int dom = a.active[blockIdx.x];
  if (a.my_events && blockIdx.x == 0 && threadIdx.x == 0) *a.my_events = 0;
  __shared__ int cnt_s;
  if (threadIdx.x == 0) cnt_s = 0;
  __syncthreads();
  const int64_t key = static_cast<int64_t>(a.pid) * t.L + dom;
  const int off = t.pl_off[key], cnt = t.pl_cnt[key];
  int32_t* cs = a.cand_slot + static_cast<int64_t>(dom) * t.cmax;
  uint8_t* cb = a.cand_buf + static_cast<int64_t>(dom) * t.cmax;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const int s = t.pl_pool[off + i];
    const int k = atomicAdd(&cnt_s, t.lazy[s] ? 2 : 1);
    if (k + (t.lazy[s] ? 2 : 1) > t.cmax) {
      set_err(t, DERR_CANDIDATES);
      continue;
    }
    cs[k] = s;
    cb[k] = 0;
    if (t.lazy[s]) {
      cs[k + 1] = s;
      cb[k + 1] = 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) a.cand_n[dom] = min(cnt_s, t.cmax);
}

// ============================================================================ K1
// S~[t][c] = <k_t, r32_c> / (|k_t| |r_c|) in fp32 (CUDA cores). |S~ - S| is bounded by a few
// 1e-6 for unit-scale data; the resolve kernel uses margin = 1e-4.
constexpr int AT = 32;  // tokens per CTA
constexpr int AC = 64;  // candidates per tile
__global__ void __launch_bounds__(256) k_approx(DevTables t, IngestArgs a) {
  extern __shared__ float sm[];
  const int d = t.d, dp = d + 1;
  float* kt = sm;                  // [AT][d+1]
  float* rt = kt + AT * dp;        // [AC][d+1]
  float* ink = rt + AC * dp;       // [AT]
  float* inr = ink + AT;           // [AC]
  const int dom = a.active[blockIdx.y];
  const int t0 = blockIdx.x * AT;
  if (t0 >= a.T) return;
  const int n = a.cand_n[dom];
  const int nt = min(AT, a.T - t0);
  const void* fk = a.fk;
  for (int i = threadIdx.x; i < AT * d; i += blockDim.x) {
    const int r = i / d, c = i % d;
    kt[r * dp + c] = r < nt ? ld_kv(fk, (static_cast<int64_t>(dom) * t.tmax + t0 + r) * d + c, t.kv_bf16) : 0.f;
  }
  __syncthreads();
  if (threadIdx.x < AT) {
    float s = 0.f;
    for (int c = 0; c < d; ++c) s += kt[threadIdx.x * dp + c] * kt[threadIdx.x * dp + c];
    ink[threadIdx.x] = s > 0.f ? rsqrtf(s) : 0.f;
  }
  const int32_t* cs = a.cand_slot + static_cast<int64_t>(dom) * t.cmax;
  const uint8_t* cb = a.cand_buf + static_cast<int64_t>(dom) * t.cmax;
  float* out = a.approx + (static_cast<int64_t>(dom) * t.tmax + t0) * t.cmax;
  const int tp = threadIdx.x / 16, cq = threadIdx.x % 16;
  for (int c0 = 0; c0 < n; c0 += AC) {
    __syncthreads();
    for (int i = threadIdx.x; i < AC * d; i += blockDim.x) {
      const int r = i / d, c = i % d;
      float v = 0.f;
      if (c0 + r < n) {
        const int s = cs[c0 + r];
        v = cb[c0 + r] ? t.brep32[static_cast<int64_t>(s) * d + c] : t.rep32[static_cast<int64_t>(s) * d + c];
      }
      rt[r * dp + c] = v;
    }
    if (threadIdx.x < AC) {
      float nr = 0.f;
      if (c0 + threadIdx.x < n) {
        const int s = cs[c0 + threadIdx.x];
        nr = static_cast<float>(cb[c0 + threadIdx.x] ? t.bnorm[s] : t.rnorm[s]);
      }
      inr[threadIdx.x] = nr > 0.f ? 1.f / nr : 0.f;
    }
    __syncthreads();
    float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    const float* k0 = kt + (2 * tp) * dp;
    const float* k1 = k0 + dp;
    for (int c = 0; c < d; ++c) {
      const float x0 = k0[c], x1 = k1[c];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float y = rt[(4 * cq + j) * dp + c];
        acc[0][j] = fmaf(x0, y, acc[0][j]);
        acc[1][j] = fmaf(x1, y, acc[1][j]);
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int tt = 2 * tp + i, cc = c0 + 4 * cq + j;
        if (tt < nt && cc < n) out[static_cast<int64_t>(tt) * t.cmax + cc] = acc[i][j] * ink[tt] * inr[4 * cq + j];
      }
  }
}

// ============================================================================ K1b
// Per (domain, token): the TOPM best approximate candidates, the (TOPM+1)-th value, and the
// EXACT cosine of each of those TOPM candidates against the launch-time representative -- valid
// for as long as the candidate stays untouched, so the sequential resolve rarely needs a
// global-memory chain. One warp per token.
__global__ void __launch_bounds__(256) k_topm(DevTables t, IngestArgs a) {
  extern __shared__ float rowsm[];  // [8 warps][cmax]
  const int dom = a.active[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tt = blockIdx.x * 8 + warp;
  if (tt >= a.T || tt < a.cursor[dom]) return;
  const int n = a.cand_n[dom];
  const int d = t.d;
  float* row = rowsm + warp * t.cmax;
  const float* src = a.approx + (static_cast<int64_t>(dom) * t.tmax + tt) * t.cmax;
  for (int c = lane; c < n; c += 32) row[c] = src[c];
  __syncwarp();
  const int64_t o = (static_cast<int64_t>(dom) * t.tmax + tt);
  int my_c = -1;  // lane r < TOPM keeps the r-th candidate
  for (int r = 0; r <= TOPM; ++r) {
    float bv = -INFINITY;
    int bi = -1;
    for (int c = lane; c < n; c += 32)
      if (row[c] > bv || (row[c] == bv && bi >= 0 && c < bi)) {
        bv = row[c];
        bi = c;
      }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float ov = __shfl_xor_sync(kFull, bv, off);
      const int oi = __shfl_xor_sync(kFull, bi, off);
      if (ov > bv || (ov == bv && oi >= 0 && (bi < 0 || oi < bi))) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == r) my_c = bi;
    if (lane == 0) {
      if (r < TOPM) {
        a.topm_idx[o * TOPM + r] = static_cast<int16_t>(bi);
        a.topm_val[o * TOPM + r] = bi >= 0 ? bv : -INFINITY;
      } else {
        a.topm_next[o] = bi >= 0 ? bv : -INFINITY;
      }
    }
    if (bi >= 0 && lane == (bi & 31)) row[bi] = -INFINITY;
    __syncwarp();
  }
  // exact cosines: lanes 0..TOPM-1 one candidate each, lane TOPM the key norm
  const int64_t kbase = o * d;
  double acc = 0.0, nr = 1.0;
  if (lane < TOPM && my_c >= 0) {
    const int s = a.cand_slot[static_cast<int64_t>(dom) * t.cmax + my_c];
    const bool ib = a.cand_buf[static_cast<int64_t>(dom) * t.cmax + my_c];
    const double* rp = (ib ? t.brep64 : t.rep64) + static_cast<int64_t>(s) * d;
    nr = ib ? t.bnorm[s] : t.rnorm[s];
#pragma unroll 16
    for (int i = 0; i < d; ++i) acc = dadd(acc, dmul(static_cast<double>(ld_kv(a.fk, kbase + i, t.kv_bf16)), rp[i]));
  } else if (lane == TOPM) {
#pragma unroll 16
    for (int i = 0; i < d; ++i) {
      const double x = static_cast<double>(ld_kv(a.fk, kbase + i, t.kv_bf16));
      acc = dadd(acc, dmul(x, x));
    }
    acc = __dsqrt_rn(acc);
  }
  const double nk = __shfl_sync(kFull, acc, TOPM);
  if (lane < TOPM) a.topm_exact[o * TOPM + lane] = my_c >= 0 ? clamp1(ddiv(acc, dmul(nk, nr))) : -3.0;
}

// ============================================================================ K2
// One warp per domain: the sequential on_insert chain of the frame (maintainer.cpp:88-176),
// exact in fp64. Per token t:
//   argmax(t) over exact cosines (precomputed for untouched top-M candidates by K1b, computed
//   in the previous chain phase for clusters touched earlier in this launch),
//   Eq. 3/4 update of the winner into pending shared buffers (elementwise),
//   ONE chain phase in which each lane runs a d-long sequential fp64 sum out of shared memory:
//   sq_dist(k_t, r') (vecmath.hpp:42-51), |r'|, |buf'| for token t and the exact dots of token
//   t+1 against every touched candidate (with the winner's pending state),
//   Eq. 5 decision for t and commit; K/V rows are copied later by K3 (off the chain).
// Winner state lives in shared memory (HOT entries); pages come from a per-domain pool.
constexpr int HOT = 32;
constexpr int RELMAX = 96;
constexpr int TLMAX = 96;
constexpr int SPECIAL_LANES = 3;
constexpr uint8_t EV_CHAIN = 0, EV_PEND = 1, EV_FRESH = 2, EV_PRE = 3, EV_SLOW = 4, EV_DEAD = 0xff;

struct ResolveShared {
  int hslot[HOT], hcl[HOT], hcb[HOT];  // slot, its live / buffer candidate index (-1 none)
  double hrn[HOT], hbn[HOT], hvar[HOT];
  long long hstat[HOT], hnmem[HOT];
  int hnbuf[HOT], hnp[HOT], hlast[HOT], hfill[HOT], hbnp[HOT], hblast[HOT], hbfill[HOT];
  uint8_t hlazy[HOT], hresid[HOT], hdirty[HOT];
  int nhot;
  int tl[TLMAX];  // touched candidate indices
  int ntl;
  int e_a[RELMAX], e_b[RELMAX];  // chain operands as offsets (doubles) into the shared block
  const double* e_gptr[RELMAX];  // global representative (EV_SLOW)
  double e_nr[RELMAX], e_dot[RELMAX];
  long long e_key[RELMAX];
  int e_cand[RELMAX];
  uint8_t e_var[RELMAX];
  int ne;
  int sel[32];  // chain phase: entry index per lane
  int pool[POOL];
  int npool;
};

// Shared row arrays use a padded stride so rows of different arrays start in different banks
// (lanes of one chain phase read several arrays at the same index).
__host__ __device__ inline int padded(int d) { return d + 2; }

__device__ void hot_writeback(const DevTables& t, ResolveShared& S, const double* hrep,
                              const double* hbrep, int h) {
  if (!S.hdirty[h]) return;
  const int lane = threadIdx.x & 31, d = t.d, DS = padded(d);
  const int64_t s = S.hslot[h];
  for (int i = lane; i < d; i += 32) {
    const double r = hrep[h * DS + i];
    t.rep64[s * d + i] = r;
    t.rep32[s * d + i] = static_cast<float>(r);
    if (S.hnbuf[h] > 0) {
      const double b = hbrep[h * DS + i];
      t.brep64[s * d + i] = b;
      t.brep32[s * d + i] = static_cast<float>(b);
    }
  }
  if (lane == 0) {
    t.rnorm[s] = S.hrn[h];
    t.bnorm[s] = S.hbn[h];
    t.var[s] = S.hvar[h];
    t.stat[s] = S.hstat[h];
    t.nmem[s] = S.hnmem[h];
    t.nbuf[s] = S.hnbuf[h];
    t.lazy[s] = S.hlazy[h];
    t.npages[s] = S.hnp[h];
    t.nbpages[s] = S.hbnp[h];
    if (S.hlast[h] >= 0) t.pg_fill[S.hlast[h]] = S.hfill[h];
    if (S.hblast[h] >= 0) t.pg_fill[S.hblast[h]] = S.hbfill[h];
  }
}

// Loads a slot into the next hot entry (caller guarantees room). cl/cb: its candidate indices.
__device__ int hot_load(const DevTables& t, ResolveShared& S, double* hrep, double* hbrep, int slot,
                        int cl, int cb) {
  const int lane = threadIdx.x & 31, d = t.d, DS = padded(d);
  const int h = S.nhot;
  __syncwarp();
  for (int i = lane; i < d; i += 32) {
    hrep[h * DS + i] = t.rep64[static_cast<int64_t>(slot) * d + i];
    hbrep[h * DS + i] = t.brep64[static_cast<int64_t>(slot) * d + i];
  }
  if (lane == 0) {
    S.hslot[h] = slot;
    S.hcl[h] = cl;
    S.hcb[h] = cb;
    S.hrn[h] = t.rnorm[slot];
    S.hbn[h] = t.bnorm[slot];
    S.hvar[h] = t.var[slot];
    S.hstat[h] = t.stat[slot];
    S.hnmem[h] = t.nmem[slot];
    S.hnbuf[h] = t.nbuf[slot];
    S.hlazy[h] = t.lazy[slot];
    S.hresid[h] = t.resid[slot];
    S.hdirty[h] = 0;
    const int np = t.npages[slot], nbp = t.nbpages[slot];
    S.hnp[h] = np;
    S.hlast[h] = np > t.seal[slot] ? t.pages[static_cast<int64_t>(slot) * t.maxp + np - 1] : -1;
    S.hfill[h] = S.hlast[h] >= 0 ? t.pg_fill[S.hlast[h]] : t.P;
    S.hbnp[h] = nbp;
    S.hblast[h] = nbp > 0 ? t.bpages[static_cast<int64_t>(slot) * t.maxbp + nbp - 1] : -1;
    S.hbfill[h] = S.hblast[h] >= 0 ? t.pg_fill[S.hblast[h]] : t.P;
    S.nhot = h + 1;
  }
  __syncwarp();
  return h;
}

// Reserves the next row of a hot slot's member / buffer page list (lane 0 only).
__device__ void hot_reserve_row(const DevTables& t, ResolveShared& S, int h, bool to_buf, int& page,
                                int& row) {
  page = -1;
  row = -1;
  int& np = to_buf ? S.hbnp[h] : S.hnp[h];
  int& last = to_buf ? S.hblast[h] : S.hlast[h];
  int& fill = to_buf ? S.hbfill[h] : S.hfill[h];
  if (fill >= t.P || last < 0) {
    const int cap = to_buf ? t.maxbp : t.maxp;
    if (np >= cap) {
      set_err(t, DERR_CLUSTER_PAGES);
      return;
    }
    if (S.npool == 0) {  // refill from the shared free stack (pops only during resolve)
      const int top = atomicSub(t.free_top, POOL);
      const int got = max(0, min(POOL, top));
      if (got < POOL) atomicAdd(t.free_top, POOL - got);
      for (int i = 0; i < got; ++i) S.pool[i] = t.free_stack[top - 1 - i];
      S.npool = got;
    }
    if (S.npool == 0) {
      set_err(t, DERR_PAGES);
      return;
    }
    const int pg = S.pool[--S.npool];
    if (last >= 0) t.pg_fill[last] = t.P;
    int* list = to_buf ? t.bpages + static_cast<int64_t>(S.hslot[h]) * t.maxbp
                       : t.pages + static_cast<int64_t>(S.hslot[h]) * t.maxp;
    list[np] = pg;
    np += 1;
    last = pg;
    fill = 0;
  }
  page = last;
  row = fill++;
}

__global__ void __launch_bounds__(32) k_resolve(DevTables t, IngestArgs a) {
  extern __shared__ __align__(16) uint8_t smraw[];
  __shared__ ResolveShared S;
  const int d = t.d, cmax = t.cmax, lane = threadIdx.x;
  const int DS = padded(d);               // padded row stride (doubles)
  double* sd = reinterpret_cast<double*>(smraw);
  double* hrep = sd;                     // [HOT][DS]
  double* hbrep = hrep + HOT * DS;       // [HOT][DS]
  double* kd = hbrep + HOT * DS;         // [3][DS] key ring: rows t, t+1, t+2 (slot = t % 3)
  double* nrep = kd + 3 * DS;            // [DS] pending r'
  double* nbrep = nrep + DS;             // [DS] pending buffer mean
  double* diff = nbrep + DS;             // [DS] k_t - r'
  double* nk = diff + DS;                // [tmax]
  double* tm_exact = nk + t.tmax;        // [tmax][TOPM] staged K1b outputs
  float* tm_val = reinterpret_cast<float*>(tm_exact + static_cast<int64_t>(t.tmax) * TOPM);  // [tmax][TOPM]
  float* tm_next = tm_val + t.tmax * TOPM;                                                    // [tmax]
  int16_t* tm_idx = reinterpret_cast<int16_t*>(tm_next + t.tmax);                            // [tmax][TOPM]
  long long* ckey = reinterpret_cast<long long*>(  // [cmax] CandidateRef order key
      (reinterpret_cast<uintptr_t>(tm_idx + t.tmax * TOPM) + 15) & ~static_cast<uintptr_t>(15));
  int* cslot = reinterpret_cast<int*>(ckey + cmax);              // [cmax]
  int8_t* chot = reinterpret_cast<int8_t*>(cslot + cmax);        // [cmax] hot index or -1
  uint8_t* cbuf = reinterpret_cast<uint8_t*>(chot + cmax);       // [cmax]
  uint8_t* touched = cbuf + cmax;                                  // [cmax]
  const int OFF_HREP = 0, OFF_HBREP = HOT * DS, OFF_KD = 2 * HOT * DS, OFF_NREP = OFF_KD + 3 * DS,
            OFF_NBREP = OFF_NREP + DS, OFF_DIFF = OFF_NBREP + DS;

  const int dom = a.active[blockIdx.x];
  const int T = a.T;
  const int cur = a.cursor[dom];
  if (a.prev_events && *a.prev_events) return;  // skipped speculative round: no writes
  // some decision of this launch was decided by the CandidateRef key (an exact tie of the best
  // fp64 cosines): the wave engine then requires its speculative children in their final order
  bool any_tie = false;
  int n = a.cand_n[dom];
  for (int c = lane; c < n; c += 32) {
    const int s = a.cand_slot[static_cast<int64_t>(dom) * cmax + c];
    const uint8_t b = a.cand_buf[static_cast<int64_t>(dom) * cmax + c];
    cslot[c] = s;
    cbuf[c] = b;
    ckey[c] = 2LL * t.cid[s] + b;
    touched[c] = 0;
    chot[c] = -1;
  }
  if (lane == 0) {
    S.nhot = 0;
    S.ntl = 0;
    S.npool = a.dom_pool_n[dom];
    a.stop_t[dom] = T;
    a.stop_kind[dom] = EV_NONE;
    a.stop_slot[dom] = -1;
  }
  if (lane < POOL) S.pool[lane] = a.dom_pool[dom * POOL + lane];
  for (int tt = cur + lane; tt < T; tt += 32) {  // |k_t| (vecmath.hpp:35-40), 16-byte key loads
    double s = 0.0;
    const int64_t base = (static_cast<int64_t>(dom) * t.tmax + tt) * d;
    if (t.kv_bf16 && (d & 7) == 0) {
      const uint4* row = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.fk) + base);
      for (int i = 0; i < d / 8; i += 4) {
        uint4 w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = i + k < d / 8 ? row[i + k] : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (i + k >= d / 8) break;
          const uint32_t u4[4] = {w[k].x, w[k].y, w[k].z, w[k].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double lo = static_cast<double>(__uint_as_float(u4[q] << 16));
            const double hi = static_cast<double>(__uint_as_float(u4[q] & 0xffff0000u));
            s = dadd(s, dmul(lo, lo));
            s = dadd(s, dmul(hi, hi));
          }
        }
      }
    } else {
#pragma unroll 8
      for (int i = 0; i < d; ++i) {
        const double x = static_cast<double>(ld_kv(a.fk, base + i, t.kv_bf16));
        s = dadd(s, dmul(x, x));
      }
    }
    nk[tt] = __dsqrt_rn(s);
    a.ev_page[static_cast<int64_t>(dom) * t.tmax + tt] = -1;
  }
  {  // stage the per-token top-M lists of this launch's tokens (one latency instead of per token)
    const int64_t o0 = (static_cast<int64_t>(dom) * t.tmax + cur) * TOPM;
    const int cnt = (T - cur) * TOPM;
    for (int i = lane; i < cnt; i += 32) {
      tm_idx[cur * TOPM + i] = a.topm_idx[o0 + i];
      tm_val[cur * TOPM + i] = a.topm_val[o0 + i];
      tm_exact[cur * TOPM + i] = a.topm_exact[o0 + i];
    }
    for (int tt = cur + lane; tt < T; tt += 32) tm_next[tt] = a.topm_next[static_cast<int64_t>(dom) * t.tmax + tt];
  }
  __syncwarp();
  int n_exact = 0;
  if (cur >= T) goto done;
  if (n == 0) {  // maintainer.cpp:93-94: empty partition layer -> the host seeds a cluster
    if (lane == 0) {
      a.stop_t[dom] = cur;
      a.stop_kind[dom] = EV_SEED;
    }
    goto done;
  }
  {
    bool bad = false;  // a degenerate representative throws at its first cosine (vecmath.hpp:59)
    for (int c = lane; c < n; c += 32) {
      const int s = cslot[c];
      if ((cbuf[c] ? t.bnorm[s] : t.rnorm[s]) < 1e-12) bad = true;
    }
    if (__any_sync(kFull, bad)) {
      if (lane == 0) {
        set_err(t, DERR_DEGENERATE);
        a.stop_t[dom] = cur;
      }
      goto done;
    }
  }
  {
    const float margin2 = 2.f * a.margin;
    // key ring: kd[(t % 3) * d] holds token t; rows cur and cur+1 now, t+2 prefetched in iteration t
    for (int r = 0; r < 2 && cur + r < T; ++r)
      for (int i = lane; i < d; i += 32)
        kd[((cur + r) % 3) * DS + i] =
            static_cast<double>(ld_kv(a.fk, (static_cast<int64_t>(dom) * t.tmax + cur + r) * d + i, t.kv_bf16));
    if (lane == 0) S.ne = 0;
    __syncwarp();

    auto add = [&](int c, uint8_t var, int oa, int ob, const double* g, double nr, long long key, double dot) {
      const int k = atomicAdd(&S.ne, 1);
      if (k < RELMAX) {
        S.e_cand[k] = c;
        S.e_var[k] = var;
        S.e_a[k] = oa;
        S.e_b[k] = ob;
        S.e_gptr[k] = g;
        S.e_nr[k] = nr;
        S.e_key[k] = key;
        S.e_dot[k] = dot;
      } else {
        set_err(t, DERR_CANDIDATES);
      }
    };
    auto flush_hot = [&]() {
      for (int i = 0; i < S.nhot; ++i) hot_writeback(t, S, hrep, hbrep, i);
      for (int c = lane; c < n; c += 32) chot[c] = -1;
      __syncwarp();
      if (lane == 0) S.nhot = 0;
      __syncwarp();
    };

    // Entries of token tn. w: the winner of tn-1 (slot, hot index) whose statistics are pending.
    auto build_entries = [&](int tn, int w_slot, bool w_isbuf, bool fresh_possible, int w_h) {
      const int64_t o = static_cast<int64_t>(dom) * t.tmax + tn;
      if (lane == 0) S.ne = 0;
      __syncwarp();
      // (a) touched candidates: exact chain on their current (hot or pending) state
      for (int i = lane; i < S.ntl; i += 32) {
        const int c = S.tl[i];
        const int s = cslot[c];
        const bool ib = cbuf[c];
        const int h = chot[c];
        if (s == w_slot) {
          if (!ib) {
            add(c, EV_PEND, 0, OFF_NREP, nullptr, 0.0, ckey[c], 0.0);
          } else if (w_isbuf) {
            add(c, EV_PEND, 0, OFF_NBREP, nullptr, 0.0, ckey[c], 0.0);
          } else {  // live winner with a registered buffer: ABSORB keeps it, DEFER moves it
            add(c, EV_CHAIN, 0, OFF_HBREP + w_h * DS, nullptr, S.hbn[w_h], ckey[c], 0.0);
            add(c, EV_PEND, 0, OFF_NBREP, nullptr, 0.0, ckey[c], 0.0);
          }
        } else if (h >= 0) {
          add(c, EV_CHAIN, 0, (ib ? OFF_HBREP : OFF_HREP) + h * DS, nullptr, ib ? S.hbn[h] : S.hrn[h], ckey[c], 0.0);
        } else {  // touched earlier, flushed out of the cache: global state (written back)
          add(c, EV_SLOW, 0, 0, (ib ? t.brep64 : t.rep64) + static_cast<int64_t>(s) * d,
              ib ? t.bnorm[s] : t.rnorm[s], ckey[c], 0.0);
        }
      }
      if (fresh_possible && lane == 0)  // the buffer a DEFER would register (index.cpp:153-160)
        add(-2, EV_FRESH, 0, OFF_NBREP, nullptr, 0.0, 2LL * t.cid[w_slot] + 1, 0.0);
      // (b) untouched candidates within 2*margin of the best untouched approximate score
      const int16_t* ti = tm_idx + tn * TOPM;
      int first_untouched;
      {
        bool u = false, stop = false;
        if (lane < TOPM) {
          const int c = ti[lane];
          stop = c < 0;
          u = !stop && !touched[c] && cslot[c] != w_slot;
        }
        const unsigned um = __ballot_sync(kFull, u), sm = __ballot_sync(kFull, stop);
        // the lists are dense: -1 entries only trail; first untouched before the first -1
        const int fu = um ? __ffs(um) - 1 : -1;
        const int fs = sm ? __ffs(sm) - 1 : 32;
        first_untouched = (fu >= 0 && fu < fs) ? fu : -1;
      }
      const float bu = first_untouched >= 0 ? tm_val[tn * TOPM + first_untouched] : -INFINITY;
      const float thr = bu - margin2;
      const bool complete = first_untouched >= 0 && !(tm_next[tn] >= thr);
      if (complete) {
        if (lane < TOPM) {
          const int c = ti[lane];
          if (c >= 0 && !touched[c] && cslot[c] != w_slot && tm_val[tn * TOPM + lane] >= thr) {
            const double ex = tm_exact[tn * TOPM + lane];
            if (isnan(ex)) {  // not computed by the tile kernel: exact from the representative
              const int s = cslot[c];
              const bool ib = cbuf[c];
              add(c, EV_SLOW, 0, 0, (ib ? t.brep64 : t.rep64) + static_cast<int64_t>(s) * d,
                  ib ? t.bnorm[s] : t.rnorm[s], ckey[c], 0.0);
            } else {
              add(c, EV_PRE, 0, 0, nullptr, 0.0, ckey[c], ex);
            }
          }
        }
      } else {  // rare: scan the whole approximate row
        for (int c = lane; c < n; c += 32) {
          if (touched[c] || cslot[c] == w_slot) continue;
          const float v = a.approx[o * cmax + c];
          if (first_untouched < 0 || v >= thr) {
            const int s = cslot[c];
            const bool ib = cbuf[c];
            add(c, EV_SLOW, 0, 0, (ib ? t.brep64 : t.rep64) + static_cast<int64_t>(s) * d,
                ib ? t.bnorm[s] : t.rnorm[s], ckey[c], 0.0);
          }
        }
      }
      __syncwarp();
    };

    // exact dots of the chain entries against the key at offset `koff`; with `specials` the
    // top three lanes of the first pass run |buf'|^2, |r'|^2 and sq_dist(k_t, r') for token t
    auto chain_phase = [&](int koff, const double* kq, bool specials, double& sq, double& rn, double& bn) {
      const int ne = min(S.ne, RELMAX);
      // slow entries (global representatives): one lane each, before the shared chain
      for (int e = lane; e < ne; e += 32)
        if (S.e_var[e] == EV_SLOW) {
          const double* g = S.e_gptr[e];
          double acc = 0.0;
#pragma unroll 16
          for (int i = 0; i < d; ++i) acc = dadd(acc, dmul(kq[i], g[i]));
          S.e_dot[e] = acc;
        }
      // compact the shared-chain entries in order
      const int dot_lanes0 = specials ? 32 - SPECIAL_LANES : 32;
      sq = rn = bn = 0.0;
      int pos = 0;  // next entry to consider
      for (int pass = 0;; ++pass) {
        const int lanes_here = pass == 0 ? dot_lanes0 : 32;
        const bool sp_pass = pass == 0 && specials;
        // find this lane's entry: the (lane)-th chain entry at or after pos (ballots over windows
        // of 32 entries instead of a per-lane serial scan)
        int taken = 0, p = pos;
        while (p < ne && taken < lanes_here) {
          const int e = p + lane;
          uint8_t v = EV_DEAD;
          if (e < ne) v = S.e_var[e];
          const bool isc = v == EV_CHAIN || v == EV_PEND || v == EV_FRESH;
          unsigned m = __ballot_sync(kFull, isc);
          const int need = lanes_here - taken;
          int span = min(32, ne - p);
          if (__popc(m) > need) {  // keep the lowest `need` chain entries; the window ends after them
            unsigned rest = m;
            for (int i = 0; i < need; ++i) rest &= rest - 1;
            m ^= rest;
            span = 32 - __clz(m);
          }
          if ((m >> lane) & 1u) S.sel[taken + __popc(m & ((1u << lane) - 1u))] = e;
          taken += __popc(m);
          p += span;
        }
        __syncwarp();
        const int mine = lane < taken ? S.sel[lane] : -1;
        __syncwarp();  // S.sel is rewritten by the next pass
        if (taken == 0 && !sp_pass) break;
        int oa = -1, ob = -1;
        if (mine >= 0) {
          oa = koff;
          ob = S.e_b[mine];
        } else if (sp_pass && lane >= dot_lanes0) {
          const int spc = lane - dot_lanes0;  // 0 buf', 1 r', 2 k - r'
          oa = spc == 0 ? OFF_NBREP : (spc == 1 ? OFF_NREP : OFF_DIFF);
          ob = oa;
        }
        double acc = 0.0;
        if (oa >= 0) {
          const double* A = sd + oa;
          const double* B = sd + ob;
#pragma unroll 16
          for (int i = 0; i < d; ++i) acc = dadd(acc, dmul(A[i], B[i]));
        }
        if (mine >= 0) S.e_dot[mine] = acc;
        if (sp_pass) {  // the two norms' square roots on their own lanes, in parallel
          const double rt = lane == dot_lanes0 || lane == dot_lanes0 + 1 ? __dsqrt_rn(acc) : acc;
          bn = __shfl_sync(kFull, rt, dot_lanes0);
          rn = __shfl_sync(kFull, rt, dot_lanes0 + 1);
          sq = __shfl_sync(kFull, rt, dot_lanes0 + 2);
        }
        pos = p;
        if (pos >= ne) break;
      }
      __syncwarp();
      n_exact += ne;
    };

    double sq = 0.0, rn = 0.0, bn = 0.0;
    build_entries(cur, -1, false, false, 0);
    chain_phase(OFF_KD + (cur % 3) * DS, kd + (cur % 3) * DS, false, sq, rn, bn);
    constexpr int KPL = 8;  // key elements per lane held in flight (d <= 256)
    long long pr[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // phase cycles | slow, scans, tokens, entries
    const bool prof_on = a.prof_on != 0;
    long long c0 = prof_on ? clock64() : 0, c1;
#define PROF(k) if (prof_on) { c1 = clock64(); pr[k] += c1 - c0; c0 = c1; }
    for (int tt = cur; tt < T; ++tt) {
      // prefetch the key of tt + 2 as raw 32-bit words (converted only at the end of the iteration,
      // so no instruction here waits for the load)
      uint32_t kpre[KPL];
      const int words = t.kv_bf16 ? d / 2 : d;
      const uint32_t* krow = reinterpret_cast<const uint32_t*>(a.fk) + (static_cast<int64_t>(dom) * t.tmax + tt + 2) * words;
#pragma unroll
      for (int j = 0; j < KPL; ++j) {
        const int w = lane + 32 * j;
        kpre[j] = (tt + 2 < T && w < words) ? krow[w] : 0u;
      }
      const double nkt = nk[tt];
      if (nkt < 1e-12) {
        if (lane == 0) {
          set_err(t, DERR_DEGENERATE);
          a.stop_t[dom] = tt;
        }
        break;
      }
      // ---- argmax(tt) (CandidateRef order tie-break)
      double bs = -3.0;
      long long bk = LLONG_MAX;
      int bp = -1;
      bool ltie = false;
      for (int e = lane; e < min(S.ne, RELMAX); e += 32) {
        const uint8_t v = S.e_var[e];
        if (v == EV_DEAD) continue;
        double cs;
        if (v == EV_PRE) {
          cs = S.e_dot[e];
        } else {
          const double nr = S.e_nr[e];
          if (nr < 1e-12) set_err(t, DERR_DEGENERATE);
          cs = clamp1(ddiv(S.e_dot[e], dmul(nkt, nr)));
        }
        if (cs == bs) ltie = true;
        else if (cs > bs) ltie = false;
        if (better(cs, S.e_key[e], bs, bk)) {
          bs = cs;
          bk = S.e_key[e];
          bp = e;
        }
      }
      const double lbs = bs;
      warp_best(bs, bk, bp);
      {
        const bool has = lbs == bs;
        if (__popc(__ballot_sync(kFull, has)) >= 2 || __any_sync(kFull, has && ltie)) any_tie = true;
      }
      const int bc = S.e_cand[bp];
      const int w = cslot[bc];
      const bool isbuf = cbuf[bc];
      PROF(0)
      // ---- winner into the hot cache
      int h = chot[bc];
      if (h < 0) {
        if (S.nhot >= HOT) flush_hot();
        // candidate indices of the slot (live / buffer)
        int cl = -1, cb = -1;
        for (int c = lane; c < n; c += 32)
          if (cslot[c] == w) {
            if (cbuf[c]) cb = c; else cl = c;
          }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          cl = max(cl, __shfl_xor_sync(kFull, cl, off));
          cb = max(cb, __shfl_xor_sync(kFull, cb, off));
        }
        h = hot_load(t, S, hrep, hbrep, w, cl, cb);
        if (cl >= 0 && lane == 0) chot[cl] = static_cast<int8_t>(h);
        if (cb >= 0 && lane == 0) chot[cb] = static_cast<int8_t>(h);
      }
      // mark the winner's candidates touched (they enter the touched list once)
      if (lane == 0) {
        const int cl = S.hcl[h], cb = S.hcb[h];
        if (cl >= 0 && !touched[cl]) {
          touched[cl] = 1;
          if (S.ntl < TLMAX) S.tl[S.ntl++] = cl; else set_err(t, DERR_CANDIDATES);
        }
        if (cb >= 0 && !touched[cb]) {
          touched[cb] = 1;
          if (S.ntl < TLMAX) S.tl[S.ntl++] = cb; else set_err(t, DERR_CANDIDATES);
        }
      }
      PROF(1)
      // Eq. 5 threshold of the winner, loaded early so its latency hides behind the chain phase
      const int64_t npre_w = S.hnmem[h];
      const double tau_w = __ldg(&t.tau_tab[npre_w < t.tau_len ? npre_w : t.tau_len - 1]);
      // ---- Eq. 3/4 into pending buffers (maintainer.cpp:16-25, index.cpp:181-188)
      const int kb = tt % 3, kn = (tt + 1) % 3;
      const double* kt = kd + kb * DS;
      const double dn = static_cast<double>(S.hstat[h]);
      const int nb = S.hnbuf[h];
      const double dnb = static_cast<double>(nb);
      // the buffer mean can only move on BUFJOIN or DEFER (a Host cluster under the deferred policy)
      const bool buf_may_move = isbuf || (S.hresid[h] != 0 && a.defer);
      {  // every element shares the divisor n + 1: one correctly rounded reciprocal + Markstein
        const double b1 = dadd(dn, 1.0), y1 = ddiv(1.0, b1);
        const double bb = dadd(dnb, 1.0), yb = ddiv(1.0, bb);
        for (int i = lane; i < d; i += 32) {
          const double r = div_rcp(dadd(dmul(dn, hrep[h * DS + i]), kt[i]), b1, y1);
          nrep[i] = r;
          diff[i] = dsub(kt[i], r);
          if (buf_may_move) nbrep[i] = nb == 0 ? kt[i] : div_rcp(dadd(dmul(dnb, hbrep[h * DS + i]), kt[i]), bb, yb);
        }
      }
      const bool has_next = tt + 1 < T;
      const bool fresh_possible = !isbuf && S.hresid[h] != 0 && a.defer && nb == 0;
      __syncwarp();
      PROF(2)
      if (has_next) {
        build_entries(tt + 1, w, isbuf, fresh_possible, h);
      } else {
        if (lane == 0) S.ne = 0;
        __syncwarp();
      }
      PROF(3)
      if (prof_on) {
        if (lane == 0) {
          int ns = 0;
          for (int e = 0; e < min(S.ne, RELMAX); ++e) ns += S.e_var[e] == EV_SLOW;
          pr[8] += ns;
          pr[10] += 1;
          pr[11] += min(S.ne, RELMAX);
        }
        c0 = clock64();
      }
      chain_phase(OFF_KD + kn * DS, kd + kn * DS, true, sq, rn, bn);
      PROF(4)
      const double varn = ddiv(dadd(dmul(dn, S.hvar[h]), sq), dadd(dn, 1.0));
      int kind;
      if (isbuf) {
        kind = EV_BUFJOIN;
      } else {
        if (varn <= tau_w)
          kind = EV_ABSORB;
        else if (S.hresid[h] == 0)
          kind = EV_SPLIT;
        else if (a.defer)
          kind = EV_DEFER;
        else
          kind = EV_EAGER;
      }
      if (kind == EV_SPLIT || kind == EV_EAGER) {  // host slow path; nothing committed
        if (lane == 0) {
          a.stop_t[dom] = tt;
          a.stop_kind[dom] = kind;
          a.stop_slot[dom] = w;
        }
        break;
      }
      // ---- resolve the pending variants of the next token's entries
      const bool buf_moved = kind == EV_BUFJOIN || kind == EV_DEFER;
      for (int e = lane; e < min(S.ne, RELMAX); e += 32) {
        const uint8_t v = S.e_var[e];
        const int c = S.e_cand[e];
        if (v == EV_PEND) {
          const bool ib = cbuf[c];
          if (ib && !buf_moved) {
            S.e_var[e] = EV_DEAD;
          } else {
            S.e_nr[e] = ib ? bn : rn;
          }
        } else if (v == EV_CHAIN && c >= 0 && cslot[c] == w && cbuf[c] && buf_moved) {
          S.e_var[e] = EV_DEAD;  // old buffer state superseded
        } else if (v == EV_FRESH) {
          if (kind == EV_DEFER && nb == 0) {
            S.e_cand[e] = n;  // the new candidate index (registered below)
            S.e_nr[e] = bn;
            S.e_var[e] = EV_PEND;
          } else {
            S.e_var[e] = EV_DEAD;
          }
        }
      }
      PROF(5)
      // ---- commit
      for (int i = lane; i < d; i += 32) {
        hrep[h * DS + i] = nrep[i];
        if (buf_moved) hbrep[h * DS + i] = nbrep[i];
      }
      __syncwarp();  // every lane read S.hvar[h] / the pending entries above (racecheck: WAR)
      if (lane == 0) {
        S.hdirty[h] = 1;
        S.hrn[h] = rn;
        S.hvar[h] = varn;
        S.hstat[h] += 1;
        if (kind == EV_ABSORB) S.hnmem[h] += 1;
        if (buf_moved) {
          S.hbn[h] = bn;
          S.hnbuf[h] = nb + 1;
        }
        if (kind == EV_DEFER) S.hlazy[h] = 1;
        const int64_t frow = static_cast<int64_t>(dom) * t.tmax + tt;
        int page, row;
        hot_reserve_row(t, S, h, buf_moved, page, row);
        a.ev_page[frow] = page;
        a.ev_row[frow] = row;
        a.ev_kind[frow] = kind;
        a.ev_slot[frow] = w;
        if (a.ring_slot >= 0) t.ring_owner[(static_cast<int64_t>(dom) * t.W + a.ring_slot) * t.tmax + tt] = w;
        if (kind == EV_DEFER && nb == 0) {  // register the new buffer candidate
          if (n < cmax) {
            cslot[n] = w;
            cbuf[n] = 1;
            ckey[n] = 2LL * t.cid[w] + 1;
            touched[n] = 1;
            chot[n] = static_cast<int8_t>(h);
            S.hcb[h] = n;
            if (S.ntl < TLMAX) S.tl[S.ntl++] = n; else set_err(t, DERR_CANDIDATES);
          } else {
            set_err(t, DERR_CANDIDATES);
          }
        }
      }
      if (kind == EV_DEFER && nb == 0) n = min(n + 1, cmax);
      PROF(6)
      if (tt + 2 < T) {
        double* kr = kd + ((tt + 2) % 3) * DS;
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
          const int w = lane + 32 * j;
          if (w < words) {
            if (t.kv_bf16) {
              kr[2 * w] = static_cast<double>(__uint_as_float(kpre[j] << 16));
              kr[2 * w + 1] = static_cast<double>(__uint_as_float(kpre[j] & 0xffff0000u));
            } else {
              kr[w] = static_cast<double>(__uint_as_float(kpre[j]));
            }
          }
        }
      }
      __syncwarp();
      PROF(7)
    }
#undef PROF
    if (lane == 0 && prof_on)
      for (int k = 0; k < 12; ++k) a.prof[dom * 16 + k] = pr[k];
  }
done:
  __syncwarp();
  for (int i = 0; i < S.nhot; ++i) hot_writeback(t, S, hrep, hbrep, i);
  if (lane < POOL) a.dom_pool[dom * POOL + lane] = S.pool[lane];
  if (lane == 0) {
    a.dom_pool_n[dom] = S.npool;
    a.n_exact[dom] = n_exact;
    if (a.tie) a.tie[dom] = any_tie ? 1 : 0;
  }
}

// ============================================================================ K3
// One warp per frame row of the launch's token range: the row's K and V (16-byte lane chunks,
// loaded once) go to the window ring page of the frame and, when the resolve kernel committed the
// token, to the (page, row) it reserved in the cluster's page list.
__global__ void k_store_rows(DevTables t, IngestArgs a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (launched as a dependent of K2)
  const int dom = a.active[blockIdx.y];
  if (a.err_copy && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *a.err_copy = *t.err;
  if (a.prev_events && *a.prev_events) return;  // skipped speculative round: no writes
  if (a.my_events && blockIdx.x == 0 && threadIdx.x == 0 && a.stop_t[dom] < a.T) atomicOr(a.my_events, 1);
  const int rb = t.d * t.es;
  const int warps = blockDim.x / 32, warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int cur = a.cursor[dom];
  const int half = lane >> 4, hl = lane & 15;  // lanes 0-15: K, lanes 16-31: V
  for (int tt = cur + blockIdx.x * warps + warp; tt < a.T; tt += gridDim.x * warps) {
    const int64_t frow = static_cast<int64_t>(dom) * t.tmax + tt;
    const int page = a.ev_page[frow];
    const int row = page >= 0 ? a.ev_row[frow] : 0;
    const uint8_t* src = static_cast<const uint8_t*>(half ? a.fv : a.fk) + frow * rb;
    // ring_slot < 0: entries inserted outside a frame (Maintainer::on_insert), no window row
    uint8_t* dring = nullptr;
    if (a.ring_slot >= 0) {
      const int rpage = t.ring_pages[(static_cast<int64_t>(dom) * t.W + a.ring_slot) * t.rpp + tt / t.P];
      dring = (half ? page_v(t, rpage) : page_k(t, rpage)) + static_cast<int64_t>(tt % t.P) * rb;
    }
    uint8_t* dclu = page >= 0 ? (half ? page_v(t, page) : page_k(t, page)) + static_cast<int64_t>(row) * rb : nullptr;
    for (int o = hl * 16; o < rb; o += 16 * 16) {
      const uint4 v = *reinterpret_cast<const uint4*>(src + o);
      if (dring) *reinterpret_cast<uint4*>(dring + o) = v;
      if (dclu) *reinterpret_cast<uint4*>(dclu + o) = v;
    }
  }
}

// Window-ring rows only (frames buffered for the batch build, which routes nothing yet).
__global__ void k_ring_rows(DevTables t, const uint8_t* fk, const uint8_t* fv, int T, int rs) {
  const int dom = blockIdx.y;
  const int rb = t.d * t.es;
  const int warps = blockDim.x / 32, warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int half = lane >> 4, hl = lane & 15;
  for (int tt = blockIdx.x * warps + warp; tt < T; tt += gridDim.x * warps) {
    const int64_t frow = static_cast<int64_t>(dom) * t.tmax + tt;
    const uint8_t* src = (half ? fv : fk) + frow * rb;
    const int rpage = t.ring_pages[(static_cast<int64_t>(dom) * t.W + rs) * t.rpp + tt / t.P];
    uint8_t* dring = (half ? page_v(t, rpage) : page_k(t, rpage)) + static_cast<int64_t>(tt % t.P) * rb;
    for (int o = hl * 16; o < rb; o += 16 * 16) *reinterpret_cast<uint4*>(dring + o) = *reinterpret_cast<const uint4*>(src + o);
  }
}

// ============================================================================ ring write
// Frame start: the ring slot's ownership entries are reset (the resolve kernel then records the
// owner of every routed token) and its page fills / token count set; the rows themselves are
// copied by K3 after the resolve, together with the cluster rows.
__global__ void k_ring_write(DevTables t, const uint8_t* fk, const uint8_t* fv, int T, int rs) {
  const int dom = blockIdx.y;
  for (int tt = blockIdx.x * blockDim.x + threadIdx.x; tt < t.tmax; tt += gridDim.x * blockDim.x)
    t.ring_owner[(static_cast<int64_t>(dom) * t.W + rs) * t.tmax + tt] = -1;
  if (blockIdx.x == 0 && threadIdx.x < t.rpp) {
    const int j = threadIdx.x;
    const int page = t.ring_pages[(static_cast<int64_t>(dom) * t.W + rs) * t.rpp + j];
    t.pg_fill[page] = max(0, min(t.P, T - j * t.P));
  }
  if (blockIdx.x == 0 && dom == 0 && threadIdx.x == 0) t.ring_count[rs] = T;
}

// ============================================================================ store maintenance
// One CTA per run: the run's pages are claimed at once (the free-stack pops in the order a
// row-by-row warp_append would make them, so the layout is the same), then every thread copies
// 16-byte pieces of the run's rows. Runs of one launch target distinct (slot, list) pairs.
__global__ void __launch_bounds__(256) k_append_runs(DevTables t, const AppendRun* runs, int n_runs,
                                                     const int32_t* idx, const uint8_t* sk, const uint8_t* sv) {
  const AppendRun r = runs[blockIdx.x];
  const bool to_buf = r.to_buffer != 0;
  int* list = to_buf ? t.bpages + static_cast<int64_t>(r.slot) * t.maxbp : t.pages + static_cast<int64_t>(r.slot) * t.maxp;
  __shared__ int s_page0, s_fill0, s_room, s_base_n, s_rows;
  if (threadIdx.x == 0) {
    int* np = to_buf ? &t.nbpages[r.slot] : &t.npages[r.slot];
    const int cap = to_buf ? t.maxbp : t.maxp;
    const int n = *np;
    const int page = n > (to_buf ? 0 : t.seal[r.slot]) ? list[n - 1] : -1;  // sealed pages take no rows
    const int fill0 = page >= 0 ? t.pg_fill[page] : t.P;
    const int room = page >= 0 ? min(t.P - fill0, r.n_rows) : 0;
    int rows = r.n_rows;
    int k = (rows - room + t.P - 1) / t.P;  // fresh pages
    if (n + k > cap) {
      set_err(t, DERR_CLUSTER_PAGES);
      k = cap - n;
    }
    int top = k > 0 ? atomicSub(t.free_top, k) - k : 0;
    if (top < 0) {
      atomicAdd(t.free_top, k);
      set_err(t, DERR_PAGES);
      k = 0;
    }
    rows = min(rows, room + k * t.P);
    for (int i = 0; i < k; ++i) {
      const int pg = t.free_stack[top + k - 1 - i];
      list[n + i] = pg;
      t.pg_fill[pg] = min(t.P, rows - room - i * t.P);
    }
    *np = n + k;
    if (room > 0) t.pg_fill[page] = fill0 + room;
    s_page0 = page;
    s_fill0 = fill0;
    s_room = room;
    s_base_n = n;
    s_rows = rows;
  }
  __syncthreads();
  const int rb = t.d * t.es, pieces = rb / 16, rows = s_rows, room = s_room;
  for (int64_t q = threadIdx.x; q < static_cast<int64_t>(rows) * pieces; q += blockDim.x) {
    const int j = static_cast<int>(q / pieces), o = static_cast<int>(q - static_cast<int64_t>(j) * pieces) * 16;
    int page, pos;
    if (j < room) {
      page = s_page0;
      pos = s_fill0 + j;
    } else {
      page = list[s_base_n + (j - room) / t.P];
      pos = (j - room) % t.P;
    }
    const int64_t row = idx[r.first_row + j];
    *reinterpret_cast<uint4*>(page_k(t, page) + static_cast<int64_t>(pos) * rb + o) =
        *reinterpret_cast<const uint4*>(sk + row * rb + o);
    *reinterpret_cast<uint4*>(page_v(t, page) + static_cast<int64_t>(pos) * rb + o) =
        *reinterpret_cast<const uint4*>(sv + row * rb + o);
  }
}

__global__ void k_gather_cluster(DevTables t, int slot, int with_buf, uint8_t* sk, uint8_t* sv,
                                 int64_t row0) {
  // block b copies page b of the member list, then the buffer pages
  const int np = t.npages[slot];
  const int nbp = with_buf ? t.nbpages[slot] : 0;
  const int64_t nmem = t.nmem[slot];
  const int b = blockIdx.x;
  if (b >= np + nbp) return;
  const bool isb = b >= np;
  const int j = isb ? b - np : b;
  const int page = isb ? t.bpages[static_cast<int64_t>(slot) * t.maxbp + j]
                       : t.pages[static_cast<int64_t>(slot) * t.maxp + j];
  const int fill = t.pg_fill[page];
  // member pages may be partial mid-list (sealed by an offload): rows before page j = sum of fills
  __shared__ int before;
  if (threadIdx.x == 0) {
    int r = 0;
    const int* list = isb ? t.bpages + static_cast<int64_t>(slot) * t.maxbp : t.pages + static_cast<int64_t>(slot) * t.maxp;
    for (int i = 0; i < j; ++i) r += t.pg_fill[list[i]];
    before = r;
  }
  __syncthreads();
  const int64_t first = row0 + (isb ? nmem : 0) + before;
  const int rb = t.d * t.es;
  const uint8_t* pk = page_k(t, page);
  const uint8_t* pv = page_v(t, page);
  for (int o = threadIdx.x * 16; o < fill * rb; o += blockDim.x * 16) {
    *reinterpret_cast<uint4*>(sk + first * rb + o) = *reinterpret_cast<const uint4*>(pk + o);
    *reinterpret_cast<uint4*>(sv + first * rb + o) = *reinterpret_cast<const uint4*>(pv + o);
  }
}

__global__ void k_free_slot(DevTables t, int slot) {
  // HBM pages return to the free stack; host-tier pages belong to an extent the host frees
  const int np = t.npages[slot], nbp = t.nbpages[slot];
  __shared__ int base, nh;
  if (threadIdx.x == 0) {
    int h = 0;
    for (int i = 0; i < np; ++i) h += is_host_page(t, t.pages[static_cast<int64_t>(slot) * t.maxp + i]) ? 1 : 0;
    nh = h;
    base = atomicAdd(t.free_top, np - h + nbp);
    int k = 0;
    for (int i = 0; i < np; ++i) {
      const int pg = t.pages[static_cast<int64_t>(slot) * t.maxp + i];
      if (!is_host_page(t, pg)) t.free_stack[base + k++] = pg;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nbp; i += blockDim.x)
    t.free_stack[base + np - nh + i] = t.bpages[static_cast<int64_t>(slot) * t.maxbp + i];
  __syncthreads();
  if (threadIdx.x == 0) {
    t.seal[slot] = 0;
    t.npages[slot] = 0;
    t.nbpages[slot] = 0;
    t.nmem[slot] = 0;
    t.nbuf[slot] = 0;
    t.lazy[slot] = 0;
    t.stat[slot] = 0;
  }
}

__global__ void k_refresh_mirror(DevTables t, const int32_t* slots, int n) {
  const int i = blockIdx.x;
  if (i >= n) return;
  const int64_t s = slots[i];
  for (int c = threadIdx.x; c < t.d; c += blockDim.x) {
    t.rep32[s * t.d + c] = static_cast<float>(t.rep64[s * t.d + c]);
    if (t.nbuf[s] > 0) t.brep32[s * t.d + c] = static_cast<float>(t.brep64[s * t.d + c]);
  }
}

// compute_representative / compute_variance (index.cpp:345-362), exact order.
__global__ void k_exact_stats(DevTables t, const AppendRun* runs, int n_runs, const int32_t* idx,
                              const void* sk) {
  extern __shared__ double es[];
  double* rep = es;            // [d]
  double* sq = es + t.d;       // [blockDim]
  const int r = blockIdx.x;
  if (r >= n_runs) return;
  const AppendRun run = runs[r];
  const int d = t.d;
  const int64_t s = run.slot;
  const double inv = ddiv(1.0, static_cast<double>(run.n_rows));
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < run.n_rows; ++j)
      acc = dadd(acc, static_cast<double>(ld_kv(sk, static_cast<int64_t>(idx[run.first_row + j]) * d + c, t.kv_bf16)));
    rep[c] = dmul(acc, inv);
    t.rep64[s * d + c] = rep[c];
    t.rep32[s * d + c] = static_cast<float>(rep[c]);
  }
  __syncthreads();
  double total = 0.0;
  for (int j0 = 0; j0 < run.n_rows; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    if (j < run.n_rows) {
      const int64_t row = idx[run.first_row + j];
      double acc = 0.0;
      for (int c = 0; c < d; ++c) {
        const double df = dsub(static_cast<double>(ld_kv(sk, row * d + c, t.kv_bf16)), rep[c]);
        acc = dadd(acc, dmul(df, df));
      }
      sq[threadIdx.x] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int m = min(static_cast<int>(blockDim.x), run.n_rows - j0);
      for (int i = 0; i < m; ++i) total = dadd(total, sq[i]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    t.var[s] = ddiv(total, static_cast<double>(run.n_rows));
    double nn = 0.0;
    for (int c = 0; c < d; ++c) nn = dadd(nn, dmul(rep[c], rep[c]));
    t.rnorm[s] = __dsqrt_rn(nn);
  }
}

__global__ void k_slot_headers(DevTables t, const SlotHeader* h, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const SlotHeader x = h[i];
  t.stat[x.slot] = x.n;
  t.nmem[x.slot] = x.n;
  t.cid[x.slot] = x.cid;
  t.nbuf[x.slot] = 0;
  t.lazy[x.slot] = 0;
  t.resid[x.slot] = 0;
}

__global__ void k_init_slots(DevTables t, const uint8_t* recs, int n) {
  const uint8_t* r = recs + static_cast<int64_t>(blockIdx.x) * slot_init_bytes(t.d);
  const SlotInit& x = *reinterpret_cast<const SlotInit*>(r);
  const double* rep = reinterpret_cast<const double*>(r + sizeof(SlotInit));
  const int64_t s = x.slot;
  for (int c = threadIdx.x; c < t.d; c += blockDim.x) {
    t.rep64[s * t.d + c] = rep[c];
    if (x.has_brep) t.brep64[s * t.d + c] = rep[t.d + c];
  }
  if (threadIdx.x == 0) {
    t.rnorm[s] = x.rnorm;
    t.var[s] = x.var;
    t.stat[s] = x.stat;
    t.nmem[s] = x.nmem;
    t.cid[s] = x.cid;
    t.resid[s] = x.resid;
    t.nbuf[s] = x.nb;
    t.lazy[s] = x.lazy;
    if (x.has_brep) t.bnorm[s] = x.bnorm;
  }
}

__global__ void k_to_f32(const void* src, float* dst, int64_t n, int bf16) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = ld_kv(src, i, bf16);
}

// ============================================================================ K4
// Block-wide k-best selection by repeated arg-best (k <= 64): items (sim[i], key[i]).
__device__ int block_take_best(const double* sim, const long long* key, uint8_t* taken, int n,
                               double* red_s, long long* red_k, int* red_i) {
  double bs = -4.0;
  long long bk = LLONG_MAX;
  int bi = -1;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (!taken[i] && better(sim[i], key[i], bs, bk)) {
      bs = sim[i];
      bk = key[i];
      bi = i;
    }
  warp_best(bs, bk, bi);
  const int w = threadIdx.x / 32, nw = blockDim.x / 32;
  if ((threadIdx.x & 31) == 0) {
    red_s[w] = bs;
    red_k[w] = bk;
    red_i[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = red_s[0];
    long long k = red_k[0];
    int ii = red_i[0];
    for (int j = 1; j < nw; ++j)
      if (red_i[j] >= 0 && (ii < 0 || better(red_s[j], red_k[j], s, k))) {
        s = red_s[j];
        k = red_k[j];
        ii = red_i[j];
      }
    red_i[32] = ii;
    if (ii >= 0) taken[ii] = 1;
  }
  __syncthreads();
  const int r = red_i[32];
  __syncthreads();
  return r;
}

// exact cosine of q (fp32, norm nq) with a fp64 row (vecmath.hpp:54-61)
__device__ __forceinline__ double exact_cos(const float* q, double nq, const double* row, double nr,
                                            int d, bool& degenerate) {
  if (nq < 1e-12 || nr < 1e-12) {
    degenerate = true;
    return -2.0;
  }
  double acc = 0.0;
#pragma unroll 16
  for (int i = 0; i < d; ++i) acc = dadd(acc, dmul(static_cast<double>(q[i]), row[i]));
  return clamp1(ddiv(acc, dmul(nq, nr)));
}

// Block-wide bitonic sort of n (power of two) entries "best first" by (sim desc, key asc);
// `ord` carries the payload. Padding entries use sim = -inf, key = LLONG_MAX.
__device__ void block_bitonic(double* sim, long long* key, int* ord, int n) {
  for (int k = 2; k <= n; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const bool up = (i & k) == 0;
          const bool sw = up ? better(sim[p], key[p], sim[i], key[i]) : better(sim[i], key[i], sim[p], key[p]);
          if (sw) {
            const double ts = sim[i];
            sim[i] = sim[p];
            sim[p] = ts;
            const long long tk = key[i];
            key[i] = key[p];
            key[p] = tk;
            const int to = ord[i];
            ord[i] = ord[p];
            ord[p] = to;
          }
        }
      }
      __syncthreads();
    }
}

__host__ __device__ inline int pow2_at_least(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

// Exact top-`take` selection by rank counting: rank(i) = #entries better than i under
// (sim desc, key asc); keys are unique so ranks are a permutation. O(n^2 / threads) broadcast
// shared reads, no sorting network and only one barrier.
__device__ void block_rank_select(const double* sim, const long long* key, int n, int take, int* order) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double si = sim[i];
    const long long ki = key[i];
    int r = 0;
    for (int j = 0; j < n; ++j) r += better(sim[j], key[j], si, ki) ? 1 : 0;
    if (r < take) order[r] = i;
  }
  __syncthreads();
}

// Top-`take` (take <= 64) of n <= 1024 entries, best first under (sim desc, key asc). Each warp
// sorts 32-entry chunks in registers with a shuffle bitonic network (no block barriers), then
// warp 0 merges the sorted chunks by repeatedly taking the best chunk head. `pay` is scratch
// for the payload indices; order[r] receives the index of the r-th best entry.
__device__ void block_topk(double* sim, long long* key, int* pay, int n, int take, int* order) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nch = (n + 31) / 32;
  for (int c = warp; c < nch; c += nw) {
    const int i = c * 32 + lane;
    double s = i < n ? sim[i] : -INFINITY;
    long long k = i < n ? key[i] : LLONG_MAX;
    int p = i < n ? i : -1;
    for (int size = 2; size <= 32; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const double ps = __shfl_xor_sync(kFull, s, stride);
        const long long pk = __shfl_xor_sync(kFull, k, stride);
        const int pp = __shfl_xor_sync(kFull, p, stride);
        const bool up = (lane & size) == 0 || size == 32;
        const bool lower = (lane & stride) == 0;
        const bool pb = better(ps, pk, s, k);
        if ((lower == up) ? pb : !pb) {
          s = ps;
          k = pk;
          p = pp;
        }
      }
    sim[c * 32 + lane] = s;
    key[c * 32 + lane] = k;
    pay[c * 32 + lane] = p;
  }
  __syncthreads();
  if (warp == 0) {
    int head = 0;  // lane j walks chunk j
    for (int r = 0; r < take; ++r) {
      double bs = -INFINITY;
      long long bk = LLONG_MAX;
      int bl = -1;
      if (lane < nch && head < 32) {
        const int i = lane * 32 + head;
        bs = sim[i];
        bk = key[i];
        if (pay[i] >= 0) bl = lane;
      }
      int src = bl;
      warp_best(bs, bk, src);
      if (src < 0) break;
      if (lane == src) {
        order[r] = pay[lane * 32 + head];
        head += 1;
      }
    }
  }
  __syncthreads();
}

constexpr int K4_ROWS = 128;  // representative rows staged per chunk (d <= 128)
// fp64 rows the stage buffer holds: 128 up to d = 128, 48 for wider rows (d = 256: 98 KB)
__host__ __device__ inline int k4_stage_rows(int d) { return d <= 128 ? K4_ROWS : 48; }
constexpr float kScoreMargin = 1e-4f;  // bound on |fp32 mirror cosine - exact fp64 cosine|

__host__ __device__ inline size_t k4_smem_bytes(int d, int cmax, int parts, int W, int tmax) {
  const int nsel = cmax > parts ? cmax : parts;
  return static_cast<size_t>(d + 1) * 8 + static_cast<size_t>(nsel) * 24 + static_cast<size_t>(cmax) * 5 +
         static_cast<size_t>(k4_stage_rows(d)) * (d + 1) * 8 + static_cast<size_t>(W) * tmax * 4 + 256;
}

__global__ void __launch_bounds__(256) k_score_select(DevTables t, DecodeArgs a, int* work_ctr) {
  extern __shared__ __align__(16) uint8_t sm4[];
  const int l = blockIdx.x, d = t.d, L = t.L, DS = d + 1;
  const int P = a.n_parts_host;
  const int cmax = t.cmax;
  const int nsel = cmax > P ? cmax : P;
  uint8_t* p = sm4;
  double* qd = reinterpret_cast<double*>(p);  // query as double (exact conversion)
  p += static_cast<size_t>(d + 1) * 8;
  double* sim = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(nsel) * 8;
  long long* key = reinterpret_cast<long long*>(p);
  p += static_cast<size_t>(nsel) * 8;
  int* pay = reinterpret_cast<int*>(p);  // top-k payload scratch
  p += static_cast<size_t>(nsel) * 4;
  float* approx = reinterpret_cast<float*>(p);  // approximate candidate scores
  p += static_cast<size_t>(nsel) * 4;
  p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~static_cast<uintptr_t>(15));
  const int SR = k4_stage_rows(d);
  double* stage = reinterpret_cast<double*>(p);  // [SR][d+1] (16-byte aligned for cp.async)
  p += static_cast<size_t>(SR) * DS * 8;
  int* owners = reinterpret_cast<int*>(p);  // [W][tmax] ring owners of this domain
  p += static_cast<size_t>(t.W) * t.tmax * 4;
  int* cslot = reinterpret_cast<int*>(p);
  p += static_cast<size_t>(cmax) * 4;
  uint8_t* cbuf = p;
  __shared__ double nq_s;
  __shared__ int ncand_s, chosen[64];
  __shared__ int vers[64], nver_s;
  __shared__ int rank_slot[64], n_rank_s, order[64];
  __shared__ unsigned long long att_s;
  __shared__ int lazy_any;
  __shared__ bool degen;
  __shared__ int ring_count_s[64];
  __shared__ int sset[K4_ROWS], n_s;
  __shared__ float qf32[256];
  __shared__ double ssim[K4_ROWS];
  __shared__ long long skey[K4_ROWS];

  long long kc0 = clock64();
#define K4MARK(k) if (a.k4prof && threadIdx.x == 0) { const long long kc1 = clock64(); a.k4prof[l * 16 + (k)] = kc1 - kc0; kc0 = kc1; }
  if (l == 0 && threadIdx.x == 0) *work_ctr = 0;
  const float* q = (a.q_src ? a.q_src : a.q) + static_cast<int64_t>(l) * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float x = q[i];
    if (a.q_src) const_cast<float*>(a.q)[static_cast<int64_t>(l) * d + i] = x;
    qd[i] = static_cast<double>(x);
    qf32[i] = x;
  }
  // the window ring owners are needed after ranking; fetch them now
  {
    const int n_own = t.W * t.tmax;
    const int* src = t.ring_owner + static_cast<int64_t>(l) * n_own;
    int v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = threadIdx.x + 256 * j;
      v[j] = i < n_own ? src[i] : -1;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = threadIdx.x + 256 * j;
      if (i < n_own) owners[i] = v[j];
    }
    for (int i = threadIdx.x + 256 * 8; i < n_own; i += blockDim.x) owners[i] = src[i];
  }
  if (threadIdx.x == 0) {
    degen = false;
    att_s = 0;
    lazy_any = 0;
  }
  if (threadIdx.x < t.W && threadIdx.x < 64) ring_count_s[threadIdx.x] = t.ring_count[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
#pragma unroll 16
    for (int i = 0; i < d; ++i) s = dadd(s, dmul(qd[i], qd[i]));
    nq_s = __dsqrt_rn(s);
  }
  __syncthreads();
  const double nq = nq_s;
  if (nq < 1e-12 && threadIdx.x == 0) degen = true;
  K4MARK(0)
  // ---- stage 1: visual_topk (index.cpp:192-208): exact cosines, order (sim desc, id asc)
  for (int p0 = 0; p0 < P; p0 += SR) {
    const int rows = min(SR, P - p0);
    for (int r = threadIdx.x >> 5; r < rows; r += blockDim.x >> 5) {
      const double* src = t.vrep + static_cast<int64_t>(p0 + r) * d;
      for (int i = threadIdx.x & 31; i < d; i += 32)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(stage + r * DS + i)), "l"(src + i)
                     : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
      const double* row = stage + r * DS;
      double acc = 0.0;
#pragma unroll 16
      for (int i = 0; i < d; ++i) acc = dadd(acc, dmul(qd[i], row[i]));
      const double nr = t.vnorm[p0 + r];
      if (nr < 1e-12) degen = true;
      sim[p0 + r] = clamp1(ddiv(acc, dmul(nq, nr)));
      key[p0 + r] = p0 + r;
    }
    __syncthreads();
  }
  const int kv = min(a.k_v, P);
  if (P <= 1024)
    block_topk(sim, key, pay, P, kv, chosen);
  else
    block_rank_select(sim, key, P, kv, chosen);
  if (threadIdx.x < kv) a.parts[l * a.k_v + threadIdx.x] = chosen[threadIdx.x];
  if (threadIdx.x == 0) a.n_parts_sel[l] = kv;
  K4MARK(1)

  // ---- stage 2: semantic_topk (index.cpp:210-240) and the prefetch ranking of layer l+1
  // with this layer's query (retrieval.cpp:117-128)
  const int passes = (a.prefetch && l + 1 < L) ? 2 : 1;
  for (int pass = 0; pass < passes; ++pass) {
    const int layer = l + pass;
    const int ktake = pass == 0 ? a.k_s : a.prefetch_k;
    if (threadIdx.x == 0) ncand_s = 0;
    __syncthreads();
    for (int i = 0; i < kv; ++i) {
      const int64_t pk = static_cast<int64_t>(chosen[i]) * L + layer;
      const int off = t.pl_off[pk], cnt = t.pl_cnt[pk];
      for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
        const int s = t.pl_pool[off + j];
        const int lz = t.lazy[s];
        const int k = atomicAdd(&ncand_s, lz ? 2 : 1);
        if (k + (lz ? 2 : 1) > cmax) {
          set_err(t, DERR_CANDIDATES);
          continue;
        }
        cslot[k] = s;
        cbuf[k] = 0;
        if (lz) {
          cslot[k + 1] = s;
          cbuf[k + 1] = 1;
        }
      }
    }
    __syncthreads();
    const int nc = min(ncand_s, cmax);
    if (pass == 0 && threadIdx.x == 0) a.n_cand[l] = nc;
    int take = min(ktake, nc);
    if (take > 64) {  // ranked lists live in 64-entry shared arrays
      if (threadIdx.x == 0) set_err(t, DERR_TAKE);
      take = 64;
    }
    // (A) approximate cosines from the fp32 mirrors: rows staged with 16-byte async copies, one
    //     thread per candidate reading its row in a rotated order (conflict-free banks)
    float* st32 = reinterpret_cast<float*>(stage);  // [rows][d + 4]
    const int DS32 = d + 4;
    const int rows32 = min(nc, (2 * SR * DS) / DS32);  // what the fp64 stage buffer holds
    for (int c0 = 0; c0 < nc; c0 += rows32) {
      const int rows = min(rows32, nc - c0);
      for (int r = threadIdx.x >> 5; r < rows; r += blockDim.x >> 5) {
        const int s = cslot[c0 + r];
        const float* src = (cbuf[c0 + r] ? t.brep32 : t.rep32) + static_cast<int64_t>(s) * d;
        for (int i = (threadIdx.x & 31) * 4; i < d; i += 128)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(st32 + r * DS32 + i)), "l"(src + i)
                       : "memory");
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
      for (int r = threadIdx.x; r < rows; r += blockDim.x) {
        const int c = c0 + r;
        const float* row = st32 + r * DS32;
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        // element order rotated by the row index: banks (4r + r + i) mod 32 are distinct per lane
        int j = r & 31;
        for (int i0 = 0; i0 < d; i0 += 4) {
          a0 = fmaf(qf32[j], row[j], a0);
          j = j + 1 == d ? 0 : j + 1;
          a1 = fmaf(qf32[j], row[j], a1);
          j = j + 1 == d ? 0 : j + 1;
          a2 = fmaf(qf32[j], row[j], a2);
          j = j + 1 == d ? 0 : j + 1;
          a3 = fmaf(qf32[j], row[j], a3);
          j = j + 1 == d ? 0 : j + 1;
        }
        const int s = cslot[c];
        const bool ib = cbuf[c];
        const double nr = ib ? t.bnorm[s] : t.rnorm[s];
        if (nr < 1e-12) degen = true;
        const float sa = ((a0 + a1) + (a2 + a3)) / static_cast<float>(nq * nr);
        approx[c] = sa;
        sim[c] = static_cast<double>(sa);
        key[c] = 2LL * t.cid[s] + (ib ? 1 : 0);
      }
      __syncthreads();
    }
    K4MARK(2)
    // (B) the set S of candidates that can reach the exact top-`take`: approximate score within
    //     2*margin of the take-th best approximate score (|approx - exact| <= margin)
    if (threadIdx.x == 0) n_s = 0;
    if (take > 0 && take < nc) {
      block_topk(sim, key, pay, nc, take, order);
      const float thr = approx[order[take - 1]] - 2.f * kScoreMargin;
      for (int c = threadIdx.x; c < nc; c += blockDim.x)
        if (approx[c] >= thr) {
          const int k = atomicAdd(&n_s, 1);
          if (k < SR) sset[k] = c;
        }
    } else {
      for (int c = threadIdx.x; c < nc; c += blockDim.x) {
        const int k = atomicAdd(&n_s, 1);
        if (k < SR) sset[k] = c;
      }
    }
    __syncthreads();
    if (n_s > SR) {
      // Near-tie-heavy query (rare): S exceeds the stage. Exact cosines of EVERY candidate, SR rows
      // at a time, into sim[] (free after the threshold pass), then the exact top-`take` over all
      // of them -- the reference ranks any number of ties (index.cpp:210-240).
      for (int c0 = 0; c0 < nc; c0 += SR) {
        const int rows = min(SR, nc - c0);
        for (int r = threadIdx.x >> 5; r < rows; r += blockDim.x >> 5) {
          const double* src = (cbuf[c0 + r] ? t.brep64 : t.rep64) + static_cast<int64_t>(cslot[c0 + r]) * d;
          for (int i = threadIdx.x & 31; i < d; i += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(stage + r * DS + i)), "l"(src + i)
                         : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        for (int r = threadIdx.x; r < rows; r += blockDim.x) {
          const int c = c0 + r;
          const int s = cslot[c];
          const bool ib = cbuf[c];
          const double* row = stage + r * DS;
          double acc = 0.0;
#pragma unroll 16
          for (int i = 0; i < d; ++i) acc = dadd(acc, dmul(qd[i], row[i]));
          sim[c] = clamp1(ddiv(acc, dmul(nq, ib ? t.bnorm[s] : t.rnorm[s])));
          key[c] = 2LL * t.cid[s] + (ib ? 1 : 0);
        }
        __syncthreads();
      }
      block_rank_select(sim, key, nc, take, order);  // order[] = candidate indices
      __syncthreads();
    } else {
    const int ns_ = n_s;
    // (C) exact cosines (vecmath.hpp:54-61) for S: fp64 rows staged with 8-byte async copies,
    //     one sequential chain per candidate; exact top-`take` of S by rank counting
    for (int r = threadIdx.x >> 5; r < ns_; r += blockDim.x >> 5) {
      const int c = sset[r];
      const double* src = (cbuf[c] ? t.brep64 : t.rep64) + static_cast<int64_t>(cslot[c]) * d;
      for (int i = threadIdx.x & 31; i < d; i += 32)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(stage + r * DS + i)), "l"(src + i)
                     : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    for (int r = threadIdx.x; r < ns_; r += blockDim.x) {
      const int c = sset[r];
      const int s = cslot[c];
      const bool ib = cbuf[c];
      const double* row = stage + r * DS;
      double acc = 0.0;
#pragma unroll 16
      for (int i = 0; i < d; ++i) acc = dadd(acc, dmul(qd[i], row[i]));
      const double nr = ib ? t.bnorm[s] : t.rnorm[s];
      ssim[r] = clamp1(ddiv(acc, dmul(nq, nr)));
      skey[r] = 2LL * t.cid[s] + (ib ? 1 : 0);
    }
    __syncthreads();
    block_rank_select(ssim, skey, ns_, take, order);
    if (threadIdx.x < take) order[threadIdx.x] = sset[order[threadIdx.x]];
    __syncthreads();
    }
    K4MARK(3)
    if (threadIdx.x < take) {
      const int b = order[threadIdx.x];
      if (pass == 0) {
        rank_slot[threadIdx.x] = cslot[b];
        a.ranked_slot[l * a.k_s + threadIdx.x] = cslot[b];
        a.ranked_buf[l * a.k_s + threadIdx.x] = cbuf[b];
      } else {
        a.pf_slot[l * a.prefetch_k + threadIdx.x] = cslot[b];
        a.pf_buf[l * a.prefetch_k + threadIdx.x] = cbuf[b];
      }
    }
    if (threadIdx.x == 0) {
      if (pass == 0) {
        a.n_ranked[l] = take;
        n_rank_s = take;
      } else {
        a.n_pf[l] = take;
      }
    }
    __syncthreads();
  }
  if (passes == 1 && threadIdx.x == 0) a.n_pf[l] = 0;
  if (degen && threadIdx.x == 0) set_err(t, DERR_DEGENERATE);

  // ---- verified (dedup in rank order, retrieval.cpp:20-26), attended count, page descriptors
  __shared__ int vnp[64], vnbp[64], voff[65];
  __shared__ int ring_cnt[64], ring_off[65];
  __shared__ unsigned long long ring_mask[64];
  if (threadIdx.x == 0) {
    int nv = 0;
    for (int i = 0; i < n_rank_s; ++i) {
      const int s = rank_slot[i];
      bool dup = false;
      for (int j = 0; j < nv; ++j) dup |= vers[j] == s;
      if (!dup) vers[nv++] = s;
    }
    nver_s = nv;
    a.n_ver[l] = nv;
  }
  __syncthreads();
  const int nv = nver_s;
  const int W = t.W, rpp = t.rpp;
  if (threadIdx.x < nv) {  // per verified cluster: counts (parallel global loads)
    const int s = vers[threadIdx.x];
    a.ver_slot[l * a.k_s + threadIdx.x] = s;
    vnp[threadIdx.x] = t.npages[s];
    vnbp[threadIdx.x] = t.nbpages[s];
    atomicAdd(&att_s, static_cast<unsigned long long>(t.nmem[s] + t.nbuf[s]));
    if (t.lazy[s]) lazy_any = 1;  // a pending split: the host must settle before the next step
  }
  if (threadIdx.x < 64) {
    ring_cnt[threadIdx.x] = 0;
    ring_mask[threadIdx.x] = 0ull;
  }
  __syncthreads();
  if (threadIdx.x == 0) a.flags[l] = lazy_any;
  K4MARK(4)
  // window ring: tokens whose owner is not a verified cluster (retrieval.cpp:107-108 dedup)
  {
    unsigned long long mine = 0;
    const int n_ring = W * t.tmax;
    const int n_pad = (n_ring + blockDim.x - 1) / blockDim.x * blockDim.x;  // warp-uniform trip count
    for (int i = threadIdx.x; i < n_pad; i += blockDim.x) {
      const int rs = i / t.tmax, tt = i - rs * t.tmax;
      bool keep = i < n_ring && tt < ring_count_s[rs];
      if (keep) {
        const int own = owners[i];
        for (int j = 0; j < nv; ++j) keep &= vers[j] != own;
      }
      // page-level counts: lanes of a warp mostly share a page -> one atomic per (warp, page)
      const int pg = keep ? rs * rpp + tt / t.P : -1;
      const unsigned km = __ballot_sync(kFull, keep);
      mine += keep ? 1 : 0;
      if (km) {
        const unsigned same = __match_any_sync(kFull, pg);
        if (keep && pg < 64 && (threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&ring_cnt[pg], __popc(same));
        const unsigned long long bit = keep ? 1ull << (tt % t.P) : 0ull;  // one shared atomic per (warp, page)
        const unsigned blo = __reduce_or_sync(same, static_cast<unsigned>(bit));
        const unsigned bhi = __reduce_or_sync(same, static_cast<unsigned>(bit >> 32));
        if (keep && pg < 64 && (threadIdx.x & 31) == __ffs(same) - 1)
          atomicOr(&ring_mask[pg], (static_cast<unsigned long long>(bhi) << 32) | blo);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(kFull, mine, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&att_s, mine);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int o = 0;
    for (int j = 0; j < nv; ++j) {
      voff[j] = o;
      o += vnp[j] + vnbp[j];
    }
    voff[nv] = o;
    for (int i = 0; i < W * rpp && i < 64; ++i) {
      ring_off[i] = o;
      o += ring_cnt[i] > 0 ? 1 : 0;
    }
    ring_off[min(W * rpp, 64)] = o;
    if (o > a.max_desc) {
      set_err(t, DERR_ITEMS);
      o = a.max_desc;
    }
    a.n_desc[l] = o;
    a.n_items[l] = (o + a.chunk_pages - 1) / a.chunk_pages;
    a.attended[l] = static_cast<int64_t>(att_s);
  }
  __syncthreads();
  K4MARK(5)
  int4* desc = a.desc + static_cast<int64_t>(l) * a.max_desc;
  const int ndesc = voff[nv];
  for (int i = threadIdx.x; i < ndesc && i < a.max_desc; i += blockDim.x) {
    int j = 0;
    while (j + 1 < nv && voff[j + 1] <= i) ++j;
    const int s = vers[j];
    const int k = i - voff[j];
    const bool isb = k >= vnp[j];
    const int page = isb ? t.bpages[static_cast<int64_t>(s) * t.maxbp + (k - vnp[j])]
                         : t.pages[static_cast<int64_t>(s) * t.maxp + k];
    desc[i] = make_int4(page, t.pg_fill[page] | ((isb ? 1 : 0) << 16), -1, -1);
  }
  for (int i = threadIdx.x; i < W * rpp && i < 64; i += blockDim.x)
    if (ring_cnt[i] > 0 && ring_off[i] < a.max_desc) {
      const int rs = i / rpp, j = i % rpp;
      const int page = t.ring_pages[(static_cast<int64_t>(l) * W + rs) * rpp + j];
      desc[ring_off[i]] = make_int4(page, t.pg_fill[page] | (2 << 16), static_cast<int>(ring_mask[i] & 0xffffffffu),
                                    static_cast<int>(ring_mask[i] >> 32));
    }
  __syncthreads();
  K4MARK(6)
#undef K4MARK
  if (threadIdx.x == 0) {  // errors raised so far (this block's own are ordered before the read)
    __threadfence();
    a.errw[l] = atomicOr(t.err, 0);
  }
  if (a.n_items[l] == 0)  // nothing attended: output zeros
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
      a.out[static_cast<int64_t>(l) * d + i] = 0.f;
      for (int r = 0; r < a.peer.n; ++r) a.peer.out[r][static_cast<int64_t>(a.peer.dom_offset + l) * d + i] = 0.f;
    }
}

// Block-wide exclusive scan of one int per thread (blockDim.x a multiple of 32, <= 1024);
// `tot` (>= 32 ints of shared scratch) receives the warp totals. Returns the thread's prefix;
// *total gets the block sum. Two barriers.
__device__ __forceinline__ int block_excl_scan(int v, int* tot, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < nw ? tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) tot[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const int before = warp > 0 ? tot[warp - 1] : 0;
  *total = tot[nw - 1];
  return before + x - v;
}

// The value of the entry of rank `kth` under (v desc, key asc) among n float entries (keys unique):
// rank counting with `sp` threads per entry (partial counts combined by shuffles), so n = 256
// candidates cost 256 / sp broadcast shared reads per thread. Writes *out; ends with a barrier.
__device__ void block_kth_value(const float* v, const long long* key, int n, int kth, float* out) {
  int sp = 1;
  while (sp < 32 && n * sp * 2 <= static_cast<int>(blockDim.x)) sp <<= 1;
  const int groups = blockDim.x / sp;
  const int part = threadIdx.x & (sp - 1);
  for (int base = 0; base < n; base += groups) {
    const int i = base + static_cast<int>(threadIdx.x) / sp;
    int r = 0;
    float vi = 0.f;
    if (i < n) {
      vi = v[i];
      const long long ki = key[i];
      for (int j = part; j < n; j += sp) {
        const float vj = v[j];
        r += (vj > vi || (vj == vi && key[j] < ki)) ? 1 : 0;
      }
    }
    for (int o = sp >> 1; o > 0; o >>= 1) r += __shfl_xor_sync(kFull, r, o);
    if (i < n && part == 0 && r == kth) *out = vi;
  }
  __syncthreads();
}

// ============================================================================ K6
__device__ __forceinline__ void mbar_init(uint64_t* bar, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct StageMeta {
  int dom, item, page, fill;
  int kind, flags;                 // flags: 1 first page of item, 2 last page, 4 end of work
  unsigned long long mask;         // tokens of the page to attend (window pages: K4's dedup)
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Warp-specialised split-KV attention. Warp ATT_WARPS (the producer) walks the page descriptors
// of claimed items and issues TMA bulk copies (K rows, V rows and the domain's query) into a ring
// of STAGES shared-memory stages, with L2 evict-first hints so the streamed K/V do not evict the
// cluster representatives K4 re-reads every step; "full" mbarriers carry the transaction bytes.
// The ATT_WARPS consumer warps process a 64-token sub-tile 8 tokens per warp, 4 lanes per token
// (D/4 dims, two accumulators), keep a per-warp online softmax, and release each stage through
// an "empty" mbarrier (no CTA-wide barrier per page). At the end of an item the consumers merge
// their states (named barrier) into a partial; the last CTA to finish a domain combines them.
constexpr int ATT_THREADS = 256;
constexpr int ATT_CHUNK = 8;  // pages per attention work item (DecodeArgs::chunk_pages)
constexpr int ATT_WARPS = ATT_THREADS / 32;

template <int D, bool BF16, int STAGES>
__global__ void __launch_bounds__(ATT_THREADS + 32) k_attend(DevTables t, DecodeArgs a, int* work_ctr) {
  constexpr int ES = BF16 ? 2 : 4;
  constexpr int ROWB = D * ES;
  constexpr int OPL = D / 32;   // output dims per lane
  extern __shared__ __align__(128) uint8_t sm6[];
  const int P = t.P;
  const int64_t kv_bytes = static_cast<int64_t>(2) * P * ROWB;
  const int64_t stage_bytes = kv_bytes + D * 4;  // K rows, V rows, query (fp32)
  uint8_t* stages = sm6;
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  __shared__ StageMeta meta[STAGES];
  __shared__ int prefix[1025];
  __shared__ float wm[ATT_WARPS], wl[ATT_WARPS];
  __shared__ float wo[ATT_WARPS][D];
  __shared__ int last_flag;
  __shared__ __align__(16) int4 pqd[2][ATT_CHUNK];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int L = min(t.L, 1024);
  // stale rows past a page's fill are read unmasked (and weighted by p = 0): keep them finite
  for (int64_t i = tid; i < STAGES * stage_bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(stages)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ATT_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // launched as a programmatic dependent of K4: everything above overlapped K4's tail; the work
  // list is read only after K4 completed and flushed (a no-op without the launch attribute)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int l = tid; l < L; l += blockDim.x) prefix[l + 1] = a.n_items[l];
  __syncthreads();
  if (tid == 0) {
    prefix[0] = 0;
    for (int l = 0; l < L; ++l) prefix[l + 1] += prefix[l];
  }
  __syncthreads();
  const int total = prefix[L];

  if (warp == ATT_WARPS) {
    // ================================================================ producer warp
    if (lane != 0) return;
    const uint64_t pol = policy_evict_first();
    // Items are claimed on demand (claiming ahead parks the last items behind busy CTAs and
    // lengthens the tail); the claimed item's descriptors arrive by cp.async into shared memory.
    int cb = 0, g_cur = 0, c_dom = 0, c_j = 0, c_n = 0, p_k = 0;
    for (int it = 0;; ++it) {
      const int s = it % STAGES;
      if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
      StageMeta& m = meta[s];
      if (p_k >= c_n) {  // claim the next item
        g_cur = atomicAdd(work_ctr, 1);
        if (g_cur >= total) {
          m.flags = 4;
          mbar_arrive(&full[s]);
          break;
        }
        int lo = 0, hi = L;
        while (hi - lo > 1) {
          const int mid = (lo + hi) / 2;
          if (prefix[mid] <= g_cur) lo = mid; else hi = mid;
        }
        c_dom = lo;
        c_j = g_cur - prefix[lo];
        c_n = min(a.chunk_pages, a.n_desc[c_dom] - c_j * a.chunk_pages);
        const int4* src = a.desc + static_cast<int64_t>(c_dom) * a.max_desc + c_j * a.chunk_pages;
        for (int i = 0; i < c_n; ++i)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&pqd[cb][i])), "l"(src + i) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_all;" ::: "memory");
        p_k = 0;
      }
      const int4 dsc = pqd[cb][p_k];
      m.dom = c_dom;
      m.item = c_j;
      m.page = dsc.x;
      m.fill = dsc.y & 0xffff;
      m.kind = dsc.y >> 16;
      m.mask = (static_cast<unsigned long long>(static_cast<uint32_t>(dsc.w)) << 32) | static_cast<uint32_t>(dsc.z);
      m.flags = (p_k == 0 ? 1 : 0) | (p_k == c_n - 1 ? 2 : 0);
      const uint32_t bytes = static_cast<uint32_t>(m.fill) * ROWB;
      uint8_t* dst = stages + s * stage_bytes;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(&full[s], 2 * bytes + D * 4);
      bulk_g2s_hint(dst, page_k(t, m.page), bytes, &full[s], pol);
      bulk_g2s_hint(dst + static_cast<int64_t>(P) * ROWB, page_v(t, m.page), bytes, &full[s], pol);
      bulk_g2s(dst + kv_bytes, a.q + static_cast<int64_t>(m.dom) * D, D * 4, &full[s]);
      // the item's page PF_AHEAD ahead goes DRAM -> L2 now (no shared memory held): more bytes in
      // flight than the two shared-memory stages carry at loaded-DRAM latency
      if (a.att_pf > 0 && p_k + a.att_pf < c_n) {
        const int4 nd = pqd[cb][p_k + a.att_pf];
        if (!is_host_page(t, nd.x)) {
          const uint32_t nb = static_cast<uint32_t>(nd.y & 0xffff) * ROWB;
          if (nb) {
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(page_k(t, nd.x)), "r"(nb) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(page_v(t, nd.x)), "r"(nb) : "memory");
          }
        }
      }
      p_k += 1;
    }
    return;
  }

  // ================================================================== consumer warps
  // Lane l owns head dims [l*OPL, l*OPL + OPL) for both q.k (query in registers) and p.v. A warp
  // takes 8 tokens of a 64-token sub-tile: each lane forms 8 partial dots over its dims, a
  // transpose-reduce (7 shuffles) + 2 butterfly steps leaves token j's full score in the lanes
  // whose bits 4,3,2 encode j; softmax statistics then need 3 shuffles each.
  float m_run = -INFINITY, l_run = 0.f;
  float o_run[OPL];
  float qr[OPL];
#pragma unroll
  for (int i = 0; i < OPL; ++i) o_run[i] = qr[i] = 0.f;
  int cur_dom = -1;
  const float sl2 = a.scale_log2;
  const int my_tok = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);

  for (int it = 0;; ++it) {
    const int s = it % STAGES;
    mbar_wait(&full[s], (it / STAGES) & 1);
    const StageMeta& m = meta[s];
    const int flags = m.flags;
    if (flags & 4) break;
    const int fill = m.fill;
    const uint8_t* Ks = stages + s * stage_bytes;
    const uint8_t* Vs = Ks + static_cast<int64_t>(P) * ROWB;
    if (m.dom != cur_dom) {  // the domain's query (carried by every stage)
      const float* qs = reinterpret_cast<const float*>(Ks + kv_bytes);
#pragma unroll
      for (int i = 0; i < OPL; ++i) qr[i] = qs[lane * OPL + i];
      cur_dom = m.dom;
    }
    for (int tb = 0; tb < ((a.debug_flags & 1) ? 0 : fill); tb += 64) {
      const int t0 = tb + warp * 8;  // this warp's first token
      if (t0 >= fill) continue;      // warp-uniform
      // ---- partial dots: 8 tokens x OPL dims per lane. Rows at or past `fill` hold finite stale
      // data (stages are zeroed at start), so no per-token bounds tests: they are masked below.
      float v[8];
      const uint8_t* kbase = Ks + static_cast<int64_t>(t0) * ROWB + lane * OPL * ES;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float acc = 0.f;
        const uint8_t* krow = kbase + j * ROWB;
        if (BF16) {
#pragma unroll
          for (int i = 0; i < OPL; i += 2) {
            const uint32_t w = *reinterpret_cast<const uint32_t*>(krow + i * 2);
            acc = fmaf(__uint_as_float(w << 16), qr[i], acc);
            if (i + 1 < OPL) acc = fmaf(__uint_as_float(w & 0xffff0000u), qr[i + 1], acc);
          }
        } else {
#pragma unroll
          for (int i = 0; i < OPL; ++i) acc = fmaf(reinterpret_cast<const float*>(krow)[i], qr[i], acc);
        }
        v[j] = acc;
      }
      // ---- transpose-reduce: xor 16 (8 -> 4 values), xor 8 (4 -> 2), xor 4 (2 -> 1)
      float w4[4], w2[2];
      const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float send = b4 ? v[i] : v[i + 4];
        const float keep = b4 ? v[i + 4] : v[i];
        w4[i] = keep + __shfl_xor_sync(kFull, send, 16);
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const float send = b3 ? w4[i] : w4[i + 2];
        const float keep = b3 ? w4[i + 2] : w4[i];
        w2[i] = keep + __shfl_xor_sync(kFull, send, 8);
      }
      float dot;
      {
        const float send = b2 ? w2[0] : w2[1];
        const float keep = b2 ? w2[1] : w2[0];
        dot = keep + __shfl_xor_sync(kFull, send, 4);
      }
      dot += __shfl_xor_sync(kFull, dot, 1);
      dot += __shfl_xor_sync(kFull, dot, 2);
      // lane holds token my_tok = (b4,b3,b2) of this warp's 8
      const int tok = t0 + my_tok;
      const bool valid = tok < fill && ((m.mask >> tok) & 1ull);  // window pages: K4's dedup mask
      const float sc = valid ? dot * sl2 : -INFINITY;
      float mx = sc;
      mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 4));
      mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 8));
      mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 16));
      const float m_new = fmaxf(m_run, mx);
      if (m_new == -INFINITY) continue;  // warp-uniform
      const float alpha = exp2f(m_run - m_new);
      const float pr = valid ? exp2f(sc - m_new) : 0.f;
      float psum = (lane & 3) == 0 ? pr : 0.f;
      psum += __shfl_xor_sync(kFull, psum, 4);
      psum += __shfl_xor_sync(kFull, psum, 8);
      psum += __shfl_xor_sync(kFull, psum, 16);
      l_run = l_run * alpha + psum;
#pragma unroll
      for (int i = 0; i < OPL; ++i) o_run[i] *= alpha;
      m_run = m_new;
      // ---- p.v: token j's probability lives in lane (j>>2&1)*16 + (j>>1&1)*8 + (j&1)*4
      const uint8_t* vbase = Vs + static_cast<int64_t>(t0) * ROWB + lane * OPL * ES;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int src = ((j >> 2) & 1) * 16 + ((j >> 1) & 1) * 8 + (j & 1) * 4;
        const float pj = __shfl_sync(kFull, pr, src);  // 0 for masked / past-fill tokens
        const uint8_t* vrow = vbase + j * ROWB;
        if (BF16) {
#pragma unroll
          for (int i = 0; i < OPL; i += 2) {
            const uint32_t w = *reinterpret_cast<const uint32_t*>(vrow + i * 2);
            o_run[i] = fmaf(pj, __uint_as_float(w << 16), o_run[i]);
            if (i + 1 < OPL) o_run[i + 1] = fmaf(pj, __uint_as_float(w & 0xffff0000u), o_run[i + 1]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < OPL; ++i) o_run[i] = fmaf(pj, reinterpret_cast<const float*>(vrow)[i], o_run[i]);
        }
      }
    }
    const int dom = m.dom, item = m.item;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // stage s released by this warp
    if (flags & 2) {  // item done: merge the warps, write the partial, maybe combine the domain
      if (lane == 0) {
        wm[warp] = m_run;
        wl[warp] = l_run;
      }
#pragma unroll
      for (int i = 0; i < OPL; ++i) wo[warp][lane * OPL + i] = o_run[i];
      named_sync(1, ATT_THREADS);
      float M = -INFINITY;
      for (int w = 0; w < ATT_WARPS; ++w) M = fmaxf(M, wm[w]);
      const int64_t pi = static_cast<int64_t>(dom) * a.max_items + item;
      for (int c = tid; c < D; c += ATT_THREADS) {
        float o = 0.f;
        for (int w = 0; w < ATT_WARPS; ++w)
          if (wm[w] != -INFINITY) o += wo[w][c] * exp2f(wm[w] - M);
        a.part_o[pi * D + c] = o;
      }
      if (tid == 0) {
        float lsum = 0.f;
        for (int w = 0; w < ATT_WARPS; ++w)
          if (wm[w] != -INFINITY) lsum += wl[w] * exp2f(wm[w] - M);
        a.part_ml[pi * 2] = M;
        a.part_ml[pi * 2 + 1] = lsum;
      }
      // the consumers' partial writes are ordered before the barrier; ONE gpu-scope fence by the
      // signalling thread after it is cumulative over them (as a grid barrier's release), so the
      // other 255 threads no longer stall on a membar per item
      named_sync(1, ATT_THREADS);
      if (tid == 0) {
        __threadfence();
        last_flag = (atomicAdd(&a.dom_done[dom], 1) + 1 == a.n_items[dom]);
      }
      named_sync(1, ATT_THREADS);
      if (last_flag) {  // split-KV combine of all partials of the domain
        __threadfence();
        const int ni = a.n_items[dom];
        const float* ml = a.part_ml + static_cast<int64_t>(dom) * a.max_items * 2;
        float MM = -INFINITY;
        for (int i = 0; i < ni; ++i) MM = fmaxf(MM, ml[2 * i]);
        for (int c = tid; c < D; c += ATT_THREADS) {
          float num = 0.f, den = 0.f;
          for (int i = 0; i < ni; ++i) {
            if (ml[2 * i] == -INFINITY) continue;
            const float w = exp2f(ml[2 * i] - MM);
            num += w * a.part_o[(static_cast<int64_t>(dom) * a.max_items + i) * D + c];
            den += w * ml[2 * i + 1];
          }
          const float v = den > 0.f ? num / den : 0.f;
          a.out[static_cast<int64_t>(dom) * D + c] = v;
          if (a.peer.n) {  // fused exchange: the row goes straight to every rank over peer memory
            for (int r = 0; r < a.peer.n; ++r) a.peer.out[r][static_cast<int64_t>(a.peer.dom_offset + dom) * D + c] = v;
          }
        }
        if (tid == 0) a.dom_done[dom] = 0;
      }
      m_run = -INFINITY;
      l_run = 0.f;
#pragma unroll
      for (int i = 0; i < OPL; ++i) o_run[i] = 0.f;
      named_sync(1, ATT_THREADS);  // wo / last_flag reuse
    }
  }
}

// Attention for head widths without a K6 instantiation (d not in {32, 64, 128, 256}; the
// reference's own tests use d = 8, 16, ...): one CTA per domain walks the domain's page
// descriptors (the same work list K6 reads), a warp per token with lanes over the dims
// (warp-reduced q.k), online softmax in exp2 space per warp, warps merged at the end. Not a
// bandwidth path -- the headline shapes take K6.
constexpr int AG_WARPS = 8;
constexpr int AG_MAXD = 256;
__global__ void __launch_bounds__(AG_WARPS * 32) k_attend_generic(DevTables t, DecodeArgs a) {
  const int l = blockIdx.x, d = t.d, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ float qs[AG_MAXD];
  __shared__ float wm[AG_WARPS], wl[AG_WARPS];
  __shared__ float wo[AG_WARPS][AG_MAXD];
  if (a.n_items[l] == 0) return;  // K4 wrote the zero row
  for (int i = threadIdx.x; i < d; i += blockDim.x) qs[i] = a.q[static_cast<int64_t>(l) * d + i];
  __syncthreads();
  float m = -INFINITY, lsum = 0.f, o[AG_MAXD / 32];
#pragma unroll
  for (int k = 0; k < AG_MAXD / 32; ++k) o[k] = 0.f;
  const int nd = a.n_desc[l];
  int tok = 0;  // running token index over the domain's attended pages
  for (int di = 0; di < nd; ++di) {
    const int4 dsc = a.desc[static_cast<int64_t>(l) * a.max_desc + di];
    const int fill = dsc.y & 0xffff;
    const unsigned long long mask =
        (static_cast<unsigned long long>(static_cast<uint32_t>(dsc.w)) << 32) | static_cast<uint32_t>(dsc.z);
    const uint8_t* kp = page_k(t, dsc.x);
    const uint8_t* vp = page_v(t, dsc.x);
    for (int r = 0; r < fill; ++r, ++tok) {
      if (((mask >> r) & 1ull) == 0 || tok % AG_WARPS != warp) continue;
      float dot = 0.f;
      for (int i = lane; i < d; i += 32) {
        const float kv = t.kv_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(kp)[static_cast<int64_t>(r) * d + i])
                                   : reinterpret_cast<const float*>(kp)[static_cast<int64_t>(r) * d + i];
        dot = fmaf(qs[i], kv, dot);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
      const float s2 = dot * a.scale_log2;
      const float mn = fmaxf(m, s2);
      const float corr = exp2f(m - mn), p = exp2f(s2 - mn);
      lsum = lsum * corr + p;
#pragma unroll
      for (int k = 0; k < AG_MAXD / 32; ++k) {
        const int i = lane + 32 * k;
        if (i < d) {
          const float vv = t.kv_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(vp)[static_cast<int64_t>(r) * d + i])
                                     : reinterpret_cast<const float*>(vp)[static_cast<int64_t>(r) * d + i];
          o[k] = o[k] * corr + p * vv;
        }
      }
      m = mn;
    }
  }
  if (lane == 0) {
    wm[warp] = m;
    wl[warp] = lsum;
  }
#pragma unroll
  for (int k = 0; k < AG_MAXD / 32; ++k)
    if (lane + 32 * k < d) wo[warp][lane + 32 * k] = o[k];
  __syncthreads();
  float M = -INFINITY;
  for (int w = 0; w < AG_WARPS; ++w) M = fmaxf(M, wm[w]);
  float den = 0.f;
  for (int w = 0; w < AG_WARPS; ++w)
    if (wm[w] != -INFINITY) den += wl[w] * exp2f(wm[w] - M);
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float num = 0.f;
    for (int w = 0; w < AG_WARPS; ++w)
      if (wm[w] != -INFINITY) num += wo[w][i] * exp2f(wm[w] - M);
    const float v = den > 0.f ? num / den : 0.f;
    a.out[static_cast<int64_t>(l) * d + i] = v;
    for (int r = 0; r < a.peer.n; ++r) a.peer.out[r][static_cast<int64_t>(a.peer.dom_offset + l) * d + i] = v;
  }
}

// flat top-k over an explicit candidate list (one CTA). The (sim, key, taken) arrays live in
// shared memory when they fit, else in the caller's global scratch (`gscratch`, n * 17 bytes).
__global__ void __launch_bounds__(256) k_flat_topk(DevTables t, const float* q, const int32_t* slots,
                                                   const uint8_t* bufs, int n, int k, int32_t* out,
                                                   uint8_t* gscratch) {
  extern __shared__ uint8_t smf[];
  double* sim = reinterpret_cast<double*>(gscratch ? gscratch : smf);
  long long* key = reinterpret_cast<long long*>(sim + n);
  uint8_t* taken = reinterpret_cast<uint8_t*>(key + n);
  __shared__ double red_s[32];
  __shared__ long long red_k[32];
  __shared__ int red_i[33];
  __shared__ float qf[256];
  __shared__ double nq;
  const int d = t.d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) qf[i] = q[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < d; ++i) s = dadd(s, dmul(static_cast<double>(qf[i]), static_cast<double>(qf[i])));
    nq = __dsqrt_rn(s);
  }
  __syncthreads();
  bool dg = false;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    if (!slots) {  // visual_topk (index.cpp:192-208): partitions 0..n-1, ties to the lower id
      sim[c] = exact_cos(qf, nq, t.vrep + static_cast<int64_t>(c) * d, t.vnorm[c], d, dg);
      key[c] = c;
    } else {
      const int s = slots[c];
      const bool ib = bufs[c];
      sim[c] = exact_cos(qf, nq, (ib ? t.brep64 : t.rep64) + static_cast<int64_t>(s) * d,
                         ib ? t.bnorm[s] : t.rnorm[s], d, dg);
      key[c] = 2LL * t.cid[s] + (ib ? 1 : 0);
    }
    taken[c] = 0;
  }
  if (dg) set_err(t, DERR_DEGENERATE);
  __syncthreads();
  const int take = min(n, k);
  for (int i = 0; i < take; ++i) {
    const int b = block_take_best(sim, key, taken, n, red_s, red_k, red_i);
    if (threadIdx.x == 0) out[i] = b;
  }
}

}  // namespace

// ============================================================================ launchers

int launch_build_cands(const DevTables& t, const IngestArgs& a, cudaStream_t st) {
  launch_pdl(k_build_cands, dim3(a.n_active), dim3(256), 0, st, t, a);
  return 1;
}

int launch_approx(const DevTables& t, const IngestArgs& a, cudaStream_t st) {
  const int dp = t.d + 1;
  const size_t smem = static_cast<size_t>(AT * dp + AC * dp + AT + AC) * 4;
  if (!smem_optin(reinterpret_cast<const void*>(k_approx), smem)) return 0;
  dim3 g((a.T + AT - 1) / AT, a.n_active);
  k_approx<<<g, 256, smem, st>>>(t, a);
  return 1;
}

int launch_resolve(const DevTables& t, const IngestArgs& a, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(HOT) * 2 * padded(t.d) * 8 + static_cast<size_t>(6) * padded(t.d) * 8 +
                      static_cast<size_t>(t.tmax) * (8 + TOPM * (8 + 4 + 2) + 4) + 16 +
                      static_cast<size_t>(t.cmax) * (8 + 4 + 3) + 64;
  if (!smem_optin(reinterpret_cast<const void*>(k_resolve), smem)) return 0;
  k_resolve<<<a.n_active, 32, smem, st>>>(t, a);
  return 1;
}

int launch_store_rows(const DevTables& t, const IngestArgs& a, cudaStream_t st) {
  dim3 g((a.T + 7) / 8, a.n_active);  // one warp per row
  launch_pdl(k_store_rows, g, dim3(256), 0, st, t, a);
  return 1;
}

int launch_topm(const DevTables& t, const IngestArgs& a, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(8) * t.cmax * 4;
  if (!smem_optin(reinterpret_cast<const void*>(k_topm), smem)) return 0;
  dim3 g((a.T + 7) / 8, a.n_active);
  k_topm<<<g, 256, smem, st>>>(t, a);
  return 1;
}

int launch_ring_write(const DevTables& t, const void* fk, const void* fv, int32_t T, int32_t rs,
                      cudaStream_t st) {
  dim3 g(1, t.L);
  k_ring_write<<<g, 256, 0, st>>>(t, static_cast<const uint8_t*>(fk), static_cast<const uint8_t*>(fv), T, rs);
  return 1;
}

int launch_ring_rows(const DevTables& t, const void* fk, const void* fv, int32_t T, int32_t rs, cudaStream_t st) {
  dim3 g((T + 7) / 8, t.L);
  k_ring_rows<<<g, 256, 0, st>>>(t, static_cast<const uint8_t*>(fk), static_cast<const uint8_t*>(fv), T, rs);
  return 1;
}

int launch_append_runs(const DevTables& t, const AppendRun* runs, int32_t n_runs, const int32_t* idx,
                       const void* sk, const void* sv, cudaStream_t st) {
  if (n_runs <= 0) return 0;
  k_append_runs<<<n_runs, 256, 0, st>>>(t, runs, n_runs, idx, static_cast<const uint8_t*>(sk),
                                       static_cast<const uint8_t*>(sv));
  return 1;
}

int launch_gather_cluster(const DevTables& t, int32_t slot, int32_t with_buf, void* sk, void* sv,
                          int64_t row0, cudaStream_t st) {
  const int blocks = t.maxp + (with_buf ? t.maxbp : 0);
  k_gather_cluster<<<blocks, 128, 0, st>>>(t, slot, with_buf, static_cast<uint8_t*>(sk),
                                           static_cast<uint8_t*>(sv), row0);
  return 1;
}

int launch_free_slot_pages(const DevTables& t, int32_t slot, cudaStream_t st) {
  k_free_slot<<<1, 128, 0, st>>>(t, slot);
  return 1;
}

int launch_refresh_mirror(const DevTables& t, const int32_t* slots, int32_t n, cudaStream_t st) {
  if (n <= 0) return 0;
  k_refresh_mirror<<<n, 128, 0, st>>>(t, slots, n);
  return 1;
}

int launch_exact_stats(const DevTables& t, const AppendRun* runs, int32_t n_runs, const int32_t* idx,
                       const void* sk, cudaStream_t st) {
  if (n_runs <= 0) return 0;
  const int threads = 128;
  const size_t smem = static_cast<size_t>(t.d + threads) * 8;
  k_exact_stats<<<n_runs, threads, smem, st>>>(t, runs, n_runs, idx, sk);
  return 1;
}

int launch_slot_headers(const DevTables& t, const SlotHeader* h, int32_t n, cudaStream_t st) {
  if (n <= 0) return 0;
  k_slot_headers<<<(n + 127) / 128, 128, 0, st>>>(t, h, n);
  return 1;
}

int launch_init_slots(const DevTables& t, const void* recs, int32_t n, cudaStream_t st) {
  if (n <= 0) return 0;
  k_init_slots<<<n, 128, 0, st>>>(t, static_cast<const uint8_t*>(recs), n);
  return 1;
}

int launch_to_f32(const DevTables& t, const void* src, float* dst, int64_t n, cudaStream_t st) {
  if (n <= 0) return 0;
  const int blocks = static_cast<int>((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  k_to_f32<<<blocks, 256, 0, st>>>(src, dst, n, t.kv_bf16);
  return 1;
}

int launch_flat_topk(const DevTables& t, const float* q, const int32_t* slots, const uint8_t* bufs,
                     int32_t n, int32_t k, int32_t* out, uint8_t* gscratch, cudaStream_t st) {
  const size_t bytes = static_cast<size_t>(n) * 17 + 16;
  const bool in_smem = bytes + 2048 <= static_cast<size_t>(device_smem_optin()) &&
                       smem_optin(reinterpret_cast<const void*>(k_flat_topk), bytes);
  if (!in_smem && !gscratch) return 0;
  k_flat_topk<<<1, 256, in_smem ? bytes : 0, st>>>(t, q, slots, bufs, n, k, out, in_smem ? nullptr : gscratch);
  return 1;
}

namespace {
int att_stages() {
  static const int stages = [] {
    const char* e = getenv("KVC_ATT_STAGES");
    const int s = e ? atoi(e) : 2;  // 2 stages -> 3 CTAs per SM (latency-bound consumers need the warps)
    return (s < 2 || s > 4) ? 2 : s;
  }();
  return stages;
}

template <int D, bool BF16, int STAGES>
int launch_attend_s(const DevTables& t, const DecodeArgs& a, cudaStream_t st, bool pdl) {
  const size_t smem = static_cast<size_t>(STAGES) * (2 * t.P * D * (BF16 ? 2 : 4) + D * 4);
  const void* fn = reinterpret_cast<const void*>(k_attend<D, BF16, STAGES>);
  if (!smem_optin(fn, smem)) return 0;  // the context constructor rejects such shapes
  const int per_sm = occupancy(fn, ATT_THREADS + 32, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(device_sms() * per_sm));
  cfg.blockDim = dim3(ATT_THREADS + 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr_pdl[1];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr_pdl;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_attend<D, BF16, STAGES>, t, a, a.work_ctr);
  return 1;
}

// Pipeline depth: KVC_ATT_STAGES (2..4) overrides the default of 2 (measured on B200: 2 stages x 3
// CTAs per SM beat 3 stages x 2 CTAs, 97 vs 104 us for config 2).
template <int D, bool BF16>
int launch_attend_t(const DevTables& t, const DecodeArgs& a, cudaStream_t st, bool pdl) {
  const int stages = att_stages();
  if (stages == 2) return launch_attend_s<D, BF16, 2>(t, a, st, pdl);
  if (stages == 4) return launch_attend_s<D, BF16, 4>(t, a, st, pdl);
  return launch_attend_s<D, BF16, 3>(t, a, st, pdl);
}
}  // namespace

namespace {
__global__ void k_peer_signal(unsigned long long* f0, unsigned long long* f1, unsigned long long* f2,
                              unsigned long long* f3, unsigned long long* f4, unsigned long long* f5,
                              unsigned long long* f6, unsigned long long* f7, int n, int rank,
                              unsigned long long step) {
  unsigned long long* f[8] = {f0, f1, f2, f3, f4, f5, f6, f7};
  const int r = threadIdx.x;
  __threadfence_system();  // this rank's output stores (earlier kernels) before the flag
  if (r < n) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f[r] + rank), "l"(step) : "memory");
}

__global__ void k_peer_wait(const unsigned long long* flags, int n, unsigned long long step) {
  if (threadIdx.x != 0) return;
  for (int q = 0; q < n; ++q) {
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + q) : "memory");
      if (v >= step) break;
      __nanosleep(200);
    }
  }
}
}  // namespace

int launch_peer_signal(unsigned long long* const* flags, int n, int rank, unsigned long long step, cudaStream_t st) {
  unsigned long long* f[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  for (int i = 0; i < n && i < 8; ++i) f[i] = flags[i];
  k_peer_signal<<<1, 32, 0, st>>>(f[0], f[1], f[2], f[3], f[4], f[5], f[6], f[7], n, rank, step);
  return 1;
}

int launch_peer_wait(const unsigned long long* my_flags, int n, unsigned long long step, cudaStream_t st) {
  k_peer_wait<<<1, 32, 0, st>>>(my_flags, n, step);
  return 1;
}

size_t attend_smem_bytes(int d, int page_tokens, bool bf16) {
  return static_cast<size_t>(att_stages()) * (2 * static_cast<size_t>(page_tokens) * d * (bf16 ? 2 : 4) + d * 4);
}

int launch_attend(const DevTables& t, const DecodeArgs& a, cudaStream_t st) {
  switch (t.d * 2 + t.kv_bf16) {
    case 64: return launch_attend_t<32, false>(t, a, st, false);
    case 65: return launch_attend_t<32, true>(t, a, st, false);
    case 128: return launch_attend_t<64, false>(t, a, st, false);
    case 129: return launch_attend_t<64, true>(t, a, st, false);
    case 256: return launch_attend_t<128, false>(t, a, st, false);
    case 257: return launch_attend_t<128, true>(t, a, st, false);
    case 512: return launch_attend_t<256, false>(t, a, st, false);
    case 513: return launch_attend_t<256, true>(t, a, st, false);
    default:
      if (t.d > AG_MAXD) return 0;
      k_attend_generic<<<t.L, AG_WARPS * 32, 0, st>>>(t, a);
      return 1;
  }
}

int launch_decode(const DevTables& t, const DecodeArgs& a, cudaStream_t st, cudaEvent_t* ev, cudaEvent_t k4_done) {
  if (ev) cudaEventRecord(ev[0], st);
  // K4 v3 (select.cu) whenever the shape fits it (d <= 128, d % 4 == 0, page_tokens % 32 == 0,
  // lists <= 64); otherwise, or with KVC_K4=v1 (read per step), the general staged variant
  // k_score_select (any d <= 256, any page size)
  const char* kv_env = getenv("KVC_K4");
  const bool force_v1 = kv_env && kv_env[0] == 'v' && kv_env[1] == '1';
  bool used3 = false;
  if (!force_v1 && launch_select3(t, a, st)) {
    used3 = true;
  } else {
    const size_t smem4 = k4_smem_bytes(t.d, t.cmax, a.n_parts_host, t.W, t.tmax);
    if (!smem_optin(reinterpret_cast<const void*>(k_score_select), smem4)) return 0;
    if (a.fr_on) cudaMemsetAsync(a.fr_n, 0, static_cast<size_t>(t.L) * 4, st);  // (fetch-on-read is K4 v3's)
    k_score_select<<<t.L, 256, smem4, st>>>(t, a, a.work_ctr);
  }
  // K6 is a programmatic dependent of K4 (PDL: its launch and prologue overlap K4) unless an event
  // has to be recorded between them (timing mode); k4_done then follows K6
  static int pdl_env = -1;
  if (pdl_env < 0) {
    const char* e = getenv("KVC_PDL");
    pdl_env = (e && e[0] == '0') ? 0 : 1;
  }
  const bool pdl = pdl_env && !ev && used3;
  int n = 1;
  if (a.fr_on && used3) n += launch_fetch_read(t, a, st, pdl);  // K4 -> fetch-on-read copies -> K6
  if (ev) cudaEventRecord(ev[1], st);
  if (k4_done && !pdl) cudaEventRecord(k4_done, st);
  switch (t.d * 2 + t.kv_bf16) {
    case 64: n += launch_attend_t<32, false>(t, a, st, pdl); break;
    case 65: n += launch_attend_t<32, true>(t, a, st, pdl); break;
    case 128: n += launch_attend_t<64, false>(t, a, st, pdl); break;
    case 129: n += launch_attend_t<64, true>(t, a, st, pdl); break;
    case 256: n += launch_attend_t<128, false>(t, a, st, pdl); break;
    case 257: n += launch_attend_t<128, true>(t, a, st, pdl); break;
    case 512: n += launch_attend_t<256, false>(t, a, st, pdl); break;
    case 513: n += launch_attend_t<256, true>(t, a, st, pdl); break;
    default:
      if (t.d <= AG_MAXD) {  // head widths K6 is not instantiated for
        k_attend_generic<<<t.L, AG_WARPS * 32, 0, st>>>(t, a);
        n += 1;
      }
      break;
  }
  if (k4_done && pdl) cudaEventRecord(k4_done, st);
  if (ev) {
    cudaEventRecord(ev[2], st);
    cudaEventRecord(ev[3], st);
  }
  return n;
}

}  // namespace kvc
