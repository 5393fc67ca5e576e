// resolve_spec.cu -- K2': speculate-and-verify resolve of one frame's inserts per domain.
//
// The reference inserts a frame's tokens one by one (Maintainer::on_insert,
// maintainer.cpp:88-176): arg-best over exact fp64 cosines against the *current* cluster
// states, Eq. 3/4 update of the winner, Eq. 5 test, branch. The sequential kernel (k_resolve)
// follows that chain token by token. This kernel breaks the chain:
//
//  * Given the routing (which candidate each token joins), the states are independent chains:
//    each ELEMENT of a representative evolves on its own, r'_i = (n r_i + k_i)/(n+1), with n
//    known in advance (stat_count + position in the cluster's chain) -- one thread per
//    (cluster, element) runs it without any synchronisation; the d-long sequential sums
//    (|k-r'|^2, |r'|, |b'|) of different tokens are independent (one thread per token); the
//    scalar variance / member-count recurrence and the decisions are one thread per cluster.
//  * Divisions on those chains use a precomputed correctly rounded reciprocal y = RN(1/(n+1))
//    and two FMA remainder corrections; the last one is Markstein's theorem (y within half an
//    ulp of 1/b and a faithful quotient q give RN(q + (a - bq) y) = RN(a/b)), so the result is
//    bit-identical to __ddiv_rn (checked on the device by kvc_debug_div_check).
//  * The routing is speculated from K1b's exact launch-time cosines and VERIFIED token by token
//    against the states it produces: a candidate whose state moved from r0 to r' has
//    |cos(k, r') - cos(k, r0)| <= |r'/|r'| - r0/|r0|| <= 2 |r' - r0| / |r0|; an untouched
//    candidate is bounded by its exact launch-time cosine (K1b) or its approximate score +
//    margin. Only candidates whose upper bound reaches the winner's lower bound get an exact
//    fp64 cosine in the reference's summation order; the CandidateRef arg-best then decides.
//  * The first token whose verified winner differs from the speculation restarts the
//    speculation there with the corrected winners (the prefix before it is exact). Each round
//    fixes at least one token, so the loop terminates.
//
// Every committed quantity is computed with the reference's operation order, so the state is
// bit-identical to the sequential kernel's. Output contract == k_resolve (ev_kind / ev_slot /
// ev_page / ev_row, ring owner, stop token / kind / slot, table writeback).
#include <cfloat>
#include <climits>

#include "devmath.cuh"

namespace kvc {
namespace {

using namespace dm;

constexpr int RS_THREADS = 512;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int FRESH_MAX = 64;  // buffers registered (DEFER onto an empty buffer) per launch
constexpr double kSlack = 1e-12;
constexpr double kApproxEps = 1e-11;  // |warp-parallel fp64 cosine - sequential cosine| bound (d <= 256)
constexpr double kMoveApprox = 1e-3;  // movement bound past which a touched candidate is settled by it


struct SpecSmem {
  uint32_t* keys;
  int ksw;  // keys: [Tl][ksw] 32-bit words (row padded by one word: conflict-free columns)
  long long* ckey;
  double* cnorm;
  int32_t* cslot;
  int16_t *sib, *cts;
  uint8_t* cbuf;
  int16_t *fr_birth, *fr_lc;
  int32_t *req_u, *req_ts;
  // per relative token [tmax]
  double *a_var, *a_rn, *a_bn, *sq, *db, *nk, *rcp, *rcpb;
  long long *a_stat, *a_nmem;
  int32_t* a_nbuf;
  int16_t *win, *vwin, *tsof, *ctok, *pos;
  uint8_t *kind, *a_lazy;
  double* tauw;  // [2 tmax] tau(nmem0 + j) per touched slot, at ts_off + ts
  // per touched slot [tmax]
  double *ts_var0, *ts_rn0, *ts_bn0;
  unsigned long long* ts_dbmax;  // ord_bits of the largest buffer movement bound
  long long *ts_stat0, *ts_nmem0, *ts_cid;
  int32_t *ts_slot, *ts_off, *ts_cnt, *ts_fill, *ts_nbuf0, *ts_np, *ts_nbp, *ts_fb;
  int16_t *ts_lc, *ts_cb;
  uint8_t *ts_lazy0, *ts_resid;
  int32_t *ts_np0, *ts_last, *ts_fill0, *ts_nbp0, *ts_blast, *ts_bfill0;  // page metadata at launch
  int32_t* ts_pbase;  // first new page of the slot in pagebuf (commit)
  double* ts_dsum;    // sum over the slot's chain of |r'_j - r'_{j-1}| (bounds |r' - r0|)
  // K1b outputs staged once: per relative token the top-M candidates, exact cosines, next value
  int16_t* tm_idx;
  double* tm_ex;
  float* tm_next;
  int32_t* pagebuf;
  int pagecap;
};

// One carving routine for host (base == nullptr: size only) and device.
__host__ __device__ inline size_t spec_carve(uint8_t* base, SpecSmem* s, int d, int es, int T, int tmax,
                                             int cmax) {
  size_t off = 0;
  auto take = [&](size_t bytes, size_t align) -> uint8_t* {
    off = (off + align - 1) & ~(align - 1);
    uint8_t* p = base ? base + off : nullptr;
    off += bytes;
    return p;
  };
  const int ksw = d * es / 4 + 1;
  s->ksw = ksw;
  s->keys = reinterpret_cast<uint32_t*>(take(static_cast<size_t>(T) * ksw * 4, 16));
  s->ckey = reinterpret_cast<long long*>(take(static_cast<size_t>(cmax) * 8, 8));
  s->cnorm = reinterpret_cast<double*>(take(static_cast<size_t>(cmax) * 8, 8));
  s->cslot = reinterpret_cast<int32_t*>(take(static_cast<size_t>(cmax) * 4, 4));
  s->sib = reinterpret_cast<int16_t*>(take(static_cast<size_t>(cmax) * 2, 2));
  s->cts = reinterpret_cast<int16_t*>(take(static_cast<size_t>(cmax) * 2, 2));
  s->cbuf = take(static_cast<size_t>(cmax), 1);
  s->fr_birth = reinterpret_cast<int16_t*>(take(FRESH_MAX * 2, 2));
  s->fr_lc = reinterpret_cast<int16_t*>(take(FRESH_MAX * 2, 2));
  s->req_u = reinterpret_cast<int32_t*>(take(FRESH_MAX * 4, 4));
  s->req_ts = reinterpret_cast<int32_t*>(take(FRESH_MAX * 4, 4));
  const size_t n = static_cast<size_t>(tmax);
  s->a_var = reinterpret_cast<double*>(take(n * 8, 8));
  s->a_rn = reinterpret_cast<double*>(take(n * 8, 8));
  s->a_bn = reinterpret_cast<double*>(take(n * 8, 8));
  s->sq = reinterpret_cast<double*>(take(n * 8, 8));
  s->db = reinterpret_cast<double*>(take(n * 8, 8));
  s->nk = reinterpret_cast<double*>(take(n * 8, 8));
  s->rcp = reinterpret_cast<double*>(take(n * 8, 8));
  s->rcpb = reinterpret_cast<double*>(take(n * 8, 8));
  s->a_stat = reinterpret_cast<long long*>(take(n * 8, 8));
  s->a_nmem = reinterpret_cast<long long*>(take(n * 8, 8));
  s->tauw = reinterpret_cast<double*>(take(2 * n * 8, 8));
  s->ts_var0 = reinterpret_cast<double*>(take(n * 8, 8));
  s->ts_rn0 = reinterpret_cast<double*>(take(n * 8, 8));
  s->ts_bn0 = reinterpret_cast<double*>(take(n * 8, 8));
  s->ts_dbmax = reinterpret_cast<unsigned long long*>(take(n * 8, 8));
  s->ts_stat0 = reinterpret_cast<long long*>(take(n * 8, 8));
  s->ts_nmem0 = reinterpret_cast<long long*>(take(n * 8, 8));
  s->ts_cid = reinterpret_cast<long long*>(take(n * 8, 8));
  s->a_nbuf = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->ts_slot = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->ts_off = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->ts_cnt = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->ts_fill = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->ts_nbuf0 = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->ts_np = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->ts_nbp = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->ts_fb = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->win = reinterpret_cast<int16_t*>(take(n * 2, 2));
  s->vwin = reinterpret_cast<int16_t*>(take(n * 2, 2));
  s->tsof = reinterpret_cast<int16_t*>(take(n * 2, 2));
  s->ctok = reinterpret_cast<int16_t*>(take(n * 2, 2));
  s->pos = reinterpret_cast<int16_t*>(take(n * 2, 2));
  s->ts_lc = reinterpret_cast<int16_t*>(take(n * 2, 2));
  s->ts_cb = reinterpret_cast<int16_t*>(take(n * 2, 2));
  s->kind = take(n, 1);
  s->a_lazy = take(n, 1);
  s->ts_lazy0 = take(n, 1);
  s->ts_resid = take(n, 1);
  s->ts_np0 = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->ts_last = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->ts_fill0 = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->ts_nbp0 = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->ts_blast = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->ts_bfill0 = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->ts_pbase = reinterpret_cast<int32_t*>(take(n * 4, 4));
  s->tm_ex = reinterpret_cast<double*>(take(n * TOPM * 8, 8));
  s->tm_next = reinterpret_cast<float*>(take(n * 4, 4));
  s->tm_idx = reinterpret_cast<int16_t*>(take(n * TOPM * 2, 16));
  s->ts_dsum = reinterpret_cast<double*>(take(n * 8, 8));
  s->pagecap = 3 * tmax + 8;
  s->pagebuf = reinterpret_cast<int32_t*>(take(static_cast<size_t>(s->pagecap) * 4, 4));
  return (off + 15) & ~static_cast<size_t>(15);
}

__device__ __forceinline__ double keyd(const SpecSmem& S, int u, int i, bool bf16) {
  if (bf16) {
    const uint32_t w = S.keys[u * S.ksw + (i >> 1)];
    return static_cast<double>(__uint_as_float((i & 1) ? (w & 0xffff0000u) : (w << 16)));
  }
  return static_cast<double>(__uint_as_float(S.keys[u * S.ksw + i]));
}

__device__ __forceinline__ bool buf_move(uint8_t k) { return k == EV_BUFJOIN || k == EV_DEFER; }

// Snapshot layout: element i of token u at ((i/4) tmax + u) 4 + i%4 -- a warp storing 32
// consecutive elements of one token writes 8 full sectors, a thread per token reads its
// elements as 32-byte quads that are contiguous across consecutive tokens.
__device__ __forceinline__ int64_t sidx(int i, int u, int tmax) {
  return (static_cast<int64_t>(i >> 2) * tmax + u) * 4 + (i & 3);
}

// Monotone 64-bit image of a double (block-wide max via integer atomics).
__device__ __forceinline__ unsigned long long ord_bits(double x) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_ord(unsigned long long o) {
  const unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
  return __longlong_as_double(static_cast<long long>(b));
}

// Block-wide exclusive scan of v over [0, n) by warp 0 (returns the total to lane 0).
__device__ int warp0_exscan(const int32_t* in_a, const int32_t* in_b, int32_t* out, int n, int lane) {
  int run = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const int v = i < n ? in_a[i] + (in_b ? in_b[i] : 0) : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (i < n) out[i] = run + x - v;
    run += __shfl_sync(kFull, x, 31);
  }
  return run;
}

// fp32 routing simulation for relaunch rounds (see the kernel): up to SIM_SLOTS touched candidates
// cached in the per-token scratch arrays a_var .. db (free until the first round's phase B).
constexpr int SIM_SLOTS = 12;
__device__ void simulate_routing(const DevTables& t, SpecSmem& S, const IngestArgs& a, int dom, int Tl, int nl,
                                 bool bf16, int lane) {
  const int d = t.d, q = d / 32;  // dimensions per lane (d % 32 == 0 here; else only partially)
  if (d % 32 != 0) return;
  const size_t room = 5 * static_cast<size_t>(t.tmax) * 8;
  const size_t per = static_cast<size_t>(d) * 4 + 16;
  const int slots = min(SIM_SLOTS, static_cast<int>(room / per));
  if (slots < 2) return;
  float* rep = reinterpret_cast<float*>(S.a_var);              // [slots][d]
  float* rn = rep + static_cast<size_t>(slots) * d;           // [slots] |rep|
  float* cnt = rn + slots;                                     // [slots] n
  for (int c = lane; c < nl; c += 32) S.cts[c] = -1;           // candidate -> slot
  __syncwarp();
  int used = 0;
  // the winner's updated state against the NEXT token, reduced together with its norm (one
  // butterfly instead of two when consecutive tokens meet the same cluster)
  int pre_sl = -1;
  float pre_dot = 0.f;
  float x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = j < q ? static_cast<float>(keyd(S, 0, lane + 32 * j, bf16)) : 0.f;
  for (int u = 0; u < Tl; ++u) {
    float xn[8];  // the next token's elements (for the fused reduction below)
#pragma unroll
    for (int j = 0; j < 8; ++j) xn[j] = (j < q && u + 1 < Tl) ? static_cast<float>(keyd(S, u + 1, lane + 32 * j, bf16)) : 0.f;
    const float nk = static_cast<float>(S.nk[u]);
    // lane k < TOPM holds top-M entry k: launch-time value when untouched; the touched ones get
    // the simulated state's cosine, one warp-wide dot each
    const int c = lane < TOPM ? S.tm_idx[u * TOPM + lane] : -1;
    const int csl = c >= 0 ? S.cts[c] : -1;
    float v = -INFINITY;
    if (c >= 0 && csl < 0) {
      const double e = S.tm_ex[u * TOPM + lane];
      v = isnan(e) ? -INFINITY : static_cast<float>(e);
    }
    long long key = c >= 0 ? S.ckey[c] : LLONG_MAX;
    if (c >= 0 && csl >= 0 && csl == pre_sl) v = pre_dot / (nk * rn[csl]);
    unsigned tm = __ballot_sync(0xffffffffu, c >= 0 && csl >= 0 && csl != pre_sl);
    while (tm) {
      const int k = __ffs(tm) - 1;
      tm &= tm - 1;
      const int sl = __shfl_sync(0xffffffffu, csl, k);
      float p = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < q) p = fmaf(x[j], rep[sl * d + lane + 32 * j], p);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
      if (lane == k) v = p / (nk * rn[sl]);
    }
    // arg-best over the top-M lanes (value desc, key asc)
    float bs = v;
    long long bk = key;
    int bc = c;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      const float so = __shfl_xor_sync(0xffffffffu, bs, o);
      const long long ko = __shfl_xor_sync(0xffffffffu, bk, o);
      const int co = __shfl_xor_sync(0xffffffffu, bc, o);
      if (so > bs || (so == bs && ko < bk)) {
        bs = so;
        bk = ko;
        bc = co;
      }
    }
    bc = __shfl_sync(0xffffffffu, bc, 0);
    if (bc < 0 || __shfl_sync(0xffffffffu, bs, 0) == -INFINITY) return;  // no proposal past here
    if (lane == 0) S.win[u] = static_cast<int16_t>(bc);
    int sl = S.cts[bc];
    __syncwarp();  // every lane read the map before lane 0 may rewrite it (racecheck: WAR)
    if (sl < 0 && used < slots) {  // the winner's launch-time state into a slot
      sl = used++;
      const int64_t sg = S.cslot[bc];
      const float* src = (S.cbuf[bc] ? t.brep32 : t.rep32) + sg * d;
      float ss = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < q) {
          const float r = src[lane + 32 * j];
          rep[sl * d + lane + 32 * j] = r;
          ss = fmaf(r, r, ss);
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) {
        rn[sl] = sqrtf(ss);
        cnt[sl] = static_cast<float>(S.cbuf[bc] ? t.nbuf[sg] : t.stat[sg]);
        S.cts[bc] = static_cast<int16_t>(sl);
      }
    }
    __syncwarp();
    pre_sl = -1;
    if (sl >= 0) {  // Eq. 3 in fp32: r' = (n r + k) / (n + 1)
      const float n = cnt[sl], inv = 1.f / (n + 1.f);
      float ss = 0.f, pn = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < q) {
          const int i = lane + 32 * j;
          const float r = (n * rep[sl * d + i] + x[j]) * inv;
          rep[sl * d + i] = r;
          ss = fmaf(r, r, ss);
          pn = fmaf(xn[j], r, pn);
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
        pn += __shfl_xor_sync(0xffffffffu, pn, o);
      }
      __syncwarp();  // (every lane read cnt[sl] above)
      if (lane == 0) {
        rn[sl] = sqrtf(ss);
        cnt[sl] = n + 1.f;
      }
      pre_sl = sl;
      pre_dot = pn;
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = xn[j];
  }
}

__global__ void __launch_bounds__(RS_THREADS, 1) k_resolve_spec(DevTables t, IngestArgs a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (launched as a dependent of K1)
  extern __shared__ __align__(16) uint8_t smraw[];
  SpecSmem S;
  spec_carve(smraw, &S, t.d, t.es, a.T, t.tmax, t.cmax);
  __shared__ int sh_nts, sh_te, sh_tfail, sh_nreq, sh_bad, sh_ntot, sh_nfresh, sh_ptotal, sh_nexact, sh_tie;
  __shared__ long long sh_prof[16];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = t.d, tmax = t.tmax, cmax = t.cmax;
  const int dom = a.active[blockIdx.x];
  const int T = a.T, cur = a.cursor[dom];
  const int Tl = T - cur;
  const int nl = a.cand_n[dom];
  const bool bf16 = t.kv_bf16 != 0;
  const double margin = static_cast<double>(a.margin);
  double* rsnap = a.rsnap + static_cast<int64_t>(dom) * d * tmax;
  double* bsnap = a.bsnap + static_cast<int64_t>(dom) * d * tmax;
  const int64_t orow0 = static_cast<int64_t>(dom) * tmax + cur;
  long long c0 = clock64();
  auto prof = [&](int k) {
    if (tid == 0) {
      const long long c1 = clock64();
      sh_prof[k] += c1 - c0;
      c0 = c1;
    }
  };

  // speculative round after a frame that stopped for host events: write nothing at all (the
  // outcome arrays still hold that frame's first round, which its relaunches copy back whole)
  if (a.prev_events && *a.prev_events) return;
  if (tid < 16) sh_prof[tid] = 0;
  if (tid == 0 && a.tie) a.tie[dom] = 0;  // (early returns below decide nothing)
  if (tid == 0) {
    a.stop_t[dom] = T;
    a.stop_kind[dom] = EV_NONE;
    a.stop_slot[dom] = -1;
    sh_bad = INT_MAX;
    sh_nexact = 0;
    sh_tie = 0;
  }
  for (int u = tid; u < Tl; u += RS_THREADS) a.ev_page[orow0 + u] = -1;
  if (Tl <= 0) return;
  if (nl == 0) {  // maintainer.cpp:93-94: empty partition layer -> the host seeds a cluster
    if (tid == 0) {
      a.stop_t[dom] = cur;
      a.stop_kind[dom] = EV_SEED;
    }
    return;
  }

  // ------------------------------------------------------------------ phase 0: inputs
  for (int c = tid; c < nl; c += RS_THREADS) {
    const int s = a.cand_slot[static_cast<int64_t>(dom) * cmax + c];
    const uint8_t b = a.cand_buf[static_cast<int64_t>(dom) * cmax + c];
    S.cslot[c] = s;
    S.cbuf[c] = b;
    S.ckey[c] = 2LL * t.cid[s] + b;
    const double nr = b ? t.bnorm[s] : t.rnorm[s];
    S.cnorm[c] = nr;
    S.sib[c] = -1;
    if (nr < 1e-12) atomicMin(&sh_bad, -1);  // degenerate representative (vecmath.hpp:59)
  }
  {
    const int rw = d * t.es / 4;  // words per key row (<= 256)
    const uint32_t* fkw = static_cast<const uint32_t*>(a.fk) + orow0 * rw;
    constexpr int RB = 4;  // rows per warp per batch, all loads in flight together
    for (int u0 = warp * RB; u0 < Tl; u0 += RS_WARPS * RB) {
      uint32_t v[RB][8];
#pragma unroll
      for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int w = lane + 32 * k;
          v[r][k] = (u0 + r < Tl && w < rw) ? __ldg(fkw + (u0 + r) * rw + w) : 0u;
        }
#pragma unroll
      for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int w = lane + 32 * k;
          if (u0 + r < Tl && w < rw) S.keys[(u0 + r) * S.ksw + w] = v[r][k];
        }
    }
  }
  __syncthreads();
  prof(11);
  // K0 places a lazy cluster's buffer candidate right after its live candidate
  for (int c = tid; c < nl; c += RS_THREADS)
    if (S.cbuf[c]) {
      S.sib[c] = static_cast<int16_t>(c - 1);
      S.sib[c - 1] = static_cast<int16_t>(c);
    }
  // K1b outputs of this launch's tokens (coalesced)
  for (int i = tid; i < Tl * TOPM; i += RS_THREADS) {
    S.tm_idx[i] = a.topm_idx[orow0 * TOPM + i];
    S.tm_ex[i] = a.topm_exact[orow0 * TOPM + i];
  }
  for (int u = tid; u < Tl; u += RS_THREADS) S.tm_next[u] = a.topm_next[orow0 + u];
  __syncthreads();
  prof(12);
  // key norms (vecmath.hpp:35-40) and the initial speculation: arg-best of K1b's exact
  // launch-time cosines (CandidateRef tie-break)
  for (int u = tid; u < Tl; u += RS_THREADS) {
    int ci[TOPM];
    double cv[TOPM];
#pragma unroll
    for (int k = 0; k < TOPM; ++k) {
      ci[k] = S.tm_idx[u * TOPM + k];
      cv[k] = S.tm_ex[u * TOPM + k];
    }
    double s = 0.0;
    for (int i = 0; i < d; ++i) {
      const double x = keyd(S, u, i, bf16);
      s = dadd(s, dmul(x, x));
    }
    const double nk = __dsqrt_rn(s);
    S.nk[u] = nk;
    if (nk < 1e-12) atomicMin(&sh_bad, u);
    double bs = -INFINITY;
    long long bk = LLONG_MAX;
    int bc = 0;
#pragma unroll
    for (int k = 0; k < TOPM; ++k) {
      const int c = ci[k];
      if (c >= 0 && better(cv[k], S.ckey[c], bs, bk)) {
        bs = cv[k];
        bk = S.ckey[c];
        bc = c;
      }
    }
    S.win[u] = static_cast<int16_t>(bc);
    S.kind[u] = EV_NONE;
  }
  __syncthreads();
  if (sh_bad != INT_MAX) {
    if (tid == 0) {
      set_err(t, DERR_DEGENERATE);
      a.stop_t[dom] = cur + (sh_bad < 0 ? 0 : sh_bad);
    }
    return;
  }
  if (tid == 0) {
    sh_ntot = nl;
    sh_nfresh = 0;
  }
  // Relaunch rounds (after a split: the fresh children absorb most of the remaining tokens and
  // move by ~1/n per absorb, so the launch-time speculation above fails at almost every token):
  // warp 0 simulates the routing sequentially in fp32 -- touched candidates' states updated by
  // Eq. 3 in fp32, their cosines re-evaluated per token, untouched ones from K1b's exact
  // launch-time values -- and speculates its winners instead. The simulation only proposes;
  // every decision is still verified exactly below, so a wrong proposal costs a round, never
  // exactness.
  if (a.exact_all && warp == 0 && d <= 256) simulate_routing(t, S, a, dom, Tl, nl, bf16, lane);
  __syncthreads();
  prof(0);

  int t0 = 0;
  int iters = 0;
  for (;;) {
    ++iters;
    __syncthreads();
    const int ntot = sh_ntot;
    // ---------------------------------------------------------------- A: touched-slot table
    for (int c = tid; c < ntot; c += RS_THREADS) S.cts[c] = -1;
    __syncthreads();
    for (int u = tid; u < Tl; u += RS_THREADS) {
      const int c = S.win[u];
      S.cts[S.cbuf[c] ? S.sib[c] : c] = -2;
    }
    __syncthreads();
    if (warp == 0) {
      int nts = 0;
      for (int base = 0; base < ntot; base += 32) {
        const int c = base + lane;
        const bool f = c < ntot && S.cts[c] == -2;
        const unsigned m = __ballot_sync(kFull, f);
        if (f) {
          const int idx = nts + __popc(m & ((1u << lane) - 1u));
          if (idx < tmax) {
            S.cts[c] = static_cast<int16_t>(idx);
            S.ts_lc[idx] = static_cast<int16_t>(c);
          } else {
            set_err(t, DERR_CANDIDATES);
            S.cts[c] = -1;
          }
        }
        nts += __popc(m);
      }
      if (lane == 0) sh_nts = min(nts, tmax);
    }
    __syncthreads();
    const int nts = sh_nts;
    for (int ts = tid; ts < nts; ts += RS_THREADS) {
      const int lc = S.ts_lc[ts];
      const int s = S.cslot[lc];
      const int cb = S.sib[lc];
      S.ts_slot[ts] = s;
      S.ts_cb[ts] = static_cast<int16_t>(cb);
      if (cb >= 0) S.cts[cb] = static_cast<int16_t>(ts);
      S.ts_var0[ts] = t.var[s];
      S.ts_rn0[ts] = t.rnorm[s];
      S.ts_bn0[ts] = t.bnorm[s];
      S.ts_stat0[ts] = t.stat[s];
      S.ts_nmem0[ts] = t.nmem[s];
      S.ts_cid[ts] = t.cid[s];
      S.ts_nbuf0[ts] = t.nbuf[s];
      S.ts_lazy0[ts] = t.lazy[s];
      S.ts_resid[ts] = t.resid[s];
      S.ts_cnt[ts] = 0;
      S.ts_fill[ts] = 0;
      S.ts_dsum[ts] = 0.0;
      S.ts_dbmax[ts] = 0ull;
      S.ts_fb[ts] = INT_MAX;
      const int np = t.npages[s], nbp = t.nbpages[s];
      const int last = np > t.seal[s] ? t.pages[static_cast<int64_t>(s) * t.maxp + np - 1] : -1;
      const int blast = nbp > 0 ? t.bpages[static_cast<int64_t>(s) * t.maxbp + nbp - 1] : -1;
      S.ts_np0[ts] = np;
      S.ts_nbp0[ts] = nbp;
      S.ts_last[ts] = last;
      S.ts_blast[ts] = blast;
      S.ts_fill0[ts] = last >= 0 ? t.pg_fill[last] : t.P;
      S.ts_bfill0[ts] = blast >= 0 ? t.pg_fill[blast] : t.P;
    }
    __syncthreads();
    // ---------------------------------------------------------------- B: chains (stable sort)
    for (int u = tid; u < Tl; u += RS_THREADS) {
      const int c = S.win[u];
      const int ts = S.cts[S.cbuf[c] ? S.sib[c] : c];
      S.tsof[u] = static_cast<int16_t>(ts);
      atomicAdd(&S.ts_cnt[ts], 1);
    }
    __syncthreads();
    if (warp == 0) {
      warp0_exscan(S.ts_cnt, nullptr, S.ts_off, nts, lane);
      __syncwarp();
      for (int base = 0; base < Tl; base += 32) {
        const int u = base + lane;
        const int key = u < Tl ? S.tsof[u] : -1 - lane;
        const unsigned peers = __match_any_sync(kFull, key);
        if (u < Tl) {
          const int p = S.ts_fill[key] + __popc(peers & ((1u << lane) - 1u));
          S.ctok[S.ts_off[key] + p] = static_cast<int16_t>(u);
          S.pos[u] = static_cast<int16_t>(p);
        }
        __syncwarp();
        if (u < Tl && lane == 31 - __clz(peers)) S.ts_fill[key] += __popc(peers);
        __syncwarp();
      }
    }
    if (tid == 0) {
      sh_te = Tl;
      sh_nreq = 0;
      sh_tfail = INT_MAX;
    }
    __syncthreads();
    // reciprocals of the Eq. 3/4 denominators and the Eq. 5 threshold window of each slot
    for (int u = t0 + tid; u < Tl; u += RS_THREADS) {
      const int ts = S.tsof[u];
      S.rcp[u] = ddiv(1.0, static_cast<double>(S.ts_stat0[ts] + S.pos[u] + 1));
    }
    for (int i = tid; i < Tl + nts; i += RS_THREADS) {  // tau(nmem0 + j), j < cnt, per slot
      int lo = 0, hi = nts - 1;  // the slot whose window [off + ts, off + ts + cnt] holds i
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (S.ts_off[mid] + mid <= i) lo = mid; else hi = mid - 1;
      }
      const int ts = lo;
      const long long j = i - (S.ts_off[ts] + ts);
      if (j < S.ts_cnt[ts]) {
        const long long n = S.ts_nmem0[ts] + j;
        S.tauw[i] = __ldg(&t.tau_tab[n < t.tau_len ? n : t.tau_len - 1]);
      }
    }
    // the chains below read other threads' reciprocals (S.rcp) and thresholds (S.tauw)
    // (compute-sanitizer racecheck: RAW hazard without this barrier)
    __syncthreads();
    prof(1);
    // ---------------------------------------------------------------- C: representative chains
    // one thread per (slot, element): r_i <- (n r_i + k_i) / (n + 1) over the slot's tokens
    for (int e = tid; e < nts * d; e += RS_THREADS) {
      const int ts = e / d, i = e - ts * d;
      const int off = S.ts_off[ts], cnt = S.ts_cnt[ts];
      int j = 0;
      while (j < cnt && S.ctok[off + j] < t0) ++j;
      if (j == cnt) continue;
      double r = j > 0 ? rsnap[sidx(i, S.ctok[off + j - 1], tmax)]
                       : t.rep64[static_cast<int64_t>(S.ts_slot[ts]) * d + i];
      double dn = static_cast<double>(S.ts_stat0[ts] + j);
      int u = S.ctok[off + j];
      int u1 = j + 1 < cnt ? S.ctok[off + j + 1] : u;
      double x = keyd(S, u, i, bf16), y = S.rcp[u];
      for (; j < cnt; ++j) {  // operands of the next step load while this one computes
        const int u2 = j + 2 < cnt ? S.ctok[off + j + 2] : u1;
        const double xn = keyd(S, u1, i, bf16), yn = S.rcp[u1];
        const double den = dadd(dn, 1.0);
        r = div_rcp(dadd(dmul(dn, r), x), den, y);  // Eq. 3 (maintainer.cpp:16-25)
        rsnap[sidx(i, u, tmax)] = r;
        dn = den;
        u = u1;
        u1 = u2;
        x = xn;
        y = yn;
      }
    }
    __syncthreads();
    prof(2);
    // ---------------------------------------------------------------- D: per-token exact sums
    for (int u = t0 + tid; u < Tl; u += RS_THREADS) {
      const int ts = S.tsof[u];
      const double2* rp = reinterpret_cast<const double2*>(rsnap) + static_cast<int64_t>(u) * 2;
      const int64_t qs = static_cast<int64_t>(tmax) * 2;  // double2 stride between quads
      double a_sq = 0.0, a_rn = 0.0;
      constexpr int QB = 4;  // quads per batch (16 elements), next batch in flight
      const int nq = d >> 2;
      double2 cb[2 * QB], nb[2 * QB];
#pragma unroll
      for (int k = 0; k < QB; ++k) {
        cb[2 * k] = k < nq ? rp[k * qs] : make_double2(0.0, 0.0);
        cb[2 * k + 1] = k < nq ? rp[k * qs + 1] : make_double2(0.0, 0.0);
      }
      for (int q0 = 0; q0 < nq; q0 += QB) {
#pragma unroll
        for (int k = 0; k < QB; ++k) {
          const int q = q0 + QB + k;
          nb[2 * k] = q < nq ? rp[q * qs] : make_double2(0.0, 0.0);
          nb[2 * k + 1] = q < nq ? rp[q * qs + 1] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int k = 0; k < QB; ++k) {
          if (q0 + k < nq) {
            const int i = (q0 + k) * 4;
            const double r4[4] = {cb[2 * k].x, cb[2 * k].y, cb[2 * k + 1].x, cb[2 * k + 1].y};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const double df = dsub(keyd(S, u, i + e, bf16), r4[e]);
              a_sq = dadd(a_sq, dmul(df, df));       // sq_dist(key, r') (vecmath.hpp:42-51)
              a_rn = dadd(a_rn, dmul(r4[e], r4[e]));  // norm(r')
            }
          }
        }
#pragma unroll
        for (int k = 0; k < 2 * QB; ++k) cb[k] = nb[k];
      }
      S.sq[u] = a_sq;
      S.a_rn[u] = __dsqrt_rn(a_rn);
      S.a_stat[u] = S.ts_stat0[ts] + S.pos[u] + 1;
    }
    __syncthreads();
    prof(3);
    // Movement bound of each slot: r'_j - r'_{j-1} = (k - r_{j-1}) / (n+1) and
    // k - r'_j = (k - r_{j-1}) n / (n+1), so |r'_j - r'_{j-1}| = sqrt(sq_j) / n; the sum over the
    // slot's chain bounds |r' - r0| for every state of the launch (warp-aggregated adds).
    for (int u0 = warp * 32; u0 < Tl; u0 += RS_THREADS) {
      const int u = u0 + lane;
      const bool ok = u < Tl;
      const int ts = ok ? S.tsof[u] : -1;
      const double v = ok ? sqrt(S.sq[u]) / static_cast<double>(S.ts_stat0[ts] + S.pos[u]) : 0.0;
      unsigned pend = __ballot_sync(kFull, ok);
      while (pend) {
        const int lead = __ffs(pend) - 1;
        const int tl = __shfl_sync(kFull, ts, lead);
        double m = (ok && ts == tl) ? v : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(kFull, m, o);
        if (lane == lead) atomicAdd(&S.ts_dsum[tl], m);
        pend &= ~__ballot_sync(kFull, ok && ts == tl);
      }
    }
    __syncthreads();
    prof(4);
    // ---------------------------------------------------------------- E1: variance chains
    // Eq. 4 var' = (n var + |k - r'|^2) / (n+1) runs for every routed token whatever the branch
    // (maintainer.cpp:114-117, 127-130), so it is a pure scalar chain per slot.
    for (int ts = tid; ts < nts; ts += RS_THREADS) {
      const int off = S.ts_off[ts], cnt = S.ts_cnt[ts];
      int j = 0;
      while (j < cnt && S.ctok[off + j] < t0) ++j;
      if (j == cnt) continue;
      double var = j > 0 ? S.a_var[S.ctok[off + j - 1]] : S.ts_var0[ts];
      double dn = static_cast<double>(S.ts_stat0[ts] + j);
      int u = S.ctok[off + j];
      int u1 = j + 1 < cnt ? S.ctok[off + j + 1] : u;
      double sq = S.sq[u], y = S.rcp[u];
      for (; j < cnt; ++j) {
        const int u2 = j + 2 < cnt ? S.ctok[off + j + 2] : u1;
        const double sqn = S.sq[u1], yn = S.rcp[u1];
        const double den = dadd(dn, 1.0);
        var = div_rcp(dadd(dmul(dn, var), sq), den, y);
        S.a_var[u] = var;
        dn = den;
        u = u1;
        u1 = u2;
        sq = sqn;
        y = yn;
      }
    }
    __syncthreads();
    prof(5);
    // ---------------------------------------------------------------- E2: decisions per slot
    // One warp per slot. A pass assumes every non-buffer token from `pos` absorbs, so the
    // member count before chain position j is known by a prefix count; the Eq. 5 tests of the
    // whole pass run in parallel and the first failure is the next non-absorb branch. A split /
    // eager split ends the slot; a deferred mark starts the next pass after it.
    for (int ts = warp; ts < nts; ts += RS_WARPS) {
      const int off = S.ts_off[ts], cnt = S.ts_cnt[ts];
      int pos = 0;
      while (pos < cnt && S.ctok[off + pos] < t0) ++pos;
      if (pos == cnt) continue;
      int nmi, nbuf;  // members added since launch (tau window index), buffered entries
      uint8_t lazy;
      if (pos > 0) {
        const int up = S.ctok[off + pos - 1];
        nmi = static_cast<int>(S.a_nmem[up] - S.ts_nmem0[ts]);
        nbuf = S.a_nbuf[up];
        lazy = S.a_lazy[up];
      } else {
        nmi = 0;
        nbuf = S.ts_nbuf0[ts];
        lazy = S.ts_lazy0[ts];
      }
      const long long nmem0 = S.ts_nmem0[ts];
      const uint8_t over = S.ts_resid[ts] ? (a.defer ? EV_DEFER : EV_EAGER) : EV_SPLIT;
      const double* tw = S.tauw + off + ts;
      const unsigned lt = (1u << lane) - 1u, le = (2u << lane) - 1u;
      while (pos < cnt) {
        int jfail = cnt, carry = 0;
        for (int base = pos; base < cnt; base += 32) {
          const int jj = base + lane;
          const bool in = jj < cnt;
          const int u = in ? S.ctok[off + jj] : 0;
          const bool isb = in && S.cbuf[S.win[u]] != 0;
          const unsigned nbm = __ballot_sync(kFull, in && !isb);
          bool ok = true;
          if (in && !isb) ok = S.a_var[u] <= tw[nmi + carry + __popc(nbm & lt)];  // Eq. 5
          const unsigned fm = __ballot_sync(kFull, !ok);
          if (fm) {
            jfail = base + __ffs(fm) - 1;
            break;
          }
          carry += __popc(nbm);
        }
        int cm = 0, cbf = 0;  // absorbs / buffer joins of [pos, jfail)
        for (int base = pos; base < jfail; base += 32) {
          const int jj = base + lane;
          const bool in = jj < jfail;
          const int u = in ? S.ctok[off + jj] : 0;
          const bool isb = in && S.cbuf[S.win[u]] != 0;
          const unsigned mm = __ballot_sync(kFull, in && !isb), bm = __ballot_sync(kFull, isb);
          if (in) {
            S.kind[u] = isb ? EV_BUFJOIN : EV_ABSORB;  // maintainer.cpp:112-137
            S.a_nmem[u] = nmem0 + nmi + cm + __popc(mm & le);
            S.a_nbuf[u] = nbuf + cbf + __popc(bm & le);
            S.a_lazy[u] = lazy;
          }
          cm += __popc(mm);
          cbf += __popc(bm);
        }
        nmi += cm;
        nbuf += cbf;
        if (jfail >= cnt) break;
        const int u = S.ctok[off + jfail];
        if (over != EV_DEFER) {  // maintainer.cpp:139-166: split / eager split, host slow path
          if (lane == 0) {
            S.kind[u] = over;
            atomicMin(&sh_te, u);
          }
          for (int jj = jfail + 1 + lane; jj < cnt; jj += 32) S.kind[S.ctok[off + jj]] = EV_NONE;
          break;
        }
        if (lane == 0) {  // maintainer.cpp:170-175: deferred mark, the entry parks in the buffer
          S.kind[u] = EV_DEFER;
          if (nbuf == 0 && S.ts_cb[ts] < 0) {
            const int q = atomicAdd(&sh_nreq, 1);
            if (q < FRESH_MAX) {
              S.req_u[q] = u;
              S.req_ts[q] = ts;
            }
          }
          S.a_nmem[u] = nmem0 + nmi;
          S.a_nbuf[u] = nbuf + 1;
          S.a_lazy[u] = 1;
        }
        nbuf += 1;
        lazy = 1;
        pos = jfail + 1;
      }
    }
    __syncthreads();
    prof(6);
    const int te = sh_te;
    // register the new buffer candidates (index.cpp register_buffer) in birth order
    if (tid == 0) {
      const int nq = min(sh_nreq, FRESH_MAX);
      if (sh_nreq > FRESH_MAX) set_err(t, DERR_CANDIDATES);
      for (int i = 1; i < nq; ++i)  // insertion sort by birth token
        for (int j = i; j > 0 && S.req_u[j - 1] > S.req_u[j]; --j) {
          const int tu = S.req_u[j], tt = S.req_ts[j];
          S.req_u[j] = S.req_u[j - 1];
          S.req_ts[j] = S.req_ts[j - 1];
          S.req_u[j - 1] = tu;
          S.req_ts[j - 1] = tt;
        }
      for (int i = 0; i < nq; ++i) {
        if (S.req_u[i] >= te) break;
        const int ts = S.req_ts[i];
        const int idx = sh_ntot;
        if (idx >= cmax || sh_nfresh >= FRESH_MAX) {
          set_err(t, DERR_CANDIDATES);
          break;
        }
        const int lc = S.ts_lc[ts];
        S.cslot[idx] = S.ts_slot[ts];
        S.cbuf[idx] = 1;
        S.ckey[idx] = 2LL * S.ts_cid[ts] + 1;
        S.cnorm[idx] = 0.0;
        S.sib[idx] = static_cast<int16_t>(lc);
        S.sib[lc] = static_cast<int16_t>(idx);
        S.cts[idx] = static_cast<int16_t>(ts);
        S.ts_cb[ts] = static_cast<int16_t>(idx);
        S.fr_birth[sh_nfresh] = static_cast<int16_t>(S.req_u[i]);
        S.fr_lc[sh_nfresh] = static_cast<int16_t>(lc);
        sh_nfresh += 1;
        sh_ntot = idx + 1;
      }
    }
    // reciprocals of the buffer-mean denominators; first buffer move of each slot
    for (int u = tid; u < te; u += RS_THREADS)
      if (buf_move(S.kind[u])) {
        if (u >= t0) S.rcpb[u] = ddiv(1.0, static_cast<double>(S.a_nbuf[u]));
        else atomicMax(&S.ts_dbmax[S.tsof[u]], ord_bits(S.db[u]));
        atomicMin(&S.ts_fb[S.tsof[u]], u);
      }
    __syncthreads();
    // ---------------------------------------------------------------- F: buffer-mean chains
    for (int e = tid; e < nts * d; e += RS_THREADS) {
      const int ts = e / d, i = e - ts * d;
      const int off = S.ts_off[ts], cnt = S.ts_cnt[ts];
      if (S.ts_fb[ts] >= te) continue;
      int j = 0;
      while (j < cnt && S.ctok[off + j] < t0) ++j;
      int ub = -1;
      for (int q = j - 1; q >= 0; --q)
        if (buf_move(S.kind[S.ctok[off + q]])) {
          ub = S.ctok[off + q];
          break;
        }
      double b = ub >= 0 ? bsnap[sidx(i, ub, tmax)] : t.brep64[static_cast<int64_t>(S.ts_slot[ts]) * d + i];
      for (; j < cnt; ++j) {
        const int u = S.ctok[off + j];
        if (u >= te) break;
        if (!buf_move(S.kind[u])) continue;
        const int nb = S.a_nbuf[u] - 1;
        const double x = keyd(S, u, i, bf16);
        const double dnb = static_cast<double>(nb);
        // buffer running mean (index.cpp:177-190)
        b = nb == 0 ? x : div_rcp(dadd(dmul(dnb, b), x), dadd(dnb, 1.0), S.rcpb[u]);
        bsnap[sidx(i, u, tmax)] = b;
      }
    }
    __syncthreads();
    for (int u = t0 + tid; u < te; u += RS_THREADS) {
      if (!buf_move(S.kind[u])) continue;
      const int ts = S.tsof[u];
      const int cb = S.ts_cb[ts];
      const bool launch_buf = cb >= 0 && cb < nl;
      const double* b0 = t.brep64 + static_cast<int64_t>(S.ts_slot[ts]) * d;
      double a_bn = 0.0, a_d = 0.0;
#pragma unroll 4
      for (int i = 0; i < d; ++i) {
        const double b = bsnap[sidx(i, u, tmax)];
        a_bn = dadd(a_bn, dmul(b, b));
        if (launch_buf) {
          const double ed = b - b0[i];
          a_d += ed * ed;
        }
      }
      S.a_bn[u] = __dsqrt_rn(a_bn);
      const double dbu = launch_buf ? 2.0 * sqrt(a_d) / S.ts_bn0[ts] * (1.0 + kSlack) + kSlack : INFINITY;
      S.db[u] = dbu;
      atomicMax(&S.ts_dbmax[ts], ord_bits(dbu));
    }
    __syncthreads();
    prof(7);
    // ---------------------------------------------------------------- H: verification
    {
      const int ntot2 = sh_ntot, nfresh = sh_nfresh;
      const int uend = min(te, Tl - 1);
      auto alive = [&](int c, int u) -> bool {
        if (c < nl) return true;
        const int k = c - nl;
        return k < nfresh && S.fr_birth[k] < u;
      };
      // first token that changes candidate c's state (INT_MAX: none this launch)
      auto first_change = [&](int c) -> int {
        const int ts = S.cts[c];
        if (ts < 0) return INT_MAX;
        return S.cbuf[c] ? S.ts_fb[ts] : S.ctok[S.ts_off[ts]];
      };
      // bound on the cosine movement of a candidate touched in this launch
      auto delta_max = [&](int c) -> double {
        const int ts = S.cts[c];
        if (S.cbuf[c]) return from_ord(S.ts_dbmax[ts]);
        return 2.0 * S.ts_dsum[ts] * (1.0 + 1e-9) / S.ts_rn0[ts] + 1e-11;
      };
      // last token before u that changed c's state (-1: launch state); binary search
      auto last_change = [&](int c, int u) -> int {
        const int ts = S.cts[c];
        if (ts < 0) return -1;
        const int off = S.ts_off[ts];
        int lo = 0, hi = S.ts_cnt[ts];  // first index with ctok >= u
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (S.ctok[off + mid] < u) lo = mid + 1; else hi = mid;
        }
        for (int j = lo - 1; j >= 0; --j) {
          const int v = S.ctok[off + j];
          if (!S.cbuf[c] || buf_move(S.kind[v])) return v;
        }
        return -1;
      };
      auto exact_at = [&](int c, int u, int st) -> double {
        const bool isb = S.cbuf[c];
        const double* p;
        int64_t stride;
        double nr;
        if (st >= 0) {  // snapshot of token st (tile layout)
          p = (isb ? bsnap : rsnap) + static_cast<int64_t>(st) * 4;
          stride = 0;
          nr = isb ? S.a_bn[st] : S.a_rn[st];
        } else {
          p = (isb ? t.brep64 : t.rep64) + static_cast<int64_t>(S.cslot[c]) * d;
          stride = 1;
          nr = S.cnorm[c];
        }
        if (nr < 1e-12) set_err(t, DERR_DEGENERATE);
        double acc = 0.0;
#pragma unroll 4
        for (int i = 0; i < d; ++i) {
          const double v = stride ? p[i] : p[static_cast<int64_t>(i >> 2) * tmax * 4 + (i & 3)];
          acc = dadd(acc, dmul(keyd(S, u, i, bf16), v));
        }
        return clamp1(ddiv(acc, dmul(S.nk[u], nr)));  // cosine_sim (vecmath.hpp:53-63)
      };
      // The same cosine from a warp-parallel fp64 sum (every lane calls it with the same c): the
      // lanes' partial sums and the tree differ from the sequential order only by rounding, so
      // |approx - exact| <= 2 gamma_d + O(u) < kApproxEps in cosine units -- tight enough that
      // only near-ties still need the sequential value. NaN: degenerate (the exact path raises it).
      auto approx_at = [&](int c, int u, int st) -> double {
        const bool isb = S.cbuf[c];
        double part = 0.0, nr;
        if (st >= 0) {
          const double* p = (isb ? bsnap : rsnap) + static_cast<int64_t>(st) * 4;
          nr = isb ? S.a_bn[st] : S.a_rn[st];
          for (int i = lane; i < d; i += 32) part += keyd(S, u, i, bf16) * p[static_cast<int64_t>(i >> 2) * tmax * 4 + (i & 3)];
        } else {
          const double* p = (isb ? t.brep64 : t.rep64) + static_cast<int64_t>(S.cslot[c]) * d;
          nr = S.cnorm[c];
          for (int i = lane; i < d; i += 32) part += keyd(S, u, i, bf16) * p[i];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
        return nr < 1e-12 ? NAN : part / (S.nk[u] * nr);
      };
      int n_ex = 0;
      // relaunch rounds (fresh children) use the warp-parallel cosine for any sizeable movement;
      // first rounds keep the movement bound (their clusters barely move, and the sequential
      // values of the few ambiguous candidates run on parallel lanes)
      const double move_approx = a.exact_all ? kMoveApprox : 3.0 * kMoveApprox;
      for (int u = t0 + warp; u <= uend; u += RS_WARPS) {
        const int64_t orow = orow0 + u;
        const int w = S.win[u];
        static_assert(TOPM == 8, "top-M row is one 16-byte vector");
        const int4 tv = *reinterpret_cast<const int4*>(S.tm_idx + u * TOPM);
        auto in_topm = [&](int c, double& ex) -> bool {
          const unsigned w[4] = {static_cast<unsigned>(tv.x), static_cast<unsigned>(tv.y),
                                 static_cast<unsigned>(tv.z), static_cast<unsigned>(tv.w)};
          int k = -1;
#pragma unroll
          for (int h = 0; h < 8; ++h) {
            const int v = static_cast<int16_t>((w[h >> 1] >> (16 * (h & 1))) & 0xffffu);
            if (v == c && k < 0) k = h;
          }
          if (k < 0) return false;
          ex = S.tm_ex[u * TOPM + k];
          return true;
        };
        const int my_ti = lane < TOPM ? S.tm_idx[u * TOPM + lane] : -1;
        const float* arow = a.approx + orow * cmax;
        const bool w_alive = alive(w, u);
        const bool w_touched = w_alive && first_change(w) < u;
        double exw = 0.0;
        // top-M entries far below the best carry NaN (exact not computed by the tile kernel)
        const bool inw = w < nl && in_topm(w, exw) && !isnan(exw);
        bool wknown = w_alive && !w_touched && inw;
        double lowW;
        if (!w_alive) {
          lowW = -INFINITY;
        } else if (w >= nl) {  // a buffer registered in this launch: no launch-time value
          double v = 0.0;
          if (lane == 0) {
            v = exact_at(w, u, last_change(w, u));
            ++n_ex;
          }
          exw = __shfl_sync(kFull, v, 0);
          wknown = true;
          lowW = exw;
        } else if (wknown) {
          lowW = exw;
        } else if (w_touched && delta_max(w) > move_approx &&
                   (a.exact_all || !(static_cast<double>(S.tm_next[u]) + margin <
                                     (inw ? exw : static_cast<double>(arow[w]) - margin) - delta_max(w)))) {
          // its state moved far (a fresh child after a split): the warp-parallel value less its
          // bound, instead of the movement bound (first rounds: only when the movement bound is
          // too loose to confine the candidates to the top-M list)
          const double ap = approx_at(w, u, last_change(w, u));
          lowW = isnan(ap) ? -INFINITY : ap - kApproxEps;
        } else {
          const double base = inw ? exw : static_cast<double>(arow[w]) - margin;
          lowW = base - (w_touched ? delta_max(w) : 0.0);
        }
        double bs = -INFINITY;
        long long bk = LLONG_MAX;
        int bp = -1;
        if (wknown && lane == 0) {
          bs = exw;
          bk = S.ckey[w];
          bp = w;
        }
        bool amb = false;
        bool ltie = false;  // this lane's best value was reached by two of its candidates
        // far-moved touched candidates the movement bound could not exclude, settled below by the
        // warp-parallel cosine (two per lane; a third goes to the sequential value at once)
        int pend0 = -1, pend1 = -1;
        // c != w, alive at u; touched: its state changed before u
        auto consider = [&](int c, bool touched, bool deferred) {
          double v = 0.0;
          bool have = false;
          if (c < nl && !deferred) {
            double ex;
            const bool in = in_topm(c, ex) && !isnan(ex);
            if (!touched && in) {  // untouched, exact launch-time value known
              if (ex < lowW) return;
              v = ex;
              have = true;
            } else {
              const double dm = touched ? delta_max(c) : 0.0;
              const double base = in ? ex : static_cast<double>(arow[c]) + margin;
              if (base + dm < lowW) return;
              if (dm > move_approx) {
                if (pend0 < 0) {
                  pend0 = c;
                  return;
                }
                if (pend1 < 0) {
                  pend1 = c;
                  return;
                }
              }
            }
          }
          amb = true;
          if (!have) {
            v = exact_at(c, u, touched ? last_change(c, u) : -1);
            ++n_ex;
          }
          if (v == bs) ltie = true;
          else if (v > bs) ltie = false;
          if (better(v, S.ckey[c], bs, bk)) {
            bs = v;
            bk = S.ckey[c];
            bp = c;
          }
        };
        const float tnext = S.tm_next[u];
        if (w_alive && static_cast<double>(tnext) + margin < lowW) {
          // untouched candidates outside the top-M list are bounded by tnext + margin
          if (lane < TOPM) {
            const int c = my_ti;
            if (c >= 0 && c != w && first_change(c) >= u) consider(c, false, false);
          }
          for (int ts = lane; ts < nts; ts += 32) {
            const int lc = S.ts_lc[ts];
            if (lc != w && S.ctok[S.ts_off[ts]] < u) consider(lc, true, false);
            const int cb = S.ts_cb[ts];
            if (cb >= 0 && cb != w && alive(cb, u) && S.ts_fb[ts] < u) consider(cb, true, false);
          }
        } else {
          for (int c = lane; c < ntot2; c += 32)
            if (c != w && alive(c, u)) consider(c, first_change(c) < u, false);
        }
        for (int r = 0; r < 2; ++r) {
          const int mine = r == 0 ? pend0 : pend1;
          unsigned m = __ballot_sync(kFull, mine >= 0);
          while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            const int c = __shfl_sync(kFull, mine, src);
            const double ap = approx_at(c, u, last_change(c, u));
            if (lane == src && (isnan(ap) || ap + kApproxEps >= lowW)) consider(c, true, true);
          }
        }
        const bool any = __any_sync(kFull, amb);
        if (any && !wknown && w_alive && lane == 0) {
          const double v = exact_at(w, u, w_touched ? last_change(w, u) : -1);
          ++n_ex;
          if (v == bs) ltie = true;
          else if (v > bs) ltie = false;
          if (better(v, S.ckey[w], bs, bk)) {
            bs = v;
            bk = S.ckey[w];
            bp = w;
          }
        }
        const double lbs = bs;
        warp_best(bs, bk, bp);
        if (any) {  // an exact tie of the best fp64 cosines decided by the key (IngestArgs::tie)
          const bool has = lbs == bs;
          if ((__popc(__ballot_sync(kFull, has)) >= 2 || __any_sync(kFull, has && ltie)) && lane == 0) sh_tie = 1;
        }
        const int vw = any ? bp : w;
        if (lane == 0) {
          S.vwin[u] = static_cast<int16_t>(vw);
          if (vw != w) atomicMin(&sh_tfail, u);
        }
      }
      for (int o = 16; o > 0; o >>= 1) n_ex += __shfl_xor_sync(kFull, n_ex, o);
      if (lane == 0 && n_ex) atomicAdd(&sh_nexact, n_ex);
    }
    __syncthreads();
    prof(8);
    const int tfail = sh_tfail;
    if (tfail > min(te, Tl - 1)) break;  // speculation verified up to the stop token
    // ---------------------------------------------------------------- restart at tfail
    t0 = tfail;
    for (int u = t0 + tid; u <= min(te, Tl - 1); u += RS_THREADS) S.win[u] = S.vwin[u];
    __syncthreads();
    if (tid == 0) {  // drop buffers registered at or after the restart token
      while (sh_nfresh > 0 && S.fr_birth[sh_nfresh - 1] >= t0) {
        sh_nfresh -= 1;
        S.sib[S.fr_lc[sh_nfresh]] = -1;
        sh_ntot -= 1;
      }
    }
    __syncthreads();
    for (int u = t0 + tid; u < Tl; u += RS_THREADS) {
      const int c = S.win[u];
      if (c >= sh_ntot) S.win[u] = S.fr_lc[c - nl];
    }
  }

  // ------------------------------------------------------------------ commit
  const int te = sh_te;
  const int stop = min(te, Tl);
  const int nts = sh_nts;
  for (int u = tid; u < stop; u += RS_THREADS) {
    const int s = S.cslot[S.win[u]];
    a.ev_kind[orow0 + u] = S.kind[u];
    a.ev_slot[orow0 + u] = s;
    if (a.ring_slot >= 0) t.ring_owner[(static_cast<int64_t>(dom) * t.W + a.ring_slot) * tmax + cur + u] = s;
  }
  // rank of each committed token among its slot's member / buffer rows (warp per slot)
  for (int ts = warp; ts < nts; ts += RS_WARPS) {
    const int off = S.ts_off[ts], cnt = S.ts_cnt[ts];
    int m = 0, b = 0;
    for (int base = 0; base < cnt; base += 32) {
      const int j = base + lane;
      const int u = j < cnt ? S.ctok[off + j] : INT_MAX;
      const bool ok = u < stop;
      const bool ism = ok && S.kind[u] == EV_ABSORB, isb = ok && !ism;
      const unsigned mm = __ballot_sync(kFull, ism), mb = __ballot_sync(kFull, isb);
      const unsigned lt = (1u << lane) - 1u;
      if (ism) S.vwin[u] = static_cast<int16_t>(m + __popc(mm & lt));  // member-row rank
      if (isb) S.vwin[u] = static_cast<int16_t>(b + __popc(mb & lt));  // buffer-row rank
      m += __popc(mm);
      b += __popc(mb);
    }
    if (lane == 0) {
      const int room = S.ts_last[ts] >= 0 ? t.P - S.ts_fill0[ts] : 0;
      const int broom = S.ts_blast[ts] >= 0 ? t.P - S.ts_bfill0[ts] : 0;
      int need_m = m > room ? (m - room + t.P - 1) / t.P : 0;
      int need_b = b > broom ? (b - broom + t.P - 1) / t.P : 0;
      if (S.ts_np0[ts] + need_m > t.maxp || S.ts_nbp0[ts] + need_b > t.maxbp) {
        set_err(t, DERR_CLUSTER_PAGES);
        need_m = need_b = 0;
      }
      S.ts_np[ts] = need_m;
      S.ts_nbp[ts] = need_b;
      S.ts_fb[ts] = m;    // (reused) committed member rows
      S.ts_fill[ts] = b;  // (reused) committed buffer rows
    }
  }
  __syncthreads();
  if (warp == 0) {
    const int total = warp0_exscan(S.ts_np, S.ts_nbp, S.ts_pbase, nts, lane);
    if (lane == 0) {
      const int want = min(total, S.pagecap);
      if (total > S.pagecap) set_err(t, DERR_PAGES);
      int k = 0;
      int pn = a.dom_pool_n[dom];
      while (k < want && pn > 0) S.pagebuf[k++] = a.dom_pool[dom * POOL + (--pn)];
      a.dom_pool_n[dom] = pn;
      const int rest = want - k;
      if (rest > 0) {
        const int top = atomicSub(t.free_top, rest);
        const int got = max(0, min(rest, top));
        if (got < rest) {
          atomicAdd(t.free_top, rest - got);
          set_err(t, DERR_PAGES);
        }
        for (int i = 0; i < got; ++i) S.pagebuf[k++] = t.free_stack[top - 1 - i];
      }
      sh_ptotal = k;
    }
  }
  __syncthreads();
  for (int ts = warp; ts < nts; ts += RS_WARPS) {
    const int off = S.ts_off[ts], cnt = S.ts_cnt[ts];
    if (cnt == 0 || S.ctok[off] >= stop) continue;
    const int s = S.ts_slot[ts];
    const int pbase = S.ts_pbase[ts];
    const int m = S.ts_fb[ts], b = S.ts_fill[ts];
    const int np0 = S.ts_np0[ts], nbp0 = S.ts_nbp0[ts];
    const int last = S.ts_last[ts], blast = S.ts_blast[ts];
    const int fill = S.ts_fill0[ts], bfill = S.ts_bfill0[ts];
    const int room = last >= 0 ? t.P - fill : 0, broom = blast >= 0 ? t.P - bfill : 0;
    const int nm = S.ts_np[ts], nbn = S.ts_nbp[ts];
    const int avail_m = min(nm, max(0, sh_ptotal - pbase));
    const int avail_b = min(nbn, max(0, sh_ptotal - pbase - nm));
    int ulast = -1, ublast = -1;
    for (int base = 0; base < cnt; base += 32) {
      const int j = base + lane;
      const int u = j < cnt ? S.ctok[off + j] : INT_MAX;
      const bool mine = u < stop;
      const bool tob = mine && S.kind[u] != EV_ABSORB;
      if (mine) {
        const int rank = S.vwin[u];
        const int rm = tob ? broom : room;
        const int navail = tob ? avail_b : avail_m;
        int page = -1, row = -1;
        if (rank < rm) {
          page = tob ? blast : last;
          row = (tob ? bfill : fill) + rank;
        } else {
          const int q = rank - rm, pi = q / t.P;
          if (pi < navail) {
            page = S.pagebuf[(tob ? pbase + nm : pbase) + pi];
            row = q - pi * t.P;
          }
        }
        a.ev_page[orow0 + u] = page;
        a.ev_row[orow0 + u] = row;
      }
      const unsigned mm = __ballot_sync(kFull, mine);
      if (mm) ulast = S.ctok[off + base + 31 - __clz(mm)];
      const unsigned mb = __ballot_sync(kFull, mine && buf_move(S.kind[u]));
      if (mb) ublast = S.ctok[off + base + 31 - __clz(mb)];
    }
    // page lists and fills
    int* list = t.pages + static_cast<int64_t>(s) * t.maxp;
    int* blist = t.bpages + static_cast<int64_t>(s) * t.maxbp;
    for (int k = lane; k < avail_m; k += 32) {
      const int pg = S.pagebuf[pbase + k];
      list[np0 + k] = pg;
      t.pg_fill[pg] = min(t.P, m - room - k * t.P);
    }
    for (int k = lane; k < avail_b; k += 32) {
      const int pg = S.pagebuf[pbase + nm + k];
      blist[nbp0 + k] = pg;
      t.pg_fill[pg] = min(t.P, b - broom - k * t.P);
    }
    if (lane == 0) {
      if (m > 0 && last >= 0) t.pg_fill[last] = min(t.P, fill + m);
      if (b > 0 && blast >= 0) t.pg_fill[blast] = min(t.P, bfill + b);
      t.npages[s] = np0 + avail_m;
      t.nbpages[s] = nbp0 + avail_b;
      t.rnorm[s] = S.a_rn[ulast];
      t.var[s] = S.a_var[ulast];
      t.stat[s] = S.a_stat[ulast];
      t.nmem[s] = S.a_nmem[ulast];
      t.nbuf[s] = S.a_nbuf[ulast];
      t.lazy[s] = S.a_lazy[ulast];
      if (ublast >= 0) t.bnorm[s] = S.a_bn[ublast];
    }
    for (int i = lane; i < d; i += 32) {
      const double r = rsnap[sidx(i, ulast, tmax)];
      t.rep64[static_cast<int64_t>(s) * d + i] = r;
      t.rep32[static_cast<int64_t>(s) * d + i] = static_cast<float>(r);
      if (ublast >= 0) {
        const double bv = bsnap[sidx(i, ublast, tmax)];
        t.brep64[static_cast<int64_t>(s) * d + i] = bv;
        t.brep32[static_cast<int64_t>(s) * d + i] = static_cast<float>(bv);
      }
    }
  }
  if (tid == 0 && te < Tl) {  // host event (split / eager split) at the stop token
    a.stop_t[dom] = cur + te;
    a.stop_kind[dom] = S.kind[te];
    a.stop_slot[dom] = S.cslot[S.win[te]];
  }
  prof(9);
  if (tid == 0) {
    a.n_exact[dom] = sh_nexact;
    if (a.tie) a.tie[dom] = sh_tie;
    for (int k = 0; k < 10; ++k) a.prof[dom * 16 + k] = sh_prof[k];
    a.prof[dom * 16 + 10] = iters;
  }
}

// Device check of div_rcp against __ddiv_rn on random operands (a in +-[2^-30, 2^4], integer
// b in [1, max_den]); counts mismatching bit patterns.
__global__ void k_div_check(uint64_t n, uint64_t seed, int max_den, unsigned long long* bad) {
  uint64_t x = seed ^ (0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1));
  unsigned long long nb = 0;
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    const double m = 1.0 + static_cast<double>(x >> 12) * 0x1p-52;  // [1, 2)
    const int e = static_cast<int>((x >> 3) % 35) - 30;
    double a = ldexp(m, e);
    if (x & 1) a = -a;
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    // max_den > 0: integer divisors (counts); otherwise real divisors in [2^-8, 2^8) (norms)
    const double b = max_den > 0 ? static_cast<double>(1 + (x % static_cast<uint64_t>(max_den)))
                                 : ldexp(1.0 + static_cast<double>(x >> 12) * 0x1p-52, static_cast<int>((x >> 4) % 16) - 8);
    if (max_den <= 0) a = static_cast<double>(static_cast<float>(a));  // unit rows: float numerators
    const double y = __ddiv_rn(1.0, b);
    const double q = div_rcp(a, b, y);
    if (__double_as_longlong(q) != __double_as_longlong(__ddiv_rn(a, b))) ++nb;
  }
  if (nb) atomicAdd(bad, nb);
}

}  // namespace

int launch_resolve_spec(const DevTables& t, const IngestArgs& a, cudaStream_t st) {
  if (t.d % 4 != 0 || t.d > 256 || t.tmax > 32767 || t.cmax > 32767) return 0;
  SpecSmem s;
  const size_t smem = spec_carve(nullptr, &s, t.d, t.es, a.T, t.tmax, t.cmax);
  if (smem > static_cast<size_t>(device_smem_optin() - 1024)) return 0;
  if (!smem_optin(reinterpret_cast<const void*>(k_resolve_spec), smem)) return 0;
  launch_pdl(k_resolve_spec, dim3(a.n_active), dim3(RS_THREADS), smem, st, t, a);
  return 1;
}

uint64_t debug_div_check(uint64_t n, uint64_t seed, int max_den) {
  unsigned long long* bad = nullptr;
  if (cudaMalloc(&bad, 8) != cudaSuccess) return ~0ull;
  cudaMemset(bad, 0, 8);
  k_div_check<<<1184, 256>>>(n, seed, max_den, bad);
  unsigned long long h = ~0ull;
  cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
  cudaFree(bad);
  return h;
}

}  // namespace kvc
