// assign_tc.cu -- K1' (tensor cores): the frame's token x candidate distance tile on tcgen05.
//
// Replaces K1 (fp32 SIMT tile) + K1b (per-token top-M) for bf16 frames. Per domain one CTA:
//   * TMA (cp.async.bulk.tensor, 128-byte swizzle) loads the frame's keys [T<=256][d] bf16 as
//     two M=128 tiles;
//   * the candidates' representatives are gathered from the fp32 mirrors and split into a bf16
//     hi/lo pair (r ~= hi + lo to 2^-17 relative), written in the same swizzled K-major layout;
//   * one elected thread issues tcgen05.mma (kind::f16, M=128, N=256, K=16, fp32 accumulate)
//     hi and lo passes into TMEM (2 tiles x 256 columns);
//   * eight epilogue warps tcgen05.ld their token rows, scale by 1/(|k||r|) to the approximate
//     cosine, store the tile row (read by the resolve kernels' rare slow paths), keep the top-8
//     and the 9th value in registers, then compute the top-8's EXACT fp64 cosines against the
//     launch-time representatives in the reference's summation order (vecmath.hpp:53-63).
// Error of the approximate cosine: split residual 2^-17 + fp32 accumulation over 2 x d products;
// the resolve kernels certify with margin kTcMargin (checked on the device by
// tests/test_kernels_gpu.py against the exact cosines).
#include <cuda.h>

#include <cfloat>

#include "devmath.cuh"

namespace kvc {
namespace {

using namespace dm;

constexpr int AS_THREADS = 256;  // 8 warps: warps 0-3 token tile 0, warps 4-7 token tile 1
constexpr int NCH = 256;         // candidates per MMA (N)
constexpr int KB = 64;           // bf16 elements per 128-byte swizzle row
constexpr uint32_t TMEM_COLS = 512;

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
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128-byte swizzle UMMA shared-memory descriptor (8-row atoms of 128 B, SBO 1024 B).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr & 0x3FFFF) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}
// kind::f16 instruction descriptor: bf16 x bf16 -> fp32, K-major A and B, M = 128, N = NCH.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(NCH >> 3) << 17) |
                            (static_cast<uint32_t>(128 >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accum)
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = __uint_as_float(r[j]);
}

__host__ __device__ inline size_t tc_smem_bytes(int d) {
  const size_t kh = static_cast<size_t>(d / KB);
  return 1024 /*align slack*/ + 2 * kh * 128 * 128 /*A*/ + 2 * kh * NCH * 128 /*B hi, lo*/ +
         NCH * 4 /*inv norms*/ + NCH * 8 /*candidate rows*/ + 64 /*barriers*/;
}

// Element i of token row r of a swizzled [128 rows][128 B] key tile (kh = i / 64 selects the tile).
__device__ __forceinline__ uint32_t a_word(const uint8_t* tile0, int KH, int r, int i) {
  const int kh = i / KB, byte = (i % KB) * 2;
  const uint8_t* p = tile0 + kh * 128 * 128 + r * 128 + ((((byte >> 4) ^ (r & 7)) << 4) | (byte & 15));
  return *reinterpret_cast<const uint32_t*>(p);  // elements i, i+1 (i even)
}

__global__ void __launch_bounds__(AS_THREADS, 1) k_assign_tc(DevTables t, IngestArgs a,
                                                             const __grid_constant__ CUtensorMap tmk) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (launched as a dependent of K0)
  extern __shared__ uint8_t smraw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  const int d = t.d, KH = d / KB;
  uint8_t* sA = base;                               // [2][KH][128 rows][128 B]
  uint8_t* sBh = sA + 2 * KH * 128 * 128;           // [KH][NCH rows][128 B]
  uint8_t* sBl = sBh + KH * NCH * 128;
  float* inr = reinterpret_cast<float*>(sBl + KH * NCH * 128);
  const float** crow = reinterpret_cast<const float**>(inr + NCH);  // candidate fp32 rows of the chunk
  uint64_t* bars = reinterpret_cast<uint64_t*>(crow + NCH);  // [0] keys loaded, [1] mma done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int dom = a.active[blockIdx.x];
  const int T = a.T, n = a.cand_n[dom], cmax = t.cmax;
  const int mtiles = T > 128 ? 2 : 1;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tid == 0) {  // keys: TMA, one box of 64 x 128 per (token tile, K half)
    mbar_expect(&bars[0], static_cast<uint32_t>(mtiles * KH * 128 * 128));
    for (int mt = 0; mt < mtiles; ++mt)
      for (int kh = 0; kh < KH; ++kh) tma_load_3d(sA + (mt * KH + kh) * 128 * 128, &tmk, kh * KB, mt * 128, dom, &bars[0]);
  }

  // this thread's token (row of the TMA-loaded key tile)
  const int mt = warp >> 2;
  const int mr = (warp & 3) * 32 + lane;
  const int m = mt * 128 + mr;
  const bool tok_ok = m < T && mt < mtiles;
  const uint8_t* atile = sA + mt * KH * 128 * 128;
  float ink = 0.f;
  float tv[TOPM + 1];
  int ti[TOPM + 1];
#pragma unroll
  for (int k = 0; k <= TOPM; ++k) {
    tv[k] = -INFINITY;
    ti[k] = -1;
  }
  const int32_t* cs = a.cand_slot + static_cast<int64_t>(dom) * cmax;
  const uint8_t* cbuf = a.cand_buf + static_cast<int64_t>(dom) * cmax;
  float* arow = a.approx + (static_cast<int64_t>(dom) * t.tmax + m) * cmax;

  uint32_t phase = 0;
  for (int c0 = 0; c0 < n; c0 += NCH) {
    const int nc = min(NCH, n - c0);
    // B: representatives as bf16 hi / lo, swizzled K-major rows (zero rows past nc). Row
    // pointers first, then each warp streams whole rows (coalesced), RB rows in flight.
    for (int r = tid; r < NCH; r += AS_THREADS) {
      float nr = 0.f;
      const float* src = nullptr;
      if (r < nc) {
        const int s = cs[c0 + r];
        const bool ib = cbuf[c0 + r];
        src = (ib ? t.brep32 : t.rep32) + static_cast<int64_t>(s) * d;
        nr = static_cast<float>(ib ? t.bnorm[s] : t.rnorm[s]);
      }
      crow[r] = src;
      inr[r] = nr > 0.f ? 1.f / nr : 0.f;
    }
    __syncthreads();
    {
      constexpr int RB = 8;
      const int q4 = d / 4;  // float4 per row (<= 32: one per lane)
      for (int r0 = warp * RB; r0 < NCH; r0 += 8 * RB) {
        float4 v[RB];
#pragma unroll
        for (int k = 0; k < RB; ++k) {
          const float* src = crow[r0 + k];
          v[k] = (src && lane < q4) ? __ldg(reinterpret_cast<const float4*>(src) + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < RB; ++k) {
          if (lane < q4) {
            const int r = r0 + k;
            const __nv_bfloat162 h01 = __floats2bfloat162_rn(v[k].x, v[k].y), h23 = __floats2bfloat162_rn(v[k].z, v[k].w);
            const float2 f01 = __bfloat1622float2(h01), f23 = __bfloat1622float2(h23);
            const __nv_bfloat162 l01 = __floats2bfloat162_rn(v[k].x - f01.x, v[k].y - f01.y);
            const __nv_bfloat162 l23 = __floats2bfloat162_rn(v[k].z - f23.x, v[k].w - f23.y);
            const int e = 4 * lane, kh = e / KB, byte = (e % KB) * 2;
            const int off = kh * NCH * 128 + r * 128 + ((((byte >> 4) ^ (r & 7)) << 4) | (byte & 15));
            uint2 hv, lv;
            hv.x = *reinterpret_cast<const uint32_t*>(&h01);
            hv.y = *reinterpret_cast<const uint32_t*>(&h23);
            lv.x = *reinterpret_cast<const uint32_t*>(&l01);
            lv.y = *reinterpret_cast<const uint32_t*>(&l23);
            *reinterpret_cast<uint2*>(sBh + off) = hv;
            *reinterpret_cast<uint2*>(sBl + off) = lv;
          }
        }
      }
    }
    if (c0 == 0) {  // 1/|k| (fp32) from the TMA-loaded key tile
      mbar_wait(&bars[0], 0);
      if (tok_ok) {
        float s2 = 0.f;
        for (int i = 0; i < d; i += 2) {
          const uint32_t w = a_word(atile, KH, mr, i);
          const float lo = __uint_as_float(w << 16), hi = __uint_as_float(w & 0xffff0000u);
          s2 = fmaf(lo, lo, s2);
          s2 = fmaf(hi, hi, s2);
        }
        ink = s2 > 0.f ? rsqrtf(s2) : 0.f;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      for (int t2 = 0; t2 < mtiles; ++t2) {
        const uint32_t dcol = tmem + static_cast<uint32_t>(t2 * NCH);
        for (int kh = 0; kh < KH; ++kh)
#pragma unroll
          for (int ks = 0; ks < KB / 16; ++ks) {
            const uint64_t ad = sw128_desc(smem_u32(sA + (t2 * KH + kh) * 128 * 128) + ks * 32);
            const uint64_t bh = sw128_desc(smem_u32(sBh + kh * NCH * 128) + ks * 32);
            const uint64_t bl = sw128_desc(smem_u32(sBl + kh * NCH * 128) + ks * 32);
            mma_bf16(dcol, ad, bh, (kh | ks) != 0);
            mma_bf16(dcol, ad, bl, 1u);
          }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bars[1]))
                   : "memory");
    }
    mbar_wait(&bars[1], phase);
    phase ^= 1;
    tc_fence_after();
    if (mt < mtiles) {
      const uint32_t tbase = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + static_cast<uint32_t>(mt * NCH);
#pragma unroll 1
      for (int cb = 0; cb < nc; cb += 8) {  // 8 columns per tcgen05.ld keeps the loop body small
        float v[8];
        tmem_ld8(tbase + static_cast<uint32_t>(cb), v);  // warp-collective
        if (tok_ok) {
          const float sc = ink;
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] *= sc * inr[cb + j];
          if (cb + 8 <= nc) {
            *reinterpret_cast<float4*>(arow + c0 + cb) = make_float4(v[0], v[1], v[2], v[3]);
            *reinterpret_cast<float4*>(arow + c0 + cb + 4) = make_float4(v[4], v[5], v[6], v[7]);
          } else {
            for (int j = 0; j < nc - cb; ++j) arow[c0 + cb + j] = v[j];
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float x = v[j];
            if (cb + j < nc && x > tv[TOPM]) {  // insertion keeps (value desc, index asc)
              tv[TOPM] = x;
              ti[TOPM] = c0 + cb + j;
#pragma unroll
              for (int k = TOPM; k > 0; --k) {
                const bool sw = tv[k] > tv[k - 1];
                const float fa = tv[k], fb = tv[k - 1];
                const int ia = ti[k], ib = ti[k - 1];
                tv[k] = sw ? fb : fa;
                tv[k - 1] = sw ? fa : fb;
                ti[k] = sw ? ib : ia;
                ti[k - 1] = sw ? ia : ib;
              }
            }
          }
        }
      }
    }
    tc_fence_before();
    __syncthreads();
  }

  // Exact fp64 cosines (vecmath.hpp:53-63) of the top-M entries that can decide the token's
  // arg-best: those within 2 margins of the best approximate score (the others are NaN = "not
  // computed"; the resolve kernels bound them by approx + margin instead). Keys come from the
  // key tile in shared memory; the fp64 representatives of the union of every token's needed
  // candidates (a frame's tokens share few clusters) are staged once into shared memory (the B
  // tiles are free after the last MMA), so the sequential dot chains read at shared-memory
  // latency instead of one L2 round trip per step. Same operands, same order: same bits.
  const float cut = tv[0] - 2.f * a.margin;
  __shared__ int s_nx;
  int* mark = reinterpret_cast<int*>(sBh);  // [n] candidate -> staged row (or -1)
  const int xs = d + 1;                     // odd row stride (doubles): rows spread over the banks
  const int mark_bytes = (cmax * 4 + 15) & ~15;
  double* xrows = reinterpret_cast<double*>(sBh + mark_bytes);
  const int xcap = (2 * KH * NCH * 128 - mark_bytes) / (xs * 8);
  for (int c = tid; c < n; c += AS_THREADS) mark[c] = 0;
  __syncthreads();
  if (tok_ok)
#pragma unroll
    for (int k = 0; k < TOPM; ++k)
      if (ti[k] >= 0 && (a.exact_all || tv[k] >= cut)) mark[ti[k]] = 1;
  __syncthreads();
  if (warp == 0) {  // compact: staged row index in candidate order
    int nb = 0;
    for (int c0 = 0; c0 < n; c0 += 32) {
      const int c = c0 + lane;
      const bool mk = c < n && mark[c] != 0;
      const unsigned bal = __ballot_sync(0xffffffffu, mk);
      if (c < n) mark[c] = mk ? nb + __popc(bal & ((1u << lane) - 1u)) : -1;
      nb += __popc(bal);
    }
    if (lane == 0) s_nx = nb;
  }
  __syncthreads();
  for (int c = warp; c < n; c += AS_THREADS / 32) {  // one warp per staged row, lanes over dims
    const int x = mark[c];
    if (x < 0 || x >= xcap) continue;
    const int s = cs[c];
    const double* src = (cbuf[c] ? t.brep64 : t.rep64) + static_cast<int64_t>(s) * d;
    for (int i = lane; i < d; i += 32) xrows[x * xs + i] = src[i];
  }
  __syncthreads();
  if (tok_ok) {
    const int64_t o = static_cast<int64_t>(dom) * t.tmax + m;
    const double* rp[TOPM];
    double nr[TOPM];
#pragma unroll
    for (int k = 0; k < TOPM; ++k) {
      const int c = ti[k];
      rp[k] = nullptr;
      nr[k] = 1.0;
      if (c >= 0 && (a.exact_all || tv[k] >= cut)) {
        const int s = cs[c];
        const bool ib = cbuf[c];
        const int x = mark[c];
        rp[k] = x < xcap ? xrows + x * xs : (ib ? t.brep64 : t.rep64) + static_cast<int64_t>(s) * d;
        nr[k] = ib ? t.bnorm[s] : t.rnorm[s];
      }
    }
    double acc[TOPM];
#pragma unroll
    for (int k = 0; k < TOPM; ++k) acc[k] = 0.0;
    double sk = 0.0;
    for (int i = 0; i < d; i += 2) {
      const uint32_t w = a_word(atile, KH, mr, i);
      const double x0 = static_cast<double>(__uint_as_float(w << 16));
      const double x1 = static_cast<double>(__uint_as_float(w & 0xffff0000u));
      sk = dadd(sk, dmul(x0, x0));
      sk = dadd(sk, dmul(x1, x1));
#pragma unroll
      for (int k = 0; k < TOPM; ++k)
        if (rp[k]) {
          const double r0 = rp[k][i], r1 = rp[k][i + 1];  // shared (staged) or global (overflow)
          acc[k] = dadd(acc[k], dmul(x0, r0));
          acc[k] = dadd(acc[k], dmul(x1, r1));
        }
    }
    const double nk = __dsqrt_rn(sk);
#pragma unroll
    for (int k = 0; k < TOPM; ++k) {
      a.topm_idx[o * TOPM + k] = static_cast<int16_t>(ti[k]);
      a.topm_val[o * TOPM + k] = ti[k] >= 0 ? tv[k] : -INFINITY;
      a.topm_exact[o * TOPM + k] = ti[k] < 0 ? -3.0 : (rp[k] ? clamp1(ddiv(acc[k], dmul(nk, nr[k]))) : NAN);
    }
    a.topm_next[o] = ti[TOPM] >= 0 ? tv[TOPM] : -INFINITY;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// Self-check of the last distance tile: max |approx - exact| over every (token, candidate) of the
// active domains, candidates outside a token's top-M list scoring above its (M+1)-th value, and
// top-M exact values differing from a fresh exact cosine. out: [ord(max err), violations, mismatches].
__global__ void k_assign_err(DevTables t, IngestArgs a, unsigned long long* out) {
  const int dom = a.active[blockIdx.x];
  const int n = a.cand_n[dom], T = a.T, d = t.d, cmax = t.cmax;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int u = warp; u < T; u += nw) {
    const int64_t o = static_cast<int64_t>(dom) * t.tmax + u;
    double sk = 0.0;
    for (int i = 0; i < d; ++i) {
      const double x = ld_kv(a.fk, o * d + i, t.kv_bf16);
      sk = dadd(sk, dmul(x, x));
    }
    const double nk = __dsqrt_rn(sk);
    const float tnext = a.topm_next[o];
    for (int c = lane; c < n; c += 32) {
      const int s = a.cand_slot[static_cast<int64_t>(dom) * cmax + c];
      const bool ib = a.cand_buf[static_cast<int64_t>(dom) * cmax + c];
      const double* rp = (ib ? t.brep64 : t.rep64) + static_cast<int64_t>(s) * d;
      double acc = 0.0;
      for (int i = 0; i < d; ++i) acc = dadd(acc, dmul(static_cast<double>(ld_kv(a.fk, o * d + i, t.kv_bf16)), rp[i]));
      const double ex = clamp1(ddiv(acc, dmul(nk, ib ? t.bnorm[s] : t.rnorm[s])));
      const double ap = a.approx[o * cmax + c];
      const double err = fabs(ap - ex);
      const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(err));
      atomicMax(&out[0], b);  // non-negative doubles order like their bit patterns
      int k = -1;
      for (int j = 0; j < TOPM; ++j)
        if (a.topm_idx[o * TOPM + j] == c) k = j;
      if (k < 0 && ap > tnext) atomicAdd(&out[1], 1ull);
      const double tx = k >= 0 ? a.topm_exact[o * TOPM + k] : 0.0;  // NaN: not computed (far below the best)
      if (k >= 0 && !isnan(tx) && tx != ex) atomicAdd(&out[2], 1ull);
      if (k >= 0 && isnan(tx) && ap >= a.topm_val[o * TOPM] - 2.0 * a.margin) atomicAdd(&out[2], 1ull);
    }
  }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace

bool assign_tc_supported(const DevTables& t) {
  return t.kv_bf16 && (t.d == 64 || t.d == 128) && t.tmax <= 256;
}

bool make_key_tensor_map(void* map, const void* keys, int d, int tmax, int L) {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return false;
    fn = reinterpret_cast<EncodeTiled>(p);
  }
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(tmax), static_cast<cuuint64_t>(L)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(d) * 2, static_cast<cuuint64_t>(d) * 2 * tmax};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(KB), 128u, 1u};
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  const CUresult r = fn(static_cast<CUtensorMap*>(map), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(keys),
                        dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int launch_assign_err(const DevTables& t, const IngestArgs& a, unsigned long long* out, cudaStream_t st) {
  k_assign_err<<<a.n_active, 256, 0, st>>>(t, a, out);
  return 1;
}

int launch_assign_tc(const DevTables& t, const IngestArgs& a, const void* key_map, cudaStream_t st) {
  const size_t smem = tc_smem_bytes(t.d);
  if (!smem_optin(reinterpret_cast<const void*>(k_assign_tc), smem)) return 0;
  launch_pdl(k_assign_tc, dim3(a.n_active), dim3(AS_THREADS), smem, st, t, a, *static_cast<const CUtensorMap*>(key_map));
  return 1;
}

}  // namespace kvc
