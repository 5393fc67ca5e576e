// tiers.cu -- physical host tier of the cluster-contiguous store (K5).
//
// The reference's TieredStore (store.cpp:95-130) moves a cluster between Device and Host as ONE
// batched transfer of its entries. Here a Host-resident cluster's member pages live in a
// contiguous extent of pinned, mapped host pages (the cluster's pages back to back), so a fetch
// or an offload is one cudaMemcpyAsync per cluster on the transfer stream between that extent and
// a contiguous staging run in HBM. The kernels below move pages between the (scattered) HBM page
// pool and the staging run and rewrite the page tables; the bulk bytes of queued migrations cross
// the host link on the copy engines. The one exception is fetch-on-read (k_fetch_read): the pages
// of host-resident clusters a decode step selected are copied by SM loads between K4 and K6,
// because K6 needs them within the step anyway (the reference fetches every verified cluster,
// retrieval.cpp:76-89); K6 then reads the fresh (L2-resident) HBM copies.
#include "devmath.cuh"

namespace kvc {

namespace {

using namespace dm;

// 16-byte vectorised copy of one page by one CTA (page_bytes is a multiple of 16).
__device__ __forceinline__ void copy_page(uint8_t* dst, const uint8_t* src, int64_t bytes) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
  const int64_t n = bytes / 16;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) d[i] = s[i];
}

// Member pages to move, 0 when every one is already in the host tier (nothing to offload).
__global__ void k_tier_count(DevTables t, const int32_t* slots, int n, int32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int np = t.npages[slots[i]];
  const int* list = t.pages + static_cast<int64_t>(slots[i]) * t.maxp;
  int dev = 0;
  for (int p = 0; p < np; ++p) dev += is_host_page(t, list[p]) ? 0 : 1;
  out[i] = dev > 0 ? np : 0;
}

// Fetch-on-read copies (DecodeArgs::fr_jobs, listed by K4): one CTA per page, 8 x 16 B loads per
// thread in flight (a 32 KB page in one round trip over the host link); then the page table
// entry and the fill move to the HBM page. K6 (a programmatic dependent) waits for this grid.
__global__ void __launch_bounds__(256) k_fetch_read(DevTables t, DecodeArgs a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  int any = 0;
  for (int l = threadIdx.x; l < t.L; l += blockDim.x) any |= a.fr_nj[l];
  if (!__syncthreads_or(any)) return;  // a hot step: nothing to copy
  const int64_t n16 = t.page_bytes / 16;
  int base = 0, g = blockIdx.x;
  for (int l = 0; l < t.L; ++l) {
    const int nj = a.fr_nj[l];
    for (; g < base + nj; g += gridDim.x) {
      const int4 j = a.fr_jobs[static_cast<int64_t>(l) * a.max_desc + (g - base)];
      const uint4* src = reinterpret_cast<const uint4*>(page_k(t, j.x));
      uint4* dst = reinterpret_cast<uint4*>(page_k(t, j.y));
      for (int64_t i0 = 0; i0 < n16; i0 += 8 * 256) {
        uint4 r[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t i = i0 + u * 256 + threadIdx.x;
          if (i < n16) r[u] = src[i];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t i = i0 + u * 256 + threadIdx.x;
          if (i < n16) dst[i] = r[u];
        }
      }
      if (threadIdx.x == 0) {
        t.pg_fill[j.y] = t.pg_fill[j.x];
        t.pages[static_cast<int64_t>(j.z) * t.maxp + j.w] = j.y;
      }
    }
    base += nj;
  }
}

// grid (x: pages, y: clusters): member page p of cluster y -> staging page stage0 + p. Pages already
// in the host tier (a re-offload of a cluster with a device tail) are read through the mapping.
__global__ void k_tier_gather(DevTables t, const TierMove* mv, uint8_t* stage) {
  const TierMove m = mv[blockIdx.y];
  if (m.slot < 0) return;  // dropped from the batch
  for (int p = blockIdx.x; p < m.n_pages; p += gridDim.x) {
    const int pg = t.pages[static_cast<int64_t>(m.slot) * t.maxp + p];
    copy_page(stage + (m.stage0 + p) * t.page_bytes, page_k(t, pg), t.page_bytes);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) t.seal[m.slot] = max(t.seal[m.slot], m.n_pages);
}

// One thread per cluster: pages [0, n) become host pages host0 + i (fills carried over); the HBM
// ones go back to the free stack. No kernel pops pages concurrently (stream order).
__global__ void k_tier_commit_offload(DevTables t, const TierMove* mv, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const TierMove m = mv[i];
  if (m.slot < 0) return;
  int* list = t.pages + static_cast<int64_t>(m.slot) * t.maxp;
  int nd = 0;
  for (int p = 0; p < m.n_pages; ++p) nd += is_host_page(t, list[p]) ? 0 : 1;
  const int base = atomicAdd(t.free_top, nd);
  int k = 0;
  for (int p = 0; p < m.n_pages; ++p) {
    const int old = list[p];
    const int hp = static_cast<int>(t.max_pages + m.host0 + p);
    t.pg_fill[hp] = t.pg_fill[old];
    if (!is_host_page(t, old)) t.free_stack[base + k++] = old;
    list[p] = hp;
  }
}

// grid (x: pages, y: clusters). Each host page of cluster y (an id inside its extent) gets a fresh
// HBM page popped by the block that copies it from staging; the new ids go to newp[y][p] and are
// installed by k_tier_fetch_tables.
__global__ void k_tier_commit_fetch(DevTables t, const TierMove* mv, const uint8_t* stage, int32_t* newp) {
  const TierMove m = mv[blockIdx.y];
  if (m.slot < 0) return;
  int* list = t.pages + static_cast<int64_t>(m.slot) * t.maxp;
  const int np = t.npages[m.slot];
  int32_t* out = newp + static_cast<int64_t>(blockIdx.y) * t.maxp;
  __shared__ int s_new[1];
  for (int p = blockIdx.x; p < np; p += gridDim.x) {
    const int old = list[p];
    if (!is_host_page(t, old)) continue;
    const int64_t rel = static_cast<int64_t>(old) - t.max_pages - m.host0;
    if (rel < 0 || rel >= m.n_pages) {  // not in this extent: table and host disagree
      if (threadIdx.x == 0) set_err(t, DERR_TIER);
      continue;
    }
    if (threadIdx.x == 0) {
      const int top = atomicSub(t.free_top, 1) - 1;
      if (top < 0) {
        atomicAdd(t.free_top, 1);
        set_err(t, DERR_PAGES);
        s_new[0] = -1;
      } else {
        s_new[0] = t.free_stack[top];
      }
    }
    __syncthreads();
    const int pg = s_new[0];
    if (pg >= 0) copy_page(page_k(t, pg), stage + (m.stage0 + rel) * t.page_bytes, t.page_bytes);
    if (threadIdx.x == 0) out[p] = pg;
    __syncthreads();
  }
}

// Second pass of the fetch commit: the new ids replace the host ids (a separate launch so no block
// of the copy pass can observe a half-rewritten list).
__global__ void k_tier_fetch_tables(DevTables t, const TierMove* mv, int n, const int32_t* newp) {
  const int y = blockIdx.x;
  if (y >= n) return;
  const TierMove m = mv[y];
  if (m.slot < 0) return;
  int* list = t.pages + static_cast<int64_t>(m.slot) * t.maxp;
  const int np = t.npages[m.slot];
  const int32_t* in = newp + static_cast<int64_t>(y) * t.maxp;
  for (int p = threadIdx.x; p < np; p += blockDim.x) {
    const int old = list[p];
    if (!is_host_page(t, old)) continue;
    const int64_t rel = static_cast<int64_t>(old) - t.max_pages - m.host0;
    if (rel < 0 || rel >= m.n_pages) continue;
    const int pg = in[p];
    if (pg < 0) continue;  // pool exhausted (error raised): the page stays readable in the host tier
    t.pg_fill[pg] = t.pg_fill[old];
    list[p] = pg;
  }
}

}  // namespace

int launch_tier_count(const DevTables& t, const int32_t* slots, int32_t n, int32_t* out, cudaStream_t st) {
  if (n <= 0) return 0;
  k_tier_count<<<(n + 255) / 256, 256, 0, st>>>(t, slots, n, out);
  return 1;
}

int launch_fetch_read(const DevTables& t, const DecodeArgs& a, cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * device_sms()));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_fetch_read, t, a);
  return 1;
}

int launch_tier_gather(const DevTables& t, const TierMove* mv, int32_t n, int32_t max_pages_per_cluster,
                       uint8_t* stage, cudaStream_t st) {
  if (n <= 0) return 0;
  const dim3 grid(static_cast<unsigned>(max(1, min(max_pages_per_cluster, 64))), static_cast<unsigned>(n));
  k_tier_gather<<<grid, 256, 0, st>>>(t, mv, stage);
  return 1;
}

int launch_tier_commit_offload(const DevTables& t, const TierMove* mv, int32_t n, cudaStream_t st) {
  if (n <= 0) return 0;
  k_tier_commit_offload<<<(n + 127) / 128, 128, 0, st>>>(t, mv, n);
  return 1;
}

int launch_tier_commit_fetch(const DevTables& t, const TierMove* mv, int32_t n, int32_t max_pages_per_cluster,
                             const uint8_t* stage, int32_t* scratch, cudaStream_t st) {
  if (n <= 0) return 0;
  const dim3 grid(static_cast<unsigned>(max(1, min(max_pages_per_cluster, 64))), static_cast<unsigned>(n));
  k_tier_commit_fetch<<<grid, 256, 0, st>>>(t, mv, stage, scratch);
  k_tier_fetch_tables<<<n, 128, 0, st>>>(t, mv, n, scratch);
  return 2;
}

}  // namespace kvc
