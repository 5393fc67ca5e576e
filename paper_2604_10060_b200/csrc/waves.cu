// waves.cu -- device side of the parallel settle of ingest host events (context_waves.cpp).
//
// The reference settles a frame's splits one after another (maintainer.cpp:88-176 per insert in
// layer-major order; the split seed is mix_seed(seed, split_counter_++), maintainer.cpp:222). A
// split only changes its own domain's clusters, so the wave engine settles the pending events of
// every domain at once with predicted counters, verifies each prediction afterwards, and rolls a
// domain back to the snapshot taken at its first event when a prediction changed its k-means.
// These kernels are the batched pieces of that engine: staging of many clusters, slot snapshots
// and their restore, batched page release, partition-list and cluster-id scatters.
#include "kvc_core.hpp"

namespace kvc {

namespace {

// One block per job: the slot's member rows (page order), then its buffer rows, then (frame_row
// >= 0) one frame key/value row, into staging rows [row0, ...).
__global__ void __launch_bounds__(256) k_gather_batch(DevTables t, const GatherJob* jobs, const uint8_t* fk,
                                                      const uint8_t* fv, uint8_t* sk, uint8_t* sv) {
  const GatherJob j = jobs[blockIdx.x];
  const int rb = t.d * t.es;
  int64_t row = j.row0;
  if (j.slot >= 0) {
    const int np = t.npages[j.slot];
    const int nbp = j.with_buf ? t.nbpages[j.slot] : 0;
    for (int b = 0; b < np + nbp; ++b) {
      const bool isb = b >= np;
      const int page = isb ? t.bpages[static_cast<int64_t>(j.slot) * t.maxbp + (b - np)]
                           : t.pages[static_cast<int64_t>(j.slot) * t.maxp + b];
      const int fill = t.pg_fill[page];
      const uint8_t* pk = page_k(t, page);
      const uint8_t* pv = page_v(t, page);
      for (int o = threadIdx.x * 16; o < fill * rb; o += blockDim.x * 16) {
        *reinterpret_cast<uint4*>(sk + row * rb + o) = *reinterpret_cast<const uint4*>(pk + o);
        *reinterpret_cast<uint4*>(sv + row * rb + o) = *reinterpret_cast<const uint4*>(pv + o);
      }
      row += fill;
    }
  }
  if (threadIdx.x == 0 && j.count_out) *j.count_out = static_cast<int32_t>(row - j.row0) + (j.frame_row >= 0 ? 1 : 0);
  if (j.frame_row >= 0)
    for (int o = threadIdx.x * 16; o < rb; o += blockDim.x * 16) {
      *reinterpret_cast<uint4*>(sk + row * rb + o) = *reinterpret_cast<const uint4*>(fk + j.frame_row * rb + o);
      *reinterpret_cast<uint4*>(sv + row * rb + o) = *reinterpret_cast<const uint4*>(fv + j.frame_row * rb + o);
    }
}

// k_free_slot for a list of slots (one block each): HBM pages back to the free stack.
__global__ void k_free_slots(DevTables t, const int32_t* slots, int n) {
  const int slot = slots[blockIdx.x];
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

__device__ __forceinline__ uint8_t* snap_rec(uint8_t* arena, int64_t e, int d) {
  return arena + e * static_cast<int64_t>(slot_snap_bytes(d));
}

// Snapshot of the ingest-mutable state of slots[e] into record e (one block per slot).
__global__ void k_snap_slots(DevTables t, const int32_t* slots, int n, uint8_t* arena) {
  const int e = blockIdx.x;
  const int64_t s = slots[e];
  uint8_t* r = snap_rec(arena, e, t.d);
  SlotSnap& h = *reinterpret_cast<SlotSnap*>(r);
  double* rep = reinterpret_cast<double*>(r + sizeof(SlotSnap));
  double* brep = rep + t.d;
  float* rep32 = reinterpret_cast<float*>(brep + t.d);
  float* brep32 = rep32 + t.d;
  for (int c = threadIdx.x; c < t.d; c += blockDim.x) {
    rep[c] = t.rep64[s * t.d + c];
    brep[c] = t.brep64[s * t.d + c];
    rep32[c] = t.rep32[s * t.d + c];
    brep32[c] = t.brep32[s * t.d + c];
  }
  if (threadIdx.x == 0) {
    h.slot = static_cast<int32_t>(s);
    h.npages = t.npages[s];
    h.nbpages = t.nbpages[s];
    h.nbuf = t.nbuf[s];
    h.stat = t.stat[s];
    h.nmem = t.nmem[s];
    h.cid = t.cid[s];
    h.lazy = t.lazy[s];
    h.resid = t.resid[s];
    h.fill_m = h.npages > 0 ? t.pg_fill[t.pages[s * t.maxp + h.npages - 1]] : 0;
    h.fill_b = h.nbpages > 0 ? t.pg_fill[t.bpages[s * t.maxbp + h.nbpages - 1]] : 0;
    h.var = t.var[s];
    h.rnorm = t.rnorm[s];
    h.bnorm = t.bnorm[s];
  }
}

// Restores records idx[i] (one block each): the pages appended since the snapshot go back to
// the free stack, the tail pages get their fill back, every statistic its snapshot value.
__global__ void k_restore_slots(DevTables t, const int32_t* idx, int n, const uint8_t* arena) {
  const uint8_t* r = arena + static_cast<int64_t>(idx[blockIdx.x]) * slot_snap_bytes(t.d);
  const SlotSnap& h = *reinterpret_cast<const SlotSnap*>(r);
  const double* rep = reinterpret_cast<const double*>(r + sizeof(SlotSnap));
  const double* brep = rep + t.d;
  const float* rep32 = reinterpret_cast<const float*>(brep + t.d);
  const float* brep32 = rep32 + t.d;
  const int64_t s = h.slot;
  for (int c = threadIdx.x; c < t.d; c += blockDim.x) {
    t.rep64[s * t.d + c] = rep[c];
    t.brep64[s * t.d + c] = brep[c];
    t.rep32[s * t.d + c] = rep32[c];
    t.brep32[s * t.d + c] = brep32[c];
  }
  if (threadIdx.x == 0) {
    const int np = t.npages[s], nbp = t.nbpages[s];
    const int extra = max(0, np - h.npages) + max(0, nbp - h.nbpages);
    if (extra > 0) {
      int base = atomicAdd(t.free_top, extra);
      for (int i = h.npages; i < np; ++i) t.free_stack[base++] = t.pages[s * t.maxp + i];
      for (int i = h.nbpages; i < nbp; ++i) t.free_stack[base++] = t.bpages[s * t.maxbp + i];
    }
    t.npages[s] = h.npages;
    t.nbpages[s] = h.nbpages;
    if (h.npages > 0) t.pg_fill[t.pages[s * t.maxp + h.npages - 1]] = h.fill_m;
    if (h.nbpages > 0) t.pg_fill[t.bpages[s * t.maxbp + h.nbpages - 1]] = h.fill_b;
    t.nbuf[s] = h.nbuf;
    t.stat[s] = h.stat;
    t.nmem[s] = h.nmem;
    t.cid[s] = h.cid;
    t.lazy[s] = h.lazy;
    t.resid[s] = h.resid;
    t.var[s] = h.var;
    t.rnorm[s] = h.rnorm;
    t.bnorm[s] = h.bnorm;
  }
}

// Partition-list scatter: record i = {key (pid * L + layer), off, n} followed by n slots.
__global__ void k_pl_scatter(DevTables t, const int32_t* recs, const int32_t* rec_off, int n) {
  const int32_t* r = recs + rec_off[blockIdx.x];
  const int key = r[0], off = r[1], cnt = r[2];
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) t.pl_pool[off + i] = r[3 + i];
  if (threadIdx.x == 0) {
    t.pl_off[key] = off;
    t.pl_cnt[key] = cnt;
  }
}

__global__ void k_read_vars(DevTables t, const int32_t* slots, int n, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = t.var[slots[i]];
}

__global__ void k_set_cids(DevTables t, const SlotCid* x, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) t.cid[x[i].slot] = x[i].cid;
}

}  // namespace

int launch_gather_batch(const DevTables& t, const GatherJob* jobs, int32_t n, const void* fk, const void* fv,
                        void* sk, void* sv, cudaStream_t st) {
  if (n <= 0) return 0;
  k_gather_batch<<<n, 256, 0, st>>>(t, jobs, static_cast<const uint8_t*>(fk), static_cast<const uint8_t*>(fv),
                                    static_cast<uint8_t*>(sk), static_cast<uint8_t*>(sv));
  return 1;
}

int launch_free_slots(const DevTables& t, const int32_t* slots, int32_t n, cudaStream_t st) {
  if (n <= 0) return 0;
  k_free_slots<<<n, 128, 0, st>>>(t, slots, n);
  return 1;
}

int launch_snap_slots(const DevTables& t, const int32_t* slots, int32_t n, void* arena, cudaStream_t st) {
  if (n <= 0) return 0;
  k_snap_slots<<<n, 128, 0, st>>>(t, slots, n, static_cast<uint8_t*>(arena));
  return 1;
}

int launch_restore_slots(const DevTables& t, const int32_t* idx, int32_t n, const void* arena, cudaStream_t st) {
  if (n <= 0) return 0;
  k_restore_slots<<<n, 128, 0, st>>>(t, idx, n, static_cast<const uint8_t*>(arena));
  return 1;
}

int launch_pl_scatter(const DevTables& t, const int32_t* recs, const int32_t* rec_off, int32_t n, cudaStream_t st) {
  if (n <= 0) return 0;
  k_pl_scatter<<<n, 128, 0, st>>>(t, recs, rec_off, n);
  return 1;
}

int launch_read_vars(const DevTables& t, const int32_t* slots, int32_t n, double* out, cudaStream_t st) {
  if (n <= 0) return 0;
  k_read_vars<<<(n + 127) / 128, 128, 0, st>>>(t, slots, n, out);
  return 1;
}

int launch_set_cids(const DevTables& t, const SlotCid* x, int32_t n, cudaStream_t st) {
  if (n <= 0) return 0;
  k_set_cids<<<(n + 255) / 256, 256, 0, st>>>(t, x, n);
  return 1;
}

}  // namespace kvc
