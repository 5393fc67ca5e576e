// Microbenchmark: latency / throughput (cycles) of fp64 ops and shared loads on one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x, int n) {
  __shared__ double sm[1024];
  __shared__ float smf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + i * 1e-9; smf[i] = 1.0f + i * 1e-6f; }
  __syncthreads();
  double a = x, b = x * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
  // 8 independent chains: throughput
  double c0 = x, c1 = x, c2 = x, c3 = x, c4 = x, c5 = x, c6 = x, c7 = x;
  for (int i = 0; i < n; ++i) {
    c0 = __dadd_rn(c0, b); c1 = __dadd_rn(c1, b); c2 = __dadd_rn(c2, b); c3 = __dadd_rn(c3, b);
    c4 = __dadd_rn(c4, b); c5 = __dadd_rn(c5, b); c6 = __dadd_rn(c6, b); c7 = __dadd_rn(c7, b);
  }
  long long t2 = clock64();
  double acc = 0.0;
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) acc = __dadd_rn(acc, __dmul_rn(sm[i], sm[(i + 3) & 1023]));
  long long t3 = clock64();
  double acc2 = 0.0;
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) acc2 = __dadd_rn(acc2, __dmul_rn((double)smf[i], sm[i]));
  long long t4 = clock64();
  // register-only dot (no loads): dmul of registers
  double acc3 = 0.0, r0 = x, r1 = b;
  for (int i = 0; i < n; ++i) acc3 = __dadd_rn(acc3, __dmul_rn(r0, r1));
  long long t5 = clock64();
  float f = (float)x;
  for (int i = 0; i < n; ++i) f = __shfl_xor_sync(0xffffffff, f, 1) + 1.0f;
  long long t6 = clock64();
  // the Eq. 3/4 element chain of one cluster (maintainer.cpp:16-25): r' = (n r + k) / (n + 1),
  // each insert depending on the previous r (correctly rounded division, as the device chains)
  double r = x, nn = 3.0;
  for (int i = 0; i < n; ++i) { r = __ddiv_rn(__dadd_rn(__dmul_rn(nn, r), b), __dadd_rn(nn, 1.0)); nn = __dadd_rn(nn, 1.0); }
  long long t7 = clock64();
  double dv = x;
  for (int i = 0; i < n; ++i) dv = __ddiv_rn(dv, 1.0000001);
  long long t8 = clock64();
  out[threadIdx.x] = a + acc + acc2 + acc3 + f + c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7 + r + dv;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; cyc[6] = t7 - t6; cyc[7] = t8 - t7; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
  const int n = 1024;
  k<<<1, 32>>>(o, c, 1.5, n); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1.5, n); cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
  printf("{\"dadd_chain_cycles\": %.2f, \"dadd_indep_cycles\": %.3f, \"lds_dot_cycles_per_elem\": %.2f, "
         "\"f32lds_dot_cycles_per_elem\": %.2f, \"reg_dot_cycles_per_elem\": %.2f, \"shfl_cycles\": %.2f, "
         "\"eq34_element_chain_cycles\": %.2f, \"ddiv_chain_cycles\": %.2f}\n",
         h[0] / (double)n, h[1] / (8.0 * n), h[2] / 1024.0, h[3] / 1024.0, h[4] / (double)n, h[5] / (double)n,
         h[6] / (double)n, h[7] / (double)n);
  return 0;
}
