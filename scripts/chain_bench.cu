// Microbenchmark: cycles per step of the resolve chains (one thread, others parked at a barrier).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double div_rcp(double a, double b, double y) {
  const double q1 = __dmul_rn(a, y);
  const double r1 = __fma_rn(-q1, b, a);
  const double q2 = __fma_rn(r1, y, q1);
  const double r2 = __fma_rn(-q2, b, a);
  return __fma_rn(r2, y, q2);
}
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ double sq[256], rc[256], tw[256];
  __shared__ short ctok[256], win[256];
  __shared__ unsigned char cb[256], kind[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    sq[i] = 1e-3 * (i % 7); rc[i] = 1.0 / (1000 + i); tw[i] = 0.5; ctok[i] = i; win[i] = i % 3; cb[i] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double var = 0.01, dn = 1000.0;
    long long t0 = clock64();
    for (int j = 0; j < n; ++j) {  // pure chain
      const double den = __dadd_rn(dn, 1.0);
      var = div_rcp(__dadd_rn(__dmul_rn(dn, var), sq[j & 255]), den, rc[j & 255]);
      dn = den;
    }
    long long t1 = clock64();
    double var2 = 0.01; dn = 1000.0;
    for (int j = 0; j < n; ++j) {  // ddiv chain
      const double den = __dadd_rn(dn, 1.0);
      var2 = __ddiv_rn(__dadd_rn(__dmul_rn(dn, var2), sq[j & 255]), den);
      dn = den;
    }
    long long t2 = clock64();
    // decision-loop shape: indirect loads, compare, stores
    double var3 = 0.01; dn = 1000.0; long long nmem = 0; int u = ctok[0];
    double s = sq[u], y = rc[u]; bool ib = cb[win[u]]; double tcur = tw[0];
    for (int j = 0; j < n; ++j) {
      const int un = j + 1 < n ? ctok[(j + 1) & 255] : u;
      const double sn = sq[un], yn = rc[un]; const bool ibn = cb[win[un]];
      const long long tix = nmem + 1; const double tnx = tw[tix & 255];
      const double den = __dadd_rn(dn, 1.0);
      const double vn = div_rcp(__dadd_rn(__dmul_rn(dn, var3), s), den, y);
      unsigned char kk = ib ? 2 : (vn <= tcur ? 1 : 3);
      kind[u] = kk;
      var3 = vn;
      if (kk == 1) { nmem += 1; tcur = tnx; }
      dn = den; u = un; s = sn; y = yn; ib = ibn;
    }
    long long t3 = clock64();
    double a = 1.0;
    for (int j = 0; j < n; ++j) a = __dadd_rn(a, 1e-9);
    long long t4 = clock64();
    double f = 1.0;
    for (int j = 0; j < n; ++j) f = __fma_rn(f, 1.0000001, 1e-9);
    long long t5 = clock64();
    out[0] = var + var2 + var3 + a + f + nmem;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
  }
  __syncthreads();
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64); cudaMalloc(&c, 64);
  const int n = 4096;
  for (int threads : {32, 512}) {
    k<<<1, threads>>>(o, c, n); cudaDeviceSynchronize();
    k<<<1, threads>>>(o, c, n); cudaDeviceSynchronize();
    long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
    printf("threads %d: chain(div_rcp) %.1f | chain(ddiv) %.1f | decision loop %.1f | dadd %.1f | dfma %.1f cycles/step\n",
           threads, h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n);
  }
  return 0;
}
