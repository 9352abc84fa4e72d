// Dependent-chain latency of DMMA.8x8x4 and DFMA on sm_100a (one warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_chain(double* out, int iters, long long* cyc) {
  double d0 = threadIdx.x, d1 = 1.0, a = 1e-3, b = 2e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (d0 == 1234.5) out[0] = d0 + d1;
}
__global__ void dfma_chain(double* out, int iters, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) x = fma(x, 0.999999, 1e-9);
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (x == 1234.5) out[0] = x;
}
int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 64); cudaMalloc(&cyc, 8);
  for (int rep = 0; rep < 2; rep++) {
    dmma_chain<<<1, 32>>>(out, 4096, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DMMA.8x8x4 dependent latency: %.1f cycles\n", h / 4096.0);
    dfma_chain<<<1, 32>>>(out, 4096, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.1f cycles\n", h / 4096.0);
  }
  return 0;
}
