// FP64 peak microbenchmark for B200 (sm_100a): DFMA (CUDA cores) and DMMA
// (mma.sync f64 tensor path, m8n8k4 and m16n8k16 shapes).  Used to fix the
// roofline denominator for the factorization kernels.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double r[8];
#pragma unroll
  for (int i = 0; i < 8; i++) r[i] = threadIdx.x * 1e-7 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += r[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma884_kernel(double* out, int iters) {
  double acc[8][2];
  double a = 1e-3 * (threadIdx.x & 7), b = 2e-3 * (threadIdx.x >> 3);
#pragma unroll
  for (int i = 0; i < 8; i++) { acc[i][0] = 0; acc[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma16816_kernel(double* out, int iters) {
  double acc[4][4];
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = 1e-3 * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < 4; i++) b[i] = 2e-3 * (threadIdx.x - i);
#pragma unroll
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) acc[i][j] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) s += acc[i][j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct Cfg { const char* name; int kind; int threads; int bps; };
  Cfg cfgs[] = {{"dfma", 0, 256, 4}, {"dfma", 0, 512, 2}, {"dfma", 0, 1024, 2},
                {"dmma_m8n8k4", 1, 128, 4}, {"dmma_m8n8k4", 1, 256, 4}, {"dmma_m8n8k4", 1, 512, 2},
                {"dmma_m16n8k16", 2, 128, 4}, {"dmma_m16n8k16", 2, 256, 4}, {"dmma_m16n8k16", 2, 512, 2}};
  for (auto& c : cfgs) {
    int iters = 20000;
    double best = 0;
    for (int rep = 0; rep < 6; rep++) {
      cudaEventRecord(e0);
      if (c.kind == 0) dfma_kernel<<<sms * c.bps, c.threads>>>(out, iters, 0.999999, 1e-9);
      else if (c.kind == 1) dmma884_kernel<<<sms * c.bps, c.threads>>>(out, iters);
      else dmma16816_kernel<<<sms * c.bps, c.threads>>>(out, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops;
      long long thr = (long long)sms * c.bps * c.threads;
      if (c.kind == 0) flops = 2.0 * 8 * iters * thr;
      else if (c.kind == 1) flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * (thr / 32);
      else flops = 2.0 * 16 * 8 * 16 * 4 * (double)iters * (thr / 32);
      double tf = flops / (ms * 1e-3) / 1e12;
      if (rep > 0 && tf > best) best = tf;
    }
    printf("{\"kernel\": \"%s\", \"threads\": %d, \"blocks_per_sm\": %d, \"tflops\": %.3f}\n", c.name, c.threads, c.bps, best);
  }
  CK(cudaGetLastError());
  return 0;
}
