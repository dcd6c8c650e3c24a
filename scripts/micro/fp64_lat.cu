// Microbenchmark: latency of dependent fp64 ops on this GPU (one warp).
#include <cstdio>
#include <cstdint>
__global__ void k_dfma(double* out, long long* cyc, double a, double b, int n) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __fma_rn(x, a, b); x = __fma_rn(x, a, b); x = __fma_rn(x, a, b); x = __fma_rn(x, a, b); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_dadd(double* out, long long* cyc, double a, double b, int n) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __dadd_rn(x, a); x = __dadd_rn(x, b); x = __dadd_rn(x, a); x = __dadd_rn(x, b); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_ffma(float* out, long long* cyc, float a, float b, int n) {
  float x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __fmaf_rn(x, a, b); x = __fmaf_rn(x, a, b); x = __fmaf_rn(x, a, b); x = __fmaf_rn(x, a, b); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_dsel(double* out, long long* cyc, double a, double b, int n) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x < a ? b : x; x = x + 1e-300; x = x < b ? a : x; x = x + 1e-300; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
// throughput: many independent chains, many warps
__global__ void k_dfma_tp(double* out, double a, double b, int n) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < n; ++i) {
    x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b); x3 = __fma_rn(x3, a, b);
    x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b); x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  double* d; float* f; long long* c; long long h;
  cudaMalloc(&d, 1 << 26); cudaMalloc(&f, 1 << 20); cudaMalloc(&c, 8);
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    k_dfma<<<1, 32>>>(d, c, 0.999, 1e-3, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent: %.2f cyc/op\n", (double)h / (4.0 * n));
    k_dadd<<<1, 32>>>(d, c, 0.5, -0.5, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent: %.2f cyc/op\n", (double)h / (4.0 * n));
    k_ffma<<<1, 32>>>(f, c, 0.999f, 1e-3f, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("FFMA dependent: %.2f cyc/op\n", (double)h / (4.0 * n));
    k_dsel<<<1, 32>>>(d, c, 0.5, 0.25, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DSETP+FSEL+DADD dependent pair: %.2f cyc/(cmp+sel+add)\n", (double)h / (2.0 * n));
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 4; w <= 32; w *= 2) {
    k_dfma_tp<<<148 * 4, 32 * w / 4>>>(d, 0.999, 1e-3, 1000);
    cudaEventRecord(e0);
    k_dfma_tp<<<148 * 4, 32 * w / 4>>>(d, 0.999, 1e-3, 1000);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 1000 * 148 * 4 * 32 * w / 4;
    printf("DFMA throughput, %d warps/SM: %.1f TFLOP/s\n", w, flops / ms / 1e9);
  }
  return 0;
}
