// HBM throughput by read:write stream mix on this GPU (roofline context for
// the write-heavy step kernel: ~0.37 R : 0.63 W at mid-day).  Each thread
// moves 16-byte vectors: R read streams summed into W write streams,
// grid-stride, 512 MB per stream (>> L2).  nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o rw_mix rw_mix.cu && ./rw_mix
#include <cstdio>
#include <cuda_runtime.h>

template <int R, int W>
__global__ void k(const float4* __restrict__ in, float4* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 s = make_float4(1.f, 2.f, 3.f, 4.f);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float4 v = __ldcs(in + r * n + i);
      s.x += v.x, s.y += v.y, s.z += v.z, s.w += v.w;
    }
#pragma unroll
    for (int w = 0; w < W; ++w) __stcs(out + w * n + i, s);
  }
}

template <int R, int W>
void run(const float4* in, float4* out, size_t n, int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = sms * 8;
  k<R, W><<<grid, 256>>>(in, out, n);
  cudaEventRecord(a);
  const int reps = 10;
  for (int i = 0; i < reps; ++i) k<R, W><<<grid, 256>>>(in, out, n);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)(R + W) * n * 16 * reps;
  printf("R:W = %d:%d  %8.1f GB/s  (write share %.2f)\n", R, W, bytes / ms / 1e6, (double)W / (R + W));
}

int main() {
  const size_t n = (512ull << 20) / 16;  // float4s per stream
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float4 *in, *out;
  cudaMalloc(&in, 5 * n * 16);
  cudaMalloc(&out, 5 * n * 16);
  cudaMemset(in, 0, 5 * n * 16);
  run<1, 0>(in, out, n, sms);
  run<0, 1>(in, out, n, sms);
  run<1, 1>(in, out, n, sms);
  run<2, 3>(in, out, n, sms);
  run<3, 5>(in, out, n, sms);
  run<1, 2>(in, out, n, sms);
  run<1, 3>(in, out, n, sms);
  return 0;
}
