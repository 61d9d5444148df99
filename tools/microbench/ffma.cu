// Microbenchmark: FFMA vs FFMA2 (fma.rn.f32x2) issue/throughput on sm_100a, and a float4 copy.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_ffma(float *out, float a, float b) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; i++) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) acc[i] = fmaf(acc[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float *out, float a, float b) {
  unsigned long long acc[8];
#pragma unroll
  for (int i = 0; i < 8; i++) {
    float2 v = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    acc[i] = *reinterpret_cast<unsigned long long *>(&v);
  }
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long A = *reinterpret_cast<unsigned long long *>(&av);
  unsigned long long B = *reinterpret_cast<unsigned long long *>(&bv);
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(A), "l"(B));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) { float2 v = *reinterpret_cast<float2 *>(&acc[i]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_copy(const float4 *__restrict__ in, float4 *__restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) out[i] = in[i];
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d l2=%d MB smemPerSM=%zu\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerMultiprocessor);
  int sms = p.multiProcessorCount;
  float *out; cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; rep++)
  for (int bs : {256, 512, 1024}) {
    int grid = sms * (2048 / bs);
    k_ffma<<<grid, bs>>>(out, 0.999f, 1e-3f);
    cudaEventRecord(e0); k_ffma<<<grid, bs>>>(out, 0.999f, 1e-3f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * ITERS * (double)grid * bs;
    k_ffma2<<<grid, bs>>>(out, 0.999f, 1e-3f);
    cudaEventRecord(e0); k_ffma2<<<grid, bs>>>(out, 0.999f, 1e-3f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms2; cudaEventElapsedTime(&ms2, e0, e1);
    printf("bs=%d FFMA %.1f TFLOP/s   FFMA2 %.1f TFLOP/s\n", bs, fl / ms / 1e9, fl / ms2 / 1e9);
  }
  size_t n = (size_t)1 << 28;  // 1 GiB of floats per buffer
  float4 *a, *b; cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4); cudaMemset(a, 0, n * 4);
  for (int g : {sms * 4, sms * 8, sms * 16}) {
    k_copy<<<g, 512>>>(a, b, n / 4);
    cudaEventRecord(e0); for (int r = 0; r < 5; r++) k_copy<<<g, 512>>>(a, b, n / 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy grid=%d %.1f GB/s\n", g, 5.0 * 2 * n * 4 / ms / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
