// Microbenchmark: FMA-pipe throughput per instruction form on sm_100a (development tool).
// 16 independent chains per thread, 2048 threads per SM; prints lane-ops per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  float2 v = make_float2(a, b);
  return *reinterpret_cast<unsigned long long *>(&v);
}
__device__ __forceinline__ float upk(unsigned long long v) {
  float2 f = *reinterpret_cast<float2 *>(&v);
  return f.x + f.y;
}

// FFMA, 3 register sources
__global__ void k_ffma_reg(float *out, const float *in) {
  float x[16], acc[16];
  const float y = in[threadIdx.x & 7];
#pragma unroll
  for (int i = 0; i < 16; i++) { x[i] = in[i + 8]; acc[i] = threadIdx.x * 1e-3f + i; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc[i]) : "f"(x[i]), "f"(y));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// FFMA with an immediate multiplier
__global__ void k_ffma_imm(float *out, const float *in) {
  float x[16], acc[16];
#pragma unroll
  for (int i = 0; i < 16; i++) { x[i] = in[i + 8]; acc[i] = threadIdx.x * 1e-3f + i; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) asm volatile("fma.rn.f32 %0, %1, 0f3F7FBE77, %0;" : "+f"(acc[i]) : "f"(x[i]));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
struct Taps { float c[16]; };
// FFMA with a kernel-parameter (constant bank) multiplier
__global__ void k_ffma_cb(float *out, const float *in, const __grid_constant__ Taps t) {
  float x[16], acc[16];
#pragma unroll
  for (int i = 0; i < 16; i++) { x[i] = in[i + 8]; acc[i] = threadIdx.x * 1e-3f + i; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) acc[i] = fmaf(x[i], t.c[i], acc[i]);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// FADD, 2 register sources
__global__ void k_fadd(float *out, const float *in) {
  float x[16], acc[16];
#pragma unroll
  for (int i = 0; i < 16; i++) { x[i] = in[i + 8]; acc[i] = threadIdx.x * 1e-3f + i; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(acc[i]) : "f"(x[i]));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// FFMA2, 3 register-pair sources
__global__ void k_ffma2(float *out, const float *in) {
  unsigned long long x[8], acc[8];
  const unsigned long long y = pk(in[threadIdx.x & 7], in[1]);
#pragma unroll
  for (int i = 0; i < 8; i++) { x[i] = pk(in[i + 8], in[i + 9]); acc[i] = pk(threadIdx.x * 1e-3f + i, i); }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i]) : "l"(x[i]), "l"(y));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += upk(acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// FADD2
__global__ void k_fadd2(float *out, const float *in) {
  unsigned long long x[8], acc[8];
#pragma unroll
  for (int i = 0; i < 8; i++) { x[i] = pk(in[i + 8], in[i + 9]); acc[i] = pk(threadIdx.x * 1e-3f + i, i); }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc[i]) : "l"(x[i]));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += upk(acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mixed: per iteration 1 FADD2 + 1 FFMA2 (the symmetric-fold pattern) on 8 chains
__global__ void k_mix(float *out, const float *in) {
  unsigned long long x[8], acc[8], z[8];
  const unsigned long long y = pk(in[threadIdx.x & 7], in[1]);
#pragma unroll
  for (int i = 0; i < 8; i++) { x[i] = pk(in[i + 8], in[i + 9]); z[i] = x[i]; acc[i] = pk(threadIdx.x * 1e-3f + i, i); }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      unsigned long long t;
      asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(x[i]), "l"(z[(i + 1) & 7]));
      asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i]) : "l"(t), "l"(y));
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += upk(acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount, clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *out, *in;
  cudaMalloc(&out, sizeof(float) * sms * 2048);
  cudaMalloc(&in, sizeof(float) * 64);
  float h[64];
  for (int i = 0; i < 64; i++) h[i] = 0.5f + 1e-3f * i;
  cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  Taps t;
  for (int i = 0; i < 16; i++) t.c[i] = 0.99f + 1e-4f * i;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int bs = 256, grid = sms * 8;
  auto run = [&](const char *name, auto launch, double lane_ops_per_thread) {
    launch();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = lane_ops_per_thread * grid * bs;
    double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
    printf("%-10s %8.3f ms  %7.1f lane-ops/clk/SM (at the %d MHz rated clock)  %.1f Gop/s\n", name, ms, per_clk_sm,
           clk / 1000, ops / ms / 1e6);
  };
  for (int rep = 0; rep < 2; rep++) {
    run("ffma_reg", [&] { k_ffma_reg<<<grid, bs>>>(out, in); }, 16.0 * ITERS);
    run("ffma_imm", [&] { k_ffma_imm<<<grid, bs>>>(out, in); }, 16.0 * ITERS);
    run("ffma_cb", [&] { k_ffma_cb<<<grid, bs>>>(out, in, t); }, 16.0 * ITERS);
    run("fadd", [&] { k_fadd<<<grid, bs>>>(out, in); }, 16.0 * ITERS);
    run("ffma2", [&] { k_ffma2<<<grid, bs>>>(out, in); }, 16.0 * ITERS);
    run("fadd2", [&] { k_fadd2<<<grid, bs>>>(out, in); }, 16.0 * ITERS);
    run("mix", [&] { k_mix<<<grid, bs>>>(out, in); }, 32.0 * ITERS);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
