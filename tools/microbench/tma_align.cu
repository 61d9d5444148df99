// Does a TMA tiled load accept a box whose x start is not 16-byte aligned in global memory?
// Loads a (36 x 2) fp32 box at x = 0, 1, 2, 3 of a 64 x 4 tensor and checks the shared copy.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void k(const __grid_constant__ CUtensorMap map, float *out, int x0) {
  __shared__ __align__(128) float buf[2 * 36];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)), "r"(2 * 36 * 4));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"((unsigned)__cvta_generic_to_shared(buf)), "l"(&map), "r"(x0), "r"(1), "r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W; }" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
    for (int i = 0; i < 72; i++) out[i] = buf[i];
  }
}

int main() {
  float h[64 * 4];
  for (int i = 0; i < 256; i++) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, sizeof h);
  cudaMalloc(&o, 72 * 4);
  cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                           const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                           CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                           CUtensorMapFloatOOBfill)>(fn);
  CUtensorMap map;
  cuuint64_t dims[2] = {64, 4}, strides[1] = {64 * 4};
  cuuint32_t box[2] = {36, 2}, es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  const int xs[7] = {0, 4, -4, 2, 1, -2, -3};
  for (int xi = 0; xi < 7; xi++) {
    const int x0 = xs[xi];
    k<<<1, 32>>>(map, o, x0);
    cudaError_t e = cudaDeviceSynchronize();
    float ho[72];
    cudaMemcpy(ho, o, sizeof ho, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int rr = 0; rr < 2; rr++)
      for (int c = 0; c < 36; c++) {
        int gx = x0 + c;
        float want = (gx >= 0 && gx < 64) ? h[(1 + rr) * 64 + gx] : 0.f;
        if (ho[rr * 36 + c] != want) bad++;
      }
    printf("x0=%d err=%s mismatches=%d\n", x0, cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
