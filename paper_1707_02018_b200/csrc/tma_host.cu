// Host-side TMA descriptor encoding for libwl (cuTensorMapEncodeTiled through the runtime's
// driver entry point, so the library has no link-time dependency on libcuda).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "wl_internal.h"

namespace wl {
namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

}  // namespace

bool encode_tmap_3d(void *map, int elem_bytes, const void *base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                    uint64_t s2, uint32_t box0, uint32_t box1) {
  // Encoding costs microseconds of host time per descriptor; operators called repeatedly on
  // the same buffers (solver loops, benchmarks) reuse the cached descriptor.
  using Key = std::tuple<int, const void *, uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t>;
  static std::mutex mu;
  static std::map<Key, CUtensorMap> cache;
  const Key key(elem_bytes, base, d0, d1, d2, s1, s2, box0, box1);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *reinterpret_cast<CUtensorMap *>(map) = it->second;
      return true;
    }
  }
  EncodeTiledFn enc = encode_tiled_fn();
  if (!enc || !base || (reinterpret_cast<uintptr_t>(base) & 15) || (s1 & 15) || (s2 & 15)) return false;
  if (box0 == 0 || box1 == 0 || box0 > 256 || box1 > 256 || (box0 * (uint32_t)elem_bytes) % 16) return false;
  cuuint64_t dims[3] = {d0, d1, d2 > 0 ? d2 : 1};
  cuuint64_t strides[2] = {s1, s2 > 0 ? s2 : s1 * d1};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap *>(map),
                   elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                   const_cast<void *>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache[key] = *reinterpret_cast<CUtensorMap *>(map);
  return true;
}

bool tma_enabled() {
  static const bool v = getenv("WL_NO_TMA") == nullptr;
  return v;
}

bool zero_taps_enabled() {
  static const bool v = getenv("WL_ALL_TAPS") == nullptr;
  return v;
}

int match_tap_range(const double *lo, const double *hi, int L) {
  if (L != 10) return 0;
  auto range = [&](const double *f, int &a, int &b) {
    a = L;
    b = 0;
    for (int j = 0; j < L; j++)
      if (f[j] != 0.0) {
        a = std::min(a, j);
        b = std::max(b, j + 1);
      }
  };
  int l0, l1, h0, h1;
  range(lo, l0, l1);
  range(hi, h0, h1);
  if (l0 == 2 && l1 == 9 && h0 == 0 && h1 == 9) return 1;
  if (l0 == 1 && l1 == 10 && h0 == 1 && h1 == 8) return 2;
  return 0;
}

bool balanced_runs() {
  // measured on B200: balanced runs lose badly (cfg5 W* level 1 170 vs 108 us, grad 666 vs 561 us):
  // strips that no longer stream the same rows at the same time break the DRAM page locality of
  // their 0.5 KB box rows.  Banded unless WL_BALANCED is set (A/B).
  static const bool v = getenv("WL_BALANCED") != nullptr;
  return v;
}

bool plain_enabled() {
  static const bool v = getenv("WL_NO_PLAIN") == nullptr;
  return v;
}

bool multi_enabled() {
  // measured on B200 (graph replay): the cooperative multi-level tail lost to per-level PDL
  // launches (cfg4 W* 96 vs 80 us, cfg2 W* 26 vs 17 us): off unless WL_MULTI is set
  static const bool v = getenv("WL_MULTI") != nullptr;
  return v;
}

bool pdl_enabled(char kind) {
  static const char *off = [] {
    // measured on B200 (cfg5 grad -1.3 %, cfg3 grad -2.7 %, cfg4 W* neutral): the long blur and
    // the long analysis launches do better without early launch (their CTAs, pre-placed while the
    // previous kernel drains, cost that kernel's tail more than they save)
    const char *e = getenv("WL_NO_PDL");
    return e ? e : "bA";
  }();
  return strchr(off, kind) == nullptr;
}

int short_run_max(int dflt, char kind) {
  static const int v = [] {
    const char *e = getenv("WL_SHORT_MAX");
    return e ? atoi(e) : -1;
  }();
  static const int va = [] {
    const char *e = getenv("WL_SHORT_MAX_A");  // analysis only
    return e ? atoi(e) : -1;
  }();
  static const int vs = [] {
    const char *e = getenv("WL_SHORT_MAX_S");  // synthesis only
    return e ? atoi(e) : -1;
  }();
  const int k = kind == 'a' ? va : (kind == 's' ? vs : -1);
  return k >= 0 ? k : (v >= 0 ? v : dflt);
}

cudaError_t kernel_resident(const void *kern, int nt, size_t smem, long long *resident) {
  static std::mutex mu;
  static std::map<std::tuple<const void *, int, int, size_t>, long long> cache;
  static std::map<std::pair<const void *, int>, size_t> opted;  // largest smem opted in per (kernel, device)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_tuple(kern, dev, nt, smem);
  std::lock_guard<std::mutex> g(mu);
  // the opt-in only ever grows: a later, smaller request must not lower it below a size
  // another (cached) launch of the same kernel relies on
  size_t &cur = opted[std::make_pair(kern, dev)];
  if (smem > cur) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cur = smem;
  }
  auto it = cache.find(key);
  if (it != cache.end()) {
    *resident = it->second;
    return cudaSuccess;
  }
  int sms = 0, occ = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, smem);
  if (e != cudaSuccess) return e;
  const long long r = (long long)sms * (occ > 0 ? occ : 1);
  cache[key] = r;
  *resident = r;
  return cudaSuccess;
}

}  // namespace wl
