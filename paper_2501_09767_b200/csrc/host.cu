// Host-side plumbing for liblemo: error reporting, TMA descriptor encoding
// (driver entry point fetched at run time, so the library does not link
// libcuda directly) and a small per-process descriptor cache keyed by
// (device, pointer, shape, box) -- one process may drive several GPUs and the
// same virtual address may back different allocations on different devices.
// The library never allocates device memory (the split-K tail scratch below
// is the one library-owned buffer, one per device and stream).
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "gemm.cuh"
#include "lemo_internal.h"

namespace lemo {

static thread_local std::string g_last_error;

void set_error(const char* where, int code) {
  char buf[512];
  const char* msg = cudaGetErrorString((cudaError_t)code);
  snprintf(buf, sizeof(buf), "%s: error %d (%s)", where, code, msg ? msg : "?");
  g_last_error = buf;
}

void set_error_msg(const char* msg) { g_last_error = msg; }

const char* last_error() { return g_last_error.c_str(); }

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
  });
  return fn;
}

struct TmaKey {
  uint64_t base, rows, cols, ld, box;
  int dev;
  bool operator==(const TmaKey& o) const {
    return base == o.base && rows == o.rows && cols == o.cols && ld == o.ld && box == o.box &&
           dev == o.dev;
  }
};
struct TmaKeyHash {
  size_t operator()(const TmaKey& k) const {
    uint64_t h = (k.base ^ ((uint64_t)k.dev << 56)) * 0x9E3779B97F4A7C15ull;
    h ^= (k.rows + 0x632BE59BD9B4E019ull + (h << 6) + (h >> 2));
    h ^= (k.cols + 0x85EBCA77C2B2AE63ull + (h << 6) + (h >> 2));
    h ^= (k.ld + (h << 6) + (h >> 2));
    h ^= (k.box + (h << 6) + (h >> 2));
    return (size_t)h;
  }
};

static std::mutex g_tma_mu;
static std::unordered_map<TmaKey, CUtensorMap, TmaKeyHash> g_tma_cache;

static int make_tma_2d(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols,
                       uint64_t ld_elems, uint32_t box_rows, bool f32);

int make_tma_bf16_2d(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols,
                     uint64_t ld_elems, uint32_t box_rows) {
  return make_tma_2d(out, base, rows, cols, ld_elems, box_rows, false);
}

int make_tma_f32_2d(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols,
                    uint64_t ld_elems, uint32_t box_rows) {
  return make_tma_2d(out, base, rows, cols, ld_elems, box_rows, true);
}

// box = (128 B of columns) x box_rows, SWIZZLE_128B; f32 keys are tagged in `box`
static int make_tma_2d(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols,
                       uint64_t ld_elems, uint32_t box_rows, bool f32) {
  const uint64_t esz = f32 ? 4 : 2;
  int dev = 0;
  cudaGetDevice(&dev);
  TmaKey key{(uint64_t)base, rows, cols, ld_elems, box_rows | (f32 ? (1ull << 40) : 0ull), dev};
  {
    std::lock_guard<std::mutex> lk(g_tma_mu);
    auto it = g_tma_cache.find(key);
    if (it != g_tma_cache.end()) {
      *out = it->second;
      return 0;
    }
  }
  auto fn = get_encode_fn();
  if (!fn) {
    set_error_msg("cuTensorMapEncodeTiled unavailable");
    return LEMO_ERR_REPORTED;
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld_elems * esz) & 15)) {
    set_error_msg("TMA operand must be 16-byte aligned with a 16-byte multiple row pitch");
    return LEMO_ERR_REPORTED;
  }
  cuuint64_t gdim[2] = {cols, rows};
  cuuint64_t gstride[1] = {ld_elems * esz};
  cuuint32_t box[2] = {(cuuint32_t)(128 / esz), box_rows};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = fn(out, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                  2, const_cast<void*>(base), gdim,
                  gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[256];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d) rows=%llu cols=%llu ld=%llu",
             (int)r, (unsigned long long)rows, (unsigned long long)cols,
             (unsigned long long)ld_elems);
    set_error_msg(buf);
    return LEMO_ERR_REPORTED;
  }
  std::lock_guard<std::mutex> lk(g_tma_mu);
  if (g_tma_cache.size() > 8192) g_tma_cache.clear();
  g_tma_cache.emplace(key, *out);
  return 0;
}

bool pair_tail_enabled() {
  static const int env = getenv("LEMO_GEMM_TAIL") ? atoi(getenv("LEMO_GEMM_TAIL")) : 1;
  return env != 0;
}

namespace {
struct TailWs {
  float* ws = nullptr;
  int* ctr = nullptr;
};
std::mutex g_tail_mu;
std::unordered_map<std::string, TailWs> g_tail_ws;
}  // namespace

int pair_tail_workspace(cudaStream_t stream, int units, int tiles, float** ws, int** ctr) {
  // sized once for the largest possible tail (one unit per cluster)
  const int max_units = gemm_num_sms() / 2;
  if (units > max_units || tiles > max_units) return (int)cudaErrorInvalidValue;
  int dev = 0;
  cudaGetDevice(&dev);
  const std::string key = std::to_string(dev) + ":" + std::to_string((uintptr_t)stream);
  std::lock_guard<std::mutex> lk(g_tail_mu);
  auto it = g_tail_ws.find(key);
  if (it == g_tail_ws.end()) {
    TailWs t;
    const size_t bytes = (size_t)max_units * 2 * 128 * 256 * sizeof(float);
    cudaError_t e = cudaMalloc(&t.ws, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&t.ctr, (size_t)max_units * 2 * sizeof(int));
    if (e == cudaSuccess) e = cudaMemsetAsync(t.ctr, 0, (size_t)max_units * 2 * sizeof(int), stream);
    if (e != cudaSuccess) return (int)e;
    it = g_tail_ws.emplace(key, t).first;
  }
  *ws = it->second.ws;
  *ctr = it->second.ctr;
  return 0;
}

int gemm_num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = kNumSMs;
  }
  return n;
}

}  // namespace lemo

extern "C" {

const char* lemo_last_error(void) { return lemo::last_error(); }

int lemo_version(void) { return LEMO_ABI_VERSION; }

void lemo_clear_descriptor_cache(void) {
  std::lock_guard<std::mutex> lk(lemo::g_tma_mu);
  lemo::g_tma_cache.clear();
}

}  // extern "C"
