// Host helpers: thread-local error string, launch checks, device queries and
// TMA tensor-map encoding through the driver entry point.
#include "host.h"

#include <atomic>

#include "../../include/ppmoe_capi.h"

namespace ppmoe {

static thread_local std::string g_last_error;
static std::atomic<unsigned long long> g_launches{0};  // diagnostic: kernels launched by this library

int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

const char* last_error() { return g_last_error.c_str(); }

int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(kErrCuda, "%s: launch failed: %s", what, cudaGetErrorString(e));
  return kOk;
}

int num_sms() {
  static thread_local int cached_dev = -1, cached = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev) {
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    cached_dev = dev;
  }
  return cached;
}

static thread_local int g_gemm_sm_budget = 0;
int gemm_ctas() {
  const int n = num_sms();
  return (g_gemm_sm_budget > 0 && g_gemm_sm_budget < n) ? g_gemm_sm_budget : n;
}

int max_smem_optin() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

int make_tmap_2d(CUtensorMap* map, const void* base, int dtype, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                 uint32_t box_inner, uint32_t box_outer) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return set_error(kErrCuda, "cuTensorMapEncodeTiled unavailable from the driver");
  if (row_bytes % 16 != 0)
    return set_error(kErrUnsupported, "TMA needs 16-byte aligned row pitch (got %llu bytes)",
                     static_cast<unsigned long long>(row_bytes));
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0) return set_error(kErrUnsupported, "TMA base must be 16-byte aligned");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, dtype == 0 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(kErrCuda, "cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu box=%ux%u", int(r),
                     static_cast<unsigned long long>(inner), static_cast<unsigned long long>(outer), box_inner,
                     box_outer);
  return kOk;
}

}  // namespace ppmoe

extern "C" {

int ppmoe_version(void) { return 1; }
const char* ppmoe_last_error(void) { return ppmoe::last_error(); }
int ppmoe_num_sms(void) { return ppmoe::num_sms(); }
int ppmoe_set_gemm_sm_budget(int sms) {
  if (sms < 0) return ppmoe::set_error(ppmoe::kErrInvalidArg, "sm budget must be >= 0 (0 = all SMs)");
  ppmoe::g_gemm_sm_budget = sms;
  return 0;
}
unsigned long long ppmoe_kernel_launches(void) { return ppmoe::g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
