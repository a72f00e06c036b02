// Host-side helpers shared by the C-ABI translation units: error reporting,
// launch checking and TMA tensor-map encoding (driver entry point fetched at
// run time, so the library links only against the CUDA runtime).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

namespace ppmoe {

enum Status : int {
  kOk = 0,
  kErrInvalidArg = -1,  // maps to ValueError on the Python side
  kErrCuda = -2,        // maps to RuntimeError
  kErrUnsupported = -3, // maps to ValueError (shape not supported by this build)
  kErrWorkspace = -4,
};

int set_error(int code, const char* fmt, ...);
const char* last_error();
int check_launch(const char* what);
int num_sms();
// CTAs for the persistent GEMM grids: all SMs unless a budget was set (to leave SMs to
// a concurrently running collective).
int gemm_ctas();
int max_smem_optin();

// Encodes a 2-D bf16/fp32 tensor map with SWIZZLE_128B boxes of box_inner x box_outer
// elements. `inner` is the contiguous extent, `outer` the row count, `row_bytes` the
// row pitch.
int make_tmap_2d(CUtensorMap* map, const void* base, int dtype, uint64_t inner, uint64_t outer,
                 uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer);

}  // namespace ppmoe

#define PPMOE_REQUIRE(cond, ...)                                   \
  do {                                                             \
    if (!(cond)) return ::ppmoe::set_error(::ppmoe::kErrInvalidArg, __VA_ARGS__); \
  } while (0)

#define PPMOE_CUDA(call)                                                                     \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return ::ppmoe::set_error(::ppmoe::kErrCuda, "%s failed: %s", #call, cudaGetErrorString(e_)); \
  } while (0)
