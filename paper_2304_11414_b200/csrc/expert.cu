// Expert FFN forward/backward entry points: the six grouped GEMMs of one MoE
// layer step (fc1/fc2 forward, fc2/fc1 data-gradient, fc2/fc1 weight-gradient)
// plus the bias-gradient column sums.  bf16 runs on the tcgen05/TMA kernel,
// fp32 (reference-precision mode) on the CUDA-core kernel.
#include "../../include/ppmoe_capi.h"
#include "epilogues.cuh"
#include "grouped_gemm.cuh"
#include "host.h"

#include <cstdlib>
#include <cstring>

namespace ppmoe {

using bf16 = __nv_bfloat16;
constexpr int kBN = 256;

// Which tcgen05 kernel runs a grouped GEMM.  Default: the CTA-pair (cta_group::2,
// 256x256) kernel (fastest in interleaved A/B runs of the whole C2 step, tools/ab.py).
// PPMOE_GEMM=single forces the 1-CTA 128x256 kernel; PPMOE_GEMM=auto uses the 1-CTA
// kernel for token-segment GEMMs with a long K (fc2 forward, fc1 data-gradient), which
// in isolation (ncu) move ~40 % less DRAM.
static thread_local int g_force_mode = 0;  // 0: env/default, 1: single, 2: pair
static thread_local int g_long_k = 0;      // the GEMM being launched has K >= kLongK
constexpr int kLongK = 8192;
static bool use_pair() {
  if (g_force_mode) return g_force_mode == 2;
  static const int env_mode = [] {
    const char* e = getenv("PPMOE_GEMM");
    if (e && strcmp(e, "single") == 0) return 1;
    if (e && strcmp(e, "auto") == 0) return 0;
    return 2;
  }();
  if (env_mode) return env_mode == 2;
  return !g_long_k;
}
struct LongKScope {  // marks a token-segment GEMM with a long reduction dimension
  explicit LongKScope(int K) { g_long_k = K >= kLongK; }
  ~LongKScope() { g_long_k = 0; }
};

// Narrow 256 x 128 pair tile for the long-K token GEMMs (fc2 fwd, fc1 dgrad: N = H).  With
// few expert rows per GPU (T >= 4) their 256-wide tile count leaves a ragged last wave
// (C2 T = 4: 544 tiles on 74 CTA pairs = 7.35 waves); the narrow tile doubles the tile count.
// PPMOE_NARROW: 0 never (default), 1 the long-K token GEMMs; ppmoe_set_gemm_narrow(1)
// selects it for the calling thread's next launches (the layer decides from its shape).
static thread_local int g_force_narrow = -1;
static bool use_narrow() {
  if (!g_long_k) return false;
  if (g_force_narrow >= 0) return g_force_narrow != 0;
  const char* e = getenv("PPMOE_NARROW");
  return e && atoi(e) != 0;
}

// Rows of a K-major B box: the pair kernel stages half of each MMA's B columns per CTA.
static uint32_t b_box_rows() { return use_pair() ? (use_narrow() ? kBN / 4 : kBN / 2) : kBN; }

// Pair-kernel tile width: 256 x 512 ("wide", two MMAs per k-step, 25 % fewer L2 -> SM
// bytes, epilogue not overlapped) or 256 x 256 (double-buffered TMEM).  PPMOE_WIDE:
// 0 = never, 1 = every GEMM, long = the long-K token GEMMs (fc2 fwd, fc1 dgrad).  Read per
// launch (A/B runs).
static thread_local int g_force_wide = -1;
// Warp-cooperative staged epilogue stores for the wide tile (PPMOE_STAGE: 0 off, 1 on,
// unset = on); its epilogue is exposed.  The 256-wide tile has no staging buffer (its
// epilogue overlaps the next tile's mainloop) and ignores the switch.  Read per launch.
static int staged_stores(bool wide) {
  const char* e = getenv("PPMOE_STAGE");
  if (!e) return wide ? 1 : 0;
  return atoi(e) != 0;
}
static bool use_wide() {
  if (g_force_wide >= 0) return g_force_wide != 0;
  const char* e = getenv("PPMOE_WIDE");
  if (!e) return false;
  if (strcmp(e, "long") == 0) return g_long_k != 0;
  return atoi(e) != 0;
}

// The soft wave synchronisation's counter: module-scope device storage (one word per device
// context, created with the module image, never cudaMalloc'd), reset on the launch stream
// before every synchronised GEMM.  Synchronised GEMMs of one device are stream-ordered.
__device__ unsigned int g_ksync_counter;

// M = 128 tail tiles of the token GEMMs (PPMOE_TAIL128=0 turns them off for A/B runs)
static bool tail128_on() {
  const char* e = getenv("PPMOE_TAIL128");  // read per launch: tools/ab_env.py switches it in-process
  return !e || atoi(e) != 0;
}
template <bool A_MN, bool B_MN, class Epi>
static int launch_tc(const CUtensorMap& ta, const CUtensorMap& tb, const GroupGeom& geo_in, const Epi& epi,
                     cudaStream_t s) {
  GroupGeom geo = geo_in;
  if (geo.ksync > 0 && geo.K_fixed > 0) {  // soft wave synchronisation (see GroupGeom::ksync)
    void* ctr = nullptr;
    PPMOE_CUDA(cudaGetSymbolAddress(&ctr, g_ksync_counter));
    PPMOE_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned int), s));
    geo.ksync_ctr = static_cast<unsigned int*>(ctr);
  } else {
    geo.ksync = 0;
  }
  if (use_pair()) {
    geo.stage = staged_stores(use_wide());
    geo.tail128 = !A_MN && !use_wide() && !use_narrow() && tail128_on();
    if (use_narrow() && !use_wide()) {
      auto kern = grouped_gemm_sm100_pair<kBN / 2, A_MN, B_MN, Epi>;
      constexpr int smem = PairSmem<kBN / 2>::kTotal;
      PPMOE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kern<<<gemm_ctas() / 2 * 2, kPairThreads, smem, s>>>(ta, tb, geo, epi);
      return check_launch("grouped_gemm_sm100_pair");
    }
    if (use_wide()) {
      auto kern = grouped_gemm_sm100_pair<2 * kBN, A_MN, B_MN, Epi>;
      constexpr int smem = PairSmem<2 * kBN>::kTotal;
      PPMOE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kern<<<gemm_ctas() / 2 * 2, kPairThreads, smem, s>>>(ta, tb, geo, epi);
      return check_launch("grouped_gemm_sm100_pair");
    }
    auto kern = grouped_gemm_sm100_pair<kBN, A_MN, B_MN, Epi>;
    constexpr int smem = PairSmem<kBN>::kTotal;
    PPMOE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<gemm_ctas() / 2 * 2, kPairThreads, smem, s>>>(ta, tb, geo, epi);
    return check_launch("grouped_gemm_sm100_pair");
  }
  auto kern = grouped_gemm_sm100<kBN, A_MN, B_MN, Epi>;
  constexpr int smem = GemmSmem<kBN>::kTotal;
  PPMOE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<gemm_ctas(), kGemmThreads, smem, s>>>(ta, tb, geo, epi);
  return check_launch("grouped_gemm_sm100");
}

template <typename T, bool A_MN, bool B_MN, class Epi>
static int launch_simt(const T* A, int lda, const T* B, int ldb, const GroupGeom& geo, int m_upper, const Epi& epi,
                       cudaStream_t s) {
  dim3 grid((geo.N + 63) / 64, (m_upper + 63) / 64, geo.G);
  if (grid.y == 0) return kOk;
  grouped_gemm_simt<T, A_MN, B_MN, Epi><<<grid, 256, 0, s>>>(A, lda, B, ldb, geo, epi);
  return check_launch("grouped_gemm_simt");
}

// Operand tensor maps: K-major -> box {64 (K), rows}; MN-major -> box {64 (MN), 64 (K)}.
static int tmap_kmajor(CUtensorMap* m, const void* p, uint64_t k_extent, uint64_t rows, uint32_t box_rows) {
  return make_tmap_2d(m, p, kBF16, k_extent, rows, k_extent * 2, 64, box_rows);
}
static int tmap_mnmajor(CUtensorMap* m, const void* p, uint64_t mn_extent, uint64_t k_rows) {
  return make_tmap_2d(m, p, kBF16, mn_extent, k_rows, mn_extent * 2, 64, 64);
}

static int check_common(int dtype, int El, int H, int F, int rows_cap) {
  PPMOE_REQUIRE(dtype == kBF16 || dtype == kF32, "dtype must be 0 (bf16) or 1 (fp32), got %d", dtype);
  PPMOE_REQUIRE(El >= 1 && El <= kMaxGroups, "local experts must be in [1, %d], got %d", kMaxGroups, El);
  PPMOE_REQUIRE(H >= 1 && F >= 1 && rows_cap >= 0, "bad expert shape H=%d F=%d rows_cap=%d", H, F, rows_cap);
  if (dtype == kBF16)
    PPMOE_REQUIRE(H % 8 == 0 && F % 8 == 0,
                  "bf16 expert path needs hidden and ffn widths divisible by 8 (TMA row pitch), got H=%d F=%d", H, F);
  return kOk;
}

// Bias gradients: column sums of a per-expert row segment.  Block = 64 columns x 8 row
// groups; each warp reads one 128-byte row slice per step; the 8 partial sums are
// combined in a fixed order (deterministic, no atomics).
template <typename T>
__global__ void __launch_bounds__(256) colsum_kernel(const T* __restrict__ src, int ld, const int* __restrict__ seg,
                                                     int N, T* __restrict__ out) {
  __shared__ float red[8][64];
  const int g = blockIdx.y;
  const int lane = threadIdx.x & 31, rg = threadIdx.x >> 5;
  const int col = blockIdx.x * 64 + 2 * lane;
  const int lo = seg[g] - seg[0];
  const int hi = seg[g + 1] - seg[0];
  float s0 = 0.f, s1 = 0.f;
  if (col < N) {
    const bool pair = col + 1 < N;
    int r = lo + rg;
#pragma unroll 4
    for (; r < hi; r += 8) {
      const T* p = src + static_cast<size_t>(r) * ld + col;
      s0 += to_f32(p[0]);
      if (pair) s1 += to_f32(p[1]);
    }
  }
  red[rg][2 * lane] = s0;
  red[rg][2 * lane + 1] = s1;
  __syncthreads();
  if (threadIdx.x < 64) {
    const int c = blockIdx.x * 64 + threadIdx.x;
    float t = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += red[q][threadIdx.x];
    if (c < N) out[static_cast<size_t>(g) * N + c] = from_f32<T>(t);
  }
}

template <typename T>
static int colsum(const void* src, int ld, const int* seg, int G, int N, void* out, cudaStream_t s) {
  if (!out) return kOk;
  dim3 grid((N + 63) / 64, G);
  colsum_kernel<T><<<grid, 256, 0, s>>>(static_cast<const T*>(src), ld, seg, N, static_cast<T*>(out));
  return check_launch("colsum");
}

// Tile order of the tcgen05 kernels (panel by default; PPMOE_ORDER=band selects the
// banded order) and the epilogue store cache policy (streaming by default;
// PPMOE_STORE=normal disables it).
static int banded_order() {
  const char* e = getenv("PPMOE_ORDER");
  return (e && strcmp(e, "band") == 0) ? 1 : 0;
}
// Tile order of the long-K token GEMMs (fc2 fwd, fc1 dgrad) alone: PPMOE_ORDER_LONG=band puts
// them in square-ish 8-tile bands (a wave reads ~8 A + ~9 B panels instead of ~5 A + all 16 B
// panels of an expert), with the wave sync keeping the bands' k-slices L2-resident.
static int banded_order_long() {
  const char* e = getenv("PPMOE_ORDER_LONG");
  if (!e) return banded_order();
  return strcmp(e, "band") == 0 ? 1 : 0;
}
// k-blocks between the soft wave barriers of the GEMMs that use them (PPMOE_KSYNC, 0 = off).
// Enabled for fc2 fwd, fc2 dgrad and fc1 dgrad: halves their DRAM traffic, which under the
// power cap buys clock; fc1 fwd measured slower with it.
static int ksync_interval() {
  const char* e = getenv("PPMOE_KSYNC");
  return e ? atoi(e) : 64;
}

static int load_hint() {
  const char* e = getenv("PPMOE_HINT");
  return (e && strcmp(e, "1") == 0) ? 1 : 0;
}
// Epilogue store flavour: 0 = plain 16-byte stores (default), 1 = 16-byte evict-first
// (PPMOE_STORE=cs), 2 = 32-byte stores (PPMOE_STORE=v8; measured 5 % slower in the C2
// step).  Read per launch (A/B runs).
static int stream_stores() {
  const char* e = getenv("PPMOE_STORE");
  if (e && strcmp(e, "cs") == 0) return 1;
  if (e && strcmp(e, "v8") == 0) return 2;
  return 0;
}

// Bias gradient from per-32-row-block column partials: out[g][c] = sum of the blocks of
// segment g, in block order (deterministic).
template <typename T>
__global__ void colsum_parts_kernel(const float* __restrict__ part, const int* __restrict__ seg, int N,
                                    T* __restrict__ out) {
  const int g = blockIdx.y;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= N) return;
  const int b0 = (seg[g] - seg[0]) >> 5, b1 = (seg[g + 1] - seg[0]) >> 5;
  float a0 = 0.f, a1 = 0.f;
  int b = b0;
  for (; b + 2 <= b1; b += 2) {
    a0 += part[static_cast<size_t>(b) * N + col];
    a1 += part[static_cast<size_t>(b + 1) * N + col];
  }
  if (b < b1) a0 += part[static_cast<size_t>(b) * N + col];
  out[static_cast<size_t>(g) * N + col] = from_f32<T>(a0 + a1);
}

template <typename T>
static int colsum_parts(const float* part, const int* seg, int G, int N, void* out, cudaStream_t s) {
  if (!out) return kOk;
  dim3 grid((N + 255) / 256, G);
  colsum_parts_kernel<T><<<grid, 256, 0, s>>>(part, seg, N, static_cast<T*>(out));
  return check_launch("colsum_parts");
}

static GroupGeom geom(int G, int N, int M_fixed, int K_fixed, const int* seg, int a_seg, int a_stride, int b_seg,
                      int b_stride) {
  GroupGeom g;
  g.rlo = nullptr;
  g.rhi = nullptr;
  g.banded = banded_order();
  {
    const char* e = getenv("PPMOE_NFAST");
    g.nfast = e ? atoi(e) : -1;
  }
  g.ksync_ctr = nullptr;
  g.ksync = 0;
  g.stage = 0;
  g.tail128 = 0;
  g.hint = load_hint();
  g.G = G;
  g.N = N;
  g.M_fixed = M_fixed;
  g.K_fixed = K_fixed;
  g.seg = seg;
  g.a_seg = a_seg;
  g.a_stride = a_stride;
  g.b_seg = b_seg;
  g.b_stride = b_stride;
  return g;
}

static int fc2_fwd_impl(int dtype, const void* Act, const void* down, const void* bias_down, const int* seg, int El,
                        int H, int F, int rows_cap, const int* row_lo, const int* row_hi, const int* tok_local,
                        const float* w_local, int weight_scaling, float dropout_p, const unsigned long long* drop,
                        void* Y, void* Y2, float* out_acc, float* const* owner_acc, int owner_rows, void* const* owner_slots,
                        const int* pair_pos, int K, void* stream) {
  if (int rc = check_common(dtype, El, H, F, rows_cap)) return rc;
  PPMOE_REQUIRE((row_lo == nullptr) == (row_hi == nullptr), "row_lo and row_hi must both be given or both be NULL");
  PPMOE_REQUIRE(dropout_p >= 0.f && dropout_p < 1.f, "dropout probability must be in [0, 1), got %g", dropout_p);
  PPMOE_REQUIRE(dropout_p == 0.f || drop, "dropout needs its stream descriptor (ppmoe_dropout_stream)");
  PPMOE_REQUIRE(!(out_acc && owner_acc), "give at most one of out_acc / owner_acc");
  PPMOE_REQUIRE(!owner_acc || owner_rows >= 1, "owner_acc needs owner_rows >= 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  LongKScope long_k(F);
  GroupGeom geo = geom(El, H, 0, F, seg, 1, 0, 0, F);
  geo.rlo = row_lo;
  geo.rhi = row_hi;
  geo.ksync = ksync_interval();
  geo.banded = banded_order_long();
  if (rows_cap == 0) return kOk;
  if (dtype == kBF16) {
    CUtensorMap ta, tb;
    if (int rc = tmap_kmajor(&ta, Act, F, rows_cap, kBM)) return rc;
    if (int rc = tmap_mnmajor(&tb, down, H, static_cast<uint64_t>(El) * F)) return rc;
    EpiFc2Fwd<bf16> epi{static_cast<bf16*>(Y), static_cast<bf16*>(Y2), static_cast<const bf16*>(bias_down), H, seg,
                        tok_local, w_local, weight_scaling, out_acc, stream_stores(), dropout_p, drop, owner_acc,
                        owner_rows, reinterpret_cast<bf16* const*>(owner_slots), pair_pos, K};
    return launch_tc<false, true>(ta, tb, geo, epi, s);
  }
  PPMOE_REQUIRE(!owner_slots, "owner slots are a bf16 path");
  EpiFc2Fwd<float> epi{static_cast<float*>(Y), static_cast<float*>(Y2), static_cast<const float*>(bias_down), H, seg,
                       tok_local, w_local, weight_scaling, out_acc, 0, dropout_p, drop, owner_acc, owner_rows,
                       nullptr, nullptr, 0};
  return launch_simt<float, false, true>(static_cast<const float*>(Act), F, static_cast<const float*>(down), H, geo,
                                         rows_cap, epi, s);
}

}  // namespace ppmoe

using namespace ppmoe;

extern "C" {

int ppmoe_set_gemm_narrow(int narrow) {
  PPMOE_REQUIRE(narrow >= -1 && narrow <= 1, "gemm narrow: -1 env/default, 0 off, 1 long-K token GEMMs");
  g_force_narrow = narrow;
  return kOk;
}

int ppmoe_set_gemm_mode(int mode) {
  PPMOE_REQUIRE(mode >= 0 && mode <= 2, "gemm mode: 0 auto/env, 1 single-CTA, 2 CTA pair");
  g_force_mode = mode;
  return kOk;
}

int ppmoe_expert_fc1_fwd(int dtype, const void* Xs, const void* up, const void* bias_up, const int* seg, int El, int H,
                         int F, int rows_cap, const int* row_lo, const int* row_hi, void* GeluGrad, void* Act,
                         void* stream) {
  if (int rc = check_common(dtype, El, H, F, rows_cap)) return rc;
  PPMOE_REQUIRE((row_lo == nullptr) == (row_hi == nullptr), "row_lo and row_hi must both be given or both be NULL");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  GroupGeom geo = geom(El, F, 0, H, seg, 1, 0, 0, H);
  geo.rlo = row_lo;
  geo.rhi = row_hi;
  if (rows_cap == 0) return kOk;
  if (dtype == kBF16) {
    CUtensorMap ta, tb;
    if (int rc = tmap_kmajor(&ta, Xs, H, rows_cap, kBM)) return rc;
    if (int rc = tmap_mnmajor(&tb, up, F, static_cast<uint64_t>(El) * H)) return rc;
    EpiFc1Fwd<bf16> epi{static_cast<bf16*>(GeluGrad), static_cast<bf16*>(Act), static_cast<const bf16*>(bias_up), F, seg, stream_stores()};
    return launch_tc<false, true>(ta, tb, geo, epi, s);
  }
  EpiFc1Fwd<float> epi{static_cast<float*>(GeluGrad), static_cast<float*>(Act), static_cast<const float*>(bias_up), F, seg, 0};
  return launch_simt<float, false, true>(static_cast<const float*>(Xs), H, static_cast<const float*>(up), F, geo,
                                         rows_cap, epi, s);
}


int ppmoe_expert_fc2_fwd(int dtype, const void* Act, const void* down, const void* bias_down, const int* seg, int El,
                         int H, int F, int rows_cap, const int* row_lo, const int* row_hi, const int* tok_local,
                         const float* w_local, int weight_scaling, float dropout_p, const unsigned long long* drop_stream,
                         void* Y, void* Y2, float* out_acc, void* stream) {
  return fc2_fwd_impl(dtype, Act, down, bias_down, seg, El, H, F, rows_cap, row_lo, row_hi, tok_local, w_local,
                      weight_scaling, dropout_p, drop_stream, Y, Y2, out_acc, nullptr, 0, nullptr, nullptr, 0, stream);
}

int ppmoe_expert_fc2_fwd_owner(int dtype, const void* Act, const void* down, const void* bias_down, const int* seg,
                               int El, int H, int F, int rows_cap, const int* tok_local, const float* w_local,
                               int weight_scaling, float dropout_p, const unsigned long long* drop_stream, void* Y,
                               float* const* owner_acc, void* const* owner_slots, const int* pair_pos, int K,
                               int owner_rows, void* stream) {
  PPMOE_REQUIRE((owner_acc != nullptr) != (owner_slots != nullptr), "give exactly one of owner_acc / owner_slots");
  PPMOE_REQUIRE(!owner_slots || (pair_pos && K >= 1 && K <= 2), "owner slots need pair_pos and k <= 2");
  return fc2_fwd_impl(dtype, Act, down, bias_down, seg, El, H, F, rows_cap, nullptr, nullptr, tok_local, w_local,
                      weight_scaling, dropout_p, drop_stream, Y, nullptr, nullptr, owner_acc, owner_rows, owner_slots,
                      pair_pos, K, stream);
}

int ppmoe_expert_fc2_dgrad(int dtype, const void* dY, const void* down, const void* GeluGrad, const int* seg, int El, int H,
                           int F, int rows_cap, void* dH, float* dh_colsum_part, void* stream) {
  if (int rc = check_common(dtype, El, H, F, rows_cap)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  GroupGeom geo = geom(El, F, 0, H, seg, 1, 0, 0, F);
  geo.ksync = ksync_interval();
  if (rows_cap == 0) return kOk;
  if (dtype == kBF16) {
    CUtensorMap ta, tb;
    if (int rc = tmap_kmajor(&ta, dY, H, rows_cap, kBM)) return rc;
    if (int rc = tmap_kmajor(&tb, down, H, static_cast<uint64_t>(El) * F, b_box_rows())) return rc;
    EpiFc2Dgrad<bf16> epi{static_cast<bf16*>(dH), static_cast<const bf16*>(GeluGrad), F, seg, stream_stores(),
                          dh_colsum_part};
    return launch_tc<false, false>(ta, tb, geo, epi, s);
  }
  PPMOE_REQUIRE(dh_colsum_part == nullptr, "column-sum partials are produced by the bf16 tcgen05 path only");
  EpiFc2Dgrad<float> epi{static_cast<float*>(dH), static_cast<const float*>(GeluGrad), F, seg, 0, nullptr};
  return launch_simt<float, false, false>(static_cast<const float*>(dY), H, static_cast<const float*>(down), H, geo,
                                          rows_cap, epi, s);
}

int ppmoe_expert_fc1_dgrad(int dtype, const void* dH, const void* up, const int* seg, int El, int H, int F,
                           int rows_cap, const int* tok_local, float* dx_acc, void* dXs, void* stream) {
  PPMOE_REQUIRE((dx_acc == nullptr) != (dXs == nullptr), "give exactly one of dx_acc (scatter-add) or dXs (rows)");
  if (int rc = check_common(dtype, El, H, F, rows_cap)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  LongKScope long_k(F);
  GroupGeom geo = geom(El, H, 0, F, seg, 1, 0, 0, H);
  geo.ksync = ksync_interval();
  geo.banded = banded_order_long();
  if (rows_cap == 0) return kOk;
  if (dtype == kBF16) {
    CUtensorMap ta, tb;
    if (int rc = tmap_kmajor(&ta, dH, F, rows_cap, kBM)) return rc;
    if (int rc = tmap_kmajor(&tb, up, F, static_cast<uint64_t>(El) * H, b_box_rows())) return rc;
    EpiFc1Dgrad<bf16> epi{dx_acc, static_cast<bf16*>(dXs), H, seg, tok_local, stream_stores()};
    return launch_tc<false, false>(ta, tb, geo, epi, s);
  }
  EpiFc1Dgrad<float> epi{dx_acc, static_cast<float*>(dXs), H, seg, tok_local, 0};
  return launch_simt<float, false, false>(static_cast<const float*>(dH), F, static_cast<const float*>(up), F, geo,
                                          rows_cap, epi, s);
}

int ppmoe_expert_fc2_wgrad(int dtype, const void* Act, const void* dY, const int* seg, int El, int H, int F,
                           int rows_cap, void* dDown, void* dBiasDown, const float* dy_colsum_part, void* stream) {
  if (int rc = check_common(dtype, El, H, F, rows_cap)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  GroupGeom geo = geom(El, H, F, 0, seg, 1, 0, 1, 0);
  if (dtype == kBF16) {
    if (rows_cap > 0) {
      CUtensorMap ta, tb;
      if (int rc = tmap_mnmajor(&ta, Act, F, rows_cap)) return rc;
      if (int rc = tmap_mnmajor(&tb, dY, H, rows_cap)) return rc;
      EpiWgrad<bf16> epi{static_cast<bf16*>(dDown), F, H, stream_stores()};
      if (int rc = launch_tc<true, true>(ta, tb, geo, epi, s)) return rc;
    } else {
      PPMOE_CUDA(cudaMemsetAsync(dDown, 0, static_cast<size_t>(El) * F * H * 2, s));
    }
    if (dy_colsum_part) return colsum_parts<bf16>(dy_colsum_part, seg, El, H, dBiasDown, s);
    return colsum<bf16>(dY, H, seg, El, H, dBiasDown, s);
  }
  EpiWgrad<float> epi{static_cast<float*>(dDown), F, H, 0};
  if (int rc = launch_simt<float, true, true>(static_cast<const float*>(Act), F, static_cast<const float*>(dY), H, geo,
                                              F, epi, s))
    return rc;
  return colsum<float>(dY, H, seg, El, H, dBiasDown, s);
}

int ppmoe_expert_fc1_wgrad(int dtype, const void* Xs, const void* dH, const int* seg, int El, int H, int F,
                           int rows_cap, void* dUp, void* dBiasUp, const float* dh_colsum_part, void* stream) {
  if (int rc = check_common(dtype, El, H, F, rows_cap)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  GroupGeom geo = geom(El, F, H, 0, seg, 1, 0, 1, 0);
  if (dtype == kBF16) {
    if (rows_cap > 0) {
      CUtensorMap ta, tb;
      if (int rc = tmap_mnmajor(&ta, Xs, H, rows_cap)) return rc;
      if (int rc = tmap_mnmajor(&tb, dH, F, rows_cap)) return rc;
      EpiWgrad<bf16> epi{static_cast<bf16*>(dUp), H, F, stream_stores()};
      if (int rc = launch_tc<true, true>(ta, tb, geo, epi, s)) return rc;
    } else {
      PPMOE_CUDA(cudaMemsetAsync(dUp, 0, static_cast<size_t>(El) * H * F * 2, s));
    }
    if (dh_colsum_part) return colsum_parts<bf16>(dh_colsum_part, seg, El, F, dBiasUp, s);
    return colsum<bf16>(dH, F, seg, El, F, dBiasUp, s);
  }
  EpiWgrad<float> epi{static_cast<float*>(dUp), H, F, 0};
  if (int rc = launch_simt<float, true, true>(static_cast<const float*>(Xs), H, static_cast<const float*>(dH), F, geo,
                                              H, epi, s))
    return rc;
  return colsum<float>(dH, F, seg, El, F, dBiasUp, s);
}

int ppmoe_gemm_selftest(int mode, int use_tc, int dtype, const void* A, const void* B, const int* seg, int G, int M,
                        int N, int K, int rows_cap, void* D, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PPMOE_REQUIRE(mode >= 0 && mode <= 2, "mode must be 0..2");
  PPMOE_REQUIRE(use_tc >= 0 && use_tc <= 5,
                "use_tc: 0 CUDA cores, 1 default tcgen05, 2 1-CTA, 3 CTA pair 256x256, 4 CTA pair 256x512, "
                "5 CTA pair 256x128");
  struct ForceGuard {
    explicit ForceGuard(int m, int w, int nr) {
      g_force_mode = m;
      g_force_wide = w;
      g_force_narrow = nr;
      if (nr == 1) g_long_k = 1;
    }
    ~ForceGuard() {
      g_force_mode = 0;
      g_force_wide = -1;
      g_force_narrow = -1;
      g_long_k = 0;
    }
  } guard(use_tc >= 2 ? (use_tc >= 3 ? 2 : 1) : 0, use_tc == 4 ? 1 : (use_tc == 3 || use_tc == 5 ? 0 : -1),
          use_tc == 5 ? 1 : 0);
  PPMOE_REQUIRE(G >= 1 && G <= kMaxGroups, "bad group count %d", G);
  PPMOE_REQUIRE(!use_tc || dtype == kBF16, "tcgen05 path is bf16 only");
  if (mode == 0) {  // D[seg rows x N] = A[seg rows x K] * B_g[K x N] (B MN-major)
    GroupGeom geo = geom(G, N, 0, K, seg, 1, 0, 0, K);
    if (use_tc) {
      CUtensorMap ta, tb;
      if (int rc = tmap_kmajor(&ta, A, K, rows_cap, kBM)) return rc;
      if (int rc = tmap_mnmajor(&tb, B, N, static_cast<uint64_t>(G) * K)) return rc;
      return launch_tc<false, true>(ta, tb, geo, EpiStore<float>{static_cast<float*>(D), N, seg, 1, 0}, s);
    }
    if (dtype == kBF16)
      return launch_simt<bf16, false, true>(static_cast<const bf16*>(A), K, static_cast<const bf16*>(B), N, geo, rows_cap,
                                            EpiStore<float>{static_cast<float*>(D), N, seg, 1, 0}, s);
    return launch_simt<float, false, true>(static_cast<const float*>(A), K, static_cast<const float*>(B), N, geo,
                                           rows_cap, EpiStore<float>{static_cast<float*>(D), N, seg, 1, 0}, s);
  }
  if (mode == 1) {  // D[g][M x N] = A_g^T * B_g with K from segments (both MN-major)
    GroupGeom geo = geom(G, N, M, 0, seg, 1, 0, 1, 0);
    if (use_tc) {
      CUtensorMap ta, tb;
      if (int rc = tmap_mnmajor(&ta, A, M, rows_cap)) return rc;
      if (int rc = tmap_mnmajor(&tb, B, N, rows_cap)) return rc;
      return launch_tc<true, true>(ta, tb, geo, EpiStore<float>{static_cast<float*>(D), N, seg, 0, M}, s);
    }
    if (dtype == kBF16)
      return launch_simt<bf16, true, true>(static_cast<const bf16*>(A), M, static_cast<const bf16*>(B), N, geo, M,
                                           EpiStore<float>{static_cast<float*>(D), N, seg, 0, M}, s);
    return launch_simt<float, true, true>(static_cast<const float*>(A), M, static_cast<const float*>(B), N, geo, M,
                                          EpiStore<float>{static_cast<float*>(D), N, seg, 0, M}, s);
  }
  // mode 2: D[seg rows x N] = A[seg rows x K] * B_g^T, B_g [N x K] K-major
  GroupGeom geo = geom(G, N, 0, K, seg, 1, 0, 0, N);
  if (use_tc) {
    CUtensorMap ta, tb;
    if (int rc = tmap_kmajor(&ta, A, K, rows_cap, kBM)) return rc;
    if (int rc = tmap_kmajor(&tb, B, K, static_cast<uint64_t>(G) * N, b_box_rows())) return rc;
    return launch_tc<false, false>(ta, tb, geo, EpiStore<float>{static_cast<float*>(D), N, seg, 1, 0}, s);
  }
  if (dtype == kBF16)
    return launch_simt<bf16, false, false>(static_cast<const bf16*>(A), K, static_cast<const bf16*>(B), K, geo, rows_cap,
                                           EpiStore<float>{static_cast<float*>(D), N, seg, 1, 0}, s);
  return launch_simt<float, false, false>(static_cast<const float*>(A), K, static_cast<const float*>(B), K, geo,
                                          rows_cap, EpiStore<float>{static_cast<float*>(D), N, seg, 1, 0}, s);
}

}  // extern "C"
