// PPMoE tensor-parallel exchange over NVLink / NVSwitch peer memory.
//
// The reference sums the T ranks' [N x H] partial outputs with one all-reduce per pass
// (reduce_from_tensor_parallel_region, moe.py:307; dX in tp_region backward,
// collectives.py:205-228).  Those partials are sparse by token: token t has at most k
// nonzero contributions, each produced by the rank owning the pair's expert.  So instead
// of a generic all-reduce this file implements the exchange as
//   1. barrier (every rank's expert rows are final),
//   2. owner gather: rank r owns tokens [r N/T, (r+1) N/T) and sums, in slot order, the k
//      expert rows of each owned token straight out of the peers' memory (P2P loads),
//   3. barrier, then every rank pulls the other owners' finished rows (all-gather).
// Deterministic (slot order, no atomics), no fp32 [N x H] accumulator, and the bytes on
// NVLink are k/T-sparse reads plus one all-gather instead of a dense all-reduce.
//
// Peer buffers come from cudaIpc handles exchanged by the host (paper_2304_11414_b200/
// nvlink.py).  Barriers are flag writes with release/acquire at system scope into a
// signal pad on every peer, with a bounded spin (a stuck peer reports an error instead
// of hanging the GPU).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "../../include/ppmoe_capi.h"
#include "common.cuh"
#include "host.h"

namespace ppmoe {

constexpr int kNvlMaxRanks = 8;
constexpr int kNvlChannels = 16;

// The group's peer pointers travel by value in the kernel parameters (no device tables).
template <typename T>
struct PeerSet {
  T* p[kNvlMaxRanks];
};

template <typename T>
static PeerSet<T> peer_set(const void* const* host_ptrs, int n) {
  PeerSet<T> s{};
  for (int i = 0; i < n && host_ptrs; ++i) s.p[i] = static_cast<T*>(const_cast<void*>(host_ptrs[i]));
  return s;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// pads.p[q] = rank q's signal pad ([kNvlChannels][kNvlMaxRanks] uint32, mapped here).
__global__ void nvl_barrier_kernel(const __grid_constant__ PeerSet<uint32_t> pads, int T, int rank, int ch, uint32_t epoch,
                                   int* __restrict__ err, long long timeout_cycles) {
  const int q = threadIdx.x;
  if (q < T) {
    __threadfence_system();  // everything this GPU wrote before the barrier is visible to peers
    st_release_sys(pads.p[q] + ch * kNvlMaxRanks + rank, epoch);
    const uint32_t* mine = pads.p[rank] + ch * kNvlMaxRanks + q;
    const long long t0 = clock64();
    while (static_cast<int>(ld_acquire_sys(mine) - epoch) < 0) {
      if (clock64() - t0 > timeout_cycles) {
        // err is host-mapped pinned memory: a plain store + system fence reaches the host,
        // which raises at its next check (nvlink.NvlArena.check_nonblocking)
        *reinterpret_cast<volatile int*>(err) = 1;
        __threadfence_system();
        break;
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void acc_bf16x8(float (&acc)[8], const uint4& u, float s) {
  const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(hv[i]);
    acc[2 * i] = fmaf(s, f.x, acc[2 * i]);
    acc[2 * i + 1] = fmaf(s, f.y, acc[2 * i + 1]);
  }
}

__device__ __forceinline__ uint4 pack_bf16x8(const float (&a)[8]) {
  uint4 r;
  r.x = pack_bf16x2(a[0], a[1]);
  r.y = pack_bf16x2(a[2], a[3]);
  r.z = pack_bf16x2(a[4], a[5]);
  r.w = pack_bf16x2(a[6], a[7]);
  return r;
}

// Owner gather.  rows.p[q] = rank q's expert-row buffer (Y forward, dX_s backward), local
// row = sorted position - seg[q*El].  Owned tokens [t0, t1), processed in tiles of kOgTile
// tokens: the (source row, weight) of every (token, slot) and the gate-term dL rows are
// resolved once per tile into shared memory, then every thread streams its 8 columns of
// U tokens x K slots with all loads in flight before the first use.  Optional gate term
// (backward): + dl[t - t0, :] . Wg^T, dl = this rank's summed dL rows [t1-t0 x E] fp32,
// Wg [H x E] fp32: EB > 0 holds the thread's 8 columns of Wg in registers (E <= EB);
// EB < 0 is the any-E form that streams Wg per tile (loads amortised over U tokens).
constexpr int kOgTile = 32;
constexpr int kOgMaxE = 128;

__device__ __forceinline__ void multimem_store(__nv_bfloat16* mc, const uint4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void multimem_store(__nv_bfloat16* mc, const uint2& v) {
  asm volatile("multimem.st.relaxed.sys.global.v2.f32 [%0], {%1, %2};" ::"l"(mc), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void multimem_store(__nv_bfloat16* mc, const uint32_t& v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc), "r"(v) : "memory");
}

template <int CW> struct OgVec;
template <> struct OgVec<8> { using type = uint4; };
template <> struct OgVec<4> { using type = uint2; };
template <> struct OgVec<2> { using type = uint32_t; };

template <int CW>
__device__ __forceinline__ void acc_bf16(float (&acc)[CW], const typename OgVec<CW>::type& u, float s) {
  const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < CW / 2; ++i) {
    const float2 f = __bfloat1622float2(hv[i]);
    acc[2 * i] = fmaf(s, f.x, acc[2 * i]);
    acc[2 * i + 1] = fmaf(s, f.y, acc[2 * i + 1]);
  }
}

// One CTA per tile of kOgTile owned tokens x (256*CW) columns.  CW columns per thread.
// Register budgets: 4 CTAs per SM where the accumulators fit in 64 registers (more row loads
// in flight per SM: C2 backward with the gate term 128 -> 92 us, forward 79 -> 73 us), else 3;
// the grid is sized to the resident CTAs (occupancy API), so the grid-stride tile loop has
// no second partial wave.
template <int EB, int U, int KT, int CW>  // KT = k (1, 2) or 0: any k <= 8 read at run time
__global__ void __launch_bounds__(256, EB > 8 ? 3
                                           : EB == 8 ? (U * CW <= 16 ? 4 : 3)
                                           : EB == 0 ? (U * CW <= 32 ? 4 : 3)
                                                     : 1)
    nvl_owner_gather_kernel(const __grid_constant__ PeerSet<const __nv_bfloat16> rows, const int* __restrict__ seg,
                            int El, const int* __restrict__ idx, const int* __restrict__ pair_pos,
                            const float* __restrict__ w, int Kr, int H, int t0, int t1,
                            const float* __restrict__ dl, const float* __restrict__ Wg, int E,
                            __nv_bfloat16* __restrict__ out, __nv_bfloat16* __restrict__ out_sym,
                            const __grid_constant__ PeerSet<__nv_bfloat16> push, int T, int sym_mc) {
  using V = typename OgVec<CW>::type;
  constexpr int KS = KT > 0 ? KT : 8;
  constexpr int DLW = EB > 0 ? EB : (EB < 0 ? kOgMaxE : 1);
  const int K = KT > 0 ? KT : Kr;
  __shared__ const __nv_bfloat16* src[kOgTile][KS];
  __shared__ float sw[kOgTile][KS];
  __shared__ __align__(16) float sdl[kOgTile][DLW];
  const int j = (blockIdx.y * blockDim.x + threadIdx.x) * CW;
  const bool active = j < H;
  // gate-term form: this CTA's Wg columns in shared memory, [e][thread][c] so each thread
  // reads its CW columns of one expert as 16-byte vectors, conflict-free across the warp
  // (in registers they cost 32 per thread and halved the resident CTAs, which left too
  // few row loads in flight for HBM)
  // E <= 8: 32 KB static; 8 < E <= 32: 64 KB of dynamic shared memory (E 16: 4 columns per
  // thread, E 32: 2), staged once per CTA, so the gate term never re-reads Wg from L2
  static_assert(EB <= 0 || CW % 2 == 0, "vector Wg reads need CW % 2 == 0");
  constexpr bool kDynWg = EB > 8;
  __shared__ __align__(16) float swg_s[(EB > 0 && !kDynWg) ? CW * EB * 256 : 4];
  extern __shared__ __align__(16) float swg_d[];
  float* swg = kDynWg ? swg_d : swg_s;
  if constexpr (EB > 0) {
    for (int i = threadIdx.x; i < CW * EB * 256; i += blockDim.x) {
      const int c = i % CW, t = (i / CW) % 256, e = i / (CW * 256);
      const int jj = (blockIdx.y * 256 + t) * CW + c;
      swg[i] = (jj < H && e < E) ? Wg[static_cast<size_t>(jj) * E + e] : 0.f;
    }
  }
  for (int tb = t0 + blockIdx.x * kOgTile; tb < t1; tb += gridDim.x * kOgTile) {
    const int nt = min(kOgTile, t1 - tb);
    __syncthreads();  // previous tile's shared entries are consumed
    for (int i = threadIdx.x; i < kOgTile * KS; i += blockDim.x) {
      const int u = i / KS, s = i % KS;
      const __nv_bfloat16* p_src = nullptr;
      float ws = 0.f;
      if (u < nt && s < K) {
        const size_t pi = static_cast<size_t>(tb + u) * K + s;
        const int p = pair_pos[pi];
        if (p >= 0) {
          const int q = idx[pi] / El;
          p_src = rows.p[q] + static_cast<size_t>(p - seg[q * El]) * H;
          ws = w ? w[pi] : 1.f;
        }
      }
      src[u][s] = p_src;
      sw[u][s] = ws;
    }
    if constexpr (EB != 0) {
      constexpr int W = EB > 0 ? EB : 1;
      const int ew = EB > 0 ? W : E;  // register form reads all EB columns: zero-fill past E
      for (int i = threadIdx.x; i < kOgTile * ew; i += blockDim.x) {
        const int u = i / ew, e = i % ew;
        sdl[u][e] = (u < nt && e < E) ? dl[static_cast<size_t>(tb - t0 + u) * E + e] : 0.f;
      }
    }
    __syncthreads();
    if (!active) continue;
    for (int u0 = 0; u0 < nt; u0 += U) {
      V v[U][KS];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          const __nv_bfloat16* p = (s < K && u0 + u < nt) ? src[u0 + u][s] : nullptr;
          if (p) v[u][s] = *reinterpret_cast<const V*>(p + j);
          else memset(&v[u][s], 0, sizeof(V));
        }
      float acc[U][CW];
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int c = 0; c < CW; ++c) acc[u][c] = 0.f;
#pragma unroll
        for (int s = 0; s < KS; ++s)
          if (s < K) acc_bf16<CW>(acc[u], v[u][s], sw[min(u0 + u, kOgTile - 1)][s]);
      }
      if constexpr (EB > 0) {
        static_assert(EB % 4 == 0, "vector dL reads need EB % 4 == 0");
#pragma unroll
        for (int e4 = 0; e4 < EB; e4 += 4) {
          float4 d[U];
#pragma unroll
          for (int u = 0; u < U; ++u) d[u] = *reinterpret_cast<const float4*>(&sdl[min(u0 + u, kOgTile - 1)][e4]);
#pragma unroll
          for (int ee = 0; ee < 4; ++ee) {
            float wv[CW];
            if constexpr (CW % 4 == 0) {
#pragma unroll
              for (int c4 = 0; c4 < CW; c4 += 4)
                *reinterpret_cast<float4*>(&wv[c4]) =
                    *reinterpret_cast<const float4*>(&swg[((e4 + ee) * 256 + threadIdx.x) * CW + c4]);
            } else {
#pragma unroll
              for (int c2 = 0; c2 < CW; c2 += 2)
                *reinterpret_cast<float2*>(&wv[c2]) =
                    *reinterpret_cast<const float2*>(&swg[((e4 + ee) * 256 + threadIdx.x) * CW + c2]);
            }
#pragma unroll
            for (int c = 0; c < CW; c += 2)  // paired columns: FFMA2, half the FMA issue slots
#pragma unroll
              for (int u = 0; u < U; ++u) {
                const float dv = ee == 0 ? d[u].x : ee == 1 ? d[u].y : ee == 2 ? d[u].z : d[u].w;
                const float2 r = __ffma2_rn(make_float2(dv, dv), make_float2(wv[c], wv[c + 1]),
                                            make_float2(acc[u][c], acc[u][c + 1]));
                acc[u][c] = r.x;
                acc[u][c + 1] = r.y;
              }
          }
        }
      } else if constexpr (EB < 0) {
        for (int e = 0; e < E; ++e) {
          float wc[CW];
#pragma unroll
          for (int c = 0; c < CW; ++c) wc[c] = Wg[static_cast<size_t>(j + c) * E + e];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const float d = sdl[min(u0 + u, kOgTile - 1)][e];
#pragma unroll
            for (int c = 0; c < CW; ++c) acc[u][c] = fmaf(d, wc[c], acc[u][c]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u0 + u >= nt) break;
        V o;
        uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
        for (int i = 0; i < CW / 2; ++i) ow[i] = pack_bf16x2(acc[u][2 * i], acc[u][2 * i + 1]);
        const size_t off = static_cast<size_t>(tb + u0 + u) * H + j;
        *reinterpret_cast<V*>(out + off) = o;
        if (push.p[0]) {  // the owned row straight into every rank's exchange buffer (P2P stores)
          for (int q = 0; q < T; ++q) *reinterpret_cast<V*>(push.p[q] + off) = o;
        } else if (out_sym && sym_mc) {  // NVLS multicast: one store lands in every rank's buffer
          multimem_store(out_sym + off, o);
        } else if (out_sym) {
          *reinterpret_cast<V*>(out_sym + off) = o;
        }
      }
    }
  }
}

// Sum over the T ranks (rank order) of rows [t0, t1) of a [N x C] fp32 buffer (the partial
// gate-logit gradients dL): out [t1-t0 x C].
__global__ void nvl_sum_rows_kernel(const __grid_constant__ PeerSet<const float> srcs, int T, int C, int t0, int t1,
                                    float* __restrict__ out) {
  const size_t n = static_cast<size_t>(t1 - t0) * C;
  const size_t base = static_cast<size_t>(t0) * C;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float acc = 0.f;
    for (int q = 0; q < T; ++q) acc += srcs.p[q][base + i];
    out[i] = acc;
  }
}

// Owned rows of the fp32 owner accumulator -> bf16 (local output and the peer-visible
// exchange copy), zeroing the accumulator for the next pass.  rows x H, H % 4 == 0.
__global__ void nvl_cast_owned_kernel(float* __restrict__ acc, size_t n4, __nv_bfloat16* __restrict__ out,
                                      __nv_bfloat16* __restrict__ xch) {
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float4* a = reinterpret_cast<float4*>(acc) + i;
    const float4 v = *a;
    *a = make_float4(0.f, 0.f, 0.f, 0.f);
    uint2 o;
    o.x = pack_bf16x2(v.x, v.y);
    o.y = pack_bf16x2(v.z, v.w);
    reinterpret_cast<uint2*>(out)[i] = o;
    if (xch) reinterpret_cast<uint2*>(xch)[i] = o;
  }
}

// Owner-slot sum: out[t] = sum over valid slots s (pair_pos[t,s] >= 0) of slots[t-t0][s],
// for the owned tokens [t0, t0+rows); writes the local output rows and the exchange copy.
__global__ void nvl_sum_slots_kernel(const __nv_bfloat16* __restrict__ slots, int rows, int K, int H, int t0,
                                     const int* __restrict__ pair_pos, __nv_bfloat16* __restrict__ out,
                                     __nv_bfloat16* __restrict__ xch) {
  const int hv = H / 8;
  const size_t n = static_cast<size_t>(rows) * hv;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / hv), c = static_cast<int>(i % hv) * 8;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int sl = 0; sl < K; ++sl) {
      if (pair_pos[static_cast<size_t>(t0 + r) * K + sl] < 0) continue;
      const uint4 u = *reinterpret_cast<const uint4*>(slots + (static_cast<size_t>(r) * K + sl) * H + c);
      acc_bf16x8(acc, u, 1.f);
    }
    const uint4 o = pack_bf16x8(acc);
    *reinterpret_cast<uint4*>(out + static_cast<size_t>(r) * H + c) = o;
    *reinterpret_cast<uint4*>(xch + static_cast<size_t>(r) * H + c) = o;
  }
}

// All-gather (pull): out rows of every other owner's block, read from its out_sym.
__global__ void __launch_bounds__(256)
    nvl_pull_blocks_kernel(const __grid_constant__ PeerSet<const __nv_bfloat16> srcs, int T, int rank, int N, int H,
                           __nv_bfloat16* __restrict__ out) {
  const size_t row_vecs = static_cast<size_t>(H) / 8;
  for (int q0 = 1; q0 < T; ++q0) {
    const int q = (rank + q0) % T;  // stagger the sources across ranks
    const size_t lo = static_cast<size_t>(q) * N / T, hi = static_cast<size_t>(q + 1) * N / T;
    const uint4* src = reinterpret_cast<const uint4*>(srcs.p[q]) + lo * row_vecs;
    uint4* dst = reinterpret_cast<uint4*>(out) + lo * row_vecs;
    const size_t n = (hi - lo) * row_vecs;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
      const uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
      dst[i] = a;
      dst[i + stride] = b;
      dst[i + 2 * stride] = c;
      dst[i + 3 * stride] = d;
    }
    for (; i < n; i += stride) dst[i] = src[i];
  }
}

// Owner-gather CTAs per SM (PPMOE_OG_CTAS).  5 = full residency of the 48-register forms
// (ncu, C2: forward 65 -> 60 us, gate-term backward 97 -> 89 us against 4; 6 overshoots).
static int og_ctas_per_sm() {  // PPMOE_OG_CTAS overrides the grid's CTAs per SM (A/B runs)
  static int v = [] { const char* e = getenv("PPMOE_OG_CTAS"); return e ? atoi(e) : 0; }();
  return v;
}
static int og16_u() {  // tokens per thread of the 8 < E <= 16 gate-term form (PPMOE_OG16_U: 4 or 8)
  static int v = [] { const char* e = getenv("PPMOE_OG16_U"); return e ? atoi(e) : 4; }();
  return v;
}
static int og8_u() {  // tokens per thread of the E <= 8 gate-term form (PPMOE_OG8_U: 4 or 8)
  static int v = [] { const char* e = getenv("PPMOE_OG8_U"); return e ? atoi(e) : 4; }();
  return v;
}
static bool og_wide_e() {  // PPMOE_OG_WIDE_E=0: the any-E form (Wg from L2) for A/B runs
  static bool v = [] { const char* e = getenv("PPMOE_OG_WIDE_E"); return !e || atoi(e) != 0; }();
  return v;
}
static int og_fwd_cw() {
  static int v = [] { const char* e = getenv("PPMOE_OG_FWD_CW"); return e ? atoi(e) : 4; }();
  return v;
}

}  // namespace ppmoe

using namespace ppmoe;

extern "C" {

size_t ppmoe_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

int ppmoe_ipc_alloc(size_t bytes, void** ptr, void* handle) {
  PPMOE_REQUIRE(ptr && handle && bytes > 0, "bad ipc_alloc arguments");
  PPMOE_CUDA(cudaMalloc(ptr, bytes));
  PPMOE_CUDA(cudaMemset(*ptr, 0, bytes));
  PPMOE_CUDA(cudaDeviceSynchronize());
  PPMOE_CUDA(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(handle), *ptr));
  return kOk;
}

int ppmoe_ipc_open(const void* handle, void** ptr) {
  PPMOE_REQUIRE(ptr && handle, "bad ipc_open arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  PPMOE_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return kOk;
}

int ppmoe_ipc_close(void* ptr) {
  PPMOE_CUDA(cudaIpcCloseMemHandle(ptr));
  return kOk;
}

int ppmoe_ipc_free(void* ptr) {
  PPMOE_CUDA(cudaFree(ptr));
  return kOk;
}

size_t ppmoe_nvl_pad_bytes(void) { return sizeof(uint32_t) * kNvlChannels * kNvlMaxRanks; }

int ppmoe_nvl_barrier(void* const* pads, int T, int rank, int ch, unsigned int epoch, int* err,
                      long long timeout_cycles, void* stream) {
  PPMOE_REQUIRE(T >= 1 && T <= kNvlMaxRanks && rank >= 0 && rank < T, "bad barrier group T=%d rank=%d", T, rank);
  PPMOE_REQUIRE(ch >= 0 && ch < kNvlChannels, "barrier channel %d out of range", ch);
  nvl_barrier_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      peer_set<uint32_t>(pads, T), T, rank, ch, static_cast<uint32_t>(epoch), err, timeout_cycles);
  return check_launch("nvl_barrier_kernel");
}

int ppmoe_nvl_owner_gather(const void* const* rows, const int* seg, int El, const int* idx, const int* pair_pos,
                           const float* w, int N, int K, int H, int T, int rank, const float* dl, const float* Wg,
                           int E, void* out, void* out_sym, void* const* push, int sym_mc, void* stream) {
  PPMOE_REQUIRE(T >= 1 && T <= kNvlMaxRanks && rank >= 0 && rank < T, "bad group T=%d rank=%d", T, rank);
  PPMOE_REQUIRE(K >= 1 && K <= 8 && H % 8 == 0 && El >= 1, "owner gather needs 1 <= k <= 8 and hidden %% 8 == 0");
  PPMOE_REQUIRE(!sym_mc || (out_sym && !push), "multicast output needs out_sym and no push set");
  PPMOE_REQUIRE(N / T < (1 << 30), "too many tokens");
  PPMOE_REQUIRE(!dl || (Wg && E >= 1 && E <= kOgMaxE), "the gate term supports 1 <= E <= %d", kOgMaxE);
  const int t0 = static_cast<int>(static_cast<long long>(rank) * N / T);
  const int t1 = static_cast<int>(static_cast<long long>(rank + 1) * N / T);
  if (t1 <= t0) return kOk;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int tiles = (t1 - t0 + kOgTile - 1) / kOgTile;
  const auto R = peer_set<const __nv_bfloat16>(rows, T);
  auto O = static_cast<__nv_bfloat16*>(out);
  auto OS = static_cast<__nv_bfloat16*>(out_sym);
  const auto P = peer_set<__nv_bfloat16>(push, push ? T : 0);
  // persistent-ish grid over the tiles; the gate-term forms use 4 columns per thread to keep
  // Wg in registers at 3+ CTAs per SM
#define PPMOE_OG(EB, U, KT, CW)                                                                            \
  do {                                                                                                     \
    const int gy_ = (H / CW + 255) / 256;                                                                  \
    static const int occ_ = [] {                                                                           \
      int b = 0;                                                                                           \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, nvl_owner_gather_kernel<EB, U, KT, CW>, 256, 0);   \
      return b > 0 ? b : 1;                                                                                \
    }();                                                                                                   \
    const int per_sm_ = og_ctas_per_sm() > 0 ? og_ctas_per_sm() : occ_;                                    \
    nvl_owner_gather_kernel<EB, U, KT, CW><<<dim3(max(1, min(tiles, num_sms() * per_sm_ / gy_)), gy_), 256, 0, s>>>( \
        R, seg, El, idx, pair_pos, w, K, H, t0, t1, dl, Wg, E, O, OS, P, T, sym_mc);                       \
  } while (0)
  // 8 < E <= 32: Wg columns in 64 KB of dynamic shared memory, 3 CTAs per SM
#define PPMOE_OG_DYN(EB, U, KT, CW)                                                                        \
  do {                                                                                                     \
    auto kern_ = nvl_owner_gather_kernel<EB, U, KT, CW>;                                                   \
    constexpr int smem_ = CW * EB * 256 * 4;                                                               \
    PPMOE_CUDA(cudaFuncSetAttribute(kern_, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_));           \
    const int gy_ = (H / CW + 255) / 256;                                                                  \
    static const int occ_ = [&] {                                                                          \
      int b = 0;                                                                                           \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern_, 256, smem_);                                \
      return b > 0 ? b : 1;                                                                                \
    }();                                                                                                   \
    kern_<<<dim3(max(1, min(tiles, num_sms() * occ_ / gy_)), gy_), 256, smem_, s>>>(                       \
        R, seg, El, idx, pair_pos, w, K, H, t0, t1, dl, Wg, E, O, OS, P, T, sym_mc);                       \
  } while (0)
  if (!dl) {
    if (K == 2 && og_fwd_cw() == 4) PPMOE_OG(0, 8, 2, 4);
    else if (K == 2) PPMOE_OG(0, 4, 2, 8);
    else if (K == 1) PPMOE_OG(0, 8, 1, 8);
    else PPMOE_OG(0, 1, 0, 8);
  } else if (E <= 8) {
    if (K == 2 && og8_u() == 8) PPMOE_OG(8, 8, 2, 4);
    else if (K == 2) PPMOE_OG(8, 4, 2, 4);
    else if (K == 1) PPMOE_OG(8, 8, 1, 4);
    else PPMOE_OG(8, 1, 0, 4);
  } else if (E <= 16 && og_wide_e()) {
    if (K == 2 && og16_u() == 4) PPMOE_OG_DYN(16, 4, 2, 4);  // (8 tokens x 2 columns: 425 vs 230 us at C3)
    else if (K == 2) PPMOE_OG_DYN(16, 8, 2, 4);
    else if (K == 1) PPMOE_OG_DYN(16, 8, 1, 4);
    else PPMOE_OG_DYN(16, 1, 0, 4);
  } else if (E <= 32 && og_wide_e()) {
    if (K == 2) PPMOE_OG_DYN(32, 8, 2, 2);
    else if (K == 1) PPMOE_OG_DYN(32, 8, 1, 2);
    else PPMOE_OG_DYN(32, 2, 0, 2);
  } else {
    if (K == 2) PPMOE_OG(-1, 4, 2, 4);
    else PPMOE_OG(-1, 2, 0, 4);
  }
#undef PPMOE_OG
#undef PPMOE_OG_DYN
  return check_launch("nvl_owner_gather_kernel");
}

// Sliced routing over peer memory: rank q's record (its N/T tokens) is [stats 4E | idx nr*K |
// w nr*K | scores nr*E] 32-bit words; every rank copies all T records into its full routing
// tensors (rows q*nr ..) and the per-rank stats table.
__global__ void nvl_route_gather_kernel(const __grid_constant__ PeerSet<const uint32_t> recs, int T, int nr, int K,
                                        int E, uint32_t* __restrict__ idx, uint32_t* __restrict__ w,
                                        uint32_t* __restrict__ scores, uint32_t* __restrict__ stats) {
  const size_t ns = 4 * static_cast<size_t>(E), ni = static_cast<size_t>(nr) * K, nsc = static_cast<size_t>(nr) * E;
  const size_t rec = ns + 2 * ni + nsc;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < T * rec;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int q = static_cast<int>(i / rec);
    size_t o = i - q * rec;
    const uint32_t v = recs.p[q][o];
    if (o < ns) {
      stats[q * ns + o] = v;
    } else if ((o -= ns) < ni) {
      idx[q * ni + o] = v;
    } else if ((o -= ni) < ni) {
      w[q * ni + o] = v;
    } else {
      scores[q * nsc + (o - ni)] = v;
    }
  }
}

int ppmoe_nvl_route_gather(const void* const* recs, int T, int nr, int K, int E, int* idx, float* w, float* scores,
                           int* stats, void* stream) {
  PPMOE_REQUIRE(T >= 1 && T <= kNvlMaxRanks && nr >= 0 && K >= 1 && E >= 1, "bad route_gather arguments");
  const size_t words = static_cast<size_t>(T) * (4 * static_cast<size_t>(E) + static_cast<size_t>(nr) * (2 * K + E));
  const int grid = static_cast<int>(std::min<size_t>((words + 255) / 256, static_cast<size_t>(num_sms()) * 4));
  nvl_route_gather_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      peer_set<const uint32_t>(recs, T), T, nr, K, E, reinterpret_cast<uint32_t*>(idx), reinterpret_cast<uint32_t*>(w),
      reinterpret_cast<uint32_t*>(scores), reinterpret_cast<uint32_t*>(stats));
  return check_launch("nvl_route_gather_kernel");
}

int ppmoe_nvl_sum_all(const void* const* srcs, int T, int count, float* out, void* stream) {
  PPMOE_REQUIRE(T >= 1 && T <= kNvlMaxRanks && count >= 0, "bad sum_all arguments");
  if (count == 0) return kOk;
  const int grid = std::min((count + 255) / 256, num_sms() * 4);
  nvl_sum_rows_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(peer_set<const float>(srcs, T), T, count, 0,
                                                                            1, out);
  return check_launch("nvl_sum_rows_kernel");
}

int ppmoe_nvl_sum_rows(const void* const* srcs, int T, int rank, int N, int C, float* out, void* stream) {
  PPMOE_REQUIRE(T >= 1 && T <= kNvlMaxRanks && rank >= 0 && rank < T && C >= 1, "bad sum_rows arguments");
  const int t0 = static_cast<int>(static_cast<long long>(rank) * N / T);
  const int t1 = static_cast<int>(static_cast<long long>(rank + 1) * N / T);
  if (t1 <= t0) return kOk;
  const size_t n = static_cast<size_t>(t1 - t0) * C;
  const int grid = static_cast<int>(std::min<size_t>((n + 255) / 256, static_cast<size_t>(num_sms()) * 4));
  nvl_sum_rows_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(peer_set<const float>(srcs, T), T, C, t0,
                                                                            t1, out);
  return check_launch("nvl_sum_rows_kernel");
}

int ppmoe_nvl_pull_blocks(const void* const* srcs, int T, int rank, int N, int H, void* out, void* stream) {
  PPMOE_REQUIRE(T >= 1 && T <= kNvlMaxRanks && rank >= 0 && rank < T, "bad group T=%d rank=%d", T, rank);
  PPMOE_REQUIRE(H % 8 == 0, "pull needs hidden %% 8 == 0");
  if (T == 1 || N == 0) return kOk;
  nvl_pull_blocks_kernel<<<num_sms() * 4, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      peer_set<const __nv_bfloat16>(srcs, T), T, rank, N, H, static_cast<__nv_bfloat16*>(out));
  return check_launch("nvl_pull_blocks_kernel");
}

int ppmoe_nvl_cast_owned(float* acc, int rows, int H, void* out_rows, void* xch_rows, void* stream) {
  PPMOE_REQUIRE(rows >= 0 && H % 4 == 0, "cast_owned needs hidden %% 4 == 0");
  const size_t n4 = static_cast<size_t>(rows) * H / 4;
  if (n4 == 0) return kOk;
  const int grid = static_cast<int>(std::min<size_t>((n4 + 255) / 256, static_cast<size_t>(num_sms()) * 8));
  nvl_cast_owned_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      acc, n4, static_cast<__nv_bfloat16*>(out_rows), static_cast<__nv_bfloat16*>(xch_rows));
  return check_launch("nvl_cast_owned_kernel");
}

int ppmoe_nvl_sum_slots(const void* slots, int rows, int K, int H, int t0, const int* pair_pos, void* out_rows,
                        void* xch_rows, void* stream) {
  PPMOE_REQUIRE(rows >= 0 && K >= 1 && K <= 8 && H % 8 == 0, "bad sum_slots arguments");
  const size_t n = static_cast<size_t>(rows) * (H / 8);
  if (n == 0) return kOk;
  const int grid = static_cast<int>(std::min<size_t>((n + 255) / 256, static_cast<size_t>(num_sms()) * 8));
  nvl_sum_slots_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(slots), rows, K, H, t0, pair_pos, static_cast<__nv_bfloat16*>(out_rows),
      static_cast<__nv_bfloat16*>(xch_rows));
  return check_launch("nvl_sum_slots_kernel");
}

int ppmoe_nvl_pull_range_ce(const void* const* srcs, int T, int rank, int N, int H, int q_lo, int q_hi, void* out,
                            void* stream) {
  PPMOE_REQUIRE(T >= 1 && T <= kNvlMaxRanks && rank >= 0 && rank < T, "bad group T=%d rank=%d", T, rank);
  PPMOE_REQUIRE(0 <= q_lo && q_lo <= q_hi && q_hi <= T, "bad owner range [%d, %d)", q_lo, q_hi);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t row = static_cast<size_t>(H) * 2;
  for (int q = q_lo; q < q_hi; ++q) {
    if (q == rank) continue;
    const size_t lo = static_cast<size_t>(q) * N / T, hi = static_cast<size_t>(q + 1) * N / T;
    if (hi > lo)
      PPMOE_CUDA(cudaMemcpyAsync(static_cast<char*>(out) + lo * row, static_cast<const char*>(srcs[q]) + lo * row,
                                 (hi - lo) * row, cudaMemcpyDeviceToDevice, s));
  }
  return kOk;
}

int ppmoe_nvl_pull_blocks_ce(const void* const* srcs, int T, int rank, int N, int H, void* out, void* stream) {
  PPMOE_REQUIRE(T >= 1 && T <= kNvlMaxRanks && rank >= 0 && rank < T, "bad group T=%d rank=%d", T, rank);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t row = static_cast<size_t>(H) * 2;
  // One copy-engine transfer per peer block, each on its own stream so the T-1 transfers
  // run concurrently on different copy engines (forked from / joined back to `stream`).
  static thread_local cudaStream_t side[kNvlMaxRanks] = {};
  static thread_local cudaEvent_t fork = nullptr, join[kNvlMaxRanks] = {};
  static thread_local int dev_of = -1;
  int dev = 0;
  PPMOE_CUDA(cudaGetDevice(&dev));
  if (dev_of != dev) {
    for (int i = 0; i < kNvlMaxRanks; ++i) {
      PPMOE_CUDA(cudaStreamCreateWithFlags(&side[i], cudaStreamNonBlocking));
      PPMOE_CUDA(cudaEventCreateWithFlags(&join[i], cudaEventDisableTiming));
    }
    PPMOE_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    dev_of = dev;
  }
  const char* ser = getenv("PPMOE_CE_SERIAL");
  const bool split = !(ser && ser[0] == '1');
  if (split) PPMOE_CUDA(cudaEventRecord(fork, s));
  for (int q0 = 1; q0 < T; ++q0) {
    const int q = (rank + q0) % T;  // staggered sources
    const size_t lo = static_cast<size_t>(q) * N / T, hi = static_cast<size_t>(q + 1) * N / T;
    if (hi <= lo) continue;
    cudaStream_t cs = split ? side[q0] : s;
    if (split) PPMOE_CUDA(cudaStreamWaitEvent(cs, fork, 0));
    PPMOE_CUDA(cudaMemcpyAsync(static_cast<char*>(out) + lo * row, static_cast<const char*>(srcs[q]) + lo * row,
                               (hi - lo) * row, cudaMemcpyDeviceToDevice, cs));
    if (split) {
      PPMOE_CUDA(cudaEventRecord(join[q0], cs));
      PPMOE_CUDA(cudaStreamWaitEvent(s, join[q0], 0));
    }
  }
  return kOk;
}

}  // extern "C"
