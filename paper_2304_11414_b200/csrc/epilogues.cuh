// Epilogue functors for the grouped expert GEMMs.  Each is applied to one row
// (`m` within expert `g`; `row` = its local position in the padded dispatch buffer
// for token-segment outputs) and W consecutive output columns starting at `n0`,
// with the fp32 accumulator values `v` read straight from TMEM (or registers in
// the CUDA-core path).
#pragma once

#include <type_traits>

#include "common.cuh"

namespace ppmoe {

// `cs`: 2 = 32-byte stores, 1 = 16-byte stores with the streaming (evict-first) cache
// policy, 0 = plain 16-byte stores (default: measured fastest in the C2 step).
template <typename T, int W>
__device__ __forceinline__ void store_row(T* p, const float (&x)[W], int valid, int cs = 0) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (cs == 2 && valid >= W && (W % 16 == 0) && (reinterpret_cast<uintptr_t>(p) & 31) == 0) {
      // 32-byte stores: every lane writes whole L2 sectors (the lanes of a warp hold
      // different rows, so 16-byte stores left each sector half written per instruction)
#pragma unroll
      for (int j = 0; j < W; j += 16) {
        uint32_t u[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) u[i] = pack_bf16x2(x[j + 2 * i], x[j + 2 * i + 1]);
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p + j), "r"(u[0]), "r"(u[1]),
                     "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7])
                     : "memory");
      }
      return;
    }
    if (valid >= W && (W % 8 == 0) && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int j = 0; j < W; j += 8) {
        uint4 u;
        u.x = pack_bf16x2(x[j], x[j + 1]);
        u.y = pack_bf16x2(x[j + 2], x[j + 3]);
        u.z = pack_bf16x2(x[j + 4], x[j + 5]);
        u.w = pack_bf16x2(x[j + 6], x[j + 7]);
        if (cs == 1) st_cs_v4(p + j, u);
        else *reinterpret_cast<uint4*>(p + j) = u;
      }
      return;
    }
    if (valid >= W && (W % 4 == 0) && (reinterpret_cast<uintptr_t>(p) & 7) == 0) {
#pragma unroll
      for (int j = 0; j < W; j += 4) {
        uint2 u;
        u.x = pack_bf16x2(x[j], x[j + 1]);
        u.y = pack_bf16x2(x[j + 2], x[j + 3]);
        *reinterpret_cast<uint2*>(p + j) = u;
      }
      return;
    }
  } else {
    if (valid >= W && (W % 4 == 0) && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int j = 0; j < W; j += 4) *reinterpret_cast<float4*>(p + j) = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < W; ++j)
    if (j < valid) p[j] = from_f32<T>(x[j]);
}

template <typename T, int W>
__device__ __forceinline__ void load_row(const T* p, float (&x)[W], int valid) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (valid >= W && (W % 8 == 0) && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int j = 0; j < W; j += 8) {
        uint4 u = *reinterpret_cast<const uint4*>(p + j);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float2 f = __bfloat1622float2(h[i]);
          x[j + 2 * i] = f.x;
          x[j + 2 * i + 1] = f.y;
        }
      }
      return;
    }
  } else {
    if (valid >= W && (W % 4 == 0) && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int j = 0; j < W; j += 4) {
        float4 f = *reinterpret_cast<const float4*>(p + j);
        x[j] = f.x;
        x[j + 1] = f.y;
        x[j + 2] = f.z;
        x[j + 3] = f.w;
      }
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < W; ++j) x[j] = j < valid ? to_f32(p[j]) : 0.f;
}

template <int W>
__device__ __forceinline__ void scatter_add_row(float* p, const float (&x)[W], float s, int valid) {
  if (valid >= W && (W % 4 == 0) && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
    for (int j = 0; j < W; j += 4) red_add_v4(p + j, s * x[j], s * x[j + 1], s * x[j + 2], s * x[j + 3]);
    return;
  }
#pragma unroll
  for (int j = 0; j < W; ++j)
    if (j < valid) atomicAdd(p + j, s * x[j]);
}

// Warp-cooperative row store through a per-warp shared-memory staging area (32 rows x
// kStageStride bytes).  The tcgen05 epilogue holds one output row per lane, so a plain
// store instruction touches 32 rows; staging turns each 32-column chunk into four
// instructions of 8 rows x 64 contiguous bytes (4x fewer L1 store wavefronts).  Every lane
// of the warp must call it (convergent); `p` = this lane's destination or null.
__device__ __forceinline__ void stage_store32(uint8_t* buf, __nv_bfloat16* p, const float (&x)[32], int valid) {
  const int lane = threadIdx.x & 31;
  if (valid < 32) {  // ragged last chunk of a row (N % 32 != 0): direct stores
    if (p) store_row<__nv_bfloat16, 32>(p, x, valid);
    return;
  }
  uint4* mine = reinterpret_cast<uint4*>(buf + lane * kStageStride);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint4 u;
    u.x = pack_bf16x2(x[8 * j], x[8 * j + 1]);
    u.y = pack_bf16x2(x[8 * j + 2], x[8 * j + 3]);
    u.z = pack_bf16x2(x[8 * j + 4], x[8 * j + 5]);
    u.w = pack_bf16x2(x[8 * j + 6], x[8 * j + 7]);
    mine[j] = u;
  }
  const unsigned long long pp = reinterpret_cast<unsigned long long>(p);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = 8 * i + (lane >> 2), seg = lane & 3;
    const unsigned long long q = __shfl_sync(0xffffffffu, pp, r);
    const uint4 u = *reinterpret_cast<const uint4*>(buf + r * kStageStride + seg * 16);
    if (q) *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(q) + seg * 8) = u;
  }
  __syncwarp();
}

// fc1 forward: a = X_e * up_e + bias_up ; Act = GeLU(a), and GeLU'(a) saved for the
// backward so the fc2 data-gradient epilogue is a plain multiply (moe.py:101-104,
// tensor.py:199-207).
template <typename T>
struct EpiFc1Fwd {
  T* gelu_grad;
  T* act;
  const T* bias;  // [G*F] or null
  int F;
  const int* seg;
  int cs;
  template <int W>
  __device__ __forceinline__ void apply(int g, int m, int row, int n0, const float (&v)[W]) const {
    const int valid = min(W, F - n0);
    float b[W];
    if (bias) load_row<T, W>(bias + static_cast<size_t>(g) * F + n0, b, valid);
    else
#pragma unroll
      for (int j = 0; j < W; ++j) b[j] = 0.f;
    float d[W], a[W];
    static_assert(W % 2 == 0, "paired GeLU");
#ifdef PPMOE_GELU_SCALAR  // dev A/B: the one-element-at-a-time form
#pragma unroll
    for (int j = 0; j < W; ++j) gelu_and_grad(v[j] + b[j], a[j], d[j]);
#else
#pragma unroll
    for (int j = 0; j < W; j += 2) {
      float2 aa, dd;
      gelu_and_grad2(__fadd2_rn(make_float2(v[j], v[j + 1]), make_float2(b[j], b[j + 1])), aa, dd);
      a[j] = aa.x;
      a[j + 1] = aa.y;
      d[j] = dd.x;
      d[j + 1] = dd.y;
    }
#endif
    const size_t off = static_cast<size_t>(row) * F + n0;
    store_row<T, W>(gelu_grad + off, d, valid, cs);
    store_row<T, W>(act + off, a, valid, cs);
  }
};

// fc2 forward + combine: Y = Act * down_e + bias_down (saved pre-scale for the
// backward), out[tok] += w * Y  (moe.py:104-107 + scale_rows + index_assign,
// tensor.py:184-196, 244-272; top-k contributions summed).
template <typename T>
struct EpiFc2Fwd {
  T* y;
  T* y2;          // optional second copy of Y (peer-visible buffer of the NVLink exchange)
  const T* bias;  // [G*H] or null
  int H;
  const int* seg;
  const int* tok;  // [rows] local token id per row, -1 for padding
  const float* w;  // [rows] gate weight per row
  int weight_scaling;
  float* out_acc;  // [N*H] fp32, zero-initialised
  int cs;
  float drop_p;             // inverted dropout on the expert output (tensor.py:315-330)
  const unsigned long long* drop;  // the reference's Philox dropout stream (common.cuh), or null
  // Owner mode (NVLink exchange): the weighted row goes straight into the fp32 accumulator
  // of the rank owning the token (owner_acc = device table of T peer pointers, each
  // [owner_rows x H]), over NVLink, tile by tile while the GEMM runs.
  float* const* owner_acc;
  int owner_rows;
  // Owner-slot mode: w*Y (bf16) stored into slot s of the owning rank's [owner_rows x K x H]
  // buffer with plain P2P stores (slot = the pair's top-k slot, found from pair_pos).
  T* const* owner_slots;
  const int* pair_pos;
  int K;
  // staged-store interface (plain Y / Y2 row stores only)
  static constexpr bool kStageable = std::is_same<T, __nv_bfloat16>::value;
  __device__ __forceinline__ bool stage_ok() const { return !out_acc && !owner_acc && !owner_slots; }
  __device__ __forceinline__ int stage_n() const { return H; }
  __device__ __forceinline__ void stage_values(int g, int row, int n0, const float (&v)[32], float (&x)[32]) const {
    float b[32];
    if (bias) load_row<T, 32>(bias + static_cast<size_t>(g) * H + n0, b, min(32, H - n0));
    else
#pragma unroll
      for (int j = 0; j < 32; ++j) b[j] = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = v[j] + b[j];
    if (drop_p > 0.f) {
      const float inv = 1.f / (1.f - drop_p);
      const uint32_t kb = drop_keep_bits<32>(drop, drop_row_draw(drop, seg, g, row, H) + n0);
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = ((kb >> j) & 1u) ? x[j] * inv : 0.f;
    }
  }
  __device__ __forceinline__ T* stage_dst(int g, int m, int row, int n0, int which) const {
    T* base = which == 0 ? y : y2;
    return base ? base + static_cast<size_t>(row) * H + n0 : nullptr;
  }
  __device__ __forceinline__ bool stage_second() const { return y2 != nullptr; }
  template <int W>
  __device__ __forceinline__ void apply(int g, int m, int row, int n0, const float (&v)[W]) const {
    const int valid = min(W, H - n0);
    float b[W];
    if (bias) load_row<T, W>(bias + static_cast<size_t>(g) * H + n0, b, valid);
    else
#pragma unroll
      for (int j = 0; j < W; ++j) b[j] = 0.f;
    float x[W];
    if constexpr (W % 2 == 0) {
#pragma unroll
      for (int j = 0; j < W; j += 2) {  // paired fp32 adds
        const float2 r = __fadd2_rn(make_float2(v[j], v[j + 1]), make_float2(b[j], b[j + 1]));
        x[j] = r.x;
        x[j + 1] = r.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < W; ++j) x[j] = v[j] + b[j];
    }
    if (drop_p > 0.f) {
      static_assert(W <= 32, "dropout keep bits cover at most 32 columns");
      const float inv = 1.f / (1.f - drop_p);
      const uint32_t kb = drop_keep_bits<W>(drop, drop_row_draw(drop, seg, g, row, H) + n0);
#pragma unroll
      for (int j = 0; j < W; ++j) x[j] = ((kb >> j) & 1u) ? x[j] * inv : 0.f;
    }
    store_row<T, W>(y + static_cast<size_t>(row) * H + n0, x, valid, cs);
    if (y2) store_row<T, W>(y2 + static_cast<size_t>(row) * H + n0, x, valid, 0);
    if (!out_acc && !owner_acc && !owner_slots) return;  // gather-combine mode: the combine reads Y afterwards
    const int t = tok[row];
    if (t >= 0 && owner_slots) {
      const float s = weight_scaling ? w[row] : 1.f;
      const int q = t / owner_rows;
      const int slot = (K == 1 || pair_pos[static_cast<size_t>(t) * K] == row + seg[0]) ? 0 : 1;
      float xs[W];
#pragma unroll
      for (int j = 0; j < W; ++j) xs[j] = s * x[j];
      store_row<T, W>(owner_slots[q] + (static_cast<size_t>(t - q * owner_rows) * K + slot) * H + n0, xs, valid, 0);
      return;
    }
    if (t >= 0) {
      const float s = weight_scaling ? w[row] : 1.f;
      float* dst;
      if (owner_acc) {
        const int q = t / owner_rows;
        dst = owner_acc[q] + static_cast<size_t>(t - q * owner_rows) * H;
      } else {
        dst = out_acc + static_cast<size_t>(t) * H;
      }
      scatter_add_row<W>(dst + n0, x, s, valid);
    }
  }
};

// fc2 data-gradient: dH = (dY * down_e^T) .* GeLU'(a)        (tensor.py:134-138, 204-207)
template <typename T>
struct EpiFc2Dgrad {
  T* dh;
  const T* gelu_grad;
  int F;
  const int* seg;
  int cs;
  // Optional [rows/32 x F] fp32 partial column sums of dH (bias_up gradient, tensor.py:154)
  // per 32-row block: needs the 32 lanes of a warp on 32 consecutive rows (tcgen05 kernels).
  float* colsum_part;
  template <int W>
  __device__ __forceinline__ void apply(int g, int m, int row, int n0, const float (&v)[W]) const {
    const int valid = min(W, F - n0);
    const size_t off = static_cast<size_t>(row) * F + n0;
    float gd[W];
    load_row<T, W>(gelu_grad + off, gd, valid);
    float x[W];
    if constexpr (W % 2 == 0) {
#pragma unroll
      for (int j = 0; j < W; j += 2) {  // paired fp32 multiplies
        const float2 r = __fmul2_rn(make_float2(v[j], v[j + 1]), make_float2(gd[j], gd[j + 1]));
        x[j] = r.x;
        x[j + 1] = r.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < W; ++j) x[j] = v[j] * gd[j];
    }
    store_row<T, W>(dh + off, x, valid, cs);
    if constexpr (W == 32) {
      if (colsum_part) {
        // the column sums use the bf16-rounded dH, exactly what the colsum pass would read
#pragma unroll
        for (int j = 0; j < W; ++j) x[j] = to_f32(from_f32<T>(x[j]));
        const float cs_val = warp_column_sums32(x);
        const int lane = threadIdx.x & 31;
        if (lane < valid) colsum_part[static_cast<size_t>(row >> 5) * F + n0 + lane] = cs_val;
      }
    }
  }
};

// fc1 data-gradient scattered back to token rows: dX[tok] += dH * up_e^T
// (index_select backward, tensor.py:235-239).
template <typename T>
struct EpiFc1Dgrad {
  float* dx_acc;  // [N*H] fp32 scatter-add target, or
  T* dxs;         // [rows*H] per-row store (gather-combined later by ppmoe_gate_grads)
  int H;
  const int* seg;
  const int* tok;
  int cs;
  static constexpr bool kStageable = std::is_same<T, __nv_bfloat16>::value;
  __device__ __forceinline__ bool stage_ok() const { return dxs != nullptr; }
  __device__ __forceinline__ int stage_n() const { return H; }
  __device__ __forceinline__ void stage_values(int, int, int, const float (&v)[32], float (&x)[32]) const {
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = v[j];
  }
  __device__ __forceinline__ T* stage_dst(int, int, int row, int n0, int) const {
    return dxs + static_cast<size_t>(row) * H + n0;
  }
  __device__ __forceinline__ bool stage_second() const { return false; }
  template <int W>
  __device__ __forceinline__ void apply(int g, int m, int row, int n0, const float (&v)[W]) const {
    const int valid = min(W, H - n0);
    if (dxs) {
      store_row<T, W>(dxs + static_cast<size_t>(row) * H + n0, v, valid, cs);
      return;
    }
    const int t = tok[row];
    if (t < 0) return;
    scatter_add_row<W>(dx_acc + static_cast<size_t>(t) * H + n0, v, 1.f, valid);
  }
};

// Weight gradient of one expert matrix: out[g][m][n]  (tensor.py:134-138, A^T * g).
template <typename T>
struct EpiWgrad {
  T* out;  // [G*M*N]
  int M;
  int N;
  int cs;
  static constexpr bool kStageable = std::is_same<T, __nv_bfloat16>::value;
  __device__ __forceinline__ bool stage_ok() const { return true; }
  __device__ __forceinline__ int stage_n() const { return N; }
  __device__ __forceinline__ void stage_values(int, int, int, const float (&v)[32], float (&x)[32]) const {
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = v[j];
  }
  __device__ __forceinline__ T* stage_dst(int g, int m, int, int n0, int) const {
    return m < M ? out + (static_cast<size_t>(g) * M + m) * N + n0 : nullptr;
  }
  __device__ __forceinline__ bool stage_second() const { return false; }
  template <int W>
  __device__ __forceinline__ void apply(int g, int m, int row, int n0, const float (&v)[W]) const {
    if (m >= M) return;
    const int valid = min(W, N - n0);
    store_row<T, W>(out + (static_cast<size_t>(g) * M + m) * N + n0, v, valid, cs);
  }
};

// Plain store into a dense [M x N] per-group output (used by the GEMM self-test).
template <typename T>
struct EpiStore {
  T* out;
  int N;
  const int* seg;
  int ldo_rows_from_seg;  // 1: row = local segment row, 0: row = g*M_fixed + m
  int M_fixed;
  template <int W>
  __device__ __forceinline__ void apply(int g, int m, int row, int n0, const float (&v)[W]) const {
    if (!ldo_rows_from_seg && m >= M_fixed) return;
    const int orow = ldo_rows_from_seg ? row : g * M_fixed + m;
    const int valid = min(W, N - n0);
    store_row<T, W>(out + static_cast<size_t>(orow) * N + n0, v, valid);
  }
};

}  // namespace ppmoe
