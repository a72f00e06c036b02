// Token data movement and the small backward kernels of the PPMoE layer:
//   gather_bulk_kernel   index-slice of replicated hidden rows into the padded
//                        expert-major buffer, bulk-TMA (cp.async.bulk) staged
//                        through a shared-memory ring (index_select, tensor.py:226-241;
//                        the paper's replacement for the all-to-all dispatch).
//   cast_kernel          fp32 combine accumulator -> output dtype.
//   bwd_dy_kernel        dY = w * dOut[tok], dw = <dOut[tok], Y>  (scale_rows and
//                        index_assign backward, tensor.py:190-194, 264-270).
//   gate_bwd_kernel      dL = s .* (dS - <dS, s>) with dS from dw and the aux loss
//                        (gather_rowwise / softmax / aux_loss backward,
//                        tensor.py:218-221, 287-291, moe.py:211-223).
//   gate_grads_kernel    dX = dx_acc + dL Wg^T and per-chunk X^T dL partials
//                        (matmul backward of the gate projection, tensor.py:134-138).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "../../include/ppmoe_capi.h"
#include "common.cuh"
#include "host.h"

namespace ppmoe {

__host__ __device__ inline size_t align_to(size_t v, size_t a) { return (v + a - 1) / a * a; }

// ------------------------------------------------------------------ gather

constexpr int kGatherThreads = 128;
constexpr int kGatherLag = 8;  // store groups allowed in flight before a slot is recycled

template <typename T, int LAG>
__global__ void __launch_bounds__(kGatherThreads)
    gather_bulk_kernel(const T* __restrict__ X, int H, const int* __restrict__ seg, int El,
                       const int* __restrict__ tok_sorted, const float* __restrict__ w_sorted, T* __restrict__ Xs,
                       int* __restrict__ tok_local, float* __restrict__ w_local, int R, int per) {
  extern __shared__ __align__(128) unsigned char sm[];
  const uint32_t row_bytes = static_cast<uint32_t>(H) * sizeof(T);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
  unsigned char* zero = sm + align_to(static_cast<size_t>(R) * 8, 128);
  int* stok = reinterpret_cast<int*>(zero + align_to(row_bytes, 128));  // this CTA's source tokens
  unsigned char* slots = reinterpret_cast<unsigned char*>(stok) + align_to(static_cast<size_t>(per) * 4, 128);
  const int s0 = seg[0];
  const int rows = seg[El] - s0;
  // this CTA's contiguous row range; its source token ids are staged in shared memory so the
  // issuing thread never waits on a global load (it used to, once per row)
  const int r0 = min(rows, static_cast<int>(blockIdx.x) * per);
  const int n = min(rows, r0 + per) - r0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int tok = tok_sorted[s0 + r0 + i];
    stok[i] = tok;
    tok_local[r0 + i] = tok;
    w_local[r0 + i] = w_sorted ? w_sorted[s0 + r0 + i] : 1.f;
  }
  for (uint32_t i = threadIdx.x; i < row_bytes / 16; i += blockDim.x) reinterpret_cast<uint4*>(zero)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < R; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x != 0) return;
  auto issue = [&](int i) {
    const int slot = i % R;
    const int tok = stok[i];
    if (tok >= 0) {
      mbar_arrive_expect_tx(&bars[slot], row_bytes);
      bulk_load(slots + static_cast<size_t>(slot) * row_bytes, X + static_cast<size_t>(tok) * H, row_bytes, &bars[slot]);
    } else {
      mbar_arrive(&bars[slot]);
    }
  };
  int issued = 0;
  for (; issued < n && issued <= R - LAG; ++issued) issue(issued);
  for (int i = 0; i < n; ++i) {
    const int slot = i % R;
    const int tok = stok[i];
    mbar_wait(&bars[slot], (i / R) & 1);
    bulk_store(Xs + static_cast<size_t>(r0 + i) * H, tok >= 0 ? slots + static_cast<size_t>(slot) * row_bytes : zero,
               row_bytes);
    bulk_commit();
    if (issued < n) {
      bulk_wait_read<LAG - 1>();  // store of the row that last used this slot has left smem
      issue(issued++);
    }
  }
  bulk_wait<0>();
}

// Fallback for rows whose byte size is not a multiple of 16 or too large for the ring.
template <typename T>
__global__ void gather_warp_kernel(const T* __restrict__ X, int H, const int* __restrict__ seg, int El,
                                   const int* __restrict__ tok_sorted, const float* __restrict__ w_sorted,
                                   T* __restrict__ Xs, int* __restrict__ tok_local, float* __restrict__ w_local) {
  const int s0 = seg[0];
  const int rows = seg[El] - s0;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x / 32;
  for (int r = blockIdx.x * wpb + (threadIdx.x >> 5); r < rows; r += gridDim.x * wpb) {
    const int tok = tok_sorted[s0 + r];
    if (lane == 0) {
      tok_local[r] = tok;
      w_local[r] = w_sorted ? w_sorted[s0 + r] : 1.f;
    }
    T* dst = Xs + static_cast<size_t>(r) * H;
    if (tok >= 0) {
      const T* src = X + static_cast<size_t>(tok) * H;
      for (int j = lane; j < H; j += 32) dst[j] = src[j];
    } else {
      for (int j = lane; j < H; j += 32) dst[j] = from_f32<T>(0.f);
    }
  }
}

// ------------------------------------------------------------------ casts

template <typename T>
__global__ void cast_kernel(const float* __restrict__ src, size_t n, T* __restrict__ dst) {
  const size_t i0 = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x * 4;
  for (size_t i = i0; i < n; i += stride) {
    if (i + 4 <= n) {
      float4 v = *reinterpret_cast<const float4*>(src + i);
      if constexpr (sizeof(T) == 2) {
        uint2 u;
        u.x = pack_bf16x2(v.x, v.y);
        u.y = pack_bf16x2(v.z, v.w);
        *reinterpret_cast<uint2*>(dst + i) = u;
      } else {
        *reinterpret_cast<float4*>(dst + i) = v;
      }
    } else {
      for (size_t j = i; j < n; ++j) dst[j] = from_f32<T>(src[j]);
    }
  }
}

// ------------------------------------------------------------------ dY / dw

template <typename T>
__global__ void bwd_dy_kernel(const T* __restrict__ dOut, const T* __restrict__ Y, const int* __restrict__ seg, int El,
                              int H, const int* __restrict__ tok_local, const float* __restrict__ w_local,
                              int weight_scaling, float drop_p, const unsigned long long* __restrict__ drop,
                              T* __restrict__ dY,
                              float* __restrict__ dw) {
  const int rows = seg[El] - seg[0];
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x / 32;
  const bool vec = (H % 8 == 0);
  for (int r = blockIdx.x * wpb + (threadIdx.x >> 5); r < rows; r += gridDim.x * wpb) {
    const int tok = tok_local[r];
    T* dy = dY + static_cast<size_t>(r) * H;
    if (tok < 0) {
      for (int j = lane; j < H; j += 32) dy[j] = from_f32<T>(0.f);
      if (lane == 0) dw[r] = 0.f;
      continue;
    }
    const float s = weight_scaling ? w_local[r] : 1.f;
    const T* g = dOut + static_cast<size_t>(tok) * H;
    const T* y = Y + static_cast<size_t>(r) * H;
    float acc = 0.f;
    if (drop_p > 0.f) {  // Y is the dropped output; dY reaches the expert through the same mask
      const float inv = 1.f / (1.f - drop_p);
      const unsigned long long rd = drop_row_draw(drop, seg, segment_of(seg, El, r), r, H);
      for (int j = lane; j < H; j += 32) {
        const float gv = to_f32(g[j]);
        acc = fmaf(gv, to_f32(y[j]), acc);
        const float keep = (drop_keep_bits<1>(drop, rd + j) & 1u) ? inv : 0.f;
        dy[j] = from_f32<T>(s * gv * keep);
      }
    } else if (vec && sizeof(T) == 2) {
      for (int j = lane * 8; j < H; j += 256) {
        uint4 gu = *reinterpret_cast<const uint4*>(g + j);
        uint4 yu = *reinterpret_cast<const uint4*>(y + j);
        const __nv_bfloat162* gh = reinterpret_cast<const __nv_bfloat162*>(&gu);
        const __nv_bfloat162* yh = reinterpret_cast<const __nv_bfloat162*>(&yu);
        uint4 out;
        uint32_t* o = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float2 gf = __bfloat1622float2(gh[i]);
          float2 yf = __bfloat1622float2(yh[i]);
          acc = fmaf(gf.x, yf.x, acc);
          acc = fmaf(gf.y, yf.y, acc);
          o[i] = pack_bf16x2(s * gf.x, s * gf.y);
        }
        *reinterpret_cast<uint4*>(dy + j) = out;
      }
    } else {
      for (int j = lane; j < H; j += 32) {
        const float gv = to_f32(g[j]);
        acc = fmaf(gv, to_f32(y[j]), acc);
        dy[j] = from_f32<T>(s * gv);
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) dw[r] = weight_scaling ? acc : 0.f;
  }
}

// CTA per 32-row block: phase 1 is bwd_dy_kernel's warp-per-row pass (8 warps x 4 rows);
// phase 2 re-reads the block's freshly written dY rows (L2-hot) column-wise and writes the
// block's column sums (the bias_down gradient partials) -- no DRAM pass over dY.
template <bool DROP>
__global__ void __launch_bounds__(256)
    bwd_dy_block_kernel(const __nv_bfloat16* __restrict__ dOut, const __nv_bfloat16* __restrict__ Y,
                        const int* __restrict__ seg, int El, int H, const int* __restrict__ tok_local,
                        const float* __restrict__ w_local, int weight_scaling, float drop_p,
                        const unsigned long long* __restrict__ drop, __nv_bfloat16* __restrict__ dY,
                        float* __restrict__ dw,
                        float* __restrict__ part) {
  const int rows = seg[El] - seg[0];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nblk = rows >> 5;
  const float inv = drop_p > 0.f ? 1.f / (1.f - drop_p) : 1.f;
  for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
    const int r0 = b << 5;
    for (int rr = warp; rr < 32; rr += 8) {
      const int r = r0 + rr;
      const int tok = tok_local[r];
      __nv_bfloat16* dy = dY + static_cast<size_t>(r) * H;
      if (tok < 0) {
        for (int j = lane * 8; j < H; j += 256) *reinterpret_cast<uint4*>(dy + j) = make_uint4(0, 0, 0, 0);
        if (lane == 0) dw[r] = 0.f;
        continue;
      }
      const float sw = weight_scaling ? w_local[r] : 1.f;
      const __nv_bfloat16* g = dOut + static_cast<size_t>(tok) * H;
      const __nv_bfloat16* y = Y + static_cast<size_t>(r) * H;
      const unsigned long long rd = DROP ? drop_row_draw(drop, seg, segment_of(seg, El, r), r, H) : 0ull;
      float acc = 0.f;
#pragma unroll 4
      for (int j = lane * 8; j < H; j += 256) {
        const uint32_t kb = DROP ? drop_keep_bits<8>(drop, rd + j) : 0u;
        const uint4 gu = *reinterpret_cast<const uint4*>(g + j);
        const uint4 yu = *reinterpret_cast<const uint4*>(y + j);
        const __nv_bfloat162* gh = reinterpret_cast<const __nv_bfloat162*>(&gu);
        const __nv_bfloat162* yh = reinterpret_cast<const __nv_bfloat162*>(&yu);
        uint4 out;
        uint32_t* o = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 gf = __bfloat1622float2(gh[i]);
          const float2 yf = __bfloat1622float2(yh[i]);
          acc = fmaf(gf.x, yf.x, acc);
          acc = fmaf(gf.y, yf.y, acc);
          float d0 = sw * gf.x, d1 = sw * gf.y;
          if (DROP) {
            d0 *= ((kb >> (2 * i)) & 1u) ? inv : 0.f;
            d1 *= ((kb >> (2 * i + 1)) & 1u) ? inv : 0.f;
          }
          o[i] = pack_bf16x2(d0, d1);
        }
        *reinterpret_cast<uint4*>(dy + j) = out;
      }
      acc = warp_sum(acc);
      if (lane == 0) dw[r] = weight_scaling ? acc : 0.f;
    }
    __syncthreads();  // the block's dY rows are visible to the whole CTA
    for (int c = threadIdx.x * 2; c < H; c += 512) {
      float s0 = 0.f, s1 = 0.f;
#pragma unroll 8
      for (int rr = 0; rr < 32; ++rr) {
        const float2 v = __bfloat1622float2(
            *reinterpret_cast<const __nv_bfloat162*>(dY + static_cast<size_t>(r0 + rr) * H + c));
        s0 += v.x;
        s1 += v.y;
      }
      *reinterpret_cast<float2*>(part + static_cast<size_t>(b) * H + c) = make_float2(s0, s1);
    }
    __syncthreads();
  }
}

// Column-slab form of bwd_dy_block_kernel (default): warp w owns the 256-column chunks
// w, w+8, ... of all 32 rows of the block, so the dY column sums accumulate in registers
// in the same row order (bit-identical partials) and phase 2's L2 re-read of dY is gone.
// The per-row dot <dOut[t], Y[r]> (the dw of scale_rows' backward, tensor.py:184-196) is
// summed per warp and then over the 8 warps in a fixed order through shared memory.
// CPW = chunks per warp = ceil(H / 2048).
template <int CPW, bool DROP>  // DROP: dropout mask regenerated (a separate instantiation keeps
                                // the Philox code out of the register budget of the p = 0 path)
__global__ void __launch_bounds__(256, 8 / CPW)
    bwd_dy_cols_kernel(const __nv_bfloat16* __restrict__ dOut, const __nv_bfloat16* __restrict__ Y,
                       const int* __restrict__ seg, int El, int H, const int* __restrict__ tok_local,
                       const float* __restrict__ w_local, int weight_scaling, float drop_p,
                       const unsigned long long* __restrict__ drop, __nv_bfloat16* __restrict__ dY,
                       float* __restrict__ dw,
                       float* __restrict__ part) {
  __shared__ float red[8][33];
  const int rows = seg[El] - seg[0];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nblk = rows >> 5;
  const int nchunk = H >> 8;
  const float inv = drop_p > 0.f ? 1.f / (1.f - drop_p) : 1.f;
  for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
    const int r0 = b << 5;
    float cs[CPW][8];
#pragma unroll
    for (int q = 0; q < CPW; ++q)
#pragma unroll
      for (int i = 0; i < 8; ++i) cs[q][i] = 0.f;
#pragma unroll 2
    for (int rr = 0; rr < 32; ++rr) {
      const int r = r0 + rr;
      const int tok = tok_local[r];
      __nv_bfloat16* dy = dY + static_cast<size_t>(r) * H;
      float acc = 0.f;
      if (tok < 0) {
#pragma unroll
        for (int q = 0; q < CPW; ++q) {
          const int ch = warp + 8 * q;
          if (ch < nchunk) *reinterpret_cast<uint4*>(dy + ch * 256 + lane * 8) = make_uint4(0, 0, 0, 0);
        }
      } else {
        const float sw = weight_scaling ? w_local[r] : 1.f;
        const __nv_bfloat16* g = dOut + static_cast<size_t>(tok) * H;
        const __nv_bfloat16* y = Y + static_cast<size_t>(r) * H;
        const unsigned long long rd = DROP ? drop_row_draw(drop, seg, segment_of(seg, El, r), r, H) : 0ull;
        uint4 gu[CPW], yu[CPW];
#pragma unroll
        for (int q = 0; q < CPW; ++q) {
          const int ch = warp + 8 * q;
          if (ch < nchunk) {
            gu[q] = *reinterpret_cast<const uint4*>(g + ch * 256 + lane * 8);
            yu[q] = *reinterpret_cast<const uint4*>(y + ch * 256 + lane * 8);
          }
        }
#pragma unroll
        for (int q = 0; q < CPW; ++q) {
          const int ch = warp + 8 * q;
          if (ch >= nchunk) continue;
          const int j = ch * 256 + lane * 8;
          const uint32_t kb = DROP ? drop_keep_bits<8>(drop, rd + j) : 0u;
          const __nv_bfloat162* gh = reinterpret_cast<const __nv_bfloat162*>(&gu[q]);
          const __nv_bfloat162* yh = reinterpret_cast<const __nv_bfloat162*>(&yu[q]);
          uint4 out;
          uint32_t* o = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 gf = __bfloat1622float2(gh[i]);
            const float2 yf = __bfloat1622float2(yh[i]);
            acc = fmaf(gf.x, yf.x, acc);
            acc = fmaf(gf.y, yf.y, acc);
            float d0 = sw * gf.x, d1 = sw * gf.y;
            if (DROP) {
              d0 *= ((kb >> (2 * i)) & 1u) ? inv : 0.f;
              d1 *= ((kb >> (2 * i + 1)) & 1u) ? inv : 0.f;
            }
            o[i] = pack_bf16x2(d0, d1);
            const float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&o[i]));
            cs[q][2 * i] += v.x;
            cs[q][2 * i + 1] += v.y;
          }
          *reinterpret_cast<uint4*>(dy + j) = out;
        }
      }
      acc = warp_sum(acc);
      if (lane == 0) red[warp][rr] = acc;
    }
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      const int ch = warp + 8 * q;
      if (ch >= nchunk) continue;
      float4* p = reinterpret_cast<float4*>(part + static_cast<size_t>(b) * H + ch * 256 + lane * 8);
      p[0] = make_float4(cs[q][0], cs[q][1], cs[q][2], cs[q][3]);
      p[1] = make_float4(cs[q][4], cs[q][5], cs[q][6], cs[q][7]);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int r = r0 + threadIdx.x;
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
      dw[r] = (weight_scaling && tok_local[r] >= 0) ? s : 0.f;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ gather-combine

// out[t] = sum_s w[t,s] * R[pair_pos[t,s] - row_lo]  (+ dL[t] . Wg^T)
// over the slots whose sorted row is one of this rank's rows [seg[0], seg[El]).  Forward:
// the top-k combine of the expert outputs (scale_rows + index_assign, tensor.py:184-272);
// backward: the index_select backward of the experts' per-row dX plus the gate
// projection's dX (matmul backward, tensor.py:134-138).  A deterministic gather in slot
// order replaces the fp32 scatter-add accumulator.  Tokens with no local pair get only the
// gate term (or zero).
//
// bf16, H % CW == 0: a thread owns CW consecutive columns for all tokens of its block, so
// the gate weights of those columns (CW x EB fp32) stay in registers.  U tokens are
// processed together: their pair positions are loaded first, then all U*KS row loads
// are issued before any is consumed (memory-level parallelism of a gather).
template <int CW> struct ColVec;
template <> struct ColVec<8> { using type = uint4; };
template <> struct ColVec<4> { using type = uint2; };

template <int EB, int CW, int U, int KT>
__global__ void __launch_bounds__(256)
    combine_rows_bf16_kernel(const __nv_bfloat16* __restrict__ R, const int* __restrict__ seg, int El,
                             const int* __restrict__ pair_pos, const float* __restrict__ w, int N, int Kr, int H,
                             const float* __restrict__ dL, const float* __restrict__ Wg, int E,
                             __nv_bfloat16* __restrict__ out) {
  using V = typename ColVec<CW>::type;
  constexpr int KS = KT > 0 ? KT : 1;  // slots loaded per batch
  const int K = KT > 0 ? KT : Kr;
  const int row_lo = seg[0], row_hi = seg[El];
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) * CW;
  if (j >= H) return;
  float wg[EB > 0 ? CW : 1][EB > 0 ? EB : 1];
  if constexpr (EB > 0) {
#pragma unroll
    for (int q = 0; q < CW; ++q)
#pragma unroll
      for (int e = 0; e < EB; ++e) wg[q][e] = e < E ? Wg[static_cast<size_t>(j + q) * E + e] : 0.f;
  }
  for (int t0 = blockIdx.y * U; t0 < N; t0 += gridDim.y * U) {
    float acc[U][CW];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < CW; ++q) acc[u][q] = 0.f;
    for (int sb = 0; sb < K; sb += KS) {
      int rows[U][KS];
      float ws[U][KS];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          const int t = t0 + u, sl = sb + s;
          rows[u][s] = -1;
          ws[u][s] = 0.f;
          if (t < N) {
            const int p = pair_pos[static_cast<size_t>(t) * K + sl];
            if (p >= row_lo && p < row_hi) {
              rows[u][s] = p - row_lo;
              ws[u][s] = w ? w[static_cast<size_t>(t) * K + sl] : 1.f;
            }
          }
        }
      V v[U][KS];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          if (rows[u][s] >= 0) v[u][s] = *reinterpret_cast<const V*>(R + static_cast<size_t>(rows[u][s]) * H + j);
          else memset(&v[u][s], 0, sizeof(V));
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&v[u][s]);
#pragma unroll
          for (int i = 0; i < CW / 2; ++i) {
            const float2 f = __bfloat1622float2(hv[i]);
            acc[u][2 * i] = fmaf(ws[u][s], f.x, acc[u][2 * i]);
            acc[u][2 * i + 1] = fmaf(ws[u][s], f.y, acc[u][2 * i + 1]);
          }
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + u;
      if (t >= N) break;
      if constexpr (EB > 0) {
#pragma unroll
        for (int e = 0; e < EB; ++e) {
          const float d = e < E ? dL[static_cast<size_t>(t) * E + e] : 0.f;
#pragma unroll
          for (int q = 0; q < CW; ++q) acc[u][q] = fmaf(d, wg[q][e], acc[u][q]);
        }
      }
      V r;
      uint32_t* rw = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
      for (int i = 0; i < CW / 2; ++i) rw[i] = pack_bf16x2(acc[u][2 * i], acc[u][2 * i + 1]);
      *reinterpret_cast<V*>(out + static_cast<size_t>(t) * H + j) = r;
    }
  }
}

// Input gradient of the layer in one pass over the tokens (bf16, E <= EB, k = KT):
//   dX[t]  = sum_s dXs[pair_pos[t,s] - row_lo] + dL[t,:] . Wg^T      (index_select + matmul bwd)
//   part[blockIdx.y] += X[t]^T dL[t,:]                               (dWg partials, tensor.py:134-138)
// A CTA owns a slab of kIgSlab columns and a contiguous token range.  A producer warp
// stages, per token, the X row slab, the slab of every local pair's dXs row and dL[t] into
// a shared-memory ring with 1-D bulk copies (bytes in flight independent of registers);
// the 8 consumer warps own 4 columns per thread, whose Wg rows and dWg partial sums stay in
// registers.  Pair sums in slot order: deterministic.
constexpr int kIgSlab = 1024;    // columns per CTA
constexpr int kIgConsumers = 256;
constexpr int kIgTok = 2;        // tokens per ring stage (amortises the barrier handshake)
constexpr int kIgRingBytes = 96 * 1024;

template <int KT>
struct alignas(16) IgStage {  // per-stage control block (rows live in a separate byte ring)
  float dl[kIgTok][16];
  int valid[kIgTok][KT];
};

template <int KT>
__host__ __device__ constexpr int ig_tok_bytes() { return (KT + 1) * kIgSlab * 2; }
template <int KT>
__host__ __device__ constexpr int ig_stage_bytes() { return kIgTok * ig_tok_bytes<KT>(); }
template <int KT>
__host__ __device__ constexpr int ig_stages() { return kIgRingBytes / ig_stage_bytes<KT>(); }

template <int EB, int KT, int MINB>
__global__ void __launch_bounds__(kIgConsumers + 32, MINB)
    input_grads_ring_kernel(const __nv_bfloat16* __restrict__ dXs, const int* __restrict__ seg, int El,
                            const int* __restrict__ pair_pos, int N, int H, const __nv_bfloat16* __restrict__ X,
                            const float* __restrict__ dL, const float* __restrict__ Wg, int E,
                            __nv_bfloat16* __restrict__ dX, float* __restrict__ part) {
  constexpr int S = ig_stages<KT>();
  constexpr int SB = ig_stage_bytes<KT>();
  constexpr int TB = ig_tok_bytes<KT>();
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* ring = sm;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * SB);
  uint64_t* empty = full + S;
  IgStage<KT>* ctl = reinterpret_cast<IgStage<KT>*>(empty + S);

  const int c0 = blockIdx.x * kIgSlab;
  const int ncols = min(kIgSlab, H - c0);
  const uint32_t slab_bytes = static_cast<uint32_t>(ncols) * 2;
  const int per = (N + gridDim.y - 1) / gridDim.y;
  const int tb = blockIdx.y * per, te = min(N, tb + per);
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kIgConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (threadIdx.x >= kIgConsumers) {  // ---------------- producer warp
    const int lane = threadIdx.x & 31;
    const int row_lo = dX ? seg[0] : 0, row_hi = dX ? seg[El] : 0;
    for (int b = tb; b < te; b += 32) {  // b - tb is a multiple of kIgTok
      // one coalesced round trip for the routing of 32 tokens
      const int t = b + lane;
      int rows[KT];
      float d[EB];
#pragma unroll
      for (int s = 0; s < KT; ++s) rows[s] = -1;
#pragma unroll
      for (int e = 0; e < EB; ++e) d[e] = 0.f;
      if (t < te) {
        if (dX) {
#pragma unroll
          for (int s = 0; s < KT; ++s) {
            const int p = pair_pos[static_cast<size_t>(t) * KT + s];
            rows[s] = (p >= row_lo && p < row_hi) ? p - row_lo : -1;
          }
        }
#pragma unroll
        for (int e = 0; e < EB; ++e)
          if (e < E) d[e] = dL[static_cast<size_t>(t) * E + e];
      }
      const int nb = min(32, te - b);
      // every lane writes its token's control entry; the stage's first lane posts the bytes
      for (int l0 = 0; l0 < nb; l0 += kIgTok) {
        const int i = b - tb + l0;  // first token of the stage
        const int st = (i / kIgTok) % S;
        const int it = i / kIgTok / S;
        if (lane == l0 && it > 0) mbar_wait(&empty[st], (it - 1) & 1);
        __syncwarp();
        const int u = lane - l0;
        uint32_t bytes = 0;
        if (u >= 0 && u < kIgTok && lane < nb) {
          IgStage<KT>& c = ctl[st];
#pragma unroll
          for (int e = 0; e < EB; ++e) c.dl[u][e] = d[e];
          bytes = part ? slab_bytes : 0;
#pragma unroll
          for (int s = 0; s < KT; ++s) {
            c.valid[u][s] = rows[s] >= 0;
            if (rows[s] >= 0) bytes += slab_bytes;
          }
        }
        // total bytes of the stage's tokens, to the stage's first lane
#pragma unroll
        for (int o = 1; o < kIgTok; o <<= 1) bytes += __shfl_down_sync(0xffffffffu, bytes, o);
        __syncwarp();
        if (lane == l0) mbar_arrive_expect_tx(&full[st], bytes);
        __syncwarp();
        if (u >= 0 && u < kIgTok && lane < nb) {
          unsigned char* stg = ring + static_cast<size_t>(st) * SB + u * TB;
          if (part) bulk_load(stg, X + static_cast<size_t>(t) * H + c0, slab_bytes, &full[st]);
#pragma unroll
          for (int s = 0; s < KT; ++s)
            if (rows[s] >= 0)
              bulk_load(stg + (s + 1) * kIgSlab * 2, dXs + static_cast<size_t>(rows[s]) * H + c0, slab_bytes,
                        &full[st]);
        }
      }
    }
    return;
  }

  // ---------------------------------------------------- consumer warps
  const int jl = threadIdx.x * 4;  // local column
  const bool active = jl < ncols;
  const int j = c0 + jl;
  float2 wg[2][EB];          // (Wg[j+2p][e], Wg[j+2p+1][e])
  float2 pacc[4][EB / 2];    // (dWg[j+q][e], dWg[j+q][e+1])
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int e = 0; e < EB; ++e) {
      const bool ok = active && dX && e < E;
      wg[p][e] = make_float2(ok ? Wg[static_cast<size_t>(j + 2 * p) * E + e] : 0.f,
                             ok ? Wg[static_cast<size_t>(j + 2 * p + 1) * E + e] : 0.f);
    }
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int e = 0; e < EB / 2; ++e) pacc[q][e] = make_float2(0.f, 0.f);
  for (int i0 = 0; i0 < te - tb; i0 += kIgTok) {
    const int st = (i0 / kIgTok) % S;
    mbar_wait(&full[st], (i0 / kIgTok / S) & 1);
    const IgStage<KT>& c = ctl[st];
    if (active) {
#pragma unroll
      for (int u = 0; u < kIgTok; ++u) {
        const int t = tb + i0 + u;
        if (t >= te) break;
        const unsigned char* stg = ring + static_cast<size_t>(st) * SB + u * TB;
        float d[EB];
#pragma unroll
        for (int e = 0; e < EB; e += 4) {
          const float4 f = *reinterpret_cast<const float4*>(&c.dl[u][e]);
          d[e] = f.x, d[e + 1] = f.y, d[e + 2] = f.z, d[e + 3] = f.w;
        }
        if (dX) {
          float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
          for (int s = 0; s < KT; ++s) {
            if (c.valid[u][s]) {
              const uint2 v = *reinterpret_cast<const uint2*>(stg + (s + 1) * kIgSlab * 2 + jl * 2);
              acc[0] = __fadd2_rn(acc[0], __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.x)));
              acc[1] = __fadd2_rn(acc[1], __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.y)));
            }
          }
#pragma unroll
          for (int e = 0; e < EB; ++e) {
            const float2 dd = make_float2(d[e], d[e]);
            acc[0] = __ffma2_rn(dd, wg[0][e], acc[0]);
            acc[1] = __ffma2_rn(dd, wg[1][e], acc[1]);
          }
          uint2 o;
          o.x = pack_bf16x2(acc[0].x, acc[0].y);
          o.y = pack_bf16x2(acc[1].x, acc[1].y);
          *reinterpret_cast<uint2*>(dX + static_cast<size_t>(t) * H + j) = o;
        }
        if (part) {
          const uint2 v = *reinterpret_cast<const uint2*>(stg + jl * 2);
          const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.x));
          const float2 bb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.y));
          const float x[4] = {a.x, a.y, bb.x, bb.y};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 xx = make_float2(x[q], x[q]);
#pragma unroll
            for (int e = 0; e < EB / 2; ++e) pacc[q][e] = __ffma2_rn(xx, make_float2(d[2 * e], d[2 * e + 1]), pacc[q][e]);
          }
        }
      }
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[st]);
  }
  if (part && active) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float* p = part + (static_cast<size_t>(blockIdx.y) * H + j + q) * E;
#pragma unroll
      for (int e = 0; e < EB / 2; ++e) {
        if (2 * e < E) p[2 * e] = pacc[q][e].x;
        if (2 * e + 1 < E) p[2 * e + 1] = pacc[q][e].y;
      }
    }
  }
}

template <int KT>
constexpr size_t ig_smem_bytes() {
  return static_cast<size_t>(ig_stages<KT>()) * ig_stage_bytes<KT>() + ig_stages<KT>() * 16 +
         ig_stages<KT>() * sizeof(IgStage<KT>);
}

// Generic form (fp32, odd widths, many experts): thread per column, gate weights from L1.
template <typename T>
__global__ void __launch_bounds__(256)
    combine_rows_kernel(const T* __restrict__ R, const int* __restrict__ seg, int El, const int* __restrict__ pair_pos,
                        const float* __restrict__ w, int N, int K, int H, const float* __restrict__ dL,
                        const float* __restrict__ Wg, int E, T* __restrict__ out) {
  const int row_lo = seg[0], row_hi = seg[El];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= H) return;
  for (int t = blockIdx.y; t < N; t += gridDim.y) {
    float acc = 0.f;
    for (int sl = 0; sl < K; ++sl) {
      const int p = pair_pos[static_cast<size_t>(t) * K + sl];
      if (p >= row_lo && p < row_hi)
        acc = fmaf(w ? w[static_cast<size_t>(t) * K + sl] : 1.f, to_f32(R[static_cast<size_t>(p - row_lo) * H + j]),
                   acc);
    }
    if (dL)
      for (int e = 0; e < E; ++e) acc = fmaf(dL[static_cast<size_t>(t) * E + e], Wg[static_cast<size_t>(j) * E + e], acc);
    out[static_cast<size_t>(t) * H + j] = from_f32<T>(acc);
  }
}

// ------------------------------------------------------------------ gate backward

__global__ void gate_bwd_kernel(const float* __restrict__ scores, const int* __restrict__ idx,
                                const int* __restrict__ pair_pos, const float* __restrict__ dw,
                                const int* __restrict__ seg, int El, const int* __restrict__ cnt_top1, int N, int E,
                                int K, const float* __restrict__ aux_grad_p, float* __restrict__ dL) {
  const float aux_grad = aux_grad_p ? aux_grad_p[0] : 0.f;
  const int row_lo = seg[0], row_hi = seg[El];
  extern __shared__ float prod[];  // [TT][E] dS*s, then [TT] row sums
  const int TT = blockDim.x / E;
  float* red = prod + TT * E;
  const int tl = threadIdx.x / E, e = threadIdx.x % E;
  const int t = blockIdx.x * TT + tl;
  const bool active = tl < TT && t < N;
  float ds = 0.f, s = 0.f;
  if (active) {
    s = scores[static_cast<size_t>(t) * E + e];
    ds = aux_grad * (static_cast<float>(E) / N) * (static_cast<float>(cnt_top1[e]) / N);
    for (int k = 0; k < K; ++k) {
      const size_t pi = static_cast<size_t>(t) * K + k;
      if (idx[pi] != e) continue;
      const int pos = pair_pos[pi];
      if (pos >= row_lo && pos < row_hi) ds += dw[pos - row_lo];
    }
  }
  if (tl < TT) prod[tl * E + e] = ds * s;
  __syncthreads();
  if (threadIdx.x < TT) {
    float acc = 0.f;  // fixed order: deterministic
    for (int j = 0; j < E; ++j) acc += prod[threadIdx.x * E + j];
    red[threadIdx.x] = acc;
  }
  __syncthreads();
  if (active) dL[static_cast<size_t>(t) * E + e] = s * (ds - red[tl]);
}

// Token-chunk row ranges of every local expert segment: rows are in ascending token
// order inside a segment, so chunk c (tokens [c*N/C, (c+1)*N/C)) is a contiguous row
// range found by binary search over the segment's kept rows.
__global__ void chunk_rows_kernel(const int* __restrict__ tok_local, const int* __restrict__ seg,
                                  const int* __restrict__ kept, int El, int N, int C, int* __restrict__ row_lo,
                                  int* __restrict__ row_hi) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (C + 1) * El) return;
  const int c = i / El, g = i % El;
  const int base = seg[g] - seg[0];
  const int cnt = kept[g];
  if (c == C) {  // padding rows of the segment (token -1)
    row_lo[i] = base + cnt;
    row_hi[i] = seg[g + 1] - seg[0];
    return;
  }
  auto lower = [&](int t) {
    int lo = 0, hi = cnt;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (tok_local[base + mid] < t) lo = mid + 1;
      else hi = mid;
    }
    return base + lo;
  };
  const long long t_lo = static_cast<long long>(c) * N / C;
  const long long t_hi = static_cast<long long>(c + 1) * N / C;
  row_lo[i] = lower(static_cast<int>(t_lo));
  row_hi[i] = lower(static_cast<int>(t_hi));
}

constexpr int kGradTC = 128;  // tokens per chunk of the dWg partials

template <typename T, int CPT>
__device__ __forceinline__ void load_cols(const T* p, float (&v)[CPT]) {
  if constexpr (sizeof(T) == 2 && CPT == 2) {
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
    v[0] = a.x;
    v[1] = a.y;
  } else if constexpr (sizeof(T) == 4 && CPT == 2) {
    const float2 f = *reinterpret_cast<const float2*>(p);
    v[0] = f.x;
    v[1] = f.y;
  } else if constexpr (sizeof(T) == 2 && CPT == 4) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  } else if constexpr (sizeof(T) == 4 && CPT == 4) {
    const float4 f = *reinterpret_cast<const float4*>(p);
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  } else {
#pragma unroll
    for (int c = 0; c < CPT; ++c) v[c] = to_f32(p[c]);
  }
}

template <typename T, int CPT>
__device__ __forceinline__ void store_cols(T* p, const float (&v)[CPT]) {
  if constexpr (sizeof(T) == 2 && CPT == 2) {
    *reinterpret_cast<uint32_t*>(p) = pack_bf16x2(v[0], v[1]);
  } else if constexpr (sizeof(T) == 4 && CPT == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else if constexpr (sizeof(T) == 2 && CPT == 4) {
    uint2 u;
    u.x = pack_bf16x2(v[0], v[1]);
    u.y = pack_bf16x2(v[2], v[3]);
    *reinterpret_cast<uint2*>(p) = u;
  } else if constexpr (sizeof(T) == 4 && CPT == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
#pragma unroll
    for (int c = 0; c < CPT; ++c) p[c] = from_f32<T>(v[c]);
  }
}

// Thread = CPT adjacent hidden columns; the token loop is unrolled by 4 with all loads of
// a group issued before the FMAs (enough bytes in flight to stream at HBM rate).
template <typename T, int EB, int CPT>
__global__ void __launch_bounds__(256)
    gate_grads_kernel(const float* __restrict__ dx_acc, const T* __restrict__ X, const float* __restrict__ dL,
                      const float* __restrict__ Wg, int N, int H, int E, T* __restrict__ dX, float* __restrict__ part) {
  __shared__ float sdl[kGradTC][EB];
  const int j0 = (blockIdx.x * 256 + threadIdx.x) * CPT;
  const int c = blockIdx.y;
  const int t0 = c * kGradTC;
  for (int i = threadIdx.x; i < kGradTC * EB; i += 256) {
    const int tt = i / EB, e = i % EB;
    const int t = t0 + tt;
    sdl[tt][e] = (t < N && e < E) ? dL[static_cast<size_t>(t) * E + e] : 0.f;
  }
  __syncthreads();
  if (j0 >= H) return;
  float wg[CPT][EB], acc[CPT][EB];
#pragma unroll
  for (int q = 0; q < CPT; ++q)
#pragma unroll
    for (int e = 0; e < EB; ++e) {
      wg[q][e] = e < E ? Wg[static_cast<size_t>(j0 + q) * E + e] : 0.f;
      acc[q][e] = 0.f;
    }
  const int tn = min(kGradTC, N - t0);
  constexpr int U = 4;
  for (int tt = 0; tt < tn; tt += U) {
    float dxv[U][CPT], xv[U][CPT];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t o = static_cast<size_t>(t0 + tt + u) * H + j0;
      const bool ok = tt + u < tn;
#pragma unroll
      for (int q = 0; q < CPT; ++q) dxv[u][q] = 0.f, xv[u][q] = 0.f;
      if (ok && dX && dx_acc) load_cols<float, CPT>(dx_acc + o, dxv[u]);
      if (ok && part) load_cols<T, CPT>(X + o, xv[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (tt + u >= tn) break;
      const float* d = sdl[tt + u];
      if (dX) {
        float v[CPT];
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          v[q] = dxv[u][q];
#pragma unroll
          for (int e = 0; e < EB; ++e) v[q] = fmaf(d[e], wg[q][e], v[q]);
        }
        store_cols<T, CPT>(dX + static_cast<size_t>(t0 + tt + u) * H + j0, v);
      }
      if (part) {
#pragma unroll
        for (int q = 0; q < CPT; ++q)
#pragma unroll
          for (int e = 0; e < EB; ++e) acc[q][e] = fmaf(xv[u][q], d[e], acc[q][e]);
      }
    }
  }
  if (part) {
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      float* p = part + (static_cast<size_t>(c) * H + j0 + q) * E;
#pragma unroll
      for (int e = 0; e < EB; ++e)
        if (e < E) p[e] = acc[q][e];
    }
  }
}

// Gate-weight gradient alone (dX not wanted): part[chunk] = X[chunk tokens]^T dL[chunk tokens]
// over a slab of kDwgSlab columns (tensor.py:134-138, the matmul backward of X Wg).  X is
// read once at HBM rate: a producer warp stages kDwgTok whole token slabs plus their dL rows
// per ring stage with 1-D bulk copies (one mbarrier handshake per 16 tokens, not per token),
// and the 8 consumer warps keep 4 columns x EB experts of partial sums in registers (FFMA2).
constexpr int kDwgSlab = 1024;
constexpr int kDwgTok = 16;
constexpr int kDwgStages = 5;

template <int EB>
struct DwgGeom {
  static constexpr int kX = kDwgTok * kDwgSlab * 2;  // bytes of the X slabs of one stage
  static constexpr int kL = kDwgTok * EB * 4;        // bytes of the dL rows of one stage
  static constexpr int kStage = kX + kL;
  static constexpr size_t kSmem = static_cast<size_t>(kDwgStages) * kStage + 2 * kDwgStages * 8;
};

template <int EB>
__global__ void __launch_bounds__(kIgConsumers + 32, 1)
    dwg_bulk_kernel(const __nv_bfloat16* __restrict__ X, const float* __restrict__ dL, int N, int H, float* __restrict__ part) {
  using G = DwgGeom<EB>;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kDwgStages * G::kStage);
  uint64_t* empty = full + kDwgStages;
  const int c0 = blockIdx.x * kDwgSlab;
  const int ncols = min(kDwgSlab, H - c0);
  const uint32_t slab_bytes = static_cast<uint32_t>(ncols) * 2;
  const int per = (N + gridDim.y - 1) / gridDim.y;
  const int tb = blockIdx.y * per, te = min(N, tb + per);
  const int nstage = te > tb ? (te - tb + kDwgTok - 1) / kDwgTok : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kDwgStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kIgConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x >= kIgConsumers) {  // ---------------- producer warp
    const int lane = threadIdx.x & 31;
    for (int i = 0; i < nstage; ++i) {
      const int st = i % kDwgStages;
      const int t0 = tb + i * kDwgTok;
      const int nt = min(kDwgTok, te - t0);
      unsigned char* stg = sm + static_cast<size_t>(st) * G::kStage;
      if (lane == 0) {
        if (i >= kDwgStages) mbar_wait(&empty[st], ((i / kDwgStages) - 1) & 1);
        mbar_arrive_expect_tx(&full[st], nt * slab_bytes + nt * EB * 4);
      }
      __syncwarp();
      if (lane < nt) bulk_load(stg + lane * kDwgSlab * 2, X + static_cast<size_t>(t0 + lane) * H + c0, slab_bytes, &full[st]);
      if (lane == 31) bulk_load(stg + G::kX, dL + static_cast<size_t>(t0) * EB, nt * EB * 4, &full[st]);
    }
    return;
  }
  // ---------------------------------------------------- consumer warps
  const int jl = threadIdx.x * 4;
  const bool active = jl < ncols;
  float2 pacc[4][EB / 2];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int e = 0; e < EB / 2; ++e) pacc[q][e] = make_float2(0.f, 0.f);
  for (int i = 0; i < nstage; ++i) {
    const int st = i % kDwgStages;
    const int nt = min(kDwgTok, te - tb - i * kDwgTok);
    mbar_wait(&full[st], (i / kDwgStages) & 1);
    const unsigned char* stg = sm + static_cast<size_t>(st) * G::kStage;
    const float* dls = reinterpret_cast<const float*>(stg + G::kX);
    if (active) {
#pragma unroll 4
      for (int u = 0; u < nt; ++u) {
        const uint2 v = *reinterpret_cast<const uint2*>(stg + u * kDwgSlab * 2 + jl * 2);
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.x));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.y));
        const float x[4] = {a.x, a.y, b.x, b.y};
        float d[EB];
#pragma unroll
        for (int e = 0; e < EB; e += 4) {
          const float4 f = *reinterpret_cast<const float4*>(dls + u * EB + e);
          d[e] = f.x, d[e + 1] = f.y, d[e + 2] = f.z, d[e + 3] = f.w;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 xx = make_float2(x[q], x[q]);
#pragma unroll
          for (int e = 0; e < EB / 2; ++e) pacc[q][e] = __ffma2_rn(xx, make_float2(d[2 * e], d[2 * e + 1]), pacc[q][e]);
        }
      }
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[st]);
  }
  if (active) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float4* p = reinterpret_cast<float4*>(part + (static_cast<size_t>(blockIdx.y) * H + c0 + jl + q) * EB);
#pragma unroll
      for (int e = 0; e < EB / 2; e += 2) p[e / 2] = make_float4(pacc[q][e].x, pacc[q][e].y, pacc[q][e + 1].x, pacc[q][e + 1].y);
    }
  }
}

static int dwg_chunks(int N, int H) {
  const int gx = (H + kDwgSlab - 1) / kDwgSlab;
  return max(1, min((N + kDwgTok - 1) / kDwgTok, num_sms() / gx));
}

__global__ void dwg_reduce_kernel(const float* __restrict__ part, int C, int HE, float* __restrict__ dWg) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= HE) return;
  float s = 0.f;
  for (int c = 0; c < C; ++c) s += part[static_cast<size_t>(c) * HE + i];
  dWg[i] = s;
}

static bool dwg_bulk_ok(int dtype, int H, int E) {
  const char* e = std::getenv("PPMOE_DWG");  // PPMOE_DWG=ring: the combined input-gradient kernel (A/B)
  return !(e && std::strcmp(e, "ring") == 0) && dtype == kBF16 && H % 8 == 0 && (E == 4 || E == 8 || E == 16);
}

static int input_grads_chunks(int N, int H, int E) {
  const int gx = (H + kIgSlab - 1) / kIgSlab;
  const int per_sm = E <= 8 ? 2 : 1;
  return max(1, min(N, num_sms() * per_sm / gx));
}

static bool input_grads_fused(int dtype, int H, int K, int E) {
  return dtype == kBF16 && H % 8 == 0 && K >= 1 && K <= 4 && E <= 16;
}

template <int EB, int KT, int MINB>
static int launch_input_grads(dim3 grid, cudaStream_t s, const void* dXs, const int* seg, int El, const int* pair_pos,
                              int N, int H, const void* X, const float* dL, const float* Wg, int E, void* dX,
                              float* part) {
  constexpr size_t smem = ig_smem_bytes<KT>();
  auto kern = input_grads_ring_kernel<EB, KT, MINB>;
  PPMOE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kern<<<grid, kIgConsumers + 32, smem, s>>>(static_cast<const __nv_bfloat16*>(dXs), seg, El, pair_pos, N, H,
                                             static_cast<const __nv_bfloat16*>(X), dL, Wg, E,
                                             static_cast<__nv_bfloat16*>(dX), part);
  return check_launch("input_grads_ring_kernel");
}

// desc = [key0, key1, threshold, first draw of local experts 0..El-1]: the experts before
// e0 (on lower ranks, moe.py:294-301) consume kept[e] * H draws each, in ascending id.
__global__ void dropout_stream_kernel(const int* __restrict__ kept, int e0, int El, int H, unsigned long long key0,
                                      unsigned long long key1, unsigned long long threshold,
                                      unsigned long long first_draw, unsigned long long* __restrict__ desc) {
  if (threadIdx.x != 0) return;
  desc[0] = key0;
  desc[1] = key1;
  desc[2] = threshold;
  unsigned long long m = first_draw;
  for (int e = 0; e < e0; ++e) m += static_cast<unsigned long long>(kept[e]) * H;
  for (int g = 0; g < El; ++g) {
    desc[3 + g] = m;
    m += static_cast<unsigned long long>(kept[e0 + g]) * H;
  }
}

}  // namespace ppmoe

using namespace ppmoe;

extern "C" {

int ppmoe_gather(const void* X, int dtype, int N, int H, const int* seg, int El, const int* tok_sorted,
                 const float* w_sorted, int rows_cap, void* Xs, int* tok_local, float* w_local, void* stream) {
  PPMOE_REQUIRE(dtype == kBF16 || dtype == kF32, "bad dtype");
  PPMOE_REQUIRE(N >= 0 && H >= 1 && El >= 1, "bad gather shape");
  (void)N;
  if (rows_cap == 0) return kOk;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t esz = dtype == kBF16 ? 2 : 4;
  const size_t row_bytes = static_cast<size_t>(H) * esz;
  // PPMOE_GATHER_CTAS = CTAs per SM (1 or 2); with 2, each ring is half the size and the
  // store lag 4 instead of 8, so the loads in flight per SM stay about the same.
  const char* gc = std::getenv("PPMOE_GATHER_CTAS");
  const int per_sm = (gc && std::atoi(gc) == 2) ? 2 : 1;
  const int lag = per_sm == 2 ? 4 : kGatherLag;
  const int grid = num_sms() * per_sm;
  const int per = (rows_cap + grid - 1) / grid;  // rows per CTA (upper bound)
  const size_t tok_bytes = align_to(static_cast<size_t>(per) * 4, 128);
  const size_t budget = 200 * 1024 / per_sm;
  int R = static_cast<int>((budget - align_to(row_bytes, 128) - 512 - std::min(tok_bytes, budget / 2)) / row_bytes);
  if (R > 32) R = 32;
  if (row_bytes % 16 == 0 && R >= lag + 2 && tok_bytes <= budget / 2) {
    const size_t smem = align_to(static_cast<size_t>(R) * 8, 128) + align_to(row_bytes, 128) + tok_bytes + R * row_bytes;
    if (dtype == kBF16) {
      auto k = per_sm == 2 ? gather_bulk_kernel<__nv_bfloat16, 4> : gather_bulk_kernel<__nv_bfloat16, kGatherLag>;
      PPMOE_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      k<<<grid, kGatherThreads, smem, s>>>(static_cast<const __nv_bfloat16*>(X), H, seg, El, tok_sorted, w_sorted,
                                           static_cast<__nv_bfloat16*>(Xs), tok_local, w_local, R, per);
    } else {
      auto k = per_sm == 2 ? gather_bulk_kernel<float, 4> : gather_bulk_kernel<float, kGatherLag>;
      PPMOE_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      k<<<grid, kGatherThreads, smem, s>>>(static_cast<const float*>(X), H, seg, El, tok_sorted, w_sorted,
                                           static_cast<float*>(Xs), tok_local, w_local, R, per);
    }
    return check_launch("gather_bulk_kernel");
  }
  if (dtype == kBF16)
    gather_warp_kernel<__nv_bfloat16><<<grid * 4, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(X), H, seg, El,
                                                               tok_sorted, w_sorted, static_cast<__nv_bfloat16*>(Xs),
                                                               tok_local, w_local);
  else
    gather_warp_kernel<float><<<grid * 4, 256, 0, s>>>(static_cast<const float*>(X), H, seg, El, tok_sorted, w_sorted,
                                                       static_cast<float*>(Xs), tok_local, w_local);
  return check_launch("gather_warp_kernel");
}

int ppmoe_chunk_rows(const int* tok_local, const int* seg, const int* kept, int El, int N, int C, int* row_lo,
                     int* row_hi, void* stream) {
  PPMOE_REQUIRE(El >= 1 && N >= 0 && C >= 1, "bad chunk_rows arguments El=%d N=%d C=%d", El, N, C);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n = (C + 1) * El;
  chunk_rows_kernel<<<(n + 127) / 128, 128, 0, s>>>(tok_local, seg, kept, El, N, C, row_lo, row_hi);
  return check_launch("chunk_rows_kernel");
}

int ppmoe_combine(int dtype, const void* R, const int* seg, int El, const int* pair_pos, const float* w, int N, int K,
                  int H, const float* dL, const float* Wg, int E, void* out, void* stream) {
  PPMOE_REQUIRE(dtype == kBF16 || dtype == kF32, "bad dtype");
  PPMOE_REQUIRE(N >= 0 && H >= 1 && K >= 1 && El >= 1, "bad combine shape N=%d H=%d K=%d El=%d", N, H, K, El);
  PPMOE_REQUIRE(!dL || (Wg && E >= 1), "the gate term needs Wg and E >= 1");
  if (N == 0) return kOk;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int ctas = num_sms() * 4;
  auto launch_bf16 = [&](auto kern, int cw, int u) {
    const int gx = (H / cw + 255) / 256;
    dim3 grid(gx, max(1, min((N + u - 1) / u, ctas / gx)));
    kern<<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(R), seg, El, pair_pos, w, N, K, H, dL, Wg, E,
                              static_cast<__nv_bfloat16*>(out));
    return check_launch("combine_rows_bf16_kernel");
  };
  if (dtype == kBF16 && !dL && H % 8 == 0) {
    if (K == 2) return launch_bf16(combine_rows_bf16_kernel<0, 8, 4, 2>, 8, 4);
    if (K == 1) return launch_bf16(combine_rows_bf16_kernel<0, 8, 8, 1>, 8, 8);
    return launch_bf16(combine_rows_bf16_kernel<0, 8, 8, 0>, 8, 8);
  }
  const int gx = (H + 255) / 256;
  dim3 grid(gx, max(1, min(N, ctas / gx)));
  if (dtype == kBF16)
    combine_rows_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(R), seg, El, pair_pos, w,
                                                            N, K, H, dL, Wg, E, static_cast<__nv_bfloat16*>(out));
  else
    combine_rows_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(R), seg, El, pair_pos, w, N, K, H, dL, Wg,
                                                    E, static_cast<float*>(out));
  return check_launch("combine_rows_kernel");
}

int ppmoe_dropout_stream(const int* kept, int E, int e0, int El, int H, unsigned long long key0,
                         unsigned long long key1, unsigned long long threshold, unsigned long long first_draw,
                         unsigned long long* desc, void* stream) {
  PPMOE_REQUIRE(E >= 1 && El >= 1 && e0 >= 0 && e0 + El <= E && H >= 1, "bad dropout stream E=%d e0=%d El=%d", E, e0,
                El);
  dropout_stream_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(kept, e0, El, H, key0, key1, threshold,
                                                                         first_draw, desc);
  return check_launch("dropout_stream_kernel");
}

size_t ppmoe_input_grads_workspace_bytes(int dtype, int N, int H, int E) {
  // fused-path partials for any k, or the gate_grads fallback's, whichever is larger
  const size_t fused = static_cast<size_t>(std::max(input_grads_chunks(N, H, E), dwg_chunks(N, H))) * H * E * 4;
  return dtype == kBF16 ? std::max(fused, ppmoe_gate_grad_workspace_bytes(N, H, E))
                        : ppmoe_gate_grad_workspace_bytes(N, H, E);
}

int ppmoe_input_grads(int dtype, const void* dXs, const int* seg, int El, const int* pair_pos, int N, int K, int H,
                      const void* X, const float* dL, const float* Wg, int E, void* dX, float* dWg, void* ws,
                      size_t ws_bytes, void* stream) {
  PPMOE_REQUIRE(dtype == kBF16 || dtype == kF32, "bad dtype");
  PPMOE_REQUIRE(N >= 1 && H >= 1 && K >= 1 && El >= 1 && E >= 1 && E <= 64, "bad input-grad shape N=%d H=%d K=%d E=%d",
                N, H, K, E);
  PPMOE_REQUIRE(!dWg || ws_bytes >= ppmoe_input_grads_workspace_bytes(dtype, N, H, E), "input-grad workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!input_grads_fused(dtype, H, K, E)) {
    if (dX)
      if (int rc = ppmoe_combine(dtype, dXs, seg, El, pair_pos, nullptr, N, K, H, dL, Wg, E, dX, stream)) return rc;
    if (!dWg) return kOk;
    return ppmoe_gate_grads(nullptr, X, dtype, dL, Wg, N, H, E, nullptr, dWg, ws, ws_bytes, stream);
  }
  if (!dX && !dWg) return kOk;
  if (!dX && dwg_bulk_ok(dtype, H, E)) {  // gate-weight gradient alone: X read once at HBM rate
    const int C = dwg_chunks(N, H);
    dim3 grid((H + kDwgSlab - 1) / kDwgSlab, C);
    float* part = static_cast<float*>(ws);
    auto launch = [&](auto kern, size_t smem) {
      PPMOE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      kern<<<grid, kIgConsumers + 32, smem, s>>>(static_cast<const __nv_bfloat16*>(X), dL, N, H, part);
      return check_launch("dwg_bulk_kernel");
    };
    int rc = E == 4 ? launch(dwg_bulk_kernel<4>, DwgGeom<4>::kSmem)
             : E == 8 ? launch(dwg_bulk_kernel<8>, DwgGeom<8>::kSmem) : launch(dwg_bulk_kernel<16>, DwgGeom<16>::kSmem);
    if (rc) return rc;
    const int HE = H * E;
    dwg_reduce_kernel<<<(HE + 255) / 256, 256, 0, s>>>(part, C, HE, static_cast<float*>(dWg));
    return check_launch("dwg_reduce_kernel");
  }
  const int C = input_grads_chunks(N, H, E);
  dim3 grid((H + kIgSlab - 1) / kIgSlab, C);
  float* part = dWg ? static_cast<float*>(ws) : nullptr;
  int rc;
#define PPMOE_IG(EB, KT, MINB) \
  rc = launch_input_grads<EB, KT, MINB>(grid, s, dXs, seg, El, pair_pos, N, H, X, dL, Wg, E, dX, part)
  if (E <= 8) {
    switch (K) {
      case 1: PPMOE_IG(8, 1, 2); break;
      case 2: PPMOE_IG(8, 2, 2); break;
      case 3: PPMOE_IG(8, 3, 2); break;
      default: PPMOE_IG(8, 4, 2); break;
    }
  } else {
    switch (K) {
      case 1: PPMOE_IG(16, 1, 1); break;
      case 2: PPMOE_IG(16, 2, 1); break;
      case 3: PPMOE_IG(16, 3, 1); break;
      default: PPMOE_IG(16, 4, 1); break;
    }
  }
#undef PPMOE_IG
  if (rc) return rc;
  if (dWg) {
    const int HE = H * E;
    dwg_reduce_kernel<<<(HE + 255) / 256, 256, 0, s>>>(part, C, HE, dWg);
    return check_launch("dwg_reduce_kernel");
  }
  return kOk;
}

int ppmoe_cast_out(const float* acc, int n, void* out, int dtype, void* stream) {
  PPMOE_REQUIRE(dtype == kBF16 || dtype == kF32, "bad dtype");
  if (n <= 0) return kOk;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int grid = num_sms() * 4;
  if (dtype == kBF16) cast_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(acc, n, static_cast<__nv_bfloat16*>(out));
  else cast_kernel<float><<<grid, 256, 0, s>>>(acc, n, static_cast<float*>(out));
  return check_launch("cast_kernel");
}

int ppmoe_bwd_dy(int dtype, const void* dOut, const void* Y, const int* seg, int El, int H, int rows_cap,
                 const int* tok_local, const float* w_local, int weight_scaling, float dropout_p,
                 const unsigned long long* drop_stream, void* dY, float* dw, float* dy_colsum_part, void* stream) {
  PPMOE_REQUIRE(dropout_p >= 0.f && dropout_p < 1.f, "dropout probability must be in [0, 1), got %g", dropout_p);
  PPMOE_REQUIRE(dropout_p == 0.f || drop_stream, "dropout needs its stream descriptor (ppmoe_dropout_stream)");
  if (dy_colsum_part) {
    PPMOE_REQUIRE(dtype == kBF16 && H % 256 == 0,
                  "dY column-sum partials need the bf16 path and hidden %% 256 == 0 (H=%d)", H);
    if (rows_cap == 0) return kOk;
    const char* mode = std::getenv("PPMOE_BWD_DY");
    const int cpw = (H + 2047) / 2048;
    const bool cols = !(mode && std::strcmp(mode, "block") == 0) && cpw <= 4;
    if (cols) {
      const int grid = num_sms() * 8;
      cudaStream_t s = static_cast<cudaStream_t>(stream);
      auto* g = static_cast<const __nv_bfloat16*>(dOut);
      auto* y = static_cast<const __nv_bfloat16*>(Y);
      auto* d = static_cast<__nv_bfloat16*>(dY);
      const bool drop = dropout_p > 0.f;
#define PPMOE_DY_COLS(C, D) \
  bwd_dy_cols_kernel<C, D><<<grid, 256, 0, s>>>(g, y, seg, El, H, tok_local, w_local, weight_scaling, dropout_p, \
                                                drop_stream, d, dw, dy_colsum_part)
      if (cpw == 1) {
        if (drop) PPMOE_DY_COLS(1, true); else PPMOE_DY_COLS(1, false);
      } else if (cpw == 2) {
        if (drop) PPMOE_DY_COLS(2, true); else PPMOE_DY_COLS(2, false);
      } else {
        if (drop) PPMOE_DY_COLS(4, true); else PPMOE_DY_COLS(4, false);
      }
#undef PPMOE_DY_COLS
      return check_launch("bwd_dy_cols_kernel");
    }
    auto blk = dropout_p > 0.f ? bwd_dy_block_kernel<true> : bwd_dy_block_kernel<false>;
    blk<<<num_sms() * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const __nv_bfloat16*>(dOut), static_cast<const __nv_bfloat16*>(Y), seg, El, H, tok_local,
        w_local, weight_scaling, dropout_p, drop_stream, static_cast<__nv_bfloat16*>(dY), dw, dy_colsum_part);
    return check_launch("bwd_dy_block_kernel");
  }
  PPMOE_REQUIRE(dtype == kBF16 || dtype == kF32, "bad dtype");
  if (rows_cap == 0) return kOk;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int grid = num_sms() * 8;
  if (dtype == kBF16)
    bwd_dy_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(dOut),
                                                      static_cast<const __nv_bfloat16*>(Y), seg, El, H, tok_local,
                                                      w_local, weight_scaling, dropout_p, drop_stream,
                                                      static_cast<__nv_bfloat16*>(dY), dw);
  else
    bwd_dy_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(dOut), static_cast<const float*>(Y), seg, El, H,
                                              tok_local, w_local, weight_scaling, dropout_p, drop_stream,
                                              static_cast<float*>(dY), dw);
  return check_launch("bwd_dy_kernel");
}

int ppmoe_gate_bwd(const float* scores, const int* idx, const int* pair_pos, const float* dw, const int* seg, int El,
                   const int* counts_top1, int N, int E, int K, const float* aux_grad, float* dL, void* stream) {
  PPMOE_REQUIRE(N >= 1 && E >= 1 && E <= 256 && K >= 1 && K <= E, "bad gate backward shape N=%d E=%d K=%d", N, E, K);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int TT = 256 / E;
  if (TT < 1) TT = 1;
  const int threads = TT * E;
  const int grid = (N + TT - 1) / TT;
  gate_bwd_kernel<<<grid, threads, (TT * E + TT) * 4, s>>>(scores, idx, pair_pos, dw, seg, El, counts_top1, N, E, K,
                                               aux_grad, dL);
  return check_launch("gate_bwd_kernel");
}

size_t ppmoe_gate_grad_workspace_bytes(int N, int H, int E) {
  const size_t C = (static_cast<size_t>(N) + kGradTC - 1) / kGradTC;
  return C * H * E * 4;
}

int ppmoe_gate_grads(const float* dx_acc, const void* X, int dtype, const float* dL, const float* Wg, int N, int H,
                     int E, void* dX, float* dWg, void* ws, size_t ws_bytes, void* stream) {
  PPMOE_REQUIRE(dtype == kBF16 || dtype == kF32, "bad dtype");
  PPMOE_REQUIRE(N >= 1 && H >= 1 && E >= 1 && E <= 64, "gate gradients support 1 <= E <= 64, got E=%d", E);
  PPMOE_REQUIRE(!dWg || ws_bytes >= ppmoe_gate_grad_workspace_bytes(N, H, E), "gate-grad workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int C = (N + kGradTC - 1) / kGradTC;
  float* part = dWg ? static_cast<float*>(ws) : nullptr;
  const int cpt = (H % 2 == 0 && E <= 16) ? 2 : 1;
  dim3 grid((H + 256 * cpt - 1) / (256 * cpt), C);
#define PPMOE_GG(T, EB, CPT)                                                                                    \
  gate_grads_kernel<T, EB, CPT><<<grid, 256, 0, s>>>(dx_acc, static_cast<const T*>(X), dL, Wg, N, H, E,         \
                                                     static_cast<T*>(dX), part)
#define PPMOE_GG_E(T)                                   \
  do {                                                  \
    if (E <= 8) {                                       \
      if (cpt == 2) PPMOE_GG(T, 8, 2);                  \
      else PPMOE_GG(T, 8, 1);                           \
    } else if (E <= 16) {                               \
      if (cpt == 2) PPMOE_GG(T, 16, 2);                 \
      else PPMOE_GG(T, 16, 1);                          \
    } else if (E <= 32) {                               \
      PPMOE_GG(T, 32, 1);                               \
    } else {                                            \
      PPMOE_GG(T, 64, 1);                               \
    }                                                   \
  } while (0)
  if (dtype == kBF16) PPMOE_GG_E(__nv_bfloat16);
  else PPMOE_GG_E(float);
#undef PPMOE_GG_E
#undef PPMOE_GG
  if (int rc = check_launch("gate_grads_kernel")) return rc;
  if (dWg) {
    const int HE = H * E;
    dwg_reduce_kernel<<<(HE + 255) / 256, 256, 0, s>>>(part, C, HE, dWg);
    return check_launch("dwg_reduce_kernel");
  }
  return kOk;
}

}  // extern "C"
