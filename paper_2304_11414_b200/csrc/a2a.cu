// Kernels of the all-to-all expert-parallel comparator (the reference's DPMoE path,
// dpmoe_forward moe.py:363-469): compact send layout, owner-side regrouping map and the
// weighted row scatter-add that restores token order (index_assign, moe.py:461-467).
#include "../../include/ppmoe_capi.h"
#include "common.cuh"
#include "host.h"

namespace ppmoe {

// Compact (unpadded) expert-major layout of this rank's kept pairs: the send buffer of
// the dispatch all-to-all holds rows ordered by destination expert, then token id
// (moe.py:405-414).  Also maps every pair to its compact row.
__global__ void a2a_compact_kernel(const int* __restrict__ tok_sorted, const float* __restrict__ w_sorted,
                                   const int* __restrict__ seg, const int* __restrict__ kept, int E,
                                   const int* __restrict__ idx, const int* __restrict__ pair_pos, int NK,
                                   int* __restrict__ cstart, int* __restrict__ tok_c, float* __restrict__ w_c,
                                   int* __restrict__ pair_pos_c) {
  __shared__ int cs[129];
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int e = 0; e < E; ++e) {
      cs[e] = acc;
      acc += kept[e];
    }
    cs[E] = acc;
  }
  __syncthreads();
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e <= E; e += blockDim.x) cstart[e] = cs[e];
  // pairs -> compact rows
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < NK; i += gridDim.x * blockDim.x) {
    const int p = pair_pos[i];
    const int e = idx[i];
    pair_pos_c[i] = p < 0 ? -1 : cs[e] + (p - seg[e]);
  }
  // rows of every expert
  for (int e = 0; e < E; ++e) {
    const int n = kept[e];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
      tok_c[cs[e] + j] = tok_sorted[seg[e] + j];
      if (w_c) w_c[cs[e] + j] = w_sorted ? w_sorted[seg[e] + j] : 1.f;
    }
  }
}

// Owner side: rows arrive source-major (per source, its rows for my local experts in
// expert order).  Regroup them expert-major with sources in rank order (concat_rows of
// the gathered sections, moe.py:426-447), each expert segment padded to 128 rows.
__global__ void a2a_owner_layout_kernel(const int* __restrict__ recv_counts, int T, int El, int rows_cap,
                                        int* __restrict__ seg_out, int* __restrict__ map) {
  extern __shared__ int sh[];
  int* src_start = sh;             // [T][El] start row in the receive buffer
  int* own_start = sh + T * El;    // [El][T] start row in the owner layout
  int* segs = own_start + T * El;  // [El+1]
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int s = 0; s < T; ++s)
      for (int e = 0; e < El; ++e) {
        src_start[s * El + e] = acc;
        acc += recv_counts[s * El + e];
      }
    int o = 0;
    for (int e = 0; e < El; ++e) {
      segs[e] = o;
      int run = o;
      for (int s = 0; s < T; ++s) {
        own_start[e * T + s] = run;
        run += recv_counts[s * El + e];
      }
      o += (run - o + 127) / 128 * 128;
    }
    segs[El] = o;
  }
  __syncthreads();
  for (int e = threadIdx.x; e <= El; e += blockDim.x) seg_out[e] = segs[e];
  for (int r = threadIdx.x; r < rows_cap; r += blockDim.x) map[r] = -1;  // incl. rows past seg[El]
  __syncthreads();
  for (int e = 0; e < El; ++e)
    for (int s = 0; s < T; ++s) {
      const int n = recv_counts[s * El + e];
      const int o = own_start[e * T + s], src = src_start[s * El + e];
      for (int j = threadIdx.x; j < n; j += blockDim.x)
        if (o + j < rows_cap) map[o + j] = src + j;
    }
}

// dst[tok[r]] += w[r] * src[r] for the first nrows[0] rows (tok < 0 skipped).
template <typename T>
__global__ void scatter_rows_kernel(const T* __restrict__ src, int H, const int* __restrict__ nrows,
                                    const int* __restrict__ tok, const float* __restrict__ w, float* __restrict__ dst) {
  const int rows = nrows[0];
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x / 32;
  const bool vec = (H % 8) == 0;
  for (int r = blockIdx.x * wpb + (threadIdx.x >> 5); r < rows; r += gridDim.x * wpb) {
    const int t = tok[r];
    if (t < 0) continue;
    const float s = w ? w[r] : 1.f;
    const T* a = src + static_cast<size_t>(r) * H;
    float* d = dst + static_cast<size_t>(t) * H;
    if (vec && sizeof(T) == 2) {
      for (int j = lane * 8; j < H; j += 256) {
        const uint4 u = *reinterpret_cast<const uint4*>(a + j);
        const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&u);
        float f[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 v = __bfloat1622float2(hv[i]);
          f[2 * i] = v.x;
          f[2 * i + 1] = v.y;
        }
        red_add_v4(d + j, s * f[0], s * f[1], s * f[2], s * f[3]);
        red_add_v4(d + j + 4, s * f[4], s * f[5], s * f[6], s * f[7]);
      }
    } else {
      for (int j = lane; j < H; j += 32) atomicAdd(d + j, s * to_f32(a[j]));
    }
  }
}

// dst[map[o]] = src[o] for owner rows o < rows with map[o] >= 0: expert outputs / per-row
// input gradients from the owner's expert-major layout back to receive order (a
// permutation: plain 16-byte row copies, no atomics, no fp32 staging).
__global__ void permute_rows_kernel(const uint4* __restrict__ src, int vec_per_row, int rows,
                                    const int* __restrict__ map, uint4* __restrict__ dst) {
  const int wpb = blockDim.x / 32;
  const int lane = threadIdx.x & 31;
  for (int o = blockIdx.x * wpb + (threadIdx.x >> 5); o < rows; o += gridDim.x * wpb) {
    const int r = map[o];
    if (r < 0) continue;
    const uint4* a = src + static_cast<size_t>(o) * vec_per_row;
    uint4* d = dst + static_cast<size_t>(r) * vec_per_row;
    for (int j = lane; j < vec_per_row; j += 32) d[j] = a[j];
  }
}

}  // namespace ppmoe

using namespace ppmoe;

extern "C" {

int ppmoe_a2a_compact(const int* tok_sorted, const float* w_sorted, const int* seg, const int* kept, int E,
                      const int* idx, const int* pair_pos, int NK, int* cstart, int* tok_c, float* w_c,
                      int* pair_pos_c, void* stream) {
  PPMOE_REQUIRE(E >= 1 && E <= 128 && NK >= 0, "bad a2a_compact arguments E=%d NK=%d", E, NK);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int grid = num_sms();
  a2a_compact_kernel<<<grid, 256, 0, s>>>(tok_sorted, w_sorted, seg, kept, E, idx, pair_pos, NK, cstart, tok_c, w_c,
                                          pair_pos_c);
  return check_launch("a2a_compact_kernel");
}

int ppmoe_a2a_owner_layout(const int* recv_counts, int T, int El, int rows_cap, int* seg_out, int* map,
                           void* stream) {
  PPMOE_REQUIRE(T >= 1 && El >= 1 && T * El <= 4096, "bad owner layout T=%d El=%d", T, El);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t smem = (2 * static_cast<size_t>(T) * El + El + 1) * 4;
  a2a_owner_layout_kernel<<<1, 1024, smem, s>>>(recv_counts, T, El, rows_cap, seg_out, map);
  return check_launch("a2a_owner_layout_kernel");
}

int ppmoe_a2a_permute_rows(const void* src, int dtype, int H, int rows, const int* map, void* dst, void* stream) {
  PPMOE_REQUIRE(dtype == kBF16 || dtype == kF32, "bad dtype");
  const size_t row_bytes = static_cast<size_t>(H) * (dtype == kBF16 ? 2 : 4);
  PPMOE_REQUIRE(H >= 1 && row_bytes % 16 == 0 && rows >= 0, "permute_rows needs 16-byte rows (H=%d)", H);
  if (rows == 0) return kOk;
  const int grid = num_sms() * 4;
  permute_rows_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(src), static_cast<int>(row_bytes / 16), rows, map, static_cast<uint4*>(dst));
  return check_launch("permute_rows_kernel");
}

int ppmoe_scatter_rows(const void* src, int dtype, int H, const int* nrows, const int* tok, const float* w, float* dst,
                       void* stream) {
  PPMOE_REQUIRE(dtype == kBF16 || dtype == kF32, "bad dtype");
  PPMOE_REQUIRE(H >= 1, "bad width");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int grid = num_sms() * 4;
  if (dtype == kBF16)
    scatter_rows_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(src), H, nrows, tok, w,
                                                            dst);
  else
    scatter_rows_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(src), H, nrows, tok, w, dst);
  return check_launch("scatter_rows_kernel");
}

}  // extern "C"
