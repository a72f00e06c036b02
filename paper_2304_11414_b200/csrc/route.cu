// Routing and dispatch plan.
//
//  router_kernel    gate GEMV (fp64 accumulation of exact bf16/fp32 x fp32 products),
//                   fp64 softmax, top-k by repeated argmax (lowest id wins ties),
//                   per-block expert score sums and top-1 counts for the aux loss.
//                   Reference: gate_top1 moe.py:196-208, softmax tensor.py:212-223,
//                   aux_loss moe.py:211-223.
//  plan_*           stable counting sort of (token, slot) pairs by expert with the
//                   capacity rule, into 128-row padded segments.
//                   Reference: build_dispatch_plan moe.py:226-235, _capacity_mask
//                   moe.py:345-360.
//
// Everything is deterministic: integer histograms (exact under atomics), fixed-order
// fp64 reductions for the aux loss.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>

#include "../../include/ppmoe_capi.h"
#include "common.cuh"
#include "host.h"

namespace ppmoe {

constexpr int kRouteThreads = 256;
constexpr int kRouteTB = 32;    // tokens per block (512 blocks at 16K tokens: >3 per SM)
constexpr int kRouteTPT = 2;    // tokens per thread (each staged Wg value feeds 2 tokens)
constexpr int kRouteKS = 16;    // hidden-dimension splits per token (threads per token pair)
constexpr int kRouteHC = 512;   // hidden chunk of Wg staged as fp64 in shared memory
constexpr int kChunk = 256;     // tokens per plan chunk (one thread per token)
constexpr int kMaxE = 128;
constexpr int kMaxK = 8;

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Exact fp32 -> fp64 widening with integer ops (keeps the conversions off the FP64
// pipe, which the logit FMAs saturate).  Zero/subnormal/inf/nan take the F2F path.
__device__ __forceinline__ double f32bits_to_f64(uint32_t b) {
  const uint32_t ex = (b >> 23) & 0xFFu;
  if (ex == 0u || ex == 0xFFu) return static_cast<double>(__uint_as_float(b));
  const unsigned long long bits = (static_cast<unsigned long long>(b >> 31) << 63) |
                                  (static_cast<unsigned long long>(ex + 896u) << 52) |
                                  (static_cast<unsigned long long>(b & 0x7FFFFFu) << 29);
  return __longlong_as_double(static_cast<long long>(bits));
}

template <typename T>
__device__ __forceinline__ void load8_f64(const T* p, double* dst);
// bf16 bits -> fp64: sign | (exponent+896, mantissa) moved into the high word.  Zero,
// subnormal, inf and nan (exponent field 0 or 255) take the exact F2F path.
__device__ __forceinline__ double bf16bits_to_f64(uint32_t b) {
  const uint32_t m = b & 0x7FFFu;
  if (m - 0x80u >= 0x7F00u) return static_cast<double>(__uint_as_float(b << 16));
  const uint32_t hi = ((b & 0x8000u) << 16) | ((m << 13) + 0x38000000u);
  return __hiloint2double(static_cast<int>(hi), 0);
}

template <>
__device__ __forceinline__ void load8_f64<__nv_bfloat16>(const __nv_bfloat16* p, double* dst) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    dst[2 * i] = bf16bits_to_f64(w[i] & 0xFFFFu);
    dst[2 * i + 1] = bf16bits_to_f64(w[i] >> 16);
  }
}

template <typename T>
__device__ __forceinline__ uint4 ldg16(const T* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

template <typename T>
__device__ __forceinline__ void widen8(const uint4* u, double* dst);
// Branch-free exact widening of 8 bf16 values; zero handled by a select.  Subnormal and
// inf/nan inputs (exponent field 0 with a nonzero mantissa, or 255) are detected once per
// group and redone with F2F on a warp-uniform slow path (they never occur for finite
// activations, but exactness must not depend on that).
template <>
__device__ __forceinline__ void widen8<__nv_bfloat16>(const uint4* u, double* dst) {
  const uint32_t w[4] = {u->x, u->y, u->z, u->w};
  uint32_t special = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int hlf = 0; hlf < 2; ++hlf) {
      const uint32_t b = hlf ? (w[i] >> 16) : (w[i] & 0xFFFFu);
      const uint32_t m = b & 0x7FFFu;
      special |= (m - 1u < 0x7Fu) | (m >= 0x7F80u);
      const uint32_t mag = m ? (m << 13) + 0x38000000u : 0u;
      dst[2 * i + hlf] = __hiloint2double(static_cast<int>(((b & 0x8000u) << 16) | mag), 0);
    }
  }
  if (__any_sync(__activemask(), special)) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      dst[2 * i] = static_cast<double>(__uint_as_float(w[i] << 16));
      dst[2 * i + 1] = static_cast<double>(__uint_as_float(w[i] & 0xFFFF0000u));
    }
  }
}
template <>
__device__ __forceinline__ void widen8<float>(const uint4* u, double* dst) {
  dst[0] = f32bits_to_f64(u[0].x); dst[1] = f32bits_to_f64(u[0].y); dst[2] = f32bits_to_f64(u[0].z);
  dst[3] = f32bits_to_f64(u[0].w); dst[4] = f32bits_to_f64(u[1].x); dst[5] = f32bits_to_f64(u[1].y);
  dst[6] = f32bits_to_f64(u[1].z); dst[7] = f32bits_to_f64(u[1].w);
}
template <>
__device__ __forceinline__ void load8_f64<float>(const float* p, double* dst) {
  const uint4 a = *reinterpret_cast<const uint4*>(p);
  const uint4 b = *reinterpret_cast<const uint4*>(p + 4);
  dst[0] = f32bits_to_f64(a.x); dst[1] = f32bits_to_f64(a.y); dst[2] = f32bits_to_f64(a.z); dst[3] = f32bits_to_f64(a.w);
  dst[4] = f32bits_to_f64(b.x); dst[5] = f32bits_to_f64(b.y); dst[6] = f32bits_to_f64(b.z); dst[7] = f32bits_to_f64(b.w);
}

__host__ __device__ inline int route_eb(int E) { return E <= 8 ? 8 : 16; }

__host__ inline size_t route_smem_bytes(int E) {
  const int EB = route_eb(E);
  // staged Wg chunk (fp64), reused for the split-K partials (KS*TB == HC)
  return static_cast<size_t>(kRouteHC) * EB * 8 + static_cast<size_t>(kRouteTB) * E * 8 + 2 * kRouteTB * 8;
}

// Softmax (fp64), top-k and the per-block aux-loss sums of the kRouteTB tokens of this
// block from their logits lg[TB][E] (shared by the router kernels).
__device__ __forceinline__ void route_tail(double* lg, double* stat, int t0, int N, int E, int K,
                                           const int* __restrict__ ovr, int* __restrict__ idx, float* __restrict__ w,
                                           float* __restrict__ scores, double* __restrict__ ssum,
                                           int* __restrict__ cnt_top1) {
  const int tid = threadIdx.x;
  __syncthreads();
  // softmax statistics (row max shift, tensor.py:214-216)
  if (tid < kRouteTB) {
    const double* l = lg + tid * E;
    double mx = l[0];
    for (int j = 1; j < E; ++j) mx = fmax(mx, l[j]);
    double s = 0.0;
    for (int j = 0; j < E; ++j) s += exp(l[j] - mx);
    stat[2 * tid] = mx;
    stat[2 * tid + 1] = s;
  }
  __syncthreads();
  for (int i = tid; i < kRouteTB * E; i += blockDim.x) {
    const int tl = i / E, e = i % E;
    const double sc = exp(lg[i] - stat[2 * tl]) / stat[2 * tl + 1];
    lg[i] = sc;
    if (t0 + tl < N) scores[static_cast<size_t>(t0 + tl) * E + e] = static_cast<float>(sc);
  }
  __syncthreads();
  // top-k selection, one thread per token
  if (tid < kRouteTB && t0 + tid < N) {
    const int tt = t0 + tid;
    const double* sc = lg + tid * E;
    unsigned long long chosen[2] = {0ull, 0ull};
    for (int s = 0; s < K; ++s) {
      int best;
      if (ovr) {
        best = ovr[static_cast<size_t>(tt) * K + s];
      } else {
        best = -1;
        for (int j = 0; j < E; ++j) {
          if ((chosen[j >> 6] >> (j & 63)) & 1ull) continue;
          if (best < 0 || sc[j] > sc[best]) best = j;
        }
        chosen[best >> 6] |= 1ull << (best & 63);
      }
      idx[static_cast<size_t>(tt) * K + s] = best;
      w[static_cast<size_t>(tt) * K + s] = static_cast<float>(sc[best]);
      if (s == 0) atomicAdd(&cnt_top1[best], 1);
    }
  }
  // per-block expert score sums in token order (deterministic aux-loss reduction)
  for (int e = tid; e < E; e += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < kRouteTB && t0 + r < N; ++r) s += lg[r * E + e];
    ssum[static_cast<size_t>(blockIdx.x) * E + e] = s;
  }
}

// Gate logits X*Wg in fp64 (bf16/fp32 x fp32 products are exact in fp64), softmax,
// top-k and aux-loss partials.  Block: 64 tokens; thread = (2 tokens, 1 of 8 hidden
// splits); experts in register passes of EB.  Every lane of a warp reads the same
// staged Wg value (shared-memory broadcast).
template <typename T, int EB>
__global__ void __launch_bounds__(kRouteThreads, EB == 8 ? 2 : 1) router_kernel(const T* __restrict__ X, const float* __restrict__ Wg,
                                                               int N, int H, int E, int K, const int* __restrict__ ovr,
                                                               int* __restrict__ idx, float* __restrict__ w,
                                                               float* __restrict__ scores, double* __restrict__ ssum,
                                                               int* __restrict__ cnt_top1) {
  extern __shared__ __align__(16) unsigned char sm[];
  static_assert(kRouteKS * kRouteTB == kRouteHC, "split-K partials alias the Wg staging buffer");
  double* wsm = reinterpret_cast<double*>(sm);                 // [HC][EB]
  double* part = wsm;                                          // [KS][TB][EB] (after the last chunk)
  double* lg = wsm + kRouteHC * EB;                            // [TB][E]
  double* stat = lg + kRouteTB * E;                            // [TB][2]
  const int tid = threadIdx.x;
  const int ks = tid >> 4;                  // half-warp = one hidden split
  const int tl0 = tid & 15, tl1 = tl0 + 16;  // the thread's two tokens (block-local)
  const int t0 = blockIdx.x * kRouteTB;
  const bool ok0 = t0 + tl0 < N, ok1 = t0 + tl1 < N;
  const T* x0 = X + static_cast<size_t>(ok0 ? t0 + tl0 : 0) * H;
  const T* x1 = X + static_cast<size_t>(ok1 ? t0 + tl1 : 0) * H;

  const bool fast = (H % kRouteHC) == 0;  // whole chunks: software-pipelined path
  for (int e0 = 0; e0 < E; e0 += EB) {
    double a0[EB], a1[EB];
#pragma unroll
    for (int j = 0; j < EB; ++j) a0[j] = a1[j] = 0.0;
    if (fast) {
      // Each thread owns kSpan hidden columns of every chunk (kG groups of 8).  The x loads
      // of chunk c+1 and its Wg values are issued while chunk c computes, so HBM latency
      // overlaps the FP64 FMAs instead of draining at every chunk barrier.
      constexpr int kSpan = kRouteHC / kRouteKS;
      constexpr int kG = kSpan / 8;
      constexpr int kU = sizeof(T) == 2 ? 1 : 2;  // uint4 per 8 values
      constexpr int kWPer = kRouteHC * EB / kRouteThreads;
      const int nch = H / kRouteHC;
      uint4 sa[kG][kU], sb[kG][kU];
      float wnext[kWPer];
      auto load_x = [&](int c) {
#pragma unroll
        for (int u = 0; u < kG; ++u)
#pragma unroll
          for (int q = 0; q < kU; ++q) {
            const int off = c * kRouteHC + ks * kSpan + 8 * u + 4 * q;
            sa[u][q] = ok0 ? ldg16(x0 + off) : make_uint4(0, 0, 0, 0);
            sb[u][q] = ok1 ? ldg16(x1 + off) : make_uint4(0, 0, 0, 0);
          }
      };
      auto load_w = [&](int c) {
#pragma unroll
        for (int r = 0; r < kWPer; ++r) {
          const int i = tid + r * kRouteThreads;
          const int cc = i / EB, j = i % EB;
          wnext[r] = e0 + j < E ? __ldg(Wg + static_cast<size_t>(c * kRouteHC + cc) * E + e0 + j) : 0.f;
        }
      };
      load_x(0);
      load_w(0);
      for (int c = 0; c < nch; ++c) {
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kWPer; ++r) wsm[tid + r * kRouteThreads] = static_cast<double>(wnext[r]);
        __syncthreads();
        if (c + 1 < nch) load_w(c + 1);
#pragma unroll
        for (int u = 0; u < kG; ++u) {
          double xa[8], xb[8];
          widen8<T>(sa[u], xa);
          widen8<T>(sb[u], xb);
          if (c + 1 < nch) {  // refill this slot with the next chunk's group
#pragma unroll
            for (int q = 0; q < kU; ++q) {
              const int off = (c + 1) * kRouteHC + ks * kSpan + 8 * u + 4 * q;
              sa[u][q] = ok0 ? ldg16(x0 + off) : make_uint4(0, 0, 0, 0);
              sb[u][q] = ok1 ? ldg16(x1 + off) : make_uint4(0, 0, 0, 0);
            }
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const double* wr = wsm + (ks * kSpan + 8 * u + i) * EB;
#pragma unroll
            for (int j = 0; j < EB; j += 2) {
              const double2 wv = *reinterpret_cast<const double2*>(wr + j);
              a0[j] = fma(xa[i], wv.x, a0[j]);
              a0[j + 1] = fma(xa[i], wv.y, a0[j + 1]);
              a1[j] = fma(xb[i], wv.x, a1[j]);
              a1[j + 1] = fma(xb[i], wv.y, a1[j + 1]);
            }
          }
        }
      }
    } else {
      for (int h0 = 0; h0 < H; h0 += kRouteHC) {
        const int hc = min(kRouteHC, H - h0);
        __syncthreads();
        for (int i = tid; i < hc * EB; i += kRouteThreads) {
          const int c = i / EB, j = i % EB;
          wsm[i] = e0 + j < E ? static_cast<double>(Wg[static_cast<size_t>(h0 + c) * E + e0 + j]) : 0.0;
        }
        __syncthreads();
        for (int c = ks; c < hc; c += kRouteKS) {
          const double xa = ok0 ? static_cast<double>(to_f32(x0[h0 + c])) : 0.0;
          const double xb = ok1 ? static_cast<double>(to_f32(x1[h0 + c])) : 0.0;
#pragma unroll
          for (int j = 0; j < EB; ++j) {
            a0[j] = fma(xa, wsm[c * EB + j], a0[j]);
            a1[j] = fma(xb, wsm[c * EB + j], a1[j]);
          }
        }
      }
    }
    // deterministic split-K reduction: ks = 0..KS-1 in order
    __syncthreads();  // partials alias the Wg staging buffer
#pragma unroll
    for (int j = 0; j < EB; ++j) {
      part[(ks * kRouteTB + tl0) * EB + j] = a0[j];
      part[(ks * kRouteTB + tl1) * EB + j] = a1[j];
    }
    __syncthreads();
    for (int i = tid; i < kRouteTB * EB; i += kRouteThreads) {
      const int tl = i / EB, j = i % EB;
      if (e0 + j >= E) continue;
      double s = 0.0;
      for (int q = 0; q < kRouteKS; ++q) s += part[(q * kRouteTB + tl) * EB + j];
      lg[tl * E + e0 + j] = s;
    }
    __syncthreads();  // the next expert pass restages Wg over the partials
  }
  route_tail(lg, stat, t0, N, E, K, ovr, idx, w, scores, ssum, cnt_top1);
}

// One FP64 tensor-core MMA (DMMA 8x8x4, IEEE fp64): d += a (8x4, row) * b (4x8, col).
// Fragments: lane l holds a = A[l/4][l%4], b = B[l%4][l/4], d = D[l/4][2(l%4) + {0,1}].
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// Gate logits X*Wg on the FP64 tensor cores, then the shared softmax / top-k / aux tail.
// bf16 activations and fp32 gate weights widen exactly to fp64, so every product is exact
// and the only rounding is fp64 accumulation (as in the fp64 oracle, up to order).  A block
// owns kRouteTB = 32 tokens (4 groups of 8 = the MMA's M) x EB experts (n-tiles of 8); its 8
// warps split the hidden dimension and their partial logits are summed in a fixed order in
// shared memory (deterministic).  MMA k-step j of a 32-column chunk maps k-index q to column
// c0 + 8q + j, so a lane's A values for all 8 steps come from ONE 16-byte load of its token
// row (x[t][c0+8q .. c0+8q+7]) and its B values are Wg[c0+8q+j][n] (L1-resident).
// FP64 FMA work moves from 2 DFMA warp-instructions per 64 FMAs to one DMMA per 256.
// Exact bf16 -> fp64 of the 16-bit pattern b (normal numbers and zero; the caller routes
// subnormal / inf / nan groups through the F2F path).
__device__ __forceinline__ double bf16_fast_f64(uint32_t b) {
  const uint32_t m = b & 0x7FFFu;
  const uint32_t mag = m ? (m << 13) + 0x38000000u : 0u;
  return __hiloint2double(static_cast<int>(((b & 0x8000u) << 16) | mag), 0);
}
__device__ __forceinline__ bool bf16x8_special(const uint4& u) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
  uint32_t sp = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t lo = w[i] & 0x7FFFu, hi = (w[i] >> 16) & 0x7FFFu;
    sp |= (lo - 1u < 0x7Fu) | (lo >= 0x7F80u) | (hi - 1u < 0x7Fu) | (hi >= 0x7F80u);
  }
  return sp != 0;
}

template <int EB, int W, int MINB>
__global__ void __launch_bounds__(32 * W, MINB) router_dmma_kernel(const __nv_bfloat16* __restrict__ X,
                                                             const float* __restrict__ Wg, int N, int H, int E, int K,
                                                             const int* __restrict__ ovr, int* __restrict__ idx,
                                                             float* __restrict__ w, float* __restrict__ scores,
                                                             double* __restrict__ ssum, int* __restrict__ cnt_top1) {
  constexpr int NT = EB / 8;
  constexpr int G = kRouteTB / 8;
  extern __shared__ __align__(16) unsigned char sm[];
  double* part = reinterpret_cast<double*>(sm);  // [W][G][NT][32][2]
  double* lg = part + W * G * NT * 64;           // [TB][E]
  double* stat = lg + kRouteTB * E;              // [TB][2]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int t0 = blockIdx.x * kRouteTB;
  const int span = H / W;  // columns per warp (H % (32 W) == 0)
  const int cw0 = warp * span;
  double acc[G][NT][2];
#pragma unroll
  for (int gi = 0; gi < G; ++gi)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[gi][nt][0] = acc[gi][nt][1] = 0.0;
  const size_t xoff = static_cast<size_t>(8 * q);
  auto row_ptr = [&](int gi) {
    const int t = t0 + gi * 8 + g;
    return X + static_cast<size_t>(t < N ? t : 0) * H + xoff;
  };
  auto load_x = [&](int gi, int c) {
    return t0 + gi * 8 + g < N ? ldg16(row_ptr(gi) + c) : make_uint4(0, 0, 0, 0);
  };
  uint4 xa[G];
#pragma unroll
  for (int gi = 0; gi < G; ++gi) xa[gi] = load_x(gi, cw0);
  for (int c0 = cw0; c0 < cw0 + span; c0 += 32) {
    uint4 xn[G];
    const bool more = c0 + 32 < cw0 + span;
#pragma unroll
    for (int gi = 0; gi < G; ++gi) xn[gi] = more ? load_x(gi, c0 + 32) : make_uint4(0, 0, 0, 0);
    double b[NT][8];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int e = nt * 8 + g;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        b[nt][j] = e < E ? static_cast<double>(__ldg(Wg + static_cast<size_t>(c0 + 8 * q + j) * E + e)) : 0.0;
    }
    bool sp = false;
#pragma unroll
    for (int gi = 0; gi < G; ++gi) sp |= bf16x8_special(xa[gi]);
    const bool slow = __any_sync(0xffffffffu, sp);  // warp-uniform: subnormal/inf/nan take F2F
    // k-step j outermost: the G*NT accumulator chains are independent, so consecutive DMMAs
    // never wait on each other's result
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        const uint32_t word = j < 2 ? xa[gi].x : j < 4 ? xa[gi].y : j < 6 ? xa[gi].z : xa[gi].w;
        const uint32_t bits = (j & 1) ? (word >> 16) : (word & 0xFFFFu);
        const double a = slow ? static_cast<double>(__uint_as_float(bits << 16)) : bf16_fast_f64(bits);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma884(acc[gi][nt], a, b[nt][j]);
      }
    }
#pragma unroll
    for (int gi = 0; gi < G; ++gi) xa[gi] = xn[gi];
  }
#pragma unroll
  for (int gi = 0; gi < G; ++gi)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      double* p = part + ((((warp * G + gi) * NT + nt) * 32) + lane) * 2;
      p[0] = acc[gi][nt][0];
      p[1] = acc[gi][nt][1];
    }
  __syncthreads();
  for (int o = threadIdx.x; o < kRouteTB * E; o += blockDim.x) {  // split-K sum, warp order
    const int tl = o / E, e = o % E;
    const int gi = tl >> 3, ln = (tl & 7) * 4 + ((e & 7) >> 1), nt = e >> 3, i = e & 1;
    double v = 0.0;
#pragma unroll
    for (int ww = 0; ww < W; ++ww) v += part[((((ww * G + gi) * NT + nt) * 32) + ln) * 2 + i];
    lg[tl * E + e] = v;
  }
  route_tail(lg, stat, t0, N, E, K, ovr, idx, w, scores, ssum, cnt_top1);
}

constexpr int kRouteDmmaMaxWarps = 8;  // warps per 32-token block (hidden-dimension split)

__host__ inline size_t route_dmma_smem_bytes(int E, int W) {
  const int NT = E <= 8 ? 1 : 2;
  return static_cast<size_t>(W) * (kRouteTB / 8) * NT * 64 * 8 + static_cast<size_t>(kRouteTB) * E * 8 +
         2 * kRouteTB * 8;
}

// ------------------------------------------------------------------ tensor-core router
//
// Gate logits on the bf16 tensor cores with a rigorous error bound, exact fp64 for the rest.
// Wg (fp32) is split exactly into three bf16 pieces w = w1 + w2 + w3 (8 significant bits
// each), so every product x * w_p of a bf16 activation is exact in fp32; mma.sync
// m16n8k16 accumulates 32 columns in fp32 per piece, then the pieces are summed and folded
// into fp64 (so fp32 accumulation error stays local to 32 columns).  A fourth MMA with |x|
// and |w1| gives A_te = sum |x||w| per (token, expert), and the logit error is bounded by
// kRouteTcBound * A_te: 2 MMAs x (16 + 1) roundings of at most 2^-23 relative per fold,
// the piece sum and the |w1| vs |w| slack, times a safety factor of 4.  A token is routed
// from the approximate logits only if every adjacent gap among its top-(k+1) logits exceeds
// the sum of the two bounds (then the top-k set and slot order equal the exact ones);
// otherwise it is queued and router_fix_kernel routes it with fp64 arithmetic throughout.
constexpr double kRouteTcBound = 4.0 * 40.0 * 1.0078125 / 8388608.0;  // 4 * 40 * 2^-23 * (1 + 2^-7)
constexpr int kFinalizeThreads = 512;
constexpr int kRouteTcWarps = 4;  // warps per 16-token block (hidden-dimension split)

__device__ __forceinline__ void hmma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// w = p1 + p2 + p3 exactly (bf16 pieces, returned as raw 16-bit patterns)
__device__ __forceinline__ void split3(float w, uint32_t& p1, uint32_t& p2, uint32_t& p3) {
  const __nv_bfloat16 h1 = __float2bfloat16_rn(w);
  const float r1 = w - __bfloat162float(h1);
  const __nv_bfloat16 h2 = __float2bfloat16_rn(r1);
  const float r2 = r1 - __bfloat162float(h2);
  const __nv_bfloat16 h3 = __float2bfloat16_rn(r2);
  p1 = __bfloat16_as_ushort(h1);
  p2 = __bfloat16_as_ushort(h2);
  p3 = __bfloat16_as_ushort(h3);
}

// Exact routing of the queued tokens (the tensor-core router wrote its best guess and counted
// its top-1; both are corrected here, and the last fixer of a 16-token block rewrites the
// block's aux partial from the final scores): one kFixThreads block per token (grid-stride over
// the queue).  Thread i takes columns i, i + kFixThreads, ... four at a time with every load of
// the four issued up front (one memory round trip per four columns), fp64 logits from exact
// widening, fixed-order warp + block reduction (deterministic), fp64 softmax, top-k by argmax.
constexpr int kFixThreads = 512;
template <int EB>
__global__ void __launch_bounds__(kFixThreads) router_fix_kernel(const __nv_bfloat16* __restrict__ X,
                                                                 const float* __restrict__ Wg, int N, int H, int E,
                                                                 int K, const int* __restrict__ fix_list,
                                                                 const int* __restrict__ fix_count,
                                                                 int* __restrict__ idx, float* __restrict__ w,
                                                                 float* __restrict__ scores, int* __restrict__ cnt_top1,
                                                                 int* __restrict__ pending, double* __restrict__ ssum) {
  constexpr int U = 4;
  constexpr int NW = kFixThreads / 32;
  __shared__ double red[NW][EB];
  __shared__ double lgt[EB], ex[EB];
  __shared__ float tile[16][EB];
  __shared__ int last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int count = *fix_count;
  const unsigned short* xs = reinterpret_cast<const unsigned short*>(X);
  for (int i = blockIdx.x; i < count; i += gridDim.x) {
    const int t = fix_list[i];
    const unsigned short* xr = xs + static_cast<size_t>(t) * H;
    double a[EB];
#pragma unroll
    for (int e = 0; e < EB; ++e) a[e] = 0.0;
    for (int c0 = threadIdx.x; c0 < H; c0 += kFixThreads * U) {
      float xv[U];
      float4 wv[U][EB / 4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * kFixThreads;
        const bool ok = c < H;
        xv[u] = ok ? __uint_as_float(static_cast<uint32_t>(__ldg(xr + c)) << 16) : 0.f;
        const float* wr = Wg + static_cast<size_t>(ok ? c : 0) * E;
#pragma unroll
        for (int e4 = 0; e4 < EB / 4; ++e4) {
          if (E == EB) {  // whole rows: 16-byte loads
            wv[u][e4] = __ldg(reinterpret_cast<const float4*>(wr) + e4);
          } else {
            const int e = 4 * e4;
            wv[u][e4] = make_float4(e < E ? __ldg(wr + e) : 0.f, e + 1 < E ? __ldg(wr + e + 1) : 0.f,
                                    e + 2 < E ? __ldg(wr + e + 2) : 0.f, e + 3 < E ? __ldg(wr + e + 3) : 0.f);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double x = static_cast<double>(xv[u]);
#pragma unroll
        for (int e4 = 0; e4 < EB / 4; ++e4) {
          a[4 * e4] = fma(x, static_cast<double>(wv[u][e4].x), a[4 * e4]);
          a[4 * e4 + 1] = fma(x, static_cast<double>(wv[u][e4].y), a[4 * e4 + 1]);
          a[4 * e4 + 2] = fma(x, static_cast<double>(wv[u][e4].z), a[4 * e4 + 2]);
          a[4 * e4 + 3] = fma(x, static_cast<double>(wv[u][e4].w), a[4 * e4 + 3]);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < EB; ++e) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a[e] += __shfl_xor_sync(0xffffffffu, a[e], o);
      if (lane == 0) red[warp][e] = a[e];
    }
    __syncthreads();
    if (threadIdx.x < E) {  // fixed-order block sum; then exps and divisions one expert per thread
      double v = 0.0;
      for (int ww = 0; ww < NW; ++ww) v += red[ww][threadIdx.x];
      lgt[threadIdx.x] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double mx = lgt[0];
      for (int e = 1; e < E; ++e) mx = fmax(mx, lgt[e]);
      red[0][0] = mx;
    }
    __syncthreads();
    if (threadIdx.x < E) ex[threadIdx.x] = exp(lgt[threadIdx.x] - red[0][0]);
    __syncthreads();
    if (threadIdx.x == 0) {
      double sum = 0.0;
      for (int e = 0; e < E; ++e) sum += ex[e];
      red[0][1] = sum;
    }
    __syncthreads();
    if (threadIdx.x < E) {
      const float sc = static_cast<float>(ex[threadIdx.x] / red[0][1]);
      scores[static_cast<size_t>(t) * E + threadIdx.x] = sc;
      ex[threadIdx.x] = sc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned used = 0;
      for (int s2 = 0; s2 < K; ++s2) {
        int best = -1;
        for (int e = 0; e < E; ++e) {
          if ((used >> e) & 1u) continue;
          if (best < 0 || lgt[e] > lgt[best]) best = e;
        }
        used |= 1u << best;
        if (s2 == 0 && idx[static_cast<size_t>(t) * K] != best) {  // the queued top-1 guess was wrong
          atomicSub(&cnt_top1[idx[static_cast<size_t>(t) * K]], 1);
          atomicAdd(&cnt_top1[best], 1);
        }
        idx[static_cast<size_t>(t) * K + s2] = best;
        w[static_cast<size_t>(t) * K + s2] = static_cast<float>(ex[best]);
      }
    }
    __threadfence();  // this token's scores before the block's queued count drops
    __syncthreads();
    if (threadIdx.x == 0) last = atomicSub(&pending[t / 16], 1) == 1;
    __syncthreads();
    if (last) {  // every queued token of this 16-token block is final: rewrite its aux partial
      __threadfence();
      const int b = t / 16;
      if (threadIdx.x < 16 * E) {
        const int r = threadIdx.x / E, e = threadIdx.x % E;
        tile[r][e] = b * 16 + r < N ? __ldcg(&scores[static_cast<size_t>(b) * 16 * E + threadIdx.x]) : 0.f;
      }
      __syncthreads();
      if (threadIdx.x < E) {
        double v = 0.0;
        for (int r = 0; r < 16; ++r) v += tile[r][threadIdx.x];
        ssum[static_cast<size_t>(b) * E + threadIdx.x] = v;
      }
    }
    __syncthreads();
  }
}

// Block = 16 tokens (the MMA's M) x all experts (n-tiles of 8); its kRouteTcWarps warps split
// the hidden dimension in 32-column steps.  MMA m (0, 1) of a step maps k-slot {2q+p, 2q+8+p}
// of lane group q to columns c0 + 8q + 4m + {p, 2+p}, so a lane's A registers come from one
// 16-byte load of each of its two token rows and its B values are Wg[c0 + 8q + j][n].
// Wg pieces in MMA-fragment order, written once per call by router_tc_prep_kernel:
// [H/32 chunk][NT][lane q][lane g][m][piece 3][2 b32 words] -> a lane's B registers of one
// 32-column chunk and n-tile are 12 consecutive words (three 16-byte loads).
__global__ void router_tc_prep_kernel(const float* __restrict__ Wg, int H, int E, int NT, uint4* __restrict__ pieces,
                                      int* __restrict__ zero) {
  if (blockIdx.x == 0 && threadIdx.x <= E) zero[threadIdx.x] = 0;  // top-1 counts + fix-up count
  const int chunks = H / 32;
  const int total = chunks * NT * 32;  // one thread per (chunk, n-tile, lane)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int lane = i % 32, nt = (i / 32) % NT, c = i / (32 * NT);
    const int q = lane & 3, g = lane >> 2, e = nt * 8 + g;
    uint32_t wd[12];
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      uint32_t p[3][4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float wv = e < E ? Wg[static_cast<size_t>(c * 32 + 8 * q + 4 * m + j) * E + e] : 0.f;
        split3(wv, p[0][j], p[1][j], p[2][j]);
      }
#pragma unroll
      for (int pc = 0; pc < 3; ++pc) {
        wd[m * 6 + pc * 2] = p[pc][0] | (p[pc][1] << 16);
        wd[m * 6 + pc * 2 + 1] = p[pc][2] | (p[pc][3] << 16);
      }
    }
    uint4* dst = pieces + static_cast<size_t>(c * NT + nt) * 96 + lane;  // [chunk][n-tile][3][lane]
    dst[0] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    dst[32] = make_uint4(wd[4], wd[5], wd[6], wd[7]);
    dst[64] = make_uint4(wd[8], wd[9], wd[10], wd[11]);
  }
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }


// Block = 16 tokens (the MMA's M) x all experts (n-tiles of 8); its W warps (4, or 8 for small
// N) split the hidden dimension in 32-column steps.  MMA m (0, 1) of a step maps k-slot {2q+p, 2q+8+p}
// of lane group q to columns c0 + 8q + 4m + {p, 2+p}, so a lane's A registers are one 16-byte
// chunk of each of its two token rows, and its B registers are 12 prepared words.  Each lane
// streams its own chunks through a private cp.async ring in shared memory (S steps
// deep: the bytes in flight do not cost registers); tokens past N are zero-filled.
// Tokens whose routing the error bound cannot certify get the block's best guess and are queued
// for router_fix_kernel.  The block then writes its aux-loss partial (fp64 sums of its 16 tokens'
// stored fp32 scores, in token order) and adds its top-1 counts; route_finalize_kernel recomputes
// the partials of blocks with queued tokens once those are fixed.
template <int NT, int S, int W>
__global__ void __launch_bounds__(32 * W, NT == 1 ? (W == 4 ? 7 : 3) : 5) router_tc_kernel(
    const __nv_bfloat16* __restrict__ X, const float* __restrict__ Wg, const uint4* __restrict__ pieces, int N, int H,
    int E, int K, int* __restrict__ idx, float* __restrict__ w, float* __restrict__ scores, double* __restrict__ ssum,
    int* __restrict__ cnt_top1, int* __restrict__ fix_list, int* __restrict__ fix_count, int* __restrict__ pending) {
  constexpr int EB = NT * 8;
  // the cp.async rings and the split-K partials share one buffer (rings dead once the loop
  // ends): x chunks S steps deep, Wg pieces (L2-resident, shorter latency) two steps deep
  constexpr int PR = 3 * NT;  // 16-byte pieces chunks per lane and step
  constexpr int kXRing = W * S * 2 * 32 * 16, kRingBytes = kXRing + W * 2 * PR * 32 * 16;
  constexpr int kPartBytes = 2 * W * 16 * EB * 8;
  __shared__ __align__(16) unsigned char sbuf[kRingBytes > kPartBytes ? kRingBytes : kPartBytes];
  auto xring = reinterpret_cast<uint4(*)[S][2][32]>(sbuf);
  auto pring = reinterpret_cast<uint4(*)[2][PR][32]>(sbuf + kXRing);
  auto part = reinterpret_cast<double(*)[16][EB]>(sbuf);
  auto apart = reinterpret_cast<double(*)[16][EB]>(sbuf + kPartBytes / 2);
  __shared__ double lg[16][EB];
  __shared__ double bd[16][EB];
  __shared__ int flagged[16], top1[16];
  __shared__ int nflag;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int t0 = blockIdx.x * 16;
  const int span = H / W;
  const int cw0 = warp * span;
  const int nsteps = span / 32;
  const bool ok0 = t0 + g < N, ok1 = t0 + g + 8 < N;
  const __nv_bfloat16* x0 = X + static_cast<size_t>(ok0 ? t0 + g : 0) * H + 8 * q + cw0;
  const __nv_bfloat16* x1 = X + static_cast<size_t>(ok1 ? t0 + g + 8 : 0) * H + 8 * q + cw0;
  const uint4* pw = pieces + static_cast<size_t>(cw0 >> 5) * NT * 96 + lane;
  if (threadIdx.x == 0) nflag = 0;
  double acc[NT][4], aab[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[nt][i] = aab[nt][i] = 0.0;
  // one commit group per operand and step, issued in need order: at step s the groups up to
  // pieces(s) must have landed while x(s+1 .. s+S-1) and pieces(s+1) stay in flight
  auto issue_x = [&](int step) {
    if (step < nsteps) {
      cp_async16(smem_u32(&xring[warp][step % S][0][lane]), x0 + step * 32, ok0);
      cp_async16(smem_u32(&xring[warp][step % S][1][lane]), x1 + step * 32, ok1);
    }
    cp_async_commit();
  };
  auto issue_p = [&](int step) {
    if (step < nsteps) {
#pragma unroll
      for (int u = 0; u < PR; ++u)
        cp_async16(smem_u32(&pring[warp][step & 1][u][lane]), pw + (step * NT * 3 + u) * 32, true);
    }
    cp_async_commit();
  };
  issue_x(0);
  issue_p(0);
#pragma unroll
  for (int st = 1; st < S - 1; ++st) issue_x(st);
  for (int step = 0; step < nsteps; ++step) {
    issue_p(step + 1);
    issue_x(step + S - 1);
    cp_async_wait<S>();
    const uint4 xa = xring[warp][step % S][0][lane];
    const uint4 xb = xring[warp][step % S][1][lane];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const uint4(*ps)[32] = pring[warp][step & 1];
      const uint4 u0 = ps[3 * nt][lane], u1 = ps[3 * nt + 1][lane], u2 = ps[3 * nt + 2][lane];
      const uint32_t b[12] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w, u2.x, u2.y, u2.z, u2.w};
      float d[4][4];
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int i = 0; i < 4; ++i) d[p][i] = 0.f;
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const uint32_t a0 = m ? xa.z : xa.x, a2 = m ? xa.w : xa.y;  // row g
        const uint32_t a1 = m ? xb.z : xb.x, a3 = m ? xb.w : xb.y;  // row g + 8
#pragma unroll
        for (int pc = 0; pc < 3; ++pc) hmma16816(d[pc], a0, a1, a2, a3, b[m * 6 + pc * 2], b[m * 6 + pc * 2 + 1]);
        hmma16816(d[3], a0 & 0x7FFF7FFFu, a1 & 0x7FFF7FFFu, a2 & 0x7FFF7FFFu, a3 & 0x7FFF7FFFu,
                  b[m * 6] & 0x7FFF7FFFu, b[m * 6 + 1] & 0x7FFF7FFFu);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[nt][i] += static_cast<double>(d[0][i] + d[1][i] + d[2][i]);
        aab[nt][i] += static_cast<double>(d[3][i]);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // every warp is done with its ring before the partials overwrite it
  // C fragment: d0, d1 = (row g, experts 2q, 2q+1), d2, d3 = (row g + 8, the same experts)
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = g + (i >> 1) * 8, col = nt * 8 + 2 * q + (i & 1);
      part[warp][row][col] = acc[nt][i];
      apart[warp][row][col] = aab[nt][i];
    }
  __syncthreads();
  for (int o = threadIdx.x; o < 16 * EB; o += blockDim.x) {  // split-K sum in warp order
    const int row = o / EB, col = o % EB;
    double v = 0.0, a = 0.0;
#pragma unroll
    for (int ww = 0; ww < W; ++ww) {
      v += part[ww][row][col];
      a += apart[ww][row][col];
    }
    lg[row][col] = v;
    bd[row][col] = kRouteTcBound * a + 1e-300;
  }
  __syncthreads();
  if (threadIdx.x < 16 && t0 + threadIdx.x < N) {
    const int r = threadIdx.x;
    // top-(k+1) by repeated argmax (lowest id wins ties), then the gap test
    int ord[kMaxK + 1];
    const int m = min(K + 1, E);
    unsigned used = 0;
    for (int s2 = 0; s2 < m; ++s2) {
      int best = -1;
      for (int e = 0; e < E; ++e) {
        if ((used >> e) & 1u) continue;
        if (best < 0 || lg[r][e] > lg[r][best]) best = e;
      }
      ord[s2] = best;
      used |= 1u << best;
    }
    bool sure = true;
    for (int s2 = 0; s2 + 1 < m && s2 < K; ++s2)
      if (lg[r][ord[s2]] - lg[r][ord[s2 + 1]] <= bd[r][ord[s2]] + bd[r][ord[s2 + 1]]) sure = false;
    if (!sure) flagged[atomicAdd(&nflag, 1)] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    pending[blockIdx.x] = nflag;
    if (nflag) {
      const int base = atomicAdd(fix_count, nflag);
      for (int f = 0; f < nflag; ++f) fix_list[base + f] = t0 + flagged[f];
    }
  }
  // softmax, top-k and outputs of the 16 tokens (fp64 from the certified logits): the exps and
  // divisions one (token, expert) per thread, the max / sum / top-k per token in expert order
  __shared__ double rmx[16], rsum[16];
  if (threadIdx.x < 16) {
    const int r = threadIdx.x;
    double mx = lg[r][0];
    for (int e = 1; e < E; ++e) mx = fmax(mx, lg[r][e]);
    rmx[r] = mx;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < 16 * EB; o += blockDim.x) {
    const int r = o / EB, e = o % EB;
    if (e < E) bd[r][e] = exp(lg[r][e] - rmx[r]);
  }
  __syncthreads();
  if (threadIdx.x < 16) {
    const int r = threadIdx.x;
    double sum = 0.0;
    for (int e = 0; e < E; ++e) sum += bd[r][e];
    rsum[r] = sum;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < 16 * E; o += blockDim.x) {  // coalesced score rows
    const int r = o / E, e = o % E;
    const float sc = static_cast<float>(bd[r][e] / rsum[r]);
    bd[r][e] = sc;  // reused: the token's stored scores, for w and the aux sums
    if (t0 + r < N) scores[static_cast<size_t>(t0) * E + o] = sc;
  }
  __syncthreads();
  if (threadIdx.x < 16 && t0 + threadIdx.x < N) {
    const int r = threadIdx.x, t = t0 + r;
    unsigned used = 0;
    for (int s2 = 0; s2 < K; ++s2) {
      int best = -1;
      for (int e = 0; e < E; ++e) {
        if ((used >> e) & 1u) continue;
        if (best < 0 || lg[r][e] > lg[r][best]) best = e;
      }
      used |= 1u << best;
      idx[static_cast<size_t>(t) * K + s2] = best;
      w[static_cast<size_t>(t) * K + s2] = static_cast<float>(bd[r][best]);
      if (s2 == 0) top1[r] = best;
    }
  }
  __syncthreads();
  if (threadIdx.x < E) {  // aux partials of the block's tokens, in token order
    const int e = threadIdx.x;
    double ssc = 0.0;
    int c = 0;
    for (int r = 0; r < 16 && t0 + r < N; ++r) {
      ssc += bd[r][e];
      c += top1[r] == e;
    }
    ssum[static_cast<size_t>(blockIdx.x) * E + e] = ssc;
    if (c) atomicAdd(&cnt_top1[e], c);
  }
}

// l_aux = E * sum_e frac_e * mean_t s[t,e]  with frac from the top-1 choice (moe.py:221-223).
// Thread (j, e) sums partials j, j + J, ... of expert e (J = blockDim / E; independent loads in
// flight), then thread e adds its J sums in j order: deterministic, one memory round trip deep.
__global__ void __launch_bounds__(kFinalizeThreads) route_finalize_kernel(const double* __restrict__ ssum,
                                                                          int nblocks,
                                                                          const int* __restrict__ cnt_top1, int N,
                                                                          int E, double* __restrict__ l_aux,
                                                                          double* __restrict__ score_sums,
                                                                          int* __restrict__ counts_top1) {
  __shared__ double part[kFinalizeThreads];
  __shared__ double tot[kMaxE];
  const int J = blockDim.x / E;
  const int j = threadIdx.x / E, e = threadIdx.x % E;
  if (j < J) {
    double v = 0.0;
#pragma unroll 8
    for (int b = j; b < nblocks; b += J) v += ssum[static_cast<size_t>(b) * E + e];
    part[threadIdx.x] = v;
  }
  __syncthreads();
  if (threadIdx.x < E) {
    double v = 0.0;
    for (int jj = 0; jj < J; ++jj) v += part[jj * E + threadIdx.x];
    tot[threadIdx.x] = v;
    if (score_sums) score_sums[threadIdx.x] = v;
    if (counts_top1) counts_top1[threadIdx.x] = cnt_top1[threadIdx.x];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0, fr = 0.0;
    for (int k = 0; k < E; ++k) {
      acc += tot[k] * (static_cast<double>(cnt_top1[k]) / N);
      fr += static_cast<double>(cnt_top1[k]) / N;
    }
    l_aux[0] = acc * (static_cast<double>(E) / N);
    l_aux[1] = fr;
  }
}

// Sliced routing: every rank routed N/T tokens and the T per-rank [score sums (E fp64) |
// top-1 counts (E int32) | E pad] records were all-gathered (stats [T][4E] int32 words).  Sum them
// in rank order (deterministic, identical on every rank) and form l_aux (moe.py:211-223).
__global__ void route_combine_stats_kernel(const int* __restrict__ stats, int T, int N, int E,
                                           double* __restrict__ l_aux, int* __restrict__ counts_top1) {
  if (threadIdx.x != 0) return;
  double tot = 0.0, fr = 0.0;
  for (int e = 0; e < E; ++e) {
    double s = 0.0;
    int c = 0;
    for (int r = 0; r < T; ++r) {
      const int* rec = stats + static_cast<size_t>(r) * 4 * E;  // 16-byte aligned records
      s += reinterpret_cast<const double*>(rec)[e];
      c += rec[2 * E + e];
    }
    const double frac = static_cast<double>(c) / N;
    tot += s * frac;
    fr += frac;
    counts_top1[e] = c;
  }
  l_aux[0] = tot * (static_cast<double>(E) / N);
  l_aux[1] = fr;
}

// ------------------------------------------------------------------ dispatch plan

struct PlanWs {
  int* hist;   // [C][K][E] pairs per chunk, slot, expert
  int* base;   // [C][K][E] exclusive prefix over chunks
  int* tot;    // [K][E]
  int* kc;     // [C][E] kept pairs per chunk and expert
  int* kb;     // [C][E] exclusive prefix over chunks
  int* kflag;  // [N*K]
};

static size_t plan_ws_layout(int N, int E, int K, char* base, PlanWs* out) {
  const size_t C = (static_cast<size_t>(N) + kChunk - 1) / kChunk;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  size_t o_hist = take(C * K * E * 4), o_base = take(C * K * E * 4), o_tot = take(static_cast<size_t>(K) * E * 4),
         o_kc = take(C * E * 4), o_kb = take(C * E * 4), o_kf = take(static_cast<size_t>(N) * K * 4);
  if (out && base) {
    out->hist = reinterpret_cast<int*>(base + o_hist);
    out->base = reinterpret_cast<int*>(base + o_base);
    out->tot = reinterpret_cast<int*>(base + o_tot);
    out->kc = reinterpret_cast<int*>(base + o_kc);
    out->kb = reinterpret_cast<int*>(base + o_kb);
    out->kflag = reinterpret_cast<int*>(base + o_kf);
  }
  return off;
}

__global__ void plan_hist_kernel(const int* __restrict__ idx, int N, int E, int K, int* __restrict__ hist) {
  extern __shared__ int sh[];  // [K][E]
  for (int i = threadIdx.x; i < K * E; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int t = blockIdx.x * kChunk + threadIdx.x;
  if (t < N)
    for (int s = 0; s < K; ++s) atomicAdd(&sh[s * E + idx[static_cast<size_t>(t) * K + s]], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < K * E; i += blockDim.x) hist[static_cast<size_t>(blockIdx.x) * K * E + i] = sh[i];
}

__global__ void plan_totals_kernel(const int* __restrict__ hist, int C, int E, int K, int capacity,
                                   int* __restrict__ base, int* __restrict__ tot, int* __restrict__ counts) {
  const int KE = K * E;
  for (int j = threadIdx.x; j < KE; j += blockDim.x) {
    int run = 0;
    for (int c = 0; c < C; ++c) {
      const int v = hist[static_cast<size_t>(c) * KE + j];
      base[static_cast<size_t>(c) * KE + j] = run;
      run += v;
    }
    tot[j] = run;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int n = 0;
    for (int s = 0; s < K; ++s) n += tot[s * E + e];
    counts[e] = n;
  }
}

// Priority rank of every pair: all slot-0 pairs in ascending token id, then slot 1, ...
// (reduces to _capacity_mask's ascending global token id at K = 1).
__global__ void plan_keep_kernel(const int* __restrict__ idx, int N, int E, int K, int capacity,
                                 const int* __restrict__ base, const int* __restrict__ tot,
                                 const int* __restrict__ rank_offset, int* __restrict__ kflag,
                                 int* __restrict__ kc) {
  extern __shared__ int sh[];
  int* wc = sh;                        // [8][K][E]
  int* kcs = wc + 8 * K * E;           // [E]
  const int c = blockIdx.x;
  const int t = c * kChunk + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int i = threadIdx.x; i < 8 * K * E; i += blockDim.x) wc[i] = 0;
  for (int i = threadIdx.x; i < E; i += blockDim.x) kcs[i] = 0;
  __syncthreads();
  int ev[kMaxK];
  int rw[kMaxK];
  for (int s = 0; s < K; ++s) {
    ev[s] = t < N ? idx[static_cast<size_t>(t) * K + s] : -1;
    const unsigned m = __match_any_sync(0xffffffffu, ev[s]);
    rw[s] = __popc(m & lt);
    if (ev[s] >= 0 && rw[s] == 0) wc[(warp * K + s) * E + ev[s]] = __popc(m);
  }
  __syncthreads();
  // exclusive prefix over the 8 warps, per (slot, expert)
  for (int j = threadIdx.x; j < K * E; j += blockDim.x) {
    int run = 0;
    for (int wv = 0; wv < 8; ++wv) {
      const int v = wc[wv * K * E + j];
      wc[wv * K * E + j] = run;
      run += v;
    }
  }
  __syncthreads();
  if (t < N) {
    for (int s = 0; s < K; ++s) {
      const int e = ev[s];
      int prior = 0;
      for (int s2 = 0; s2 < s; ++s2) prior += tot[s2 * E + e];
      const long long rank = static_cast<long long>(prior) + base[(static_cast<size_t>(c) * K + s) * E + e] +
                             wc[(warp * K + s) * E + e] + rw[s] + (rank_offset ? rank_offset[s * E + e] : 0);
      const int keep = rank < capacity ? 1 : 0;
      kflag[static_cast<size_t>(t) * K + s] = keep;
      if (keep) atomicAdd(&kcs[e], 1);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x) kc[static_cast<size_t>(c) * E + i] = kcs[i];
}

__global__ void plan_offsets_kernel(const int* __restrict__ kc, int C, int E, int* __restrict__ kb,
                                    int* __restrict__ kept, int* __restrict__ seg, int* __restrict__ tok_sorted,
                                    float* __restrict__ w_sorted) {
  __shared__ int sk[kMaxE];
  __shared__ int sseg[kMaxE + 1];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int run = 0;
    for (int c = 0; c < C; ++c) {
      kb[static_cast<size_t>(c) * E + e] = run;
      run += kc[static_cast<size_t>(c) * E + e];
    }
    sk[e] = run;
    kept[e] = run;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int e = 0; e < E; ++e) {
      sseg[e] = acc;
      acc += (sk[e] + 127) / 128 * 128;
    }
    sseg[E] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e <= E; e += blockDim.x) seg[e] = sseg[e];
  // padding rows of every segment: token -1, weight 0
  for (int e = 0; e < E; ++e) {
    const int lo = sseg[e] + sk[e], hi = sseg[e + 1];
    for (int p = lo + threadIdx.x; p < hi; p += blockDim.x) {
      tok_sorted[p] = -1;
      if (w_sorted) w_sorted[p] = 0.f;
    }
  }
}

// Stable scatter: kept pairs of expert e land in ascending token order at
// seg[e] + (# kept pairs of e with a smaller token id).
__global__ void plan_scatter_kernel(const int* __restrict__ idx, const float* __restrict__ w, int N, int E, int K,
                                    const int* __restrict__ kflag, const int* __restrict__ kb,
                                    const int* __restrict__ seg, int* __restrict__ tok_sorted,
                                    float* __restrict__ w_sorted, int* __restrict__ pair_pos) {
  extern __shared__ int sh[];  // [8][E]
  const int c = blockIdx.x;
  const int t = c * kChunk + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  int ev[kMaxK], kf[kMaxK], rw[kMaxK];
  for (int s = 0; s < K; ++s) {
    ev[s] = t < N ? idx[static_cast<size_t>(t) * K + s] : -1;
    kf[s] = t < N ? kflag[static_cast<size_t>(t) * K + s] : 0;
    rw[s] = 0;
  }
  for (int e = 0; e < E; ++e) {
    unsigned mask = 0u;
    for (int s = 0; s < K; ++s) mask |= __ballot_sync(0xffffffffu, kf[s] && ev[s] == e);
    for (int s = 0; s < K; ++s)
      if (kf[s] && ev[s] == e) rw[s] = __popc(mask & lt);
    if (lane == 0) sh[warp * E + e] = __popc(mask);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int run = 0;
    for (int wv = 0; wv < 8; ++wv) {
      const int v = sh[wv * E + e];
      sh[wv * E + e] = run;
      run += v;
    }
  }
  __syncthreads();
  if (t >= N) return;
  for (int s = 0; s < K; ++s) {
    const size_t pi = static_cast<size_t>(t) * K + s;
    if (!kf[s]) {
      pair_pos[pi] = -1;
      continue;
    }
    const int e = ev[s];
    const int pos = seg[e] + kb[static_cast<size_t>(c) * E + e] + sh[warp * E + e] + rw[s];
    tok_sorted[pos] = t;
    if (w_sorted) w_sorted[pos] = w ? w[pi] : 1.f;
    pair_pos[pi] = pos;
  }
}

template <typename T, int EB>
static int launch_router(const void* X, const float* Wg, int N, int H, int E, int K, const int* ovr, int* idx, float* w,
                         float* scores, double* ssum, int* cnt, cudaStream_t s) {
  const size_t smem = route_smem_bytes(E);
  auto k = router_kernel<T, EB>;
  PPMOE_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int nb = (N + kRouteTB - 1) / kRouteTB;
  k<<<nb, kRouteThreads, smem, s>>>(static_cast<const T*>(X), Wg, N, H, E, K, ovr, idx, w, scores, ssum, cnt);
  return check_launch("router_kernel");
}

// PPMOE_ROUTER=tc (default for bf16): tensor-core logits + guard band + exact fix-up;
// dmma: FP64 tensor-core logits for every token; dfma: CUDA-core fp64.
static bool use_tc_router(int dtype, int H, int E) {
  // default for bf16 and E <= 16 (tools/ab_router.py, C2 / C3: 64 / 189 us against the DMMA
  // router's 89 / 237); PPMOE_ROUTER=dmma|dfma selects the fp64 routers
  const char* e = std::getenv("PPMOE_ROUTER");
  if (e && std::strcmp(e, "tc") != 0) return false;
  return dtype == kBF16 && H % (32 * kRouteTcWarps) == 0 && E <= 16;
}

static int launch_router_tc(const void* X, const float* Wg, int N, int H, int E, int K, int* idx, float* w,
                            float* scores, double* ssum, int* cnt, int* fix_list, int* fix_count, int* pending,
                            uint4* pieces, cudaStream_t s) {
  const auto* x = static_cast<const __nv_bfloat16*>(X);
  const int NT = E <= 8 ? 1 : 2;
  const int prep_threads = H / 32 * NT * 32;
  router_tc_prep_kernel<<<std::max(1, std::min((prep_threads + 255) / 256, num_sms() * 4)), 256, 0, s>>>(Wg, H, E, NT,
                                                                                                      pieces, cnt);
  if (int rc = check_launch("router_tc_prep_kernel")) return rc;
  const int blocks = (N + 15) / 16;
  // x two steps deep (a three-deep x ring measured 37.7 vs 35.5 us at C2, 164 vs 166 at C3).
  // Few blocks (a TP rank's N/T-token slice, <= 2 per SM) fill the SMs better with 8 warps per
  // block instead of 4, each splitting the hidden dimension further (ncu, C2 shape: 4096 tokens
  // 17.3 -> 15.5 us; 8192 tokens 23.6 -> 29 us, so only below that); PPMOE_TC_W=4|8 forces one.
  const char* we = getenv("PPMOE_TC_W");
  const int wsel = we ? atoi(we) : (blocks <= num_sms() * 2 ? 8 : 4);
  if (E <= 8 && wsel == 8 && H % 256 == 0)
    router_tc_kernel<1, 2, 8><<<blocks, 256, 0, s>>>(x, Wg, pieces, N, H, E, K, idx, w, scores, ssum, cnt, fix_list,
                                                     fix_count, pending);
  else if (E <= 8)
    router_tc_kernel<1, 2, kRouteTcWarps><<<blocks, 32 * kRouteTcWarps, 0, s>>>(
        x, Wg, pieces, N, H, E, K, idx, w, scores, ssum, cnt, fix_list, fix_count, pending);
  else
    router_tc_kernel<2, 2, kRouteTcWarps><<<blocks, 32 * kRouteTcWarps, 0, s>>>(
        x, Wg, pieces, N, H, E, K, idx, w, scores, ssum, cnt, fix_list, fix_count, pending);
  if (int rc = check_launch("router_tc_kernel")) return rc;
  const int fix_blocks = std::min(N, num_sms() * 2);
  if (E <= 8) router_fix_kernel<8><<<fix_blocks, kFixThreads, 0, s>>>(x, Wg, N, H, E, K, fix_list, fix_count, idx, w, scores, cnt,
                                                              pending, ssum);
  else router_fix_kernel<16><<<fix_blocks, kFixThreads, 0, s>>>(x, Wg, N, H, E, K, fix_list, fix_count, idx, w, scores, cnt,
                                                               pending, ssum);
  return check_launch("router_fix_kernel");
}

static bool use_dmma_router(int dtype, int H, int E) {
  const char* e = std::getenv("PPMOE_ROUTER");  // PPMOE_ROUTER=dfma: the CUDA-core fp64 kernel (A/B)
  if (e && std::strcmp(e, "dfma") == 0) return false;
  return dtype == kBF16 && H % (32 * kRouteDmmaMaxWarps) == 0 && E <= 16;
}


template <int EB, int W, int MINB>
static int launch_router_dmma_cfg(const void* X, const float* Wg, int N, int H, int E, int K, const int* ovr, int* idx,
                                  float* w, float* scores, double* ssum, int* cnt, cudaStream_t s) {
  const size_t smem = route_dmma_smem_bytes(E, W);
  auto k = router_dmma_kernel<EB, W, MINB>;
  PPMOE_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int nb = (N + kRouteTB - 1) / kRouteTB;
  k<<<nb, 32 * W, smem, s>>>(static_cast<const __nv_bfloat16*>(X), Wg, N, H, E, K, ovr, idx, w, scores, ssum, cnt);
  return check_launch("router_dmma_kernel");
}

// 8 warps per 32-token block, 2 blocks per SM.  Measured alternatives (tools/ab_router.py,
// profiles/r02_router_ab.txt): 4 warps x 4-6 blocks per SM, 3 blocks per SM (register
// spills), and a TMA shared-memory ring for X and Wg: equal or slower.
template <int EB>
static int launch_router_dmma(const void* X, const float* Wg, int N, int H, int E, int K, const int* ovr, int* idx,
                              float* w, float* scores, double* ssum, int* cnt, cudaStream_t s) {
  return launch_router_dmma_cfg<EB, 8, 2>(X, Wg, N, H, E, K, ovr, idx, w, scores, ssum, cnt, s);
}

}  // namespace ppmoe

using namespace ppmoe;

extern "C" {

// ppmoe_route workspace: aux score-sum records (one per 16 tokens; the fp64 routers use one per
// 32) | top-1 counts + the tensor-core router's fix-up count | fix-up queue, per-16-token-block
// queued counts | (with H) the Wg pieces.
static size_t route_ssum_bytes(int N, int E) {
  return align_up((static_cast<size_t>(N) + 15) / 16 * (E > 0 ? E : 1) * 8, 256);
}

size_t ppmoe_route_workspace_bytes(int N, int E, int K) {
  (void)K;
  return route_ssum_bytes(N, E) + align_up(static_cast<size_t>(E) * 4 + 4, 256) +
         align_up(align_up(static_cast<size_t>(N > 0 ? N : 1), 64) * 4 + (static_cast<size_t>(N) + 15) / 16 * 4, 256);
}

size_t ppmoe_route_workspace_bytes_h(int N, int H, int E, int K) {
  // + the tensor-core router's Wg pieces (H/32 chunks x n-tiles x 32 lanes x 48 bytes)
  const size_t nt = E <= 8 ? 1 : 2;
  return ppmoe_route_workspace_bytes(N, E, K) + align_up(static_cast<size_t>(H > 0 ? H : 1) / 32 * nt * 32 * 48 + 48, 256);
}

int ppmoe_route(const void* X, int dtype, const float* Wg, int N, int H, int E, int K, const int* route_override,
                int* idx, float* w, float* scores, double* l_aux, int* counts_top1, double* score_sums, void* ws,
                size_t ws_bytes, void* stream) {
  PPMOE_REQUIRE(dtype == kBF16 || dtype == kF32, "dtype must be 0 (bf16) or 1 (fp32)");
  PPMOE_REQUIRE(N >= 1, "aux_loss of zero tokens is undefined (N=%d)", N);
  PPMOE_REQUIRE(H >= 1 && E >= 1 && E <= kMaxE, "router needs 1 <= E <= %d, got E=%d H=%d", kMaxE, E, H);
  PPMOE_REQUIRE(K >= 1 && K <= E && K <= kMaxK, "top-k must satisfy 1 <= k <= min(E, %d), got k=%d E=%d", kMaxK, K, E);
  PPMOE_REQUIRE(ws_bytes >= ppmoe_route_workspace_bytes(N, E, K), "route workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = (N + kRouteTB - 1) / kRouteTB;
  double* ssum = static_cast<double*>(ws);
  int* cnt = reinterpret_cast<int*>(static_cast<char*>(ws) + route_ssum_bytes(N, E));
  int* fix_count = cnt + E;
  int* fix_list = reinterpret_cast<int*>(reinterpret_cast<char*>(cnt) + align_up(static_cast<size_t>(E) * 4 + 4, 256));
  int rc;
  int nparts = nb;  // aux partial records: 32-token blocks, or 16-token blocks of the tensor-core router
  const bool tc = !route_override && use_tc_router(dtype, H, E) && ws_bytes >= ppmoe_route_workspace_bytes_h(N, H, E, K);
  if (!tc) PPMOE_CUDA(cudaMemsetAsync(cnt, 0, static_cast<size_t>(E) * 4 + 4, s));  // the tc prep kernel zeroes them
  if (tc) {
    uint4* pieces = reinterpret_cast<uint4*>(static_cast<char*>(ws) + ppmoe_route_workspace_bytes(N, E, K));
    int* pending = fix_list + align_up(static_cast<size_t>(N), 64);
    rc = launch_router_tc(X, Wg, N, H, E, K, idx, w, scores, ssum, cnt, fix_list, fix_count, pending, pieces, s);
    nparts = (N + 15) / 16;
  } else if (use_dmma_router(dtype, H, E))
    rc = E <= 8 ? launch_router_dmma<8>(X, Wg, N, H, E, K, route_override, idx, w, scores, ssum, cnt, s)
                : launch_router_dmma<16>(X, Wg, N, H, E, K, route_override, idx, w, scores, ssum, cnt, s);
  else if (dtype == kBF16)
    rc = E <= 8 ? launch_router<__nv_bfloat16, 8>(X, Wg, N, H, E, K, route_override, idx, w, scores, ssum, cnt, s)
                : launch_router<__nv_bfloat16, 16>(X, Wg, N, H, E, K, route_override, idx, w, scores, ssum, cnt, s);
  else
    rc = E <= 8 ? launch_router<float, 8>(X, Wg, N, H, E, K, route_override, idx, w, scores, ssum, cnt, s)
                : launch_router<float, 16>(X, Wg, N, H, E, K, route_override, idx, w, scores, ssum, cnt, s);
  if (rc) return rc;
  route_finalize_kernel<<<1, kFinalizeThreads, 0, s>>>(ssum, nparts, cnt, N, E, l_aux, score_sums, counts_top1);
  return check_launch("route_finalize_kernel");
}

int ppmoe_route_combine_stats(const int* stats, int T, int N, int E, double* l_aux, int* counts_top1, void* stream) {
  PPMOE_REQUIRE(T >= 1 && N >= 1 && E >= 1 && E <= kMaxE, "bad route stats T=%d N=%d E=%d", T, N, E);
  route_combine_stats_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(stats, T, N, E, l_aux, counts_top1);
  return check_launch("route_combine_stats_kernel");
}

size_t ppmoe_dispatch_workspace_bytes(int N, int E, int K) { return plan_ws_layout(N, E, K, nullptr, nullptr); }

int ppmoe_dispatch_plan(const int* idx, const float* w, int N, int E, int K, int capacity, const int* rank_offset,
                        int* counts, int* kept, int* seg, int* tok_sorted, float* w_sorted, int* pair_pos,
                        int rows_cap_global, void* ws, size_t ws_bytes, void* stream) {
  PPMOE_REQUIRE(N >= 0 && E >= 1 && E <= kMaxE, "dispatch plan needs 1 <= E <= %d", kMaxE);
  PPMOE_REQUIRE(K >= 1 && K <= kMaxK && K <= E, "bad top-k %d", K);
  PPMOE_REQUIRE(capacity >= 0, "capacity must be non-negative");
  PPMOE_REQUIRE(static_cast<long long>(rows_cap_global) >= static_cast<long long>(N) * K + 128LL * E,
                "rows_cap_global too small");
  PPMOE_REQUIRE(ws_bytes >= plan_ws_layout(N, E, K, nullptr, nullptr), "dispatch workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PlanWs p;
  plan_ws_layout(N, E, K, static_cast<char*>(ws), &p);
  const int C = (N + kChunk - 1) / kChunk;
  if (C == 0) {
    PPMOE_CUDA(cudaMemsetAsync(counts, 0, E * 4, s));
    PPMOE_CUDA(cudaMemsetAsync(kept, 0, E * 4, s));
    PPMOE_CUDA(cudaMemsetAsync(seg, 0, (E + 1) * 4, s));
    return kOk;
  }
  plan_hist_kernel<<<C, kChunk, K * E * 4, s>>>(idx, N, E, K, p.hist);
  if (int rc = check_launch("plan_hist")) return rc;
  plan_totals_kernel<<<1, 1024, 0, s>>>(p.hist, C, E, K, capacity, p.base, p.tot, counts);
  if (int rc = check_launch("plan_totals")) return rc;
  plan_keep_kernel<<<C, kChunk, (8 * K * E + E) * 4, s>>>(idx, N, E, K, capacity, p.base, p.tot, rank_offset,
                                                         p.kflag, p.kc);
  if (int rc = check_launch("plan_keep")) return rc;
  plan_offsets_kernel<<<1, 1024, 0, s>>>(p.kc, C, E, p.kb, kept, seg, tok_sorted, w_sorted);
  if (int rc = check_launch("plan_offsets")) return rc;
  plan_scatter_kernel<<<C, kChunk, 8 * E * 4, s>>>(idx, w, N, E, K, p.kflag, p.kb, seg, tok_sorted, w_sorted,
                                                   pair_pos);
  return check_launch("plan_scatter");
}

}  // extern "C"
