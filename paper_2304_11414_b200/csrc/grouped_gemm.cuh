// Grouped (per-expert) GEMM on sm_100a: tcgen05.mma + TMEM accumulators, TMA-fed,
// warp-specialised, persistent over a device-side tile list.
//
//   D_g[M_g x N] = A_g[M_g x K_g] * B_g[K_g x N]      for every local expert g
//
// M_g or K_g may come from the device-side dispatch segments (`seg`, padded to
// 128 rows per expert by the dispatch plan), so no host synchronisation is
// needed between routing and the expert GEMMs.  Each operand is a 2-D global
// tensor addressed either K-major (row = M/N index, K contiguous) or MN-major
// (row = K index, M/N contiguous); both are staged with SWIZZLE_128B TMA boxes
// and described to the tensor core with the matching canonical layout.
//
// The epilogue is a functor applied per (row, 32-column chunk) straight out of
// TMEM (tcgen05.ld): bias + exact GeLU, gate-scaled scatter-add combine,
// GeLU' backward, scatter-add of dX, or the weight-gradient store.  This is the
// fused replacement of the reference's per-expert loop of
//   index_select -> matmul -> add -> gelu -> matmul -> add -> scale_rows -> index_assign
// (moe.py:294-305, tensor.py:128-272).
#pragma once

#include "common.cuh"

namespace ppmoe {

constexpr int kBM = 128;      // tile rows (UMMA M, one CTA)
constexpr int kBK = 64;       // K per pipeline stage = one 128-byte swizzle row of bf16
constexpr int kUMMAK = 16;    // K per tcgen05.mma (bf16)
constexpr int kStages = 4;
constexpr int kMaxGroups = 64;
constexpr int kGemmThreads = 256;  // warp0 TMA, warp1 MMA, warp2 TMEM alloc, warps4-7 epilogue

struct GroupGeom {
  int G;          // number of groups (local experts)
  int N;          // output columns
  int M_fixed;    // >0: every group has M = M_fixed rows; else M_g = padded segment rows
  int K_fixed;    // >0: every group has K = K_fixed; else K_g = padded segment rows
  const int* seg; // [G+1] padded segment starts (global positions; local = seg[g]-seg[0])
  int a_seg;      // A row base: 1 -> local segment start, 0 -> g * a_stride
  int a_stride;
  int b_seg;
  int b_stride;
  const int* rlo; // optional [G] local first row of each group (token chunk of a segment)
  const int* rhi; // optional [G] local end row; when set, M_g = rhi - rlo (seg ignored for rows)
  int banded;     // 1: banded 2-D tile order with L2 residency hints, 0: panel order
  int nfast;      // -1: fast dimension chosen by panel size; 0 / 1: force M / N fast
  int hint;       // panel order: load the streaming operand with evict-first priority
  // Soft wave synchronisation of the TMA producers every `ksync` k-blocks (0 = off; only
  // with K_fixed > 0): keeps the concurrent tiles' k positions together so the wave's
  // operand slices are re-used from L2 instead of re-read from DRAM.  Bounded wait.
  unsigned int* ksync_ctr;
  int ksync;
  int stage;      // pair kernel: warp-cooperative staged row stores for stageable epilogues
  int tail128;    // pair kernel: a group's last tile with 128 rows runs M = 128 MMAs (half the work)
};

// Epilogues that can hand their bf16 rows to the staged (coalesced) store path.
template <class E, class = void>
struct StageTrait {
  static constexpr bool value = false;
};
template <class E>
struct StageTrait<E, std::void_t<decltype(E::kStageable)>> {
  static constexpr bool value = E::kStageable;
};

template <int BN>
struct GemmSmem {
  static constexpr int kABytes = kBM * kBK * 2;     // 16 KB
  static constexpr int kBBytes = BN * kBK * 2;      // 32 KB at BN=256
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBarOffset = kStages * kStageBytes;
  // full[S], empty[S], tmem_full[2], tmem_empty[2], tmem base, scheduler tables
  static constexpr int kBarBytes = (2 * kStages + 4) * 8 + 16;
  static constexpr int kSchedOffset = kBarOffset + kBarBytes;
  static constexpr int kSchedBytes = (kMaxGroups + 1) * 4 * 8;
  static constexpr int kTotal = kSchedOffset + kSchedBytes + 1024;  // + alignment slack
};

// Tile scheduler tables, filled identically by every CTA from the device segments.
struct SchedTables {
  int* tile_start;  // [G+1]
  int* m_tiles;     // [G]
  int* k_blocks;    // [G]
  int* a_base;      // [G]
  int* b_base;      // [G]
  int* n_fast;      // [G] 1: walk n-tiles fastest (A panel larger than B panel), else m-tiles fastest
  int* m_rows;      // [G] valid rows of the group (epilogue row mask)
  int* row_base;    // [G] local buffer row of the group's first row
};

// Tile (m, n) of the local index inside group g.  Tiles are walked in bands of
// kBand tiles along the slow dimension with the fast dimension inside the band, so a
// wave of concurrent tiles covers a roughly square block of the output: both operand
// panels of that block are shared through L2 while the K loop streams.  The fast
// dimension is N when the A panel is the larger one.
constexpr int kBand = 8;
__device__ __forceinline__ void tile_coords(const SchedTables& t, int g, int local, int n_tiles, int& mt, int& nt,
                                            int banded) {
  const int m_tiles = t.m_tiles[g];
  if (!banded) {  // panel order: the fast dimension's whole panel shared by the wave
    if (t.n_fast[g]) {
      mt = local / n_tiles;
      nt = local % n_tiles;
    } else {
      mt = local % m_tiles;
      nt = local / m_tiles;
    }
    return;
  }
  if (t.n_fast[g]) {  // bands of kBand m-tiles (A band L2-resident), n advances slowest inside a band
    const int per_band = kBand * n_tiles;
    const int b = local / per_band, r = local % per_band;
    const int bw = min(kBand, m_tiles - b * kBand);
    mt = b * kBand + r % bw;
    nt = r / bw;
  } else {  // bands of kBand n-tiles (B band L2-resident), m advances slowest inside a band
    const int per_band = kBand * m_tiles;
    const int b = local / per_band, r = local % per_band;
    const int bw = min(kBand, n_tiles - b * kBand);
    nt = b * kBand + r % bw;
    mt = r / bw;
  }
}

// The group's last m-tile holds 128 rows (M = padded segment rows, a multiple of 128): the
// CTA pair runs it with M = 128 MMAs (64 rows per CTA) instead of 256 rows half padding.
__device__ __forceinline__ bool pair_tail(const GroupGeom& geo, const SchedTables& t, int g, int mt) {
  return geo.tail128 && t.m_rows[g] - mt * 256 <= 128;
}

__device__ __forceinline__ void sched_locate(const SchedTables& t, int G, int tile, int& g, int& local) {
  int lo = 0;
  while (lo + 1 < G && t.tile_start[lo + 1] <= tile) ++lo;
  g = lo;
  local = tile - t.tile_start[lo];
}

template <int BN, bool A_MN, bool B_MN, class Epi>
__global__ void __launch_bounds__(kGemmThreads, 1)
    grouped_gemm_sm100(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                       GroupGeom geo, Epi epi) {
  using L = GemmSmem<BN>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);

  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  int* sched = reinterpret_cast<int*>(smem + L::kSchedOffset);
  SchedTables tab{sched, sched + (kMaxGroups + 1), sched + 2 * (kMaxGroups + 1), sched + 3 * (kMaxGroups + 1),
                  sched + 4 * (kMaxGroups + 1), sched + 5 * (kMaxGroups + 1), sched + 6 * (kMaxGroups + 1),
                  sched + 7 * (kMaxGroups + 1)};

  const int warp = warp_id();
  const int lane = lane_id();
  const int G = geo.G;
  const int n_tiles = (geo.N + BN - 1) / BN;

  if (threadIdx.x == 0) {
    const int s0 = geo.seg[0];
    int acc = 0;
    for (int g = 0; g < G; ++g) {
      const int seg_lo = geo.rlo ? geo.rlo[g] : geo.seg[g] - s0;
      const int seg_rows = geo.rlo ? geo.rhi[g] - geo.rlo[g] : geo.seg[g + 1] - geo.seg[g];
      const int M = geo.M_fixed > 0 ? geo.M_fixed : seg_rows;
      const int K = geo.K_fixed > 0 ? geo.K_fixed : seg_rows;
      tab.tile_start[g] = acc;
      tab.m_tiles[g] = (M + kBM - 1) / kBM;
      tab.k_blocks[g] = (K + kBK - 1) / kBK;
      tab.a_base[g] = geo.a_seg ? seg_lo : g * geo.a_stride;
      tab.b_base[g] = geo.b_seg ? seg_lo : g * geo.b_stride;
      tab.n_fast[g] = geo.nfast >= 0 ? geo.nfast : (M > geo.N ? 1 : 0);
      tab.m_rows[g] = M;
      tab.row_base[g] = seg_lo;
      acc += tab.m_tiles[g] * n_tiles;
    }
    tab.tile_start[G] = acc;
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
  }
  constexpr uint32_t kTmemCols = 2 * BN;  // double-buffered fp32 accumulator
  if (warp == 2) tmem_alloc(tmem_base_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  const int total_tiles = tab.tile_start[G];

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        int g, local;
        sched_locate(tab, G, tile, g, local);
        int mt, nt;
        tile_coords(tab, g, local, n_tiles, mt, nt, geo.banded);
        const int kb_n = tab.k_blocks[g];
        const int abase = tab.a_base[g];
        const int bbase = tab.b_base[g];
        for (int kb = 0; kb < kb_n; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          mbar_arrive_expect_tx(&full[stage], L::kStageBytes);
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < kBM / 64; ++j)
              tma_load_2d(sa + j * (64 * kBK * 2), &tmap_a, &full[stage], mt * kBM + j * 64, abase + kb * kBK);
          } else {
            tma_load_2d(sa, &tmap_a, &full[stage], kb * kBK, abase + mt * kBM);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(sb + j * (64 * kBK * 2), &tmap_b, &full[stage], nt * BN + j * 64, bbase + kb * kBK);
          } else {
            tma_load_2d(sb, &tmap_b, &full[stage], kb * kBK, bbase + nt * BN);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(kBM, BN, A_MN, B_MN);
      // Descriptor strides (bytes). K-major: SBO = 8 rows x 128 B. MN-major: LBO = distance
      // between 64-wide MN chunks (one TMA box each), SBO = 8 K-rows x 128 B.
      constexpr uint32_t a_lbo = A_MN ? (64 * kBK * 2) : 16;
      constexpr uint32_t b_lbo = B_MN ? (64 * kBK * 2) : 16;
      constexpr uint32_t k_step_a = A_MN ? (kUMMAK * 128) : (kUMMAK * 2);
      constexpr uint32_t k_step_b = B_MN ? (kUMMAK * 128) : (kUMMAK * 2);
      int stage = 0;
      uint32_t phase = 0;
      int iter = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++iter) {
        int g, local;
        sched_locate(tab, G, tile, g, local);
        const int kb_n = tab.k_blocks[g];
        const int acc = iter & 1;
        const uint32_t acc_phase = (iter >> 1) & 1;
        mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kb_n; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * L::kStageBytes);
          const uint32_t sb = sa + L::kABytes;
#pragma unroll
          for (int k = 0; k < kBK / kUMMAK; ++k) {
            const uint64_t ad = make_sdesc(sa + k * k_step_a, a_lbo, 1024);
            const uint64_t bd = make_sdesc(sb + k * k_step_b, b_lbo, 1024);
            umma_bf16(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tmem_full[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row_in_tile = q * 32 + lane;
    int iter = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++iter) {
      int g, local;
      sched_locate(tab, G, tile, g, local);
      int mt, nt;
      tile_coords(tab, g, local, n_tiles, mt, nt, geo.banded);
      const bool has_k = tab.k_blocks[g] > 0;
      const int acc = iter & 1;
      const uint32_t acc_phase = (iter >> 1) & 1;
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      const int m = mt * kBM + row_in_tile;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float v[32];
        tmem_ld32(taddr + c * 32, v);
        if (!has_k) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f;
        }
        const int n0 = nt * BN + c * 32;
        if (n0 < geo.N && m < tab.m_rows[g]) epi.template apply<32>(g, m, tab.row_base[g] + m, n0, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

// --------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): one 256 x 256 tile per CTA pair (cluster of 2).
// CTA r of the pair stages A rows [256*mt + 128 r, +128) and B columns
// [256*nt + 128 r, +128) (32 KB per stage per CTA, 6 stages); the leader issues
// tcgen05.mma.cta_group::2 M=256 N=256, each CTA's TMEM receives its 128 rows.
// Per-SM operand traffic is 2/3 of the 1-CTA 128x256 tile.
//   full[s]      (leader) 1 arrival: the leader expects both CTAs' bytes; the peer's TMA
//                         completes its transactions on the leader's barrier
//   empty[s]     (both)   multicast commit from the leader's MMA
//   tmem_full[a] (both)   multicast commit
//   tmem_empty[a](leader) 8 arrivals: 4 epilogue warps x 2 CTAs
// BN = 512 ("wide"): one 256 x 512 tile per pair, two M=256 N=256 MMAs per k-step on the
// same A stage (CTA r stages B columns [256 j + 128 r, +128) for MMA j), 48 KB per stage,
// 4 stages, a single TMEM accumulator (512 columns).  Per tile the pair loads
// A 32 KB + B 64 KB per k-block for 2x the FLOPs of a 256 x 256 tile: 25 % fewer
// L2 -> SM bytes (the cuBLAS tile shape); the epilogue no longer overlaps the next
// tile's mainloop.
constexpr int kPairBM = 256;
// CTA-pair kernel: warp0 TMA, warp1 MMA, warps 2..9 epilogue (warp2 also allocates TMEM)
constexpr int kPairEpiWarps = 8;
constexpr int kPairThreads = 32 * (2 + kPairEpiWarps);

template <int BN>
struct PairSmem {
  static constexpr int kStages = BN > 256 ? 4 : 6;
  static constexpr int kMmaN = BN > 256 ? 256 : BN;       // N of one tcgen05.mma
  static constexpr int kNMma = BN / kMmaN;                // MMAs per k-step
  static constexpr int kAcc = BN > 256 ? 1 : 2;           // TMEM accumulator buffers
  static constexpr int kABytes = 128 * kBK * 2;          // 16 KB: this CTA's half of A
  static constexpr int kBChunk = (kMmaN / 2) * kBK * 2;  // 16 KB: this CTA's half of one MMA's B
  static constexpr int kBBytes = kNMma * kBChunk;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBarOffset = kStages * kStageBytes;
  static constexpr int kBarBytes = (2 * kStages + 4) * 8 + 16;
  static constexpr int kSchedOffset = kBarOffset + kBarBytes;
  static constexpr int kSchedBytes = (kMaxGroups + 1) * 4 * 8;
  static constexpr int kStageBufOffset = (kSchedOffset + kSchedBytes + 15) / 16 * 16;
  // staged epilogue stores exist only for the wide tile: 20 KB more shared memory on the
  // 256-wide tile shrinks its L1 carveout and cost 2-5 points of tensor-pipe activity
  static constexpr bool kHasStageBuf = BN > 256;
  static constexpr int kStageBufBytes = kHasStageBuf ? kPairEpiWarps * 32 * kStageStride : 0;
  static constexpr int kTotal = kStageBufOffset + kStageBufBytes + 1024;
};

template <int BN, bool A_MN, bool B_MN, class Epi>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
    grouped_gemm_sm100_pair(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                            GroupGeom geo, Epi epi) {
  using L = PairSmem<BN>;
  constexpr int kPairStages = L::kStages;
  constexpr int kMmaN = L::kMmaN;
  constexpr int kAcc = L::kAcc;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);

  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + kPairStages;
  uint64_t* tmem_full = empty + kPairStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  int* sched = reinterpret_cast<int*>(smem + L::kSchedOffset);
  SchedTables tab{sched, sched + (kMaxGroups + 1), sched + 2 * (kMaxGroups + 1), sched + 3 * (kMaxGroups + 1),
                  sched + 4 * (kMaxGroups + 1), sched + 5 * (kMaxGroups + 1), sched + 6 * (kMaxGroups + 1),
                  sched + 7 * (kMaxGroups + 1)};

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  const int num_pairs = gridDim.x >> 1;
  const int G = geo.G;
  const int n_tiles = (geo.N + BN - 1) / BN;

  if (threadIdx.x == 0) {
    const int s0 = geo.seg[0];
    int acc = 0;
    for (int g = 0; g < G; ++g) {
      const int seg_lo = geo.rlo ? geo.rlo[g] : geo.seg[g] - s0;
      const int seg_rows = geo.rlo ? geo.rhi[g] - geo.rlo[g] : geo.seg[g + 1] - geo.seg[g];
      const int M = geo.M_fixed > 0 ? geo.M_fixed : seg_rows;
      const int K = geo.K_fixed > 0 ? geo.K_fixed : seg_rows;
      tab.tile_start[g] = acc;
      tab.m_tiles[g] = (M + kPairBM - 1) / kPairBM;
      tab.k_blocks[g] = (K + kBK - 1) / kBK;
      tab.a_base[g] = geo.a_seg ? seg_lo : g * geo.a_stride;
      tab.b_base[g] = geo.b_seg ? seg_lo : g * geo.b_stride;
      tab.n_fast[g] = geo.nfast >= 0 ? geo.nfast : (M > geo.N ? 1 : 0);
      tab.m_rows[g] = M;
      tab.row_base[g] = seg_lo;
      acc += tab.m_tiles[g] * n_tiles;
    }
    tab.tile_start[G] = acc;
    for (int s = 0; s < kPairStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 2 * kPairEpiWarps);  // every epilogue warp of both CTAs
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
  }
  constexpr uint32_t kTmemCols = kAcc * BN;
  static_assert(kTmemCols <= 512, "TMEM holds 512 columns");
  if (warp == 2) tmem_alloc_pair(tmem_base_slot, kTmemCols);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  const int total_tiles = tab.tile_start[G];

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // soft wave barrier bookkeeping (see GroupGeom::ksync)
      const bool ksync_on = geo.ksync > 0 && geo.K_fixed > 0 && geo.ksync_ctr != nullptr;
      const int spt = ksync_on ? (tab.k_blocks[0] + geo.ksync - 1) / geo.ksync : 0;
      const int base_tiles = total_tiles / num_pairs, extra = total_tiles % num_pairs;
      const unsigned nctas = gridDim.x;
      unsigned sp = 0;
      for (int tile = pair; tile < total_tiles; tile += num_pairs) {
        int g, local;
        sched_locate(tab, G, tile, g, local);
        int mt, nt;
        tile_coords(tab, g, local, n_tiles, mt, nt, geo.banded);
        const int kb_n = tab.k_blocks[g];
        // tail tile (128 rows left in the group): each CTA's A half is 64 rows (the box still
        // loads 128; the M = 128 MMA reads the first 64 of each CTA)
        const bool tail = BN == 256 && pair_tail(geo, tab, g, mt);
        const int arow = mt * kPairBM + static_cast<int>(rank) * (tail ? 64 : 128);
        const int bcol = nt * BN + static_cast<int>(rank) * (kMmaN / 2);  // + kMmaN j for MMA j
        const int abase = tab.a_base[g];
        const int bbase = tab.b_base[g];
        // the band-resident operand is kept in L2, the streaming one is evicted first
        const bool a_res = tab.n_fast[g] != 0;
        constexpr uint64_t kNormal = 0x1000000000000000ull;
        uint64_t pol_a, pol_b;
        if (geo.banded) {
          pol_a = a_res ? kL2EvictLast : kL2EvictFirst;
          pol_b = a_res ? kL2EvictFirst : kL2EvictLast;
        } else {  // panel order: the slow dimension's operand is re-read by every wave of the
                  // group -> keep it (evict-last); the fast one is shared within a wave only
          pol_a = (geo.hint && !a_res) ? kL2EvictLast : kNormal;
          pol_b = (geo.hint && a_res) ? kL2EvictLast : kNormal;
        }
        for (int kb = 0; kb < kb_n; ++kb) {
          if (ksync_on && kb % geo.ksync == 0) {
            ++sp;
            const unsigned full_sp = static_cast<unsigned>(base_tiles * spt);
            const unsigned target = sp <= full_sp ? sp * nctas
                                                  : full_sp * nctas + (sp - full_sp) * 2u * static_cast<unsigned>(extra);
            atomicAdd(geo.ksync_ctr, 1u);
            const long long t0 = clock64();
            while (*reinterpret_cast<volatile unsigned*>(geo.ksync_ctr) < target && clock64() - t0 < 40000) {
            }
          }
          mbar_wait_sleep(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          const uint32_t fbar = mapa_shared(&full[stage], 0);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * L::kStageBytes);
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < 2; ++j)
              tma_load_2d_pair_hint(sa + j * (64 * kBK * 2), &tmap_a, fbar, arow + j * 64, abase + kb * kBK, pol_a);
          } else {
            tma_load_2d_pair_hint(sa, &tmap_a, fbar, kb * kBK, abase + arow, pol_a);
          }
#pragma unroll
          for (int j = 0; j < L::kNMma; ++j) {
            if (B_MN) {
#pragma unroll
              for (int jj = 0; jj < kMmaN / 128; ++jj)
                tma_load_2d_pair_hint(sb + j * L::kBChunk + jj * (64 * kBK * 2), &tmap_b, fbar,
                                      bcol + j * kMmaN + jj * 64, bbase + kb * kBK, pol_b);
            } else {
              tma_load_2d_pair_hint(sb + j * L::kBChunk, &tmap_b, fbar, kb * kBK, bbase + bcol + j * kMmaN, pol_b);
            }
          }
          if (++stage == kPairStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    // The whole warp runs the loop (warp-uniform descriptor math lands in uniform
    // registers, no per-instruction waterfall) and one elected lane issues each MMA: the
    // issue stream must keep up with the tensor pipe while two epilogue warps share this
    // SM sub-partition.
    if (leader) {
      constexpr uint32_t idesc256 = make_idesc_bf16(kPairBM, kMmaN, A_MN, B_MN);
      constexpr uint32_t idesc128 = make_idesc_bf16(kPairBM / 2, kMmaN, A_MN, B_MN);
      constexpr uint32_t a_lbo = A_MN ? (64 * kBK * 2) : 16;
      constexpr uint32_t b_lbo = B_MN ? (64 * kBK * 2) : 16;
      constexpr uint32_t k_step_a = A_MN ? (kUMMAK * 128) : (kUMMAK * 2);
      constexpr uint32_t k_step_b = B_MN ? (kUMMAK * 128) : (kUMMAK * 2);
      const bool elected = elect_one();
      int stage = 0;
      uint32_t phase = 0;
      int iter = 0;
#ifdef PPMOE_GEMM_STATS
      long long st_empty = 0, st_full = 0, st_t0 = clock64(), st_a;
#endif
      for (int tile = pair; tile < total_tiles; tile += num_pairs, ++iter) {
        int g, local;
        sched_locate(tab, G, tile, g, local);
        const int kb_n = tab.k_blocks[g];
        int mt_, nt_;
        tile_coords(tab, g, local, n_tiles, mt_, nt_, geo.banded);
        const uint32_t idesc = BN == 256 && pair_tail(geo, tab, g, mt_) ? idesc128 : idesc256;
        const int acc = iter % kAcc;
        const uint32_t acc_phase = (iter / kAcc) & 1;
#ifdef PPMOE_GEMM_STATS
        st_a = clock64();
#endif
        mbar_wait_cluster(&tmem_empty[acc], acc_phase ^ 1);
#ifdef PPMOE_GEMM_STATS
        st_empty += clock64() - st_a;
#endif
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kb_n; ++kb) {
#ifdef PPMOE_GEMM_STATS
          st_a = clock64();
#endif
          mbar_wait_sleep(&full[stage], phase);
#ifdef PPMOE_GEMM_STATS
          st_full += clock64() - st_a;
#endif
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * L::kStageBytes);
          const uint32_t sb = sa + L::kABytes;
#pragma unroll
          for (int k = 0; k < kBK / kUMMAK; ++k) {
            const uint64_t ad = make_sdesc(sa + k * k_step_a, a_lbo, 1024);
#pragma unroll
            for (int j = 0; j < L::kNMma; ++j) {
              const uint64_t bd = make_sdesc(sb + j * L::kBChunk + k * k_step_b, b_lbo, 1024);
              if (elected) umma_bf16_pair(d_tmem + j * kMmaN, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
            }
          }
          if (elected) umma_commit_pair_mc(&empty[stage], 0x3);
          __syncwarp();
          if (++stage == kPairStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elected) umma_commit_pair_mc(&tmem_full[acc], 0x3);
        __syncwarp();
      }
#ifdef PPMOE_GEMM_STATS
      if (lane == 0 && (pair % 16) == 0)
        printf("gemm BN=%d pair %d: tiles %d cycles %lld wait tmem_empty %lld (%.1f%%) wait full %lld (%.1f%%)\n", BN,
               pair, iter, clock64() - st_t0, st_empty, 100.0 * st_empty / (clock64() - st_t0), st_full,
               100.0 * st_full / (clock64() - st_t0));
#endif
    }
    __syncwarp();
  } else if (warp >= 2) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    // kPairEpiWarps warps: warp w reads TMEM lane quarter w % 4 (the hardware rule) and
    // one of the column halves, so two warps per SM sub-partition share each tile's
    // epilogue (latency of tcgen05.ld / the stores overlaps across them).
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    constexpr int kChunksPerWarp = BN / 32 / (kPairEpiWarps / 4);
    const int row_full = static_cast<int>(rank) * 128 + q * 32 + lane;
    // M = 128 pair MMA (tail tile): each CTA's 64 rows x N land folded in its TMEM -- lanes
    // 0-63 hold columns [0, N/2), lanes 64-127 the same rows' columns [N/2, N) (measured,
    // tools/tail_probe.py) -- so lane quarter q holds rows (q & 1) * 32 + lane of this CTA's
    // half and output columns (q >> 1) * N/2 + TMEM column
    const int row_tail = static_cast<int>(rank) * 64 + (q & 1) * 32 + lane;
    const uint32_t empty_leader = mapa_shared(&tmem_empty[0], 0);
    constexpr bool kCanStage = StageTrait<Epi>::value && L::kHasStageBuf;
    uint8_t* stage_buf = smem + L::kStageBufOffset + (warp - 2) * 32 * kStageStride;
    bool staged = false;
    if constexpr (kCanStage) staged = geo.stage && epi.stage_ok();
    int iter = 0;
    for (int tile = pair; tile < total_tiles; tile += num_pairs, ++iter) {
      int g, local;
      sched_locate(tab, G, tile, g, local);
      int mt, nt;
      tile_coords(tab, g, local, n_tiles, mt, nt, geo.banded);
      const bool has_k = tab.k_blocks[g] > 0;
      const int acc = iter % kAcc;
      const uint32_t acc_phase = (iter / kAcc) & 1;
      mbar_wait_sleep(&tmem_full[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      const bool tail = BN == 256 && pair_tail(geo, tab, g, mt);
      const int m = mt * kPairBM + (tail ? row_tail : row_full);
      // TMEM column chunks of this warp, and the output column of TMEM column 0
      const int cpw = tail ? kChunksPerWarp / 2 : kChunksPerWarp;
      const int col0 = nt * BN + (tail ? (q >> 1) * (BN / 2) : 0);
      static_assert(BN != 256 || kChunksPerWarp % 4 == 0, "64-column TMEM loads, also for the folded tail");
#pragma unroll 1
      for (int c = half * cpw; c < (half + 1) * cpw; c += 2) {
        float v[64];
        tmem_ld64(taddr + c * 32, v);
        if (!has_k) {
#pragma unroll
          for (int j = 0; j < 64; ++j) v[j] = 0.f;
        }
        const bool row_ok = m < tab.m_rows[g];
        const int n0 = col0 + c * 32;
        if constexpr (kCanStage) {
          if (staged) {  // warp-uniform
            const int row = tab.row_base[g] + m;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int nn = n0 + 32 * h;
              if (nn >= geo.N) break;
              float x[32];
              if (row_ok) epi.stage_values(g, row, nn, *reinterpret_cast<const float(*)[32]>(v + 32 * h), x);
              const int valid = min(32, epi.stage_n() - nn);
              stage_store32(stage_buf, row_ok ? epi.stage_dst(g, m, row, nn, 0) : nullptr, x, valid);
              if (epi.stage_second())
                stage_store32(stage_buf, row_ok ? epi.stage_dst(g, m, row, nn, 1) : nullptr, x, valid);
            }
            continue;
          }
        }
        if (n0 < geo.N && row_ok)
          epi.template apply<32>(g, m, tab.row_base[g] + m, n0, *reinterpret_cast<const float(*)[32]>(v));
        if (n0 + 32 < geo.N && row_ok)
          epi.template apply<32>(g, m, tab.row_base[g] + m, n0 + 32, *reinterpret_cast<const float(*)[32]>(v + 32));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(empty_leader + acc * 8);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, kTmemCols);
  }
}

// --------------------------------------------------------------------------
// CUDA-core reference grouped GEMM (fp32 mode, configs with rtol 1e-4, and
// shapes the TMA path does not take). Same geometry and epilogues.
// 64x64 tile, 256 threads, 4x4 register micro-tile.
template <typename T, bool A_MN, bool B_MN, class Epi>
__global__ void __launch_bounds__(256)
    grouped_gemm_simt(const T* __restrict__ A, int lda, const T* __restrict__ B, int ldb, GroupGeom geo, Epi epi) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int g = blockIdx.z;
  const int s0 = geo.seg[0];
  const int seg_lo = geo.rlo ? geo.rlo[g] : geo.seg[g] - s0;
  const int seg_rows = geo.rlo ? geo.rhi[g] - geo.rlo[g] : geo.seg[g + 1] - geo.seg[g];
  const int M = geo.M_fixed > 0 ? geo.M_fixed : seg_rows;
  const int K = geo.K_fixed > 0 ? geo.K_fixed : seg_rows;
  const int m0 = blockIdx.y * 64;
  const int n0 = blockIdx.x * 64;
  if (m0 >= M) return;
  const int abase = geo.a_seg ? seg_lo : g * geo.a_stride;
  const int bbase = geo.b_seg ? seg_lo : g * geo.b_stride;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      const int kk = i / 64, mm = i % 64;
      const int m = m0 + mm, k = k0 + kk;
      float va = 0.f, vb = 0.f;
      if (m < M && k < K)
        va = to_f32(A_MN ? A[static_cast<size_t>(abase + k) * lda + m] : A[static_cast<size_t>(abase + m) * lda + k]);
      const int n = n0 + mm;
      if (n < geo.N && k < K)
        vb = to_f32(B_MN ? B[static_cast<size_t>(bbase + k) * ldb + n] : B[static_cast<size_t>(bbase + n) * ldb + k]);
      As[kk][mm] = va;
      Bs[kk][mm] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m < M && n0 + tx * 4 < geo.N) epi.template apply<4>(g, m, seg_lo + m, n0 + tx * 4, acc[i]);
  }
}

}  // namespace ppmoe
