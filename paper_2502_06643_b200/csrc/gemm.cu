// gemm.cu -- K5/K6: persistent grouped bf16 GEMM on tcgen05 tensor cores.
//
// Computes, for every hosted expert segment i (rows [row0_i, row0_i + rows_i)
// of the expert-major receive layout, padded to kSegAlign rows):
//   SWIGLU=true  (K5): acc = A_i W13_i^T (N = 2F, interleaved gate/up blocks of
//                      BN/2 rows, see moe_pack_w13); D = bf16(silu(g) * u)
//   SWIGLU=false (K6): D = bf16(A_i W2_i^T)
// i.e. the Mixtral SwiGLU expert FFN (reading G5) that the paper runs between
// the two all-to-alls.  fp32 accumulation in TMEM, fixed K order, no
// split-K: results are bit-identical for a row regardless of placement or G.
//
// Structure: persistent kernel, CG = 2 CTAs per cluster (one per SM of a TPC)
// cooperating on 256 x BN tiles with tcgen05.mma.cta_group::2 (M = 256), or
// CG = 1 (M = 128).  Per CTA, 192 threads:
//   warp 0      TMA producer: its own A half [128 x 64] and B half [BN/CG x 64]
//               per stage, 128-byte swizzle; completion is signalled on the
//               leader CTA's mbarrier (cta_group::2 TMA)
//   warp 1      TMEM allocator (both CTAs) + single-thread MMA issuer (leader
//               only); tcgen05.commit multicasts stage-free / accumulator-full
//               to both CTAs
//   warps 2..5  epilogue: tcgen05.ld 32x32b of this CTA's 128 accumulator
//               rows -> SwiGLU / convert -> 16-byte global stores; arrive on
//               the leader's accumulator-empty barrier; double-buffered TMEM
// Tile order (per segment): groups of kGroupM M tiles; inside a group N tiles
// outer, M tiles fastest.  Concurrent clusters share weight tiles (B) while the
// group's activation rows (A, <= 32 MiB) stay resident in the 126 MB L2, so the
// weights are streamed from HBM once per group instead of A once per N tile.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace moe {

constexpr int BK = 64;  // 64 bf16 = 128 bytes = one swizzle row
constexpr int kGemmThreads = 192;
constexpr int kSmemBudget = 200 * 1024;
constexpr int kSchedRing = 8;  // depth of the tile-scheduler ring
constexpr int kAhead = 8;      // k-blocks before a tile's end at which the leader publishes the next tile

template <int BN, int CG, bool FUSED = false>
struct GemmCfg {
  static constexpr int A_BYTES = 128 * BK * 2;
  static constexpr int B_ROWS = BN / CG;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // fused-combine epilogue: each epilogue warp stages its 32 output rows (bf16,
  // row pitch padded by 16 bytes so the lane-per-row writes are conflict-free);
  // each row then leaves as one bulk async copy (TMA engine) to its destination
  static constexpr int STAGE_PITCH = BN * 2 + 16;
  // plain / SwiGLU epilogues: each warp stages 32-row x 32-column bf16 chunks in
  // a 2 KB buffer (dense 64-byte rows) and one lane stores each chunk with a
  // TMA 2D store (async: the warp moves on to the next TMEM chunk while the
  // copy engine writes the rows).  Measured: the output stores were costing the
  // GEMMs ~10% (profiles/r1_v17_*); an LSU variant of the staged stores measured
  // equal and was removed.
  // (one 2 KB buffer per warp: 32 dense 64-byte rows, 64-byte swizzled -- see
  // epi_store_chunk_tma; a second buffer would push K5 past the shared memory that
  // lets a k_scatter CTA co-reside with it in P2P mode)
  static constexpr int EPI_BUF = 32 * 64;
  static constexpr int STAGING = FUSED ? 4 * 32 * STAGE_PITCH : 4 * EPI_BUF;
  static constexpr int BUDGET = (FUSED ? kSmemBudget : kSmemBudget + 10 * 1024) - STAGING;
  static constexpr int STAGES = (BUDGET / STAGE_BYTES) > 8 ? 8 : (BUDGET / STAGE_BYTES);
  static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                   : (2 * BN <= 256) ? 256 : 512;
  static constexpr int SMEM =
      STAGES * STAGE_BYTES + STAGING + 1024 /*align*/ + 8192 /*seg table*/ + 512 /*barriers*/;
  static_assert((2 * STAGES + 4 + 2 * kSchedRing) * 8 + 4 + 4 * kSchedRing <= 512, "barrier area");
  static constexpr int TILE_M = 128 * CG;
};

// Tiles come in two phases.  Phase A: per segment, the M tiles made only of this
// rank's own rows (P2P overlap: they are written locally before K5 starts, so
// they run while the peers' rows are still crossing NVLink).  Phase B: every
// other M tile.  Without per-tile waits phase A is empty.
struct SegSmem {
  int nseg;
  int totalA;
  int row0[kMaxExperts];
  int wrow[kMaxExperts];   // first weight row of the segment's expert
  int mtiles[kMaxExperts];
  short mA0[kMaxExperts], mA1[kMaxExperts];  // phase-A M tiles [mA0, mA1)
  int tA0[kMaxExperts + 1];                 // phase-A tile prefix
  int tB0[kMaxExperts + 1];                 // phase-B tile prefix
};

// position p among n M tiles of one phase -> (M tile index within the phase, N tile)
__device__ __forceinline__ void raster(int group_m, int ntn, int n, int local, int& mi, int& ntile) {
  if (group_m > 0) {  // groups of group_m M tiles, N outer, M fastest (A group L2-resident)
    const int per_group = group_m * ntn;
    const int g = local / per_group;
    const int r = local % per_group;
    const int gm = min(group_m, n - g * group_m);  // M tiles in this group
    ntile = r / gm;
    mi = g * group_m + r % gm;
  } else {            // groups of -group_m N tiles, M outer, N fastest (weight group L2-resident)
    const int gfull = -group_m;
    const int per_group = gfull * n;
    const int g = local / per_group;
    const int r = local % per_group;
    const int gn = min(gfull, ntn - g * gfull);
    mi = r / gn;
    ntile = g * gfull + r % gn;
  }
}

// tile -> (A row of the tile, first weight row of the expert, N tile index, segment)
__device__ __forceinline__ void decode_tile(const SegSmem& sg, int ntn, int tile_m, int group_m, int tile, int& arow,
                                            int& wrow, int& ntile, int& seg) {
  int i = 0, mtile, mi;
  if (tile < sg.totalA) {
    while (i + 1 < sg.nseg && tile >= sg.tA0[i + 1]) ++i;
    raster(group_m, ntn, sg.mA1[i] - sg.mA0[i], tile - sg.tA0[i], mi, ntile);
    mtile = sg.mA0[i] + mi;
  } else {
    const int t = tile - sg.totalA;
    while (i + 1 < sg.nseg && t >= sg.tB0[i + 1]) ++i;
    const int nA = sg.mA1[i] - sg.mA0[i];
    raster(group_m, ntn, sg.mtiles[i] - nA, t - sg.tB0[i], mi, ntile);
    mtile = mi < sg.mA0[i] ? mi : mi + nA;
  }
  seg = i;
  arow = sg.row0[i] + mtile * tile_m;
  wrow = sg.wrow[i];
}

// One warp's 32 rows x 32 bf16 columns (lane = row, packed = its 64 bytes) ->
// D[wrow0 + r][col0 .. col0 + 32): the chunk goes to the warp's 2 KB staging
// buffer (512-byte aligned) in the TMA 64-byte swizzle -- 16-byte granule g of
// row r sits at granule g ^ ((r >> 1) & 3) -- so each 16-byte store instruction
// of the warp hits 8 distinct bank groups per 8 lanes (4 wavefronts, no
// conflicts; the unswizzled lane * 64 layout was a 16-20-way conflict, ncu
// round 1); lane 0 issues the TMA 2D store after every lane wrote its row and
// fenced it for the async proxy.
__device__ __forceinline__ void epi_store_chunk_tma(uint8_t* stg, const uint32_t (&packed)[16],
                                                    const CUtensorMap* tmD, int wrow0, int col0, int lane) {
  uint8_t* buf = stg;
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // previous chunk was read
  __syncwarp();
  uint4* mine = reinterpret_cast<uint4*>(buf + lane * 64);
  const int sw = (lane >> 1) & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    mine[i ^ sw] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d_hint(tmD, buf, col0, wrow0, l2_evict_first_policy());
    bulk_commit();
  }
}

// SwiGLU of one output: silu(g) * u = g * u / (1 + e^-g) (reading G5), with the
// MUFU exp2 and reciprocal (relative error ~1e-7, far below the bf16 rounding
// that follows) instead of an IEEE division with its slow-path branch.
__device__ __forceinline__ float silu_mul(float g, float u) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + __expf(-g)));
  return g * u * r;
}

template <int BN, bool SWIGLU, int CG, bool FUSED = false>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_grouped_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   uint16_t* __restrict__ D, int ldd, const int32_t* __restrict__ seg_meta, int E, int N, int K,
                   int group_m, const SrcWait sw, int* err, unsigned* sched, const FusedRet fr, int ksplit,
                   float* __restrict__ part, long long part_stride, const __grid_constant__ CUtensorMap tmD,
                   int n_w) {
  using C = GemmCfg<BN, CG, FUSED>;
  static_assert(!(FUSED && SWIGLU), "the fused combine applies to the down projection (K6) only");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + C::STAGES * C::A_BYTES;
  static_assert(sizeof(SegSmem) <= 8192, "segment table");
  SegSmem& sg = *reinterpret_cast<SegSmem*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES + 8192);
  uint8_t* staging = smem + C::STAGES * C::STAGE_BYTES + 8192 + 512;  // per epilogue warp (see GemmCfg)
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = bars + 2 * C::STAGES + 2;
  uint64_t* sfull = bars + 2 * C::STAGES + 4;           // tile-scheduler ring
  uint64_t* sempty = sfull + kSchedRing;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + kSchedRing);
  int* sched_tile = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = (CG == 2) ? cluster_ctarank() : 0;
  const bool leader = crank == 0;
  const int cluster_id = blockIdx.x / CG;
  const int n_clusters = gridDim.x / CG;
  const int ntn = N / BN;
  const int nkb = K / BK;

  // ---- segment table -> smem (tile prefix over segments)
  if (threadIdx.x == 0) {
    const int nseg = seg_meta[0];
    // the weights hold n_w experts; the placement of the last dispatch hosts nseg here
    // (a mismatch is a caller error: latched, and the TMA zero-fills rows past n_w)
    if (blockIdx.x == 0 && nseg != n_w) atomicOr(err, kErrWeights);
    sg.nseg = nseg;
    int accA = 0, accB = 0;
    for (int i = 0; i < nseg; ++i) {
      const int rows = seg_meta[1 + E + i];
      const int mt = (rows + C::TILE_M - 1) / C::TILE_M;
      sg.row0[i] = seg_meta[1 + i];
      sg.wrow[i] = seg_meta[1 + 2 * E + i] * N;
      sg.mtiles[i] = mt;
      int a0 = 0, a1 = 0;
      if (sw.flags != nullptr && sw.me >= 0) {  // M tiles lying inside this rank's own rows [lo, hi)
        const int32_t* own = sw.seg_src + ((long long)i * sw.G + sw.me) * 3;
        const int lo = own[0] - sg.row0[i], hi = lo + own[1];
        if (own[1] > 0) {
          a0 = min(mt, (lo + C::TILE_M - 1) / C::TILE_M);
          a1 = hi >= rows ? mt : hi / C::TILE_M;
          if (a1 < a0) a1 = a0;
        }
      }
      sg.mA0[i] = (short)a0;
      sg.mA1[i] = (short)a1;
      sg.tA0[i] = accA;
      sg.tB0[i] = accB;
      accA += (a1 - a0) * ntn;
      accB += (mt - (a1 - a0)) * ntn;
    }
    sg.tA0[nseg] = accA;
    sg.tB0[nseg] = accB;
    sg.totalA = accA;
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4 * CG);
    }
    // scheduler ring: published by the leader's producer; consumed by the MMA
    // issuer, every epilogue warp and (pair mode) the peer's producer
    for (int s = 0; s < kSchedRing; ++s) {
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], CG == 2 ? 10 : 5);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // split-K (decode-sized contexts whose tiles cannot cover the SMs): tile id t =
  // output tile t / ksplit, K slice t % ksplit; each slice's fp32 partial goes to
  // part[slice] and k_splitk_reduce sums the slices in order (deterministic)
  const int total_tiles = (sg.totalA + sg.tB0[sg.nseg]) * ksplit;

  // Dynamic tile scheduler: the leader's producer takes the next tile id from a
  // global counter (atomicAdd) and publishes it through an mbarrier ring to
  // every role of both CTAs.  Clusters that run ahead simply take more tiles,
  // so the tiles in flight are always ~one wave of consecutive ids and the
  // rasterisation group's operands stay L2-resident (a static round-robin
  // schedule lets clusters drift apart by several waves).
  auto take_tile = [&](int& seq) -> int {
    const int slot = seq % kSchedRing;
    mbar_wait_cluster(&sfull[slot], (uint32_t)((seq / kSchedRing) & 1));
    const int t = reinterpret_cast<volatile int*>(sched_tile)[slot];
    ++seq;
    return t;
  };
  // A consumer's "slot read" arrival carries no data, so it is relaxed: a release at
  // cluster scope costs the MMA issuer ~1.25k cycles per tile on its critical path
  // (profiles/r2_k5_mma_issuer_trace*.json).  The slot's tile id was read and
  // branched on before the arrival, so the load completed first.
  auto release_tile = [&](int seq_after) {
    const int slot = (seq_after - 1) % kSchedRing;
    if constexpr (CG == 2) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&sempty[slot]), 0));
    else mbar_arrive(&sempty[slot]);
  };
  (void)cluster_id;
  (void)n_clusters;

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer (every CTA loads its halves)
      int stage = 0;
      uint32_t phase = 0;
      int seq = 0;
      unsigned long long ready = 0;  // P2P: source ranks whose rows have arrived
      int ready_seg = -1;            // (per-(source, segment) flags: `ready` holds for this segment)
      // P2P: this dispatch's flag value (written by k_layout earlier on the stream)
      const unsigned epoch = sw.flags != nullptr ? *(volatile const unsigned*)sw.epoch_ptr : 0u;
      // The leader takes the next tile id from the global counter and publishes it to
      // every role kAhead k-blocks before the end of the current tile: at the tile
      // boundary the MMA issuer and the peer producer find the next tile already in
      // the ring, and this producer goes straight on to its first loads (measured at
      // the boundary before: the MMA issuer waited ~1.3k cycles for the id and ~0.7k
      // for the first data, profiles/r2_k5_mma_issuer_trace.json)
      auto fetch_publish = [&]() -> int {
        const int slot = seq % kSchedRing;
        mbar_wait_cluster(&sempty[slot], (uint32_t)(((seq / kSchedRing) & 1) ^ 1));
        const int t = (int)atomicAdd(sched, 1u);
        sched_tile[slot] = t;
        if constexpr (CG == 2) {
          st_shared_cluster_u32(mapa_shared(smem_u32(&sched_tile[slot]), 1), (uint32_t)t);
          mbar_arrive_cluster(mapa_shared(smem_u32(&sfull[slot]), 1));
        }
        mbar_arrive(&sfull[slot]);
        ++seq;
        return t;
      };
      int pending = -1;  // leader: the next tile, already published
      while (true) {
        int tile;
        if (leader) {
          tile = pending >= 0 ? pending : fetch_publish();
          pending = -1;
        } else {
          tile = take_tile(seq);
          release_tile(seq);
        }
        if (tile >= total_tiles) break;
        int arow, wrow, nt, seg;
        decode_tile(sg, ntn, C::TILE_M, group_m, tile / ksplit, arow, wrow, nt, seg);
        const int ks = tile % ksplit;
        const int kb_lo = ks * nkb / ksplit, kb_hi = (ks + 1) * nkb / ksplit;
        const int a_row = arow + (int)crank * 128;
        const int b_row = wrow + nt * BN + (int)crank * C::B_ROWS;
        if (sw.flags != nullptr) {
          // P2P overlap: wait for the source ranks whose rows this CTA's half of the
          // tile holds (system-scope acquire of their arrival flags), then order
          // those generic-proxy arrivals before the TMA (async proxy) reads
          const int32_t* ss = sw.seg_src + (long long)seg * sw.G * 3;
          if (sw.flags_se != nullptr && seg != ready_seg) {  // per-(source, segment) flags
            ready = 0;
            ready_seg = seg;
          }
          bool waited = false;
          for (int s = 0; s < sw.G; ++s) {
            if (s == sw.me || ((ready >> s) & 1ull)) continue;
            const int r0 = __ldg(ss + 3 * s), n = __ldg(ss + 3 * s + 1);
            if (n == 0 || r0 >= a_row + 128 || r0 + n <= a_row) continue;
            const unsigned* word = sw.flags_se != nullptr ? sw.flags_se + s * sw.E + __ldg(sw.seg_e + seg) : sw.flags + s;
            const unsigned long long t0 = globaltimer_ns();
            unsigned v;
            do {
              asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(word) : "memory");
              if (globaltimer_ns() - t0 > sw.timeout_ns) {
                atomicOr(err, timeout_bits(kWaitRowsK5));
                break;
              }
            } while ((int)(v - epoch) < 0);
            ready |= 1ull << s;
            waited = true;
          }
          if (waited) asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        const int kb_next = max(kb_lo, kb_hi - kAhead);
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          if (leader && kb == kb_next) pending = fetch_publish();
          mbar_wait(&empty[stage], phase ^ 1);
          if constexpr (CG == 2) {
            const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            tma_load_2d_pair(&tmA, fb, smA + stage * C::A_BYTES, kb * BK, a_row);
            tma_load_2d_pair(&tmB, fb, smB + stage * C::B_BYTES, kb * BK, b_row);
          } else {
            mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
            tma_load_2d(&tmA, &full[stage], smA + stage * C::A_BYTES, kb * BK, a_row);
            tma_load_2d(&tmB, &full[stage], smB + stage * C::B_BYTES, kb * BK, b_row);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ================= MMA issuer (single thread of the leader CTA)
      constexpr uint32_t idesc = umma_idesc_bf16(C::TILE_M, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int seq = 0;
      while (true) {
        const int tile = take_tile(seq);
        if (tile >= total_tiles) {
          release_tile(seq);
          break;
        }
        release_tile(seq);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int ks = tile % ksplit;
        const int kb_lo = ks * nkb / ksplit, kb_hi = (ks + 1) * nkb / ksplit;
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(smB + stage * C::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = umma_desc_sw128(a_addr + kk * 32), bd = umma_desc_sw128(b_addr + kk * 32);
            const uint32_t accum = (kb != kb_lo || kk != 0) ? 1u : 0u;
            if constexpr (CG == 2) umma_bf16_pair(d_tmem, ad, bd, idesc, accum);
            else umma_bf16(d_tmem, ad, bd, idesc, accum);
          }
          if constexpr (CG == 2) umma_commit_pair_mc(&empty[stage], 0x3);
          else umma_commit(&empty[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (CG == 2) umma_commit_pair_mc(&tfull[acc], 0x3);
        else umma_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ================= epilogue warps 2..5 (TMEM lane quarter = warp % 4)
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    int ce_pending = -1;  // copy-engine combine: segment of this warp's last tile, not yet counted
    const uint32_t tempty_leader0 = (CG == 2) ? mapa_shared(smem_u32(&tempty[0]), 0) : 0;
    int seq = 0;
    while (true) {
      const int tile = take_tile(seq);
      __syncwarp();
      if (lane == 0) release_tile(seq);
      if (tile >= total_tiles) break;
      int arow, wrow, nt, seg;
      decode_tile(sg, ntn, C::TILE_M, group_m, tile / ksplit, arow, wrow, nt, seg);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const long long grow = arow + (int)crank * 128 + q * 32 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      if (ksplit > 1) {
        // fp32 partial of K slice tile % ksplit (raw accumulators; the reduction
        // kernel applies the epilogue)
        float* prow = part + (long long)(tile % ksplit) * part_stride + grow * N + (long long)nt * BN;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t v[32];
          tmem_ld32(taddr + c, v);
          tmem_ld_wait();
          float4* dst = reinterpret_cast<float4*>(prow + c);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                 __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
        }
      } else if constexpr (SWIGLU) {
        uint8_t* stg = staging + (size_t)(warp - 2) * C::EPI_BUF;
        const long long wrow0 = arow + (int)crank * 128 + q * 32;  // first row of this warp
#pragma unroll 1
        for (int c = 0; c < BN / 2; c += 32) {
          uint32_t g[32], u[32];
          tmem_ld32(taddr + c, g);
          tmem_ld32(taddr + BN / 2 + c, u);
          tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float g0 = __uint_as_float(g[2 * i]), g1 = __uint_as_float(g[2 * i + 1]);
            const float u0 = __uint_as_float(u[2 * i]), u1 = __uint_as_float(u[2 * i + 1]);
            const float h0 = silu_mul(g0, u0), h1 = silu_mul(g1, u1);
            packed[i] = pack_bf16x2(h0, h1);
          }
          epi_store_chunk_tma(stg, packed, &tmD, (int)wrow0, nt * (BN / 2) + c, lane);
        }
      } else if constexpr (FUSED) {
        // Fused combine: the row belongs to source s (rows of s are contiguous in the
        // segment) and goes to s's return buffer at the item's send-order slot, over
        // NVLink.  The warp stages its 32 rows in shared memory (16-byte granules,
        // XOR-swizzled by row), releases the accumulator, then writes row by row with
        // all 32 lanes so every NVLink store is a whole contiguous row segment.
        constexpr int PITCH = C::STAGE_PITCH;
        uint8_t* stg = staging + (size_t)(warp - 2) * 32 * PITCH;
        uint8_t* my_row = stg + (size_t)lane * PITCH;
        unsigned long long dst_row = 0;
        const int32_t* ss = fr.seg_src + (long long)seg * fr.G * 3;
        for (int s = 0; s < fr.G; ++s) {
          const int r0 = __ldg(ss + 3 * s), n = __ldg(ss + 3 * s + 1);
          if (grow >= r0 && grow < r0 + n) {
            dst_row = reinterpret_cast<unsigned long long>(
                fr.ret_table[s] + ((long long)__ldg(ss + 3 * s + 2) + (grow - r0)) * ldd + (long long)nt * BN);
            break;
          }
        }
        bulk_wait_read_all();  // this lane's previous row copy has left the staging row
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t v[32];
          tmem_ld32(taddr + c, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 4; ++i)
            reinterpret_cast<uint4*>(my_row)[c / 8 + i] =
                make_uint4(pack_bf16x2(__uint_as_float(v[8 * i + 0]), __uint_as_float(v[8 * i + 1])),
                           pack_bf16x2(__uint_as_float(v[8 * i + 2]), __uint_as_float(v[8 * i + 3])),
                           pack_bf16x2(__uint_as_float(v[8 * i + 4]), __uint_as_float(v[8 * i + 5])),
                           pack_bf16x2(__uint_as_float(v[8 * i + 6]), __uint_as_float(v[8 * i + 7])));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {  // accumulator drained into smem: the MMA may reuse it
          if constexpr (CG == 2) mbar_arrive_cluster(tempty_leader0 + acc * 8);
          else mbar_arrive(&tempty[acc]);
        }
        // every lane ships its own row (a contiguous BN-column segment of the
        // destination row) with one bulk copy; the copy engine keeps the NVLink
        // stores in flight while the warp moves on to the next accumulator
        fence_proxy_async_smem();
        if (dst_row != 0) {
          bulk_s2g(reinterpret_cast<void*>(dst_row), smem_u32(my_row), BN * 2);
          bulk_commit();
        }
      } else {
        uint8_t* stg = staging + (size_t)(warp - 2) * C::EPI_BUF;
        const long long wrow0 = arow + (int)crank * 128 + q * 32;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t v[32];
          tmem_ld32(taddr + c, v);
          tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) packed[i] = pack_bf16x2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
          epi_store_chunk_tma(stg, packed, &tmD, (int)wrow0, nt * BN + c, lane);
        }
      }
      if (FUSED && ksplit > 1) {  // (never launched: split-K is not combined with the fused combine)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) mbar_arrive_cluster(tempty_leader0 + acc * 8);
          else mbar_arrive(&tempty[acc]);
        }
      }
      if constexpr (!FUSED) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) mbar_arrive_cluster(tempty_leader0 + acc * 8);
          else mbar_arrive(&tempty[acc]);
        }
        if (fr.segdone != nullptr && ksplit == 1 && lane == 0) {
          // copy-engine combine (after the accumulator is released): the previous
          // tile's stores of this warp -- every bulk group but this tile's BN / 32 --
          // are complete, then its segment's counter moves (one tile late, so the warp
          // never waits for the stores it has just issued; the copy engines read
          // through L2, a GPU-scope release orders them)
          if (ce_pending >= 0) {
            asm volatile("cp.async.bulk.wait_group %0;" ::"n"(BN / 32) : "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(fr.segdone + ce_pending) : "memory");
          }
          ce_pending = seg;
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if constexpr (FUSED) {  // peer stores complete and visible before the ready flag
      bulk_wait_all();
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __threadfence_system();
    } else {                // the epilogue's TMA stores have landed before the kernel ends
      if (lane == 0) bulk_wait_all();
      if (lane == 0 && ce_pending >= 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(fr.segdone + ce_pending) : "memory");
      }
      __syncwarp();
    }
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  // the last CTA to leave resets the scheduler counters for the next launch
  if (threadIdx.x == 0) {
    if (atomicAdd(&sched[1], 1u) == gridDim.x - 1) {
      atomicExch(&sched[0], 0u);
      atomicExch(&sched[1], 0u);
    }
  }
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS)
                   : "memory");
  }
}

// ------------------------------------------------------------------ host side
int gemm_block_n(int N, bool swiglu) {
  if (swiglu) return (N % 256 == 0 && (N / 2) % 128 == 0) ? 256 : 128;
  if (N % 256 == 0) return 256;
  if (N % 128 == 0) return 128;
  return 64;
}

int gemm_b_box_rows(int N, bool swiglu, int cg) { return gemm_block_n(N, swiglu) / cg; }

template <int BN, bool SWIGLU, int CG, bool FUSED = false>
static cudaError_t launch_impl(const void* tmA, const void* tmB, uint16_t* D, int ldd, const int32_t* seg_meta, int E,
                               int n_w, int N, int K, int num_sms, const SrcWait& sw, int* err, unsigned* sched,
                               const FusedRet& fr, cudaStream_t s, int ksplit, float* part, long long part_stride,
                               const void* tmD) {
  using C = GemmCfg<BN, CG, FUSED>;
  auto kern = k_grouped_gemm<BN, SWIGLU, CG, FUSED>;
  static unsigned long long configured = 0;  // per device
  if (first_time_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
  }
  const CUtensorMap& a = *reinterpret_cast<const CUtensorMap*>(tmA);
  const CUtensorMap& b = *reinterpret_cast<const CUtensorMap*>(tmB);
  // output map of the TMA-store epilogue (any valid map when the epilogue does not
  // use it: fused combine, split-K partials)
  const CUtensorMap& dmap = *reinterpret_cast<const CUtensorMap*>(tmD ? tmD : tmA);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((num_sms / CG) * CG);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // rasterisation group: about 32 MiB of A rows per group (K bytes per row)
  // (MOE_GEMM_GROUP_M overrides for tuning; a negative value -g selects groups
  // of g N tiles instead)
  static bool env_read = false;
  static int env_group = 0;
  if (!env_read) {
    const char* env = getenv("MOE_GEMM_GROUP_M");
    env_group = env ? atoi(env) : 0;
    env_read = true;
  }
  // measured on B200 with the dynamic scheduler (profiles/r1_v5_gemm_group_sweep.txt):
  // K = 4096 -> 16 M tiles (32 MiB of A), K = 14336 -> 8 M tiles (~58 MiB)
  const long long target = K <= 8192 ? (32ll << 20) : (64ll << 20);
  int group_m = (int)(target / ((long long)C::TILE_M * K * 2));
  if (group_m < 1) group_m = 1;
  if (group_m > 64) group_m = 64;
  if (env_group != 0) group_m = env_group;
  return cudaLaunchKernelEx(&cfg, kern, a, b, D, ldd, seg_meta, E, N, K, group_m, sw, err,
                            sched, fr, ksplit, part, part_stride, dmap, n_w);
}

cudaError_t launch_grouped_gemm(const void* tmA, const void* tmB, uint16_t* D, int ldd, const int32_t* seg_meta,
                                int E, int n_w, int N, int K, bool swiglu, int cg, int num_sms, const SrcWait& sw, int* err,
                                unsigned* sched, const FusedRet& fr, cudaStream_t s, int ksplit, float* part,
                                long long part_stride, const void* tmD) {
  const int bn = gemm_block_n(N, swiglu);
  if (ksplit < 1) ksplit = 1;
  const bool fused = fr.enabled && !swiglu;
#define MOE_GO(BN_, SW_, CG_, FU_) \
  launch_impl<BN_, SW_, CG_, FU_>(tmA, tmB, D, ldd, seg_meta, E, n_w, N, K, num_sms, sw, err, sched, fr, s, ksplit, part, \
                                  part_stride, tmD)
#define MOE_GO2(BN_, CG_) (fused ? MOE_GO(BN_, false, CG_, true) : MOE_GO(BN_, false, CG_, false))
  if (cg == 2) {
    if (swiglu) return bn == 256 ? MOE_GO(256, true, 2, false) : MOE_GO(128, true, 2, false);
    if (bn == 256) return MOE_GO2(256, 2);
    if (bn == 128) return MOE_GO2(128, 2);
    return MOE_GO2(64, 2);
  }
  if (swiglu) return bn == 256 ? MOE_GO(256, true, 1, false) : MOE_GO(128, true, 1, false);
  if (bn == 256) return MOE_GO2(256, 1);
  if (bn == 128) return MOE_GO2(128, 1);
  return MOE_GO2(64, 1);
#undef MOE_GO2
#undef MOE_GO
}

// Split-K reduction (plain GEMM): D[row][c] = bf16( sum_{slice ascending} part[slice][row][c] )
// over every row of every segment's padded M range (fp32, fixed order).
__global__ void __launch_bounds__(256) k_splitk_reduce(const float* __restrict__ part, long long part_stride, int S,
                                                       const int32_t* __restrict__ seg_meta, int E, int N, int tile_m,
                                                       uint16_t* __restrict__ D, int ldd) {
  const int nseg = seg_meta[0];
  const int c4 = N / 4;
  for (int i = 0; i < nseg; ++i) {
    const long long r0 = seg_meta[1 + i];
    const int rows = seg_meta[1 + E + i];
    const long long n = (long long)((rows + tile_m - 1) / tile_m) * tile_m * c4;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
      const long long row = r0 + p / c4;
      const int c = (int)(p % c4) * 4;
      const float* src = part + row * N + c;
      float4 acc = *reinterpret_cast<const float4*>(src);
      for (int sl = 1; sl < S; ++sl) {
        const float4 v = *reinterpret_cast<const float4*>(src + sl * part_stride);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      uint2 o;
      o.x = pack_bf16x2(acc.x, acc.y);
      o.y = pack_bf16x2(acc.z, acc.w);
      *reinterpret_cast<uint2*>(D + row * ldd + c) = o;
    }
  }
}

cudaError_t launch_splitk_reduce(const float* part, long long part_stride, int S, const int32_t* seg_meta, int E,
                                 int N, int cg, uint16_t* D, int ldd, int num_sms, cudaStream_t s) {
  k_splitk_reduce<<<2 * num_sms, 256, 0, s>>>(part, part_stride, S, seg_meta, E, N, 128 * cg, D, ldd);
  return cudaGetLastError();
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_tmap_2d(void* tmap_out, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  return make_tmap_2d_ld(tmap_out, base, rows, cols, cols, box_rows);
}

bool make_tmap_store_2d(void* tmap_out, const void* base, uint64_t rows, uint64_t cols, uint64_t ld) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {32, 32};  // one epilogue chunk: 32 rows x 32 bf16 (64-byte rows, 64-byte swizzle)
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(tmap_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_2d_ld(void* tmap_out, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                     uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(tmap_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, bool SWIGLU, int CG, bool FUSED = false>
static void preload_one() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, (const void*)k_grouped_gemm<BN, SWIGLU, CG, FUSED>);
  cudaFuncSetAttribute(k_grouped_gemm<BN, SWIGLU, CG, FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       GemmCfg<BN, CG, FUSED>::SMEM);
}

void preload_gemm_kernels() {
#define MOE_PL(CG_)                                                                                        \
  preload_one<256, true, CG_>(), preload_one<128, true, CG_>(), preload_one<256, false, CG_>(),           \
      preload_one<128, false, CG_>(), preload_one<64, false, CG_>(), preload_one<256, false, CG_, true>(), \
      preload_one<128, false, CG_, true>(), preload_one<64, false, CG_, true>()
  MOE_PL(1);
  MOE_PL(2);
#undef MOE_PL
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, (const void*)k_splitk_reduce);
}

}  // namespace moe
