// fs_gram_tc.cu — pairwise mask-overlap (Gram) matrix on 5th-gen tensor cores.
//
// Reference: similarity_matrix() issues one pair_counts() per i<j pair
// (analytics.py:174-181, _kernels_np.py:26-32): |A & B| over wet masks.  Stacking the
// binarized masks as X (k x P, 0/1) gives I = X X^T, a dense contraction over pixels.
//
// Engine: tcgen05.mma.cta_group::1.kind::i8 (u8 x u8 -> s32 accumulators in TMEM).
//  * Masks stay bit-packed in HBM (P/8 bytes each) in the tile-interleaved layout, so
//    one pixel tile of a whole 256-mask panel is a single contiguous 32 KB block.  A
//    TMA warp streams those blocks (3-D tensor map, SWIZZLE_128B/64B) into a raw SMEM
//    ring; expander warps turn each 128-px slice of every row into 0/1 bytes written
//    straight into the canonical K-major SWIZZLE_128B operand layout (one 128-B row
//    per mask); one elected thread issues the MMAs.  Both SMEM reads of the expanders
//    (swizzled raw) and their writes (swizzled operand) are bank-conflict free.
//  * Masks are tiled in panels of PANEL (128 or 256) rows.  A diagonal tile (I == J)
//    uses ONE operand panel as both A and B: every mask row is expanded once per K
//    step and read by the MMA as M rows and as N columns.
//  * PANEL = 256: two M=128 halves.  Diagonal tiles issue half 0 with N=256 and half 1
//    with N=128 (columns 128..255) — the lower-left quadrant is the transpose of the
//    upper-right one and is mirrored by the reduce kernel (3/4 of the full work).
//  * FP4 variant (diagonal tiles): tcgen05.mma.kind::mxf4.block_scale (e2m1 operands,
//    every UE8M0 block scale = 1.0, f32 accumulators), twice the int8 MMA rate.  A wet
//    bit becomes the e2m1 code 0b0010 (= 1.0), so products are exact 0/1 and the f32
//    sums are exact integers while a CTA's K chunk stays <= 2^24 px.  Because a Gram
//    entry is invariant under any permutation of the pixel (K) axis applied to both
//    operands, the expander does not keep pixel order: nibble q of output word j is bit
//    4q + j of the packed word, i.e. out_j = (w >> j-1) & 0x22222222 — two ops per 8 px.
//  * Pixels (K) are split over CTAs; each CTA writes an int32 partial tile and a reduce
//    kernel sums partials into the exact int64 Gram.  Partials are exact: a CTA's K
//    range is far below 2^31 pixels.
#include <cstdio>
#include <cstdlib>

#include "fs_bitslice.cuh"
#include "fs_tcgen05.cuh"

namespace fs {

namespace tc {

// warp roles (Cfg::k*Warp*): w0 TMEM alloc + MMA; w1..kExpWarps expanders + epilogue;
// then the TMA warp; then (FUSE) 4 per-pixel counter warps of the fused overlap pass
constexpr int kFuseBins = 288;      // SMEM histogram / RGBA table (k <= 256 -> <= 257 bins)
constexpr int kSmemBudget = 200 * 1024;
constexpr int kRawDepth = 2;

// 256-mask fused diagonal: raw ring depth (= counter warps up to 4).  4 x 32 KB raw
// units leave room for 2 operand stages.  Depth 2 (2 counter warps, 4 operand stages)
// measured slower, 1.41 vs 1.08 ms at C2: two counter warps cannot keep up
// (profiles/r3f/parts.txt)
#ifndef FS_FUSE_DEPTH_256
#define FS_FUSE_DEPTH_256 4
#endif
constexpr int kFuseDepth256 = FS_FUSE_DEPTH_256;

#ifndef FS_EXP_BATCH
#define FS_EXP_BATCH 2
#endif
constexpr uint64_t kF4MaxChunkPx = 1ull << 24;  // f32 sums stay exact below this

template <int PANEL, bool DIAG, bool FP4 = false, bool FUSE = false, int FD = 4>
struct Cfg {
  // raw ring depth.  FUSE: a multiple of the counter-warp count (unit u lives in slot
  // u % kDepth and is counted by warp u % kCntWarps), so a counter warp only ever waits
  // on its own slots, in order, and can never run a full mbarrier phase ahead of them.
  static constexpr int kDepth = FUSE ? FD : kRawDepth;
  // FUSE: counter warps; warp cw counts units cw, cw + kCntWarps, ... (FD = raw ring depth)
  static constexpr int kCntWarps = FUSE ? (FD < 4 ? FD : 4) : 0;
  static constexpr int kExtraBytes =
      FUSE ? (kCntWarps * 32 * kTileTb * 4 + 2 * kFuseBins * 4) : 0;
  static constexpr int kBudget = FUSE ? (232448 - 1024 - 256) : kSmemBudget;
  static constexpr int kRegions = DIAG ? 1 : 2;
  // expander work item = one 16-B raw chunk of one operand row per K stage (FP4: 2 per
  // row).  8 expander warps when there are >= 256 items (latency hiding: each thread's
  // loads -> expand -> stores chain is short), else 4
  static constexpr int kChunks = FP4 ? 2 : 1;
  static constexpr int kItems = PANEL * kRegions * kChunks;
  static constexpr int kExpWarps = (kItems >= 256) ? 8 : 4;
  static constexpr int kExpThreads = 32 * kExpWarps;
  static constexpr int kItemsPerThread = kItems / kExpThreads;
  static_assert(kItems % kExpThreads == 0, "expander items must split evenly");
  static constexpr int kTmaWarp = kExpWarps + 1;
  static constexpr int kCntWarp0 = kExpWarps + 2;
  static constexpr int kThreadsTotal = 32 * (kExpWarps + 2 + kCntWarps);
  static constexpr int kRawRow = (PANEL == 256 && !DIAG) ? 64 : 128;  // raw bytes/row/unit
  static constexpr int kRawPerStage = FP4 ? 32 : 16;  // raw bytes per row per K stage
  static constexpr int kStagesPerUnit = kRawRow / kRawPerStage;
  static constexpr int kRawUnitBytes = kRegions * PANEL * kRawRow;
  static constexpr int kRegionBytes = PANEL * 128;
  static constexpr int kStageBytes = kRegionBytes * kRegions;
  static constexpr int kStagesFit =
      (kBudget - kDepth * kRawUnitBytes - kExtraBytes) / kStageBytes;
  static constexpr int kStages = kStagesFit > 8 ? 8 : kStagesFit;
  // expanders fill kBatch operand stages per pass with one proxy fence: the fence waits
  // for the pass's shared stores to drain, so batching halves those waits when the
  // operand ring is deep enough to keep the MMA fed (PANEL 128: 8 stages)
  static constexpr int kBatch = (kStages >= 6 && kStagesPerUnit % 2 == 0) ? FS_EXP_BATCH : 1;
  static constexpr int kHalves = PANEL / 128;
  static constexpr uint32_t kTmemCols = (PANEL == 256 || FP4) ? 512u : 128u;
  static_assert(!FP4 || DIAG, "FP4 path is for diagonal tiles (off-diagonal accumulators fill TMEM)");
  static_assert(!FUSE || DIAG, "the fused overlap pass runs in diagonal tiles");
  // FUSE: counter warp u % kCntWarps takes unit u from slot u % kDepth.  With kDepth a
  // multiple of kCntWarps the previous occupant of that slot (unit u - kDepth) was
  // counted by the same warp, so when the warp waits for unit u the slot holds
  // u - kDepth or u and the phase parity tells them apart.  Otherwise the previous
  // occupant belongs to another warp, the expanders may still hold the slot two phases
  // back, and the parity wait would pass on stale data (the parity tests caught it with
  // 4 counter warps at depth 2 and 3).
  static_assert(!FUSE || kDepth % kCntWarps == 0, "counter warp u % kCntWarps must own slot u % kDepth");
  static constexpr int kSmemBytes = kDepth * kRawUnitBytes + kStages * kStageBytes + kExtraBytes +
                                    1024 /*align*/ + 256 /*barriers*/;
  static_assert(kStages >= 2, "operand ring too shallow");
};

template <int PANEL, bool DIAG, bool FP4, bool FUSE, int FD>
__global__ void __launch_bounds__(Cfg<PANEL, DIAG, FP4, FUSE, FD>::kThreadsTotal, 1)
    k_gram_tc(const __grid_constant__ CUtensorMap tm, uint32_t npanels, uint32_t kchunks,
              uint64_t units_per_chunk, uint64_t total_units, int32_t *__restrict__ partial,
              const OverlapArgs ov, uint32_t kmasks) {
  using C = Cfg<PANEL, DIAG, FP4, FUSE, FD>;
  constexpr int kRawDepth = C::kDepth;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  const uint32_t pad = (1024u - (raw_addr & 1023u)) & 1023u;
  uint8_t *smem = smem_raw + pad;
  const uint32_t smem_base = raw_addr + pad;
  const uint32_t raw_base = smem_base;                                  // raw ring
  const uint32_t op_base = smem_base + kRawDepth * C::kRawUnitBytes;    // operand stages
  uint8_t *extra = smem + kRawDepth * C::kRawUnitBytes + C::kStages * C::kStageBytes;
  uint32_t *cnt_tb = reinterpret_cast<uint32_t *>(extra);        // FUSE: 4 x 32 x kTileTb
  uint32_t *sh_hist = cnt_tb + C::kCntWarps * 32 * kTileTb;      // FUSE: kFuseBins
  uint32_t *sh_lut = sh_hist + kFuseBins;                        // FUSE: kFuseBins
  uint64_t *full = reinterpret_cast<uint64_t *>(extra + C::kExtraBytes);
  uint64_t *empty = full + C::kStages;
  uint64_t *raw_full = empty + C::kStages;
  uint64_t *raw_empty = raw_full + kRawDepth;
  uint64_t *tmem_full = raw_empty + kRawDepth;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  // tile decode: blockIdx.x = tile * kchunks + kc
  const uint32_t tile = blockIdx.x / kchunks;
  const uint32_t kc = blockIdx.x % kchunks;
  uint32_t I, J;
  if (DIAG) {
    I = J = tile;
  } else {
    uint32_t t = tile;
    I = 0;
    while (t >= npanels - 1 - I) {
      t -= npanels - 1 - I;
      ++I;
    }
    J = I + 1 + t;
  }
  const uint64_t u0 = (uint64_t)kc * units_per_chunk;
  const uint64_t u1 = min(u0 + units_per_chunk, total_units);
  const int nunits = u1 > u0 ? (int)(u1 - u0) : 0;
  const int nst = nunits * C::kStagesPerUnit;
  // a single 128-mask panel holding k < 128 masks: MMA N, expanded operand rows and
  // counted rows shrink to n16 = roundup(k, 16).  Rows >= k of the raw tiles are TMA
  // out-of-bounds zeros; operand rows >= n16 are never written and only feed
  // accumulator rows / columns >= k, which k_gram_reduce never reads.
  constexpr bool kNarrow = PANEL == 128 && FP4 && DIAG;
  const uint32_t kin = kmasks > I * PANEL ? kmasks - I * PANEL : 0u;
  const uint32_t n16 = kNarrow ? (kin >= 128u ? 128u : ((kin + 15u) & ~15u)) : (uint32_t)PANEL;

  if (tid == 0) {
    ptx::prefetch_tmap(&tm);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&full[s], C::kExpThreads);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kRawDepth; ++s) {
      ptx::mbar_init(&raw_full[s], 1);
      ptx::mbar_init(&raw_empty[s], FUSE ? C::kExpThreads + 32 : C::kExpThreads);
    }
    ptx::mbar_init(tmem_full, 1);
    ptx::fence_mbar_init();
  }
  const bool lut_sh = FUSE && ov.rgba != nullptr;
  if (FUSE && warp >= C::kCntWarp0) {
    for (int i = tid - 32 * C::kCntWarp0; i < kFuseBins; i += 32 * C::kCntWarps) {
      sh_hist[i] = 0;
      sh_lut[i] = lut_sh && (uint32_t)i < ov.nbins ? rgba_word(i, ov.n_inputs, ov.lut) : 0u;
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     ptx::smem_u32(tmem_slot)),
                 "n"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  if (FP4) {
    // all block scales = 1.0: SFA / SFB columns [kSfCol, kSfCol + 32), every lane
    if (warp >= 1 && warp <= 4) {
      const uint32_t lanes = (uint32_t)((warp & 3) * 32) << 16;
      tmem_st16(tmem + lanes + kSfCol, kSfOnes);
      tmem_st16(tmem + lanes + kSfCol + 16, kSfOnes);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
  }

  if (warp == 0) {
    // ===== MMA issuer =====
    if (lane == 0 && nst > 0) {
      const uint32_t idA = kNarrow ? idesc_mxf4(128, (int)(n16 > 0 ? n16 : 16))
                           : (FP4 ? idesc_mxf4(128, PANEL) : idesc_i8(128, PANEL));
      constexpr uint32_t idB = FP4 ? idesc_mxf4(128, 128) : idesc_i8(128, 128);
      const uint32_t sfa = tmem + kSfCol, sfb = tmem + kSfCol + 16;
      // descriptors = the stage-0 descriptor + byte offset / 16 (the 14-bit start field
      // never carries below 256 KB): one add per MMA keeps the lone issuing thread's
      // dependent chain short — at small N the issue loop, not the tensor pipe, sets the
      // pace (tools/probes/mma_probe.cu)
      const uint64_t d_op = sw128_desc(op_base);
      for (int j = 0; j < nst; ++j) {
        const int s = j % C::kStages;
        ptx::mbar_wait(&full[s], (uint32_t)((j / C::kStages) & 1));
        fence_after();
        const uint64_t d_a = d_op + (uint64_t)((uint32_t)(s * C::kStageBytes) >> 4);
        const uint64_t d_b = DIAG ? d_a : d_a + (uint64_t)(C::kRegionBytes >> 4);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {  // 4 MMAs of 32 B of K per 128-B operand row
          const uint32_t acc = (j > 0 || ks > 0) ? 1u : 0u;
#pragma unroll
          for (int h = 0; h < C::kHalves; ++h) {
            const uint64_t adesc = d_a + (uint64_t)((h * 128 * 128 + ks * 32) >> 4);
            if (DIAG && PANEL == 256 && h == 1) {
              // rows 128..255 x cols 128..255 only
              const uint64_t bdesc = d_b + (uint64_t)((128 * 128 + ks * 32) >> 4);
              if (FP4)
                mma_mxf4(tmem + 256u, adesc, bdesc, idB, acc, sfa, sfb);
              else
                mma_i8(tmem + 256u, adesc, bdesc, idB, acc);
            } else {
              const uint64_t bdesc = d_b + (uint64_t)((ks * 32) >> 4);
#ifndef FS_PROBE_NO_MMA  // timing experiment only: the kernel without its main MMAs
              if (FP4)
                mma_mxf4(tmem + (uint32_t)(h * PANEL), adesc, bdesc, idA, acc, sfa, sfb);
              else
                mma_i8(tmem + (uint32_t)(h * PANEL), adesc, bdesc, idA, acc);
#endif
            }
          }
        }
#ifdef FS_PROBE_PLAIN_ARRIVE  // timing experiment only (with FS_PROBE_NO_MMA)
        ptx::mbar_arrive(&empty[s]);
#else
        mma_commit(&empty[s]);
#endif
      }
      mma_commit(tmem_full);
    }
    __syncwarp();
  } else if (warp == C::kTmaWarp) {
    // ===== TMA loader: one contiguous [PANEL rows][raw row] box per region per unit =====
    if (lane == 0) {
      constexpr int kUnitsPerTile = 128 / C::kRawRow;
      for (int u = 0; u < nunits; ++u) {
        const int ru = u % kRawDepth;
        if (u >= kRawDepth) ptx::mbar_wait(&raw_empty[ru], (uint32_t)(((u / kRawDepth) - 1) & 1));
        const uint64_t gu = u0 + (uint64_t)u;
        const int c0 = (int)(gu % kUnitsPerTile) * (C::kRawRow / 4);
        const int c2 = (int)(gu / kUnitsPerTile);
        ptx::mbar_arrive_expect_tx(&raw_full[ru], C::kRawUnitBytes);
#pragma unroll
        for (int r = 0; r < C::kRegions; ++r) {
          const uint32_t panel = r == 0 ? I : J;
          ptx::tma_load_3d(smem + ru * C::kRawUnitBytes + r * PANEL * C::kRawRow, &tm, c0,
                           (int)(panel * PANEL), c2, &raw_full[ru]);
        }
      }
    }
    __syncwarp();
  } else if (FUSE && warp >= C::kCntWarp0) {
    // ===== counters: the fused overlap pass over the same raw tiles =====
    // warp cw takes units cw, cw+4, ...: lane = word of the 1024-px tile, a bit-sliced
    // adder over all PANEL mask rows, then the tile epilogue (histogram, counts, RGBA).
    const int cw = warp - C::kCntWarp0;
    uint32_t off[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      off[j] = ((((uint32_t)lane >> 2) ^ (uint32_t)j) << 4) + ((uint32_t)lane & 3u) * 4u;
    for (int u = cw; u < nunits; u += C::kCntWarps) {
      const int ru = u % kRawDepth;
      ptx::mbar_wait(&raw_full[ru], (uint32_t)((u / kRawDepth) & 1));
      const uint32_t rb = raw_base + ru * C::kRawUnitBytes;
#ifdef FS_PROBE_NO_COUNT  // timing experiment only
      __syncwarp();
      ptx::mbar_arrive(&raw_empty[ru]);
      continue;
#endif
      HSCounter<5> hc;
      hc.reset();
#pragma unroll 1
      for (int g16 = 0; g16 < (int)(n16 / 16); ++g16) {
        uint32_t d[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t addr = rb + (uint32_t)(g16 * 16 + j) * 128u + off[j & 7];
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(d[j]) : "r"(addr) : "memory");
        }
        hc.add16(d);
      }
      __syncwarp();
      ptx::mbar_arrive(&raw_empty[ru]);
      uint32_t cnt32[32];
      hc.extract1(cnt32);
#ifdef FS_PROBE_NO_EMIT  // timing experiment only
      if (cnt32[lane & 31] == 0xFFFFFFFFu) ov.counts[0] = 0;  // keep the count live
      continue;
#endif
      if (ov.partial16 != nullptr)  // multi-panel: this panel's counts, summed later
        emit_partial16(cnt32, u0 + (uint64_t)u, lane, cnt_tb + cw * 32 * kTileTb,
                       ov.partial16 + (uint64_t)I * ov.part_pitch);
      else
        emit_tile(cnt32, u0 + (uint64_t)u, lane, cnt_tb + cw * 32 * kTileTb, ov, sh_hist,
                  ov.bins != nullptr, sh_lut, lut_sh);
    }
  } else {
    // ===== expanders: raw bits (swizzled) -> 0/1 bytes in SW128 K-major operand =====
    const uint32_t ptid = (uint32_t)(tid - 32);
    constexpr int kB = C::kBatch;  // stages per pass (never straddles a raw unit)
    // item i: row (i % rows) of all regions, raw chunk (i / rows); thread ptid takes
    // items ptid, ptid + kExpThreads, ... (PANEL 256: both chunks of one row)
    const uint32_t rows_rt = kNarrow ? n16 : (uint32_t)(PANEL * C::kRegions);
    uint32_t it_r[C::kItemsPerThread], it_rr[C::kItemsPerThread], it_h[C::kItemsPerThread];
    bool it_on[C::kItemsPerThread];
#pragma unroll
    for (int m = 0; m < C::kItemsPerThread; ++m) {
      const uint32_t idx = ptid + (uint32_t)m * C::kExpThreads;
      const uint32_t row = kNarrow ? (rows_rt ? idx % rows_rt : 0u) : idx % (PANEL * C::kRegions);
      it_h[m] = kNarrow ? (rows_rt ? idx / rows_rt : 0u) : idx / (PANEL * C::kRegions);
      it_r[m] = row / PANEL;
      it_rr[m] = row % PANEL;
      it_on[m] = !kNarrow || idx < rows_rt * C::kChunks;
    }
    // raw loads of pass p + 1 are issued right after pass p's operand stores and before
    // its proxy fence, so the fence's wait for the stores to drain overlaps the next
    // pass's shared-memory load latency (the accesses are volatile asm, kept in order)
    auto load_pass = [&](int jp, uint4 (&vv)[kB][C::kItemsPerThread]) {
      const int up = jp / C::kStagesPerUnit;
      const int subp = jp % C::kStagesPerUnit;
      const int rup = up % kRawDepth;
      if (subp == 0) ptx::mbar_wait(&raw_full[rup], (uint32_t)((up / kRawDepth) & 1));
      const uint32_t rbase = raw_base + rup * C::kRawUnitBytes;
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const int sub = subp + b;
#pragma unroll
        for (int m = 0; m < C::kItemsPerThread; ++m) {
          if (!it_on[m]) continue;
          const uint32_t rr = it_rr[m];
          const uint32_t sw = C::kRawRow == 128 ? (rr & 7u) : ((rr >> 1) & 3u);
          const uint32_t rrow = rbase + it_r[m] * PANEL * C::kRawRow + rr * C::kRawRow;
          const uint32_t c = FP4 ? (uint32_t)(2 * sub) + it_h[m] : (uint32_t)sub;
          vv[b][m] = ld_shared_v4(rrow + ((c ^ sw) << 4));
        }
      }
    };
    // (one stage per pass only: with two-stage passes, the 128-mask panel, holding the
    // next pass's loads across the fence measured 2 % slower)
    constexpr bool kPrefetch = kB == 1;
    uint4 v[kB][C::kItemsPerThread];
    if (kPrefetch && nst > 0) load_pass(0, v);
    for (int j = 0; j < nst; j += kB) {
      const int u = j / C::kStagesPerUnit;
      const int sub0 = j % C::kStagesPerUnit;
      const int ru = u % kRawDepth;
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const int jj = j + b;
        if (jj >= C::kStages)
          ptx::mbar_wait(&empty[jj % C::kStages], (uint32_t)(((jj / C::kStages) - 1) & 1));
      }
      if (!kPrefetch) load_pass(j, v);
#ifndef FS_PROBE_NO_EXPAND  // timing experiment only: skip the expansion work
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const uint32_t sbase = op_base + ((j + b) % C::kStages) * C::kStageBytes;
#pragma unroll
        for (int m = 0; m < C::kItemsPerThread; ++m) {
          if (!it_on[m]) continue;
          if (FP4)  // 16 raw bytes (128 px) -> half of the 128-B operand row
            expand_row_f4(sbase + it_r[m] * C::kRegionBytes, it_rr[m], 4u * it_h[m], v[b][m]);
          else
            expand_row(sbase + it_r[m] * C::kRegionBytes, it_rr[m], v[b][m]);
        }
      }
#endif
      uint4 vn[kB][C::kItemsPerThread];
      if (kPrefetch && j + kB < nst) load_pass(j + kB, vn);
      // every writer fences its own stores into the async proxy and arrives (one
      // arrive per warp after __syncwarp measured 2 % slower at C2: 1.105 vs 1.08 ms)
#ifndef FS_PROBE_NO_FENCE  // timing experiment only (racy without the fence)
      ptx::fence_proxy_async_smem();
#endif
#pragma unroll
      for (int b = 0; b < kB; ++b) ptx::mbar_arrive(&full[(j + b) % C::kStages]);
      if (sub0 + kB == C::kStagesPerUnit) ptx::mbar_arrive(&raw_empty[ru]);
      if (kPrefetch) {
#pragma unroll
        for (int b = 0; b < kB; ++b)
#pragma unroll
          for (int m = 0; m < C::kItemsPerThread; ++m) v[b][m] = vn[b][m];
      }
    }
    // ===== epilogue: TMEM -> registers -> int32 partial tile =====
    const uint32_t q = (uint32_t)(warp & 3);  // TMEM lane quarter of this warp
    constexpr int kColGroups = C::kExpWarps / 4;  // warps sharing a lane quarter split columns
    const int cg = (warp - 1) / 4;
    int32_t *out = partial + (uint64_t)blockIdx.x * PANEL * PANEL;
    if (nst > 0) {
      ptx::mbar_wait(tmem_full, 0);
      fence_after();
    }
#pragma unroll
    for (int h = 0; h < C::kHalves; ++h) {
      const uint32_t row = h * 128 + q * 32 + lane;
      const bool lower_diag = DIAG && PANEL == 256 && h == 1;
      const int c_begin = lower_diag ? 128 : 0;
      for (int c0 = c_begin + 32 * cg; c0 < (int)n16; c0 += 32 * kColGroups) {
        uint32_t v[32];
        const uint32_t col =
            lower_diag ? (256u + (uint32_t)(c0 - 128)) : (uint32_t)(h * PANEL + c0);
        tmem_ld32(tmem + ((q * 32u) << 16) + col, v);
        if (nst == 0) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0;
        } else if (FP4) {  // exact integer-valued f32 -> int32
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = (uint32_t)__float2int_rn(__uint_as_float(v[e]));
        }
        int4 *dst = reinterpret_cast<int4 *>(out + (uint64_t)row * PANEL + c0);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          dst[e] = make_int4((int)v[4 * e], (int)v[4 * e + 1], (int)v[4 * e + 2], (int)v[4 * e + 3]);
      }
    }
    fence_before();
  }
  __syncthreads();
  if (FUSE && warp >= C::kCntWarp0 && ov.bins != nullptr) {
    for (uint32_t i = tid - 32 * C::kCntWarp0; i < ov.nbins; i += 32 * C::kCntWarps)
      if (sh_hist[i]) atomicAdd(ov.bins + i, (unsigned long long)sh_hist[i]);
    if (blockIdx.x == 0 && tid == 32 * C::kCntWarp0) {
      const uint64_t pad = total_units * 1024 - ov.pixels;  // padding counted in bin 0
      if (pad) atomicAdd(ov.bins, (unsigned long long)(0ull - pad));
    }
  }
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(C::kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// Off-diagonal 256 x 256 tiles on a CTA PAIR: tcgen05.mma.cta_group::2.kind::mxf4.
//
// A single-CTA 256 x 256 FP4 tile does not fit TMEM (2 x 256 f32 accumulator columns
// leave no room for the scale factors) and its SMEM traffic per MAC is high (both
// A halves read the whole 256-row B operand).  On a pair, CTA r (cluster rank r) owns
// rows [128 r, 128 r + 128) of panel I (its A half) and of panel J (its B half): it
// loads and expands only those 256 raw rows, the leader's MMA (M = 256, N = 256,
// K = 64) reads A and B halves from both CTAs' SMEM at the same offsets, and CTA r's
// TMEM holds D rows [128 r, 128 r + 128) x 256 columns.  Per CTA and 256-px K stage:
// 512 MMA cycles against ~576 cycles of SMEM traffic (expansion writes 32 KB, UMMA
// reads 32 KB, raw reads 8 KB), i.e. near the tensor-pipe bound at 2x the int8 rate.
//
// Synchronisation: raw ring per CTA (TMA -> local expanders); operand stage s is
// "full" on the LEADER's barrier once all 8 expander warps of both CTAs arrived
// (remote arrive through mapa for rank 1); the leader's tcgen05.commit multicasts
// "empty" and finally "tmem_full" to both CTAs.
// ---------------------------------------------------------------------------
constexpr int kPairThreads = 320;  // w0: TMEM alloc + MMA (leader); w1..8: expanders + epilogue; w9: TMA
constexpr int kPairExpWarps = 8;   // thread t < 128 expands A-half row t, t >= 128 B-half row t - 128
constexpr int kPairDepth = 2;      // raw units in flight per CTA
constexpr int kPairRawUnit = 2 * 128 * 128;  // A half + B half, 1024 px (128 B) per row
constexpr int kPairStageBytes = 2 * 128 * 128;  // A + B operand halves, 256 px per row
constexpr int kPairStages = 5;
// raw units prefetched into L2 ahead of the TMA loads (0 = off)
#ifndef FS_PAIR_L2PF
#define FS_PAIR_L2PF 0
#endif
// operand stages per proxy fence (1 or 2; a raw unit holds 4 stages)
#ifndef FS_PAIR_BATCH
#define FS_PAIR_BATCH 2
#endif
constexpr int kPairBatch = FS_PAIR_BATCH;
static_assert(kPairBatch == 1 || kPairBatch == 2, "1 or 2 stages per fence");
constexpr int kPairSmemBytes = kPairDepth * kPairRawUnit + kPairStages * kPairStageBytes + 1024 + 256;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// arrive on the barrier at the same SMEM offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t *bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(ptx::smem_u32(bar)), "r"(rank));
  // plain remote arrive (default .release.cta, like CUTLASS's ClusterBarrier::arrive):
  // the .release.cluster form costs a MEMBAR.ALL.GPU per stage; the operand writes
  // are already ordered for the tensor core by fence.proxy.async before this arrive
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// wait with cluster-scope acquire (arrivals come from the peer CTA too)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
  const uint32_t addr = ptx::smem_u32(bar);
  uint32_t done = 0;
  uint64_t spins = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;"
        "\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) break;
    if (++spins > (1ull << 26)) __trap();
  }
}
__device__ __forceinline__ void mma_mxf4_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                              uint32_t accum, uint32_t sfa, uint32_t sfb) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;"
      "\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void mma_commit_pair(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(ptx::smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
    k_gram_pair_f4(const __grid_constant__ CUtensorMap tm, uint32_t npanels, uint32_t kchunks,
                   uint64_t units_per_chunk, uint64_t total_units, int32_t *__restrict__ partial) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  const uint32_t pad = (1024u - (raw_addr & 1023u)) & 1023u;
  uint8_t *smem = smem_raw + pad;
  const uint32_t raw_base = raw_addr + pad;
  const uint32_t op_base = raw_base + kPairDepth * kPairRawUnit;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kPairDepth * kPairRawUnit +
                                                kPairStages * kPairStageBytes);
  uint64_t *empty = full + kPairStages;
  uint64_t *raw_full = empty + kPairStages;
  uint64_t *raw_empty = raw_full + kPairDepth;
  uint64_t *tmem_full = raw_empty + kPairDepth;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const uint32_t pair = blockIdx.x >> 1;
  const uint32_t tile = pair / kchunks;
  const uint32_t kc = pair % kchunks;
  uint32_t I = 0, t = tile;
  while (t >= npanels - 1 - I) {
    t -= npanels - 1 - I;
    ++I;
  }
  const uint32_t J = I + 1 + t;
  const uint64_t u0 = (uint64_t)kc * units_per_chunk;
  const uint64_t u1 = min(u0 + units_per_chunk, total_units);
  const int nunits = u1 > u0 ? (int)(u1 - u0) : 0;
  constexpr int kSub = 4;  // 256-px operand stages per 1024-px raw unit
  const int nst = nunits * kSub;

  if (tid == 0) {
    ptx::prefetch_tmap(&tm);
    for (int q = 0; q < kPairStages; ++q) {
      ptx::mbar_init(&full[q], 2 * kPairExpWarps);  // expander warps of both CTAs (leader's copy)
      ptx::mbar_init(&empty[q], 1);
    }
    for (int q = 0; q < kPairDepth; ++q) {
      ptx::mbar_init(&raw_full[q], 1);
      ptx::mbar_init(&raw_empty[q], kPairExpWarps);
    }
    ptx::mbar_init(tmem_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     ptx::smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  // block scales = 1.0 in both CTAs' scale-factor columns
  if (warp >= 1 && warp <= 4) {
    const uint32_t lanes = (uint32_t)((warp & 3) * 32) << 16;
    tmem_st16(tmem + lanes + kSfCol, kSfOnes);
    tmem_st16(tmem + lanes + kSfCol + 16, kSfOnes);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  fence_before();
  cluster_sync_all();  // barrier inits + scale factors visible pair-wide
  fence_after();

  if (warp == 0) {
    if (rank == 0 && lane == 0 && nst > 0) {
      constexpr uint32_t idesc = idesc_mxf4(256, 256);
      const uint32_t sfa = tmem + kSfCol, sfb = tmem + kSfCol + 16;
      const uint64_t d_op = sw128_desc(op_base);  // + byte offset / 16, as in k_gram_tc
      for (int j = 0; j < nst; ++j) {
        const int s = j % kPairStages;
        mbar_wait_cluster(&full[s], (uint32_t)((j / kPairStages) & 1));
        fence_after();
        const uint64_t d_a = d_op + (uint64_t)((uint32_t)(s * kPairStageBytes) >> 4);
        const uint64_t d_b = d_a + (uint64_t)((128 * 128) >> 4);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          mma_mxf4_pair(tmem, d_a + (uint64_t)(ks * 2), d_b + (uint64_t)(ks * 2), idesc,
                        (j > 0 || ks > 0) ? 1u : 0u, sfa, sfb);
        mma_commit_pair(&empty[s]);
      }
      mma_commit_pair(tmem_full);
    }
    __syncwarp();
  } else if (warp == kPairExpWarps + 1) {
    if (lane == 0) {
      for (int u = 0; u < nunits; ++u) {
        const int ru = u % kPairDepth;
#if FS_PAIR_L2PF > 0
        if (u == 0)
          for (int q = 1; q <= FS_PAIR_L2PF && q < nunits; ++q) {
            ptx::tma_prefetch_3d(&tm, 0, (int)(I * 256 + rank * 128), (int)(u0 + (uint64_t)q));
            ptx::tma_prefetch_3d(&tm, 0, (int)(J * 256 + rank * 128), (int)(u0 + (uint64_t)q));
          }
        else if (u + FS_PAIR_L2PF < nunits) {
          const int cp = (int)(u0 + (uint64_t)(u + FS_PAIR_L2PF));
          ptx::tma_prefetch_3d(&tm, 0, (int)(I * 256 + rank * 128), cp);
          ptx::tma_prefetch_3d(&tm, 0, (int)(J * 256 + rank * 128), cp);
        }
#endif
        if (u >= kPairDepth) ptx::mbar_wait(&raw_empty[ru], (uint32_t)(((u / kPairDepth) - 1) & 1));
        const int c2 = (int)(u0 + (uint64_t)u);
        ptx::mbar_arrive_expect_tx(&raw_full[ru], kPairRawUnit);
        uint8_t *dst = smem + ru * kPairRawUnit;
        ptx::tma_load_3d(dst, &tm, 0, (int)(I * 256 + rank * 128), c2, &raw_full[ru]);
        ptx::tma_load_3d(dst + 128 * 128, &tm, 0, (int)(J * 256 + rank * 128), c2, &raw_full[ru]);
      }
    }
    __syncwarp();
  } else {
    // ===== expanders: thread t expands row t % 128 of the A (t < 128) or B half =====
    const uint32_t et = (uint32_t)(tid - 32);
    const uint32_t reg = et >> 7, rr = et & 127u;
    const uint32_t sw = rr & 7u;
    // as in k_gram_tc: the next stage's raw loads go out before this stage's proxy fence
    // (within a raw unit only — with a 2-deep raw ring, waiting for the next unit before
    // releasing this one would delay its refill)
    auto load = [&](int jp, uint4 &a, uint4 &b) {
      const int up = jp / kSub, subp = jp % kSub;
      const int rup = up % kPairDepth;
      if (subp == 0) ptx::mbar_wait(&raw_full[rup], (uint32_t)((up / kPairDepth) & 1));
      const uint32_t rrow = raw_base + rup * kPairRawUnit + reg * 128 * 128 + rr * 128;
      a = ld_shared_v4(rrow + ((((uint32_t)(2 * subp)) ^ sw) << 4));
      b = ld_shared_v4(rrow + ((((uint32_t)(2 * subp + 1)) ^ sw) << 4));
    };
    uint4 v0, v1;
    bool have = false;
    if (kPairBatch == 1) {
      for (int j = 0; j < nst; ++j) {
        const int u = j / kSub, sub = j % kSub;
        const int ru = u % kPairDepth;
        const int s = j % kPairStages;
        if (!have) load(j, v0, v1);
        if (j >= kPairStages) ptx::mbar_wait(&empty[s], (uint32_t)(((j / kPairStages) - 1) & 1));
        const uint32_t obase = op_base + s * kPairStageBytes + reg * 128 * 128;
        expand_row_f4(obase, rr, 0u, v0);
        expand_row_f4(obase, rr, 4u, v1);
        uint4 n0, n1;
        have = j + 1 < nst && (j + 1) % kSub != 0;
        if (have) load(j + 1, n0, n1);
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_cluster(&full[s], 0);
          if (sub == kSub - 1) ptx::mbar_arrive(&raw_empty[ru]);
        }
        if (have) {
          v0 = n0;
          v1 = n1;
        }
      }
    } else {
      // two stages per proxy fence: stages j, j + 1 (same raw unit) expanded back to back
      for (int j = 0; j < nst; j += 2) {
        const int u = j / kSub, sub = j % kSub;
        const int ru = u % kPairDepth;
        const int s0 = j % kPairStages, s1 = (j + 1) % kPairStages;
        uint4 w0, w1;
        load(j, v0, v1);
        load(j + 1, w0, w1);
        if (j >= kPairStages) ptx::mbar_wait(&empty[s0], (uint32_t)(((j / kPairStages) - 1) & 1));
        if (j + 1 >= kPairStages)
          ptx::mbar_wait(&empty[s1], (uint32_t)((((j + 1) / kPairStages) - 1) & 1));
        const uint32_t ob0 = op_base + s0 * kPairStageBytes + reg * 128 * 128;
        const uint32_t ob1 = op_base + s1 * kPairStageBytes + reg * 128 * 128;
        expand_row_f4(ob0, rr, 0u, v0);
        expand_row_f4(ob0, rr, 4u, v1);
        expand_row_f4(ob1, rr, 0u, w0);
        expand_row_f4(ob1, rr, 4u, w1);
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_cluster(&full[s0], 0);
          mbar_arrive_cluster(&full[s1], 0);
          if (sub + 1 == kSub - 1) ptx::mbar_arrive(&raw_empty[ru]);
        }
      }
    }
    // ===== epilogue: this CTA's 128 rows x 256 columns of D =====
    const uint32_t q = (uint32_t)(warp & 3);     // TMEM lane quarter of this warp
    const int chalf = (warp - 1) / 4;            // warps 1..4: columns 0..127, 5..8: 128..255
    int32_t *out = partial + (uint64_t)pair * 256 * 256;
    if (nst > 0) {
      ptx::mbar_wait(tmem_full, 0);
      fence_after();
    }
    const uint32_t row = rank * 128 + q * 32 + lane;
    for (int c0 = chalf * 128; c0 < chalf * 128 + 128; c0 += 32) {
      uint32_t v[32];
      tmem_ld32(tmem + ((q * 32u) << 16) + (uint32_t)c0, v);
      if (nst == 0) {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0;
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = (uint32_t)__float2int_rn(__uint_as_float(v[e]));
      }
      int4 *dst = reinterpret_cast<int4 *>(out + (uint64_t)row * 256 + c0);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        dst[e] = make_int4((int)v[4 * e], (int)v[4 * e + 1], (int)v[4 * e + 2], (int)v[4 * e + 3]);
    }
    fence_before();
  }
  __syncthreads();
  cluster_sync_all();  // the leader's MMAs read this CTA's SMEM / write its TMEM
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Sum int32 partials over K chunks; scatter into the k x k Gram (both triangles).
template <int PANEL>
__global__ void k_gram_reduce(const int32_t *__restrict__ part_diag, uint32_t kc_diag,
                              const int32_t *__restrict__ part_off, uint32_t kc_off, uint32_t k,
                              uint32_t npanels, unsigned long long *__restrict__ gram) {
  const uint32_t ndiag = npanels;
  const uint32_t noff = npanels * (npanels - 1) / 2;
  const uint64_t per_tile = (uint64_t)PANEL * PANEL;
  const uint64_t total = (uint64_t)(ndiag + noff) * per_tile;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(e / per_tile);
    const uint32_t r = (uint32_t)((e % per_tile) / PANEL), c = (uint32_t)(e % PANEL);
    uint32_t I, J;
    const int32_t *base;
    uint32_t kc;
    uint32_t rr = r, cc = c;
    if (t < ndiag) {
      I = J = t;
      base = part_diag + (uint64_t)t * kc_diag * per_tile;
      kc = kc_diag;
      if (PANEL == 256 && r >= 128 && c < 128) {  // not computed: mirror quadrant
        rr = c;
        cc = r;
      }
    } else {
      uint32_t u = t - ndiag;
      I = 0;
      while (u >= npanels - 1 - I) {
        u -= npanels - 1 - I;
        ++I;
      }
      J = I + 1 + u;
      base = part_off + (uint64_t)(t - ndiag) * kc_off * per_tile;
      kc = kc_off;
    }
    const uint32_t gi = I * PANEL + r, gj = J * PANEL + c;
    if (gi >= k || gj >= k) continue;
    long long s = 0;
    for (uint32_t x = 0; x < kc; ++x) s += base[(uint64_t)x * per_tile + (uint64_t)rr * PANEL + cc];
    gram[(uint64_t)gi * k + gj] = (unsigned long long)s;
    if (I != J) gram[(uint64_t)gj * k + gi] = (unsigned long long)s;
  }
}

// Gather arbitrary slots into a contiguous tile-interleaved copy (rows 0..k-1).
__global__ void k_gather_slots(const uint32_t *__restrict__ packed, uint64_t cap,
                               const uint32_t *__restrict__ slots, uint32_t k, uint64_t ntiles,
                               uint32_t *__restrict__ dst) {
  const uint64_t total = ntiles * k * 8;  // uint4 per (tile, row): 8
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t t = e / ((uint64_t)k * 8);
    const uint32_t i = (uint32_t)((e / 8) % k), v = (uint32_t)(e % 8);
    const uint4 *src = reinterpret_cast<const uint4 *>(packed + (t * cap + slots[i]) * 32) + v;
    reinterpret_cast<uint4 *>(dst + (t * k + i) * 32)[v] = *src;
  }
}

struct Plan {
  int panel;
  uint32_t k;  // masks
  bool pair;  // off-diagonal tiles on CTA pairs (kind::mxf4, cta_group::2)
  uint32_t npanels, ndiag, noff;
  uint64_t units_diag, units_off;  // raw units along K for each tile kind
  uint32_t kc_diag, kc_off;
  uint64_t upc_diag, upc_off;
};

// K chunks per tile: the grid is ntiles * kc CTAs (or CTA pairs) over `slots` resident
// positions.  Pick the kc that keeps the machine busiest over whole waves,
// ntiles*kc / (waves * slots), preferring fewer chunks on ties (less prologue and
// partial-reduce work); a chunk keeps >= 4 units (4 K px) and respects max_upc
// (the FP4 exactness cap).
static void chunking(uint64_t total_units, uint32_t ntiles, int slots, uint32_t &kc,
                     uint64_t &upc, uint64_t max_upc = UINT64_MAX) {
  if (ntiles == 0 || total_units == 0) {
    kc = 0;
    upc = 0;
    return;
  }
  const uint64_t S = (uint64_t)(slots > 0 ? slots : 1);
  const uint64_t kc_min = (total_units + max_upc - 1) / max_upc;  // exactness cap
  uint64_t kc_max = std::max<uint64_t>(kc_min, std::min<uint64_t>(total_units / 4, 8 * S));
  if (kc_max < 1) kc_max = 1;
  double best_eff = -1.0;
  uint64_t best = kc_min > 0 ? kc_min : 1;
  for (uint64_t c = (kc_min > 0 ? kc_min : 1); c <= kc_max; ++c) {
    const uint64_t u = (total_units + c - 1) / c;  // units per chunk
    const uint64_t real = (total_units + u - 1) / u;  // chunks actually used
    if (real != c) continue;
    const uint64_t ctas = (uint64_t)ntiles * c;
    const uint64_t waves = (ctas + S - 1) / S;
    const double eff = (double)ctas / (double)(waves * S);
    if (eff > best_eff + 1e-3) {
      best_eff = eff;
      best = c;
    }
    if (waves > 4) break;  // deeper than a few waves buys nothing
  }
  upc = (total_units + best - 1) / best;
  if (upc > max_upc) upc = max_upc;
  kc = (uint32_t)((total_units + upc - 1) / upc);
}

static Plan make_plan(uint32_t k, uint64_t wpm, int num_sms, bool fp4) {
  Plan p{};
  p.k = k;
  p.panel = k <= 128 ? 128 : 256;
  p.npanels = (k + p.panel - 1) / p.panel;
  p.ndiag = p.npanels;
  p.noff = p.npanels * (p.npanels - 1) / 2;
  const uint64_t ntiles = wpm / 32;
  p.units_diag = ntiles;  // diag tiles: one 128-B raw row per tile
  p.units_off = p.panel == 256 ? ntiles * 2 : ntiles;  // 256-panel off-diag: 64-B halves
  // FP4 diagonal tiles accumulate in f32: a chunk (unit = 1024 px) must stay <= 2^24 px
  chunking(p.units_diag, p.ndiag, num_sms, p.kc_diag, p.upc_diag,
           fp4 ? kF4MaxChunkPx / 1024 : UINT64_MAX);
  p.pair = fp4 && p.panel == 256 && p.noff > 0;
  if (p.pair) {
    // one pair per two SMs; 1024-px units; f32 accumulation caps a chunk at 2^24 px
    p.units_off = ntiles;
    chunking(p.units_off, p.noff, num_sms / 2, p.kc_off, p.upc_off, kF4MaxChunkPx / 1024);
  } else {
    chunking(p.units_off, p.noff, num_sms, p.kc_off, p.upc_off);
  }
  return p;
}

}  // namespace tc

static uint64_t partial_offset(const tc::Plan &p) {
  const uint64_t per_tile = (uint64_t)p.panel * p.panel * 4;
  const uint64_t b = ((uint64_t)p.ndiag * p.kc_diag + (uint64_t)p.noff * p.kc_off) * per_tile;
  return (b + 255) / 256 * 256;
}

size_t gram_tc_workspace_bytes(uint32_t k, uint64_t wpm, int num_sms, bool fp4, bool fuse) {
  tc::Plan p = tc::make_plan(k, wpm, num_sms, fp4);
  uint64_t bytes = partial_offset(p);
  // multi-panel fused recompute: one uint16 partial-count slab per panel
  if (fuse && fp4 && p.panel == 256 && p.npanels > 1)
    bytes += (uint64_t)p.npanels * (wpm / 32) * 1024 * 2;
  return (size_t)bytes;
}

template <int PANEL, bool DIAG, bool FP4 = false, bool FUSE = false, int FD = 4>
static cudaError_t launch_one(const CUtensorMap &tm, const tc::Plan &p, int32_t *part,
                              const OverlapArgs &ov, cudaStream_t s) {
  using C = tc::Cfg<PANEL, DIAG, FP4, FUSE, FD>;
  const uint32_t ntiles = DIAG ? p.ndiag : p.noff;
  const uint32_t kc = DIAG ? p.kc_diag : p.kc_off;
  const uint64_t upc = DIAG ? p.upc_diag : p.upc_off;
  const uint64_t units = DIAG ? p.units_diag : p.units_off;
  if (ntiles == 0 || kc == 0) return cudaSuccess;
  static SmemOptIn attr;
  if (cudaError_t e = smem_opt_in(attr, tc::k_gram_tc<PANEL, DIAG, FP4, FUSE, FD>, C::kSmemBytes);
      e != cudaSuccess)
    return e;
  tc::k_gram_tc<PANEL, DIAG, FP4, FUSE, FD>
      <<<ntiles * kc, C::kThreadsTotal, C::kSmemBytes, s>>>(
          tm, p.npanels, kc, upc, units, part, ov, p.k);
  return cudaGetLastError();
}

size_t gram_tc_gather_bytes(uint32_t k, uint64_t wpm) { return (size_t)k * wpm * 4; }

// Fused single-panel FP4 recompute: 2 = k_recompute_f4 (register-staged raw units,
// fs_recompute_f4.cu, default), 1 = k_gram_tc<256, ..., FUSE> (TMA raw ring + counter
// warps).  FS_FUSED_KERNEL=1 selects the older kernel (A/B measurements).
constexpr uint32_t kRc128MinMasks = 80;

static int fused_kernel_version() {
  static const int v = [] {
    const char *e = std::getenv("FS_FUSED_KERNEL");
    return (e && e[0] == '1') ? 1 : 2;
  }();
  return v;
}

cudaError_t launch_gram_tc(const uint32_t *packed, uint64_t capacity, uint64_t wpm,
                           const uint32_t *slots, const uint32_t *host_slots, uint32_t k,
                           unsigned long long *gram, void *workspace, void *gather_ws,
                           int num_sms, bool fp4, const OverlapArgs *fuse, bool *fused,
                           cudaStream_t s) {
  if (fused) *fused = false;
  if (k == 0) return cudaSuccess;
  tc::Plan p = tc::make_plan(k, wpm, num_sms, fp4);
  const uint64_t ntiles = wpm / 32;
  // contiguous slot run -> map straight over the ensemble; else gather first
  const uint32_t *src = packed;
  uint64_t src_cap = capacity, row0 = 0;
  const int64_t first = contiguous_run(host_slots, k);
  cudaError_t e;
  // the single-panel fused recompute reads scattered slots itself (no gather pass)
  const bool rc_direct = fuse != nullptr && p.npanels == 1 && fp4 &&
                         (p.panel == 256 || k >= kRc128MinMasks) && fused_kernel_version() >= 2;
  if (first >= 0) {
    row0 = (uint64_t)first;
  } else if (rc_direct) {
    // src stays the ensemble; launch_recompute_f4 gets the slot list below
  } else {
    if (gather_ws == nullptr) return cudaErrorInvalidValue;
    uint64_t total = ntiles * k * 8;
    uint64_t grid = (total + 255) / 256;
    if (grid > (uint64_t)num_sms * 16) grid = (uint64_t)num_sms * 16;
    tc::k_gather_slots<<<(unsigned)grid, 256, 0, s>>>(packed, capacity, slots, k, ntiles,
                                                      static_cast<uint32_t *>(gather_ws));
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    src = static_cast<const uint32_t *>(gather_ws);
    src_cap = k;
  }
  const uint64_t per_tile = (uint64_t)p.panel * p.panel;
  int32_t *part_diag = reinterpret_cast<int32_t *>(workspace);
  int32_t *part_off = part_diag + (uint64_t)p.ndiag * p.kc_diag * per_tile;
  CUtensorMap tm_diag, tm_off;
  const uint32_t raw_off = p.panel == 256 ? 16u : 32u;  // box words for off-diag units
  if ((e = encode_packed_map(&tm_diag, src, src_cap, row0, k, ntiles, 32, p.panel, 1, 128)) !=
      cudaSuccess)
    return e;
  if ((e = encode_packed_map(&tm_off, src, src_cap, row0, k, ntiles, raw_off, p.panel, 1,
                             raw_off == 16 ? 64 : 128)) != cudaSuccess)
    return e;
  CUtensorMap tm_pair;
  if (p.pair && (e = encode_packed_map(&tm_pair, src, src_cap, row0, k, ntiles, 32, 128, 1, 128)) !=
                    cudaSuccess)
    return e;
  const OverlapArgs none{};
  // one panel holds every mask: its diagonal CTAs see all masks of a pixel range and
  // also produce the overlap products (counts / histogram / RGBA) from the same tiles
  const bool fuse_now = fuse != nullptr && p.npanels == 1;
  // several 256-mask panels (FP4): each diagonal CTA counts its panel's masks from the
  // tiles it already streams (uint16 partial counts); a combine pass sums the panels
  const bool fuse_multi = fuse != nullptr && p.npanels > 1 && fp4 && p.panel == 256;
  OverlapArgs ovp{};
  uint16_t *partial16 = nullptr;
  const uint64_t pitch = ntiles * 1024;
  if (fuse_multi) {
    partial16 = reinterpret_cast<uint16_t *>(static_cast<char *>(workspace) + partial_offset(p));
    ovp = *fuse;
    ovp.counts = nullptr;
    ovp.rgba = nullptr;
    ovp.bins = nullptr;
    ovp.partial16 = partial16;
    ovp.part_pitch = pitch;
  }
  if (p.panel == 128) {
    // 128-row k_recompute_f4 from k = 80 on; below it the narrow TMA-ring kernel's MMA
    // N shrinks with k and its per-unit overhead is lower (k_sweep: k = 64 0.57 vs 0.58 ms,
    // k = 100 0.60 vs 0.58, k = 128 0.67 vs 0.58; profiles/round2/kernel_search/g36)
    if (fuse_now && fp4 && k >= kRc128MinMasks && fused_kernel_version() >= 2)
      e = launch_recompute_f4(src, src_cap, row0, k, p.units_diag, p.kc_diag, p.upc_diag,
                              part_diag, *fuse, s, 1, first >= 0 ? nullptr : slots, 128);
    else if (fuse_now)
      e = fp4 ? launch_one<128, true, true, true>(tm_diag, p, part_diag, *fuse, s)
              : launch_one<128, true, false, true>(tm_diag, p, part_diag, *fuse, s);
    else
      e = fp4 ? launch_one<128, true, true>(tm_diag, p, part_diag, none, s)
              : launch_one<128, true>(tm_diag, p, part_diag, none, s);
    if (e != cudaSuccess) return e;
    if ((e = launch_one<128, false>(tm_off, p, part_off, none, s)) != cudaSuccess) return e;
  } else {
    if (fuse_now && fp4 && fused_kernel_version() >= 2)
      e = launch_recompute_f4(src, src_cap, row0, k, p.units_diag, p.kc_diag, p.upc_diag,
                              part_diag, *fuse, s, 1, first >= 0 ? nullptr : slots);
    else if (fuse_now)
      e = fp4 ? launch_one<256, true, true, true, tc::kFuseDepth256>(tm_diag, p, part_diag, *fuse, s)
              : launch_one<256, true, false, true>(tm_diag, p, part_diag, *fuse, s);
    else if (fuse_multi && fused_kernel_version() >= 2)
      e = launch_recompute_f4(src, src_cap, row0, k, p.units_diag, p.kc_diag, p.upc_diag,
                              part_diag, ovp, s, p.ndiag);
    else if (fuse_multi)
      e = launch_one<256, true, true, true, tc::kFuseDepth256>(tm_diag, p, part_diag, ovp, s);
    else
      e = fp4 ? launch_one<256, true, true>(tm_diag, p, part_diag, none, s)
              : launch_one<256, true>(tm_diag, p, part_diag, none, s);
    if (e != cudaSuccess) return e;
    if (p.pair) {
      if (p.kc_off > 0) {
        static SmemOptIn attr;
        if ((e = smem_opt_in(attr, tc::k_gram_pair_f4, tc::kPairSmemBytes)) != cudaSuccess)
          return e;
        tc::k_gram_pair_f4<<<2 * p.noff * p.kc_off, tc::kPairThreads, tc::kPairSmemBytes, s>>>(
            tm_pair, p.npanels, p.kc_off, p.upc_off, p.units_off, part_off);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
      }
    } else if ((e = launch_one<256, false>(tm_off, p, part_off, none, s)) != cudaSuccess) {
      return e;
    }
  }
  if (fused) *fused = fuse_now || fuse_multi;
  const uint64_t total = (uint64_t)(p.ndiag + p.noff) * per_tile;
  uint64_t grid = (total + 255) / 256;
  if (grid > (uint64_t)num_sms * 8) grid = (uint64_t)num_sms * 8;
  if (p.panel == 128)
    tc::k_gram_reduce<128><<<(unsigned)grid, 256, 0, s>>>(part_diag, p.kc_diag, part_off,
                                                           p.kc_off, k, p.npanels, gram);
  else
    tc::k_gram_reduce<256><<<(unsigned)grid, 256, 0, s>>>(part_diag, p.kc_diag, part_off,
                                                           p.kc_off, k, p.npanels, gram);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (fuse_multi) return launch_combine_partials(partial16, p.npanels, pitch, *fuse, s);
  return cudaSuccess;
}

}  // namespace fs
