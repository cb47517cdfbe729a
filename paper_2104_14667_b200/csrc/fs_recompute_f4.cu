// fs_recompute_f4.cu — the full recompute of one <= 256-mask panel in ONE kernel:
// exact pairwise intersections (Gram, tcgen05 kind::mxf4) AND the per-pixel overlap
// products (counts, histogram, composite RGBA) from a single read of the packed masks.
//
// Reference semantics: similarity_matrix's pair_counts loop (analytics.py:174-181,
// _kernels_np.py:26-32) and accumulate / overlap_histogram / composite_map
// (analytics.py:106-162, _kernels_np.py:16-47) of /root/reference/pkg/src/floodstream/.
//
// Template ROWS: 256 (one 256-mask panel, also the diagonal tiles of larger ensembles) or
// 128 (a single panel of 80..128 masks, one MMA of N = roundup(k, 16) per K step).
//
// Data path per 1024-px unit (one pixel tile of every mask = 256 x 128 B, contiguous in
// the tile-interleaved layout, fs_common.cuh):
//   * Two groups of 8 expander warps take alternate units (FS_RC_GROUPS = 2; group g
//     does units u = g mod 2), so a warp has two units of MMA time for one unit of its
//     serial load / count / expand chain.  A warp loads its 32 rows of the unit straight
//     from global memory into REGISTERS with fully coalesced 16-B loads (warp
//     instruction j covers 4 consecutive mask rows = 512 contiguous bytes); lane l holds
//     rows 4j + l/8 (j = 0..7), 16-B chunk c = l % 8 (pixels 128c .. 128c+127).  One lane
//     per group bulk-prefetches the unit 2 ahead into L2 (cp.async.bulk.prefetch.L2), so
//     the register loads, issued as soon as the previous unit is expanded, hit L2.  No
//     TMA ring and no raw copy in shared memory.
//   * Counting from those registers: per lane a carry-save tree over its 8 rows, then
//     two shuffle rounds over the 4 lanes holding the same chunk give each lane the
//     bit-sliced count (6 planes) of one 32-px word over the warp's 32 rows; the 8 warps'
//     partial planes (6 KB per unit) go to a per-group partial ring in shared memory and
//     3 combiner warps add them (9 planes, exact), transpose to per-pixel counts and emit
//     histogram / counts / RGBA (fs_bitslice.cuh emit_tile).
//   * Expansion from the same registers: operand stage s of the unit = word s of every
//     chunk (any pixel permutation shared by all masks leaves a Gram unchanged), so each
//     lane writes 16 B of e2m1 0/1 operand per row per stage into the SWIZZLE_128B
//     K-major ring (5 x 32 KB); one thread issues rows 0-127 x N=256 and rows 128-255 x
//     N=128 kind::mxf4 MMAs per 64-px K step (3/4 of the 256 x 256 square; the reduce
//     mirrors).
// Measured (profiles/round2/kernel_search): the tensor core's operand fetch and the
// expanders' st.shared stream do not compete (768 -> 778 cycles per stage with 32 KB of
// stores beside the MMAs); what sets the time is the MMA pipe (90 % active under ncu) and
// the handoff of each stage between the expander warps and the MMA thread.
#include "fs_bitslice.cuh"
#include "fs_tcgen05.cuh"

namespace fs {
namespace rc {

// Expander groups: 1 = eight expander warps take every unit (double-buffered registers);
// 2 = two groups of eight take alternate units (single-buffered), so each warp has two
// units of MMA time for one unit of its serial work (20 warps, 96 registers).
#ifndef FS_RC_GROUPS
#define FS_RC_GROUPS 2
#endif
constexpr int kGroups = FS_RC_GROUPS;
// every producing thread arrives on the stage / partial barriers itself (the arrive is the
// release of that thread's own stores; 1) or one lane per warp after __syncwarp (0)
#ifndef FS_RC_THREAD_ARRIVE
#define FS_RC_THREAD_ARRIVE 1
#endif
constexpr bool kThreadArrive = FS_RC_THREAD_ARRIVE != 0;
constexpr uint32_t kArrivePerWarp = kThreadArrive ? 32u : 1u;
static_assert(kGroups == 1 || kGroups == 2, "one or two expander groups");
constexpr int kCntWarps = kGroups == 1 ? 4 : 3;  // combiner + emit warps
// partial-count ring: kCntWarps slots per group; combiner c owns slot c of every group's
// ring and takes the units u with (u / kGroups) % kCntWarps == c, in order — one producer
// group and one consumer per slot, so the parity waits cannot alias
constexpr int kPartSlots = kCntWarps;
constexpr int kPartDepth = kGroups * kPartSlots;
constexpr int kPlanes = 6;                    // bit planes of a 32-row partial count
constexpr int kFuseBins = 288;
constexpr int kTbBytes = kCntWarps * 32 * kTileTb * 4;
constexpr int kSlotWords = 256 + 2;  // slot of every panel row + the slot span [lo, hi]
constexpr int kSmemMax = 232448;

// ROWS = 256: a 256-mask panel, MMAs rows 0-127 x N=256 + rows 128-255 x N=128 per K step;
// ROWS = 128: a panel of k <= 128 masks, one MMA rows 0-127 x N=roundup(k, 16).
template <int ROWS>
struct Cfg {
  static constexpr int kGW = ROWS / 32;                 // expander warps per group
  static constexpr int kExpWarps = kGW * kGroups;       // expander / epilogue warps
  static constexpr int kWarps = 1 + kExpWarps + kCntWarps;
  static constexpr int kThreads = 32 * kWarps;
  static constexpr int kCntWarp0 = 1 + kExpWarps;
  static constexpr int kPartWords = kGW * kPlanes * 32;  // per unit
  static constexpr int kStageBytes = ROWS * 128;        // ROWS rows x 128 B (256 px of e2m1)
  static constexpr int kExtraBytes = kPartDepth * kPartWords * 4 + kTbBytes +
                                     2 * kFuseBins * 4 + kSlotWords * 4;
  static constexpr int kStages = (kSmemMax - 1024 - 512 - kExtraBytes) / kStageBytes;
  static constexpr int kSmemBytes = kStages * kStageBytes + kExtraBytes + 1024 + 512;
  static_assert(kStages >= 3, "operand ring too shallow");
  static_assert(2 * (2 * kStages + 2 * kPartDepth + 1) * 4 + 12 <= 512, "barrier area");
};
// operand stages written per proxy fence + arrive (2 measured better with one expander
// group, 1 with two)
#ifndef FS_RC_BATCH
#define FS_RC_BATCH 1
#endif
// L2 prefetch distance in units: while unit u is processed, one lane bulk-prefetches unit
// u + d (cp.async.bulk.prefetch.L2, the unit's k rows x 128 B are contiguous) so the
// register loads issued two units ahead hit L2 (0 = off)
#ifndef FS_RC_L2PF
#define FS_RC_L2PF 2
#endif
constexpr int kBatch = FS_RC_BATCH;             // operand stages per proxy fence
static_assert(4 % kBatch == 0 && kBatch < 3, "batch must divide a unit's 4 stages");
__host__ __device__ constexpr int part_slot(int u) {
  return (u % kGroups) * kPartSlots + (u / kGroups) % kPartSlots;
}
__host__ __device__ constexpr int part_use(int u) { return (u / kGroups) / kPartSlots; }

// bulk L2 prefetch of one unit (k rows x 128 B, contiguous)
__device__ __forceinline__ void l2_prefetch(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// (h, l) = a + b (half adder)
__device__ __forceinline__ void ha(uint32_t &h, uint32_t &l, uint32_t a, uint32_t b) {
  h = a & b;
  l = a ^ b;
}

// bit-sliced sum of 8 words: planes p[0..3] (value 0..8)
__device__ __forceinline__ void sum8(const uint32_t (&x)[8], uint32_t (&p)[4]) {
  uint32_t t1, o1, t2, o2, t3, o3, t4, o4, f1, w1, f2, w2;
  csa(t1, o1, x[0], x[1], x[2]);
  csa(t2, o2, o1, x[3], x[4]);
  csa(t3, o3, o2, x[5], x[6]);
  ha(t4, o4, o3, x[7]);
  csa(f1, w1, t1, t2, t3);
  ha(f2, w2, w1, t4);
  p[0] = o4;
  p[1] = w2;
  p[2] = f1 ^ f2;
  p[3] = f1 & f2;
}

// bit-sliced a + b, NA planes each -> NA + 1 planes
template <int NA>
__device__ __forceinline__ void add_planes(const uint32_t *a, const uint32_t *b, uint32_t *s) {
  uint32_t c = a[0] & b[0];
  s[0] = a[0] ^ b[0];
#pragma unroll
  for (int i = 1; i < NA; ++i) {
    const uint32_t u = a[i] ^ b[i];
    s[i] = u ^ c;
    c = (a[i] & b[i]) | (u & c);
  }
  s[NA] = c;
}

__device__ __forceinline__ void expand_word(uint32_t addr, uint32_t x) {
  tc::st_shared_v4(addr, make_uint4((x << 1) & 0x22222222u, x & 0x22222222u,
                                    (x >> 1) & 0x22222222u, (x >> 2) & 0x22222222u));
}

struct Args {
  const uint32_t *src;   // packed masks (tile-interleaved)
  uint64_t cap;          // slots per tile row of `src`
  uint64_t row0;         // first slot of panel 0
  uint32_t k;            // masks in all panels (panel I holds masks 256 I .. 256 I + 255)
  const uint32_t *slots; // device slot list (mask m lives in slot slots[m]) or null:
                         // mask m in slot row0 + m (a contiguous run)
  uint64_t total_units;  // tiles of 1024 px
  uint64_t upc;          // units per CTA chunk
  uint32_t kchunks;      // CTA chunks per panel: blockIdx.x = panel * kchunks + chunk
  int32_t *partial;      // one ROWS x ROWS int32 tile per CTA
};

// kSlots: the panel's masks are read through the slot table (a.slots != nullptr)
template <int ROWS, bool kSlots>
__global__ void __launch_bounds__(Cfg<ROWS>::kThreads, 1)
    k_recompute_f4(const Args a, const OverlapArgs ov) {
  using C = Cfg<ROWS>;
  constexpr int kGW = C::kGW, kExpWarps = C::kExpWarps, kCntWarp0 = C::kCntWarp0;
  constexpr int kPartWords = C::kPartWords, kStageBytes = C::kStageBytes, kStages = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  const uint32_t pad = (1024u - (raw_addr & 1023u)) & 1023u;
  uint8_t *smem = smem_raw + pad;
  const uint32_t op_base = raw_addr + pad;
  uint32_t *part = reinterpret_cast<uint32_t *>(smem + kStages * kStageBytes);
  uint32_t *cnt_tb = part + kPartDepth * kPartWords;
  uint32_t *sh_hist = cnt_tb + kCntWarps * 32 * kTileTb;
  uint32_t *sh_lut = sh_hist + kFuseBins;
  uint32_t *sh_slot = sh_lut + kFuseBins;  // ensemble slot of panel row r; [256], [257]: span
  uint64_t *full = reinterpret_cast<uint64_t *>(sh_slot + kSlotWords);
  uint64_t *empty = full + kStages;
  uint64_t *part_full = empty + kStages;
  uint64_t *part_empty = part_full + kPartDepth;
  uint64_t *tmem_full = part_empty + kPartDepth;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  // diagonal tile `panel` of a k > 256 ensemble (the Gram of masks 256 panel ..) or the
  // single panel (panel 0); the off-diagonal tiles run on k_gram_pair_f4
  const uint32_t panel = blockIdx.x / a.kchunks;
  const uint64_t prow0 = a.row0 + (uint64_t)ROWS * panel;     // first slot of this panel
  const uint32_t pk = min((uint32_t)ROWS, a.k - (uint32_t)ROWS * panel);  // masks in it
  const uint64_t u0 = (uint64_t)(blockIdx.x % a.kchunks) * a.upc;
  const uint64_t u1 = min(u0 + a.upc, a.total_units);
  const int nunits = u1 > u0 ? (int)(u1 - u0) : 0;
  const int nst = nunits * 4;

  // expander registers: rows 4j + lane/8 of this warp's 32 rows, chunk lane % 8
  const int ew = warp - 1;
  const int grp = ew / kGW, gw = ew % kGW;  // expander group, warp within the group
  const uint32_t chunk = (uint32_t)lane & 7u;
  uint4 ra[8], rb[8];
  auto load_unit = [&](int u, uint4 (&r)[8]) {
    const uint64_t gu = u0 + (uint64_t)u;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t row = (uint32_t)(32 * gw + 4 * j) + ((uint32_t)lane >> 3);
#ifndef FS_RC_NO_LOAD  // timing experiment only: no HBM traffic, constant data
      if (row < pk) {
        const uint64_t slot = kSlots ? (uint64_t)sh_slot[row] : prow0 + row;
        r[j] = ptx::ld_nc_v4(a.src + ((gu * a.cap + slot) * 32u + 4u * chunk));
      }
      else
#else
      if (row < pk)
        r[j] = make_uint4((uint32_t)gu * 0x9E3779B9u ^ row, row * 7u, (uint32_t)gu, row ^ 5u);
      else
#endif
        r[j] = make_uint4(0u, 0u, 0u, 0u);
    }
  };
  const bool is_exp = warp >= 1 && warp <= kExpWarps;
  auto first_loads = [&] {
    if (grp < nunits) load_unit(grp, ra);
    if (kGroups == 1 && nunits > 1) load_unit(1, rb);
  };
  // a contiguous run: first unit(s) in flight before the setup below (a slot list is
  // read into shared memory by the setup first)
  if (is_exp && !kSlots) first_loads();

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], kGW * kArrivePerWarp);  // the warps of the unit's group
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kPartDepth; ++s) {
      ptx::mbar_init(&part_full[s], kGW * kArrivePerWarp);
      ptx::mbar_init(&part_empty[s], kArrivePerWarp);
    }
    ptx::mbar_init(tmem_full, 1);
    ptx::fence_mbar_init();
  }
  const bool lut_sh = ov.rgba != nullptr;
  if (kSlots && warp == kCntWarp0) {  // this panel's slots and their span
    uint32_t lo = 0xFFFFFFFFu, hi = 0u;
    for (uint32_t i = (uint32_t)lane; i < 256u; i += 32u) {
      const uint32_t sl = i < pk ? a.slots[(uint32_t)ROWS * panel + i] : 0u;
      sh_slot[i] = sl;
      if (i < pk) {
        lo = min(lo, sl);
        hi = max(hi, sl);
      }
    }
    lo = __reduce_min_sync(0xFFFFFFFFu, lo);
    hi = __reduce_max_sync(0xFFFFFFFFu, hi);
    if (lane == 0) {
      sh_slot[256] = lo;
      sh_slot[257] = hi;
    }
  }
  if (warp >= kCntWarp0) {
    for (int i = tid - 32 * kCntWarp0; i < kFuseBins; i += 32 * kCntWarps) {
      sh_hist[i] = 0;
      sh_lut[i] = lut_sh && (uint32_t)i < ov.nbins ? rgba_word(i, ov.n_inputs, ov.lut) : 0u;
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     ptx::smem_u32(tmem_slot)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (is_exp && kSlots) first_loads();
  const uint32_t tmem = *tmem_slot;
  if (warp >= 1 && warp <= 4) {  // every UE8M0 block scale = 1.0
    const uint32_t lanes = (uint32_t)((warp & 3) * 32) << 16;
    tc::tmem_st16(tmem + lanes + tc::kSfCol, tc::kSfOnes);
    tc::tmem_st16(tmem + lanes + tc::kSfCol + 16, tc::kSfOnes);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();

  if (warp == 0) {
    // ===== MMA issuer =====
    if (lane == 0 && nst > 0) {
      constexpr uint32_t idA = tc::idesc_mxf4(128, 256);
      constexpr uint32_t idB = tc::idesc_mxf4(128, 128);
      // ROWS = 128: N = roundup(k, 16) columns (rows >= k are zeros and unread)
      const uint32_t idN = tc::idesc_mxf4(128, (int)min(128u, (pk + 15u) & ~15u));
      const uint32_t sfa = tmem + tc::kSfCol, sfb = tmem + tc::kSfCol + 16;
      const uint64_t d_op = tc::sw128_desc(op_base);
      for (int j = 0; j < nst; ++j) {
        const int s = j % kStages;
        ptx::mbar_wait(&full[s], (uint32_t)((j / kStages) & 1));
        tc::fence_after();
        const uint64_t d_s = d_op + (uint64_t)((uint32_t)(s * kStageBytes) >> 4);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {  // 4 MMAs of 64 K (32 B) per 128-B operand row
          const uint32_t acc = (j > 0 || ks > 0) ? 1u : 0u;
          const uint64_t lo = d_s + (uint64_t)((ks * 32) >> 4);
          const uint64_t hi = lo + (uint64_t)((128 * 128) >> 4);
#ifndef FS_RC_NO_MMA  // timing experiment only
          if (ROWS == 256) {
            tc::mma_mxf4(tmem, lo, lo, idA, acc, sfa, sfb);          // rows 0-127 x 0-255
            tc::mma_mxf4(tmem + 256u, hi, hi, idB, acc, sfa, sfb);   // rows 128-255 x 128-255
          } else {
            tc::mma_mxf4(tmem, lo, lo, idN, acc, sfa, sfb);          // rows 0-127 x 0-(N-1)
          }
#else
          (void)hi;
          (void)idN;
#endif
        }
        tc::mma_commit(&empty[s]);
      }
      tc::mma_commit(tmem_full);
    }
    __syncwarp();
  } else if (is_exp) {
    // ===== expanders: count + expand each unit from registers =====
    const uint32_t sw_lo = ((uint32_t)lane >> 3);  // row & 7 for even j; +4 for odd j
    auto count_unit = [&](int u, uint4 (&r)[8]) {
#ifndef FS_RC_NO_COUNT  // timing experiment only
      // --- partial counts of this warp's 32 rows: 8 rows per lane, then lanes ^8, ^16
      uint32_t P[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint32_t x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = i == 0 ? r[j].x : i == 1 ? r[j].y : i == 2 ? r[j].z : r[j].w;
        sum8(x, P[i]);
      }
      const bool b3 = (lane >> 3) & 1, b4 = (lane >> 4) & 1;
      uint32_t Q[2][5];  // words (b3 ? 2 : 0) and (b3 ? 3 : 1), 5 planes
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        uint32_t mine[4], other[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const uint32_t keep = b3 ? P[2 + q][p] : P[q][p];
          const uint32_t send = b3 ? P[q][p] : P[2 + q][p];
          mine[p] = keep;
          other[p] = __shfl_xor_sync(0xFFFFFFFFu, send, 8);
        }
        add_planes<4>(mine, other, Q[q]);
      }
      uint32_t R6[kPlanes];
      {
        uint32_t mine[5], other[5];
#pragma unroll
        for (int p = 0; p < 5; ++p) {
          const uint32_t keep = b4 ? Q[1][p] : Q[0][p];
          const uint32_t send = b4 ? Q[0][p] : Q[1][p];
          mine[p] = keep;
          other[p] = __shfl_xor_sync(0xFFFFFFFFu, send, 16);
        }
        add_planes<5>(mine, other, R6);
      }
      // this lane now holds word 4c + 2 b3 + b4 of the unit (c = lane % 8)
      const uint32_t wi = 4u * chunk + 2u * (uint32_t)b3 + (uint32_t)b4;
      const int ps = part_slot(u), pu = part_use(u);
      if (pu > 0) ptx::mbar_wait(&part_empty[ps], (uint32_t)((pu - 1) & 1));
      uint32_t *dst = part + ps * kPartWords + gw * kPlanes * 32;
#pragma unroll
      for (int p = 0; p < kPlanes; ++p) dst[p * 32 + wi] = R6[p];
      if (kThreadArrive) {
        ptx::mbar_arrive(&part_full[ps]);
      } else {
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&part_full[ps]);
      }
#endif
    };
    // --- operand stages s0 .. s0 + kBatch - 1 of unit u: word s of every chunk of every
    // row; one proxy fence per batch (the fence waits for this thread's stores to drain)
    auto stage_batch = [&](int u, uint4 (&r)[8], int s0) {
#pragma unroll
      for (int b = 0; b < kBatch; ++b) {
        const int j = u * 4 + s0 + b;
        if (j >= kStages) ptx::mbar_wait(&empty[j % kStages], (uint32_t)(((j / kStages) - 1) & 1));
      }
#pragma unroll
      for (int b = 0; b < kBatch; ++b) {
        const int s = s0 + b;
        const uint32_t sbase = op_base + (uint32_t)((u * 4 + s) % kStages) * kStageBytes;
#pragma unroll
        for (int jr = 0; jr < 8; ++jr) {
          const uint32_t row = (uint32_t)(32 * gw + 4 * jr) + sw_lo;
          const uint32_t swz = (sw_lo + 4u * (uint32_t)(jr & 1)) & 7u;
          const uint32_t w = s == 0 ? r[jr].x : s == 1 ? r[jr].y : s == 2 ? r[jr].z : r[jr].w;
#ifndef FS_RC_NO_EXPAND  // timing experiment only
          expand_word(sbase + row * 128u + ((chunk ^ swz) << 4), w);
#else
          if (w == 0xFFFFFFFFu && swz == 9u) expand_word(sbase, w);  // keep w live
#endif
        }
      }
      ptx::fence_proxy_async_smem();
      if (!kThreadArrive) __syncwarp();
      if (kThreadArrive || lane == 0) {
#pragma unroll
        for (int b = 0; b < kBatch; ++b) ptx::mbar_arrive(&full[(u * 4 + s0 + b) % kStages]);
      }
    };
    auto process = [&](int u, uint4 (&r)[8]) {
#if FS_RC_L2PF > 0
      if (gw == 0 && lane == 0 && u + FS_RC_L2PF < nunits) {
        // the unit's rows: a contiguous run, or the span of the slot list when it is
        // not much wider than the panel
        const uint64_t lo = kSlots ? (uint64_t)sh_slot[256] : prow0;
        const uint32_t n = kSlots ? sh_slot[257] - sh_slot[256] + 1u : pk;
        if (n <= 2u * pk)
          l2_prefetch(a.src + ((u0 + (uint64_t)(u + FS_RC_L2PF)) * a.cap + lo) * 32u, n * 128u);
      }
#endif
      count_unit(u, r);
#pragma unroll
      for (int s0 = 0; s0 < 4; s0 += kBatch) {
        stage_batch(u, r, s0);
      }
    };
    if (kGroups == 1) {
      for (int u = 0; u < nunits; u += 2) {
        process(u, ra);
        if (u + 2 < nunits) load_unit(u + 2, ra);
        if (u + 1 < nunits) {
          process(u + 1, rb);
          if (u + 3 < nunits) load_unit(u + 3, rb);
        }
      }
    } else {
      // this group's units; the next one is requested as soon as the registers are free
      // (the other group's unit and the operand ring cover its latency)
      for (int u = grp; u < nunits; u += kGroups) {
        process(u, ra);
        if (u + kGroups < nunits) load_unit(u + kGroups, ra);
      }
    }
    // ===== epilogue: TMEM -> registers -> int32 partial tile =====
    const uint32_t q = (uint32_t)(warp & 3);  // TMEM lane quarter of this warp
    const int cg = gw / 4;                    // warps sharing a quarter split the columns
    constexpr int kColStep = 32 * (kGW / 4);
    int32_t *out = a.partial + (uint64_t)blockIdx.x * ROWS * ROWS;
    if (grp == 0 && nst > 0) {
      ptx::mbar_wait(tmem_full, 0);
      tc::fence_after();
    }
#pragma unroll
    for (int h = 0; h < ROWS / 128 && grp == 0; ++h) {  // group 0 drains the accumulators
      const uint32_t row = h * 128 + q * 32 + lane;
      const int c_begin = h == 1 ? 128 : 0;
      for (int c0 = c_begin + 32 * cg; c0 < ROWS; c0 += kColStep) {
        uint32_t v[32];
        const uint32_t col = h == 1 ? (256u + (uint32_t)(c0 - 128)) : (uint32_t)c0;
        tc::tmem_ld32(tmem + ((q * 32u) << 16) + col, v);
        if (nst == 0) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0;
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = (uint32_t)__float2int_rn(__uint_as_float(v[e]));
        }
        int4 *dst = reinterpret_cast<int4 *>(out + (uint64_t)row * ROWS + c0);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          dst[e] = make_int4((int)v[4 * e], (int)v[4 * e + 1], (int)v[4 * e + 2], (int)v[4 * e + 3]);
      }
    }
    tc::fence_before();
  } else {
    // ===== combiners: 8 partial counts -> exact per-pixel counts -> emit =====
    const int cw = warp - kCntWarp0;
    for (int u0c = cw * kGroups, u = u0c; u < nunits;
         u = (u % kGroups == kGroups - 1) ? u + 1 + (kCntWarps - 1) * kGroups : u + 1) {
#ifdef FS_RC_NO_COUNT  // timing experiment only
      break;
#endif
      const int ps = part_slot(u);
      ptx::mbar_wait(&part_full[ps], (uint32_t)(part_use(u) & 1));
      const uint32_t *src = part + ps * kPartWords + lane;
      uint32_t n[kGW][kPlanes];
#pragma unroll
      for (int w = 0; w < kGW; ++w)
#pragma unroll
        for (int p = 0; p < kPlanes; ++p) n[w][p] = src[(w * kPlanes + p) * 32];
      if (kThreadArrive) {
        ptx::mbar_arrive(&part_empty[ps]);
      } else {
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&part_empty[ps]);
      }
      uint32_t cnt32[32];
      if constexpr (kGW == 8) {  // 8 x 32 rows -> 9 planes
        uint32_t s7[4][7], s8[2][8], s9[9];
#pragma unroll
        for (int i = 0; i < 4; ++i) add_planes<6>(n[2 * i], n[2 * i + 1], s7[i]);
#pragma unroll
        for (int i = 0; i < 2; ++i) add_planes<7>(s7[2 * i], s7[2 * i + 1], s8[i]);
        add_planes<8>(s8[0], s8[1], s9);
        HSCounter<5> hc;
        hc.ones = s9[0];
        hc.twos = s9[1];
        hc.fours = s9[2];
        hc.eights = s9[3];
#pragma unroll
        for (int i = 0; i < 5; ++i) hc.H[i] = s9[4 + i];
        hc.extract1(cnt32);
      } else {  // 4 x 32 rows -> 8 planes
        uint32_t s7[2][7], s8[8];
#pragma unroll
        for (int i = 0; i < 2; ++i) add_planes<6>(n[2 * i], n[2 * i + 1], s7[i]);
        add_planes<7>(s7[0], s7[1], s8);
        HSCounter<4> hc;
        hc.ones = s8[0];
        hc.twos = s8[1];
        hc.fours = s8[2];
        hc.eights = s8[3];
#pragma unroll
        for (int i = 0; i < 4; ++i) hc.H[i] = s8[4 + i];
        hc.extract1(cnt32);
      }
#ifdef FS_RC_NO_EMIT  // timing experiment only
      if (cnt32[lane & 31] == 0xFFFFFFFFu) ov.counts[0] = 0;  // keep the count live
      continue;
#endif
      if (ov.partial16 != nullptr)  // several panels: this panel's counts, summed later
        emit_partial16(cnt32, u0 + (uint64_t)u, lane, cnt_tb + cw * 32 * kTileTb,
                       ov.partial16 + (uint64_t)panel * ov.part_pitch);
      else
        emit_tile(cnt32, u0 + (uint64_t)u, lane, cnt_tb + cw * 32 * kTileTb, ov, sh_hist,
                  ov.bins != nullptr, sh_lut, lut_sh);
    }
  }
  __syncthreads();
  if (warp >= kCntWarp0 && ov.bins != nullptr) {
    for (uint32_t i = tid - 32 * kCntWarp0; i < ov.nbins; i += 32 * kCntWarps)
      if (sh_hist[i]) atomicAdd(ov.bins + i, (unsigned long long)sh_hist[i]);
    if (blockIdx.x == 0 && tid == 32 * kCntWarp0) {
      const uint64_t padpx = a.total_units * 1024 - ov.pixels;  // padding counted in bin 0
      if (padpx) atomicAdd(ov.bins, (unsigned long long)(0ull - padpx));
    }
  }
  if (warp == 0) {
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}

}  // namespace rc

namespace {
template <int ROWS, bool SLOTS>
cudaError_t launch_rc(const rc::Args &a, const OverlapArgs &ov, unsigned grid, cudaStream_t s) {
  using C = rc::Cfg<ROWS>;
  static SmemOptIn attr;
  if (cudaError_t e = smem_opt_in(attr, rc::k_recompute_f4<ROWS, SLOTS>, (size_t)C::kSmemBytes);
      e != cudaSuccess)
    return e;
  rc::k_recompute_f4<ROWS, SLOTS><<<grid, C::kThreads, C::kSmemBytes, s>>>(a, ov);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_recompute_f4(const uint32_t *src, uint64_t cap, uint64_t row0, uint32_t k,
                                uint64_t total_units, uint32_t kchunks, uint64_t upc,
                                int32_t *partial, const OverlapArgs &ov, cudaStream_t s,
                                uint32_t npanels, const uint32_t *slots, uint32_t rows) {
  if (kchunks == 0 || npanels == 0) return cudaSuccess;
  if (rows != 128 && rows != 256) return cudaErrorInvalidValue;
  rc::Args a{src, cap, row0, k, slots, total_units, upc, kchunks, partial};
  const unsigned grid = kchunks * npanels;
  if (rows == 256)
    return slots ? launch_rc<256, true>(a, ov, grid, s) : launch_rc<256, false>(a, ov, grid, s);
  return slots ? launch_rc<128, true>(a, ov, grid, s) : launch_rc<128, false>(a, ov, grid, s);
}

}  // namespace fs
