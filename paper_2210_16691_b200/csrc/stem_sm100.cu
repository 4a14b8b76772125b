// stem_sm100.cu — the window conv kernel: convolutions whose pipelined chunk
// is the tile's input window, loaded once by one TMA box, with every filter
// tap an MMA descriptor into it (the A operand is never expanded).  Modes:
// 0 / 3 the small-channel stride-2 stem (ResNet-50 conv1, 7x7/2, 3 -> 64) on
// pixel pairs (3: four output rows per tile), 1 C = 64 stride-1 convs with the
// filter resident, 2 wider stride-1 convs with the filter streamed through its
// own ring.  The pair mode is described first:
//
// The implicit-GEMM view of conv1 has K = R*S*C = 147 with C = 3: the generic
// kernel pads every filter tap to 8 channels and gathers an im2col tile per
// chunk, which re-reads each input pixel ~9x from L2 and runs the tensor
// cores on 3/8 useful lanes (0.09 of the attainable roofline, round 1).
//
// Here x is NHWC with C = 4 (3 real channels + one zero), so one 16-byte
// shared-memory row holds a PAIR of horizontally adjacent pixels
// (2u, 2u+1) x 4 channels.  With horizontal stride 2, output column q and
// filter taps (s, s+1) of equal pair offset read pair q + o: consecutive
// output columns read consecutive 16-byte rows.  That is exactly the UMMA
// K-major no-swizzle layout (core matrix = 8 rows x 16 B):
//   M row m (output column q0+m)   -> +16 B per row   (SBO = 8 rows = 128 B)
//   K group t (tap pair offset t)  -> +16 B per group (LBO = 16 B)
// so the MMA descriptors read the im2col matrix straight out of the raw
// input rows — the core matrices of neighbouring K groups overlap, shifted by
// one row.  A tile = one output row segment of 128 columns x all K filters;
// its A chunk = the R input rows the filter covers (one 4-D TMA box of
// 128-byte pixel-pair blocks, zero-filled outside the image); per filter row
// T2/2 tcgen05.mma (M=128, N=K, K=16) with the start address moved 32 B per
// k-step.  The filter (K x R x T2 x 8, zero taps where the pairing overhangs
// the filter) stays resident in shared memory for the kernel's lifetime.
//
// Pipeline: the paper's outer level is the ring of n_stage windows
// (producer_acquire = wait empty[slot], producer_commit = expect_tx + TMA,
// consumer_wait = wait full[slot], consumer_release = tcgen05.commit ->
// empty[slot]); the inner level is the ring of n_stage_inner TMEM
// accumulators, so the epilogue of tile i (TMEM -> bf16 -> TMA store) overlaps
// the MMAs of tile i+1.  Warp 0 = TMA producer, warp 1 = TMEM allocator + MMA
// issuer, warps 2-5 = epilogue.  Persistent: CTA b walks tiles b + i*grid.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "alcop_internal.h"
#include "sm100_ptx.cuh"

namespace alcop {

int encode_tiled_map(CUtensorMap* m, CUtensorMapDataType dt, const void* base, int rank, const cuuint64_t* dims,
                     const cuuint64_t* strides_bytes, const cuuint32_t* box, const cuuint32_t* estr,
                     CUtensorMapSwizzle swz, const char* what);
bool pdl_enabled();

namespace {

constexpr int kStemThreads = 352;  // producer; MMA + 4 epilogue warps per tile parity (1, 2-5 even; 6, 7-10 odd)
constexpr uint32_t kStemStaging = 32 * 128;  // one epilogue staging buffer: 32 rows x 128 B

// kMode: 0 = pixel pairs (C = 4, stride_w 2: the ResNet-50 stem); 1 = window
// (C = 64, stride 1: a TR-output-row tile reads its (TR+R-1)-row input window
// once; tap (r, s) is the window shifted by r rows and s pixels); 2 = window
// with a streamed filter (C = 64 * CB, stride 1: per 64-channel block the
// window is one chunk of the A ring and the filter comes in chunks of TB taps
// through the B ring — the two pipelined buffers with their own stage counts)
struct StemKParams {
  int32_t P, Q, QB, num_tiles;  // tile rows (output rows / row blocks) per image, output columns, column blocks
  int32_t Pout;                 // output rows per image
  int32_t R, S, T2, o_min;      // filter rows / taps, pair groups per filter row (even), pair offset of group 0
  int32_t row_step, ph, pw;     // input rows per tile row (stride_h / TR), padding
  int32_t BN;                   // = K filters (the whole N of the GEMM view)
  int32_t stages, nacc;
  uint32_t row_bytes, slot_bytes, box_bytes, wbytes;  // window row, ring slot, TMA box, resident filter
  uint32_t acc_stride, tmem_cols, idesc;
  int32_t dn, dp, dq;           // the grid as (images, tile rows, column blocks): the tile cursor's step
  int32_t shift, blk_off;       // window: first MMA row `shift` pairs in; x coordinate of column block 0
  int32_t lwp;                  // window mode: log2 of the window row pitch WP (pixels); TR = 128 / WP
  int32_t stage_bufs;           // epilogue staging buffers per warp (1 or 2)
  int32_t stage_warps;          // epilogue warps with staging (8 with two epilogue groups, else 4)
  const uint16_t* w;            // KRSC
  int32_t dual;                 // two MMA-issuing warps (1: even tiles, 6: odd tiles); even rings only
  // kMode 2 (window + streamed filter): channel blocks of 64, filter chunks of TB taps per block, the
  // filter ring (n_stage_smem_B slots of TB x BN x 128 B)
  int32_t CB, TB, nbc, sB;
  uint32_t b_slot_bytes;
  int32_t skip;                 // -DSTEM_PROBE builds only (ALCOP_STEM_SKIP): 1 no MMA, 2 no window load, 4 no store
  int32_t bn_cta;               // filter rows staged per CTA: BN, or BN / 2 on a CTA pair (window modes)
};

template <typename OutT>
__device__ __forceinline__ uint32_t pack2s(uint32_t a, uint32_t b);
template <>
__device__ __forceinline__ uint32_t pack2s<__nv_bfloat16>(uint32_t a, uint32_t b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(a), __uint_as_float(b));
  return *reinterpret_cast<uint32_t*>(&h);
}
template <>
__device__ __forceinline__ uint32_t pack2s<__half>(uint32_t a, uint32_t b) {
  __half2 h = __floats2half2_rn(__uint_as_float(a), __uint_as_float(b));
  return *reinterpret_cast<uint32_t*>(&h);
}

// Tile cursor: tile t = (image n, tile row p, column block qb), qb fastest.
// A CTA walks t = blockIdx.x + i * grid; the cursor advances by the grid's
// (dn, dp, dq) decomposition with carries — no integer division in the tile
// loops (the divisions' dependent chains on the uniform datapath cost ~900
// clk per tile in the MMA warp).
struct StemCursor {
  int n, p, qb;
  __device__ __forceinline__ void start(const StemKParams& k, int t) {
    const int per_img = k.P * k.QB;
    n = t / per_img;
    const int rem = t - n * per_img;
    p = rem / k.QB;
    qb = rem - p * k.QB;
  }
  __device__ __forceinline__ void advance(const StemKParams& k) {
    qb += k.dq;
    int carry = qb >= k.QB;
    qb -= carry ? k.QB : 0;
    p += k.dp + carry;
    carry = p >= k.P;
    p -= carry ? k.P : 0;
    n += k.dn + carry;
  }
};

// one tcgen05.mma: this CTA's (cta_group::1) or the CTA pair's (cta_group::2,
// M = 256: A rows 0-127 from the leader's shared memory, 128-255 from the
// peer's at the same address; B's N/2-row halves from each)
template <bool kPair>
__device__ __forceinline__ void stem_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (kPair)
    ptx::umma_f16_ss_pair(d, a, b, idesc, acc);
  else
    ptx::umma_f16_ss(d, a, b, idesc, acc);
}

// Issue one tile's MMAs (one elected thread).  kR/kKS (pairs) or kR/kS
// (window) fixed at compile time unroll the whole tile (immediate descriptor
// offsets); 0 = run-time loops.
template <int kMode, int kR, int kKS, bool kPair = false>
__device__ __forceinline__ void stem_tile_mmas(const StemKParams& p, uint32_t d_tmem, uint32_t a0, uint32_t wsm) {
  using namespace ptx;
  if constexpr (kMode == 0) {
    // pairs: per filter row r, T2/2 k-steps; A rows m -> pair (m + 2j [+1]) of
    // window row r (LBO 16: overlapping core matrices), B k groups (r, 2j), (r, 2j+1)
    const uint32_t lbo_b = static_cast<uint32_t>(p.BN) * 16u;
    const uint64_t b_step = (2 * lbo_b) >> 4;
    const uint64_t a_row16 = p.row_bytes >> 4;
    const uint64_t ad = make_smem_desc(a0, 16u, 128u, kLayoutNone);
    const uint64_t bd = make_smem_desc(wsm, lbo_b, 128u, kLayoutNone);
    if constexpr (kR > 0) {
#pragma unroll
      for (int r = 0; r < kR; ++r)
#pragma unroll
        for (int j = 0; j < kKS; ++j)
          umma_f16_ss(d_tmem, ad + r * a_row16 + 2 * j, bd + (r * kKS + j) * b_step, p.idesc,
                      (r > 0 || j > 0) ? 1u : 0u);
    } else {
      const int ksteps = p.T2 / 2;
      for (int r = 0; r < p.R; ++r)
        for (int j = 0; j < ksteps; ++j)
          umma_f16_ss(d_tmem, ad + r * a_row16 + 2 * j, bd + (r * ksteps + j) * b_step, p.idesc,
                      (r > 0 || j > 0) ? 1u : 0u);
    }
  } else if constexpr (kMode == 3) {
    // stem, four output rows per tile: window row e (input row 2*p0 - 3 + e,
    // e = 0..12) is the A operand once for every output row k it feeds
    // (filter row r = e - 2k in [0, 7)), with those filter rows stacked as N
    // = count x 64 — the even rows {6, 4, 2, 0} and the odd rows {5, 3, 1}
    // are each stored descending, so the rows of one MMA are adjacent — and
    // D = the adjacent 64-column accumulators of output rows k_min..k_max.
    // Output row k starts at e = 2k (r = 0): that piece is split off with
    // accumulate = 0; every other piece accumulates.
    const uint64_t a_row16 = p.row_bytes >> 4;
    const uint64_t ad = make_smem_desc(a0, 16u, 128u, kLayoutNone);
#pragma unroll
    for (int e = 0; e < 13; ++e) {
      const int cls = e & 1;
      const int nj = cls ? 3 : 4;                         // filter rows in the class
      const int kmin = e <= 6 ? 0 : (e - 5) / 2;          // ceil((e - 6) / 2)
      const int kmax = (e / 2) < 3 ? (e / 2) : 3;
      const int j0 = ((cls ? 5 : 6) - (e - 2 * kmin)) / 2;  // class block of filter row e - 2 kmin
      const bool starts = !cls && e / 2 <= 3;             // output row kmax gets its first piece (r = 0)
      const uint32_t cbase = wsm + (cls ? 4u * 4u * 64u * 16u : 0u);
      const uint32_t lbo_b = static_cast<uint32_t>(nj) * 64u * 16u;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint64_t ade = ad + e * a_row16 + 2 * u;
        const uint32_t bt = cbase + 2u * u * lbo_b;  // pair groups 2u, 2u+1
        if (starts && u == 0) {
          const int cnt = kmax - kmin;  // rows already under way
          if (cnt > 0)
            umma_f16_ss(d_tmem + kmin * 64, ade, make_smem_desc(bt + j0 * 1024u, lbo_b, 128u, kLayoutNone),
                        (p.idesc & ~(0x3Fu << 17)) | ((cnt * 64u >> 3) << 17), 1u);
          umma_f16_ss(d_tmem + kmax * 64, ade,
                      make_smem_desc(bt + (j0 + cnt) * 1024u, lbo_b, 128u, kLayoutNone),
                      (p.idesc & ~(0x3Fu << 17)) | ((64u >> 3) << 17), 0u);
        } else {
          const int cnt = kmax - kmin + 1;
          umma_f16_ss(d_tmem + kmin * 64, ade, make_smem_desc(bt + j0 * 1024u, lbo_b, 128u, kLayoutNone),
                      (p.idesc & ~(0x3Fu << 17)) | ((cnt * 64u >> 3) << 17), 1u);
        }
      }
    }
  } else {
    // window: tap (r, s) = A rows m -> window pixel m + r*WP + s (128 B each,
    // 128B-swizzled: the swizzle follows the absolute smem address, so a
    // start moved by whole 128-byte rows reads the shifted rows, base offset
    // 0 — tools/desc_probe.cu); 4 k-steps of 16 channels per tap; B tap t =
    // BN rows x 64 channels, 128B-swizzled
    const uint64_t ad = make_smem_desc(a0, 16u, 1024u, kLayoutSW128);
    const uint64_t bd = make_smem_desc(wsm, 16u, 1024u, kLayoutSW128);
    const uint64_t a_row16 = (128u << p.lwp) >> 4;  // one window row
    const uint64_t b_tap16 = (static_cast<uint32_t>(p.bn_cta) * 128u) >> 4;
    if constexpr (kR > 0) {
#pragma unroll
      for (int r = 0; r < kR; ++r)
#pragma unroll
        for (int s = 0; s < kKS; ++s)
#pragma unroll
          for (int u = 0; u < 4; ++u)
            stem_mma<kPair>(d_tmem, ad + r * a_row16 + s * 8 + 2 * u, bd + (r * kKS + s) * b_tap16 + 2 * u, p.idesc,
                            (r > 0 || s > 0 || u > 0) ? 1u : 0u);
    } else {
      for (int r = 0; r < p.R; ++r)
        for (int s = 0; s < p.S; ++s)
#pragma unroll
          for (int u = 0; u < 4; ++u)
            stem_mma<kPair>(d_tmem, ad + r * a_row16 + s * 8 + 2 * u, bd + (r * p.S + s) * b_tap16 + 2 * u, p.idesc,
                            (r > 0 || s > 0 || u > 0) ? 1u : 0u);
    }
  }
}

// kPair (window modes 1, 2): a cluster of two CTAs computes a 256-pixel tile
// with tcgen05.mma.cta_group::2 — each CTA loads the window of its own TR
// output rows (tile rows 2u, 2u+1 of the pair tile u) and stages half of the
// filter rows (bn_cta = BN / 2), so per 128 output pixels the MMAs read half
// the filter bytes from each SM's shared memory (the port both the MMA operand
// reads and the TMA fills share, ~128 B/clk).  Both CTAs' loads complete on
// the leader's barriers, the leader's MMA warps issue for the pair, their
// commits multicast the releases to both CTAs, and each CTA's epilogue drains
// its own TMEM and hands the accumulator back on the leader's barrier.
template <typename OutT, int kMode, int kR, int kKS, bool kPair = false>
__global__ void __launch_bounds__(kStemThreads, 1)
    alcop_stem_conv_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmY,
                           const __grid_constant__ CUtensorMap tmW, const StemKParams p) {
  using namespace ptx;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t ring = smem_u32(smem);
  const uint32_t ringB = ring + p.stages * p.slot_bytes;  // kMode 2: the filter ring
  const uint32_t wsm = ringB + p.sB * p.b_slot_bytes;
  const uint32_t staging = wsm + p.wbytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.stages * p.slot_bytes + p.sB * p.b_slot_bytes + p.wbytes +
                                               p.stage_warps * p.stage_bufs * kStemStaging);
  uint64_t* full = bars;
  uint64_t* empty = full + p.stages;
  uint64_t* tfull = empty + p.stages;
  uint64_t* tempty = tfull + p.nacc;
  uint64_t* bfull = tempty + p.nacc;
  uint64_t* bempty = bfull + p.sB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bempty + p.sB);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const uint32_t rank = kPair ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmY);
    if (kMode == 2) prefetch_tmap(&tmW);
  }
  if (warp == 1) {
    if (lane == 0) {
      for (int i = 0; i < p.stages; ++i) {
        mbar_init(smem_u32(&full[i]), 1);
        mbar_init(smem_u32(&empty[i]), 1);
      }
      for (int i = 0; i < p.nacc; ++i) {
        mbar_init(smem_u32(&tfull[i]), 1);
        mbar_init(smem_u32(&tempty[i]), kPair ? 8 : 4);  // 4 epilogue warps (x 2 CTAs)
      }
      for (int i = 0; i < p.sB; ++i) {
        mbar_init(smem_u32(&bfull[i]), 1);
        mbar_init(smem_u32(&bempty[i]), 1);
      }
      fence_barrier_init();
    }
    __syncwarp();
    if constexpr (kPair) {
      tmem_alloc_pair(smem_u32(tmem_slot), p.tmem_cols);
      tmem_relinquish_pair();
    } else {
      tmem_alloc(smem_u32(tmem_slot), p.tmem_cols);
      tmem_relinquish();
    }
  }
  if constexpr (kPair) cluster_sync();  // both CTAs' barriers initialised before any remote arrive / complete_tx
  // PDL: setup overlapped the previous kernel's tail; global data from here on
  grid_dependency_wait();
  grid_launch_dependents();

  // The filter, resident in shared memory for the kernel's lifetime.
  if constexpr (kMode == 3) {
    // two classes of filter rows, each [pair group t][class block j][filter n][8
    // elements]: even rows 6, 4, 2, 0 (j = 0..3), odd rows 5, 3, 1 (j = 0..2);
    // element e = (tap parity e/4, channel e%4) as in the pair mode
    for (int idx = threadIdx.x; idx < 7 * 4 * 64; idx += blockDim.x) {
      const int n = idx & 63, rest = idx >> 6;  // rest = (class slot, t)
      const int t = rest & 3, js = rest >> 2;   // js = 0..6: even j 0..3, odd j 0..2
      const int cls = js >= 4, j = cls ? js - 4 : js;
      const int r = cls ? 5 - 2 * j : 6 - 2 * j;
      uint32_t v[4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int sx = 2 * (p.o_min + t) + h + p.pw;
        uint2 taps = make_uint2(0u, 0u);
        if (sx >= 0 && sx < p.S)
          taps = __ldg(reinterpret_cast<const uint2*>(p.w + ((static_cast<int64_t>(n) * p.R + r) * p.S + sx) * 4));
        v[2 * h] = taps.x;
        v[2 * h + 1] = taps.y;
      }
      const int nj = cls ? 3 : 4;
      const uint32_t off = (cls ? 4u * 4u * 64u * 16u : 0u) + ((t * nj + j) * 64u + n) * 16u;
      st_shared_v4(wsm + off, v[0], v[1], v[2], v[3]);
    }
  } else if constexpr (kMode == 0) {
    // B operand in the K-major no-swizzle layout [k group kg][filter n][8
    // elements] (LBO = BN*16 bytes between k groups, SBO = 128 bytes between
    // 8-filter groups).  k group kg = (filter row r, pair group t); element e
    // = (tap parity e/4, channel e%4); tap s = 2*(o_min+t) + e/4 + pad_w, zero
    // outside [0, S) (the pairing overhangs the filter by at most one tap).
    const int groups = p.R * p.T2;
    for (int idx = threadIdx.x; idx < groups * p.BN; idx += blockDim.x) {
      const int kg = idx / p.BN, n = idx - kg * p.BN;
      const int r = kg / p.T2, t = kg - r * p.T2;
      uint32_t v[4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int s = 2 * (p.o_min + t) + h + p.pw;
        uint2 taps = make_uint2(0u, 0u);
        if (s >= 0 && s < p.S)  // 4 channels of tap s: 8 bytes, 8-byte aligned (C = 4)
          taps = __ldg(reinterpret_cast<const uint2*>(p.w + ((static_cast<int64_t>(n) * p.R + r) * p.S + s) * 4));
        v[2 * h] = taps.x;
        v[2 * h + 1] = taps.y;
      }
      st_shared_v4(wsm + static_cast<uint32_t>(idx) * 16u, v[0], v[1], v[2], v[3]);
    }
  } else if constexpr (kMode == 1) {
    // B operand per tap t = (r, s): BN filter rows x 64 channels (128 B),
    // 128B-swizzled K-major ([t][n][128 B], 16-byte chunk c of row n at c ^ (n & 7))
    // (a CTA pair: filters rank * bn_cta .. + bn_cta - 1 in each CTA)
    const int rows = p.R * p.S * p.bn_cta;
    for (int idx = threadIdx.x; idx < rows * 8; idx += blockDim.x) {
      const int row = idx >> 3, c = idx & 7;
      const int t = row / p.bn_cta, n = row - t * p.bn_cta;
      const int64_t f = static_cast<int64_t>(rank) * p.bn_cta + n;
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(p.w + (f * p.R * p.S + t) * 64) + c);
      st_shared_v4(wsm + static_cast<uint32_t>(row) * 128u + ((c ^ (n & 7)) << 4), v.x, v.y, v.z, v.w);
    }
  }
  fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor cores
  tc_fence_before();
  if constexpr (kPair)
    cluster_sync();  // the leader's MMAs read the peer's filter half
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // the work unit: a CTA, or a CTA pair (cluster) walking pair tiles
  const int grid = kPair ? static_cast<int>(gridDim.x) >> 1 : static_cast<int>(gridDim.x);
  const int unit = kPair ? static_cast<int>(blockIdx.x) >> 1 : static_cast<int>(blockIdx.x);
  const int my_tiles = (p.num_tiles - unit + grid - 1) / grid;

  if (warp == 0) {
    // ======================= producer (TMA) =======================
    // the whole warp walks the loop (coordinates stay on the uniform
    // datapath), one elected lane issues
    // (a CTA pair: each CTA loads its own tile row's window and filter half,
    // completing on the leader's barriers, which the leader arms with both
    // CTAs' bytes; each waits on its own empty barriers, which the leader's
    // commits multicast)
    int slot = 0, bslot = 0;
    uint32_t phase = 0, bphase = 0;
    StemCursor cur;
    cur.start(p, unit);
    for (int tl = 0; tl < my_tiles; ++tl, cur.advance(p)) {
      const int prow = kPair ? 2 * cur.p + static_cast<int>(rank) : cur.p;  // this CTA's tile row
      for (int cb = 0; cb < (kMode == 2 ? p.CB : 1); ++cb) {
        mbar_wait(smem_u32(&empty[slot]), ((phase >> slot) & 1u) ^ 1u);  // producer_acquire (window)
        phase ^= 1u << slot;
        if (elect_one()) {
          if (p.skip & 2) {
            if (leader) mbar_arrive(smem_u32(&full[slot]));
          } else if constexpr (kPair) {
            const uint32_t fb = smem_u32(&full[slot]);
            if (leader) mbar_arrive_expect_tx(fb, 2 * p.box_bytes);        // producer_commit (both windows)
            tma_load_4d_pair(ring + slot * p.slot_bytes, &tmX, mapa_shared(fb, 0), cb * 64, cur.qb * 16 + p.blk_off,
                             prow * p.row_step - p.ph, cur.n);
          } else {
            mbar_arrive_expect_tx(smem_u32(&full[slot]), p.box_bytes);      // producer_commit
            tma_load_4d(ring + slot * p.slot_bytes, &tmX, smem_u32(&full[slot]), cb * 64, cur.qb * 16 + p.blk_off,
                        prow * p.row_step - p.ph, cur.n);
          }
        }
        __syncwarp();
        slot = slot + 1 == p.stages ? 0 : slot + 1;
        if constexpr (kMode == 2) {
          // this channel block's filter, TB taps per chunk: tap t = filter columns t*C + cb*64 .. +63
          for (int j = 0; j < p.nbc; ++j) {
            mbar_wait(smem_u32(&bempty[bslot]), ((bphase >> bslot) & 1u) ^ 1u);
            bphase ^= 1u << bslot;
            if (elect_one()) {
              const uint32_t bb = smem_u32(&bfull[bslot]);
              if (leader) mbar_arrive_expect_tx(bb, p.TB * p.BN * 128u);  // both halves: TB x BN rows
              for (int t = 0; t < p.TB; ++t) {
                const uint32_t dst = ringB + bslot * p.b_slot_bytes + t * p.bn_cta * 128u;
                const int col = (j * p.TB + t) * p.CB * 64 + cb * 64;
                if constexpr (kPair)
                  tma_load_3d_pair(dst, &tmW, mapa_shared(bb, 0), col, static_cast<int>(rank) * p.bn_cta, 0);
                else
                  tma_load_3d(dst, &tmW, bb, col, 0, 0);
              }
            }
            __syncwarp();
            bslot = bslot + 1 == p.sB ? 0 : bslot + 1;
          }
        }
      }
    }
  } else if (warp == 1 || warp == 6) {
    // ======================= MMA issuers =======================
    // warp-uniform loop, one elected lane issues: the descriptors stay in
    // uniform registers (a single-thread loop made the compiler move every
    // descriptor into uniform registers per MMA — ~250 clk per tcgen05.mma).
    // Two issuing warps take alternate tiles (their own slots and
    // accumulators: both rings are even), so one warp's barrier waits and
    // commits (~500 clk per tile) overlap the other's MMAs; each warp's
    // tcgen05.commit tracks only the MMAs it issued.
    const int first = warp == 6 ? 1 : 0;
    const int step = p.dual ? 2 : 1;
    // a commit releasing a barrier in this CTA, or in both CTAs of the pair
    auto commit = [&](uint64_t* bar) {
      if constexpr (kPair)
        umma_commit_pair_multicast(smem_u32(bar), 0x3);
      else
        umma_commit(smem_u32(bar));
    };
    if (kPair && !leader) {
      // the peer CTA issues nothing: the leader's MMAs cover both
    } else if constexpr (kMode == 2) {
      // one issuing warp (the rings carry several chunks per tile in order)
      if (warp == 1) {
        int slot = 0, bslot = 0, acc = 0;
        uint32_t phase = 0, bphase = 0, acc_phase = 0;
        const uint64_t a_row16 = (128u << p.lwp) >> 4;
        const uint64_t b_tap16 = (static_cast<uint32_t>(p.bn_cta) * 128u) >> 4;
        for (int tl = 0; tl < my_tiles; ++tl) {
          mbar_wait(smem_u32(&tempty[acc]), ((acc_phase >> acc) & 1u) ^ 1u);
          acc_phase ^= 1u << acc;
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * p.acc_stride;
          for (int cb = 0; cb < p.CB; ++cb) {
            mbar_wait(smem_u32(&full[slot]), (phase >> slot) & 1u);     // consumer_wait (window)
            phase ^= 1u << slot;
            const uint64_t ad = make_smem_desc(ring + slot * p.slot_bytes, 16u, 1024u, kLayoutSW128);
            int r = 0, sx = 0;  // tap of the chunk's first filter column
            for (int j = 0; j < p.nbc; ++j) {
              mbar_wait(smem_u32(&bfull[bslot]), (bphase >> bslot) & 1u);  // consumer_wait (filter chunk)
              bphase ^= 1u << bslot;
              tc_fence_after();
              if (elect_one()) {
                const uint64_t bd = make_smem_desc(ringB + bslot * p.b_slot_bytes, 16u, 1024u, kLayoutSW128);
                int rr = r, ss = sx;
                for (int t = 0; t < p.TB; ++t) {
#pragma unroll
                  for (int u = 0; u < 4; ++u)
                    stem_mma<kPair>(d_tmem, ad + rr * a_row16 + ss * 8 + 2 * u, bd + t * b_tap16 + 2 * u, p.idesc,
                                    (cb > 0 || j > 0 || t > 0 || u > 0) ? 1u : 0u);
                  if (++ss == p.S) {
                    ss = 0;
                    ++rr;
                  }
                }
                commit(&bempty[bslot]);                     // consumer_release (filter chunk)
                if (j == p.nbc - 1) commit(&empty[slot]);   // consumer_release (window)
                if (j == p.nbc - 1 && cb == p.CB - 1) commit(&tfull[acc]);
              }
              __syncwarp();
              sx += p.TB;
              while (sx >= p.S) {
                sx -= p.S;
                ++r;
              }
              bslot = bslot + 1 == p.sB ? 0 : bslot + 1;
            }
            slot = slot + 1 == p.stages ? 0 : slot + 1;
          }
          if (++acc == p.nacc) acc = 0;
        }
      }
    } else if (!(warp == 6 && !p.dual)) {
      int slot = first % p.stages;
      int acc = first % p.nacc;
      uint32_t phase = 0, acc_phase = 0;  // bit k: current parity of ring slot / accumulator k
      for (int tl = first; tl < my_tiles; tl += step) {
        mbar_wait(smem_u32(&tempty[acc]), ((acc_phase >> acc) & 1u) ^ 1u);  // accumulator drained
        acc_phase ^= 1u << acc;
        tc_fence_after();
        mbar_wait(smem_u32(&full[slot]), (phase >> slot) & 1u);             // consumer_wait
        phase ^= 1u << slot;
        tc_fence_after();
        if (elect_one()) {
          if (!(p.skip & 1))
            stem_tile_mmas<kMode, kR, kKS, kPair>(p, tmem_base + acc * p.acc_stride,
                                                  ring + slot * p.slot_bytes + static_cast<uint32_t>(p.shift) * 16u,
                                                  wsm);
          commit(&empty[slot]);  // consumer_release: the window slot is free once these retire
          commit(&tfull[acc]);   // accumulator ready
        }
        __syncwarp();
        slot += step;
        if (slot >= p.stages) slot -= p.stages;
        acc += step;
        if (acc >= p.nacc) acc -= p.nacc;
      }
    }
    __syncwarp();
  } else if ((warp >= 2 && warp <= 5) || (warp >= 7 && p.dual)) {
    // ======================= epilogue (warps 2-5: even tiles, 7-10: odd tiles) =======================
    // with two issuing warps the tiles split into two independent
    // MMA -> epilogue pipelines (their own accumulators); one group's TMEM
    // drain, staging and TMA store overlap the other's.  TMEM lane quarter q
    // holds tile rows m = 32q..32q+31: pairs mode, output columns q0 + m of
    // one output row; window mode, output (row m / WP, column m % WP) of the
    // tile's TR rows.
    const int q = warp & 3;
    const int first = warp >= 7 ? 1 : 0;
    const int step = p.dual ? 2 : 1;
    const uint32_t stage_base = staging + (warp >= 7 ? warp - 3 : warp - 2) * p.stage_bufs * kStemStaging;
    constexpr int kChunkCols = 128 / static_cast<int>(sizeof(OutT));
    const int nchunks = p.BN / kChunkCols;
    int buf = 0;
    int acc = first % p.nacc;
    uint32_t acc_phase = 0;
    StemCursor cur;
    cur.start(p, unit);
    if (first) cur.advance(p);
    // this warp's first output (column, row-in-tile) of the tile
    const int m0 = q * 32;
    constexpr bool kPairs = kMode == 0 || kMode == 3;
    const int col0 = kPairs ? m0 : (m0 & ((1 << p.lwp) - 1));
    const int row0 = kPairs ? 0 : (m0 >> p.lwp);
    constexpr int kSub = kMode == 3 ? 4 : 1;  // output rows per tile held side by side in TMEM (stem4)
    for (int tl = first; tl < my_tiles; tl += step, cur.advance(p), (step == 2 ? cur.advance(p) : void())) {
      mbar_wait(smem_u32(&tfull[acc]), (acc_phase >> acc) & 1u);
      acc_phase ^= 1u << acc;
      tc_fence_after();
      const uint32_t t_addr = tmem_base + acc * p.acc_stride + (static_cast<uint32_t>(q * 32) << 16);
      const int oq = cur.qb * 128 + col0;  // output column of row m0
      for (int ic = 0; ic < kSub * nchunks; ++ic) {
        const int k = kSub == 1 ? 0 : ic / nchunks, c = kSub == 1 ? ic : ic - k * nchunks;
        const uint32_t ta = t_addr + k * p.BN;
        const int prow = kPair ? 2 * cur.p + static_cast<int>(rank) : cur.p;  // this CTA's tile row
        const int op = kMode == 0 ? prow : kMode == 3 ? prow * 4 + k : prow * p.row_step + row0;  // output row
        const bool rows_live = oq < p.Q && op < p.Pout;
        uint32_t w[32];
        if constexpr (sizeof(OutT) == 4) {
          tmem_ld_32x32b_x32(ta + c * 32, w);
          tmem_wait_ld();
        } else {
          uint32_t r0[32], r1[32];
          tmem_ld_32x32b_x32(ta + c * 64, r0);
          tmem_ld_32x32b_x32(ta + c * 64 + 32, r1);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            w[i] = pack2s<OutT>(r0[2 * i], r0[2 * i + 1]);
            w[16 + i] = pack2s<OutT>(r1[2 * i], r1[2 * i + 1]);
          }
        }
        if (ic == kSub * nchunks - 1) {  // this warp's TMEM reads of the accumulator are done
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (kPair)
              mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));  // the leader's barrier
            else
              mbar_arrive(smem_u32(&tempty[acc]));
          }
        }
        if (!rows_live || (p.skip & 4)) continue;  // tile rows past the image (the M=128 tile overhangs it)
        const uint32_t sbuf = stage_base + buf * kStemStaging;
        if (lane == 0) {  // the store that last read sbuf is done
          if (p.stage_bufs == 2)
            bulk_wait_group_read<1>();
          else
            bulk_wait_group_read<0>();
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j)
          st_shared_v4(sbuf + lane * 128 + ((j ^ (lane & 7)) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2],
                       w[4 * j + 3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_4d(&tmY, sbuf, c * kChunkCols, oq, op, cur.n);
          bulk_commit_group();
        }
        buf ^= p.stage_bufs - 1;
      }
      acc += step;
      if (acc >= p.nacc) acc -= p.nacc;
    }
    if (lane == 0) bulk_wait_group_read<0>();
    __syncwarp();
  }

  tc_fence_before();
  if constexpr (kPair)
    cluster_sync();  // no CTA leaves while its peer may still signal it or read its shared memory
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (kPair)
      tmem_dealloc_pair(tmem_base, p.tmem_cols);
    else
      tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

template <typename OutT>
int launch_stem_typed(const CUtensorMap& tx, const CUtensorMap& ty, const CUtensorMap& tw, const StemKParams& kp,
                      int mode, bool pair, int grid, int smem, cudaStream_t st) {
  const bool r3 = kp.R == 3 && kp.S == 3;
  auto kern = pair ? (mode == 2 ? alcop_stem_conv_kernel<OutT, 2, 0, 0, true>
                      : r3      ? alcop_stem_conv_kernel<OutT, 1, 3, 3, true>
                                : alcop_stem_conv_kernel<OutT, 1, 0, 0, true>)
              : mode == 3 ? alcop_stem_conv_kernel<OutT, 3, 7, 2>
              : mode == 2 ? alcop_stem_conv_kernel<OutT, 2, 0, 0>
              : mode == 1 ? (r3 ? alcop_stem_conv_kernel<OutT, 1, 3, 3> : alcop_stem_conv_kernel<OutT, 1, 0, 0>)
                          : (kp.R == 7 && kp.T2 == 4 ? alcop_stem_conv_kernel<OutT, 0, 7, 2>
                                                     : alcop_stem_conv_kernel<OutT, 0, 0, 0>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_error(ALCOP_ERR_CUDA, "CudaError", cudaGetErrorString(e));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kStemThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;  // CTA pairs (window modes, cta_group 2)
  attr[1].val.clusterDim.x = pair ? 2 : 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pair ? 2 : 1;
  e = cudaLaunchKernelEx(&cfg, kern, tx, ty, tw, kp);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ALCOP_ERR_CUDA, "CudaError", cudaGetErrorString(e));
  return ALCOP_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
static int out_bytes(const alcop_conv_desc& d) { return d.out_dtype == ALCOP_F32 ? 4 : 2; }

bool stem_pairs_applicable(const alcop_conv_desc& d) {
  return d.C == 4 && d.stride_w == 2 && !d.x_halo && d.W % 16 == 0 && d.K % 16 == 0 && d.K >= 16 && d.K <= 256 &&
         (d.K * out_bytes(d)) % 128 == 0 && d.R <= 32 && d.S <= 32 && d.stride_h <= 8 && d.pad_h <= 64 &&
         d.pad_w <= 64;
}

// window row pitch: the smallest power of two >= Q + S - 1 (a valid output
// column's taps stay inside its window row), at least 16, at most 128
static int64_t window_pitch(const alcop_conv_desc& d) {
  const int64_t Q = (d.W + 2 * d.pad_w - d.S) / d.stride_w + 1;
  int64_t wp = 16;
  while (wp < Q + d.S - 1) wp *= 2;
  return wp;
}

static bool window_common(const alcop_conv_desc& d) {
  if (!(d.stride_h == 1 && d.stride_w == 1 && !d.x_halo && d.K % 16 == 0 && d.K >= 16 && d.K <= 256 &&
        (d.K * out_bytes(d)) % 128 == 0 && d.R <= 8 && d.S <= 8 && d.pad_h <= 8 && d.pad_w <= 8 &&
        (d.R > 1 || d.S > 1)))
    return false;
  // 1x1 convs stay on the GEMM kernels (both HBM-bound, tools/window1x1_probe.py)
  const int64_t wp = window_pitch(d);
  if (wp > 128) return false;
  const int64_t tr = 128 / wp;
  const int64_t P = (d.H + 2 * d.pad_h - d.R) + 1;
  // worth it only when the tile rows are mostly real output (not a 7x7 map in 8-row tiles)
  return P >= tr && (tr + d.R - 1) * wp <= 256;
}

bool window_conv_applicable(const alcop_conv_desc& d) {
  // the resident filter leaves room for a 2-slot window ring
  return d.C == 64 && window_common(d) && d.R * d.S * d.K * 128 <= 80 * 1024;
}

bool window_stream_applicable(const alcop_conv_desc& d) {
  // the window saves the im2col kernel's A re-reads: half of its L2 -> SM
  // bytes at K = 128, a third at K = 256, where the im2col kernel's deeper
  // 48 KB stages win (ResNet-50 l3 3x3: 1297 vs 1130 TFLOP/s; l2 3x3, K = 128:
  // 888 -> 1098 TFLOP/s on the window kernel)
  return d.C % 64 == 0 && d.K <= 128 && !window_conv_applicable(d) && window_common(d);
}

// the ResNet-50 stem exactly (7x7, stride 2, pad 3, K 64): four output rows
// per tile with the filter rows stacked along N (kMode 3)
static bool stem4_applicable(const alcop_conv_desc& d) {
  return stem_pairs_applicable(d) && d.R == 7 && d.S == 7 && d.stride_h == 2 && d.stride_w == 2 && d.pad_h == 3 &&
         d.pad_w == 3 && d.K == 64 && (d.H + 2 * d.pad_h - d.R) / d.stride_h + 1 >= 4;
}

// 0 = pixel pairs, 1 = window (resident filter), 2 = window (streamed filter),
// 3 = pixel pairs, four output rows per tile (the ResNet-50 stem), -1 = none
static int stem_mode(const alcop_conv_desc& d) {
  if (d.C == 4) return stem4_applicable(d) ? 3 : 0;
  if (window_conv_applicable(d)) return 1;
  if (window_stream_applicable(d)) return 2;
  return -1;
}

StemGeometry stem_pairs_geometry(const alcop_conv_desc& d) {
  StemGeometry g{};
  g.P = (d.H + 2 * d.pad_h - d.R) / d.stride_h + 1;
  g.Q = (d.W + 2 * d.pad_w - d.S) / d.stride_w + 1;
  const int mode = stem_mode(d);
  if (mode == 1 || mode == 2) {  // window modes
    const int64_t wp = window_pitch(d);
    const int64_t tr = 128 / wp;
    g.QB = 1;
    g.TR = static_cast<int32_t>(tr);
    g.WP = static_cast<int32_t>(wp);
    g.row_bytes = static_cast<uint32_t>(wp * 128);
    g.box_bytes = static_cast<uint32_t>((tr + d.R - 1) * wp * 128);
    // + S-1 pixels of slack: the taps of the tile's last (overhanging, never
    // stored) rows read past the box
    g.slot_bytes = static_cast<uint32_t>((g.box_bytes + (d.S - 1) * 128 + 1023) / 1024 * 1024);
    g.wbytes = mode == 1 ? static_cast<uint32_t>((d.R * d.S * d.K * 128 + 1023) / 1024 * 1024) : 0u;
    g.kdim = d.R * d.S * d.C;
    return g;
  }
  g.QB = (g.Q + 127) / 128;
  // tap s reads pixel 2q - pad_w + s = pair q + floor((s - pad_w) / 2)
  auto fdiv2 = [](int64_t v) { return v >= 0 ? v / 2 : -((1 - v) / 2); };
  g.o_min = static_cast<int32_t>(fdiv2(-d.pad_w));
  const int32_t o_max = static_cast<int32_t>(fdiv2(d.S - 1 - d.pad_w));
  const int32_t T = o_max - g.o_min + 1;
  g.T2 = (T + 1) & ~1;
  // window: shift (0..7) + 128 rows + T2-1 further pairs, in 8-pair (128 B) blocks
  g.NB = (7 + 128 + g.T2 - 1 + 7) / 8;
  g.row_bytes = static_cast<uint32_t>(g.NB * 128);
  // four output rows per tile (mode 3): the window covers 2 * 3 + R input rows
  const int64_t wrows = mode == 3 ? 3 * d.stride_h + d.R : d.R;
  g.TR = mode == 3 ? 4 : 1;
  g.box_bytes = static_cast<uint32_t>(wrows * g.row_bytes);
  g.slot_bytes = static_cast<uint32_t>((g.box_bytes + 1023) / 1024 * 1024);
  g.wbytes = static_cast<uint32_t>((d.R * g.T2 * d.K * 16 + 1023) / 1024 * 1024);
  g.kdim = d.R * g.T2 * 8;
  return g;
}

// filter rows staged per CTA: all K, or K / 2 on a CTA pair
static int64_t filter_rows_cta(const alcop_conv_desc& d, const alcop_schedule& s) {
  return s.cta_group == 2 ? d.K / 2 : d.K;
}
// streamed filter: taps per filter chunk (tileK = 64 x taps), ring of n_stage_smem_B chunks
static int64_t stream_b_slot_bytes(const alcop_conv_desc& d, const alcop_schedule& s) {
  return stem_mode(d) == 2 ? (s.tileK / 64) * filter_rows_cta(d, s) * 128 : 0;
}
// the resident filter (window mode 1): this CTA's rows of every tap
static int64_t resident_filter_bytes(const alcop_conv_desc& d, const alcop_schedule& s, const StemGeometry& g) {
  if (stem_mode(d) != 1) return g.wbytes;
  return (d.R * d.S * filter_rows_cta(d, s) * 128 + 1023) / 1024 * 1024;
}
static bool stem_dual(const alcop_conv_desc& d, const alcop_schedule& s) {
  return stem_mode(d) != 2 && s.n_stage_smem_A % 2 == 0 && s.n_stage_inner % 2 == 0;
}

static int64_t stem_smem_bytes_bufs(const alcop_conv_desc& d, const alcop_schedule& s, int bufs) {
  const StemGeometry g = stem_pairs_geometry(d);
  const bool streamed = stem_mode(d) == 2;
  const int64_t sB = streamed ? s.n_stage_smem_B : 0;
  const int64_t bars = 8 * (2 * s.n_stage_smem_A + 2 * s.n_stage_inner + 2 * sB) + 16;
  const int warps = stem_dual(d, s) ? 8 : 4;
  return 1024 + s.n_stage_smem_A * static_cast<int64_t>(g.slot_bytes) + sB * stream_b_slot_bytes(d, s) +
         resident_filter_bytes(d, s, g) + warps * bufs * kStemStaging + bars;
}

// two staging buffers per epilogue warp when they fit, else one
static int stem_staging_bufs(const alcop_conv_desc& d, const alcop_schedule& s) {
  return stem_smem_bytes_bufs(d, s, 2) <= kMaxSmemBytes ? 2 : 1;
}

int64_t stem_pairs_smem_bytes(const alcop_conv_desc& d, const alcop_schedule& s) {
  return stem_smem_bytes_bufs(d, s, stem_staging_bufs(d, s));
}

int validate_stem_pairs(const alcop_conv_desc& d, const alcop_schedule& s) {
  const int mode = stem_mode(d);
  if (mode < 0)
    return set_error(ALCOP_ERR_CONFIG, "Unsupported", "not a shape of the resident-filter / window conv kernel");
  const bool tk_ok = s.tileK == 64 || (mode == 2 && s.tileK == 64 * d.S);
  const bool window = mode == 1 || mode == 2;
  if (s.cta_group != 1 && !(s.cta_group == 2 && window && d.K % 32 == 0))
    return set_error(ALCOP_ERR_CONFIG, "BadSchedule",
                     "the window conv kernel runs one CTA per tile, or a CTA pair per 256-pixel tile in the window "
                     "modes (cta_group 2, K % 32 == 0)");
  if (s.tileM != kTileM * s.cta_group || !tk_ok || s.tileN != d.K)
    return set_error(ALCOP_ERR_CONFIG, "BadSchedule",
                     "the window conv kernel's tile is 128 output pixels (256 on a CTA pair) x all K filters "
                     "(tileM 128 x cta_group, tileN = K, tileK 64; streamed filter: tileK 64 or 64 x S = taps per "
                     "filter chunk)");
  if (s.stream_k != 0 || s.mode != ALCOP_MODE_FUSED)
    return set_error(ALCOP_ERR_CONFIG, "BadSchedule", "the window conv kernel runs whole tiles (FUSED, no stream-K)");
  if (mode == 2) {
    if (s.n_stage_smem_A < 1 || s.n_stage_smem_A > 4 || s.n_stage_smem_B < 1 || s.n_stage_smem_B > kMaxStages)
      return set_error(ALCOP_ERR_CONFIG, "BadSchedule", "streamed filter: window stages 1..4, filter stages 1..16");
  } else if (s.n_stage_smem_A != s.n_stage_smem_B || s.n_stage_smem_A < 1 || s.n_stage_smem_A > kMaxStages) {
    return set_error(ALCOP_ERR_CONFIG, "BadSchedule", "the window ring: equal A/B stages in 1..16");
  }
  const int max_inner = mode == 2 ? 2 : 8;
  const int64_t acc_cols = (mode == 3 ? 4 : 1) * d.K;  // mode 3: four output rows side by side
  if (s.n_stage_inner < 1 || s.n_stage_inner > max_inner || s.n_stage_inner * acc_cols > kTmemCols)
    return set_error(ALCOP_ERR_CONFIG, "TmemCapacity", "n_stage_inner accumulators of K columns exceed TMEM");
  if (stem_pairs_smem_bytes(d, s) > kMaxSmemBytes)
    return set_error(ALCOP_ERR_CONFIG, "SmemCapacity", "window / filter rings exceed shared memory");
  return ALCOP_OK;
}

int launch_conv2d_stem_pairs(const alcop_conv_desc& d, const alcop_schedule& s, const void* x, const void* wt,
                             void* y, void* stream) {
  const int mode = stem_mode(d);
  if (mode == 0 && !stem_pairs_applicable(d))
    return set_error(ALCOP_ERR_CONFIG, "Unsupported",
                     "C = 4 convs run on the stem kernel: stride_w 2, W % 16 == 0, K % 16 == 0, K <= 256, "
                     "K * out bytes % 128 == 0, no halo layout");
  if (mode < 0)
    return set_error(ALCOP_ERR_CONFIG, "Unsupported", "not a window-conv shape (C % 64, stride 1, small filter)");
  int rc = validate_stem_pairs(d, s);
  if (rc) return rc;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(wt) | reinterpret_cast<uintptr_t>(y)) & 15)
    return set_error(ALCOP_ERR_CONFIG, "Alignment", "x, w and y must be 16-byte aligned");
  const StemGeometry g = stem_pairs_geometry(d);
  if (g.P < 1 || g.Q < 1) return set_error(ALCOP_ERR_CONFIG, "BadWorkload", "empty output");
  const CUtensorMapDataType dt =
      d.in_dtype == ALCOP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const CUtensorMapDataType odt = d.out_dtype == ALCOP_F32    ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                  : d.out_dtype == ALCOP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                              : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const int ob = out_bytes(d);
  CUtensorMap tx, ty;
  const cuuint32_t one[4] = {1, 1, 1, 1};
  if (mode == 0 || mode == 3) {
    // x viewed as {64 elements = 8 pixel pairs (128 B), W/16 blocks, H, N}; box
    // = NB blocks of R consecutive rows: the tile's whole input window, zero
    // filled above/below the image and left/right of it (pairs never straddle
    // the border: W is even, pad columns come in whole out-of-range pairs)
    const cuuint64_t xdims[4] = {64, static_cast<cuuint64_t>(d.W / 16), static_cast<cuuint64_t>(d.H),
                                 static_cast<cuuint64_t>(d.N)};
    const cuuint64_t xstr[3] = {128, static_cast<cuuint64_t>(d.W * 8), static_cast<cuuint64_t>(d.H * d.W * 8)};
    const cuuint32_t xbox[4] = {64, static_cast<cuuint32_t>(g.NB), g.box_bytes / g.row_bytes, 1};
    rc = encode_tiled_map(&tx, dt, x, 4, xdims, xstr, xbox, one, CU_TENSOR_MAP_SWIZZLE_NONE, "x (stem pairs)");
  } else {
    // x as {C channels, W, H, N}; box = 64 channels x WP pixels (from
    // -pad_w) x TR+R-1 rows: the tile's input window of one channel block,
    // zero filled outside the image
    const cuuint64_t xdims[4] = {static_cast<cuuint64_t>(d.C), static_cast<cuuint64_t>(d.W),
                                 static_cast<cuuint64_t>(d.H), static_cast<cuuint64_t>(d.N)};
    const cuuint64_t xstr[3] = {static_cast<cuuint64_t>(d.C * 2), static_cast<cuuint64_t>(d.W * d.C * 2),
                                static_cast<cuuint64_t>(d.H * d.W * d.C * 2)};
    const cuuint32_t xbox[4] = {64, static_cast<cuuint32_t>(g.WP), static_cast<cuuint32_t>(g.TR + d.R - 1), 1};
    rc = encode_tiled_map(&tx, dt, x, 4, xdims, xstr, xbox, one, CU_TENSOR_MAP_SWIZZLE_128B, "x (window)");
  }
  if (rc) return rc;
  // streamed filter: w viewed as [K rows, R*S*C columns]; box = 64 channels of
  // one tap x all K filters (128B-swizzled, K-major B)
  // (a CTA pair: each CTA's box is its K / 2 filters)
  const bool pair = s.cta_group == 2;
  const int64_t bn_cta = filter_rows_cta(d, s);
  CUtensorMap tw = tx;
  if (mode == 2) {
    const cuuint64_t wdims[3] = {static_cast<cuuint64_t>(d.R * d.S * d.C), static_cast<cuuint64_t>(d.K), 1};
    const cuuint64_t wstr[2] = {static_cast<cuuint64_t>(d.R * d.S * d.C * 2),
                                static_cast<cuuint64_t>(d.K * d.R * d.S * d.C * 2)};
    const cuuint32_t wbox[3] = {64, static_cast<cuuint32_t>(bn_cta), 1};
    rc = encode_tiled_map(&tw, dt, wt, 3, wdims, wstr, wbox, one, CU_TENSOR_MAP_SWIZZLE_128B, "w (window)");
    if (rc) return rc;
  }
  // y as {K, Q, P, N}: each epilogue warp stores its 32 tile rows x 128 B
  // (window mode, WP = 16: two output rows of 16 columns)
  const int64_t wcols = (mode == 0 || mode == 3) ? 32 : std::min<int64_t>(32, g.WP);
  const cuuint64_t ydims[4] = {static_cast<cuuint64_t>(d.K), static_cast<cuuint64_t>(g.Q),
                               static_cast<cuuint64_t>(g.P), static_cast<cuuint64_t>(d.N)};
  const cuuint64_t ystr[3] = {static_cast<cuuint64_t>(d.K * ob), static_cast<cuuint64_t>(g.Q * d.K * ob),
                              static_cast<cuuint64_t>(g.P * g.Q * d.K * ob)};
  const cuuint32_t ybox[4] = {static_cast<cuuint32_t>(128 / ob), static_cast<cuuint32_t>(wcols),
                              static_cast<cuuint32_t>(32 / wcols), 1};
  rc = encode_tiled_map(&ty, odt, y, 4, ydims, ystr, ybox, one, CU_TENSOR_MAP_SWIZZLE_128B, "y (stem)");
  if (rc) return rc;

  StemKParams kp{};
  kp.Pout = static_cast<int32_t>(g.P);
  kp.P = static_cast<int32_t>(mode == 0 ? g.P : (g.P + g.TR - 1) / g.TR);  // tile rows per image
  if (pair) kp.P = (kp.P + 1) / 2;  // pair tiles: tile rows 2u (leader) and 2u + 1 (peer)
  kp.Q = static_cast<int32_t>(g.Q);
  kp.QB = static_cast<int32_t>(g.QB);
  const int64_t tiles = d.N * static_cast<int64_t>(kp.P) * g.QB;
  if (tiles > (int64_t(1) << 31) - 1) return set_error(ALCOP_ERR_CONFIG, "BadWorkload", "too many output tiles");
  kp.num_tiles = static_cast<int32_t>(tiles);
  kp.R = static_cast<int32_t>(d.R);
  kp.S = static_cast<int32_t>(d.S);
  kp.T2 = g.T2;
  kp.o_min = g.o_min;
  kp.row_step = mode == 0 ? d.stride_h : mode == 3 ? 4 * d.stride_h : g.TR;  // input rows per tile row
  kp.ph = d.pad_h;
  kp.pw = d.pad_w;
  kp.BN = static_cast<int32_t>(d.K);
  kp.stages = s.n_stage_smem_A;
  kp.nacc = s.n_stage_inner;
  kp.row_bytes = g.row_bytes;
  kp.slot_bytes = g.slot_bytes;
  kp.box_bytes = g.box_bytes;
  kp.wbytes = static_cast<uint32_t>(resident_filter_bytes(d, s, g));
  kp.bn_cta = static_cast<int32_t>(bn_cta);
  kp.acc_stride = static_cast<uint32_t>(round_up_pow2_cols((mode == 3 ? 4 : 1) * d.K));
  kp.tmem_cols = static_cast<uint32_t>(round_up_pow2_cols(kp.acc_stride * kp.nacc));
  kp.idesc = ptx::make_idesc_f16(d.in_dtype == ALCOP_BF16 ? 1u : 0u, 0u, kTileM * (pair ? 2u : 1u),
                                 static_cast<uint32_t>(d.K));
  kp.w = static_cast<const uint16_t*>(wt);
  kp.stage_bufs = stem_staging_bufs(d, s);
  int lwp = 0;
  while ((1 << lwp) < g.WP) ++lwp;
  kp.lwp = lwp;
#ifdef STEM_PROBE
  // measurement builds only (-DSTEM_PROBE, tools/stem_skip_probe.py): switch parts of the pipeline off
  static const int skip_env = [] {
    const char* e = std::getenv("ALCOP_STEM_SKIP");
    return e ? std::atoi(e) : 0;
  }();
  kp.skip = skip_env;
#else
  kp.skip = 0;
#endif
  kp.dual = stem_dual(d, s) ? 1 : 0;
  kp.stage_warps = kp.dual ? 8 : 4;
  if (mode == 2) {
    kp.CB = static_cast<int32_t>(d.C / 64);
    kp.TB = static_cast<int32_t>(s.tileK / 64);
    kp.nbc = static_cast<int32_t>(d.R * d.S / kp.TB);
    kp.sB = s.n_stage_smem_B;
    kp.b_slot_bytes = static_cast<uint32_t>(stream_b_slot_bytes(d, s));
  }
  const int sms = device_sm_count();
  if (sms <= 0) return set_error(ALCOP_ERR_CUDA, "CudaError", "no CUDA device");
  // work units (CTAs, or CTA pairs) walking the tiles
  int grid = (s.num_ctas > 0 ? s.num_ctas : sms) / (pair ? 2 : 1);
  if (grid < 1) grid = 1;
  if (grid > kp.num_tiles) grid = kp.num_tiles;
  kp.dn = grid / (kp.P * kp.QB);
  kp.dp = (grid - kp.dn * kp.P * kp.QB) / kp.QB;
  kp.dq = grid - kp.dn * kp.P * kp.QB - kp.dp * kp.QB;
  if (mode == 0 || mode == 3) {
    // column block qb reads pairs from 128*qb + o_min: block 16*qb + floor(o_min/8), `shift` pairs in
    kp.blk_off = g.o_min >= 0 ? g.o_min / 8 : -((7 - g.o_min) / 8);
    kp.shift = g.o_min - 8 * kp.blk_off;
  } else {
    kp.blk_off = -d.pad_w;  // the window's first pixel
    kp.shift = 0;
  }
  const int smem = static_cast<int>(stem_pairs_smem_bytes(d, s));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int ctas = grid * (pair ? 2 : 1);
  switch (d.out_dtype) {
    case ALCOP_F32: return launch_stem_typed<float>(tx, ty, tw, kp, mode, pair, ctas, smem, st);
    case ALCOP_BF16: return launch_stem_typed<__nv_bfloat16>(tx, ty, tw, kp, mode, pair, ctas, smem, st);
    default: return launch_stem_typed<__half>(tx, ty, tw, kp, mode, pair, ctas, smem, st);
  }
}

}  // namespace alcop
