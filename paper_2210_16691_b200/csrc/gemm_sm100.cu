// gemm_sm100.cu — the output of ALCOP's pipelining pass as an sm_100a kernel.
//
// Reference: the pass rewrites the lowered load-and-use nest
// (schedule.hpp:551-578) into the pipelined nest (pipeline_pass.hpp:753-764):
//   expand_buffers          (pipeline_pass.hpp:392-437) -> an s-slot smem ring per buffer
//   shift_and_wrap_indices  (pipeline_pass.hpp:482-552) -> producer loads chunk (v+s-1)%E
//                                                          into slot (v+s-1)%s, consumer slot v%s
//   inject_prologues        (pipeline_pass.hpp:627-682) -> s-1 chunk prologue
//   inject_sync             (pipeline_pass.hpp:689-748) -> four primitives + s-1 drains
// and the four primitives' semantics (interp.hpp:375-418) become mbarriers:
//   producer_acquire  = wait empty[slot]           (slot free: previous use released)
//   producer_commit   = arrive.expect_tx full[slot] + TMA bulk-tensor copies
//   consumer_wait     = wait full[slot]            (bytes landed -> visible)
//   consumer_release  = tcgen05.commit -> empty[slot] (arrives when the MMAs retire)
// The inner (shared->register) level of the paper is re-expressed for
// tcgen05: the "register load" of k-step u of chunk v is the smem descriptor
// (slot v%s, k-offset u) handed to tcgen05.mma, and the register double
// buffer becomes a ring of n_stage_inner TMEM accumulators rotating per
// output tile, so the epilogue of tile i overlaps the MMAs of tile i+1.
//
// Warp roles (192 threads): warp 0 = TMA producer (one lane), warp 1 = TMEM
// allocator + MMA issuer (one lane), warps 2-5 = epilogue (TMEM -> regs ->
// global).  Persistent: one CTA per SM walks tiles blockIdx.x + i*gridDim.x.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <mutex>
#include <string>
#include <type_traits>

#include "alcop_internal.h"
#include "sm100_ptx.cuh"

namespace alcop {

struct GemmKParams {
  int32_t M, N, K, batch;
  int32_t BN, BK;
  int32_t num_m, num_n, num_tiles;
  int32_t group_m;  // raster: tile rows per group (>= num_m: plain m-fastest order)
  int32_t E;  // chunks (k blocks) per output tile = pipelined loop extent
  int32_t sA, sB, tacc;
  int32_t mode;
  int32_t b_mn_major;
  uint32_t idesc;
  uint32_t a_stage_bytes, b_stage_bytes;
  uint32_t acc_stride;  // TMEM columns between accumulator buffers
  uint32_t tmem_cols;
  void* C;
  int64_t ldc, stride_c;
  alcop_event* trace;
  int32_t trace_cap;
  uint64_t* stamps;  // debug timeline: 8 globaltimer stamps per CTA (nullptr = off)
  // implicit-GEMM conv2d (kConv): output pixels m = (n, p, q) row-major,
  // reduction chunk = (r, s, channel block) matching the KRSC filter layout
  int32_t conv_P, conv_Q, conv_S, conv_Cb;  // Cb: 64-channel blocks (kConv 1) / 8-channel groups (2)
  int32_t conv_RS;                         // filter taps R*S
  int32_t conv_small_c;                    // 1: C % 64 != 0 (kConv 2); 2: stem (kConv 3)
  int32_t conv_Pb, conv_Qb;                // stem: 8-row x 16-column output blocks per image
  int32_t conv_stem5;                      // stem A map is the 5-D strided view (stored H % stride_h == 0)
  int32_t conv_sh, conv_sw, conv_ph, conv_pw;
  // atom-stacked view of A: one 4-D TMA box brings the BK/64 K atoms of a
  // chunk instead of one instruction per atom (A: BK = 128; B: B[K,N] on one CTA, BN >= 128)
  int32_t a_view, b_view;
  // CTA pair, B[K,N] with BN/2 % 64 != 0 (BN 192: halves of 96 columns): load
  // each half as two 128B-swizzled 64-column atoms (over-fetching 32 columns
  // that the MMA never reads) instead of three 64B-swizzled 32-column atoms
  int32_t b_pad;
  int32_t stage_bufs;  // epilogue staging buffers per warp (1 or 2), gemm_staging_bufs
  int32_t epi_warps;   // 4 or 8 (gemm_epi_warps)
  int32_t in_bf16;  // fused pre-op arithmetic type
  int32_t pre_op;   // 1: A -> 2A+1 before the MMA (the reference's inlined "ew")
  int32_t* sk_flags;  // stream-K: per writer cluster, partial published (8 arrivals) / consumed
};

// debug timeline buffer (set through alcop_debug_set_stamps)
static uint64_t* g_stamps = nullptr;
// programmatic dependent launch on (alcop_debug_set_pdl; env ALCOP_PDL=0 turns it off)
static bool g_pdl = [] {
  const char* e = std::getenv("ALCOP_PDL");
  return !(e && e[0] == '0');
}();

namespace {

constexpr int kThreads = 192;      // producer, MMA, 4 epilogue warps
constexpr int kThreadsEpi8 = 320;  // producer, MMA, 8 epilogue warps (short-K tiles, see kEpi)
constexpr int kThreadsSplit = 224; // + warp 6: the B producer (conv, FUSED joint ring)
constexpr int kThreadsPair = 224;  // the CTA pair: producer A, MMA, 4 epilogue warps, producer B
constexpr int kThreadsPreOp = 192 + 128;  // 4 transform warps (6-9) for the fused pre-op, one producer
constexpr int kStagingBytesPerWarp = 32 * 128;  // one staging buffer: 32 rows x 128 B

struct TileCoord {
  int b, mb, nb;
};

__device__ __forceinline__ TileCoord tile_coord(const GemmKParams& p, int tile_id) {
  TileCoord t;
  int per_batch = p.num_m * p.num_n;
  t.b = tile_id / per_batch;
  int r = tile_id - t.b * per_batch;
  // grouped raster: m fastest inside a group of group_m tile rows, groups in
  // order, so the tiles in flight at once share few A rows and B columns
  // (their panels stay L2-resident instead of streaming A once per wave)
  const int span = p.group_m * p.num_n;
  const int g = r / span;
  const int first = g * p.group_m;
  const int gs = min(p.group_m, p.num_m - first);
  const int w = r - g * span;
  t.nb = w / gs;
  t.mb = first + (w - t.nb * gs);
  return t;
}

// Role-thread layout of the producer and MMA warps: the whole warp runs the
// loop warp-uniformly (everything stays on the uniform datapath) and one
// elected lane issues (ALCOP_WARP_ROLES=1, default, measured faster), or a
// single elected thread runs it (ALCOP_WARP_ROLES=0).
#ifndef ALCOP_WARP_ROLES
#define ALCOP_WARP_ROLES 1
#endif
#if ALCOP_WARP_ROLES
#define ROLE_GUARD() true
#define ISSUE(...)                 \
  do {                             \
    if (ptx::elect_one()) {        \
      __VA_ARGS__;                 \
    }                              \
    __syncwarp();                  \
  } while (0)
#else
#define ROLE_GUARD() ptx::elect_one()
#define ISSUE(...) \
  do {             \
    __VA_ARGS__;   \
  } while (0)
#endif

template <bool kDebug>
__device__ __forceinline__ void stamp(const GemmKParams& p, int i) {
  if constexpr (kDebug) {
    if (p.stamps == nullptr) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.stamps[blockIdx.x * 8 + i] = t;
    // CTA 0: SM clock beside the globaltimer at start / end (effective SM MHz under load)
    if (blockIdx.x == 0 && (i == 0 || i == 7)) p.stamps[148 * 8 + 192 + (i == 7)] = clock64();
  }
}

// epilogue clock64 log of CTA 0, warp 2 (debug): [chunk][event]
template <bool kDebug>
__device__ __forceinline__ void epistamp(const GemmKParams& p, int warp, int lane, int c, int ev) {
  if constexpr (kDebug) {
    if (p.stamps == nullptr || blockIdx.x != 0 || warp != 2 || lane != 0 || c >= 16) return;
    p.stamps[148 * 8 + c * 4 + ev] = clock64();
  }
}

// per-chunk clock64 log of CTA 0 (debug): role 0 = producer after
// producer_acquire, 1 = MMA after consumer_wait; chunks 0..63 of the stream
template <bool kDebug>
__device__ __forceinline__ void chunkstamp(const GemmKParams& p, int role, int i) {
  if constexpr (kDebug) {
    if (p.stamps == nullptr || blockIdx.x != 0 || i >= 64) return;
    p.stamps[148 * 8 + 64 + role * 64 + i] = clock64();
  }
}

template <bool kDebug>
__device__ __forceinline__ void log_event(const GemmKParams& p, int role, int& n, int kind, int buf, int tile,
                                          int slot, int chunk, int parity, int c0, int c1, int c2, int c3) {
  if constexpr (kDebug) {
    if (p.trace == nullptr) return;
    if (n < p.trace_cap) {
      alcop_event* e = p.trace + (static_cast<int64_t>(blockIdx.x) * 2 + role) * p.trace_cap + n;
      e->kind = kind;
      e->buf = buf;
      e->tile = tile;
      e->slot = slot;
      e->chunk = chunk;
      e->parity = parity;
      e->acquired = c0;
      e->committed = c1;
      e->waited = c2;
      e->released = c3;
    }
    ++n;
  }
}

// f(x) = 2x + 1 on a packed pair of f16 / bf16 values (RNE back to the input type)
__device__ __forceinline__ uint32_t pre_op_pair(uint32_t v, int bf16) {
  if (bf16) {
    __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&v);
    float2 f = __bfloat1622float2(h);
    __nv_bfloat162 r = __floats2bfloat162_rn(fmaf(2.f, f.x, 1.f), fmaf(2.f, f.y, 1.f));
    return *reinterpret_cast<uint32_t*>(&r);
  }
  __half2 h = *reinterpret_cast<__half2*>(&v);
  float2 f = __half22float2(h);
  __half2 r = __floats2half2_rn(fmaf(2.f, f.x, 1.f), fmaf(2.f, f.y, 1.f));
  return *reinterpret_cast<uint32_t*>(&r);
}

template <typename OutT>
__device__ __forceinline__ uint32_t pack2(uint32_t a, uint32_t b);
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(uint32_t a, uint32_t b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(a), __uint_as_float(b));
  return *reinterpret_cast<uint32_t*>(&h);
}
template <>
__device__ __forceinline__ uint32_t pack2<__half>(uint32_t a, uint32_t b) {
  __half2 h = __floats2half2_rn(__uint_as_float(a), __uint_as_float(b));
  return *reinterpret_cast<uint32_t*>(&h);
}

// One shared-memory ring of the pipeline (one pipeline group of the
// reference, interp.hpp:87-94): slot cursor, per-slot phase bits and the
// group counters.  Producer and consumer each keep their own copy.
struct RingCursor {
  uint32_t phase = 0;  // bit k = current phase parity of slot k
  int slot = 0;
  int count = 0;  // acquired/committed (producer) or waited (consumer)
  int released = 0;
  __device__ __forceinline__ void advance(int s) { slot = (slot + 1 == s) ? 0 : slot + 1; }
};

// ---------------------------------------------------------------------------
// The kernel.  kJoint: both buffers carry the same n_stage, so one mbarrier
// pair per slot guards the A and B copies of a chunk together (two groups
// with identical counters — the reference's own emission when the hints are
// equal); otherwise each buffer has its own ring and lookahead.  kDebug
// compiles in the bookkeeping trace and the timeline stamps.
// ---------------------------------------------------------------------------
// kConv: 0 GEMM / BMM; 1 implicit-GEMM conv, C % 64 == 0 (one 128B-swizzled
// im2col box per chunk); 2 small-channel conv, C % 8 == 0 (eight 16-byte-wide
// im2col boxes per chunk, one per 8-channel group of a filter tap, in the
// no-swizzle K-major core-matrix layout; ResNet-50 conv1 with C padded 3 -> 8);
// 3 stem conv on a halo-padded input with S*C <= 64: one chunk = one filter
// row, whose S taps x C channels are S*C contiguous elements of the input
// row, so a tiled TMA box over an overlapping (pixel-stride) view of x loads
// the whole 128 x 64 A chunk in one 128B-swizzled copy; output tiles are
// 8 x 16 output-pixel blocks
// kEpi: epilogue warps.  8 for tiles whose main loop is one or two chunks
// (attention QK^T: K = 64), where draining the accumulator, not loading or
// multiplying, sets the per-tile time; two warps then share each TMEM lane
// quarter, taking alternate column chunks.
template <typename OutT, int BK, bool kJoint, bool kDebug, int kConv = 0, bool kPreOp = false, int kEpi = 4>
__global__ void __launch_bounds__(kPreOp ? kThreadsPreOp
                                         : (kEpi == 8 ? kThreadsEpi8
                                                      : (kJoint && !kDebug && kConv != 0 ? kThreadsSplit : kThreads)),
                                  1)
    alcop_pipelined_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                                const __grid_constant__ CUtensorMap tmC, const GemmKParams p) {
  using namespace ptx;
  constexpr int kSteps = BK / 16;             // tcgen05 k-steps per chunk (the inner loop, F)
  constexpr int kBoxK = BK >= 64 ? 64 : BK;   // K extent of one K-major swizzle atom
  constexpr int kKAtoms = BK / kBoxK;
  constexpr uint32_t kKSbo = BK >= 64 ? 1024u : 512u;  // 8 rows x swizzle width
  constexpr uint32_t kKLayout = BK >= 64 ? kLayoutSW128 : kLayoutSW64;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the 128B swizzle atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t ringA = smem_u32(smem);
  const uint32_t ringB = ringA + p.sA * p.a_stage_bytes;
  // epilogue staging: 4 warps x 2 buffers x (32 rows x 128 B), 128B-swizzled for the TMA store
  const uint32_t staging = ringB + p.sB * p.b_stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.sA * p.a_stage_bytes + p.sB * p.b_stage_bytes +
                                               kEpi * kStagingBytesPerWarp * p.stage_bufs);
  uint64_t* fullA = bars;
  uint64_t* emptyA = fullA + p.sA;
  uint64_t* fullB = kJoint ? fullA : emptyA + p.sA;
  uint64_t* emptyB = kJoint ? emptyA : fullB + p.sB;
  uint64_t* tfull = bars + 2 * p.sA + 2 * p.sB;
  uint64_t* tempty = tfull + 2;
  // fused pre-op: transform warps turn full[slot] (raw A landed) into ready[slot] (f(A) in place)
  uint64_t* ready = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ready + (kPreOp ? p.sA : 0));

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) stamp<kDebug>(p, 0);
  if (warp == 0 && elect_one()) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    prefetch_tmap(&tmC);
  }
  if (warp == 1) {
    if (elect_one()) {
      for (int i = 0; i < p.sA; ++i) {
        mbar_init(smem_u32(&fullA[i]), 1);
        mbar_init(smem_u32(&emptyA[i]), 1);
      }
      if (!kJoint) {
        for (int i = 0; i < p.sB; ++i) {
          mbar_init(smem_u32(&fullB[i]), 1);
          mbar_init(smem_u32(&emptyB[i]), 1);
        }
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(smem_u32(&tfull[i]), 1);
        mbar_init(smem_u32(&tempty[i]), kEpi);
      }
      if (kPreOp)
        for (int i = 0; i < p.sA; ++i) mbar_init(smem_u32(&ready[i]), 4);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(smem_u32(tmem_slot), p.tmem_cols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: the setup above overlapped the previous kernel's tail; from here on
  // global memory is touched, so wait for it, and let the next kernel start
  // its own setup as soon as SMs free up.
  grid_dependency_wait();
  grid_launch_dependents();
  if (threadIdx.x == 0) stamp<kDebug>(p, 1);

  const int grid = gridDim.x;
  const int my_tiles = (p.num_tiles - static_cast<int>(blockIdx.x) + grid - 1) / grid;
  const int E = p.E;
  const bool wrap = (p.mode == ALCOP_MODE_WRAP);
  // Split producer (FUSED, joint ring): a TMA issue costs the issuing thread
  // ~80 clk and a chunk is 2-5 of them, which bounded the per-chunk time near
  // or above the MMA time; warp 0 commits the chunk (arrive.expect_tx of all
  // its bytes) and loads A, warp 6 waits on the same empty barrier and loads B
  // into the same full barrier (B bytes may land before the expect_tx: the
  // phase still needs warp 0's arrival).  WRAP / debug / pre-op / split rings
  // keep one producer (the device trace logs both buffers from one thread).
  // Measured: +4-11 % on the implicit-GEMM conv layers and the CTA pairs with
  // 64-wide chunks, -1.5 % on the single-CTA GEMMs of the BERT step, so the
  // single-CTA GEMM keeps one producer.
  constexpr bool kSplit = kJoint && !kDebug && !kPreOp && kConv != 0;

  if (warp == 0 || (kSplit && warp == 6)) {
    if (ROLE_GUARD()) {
      // ======================= producer(s) (TMA) =======================
      RingCursor ra, rb;
      int nev = 0;
      TileCoord tc{0, 0, 0};
      int tc_tile = -1;
      const uint32_t a_bytes = p.a_stage_bytes, b_bytes = p.b_stage_bytes;
      auto coord = [&](int tl) {
        if (tl != tc_tile) {
          tc_tile = tl;
          tc = tile_coord(p, static_cast<int>(blockIdx.x) + tl * grid);
        }
      };
      // conv: origin of the tile's first output pixel in input coordinates
      int cv_n = 0, cv_h = 0, cv_w = 0, cv_tile = -1;
      auto issue_a = [&](uint32_t slot, uint32_t fb, int chunk) {
        if constexpr (kConv) {
          if (tc_tile != cv_tile) {
            cv_tile = tc_tile;
            const int m0 = tc.mb * kTileM;
            const int pq = p.conv_P * p.conv_Q;
            cv_n = m0 / pq;
            const int rem = m0 - cv_n * pq;
            const int pp = rem / p.conv_Q;
            cv_h = pp * p.conv_sh - p.conv_ph;
            cv_w = (rem - pp * p.conv_Q) * p.conv_sw - p.conv_pw;
          }
          if constexpr (kConv == 3) {
            // tile = 8 output rows x 16 output columns of image n; chunk = filter row
            const int per_img = p.conv_Pb * p.conv_Qb;
            const int n = tc.mb / per_img;
            const int rem = tc.mb - n * per_img;
            const int pb = rem / p.conv_Qb;
            const int qb = rem - pb * p.conv_Qb;
            if (p.conv_stem5)  // {taps, q (stride sw px), p (stride sh rows), row parity, n}: no traversal strides
              tma_load_5d(ringA + slot * a_bytes, &tmA, fb, 0, qb * 16, pb * 8 + chunk / p.conv_sh,
                          chunk % p.conv_sh, n);
            else
              tma_load_4d(ringA + slot * a_bytes, &tmA, fb, 0, qb * 16 * p.conv_sw, pb * 8 * p.conv_sh + chunk, n);
          } else if constexpr (kConv == 2) {
            // K-group G = 8 channels of one filter tap; taps past R*S re-read
            // tap 0 (their filter rows are zero-filled by the w map)
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              const int G = chunk * 8 + g;
              int tap = G / p.conv_Cb;
              const int cgrp = G - tap * p.conv_Cb;
              if (tap >= p.conv_RS) tap = 0;
              const int fs = tap % p.conv_S;
              const int fr = tap / p.conv_S;
              tma_load_im2col_4d(ringA + slot * a_bytes + g * (kTileM * 16), &tmA, fb, cgrp * 8, cv_w, cv_h, cv_n,
                                 static_cast<uint16_t>(fs), static_cast<uint16_t>(fr));
            }
          } else {
            const int cb = chunk % p.conv_Cb;
            const int rs = chunk / p.conv_Cb;
            const int fs = rs % p.conv_S;
            const int fr = rs / p.conv_S;
            tma_load_im2col_4d(ringA + slot * a_bytes, &tmA, fb, cb * 64, cv_w, cv_h, cv_n,
                               static_cast<uint16_t>(fs), static_cast<uint16_t>(fr));
          }
        } else if (kKAtoms > 1 && p.a_view) {
          tma_load_4d(ringA + slot * a_bytes, &tmA, fb, 0, tc.mb * kTileM, chunk * kKAtoms, tc.b);
        } else {
#pragma unroll
          for (int a = 0; a < kKAtoms; ++a)
            tma_load_3d(ringA + slot * a_bytes + a * (kTileM * 128), &tmA, fb, chunk * BK + a * kBoxK,
                        tc.mb * kTileM, tc.b);
        }
      };
      auto issue_b = [&](uint32_t slot, uint32_t fb, int chunk) {
        const uint32_t dst = ringB + slot * b_bytes;
        if (kConv == 3) {
          tma_load_3d(dst, &tmB, fb, 0, chunk, tc.nb * p.BN);  // filter row `chunk`: S*C taps, zero-filled to 64
        } else if (p.b_mn_major) {
          // B[K,N] row-major: BN/64 atoms of (BK rows x 128 B), box {64 N, BK K}; with the atom-stacked
          // view {64, K, N/64} one box of BN/64 atoms
          if (p.b_view)
            tma_load_4d(dst, &tmB, fb, 0, chunk * BK, tc.nb * (p.BN >> 6), tc.b);
          else
            for (int a = 0; a < (p.BN >> 6); ++a)
              tma_load_3d(dst + a * (BK * 128), &tmB, fb, tc.nb * p.BN + a * 64, chunk * BK, tc.b);
        } else {
          // B[N,K] row-major: K-major like A with BN rows
#pragma unroll
          for (int a = 0; a < kKAtoms; ++a)
            tma_load_3d(dst + a * (p.BN * 128), &tmB, fb, chunk * BK + a * kBoxK, tc.nb * p.BN, tc.b);
        }
      };
      // producer_acquire + producer_commit of one buffer's chunk
      auto load = [&](RingCursor& r, int s, uint64_t* full, uint64_t* empty, int buf, int tl, int chunk) {
        const uint32_t slot = r.slot;
        const uint32_t par = ((r.phase >> slot) & 1u) ^ 1u;
        mbar_wait(smem_u32(&empty[slot]), par);  // producer_acquire
        r.phase ^= 1u << slot;
        ++r.count;
        coord(tl);
        const uint32_t fb = smem_u32(&full[slot]);
        ISSUE(if (buf == 0) {
          mbar_arrive_expect_tx(fb, a_bytes);  // producer_commit
          issue_a(slot, fb, chunk);
        } else {
          mbar_arrive_expect_tx(fb, b_bytes);
          issue_b(slot, fb, chunk);
        } log_event<kDebug>(p, 0, nev, 0, buf, tl, slot, chunk, par, r.count, r.count, -1, -1));
        r.advance(s);
      };
      // joint ring: both buffers' copies of a chunk under one barrier pair
      // kRole: 0 = commit + A, 1 = B, 2 = both (single producer)
#ifdef GEMM_TRACE
      // measurement build only (-DGEMM_TRACE): CTA 0's producer, clock64 after each
      // acquire and after each chunk's TMA issue
      unsigned long long ptr_[64];
      int ptn_ = 0;
#endif
      auto load_joint = [&](int tl, int chunk, auto role) {
        constexpr int kRole = decltype(role)::value;
        const uint32_t slot = ra.slot;
        const uint32_t par = ((ra.phase >> slot) & 1u) ^ 1u;
        mbar_wait(smem_u32(&emptyA[slot]), par);
#ifdef GEMM_TRACE
        if (blockIdx.x == 0 && warp == 0 && ptn_ < 64) ptr_[ptn_++] = clock64();
#endif
        ra.phase ^= 1u << slot;
        if (lane == 0) chunkstamp<kDebug>(p, 0, ra.count);
        ++ra.count;
        coord(tl);
        const uint32_t fb = smem_u32(&fullA[slot]);
        ISSUE(if constexpr (kRole != 1) {
          mbar_arrive_expect_tx(fb, a_bytes + b_bytes);
          issue_a(slot, fb, chunk);
        } if constexpr (kRole != 0) issue_b(slot, fb, chunk);
              log_event<kDebug>(p, 0, nev, 0, 0, tl, slot, chunk, par, ra.count, ra.count, -1, -1);
              log_event<kDebug>(p, 0, nev, 0, 1, tl, slot, chunk, par, ra.count, ra.count, -1, -1));
#ifdef GEMM_TRACE
        if (blockIdx.x == 0 && warp == 0 && ptn_ < 64) ptr_[ptn_++] = clock64() | (1ull << 62);
#endif
        ra.advance(p.sA);
      };

      if (wrap && warp != 0) {
        // WRAP keeps one producer (warp 0)
      } else if (wrap) {
        // reference-faithful: per tile, prologue chunks 0..s-2 into slots 0..s-2
        // (pipeline_pass.hpp:647-656), then steady loads of chunk (v+s-1)%E
        // (pipeline_pass.hpp:501-509); the s-1 tail loads wrap to chunks 0..
        for (int tl = 0; tl < my_tiles; ++tl) {
          ra.slot = 0;
          rb.slot = 0;
          if constexpr (kJoint) {
            int c = 0;
            for (int i = 0; i < E + p.sA - 1; ++i) {
              load_joint(tl, c, std::integral_constant<int, 2>{});
              c = (c + 1 == E) ? 0 : c + 1;
            }
          } else {
            for (int i = 0; i < p.sA - 1; ++i) load(ra, p.sA, fullA, emptyA, 0, tl, i % E);
            for (int i = 0; i < p.sB - 1; ++i) load(rb, p.sB, fullB, emptyB, 1, tl, i % E);
            int ca = (p.sA - 1) % E, cb = (p.sB - 1) % E;
            for (int v = 0; v < E; ++v) {
              load(ra, p.sA, fullA, emptyA, 0, tl, ca);
              load(rb, p.sB, fullB, emptyB, 1, tl, cb);
              ca = (ca + 1 == E) ? 0 : ca + 1;
              cb = (cb + 1 == E) ? 0 : cb + 1;
            }
          }
        }
      } else {
        // fused: one lookahead window over the flattened (tile, chunk) stream;
        // issuing in order is enough, the empty barriers enforce the lookahead
        if constexpr (kSplit) {
          if (warp == 0) {
            for (int tl = 0; tl < my_tiles; ++tl)
              for (int c = 0; c < E; ++c) load_joint(tl, c, std::integral_constant<int, 0>{});
          } else {
            for (int tl = 0; tl < my_tiles; ++tl)
              for (int c = 0; c < E; ++c) load_joint(tl, c, std::integral_constant<int, 1>{});
          }
        } else if constexpr (kJoint) {
          for (int tl = 0; tl < my_tiles; ++tl)
            for (int c = 0; c < E; ++c) load_joint(tl, c, std::integral_constant<int, 2>{});
        } else {
          const int total = my_tiles * E;
          int ta = 0, ca = 0, tb = 0, cb = 0;  // (tile, chunk) of the next A / B load
          auto nextA = [&] { if (++ca == E) { ca = 0; ++ta; } };
          auto nextB = [&] { if (++cb == E) { cb = 0; ++tb; } };
          for (int i = 0; i < p.sA - 1 && i < total; ++i) { load(ra, p.sA, fullA, emptyA, 0, ta, ca); nextA(); }
          for (int i = 0; i < p.sB - 1 && i < total; ++i) { load(rb, p.sB, fullB, emptyB, 1, tb, cb); nextB(); }
          for (int v = 0; v < total; ++v) {
            if (v + p.sA - 1 < total) { load(ra, p.sA, fullA, emptyA, 0, ta, ca); nextA(); }
            if (v + p.sB - 1 < total) { load(rb, p.sB, fullB, emptyB, 1, tb, cb); nextB(); }
          }
        }
      }
      if (kDebug && ra.count == 1) stamp<kDebug>(p, 2);
#ifdef GEMM_TRACE
      if (blockIdx.x == 0 && warp == 0 && lane == 0)
        for (int i = 0; i < ptn_; ++i) printf("P %d %llu\n", i, ptr_[i]);
#endif
    }
    __syncwarp();
  } else if (warp == 1) {
    if (ROLE_GUARD()) {
      // ======================= MMA issuer =======================
      RingCursor ca, cb;
      int nev = 0;
      // descriptor bases (start address advances in 16-byte units in the low word)
      // small-channel conv A: no-swizzle core matrices (8 rows x 16 B), LBO =
      // next 8 K (one 128-row x 16 B box), SBO = next 8 rows
      const uint64_t adesc0 = kConv == 2 ? make_smem_desc(ringA, kTileM * 16, 128, kLayoutNone)
                                         : make_smem_desc(ringA, 16, kKSbo, kKLayout);
      uint64_t bdesc0;
      uint32_t b_big, b_small;  // B k-step advance: (u>>2)*b_big + (u&3)*b_small, in 16 B units
      if (p.b_mn_major) {
        bdesc0 = make_smem_desc(ringB, BK * 128, 1024, kLayoutSW128);
        b_small = 2048 / 16;
        b_big = 4 * b_small;
      } else {
        bdesc0 = make_smem_desc(ringB, 16, kKSbo, kKLayout);
        b_small = 2;
        b_big = static_cast<uint32_t>(p.BN) * 128 / 16;
      }
      const uint32_t a_stage16 = p.a_stage_bytes >> 4, b_stage16 = p.b_stage_bytes >> 4;
      const uint32_t idesc = p.idesc;
      // consumer_wait of one buffer
#ifdef GEMM_TRACE
      unsigned long long ctr_[64];
      int ctn_ = 0;
#endif
      auto cwait = [&](RingCursor& r, uint64_t* full, int buf, int tl, int chunk) -> uint32_t {
        const uint32_t slot = r.slot, par = (r.phase >> slot) & 1u;
        mbar_wait(smem_u32(&full[slot]), par);
#ifdef GEMM_TRACE
        if (blockIdx.x == 0 && ctn_ < 64) ctr_[ctn_++] = clock64();
#endif
        r.phase ^= 1u << slot;
        ++r.count;
        if constexpr (kDebug) ISSUE(log_event<kDebug>(p, 1, nev, 1, buf, tl, slot, chunk, par, -1, -1, r.count, r.released));
        return par;
      };
      for (int tl = 0; tl < my_tiles; ++tl) {
        const int acc = tl % p.tacc;
        const uint32_t acc_par = ((tl / p.tacc) & 1) ^ 1;
        mbar_wait(smem_u32(&tempty[acc]), acc_par);  // accumulator drained by the epilogue
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * p.acc_stride;
        if (wrap) {
          ca.slot = 0;
          cb.slot = 0;
        }
        for (int v = 0; v < E; ++v) {
          const uint32_t sa = ca.slot, sb = kJoint ? ca.slot : cb.slot;
          uint32_t pa, pb;
          if constexpr (kJoint) {
            pa = cwait(ca, kPreOp ? ready : fullA, 0, tl, v);  // consumer_wait A (+B: same barrier)
            if (lane == 0) chunkstamp<kDebug>(p, 1, ca.count - 1);
            pb = pa;
            ++cb.count;
            if constexpr (kDebug) ISSUE(log_event<kDebug>(p, 1, nev, 1, 1, tl, sb, v, pb, -1, -1, cb.count, cb.released));
          } else {
            pa = cwait(ca, fullA, 0, tl, v);  // consumer_wait A
            pb = cwait(cb, fullB, 1, tl, v);  // consumer_wait B
          }
          tc_fence_after();
          const uint64_t ad = adesc0 + sa * a_stage16;
          const uint64_t bd = bdesc0 + sb * b_stage16;
          ++ca.released;
          ++cb.released;
          ISSUE(
#pragma unroll
              for (int u = 0; u < kSteps; ++u) {
                // inner level: k-step u of chunk v reads slot v%s at k offset 16u
                const uint32_t a_off = kConv == 2 ? u * (2 * kTileM * 16 / 16)
                                       : BK >= 64 ? (u >> 2) * (kTileM * 128 / 16) + (u & 3) * 2 : u * 2;
                const uint32_t b_off = (u >> 2) * b_big + (u & 3) * b_small;
                umma_f16_ss(d_tmem, ad + a_off, bd + b_off, idesc, (v > 0 || u > 0) ? 1u : 0u);
              } umma_commit(smem_u32(&emptyA[sa]));  // consumer_release A
              if (!kJoint) umma_commit(smem_u32(&emptyB[sb]));   // consumer_release B
              log_event<kDebug>(p, 1, nev, 2, 0, tl, sa, v, pa, -1, -1, ca.count, ca.released);
              log_event<kDebug>(p, 1, nev, 2, 1, tl, sb, v, pb, -1, -1, cb.count, cb.released));
          ca.advance(p.sA);
          if (!kJoint) cb.advance(p.sB);
        }
        ISSUE(umma_commit(smem_u32(&tfull[acc])));  // accumulator ready
        if (tl == my_tiles - 1) stamp<kDebug>(p, 4);
        if (wrap) {
          // drains (pipeline_pass.hpp:739-742): consume the s-1 wrapped tail
          // groups of each buffer, A's then B's, without MMA.
          auto drain = [&](RingCursor& r, int s, uint64_t* full, uint64_t* empty, int buf) {
            for (int d = 0; d < s - 1; ++d) {
              const uint32_t slot = r.slot;
              const uint32_t par = cwait(r, full, buf, tl, (E + d) % E);
              ++r.released;
              ISSUE(mbar_arrive(smem_u32(&empty[slot]));
                    log_event<kDebug>(p, 1, nev, 2, buf, tl, slot, (E + d) % E, par, -1, -1, r.count, r.released));
              r.advance(s);
            }
          };
          if constexpr (kJoint) {
            for (int d = 0; d < p.sA - 1; ++d) {
              const uint32_t slot = ca.slot;
              const uint32_t par = cwait(ca, kPreOp ? ready : fullA, 0, tl, (E + d) % E);
              ++cb.count;
              ++ca.released;
              ++cb.released;
              ISSUE(log_event<kDebug>(p, 1, nev, 1, 1, tl, slot, (E + d) % E, par, -1, -1, cb.count, cb.released - 1);
                    mbar_arrive(smem_u32(&emptyA[slot]));
                    log_event<kDebug>(p, 1, nev, 2, 0, tl, slot, (E + d) % E, par, -1, -1, ca.count, ca.released);
                    log_event<kDebug>(p, 1, nev, 2, 1, tl, slot, (E + d) % E, par, -1, -1, cb.count, cb.released));
              ca.advance(p.sA);
            }
          } else {
            drain(ca, p.sA, fullA, emptyA, 0);
            drain(cb, p.sB, fullB, emptyB, 1);
          }
        }
      }
#ifdef GEMM_TRACE
      if (blockIdx.x == 0 && lane == 0)
        for (int i = 0; i < ctn_; ++i) printf("C %d %llu\n", i, ctr_[i]);
#endif
    }
    __syncwarp();
  } else if (kPreOp && warp >= 6) {
    // ======================= fused elementwise pre-op (warps 6-9) =======================
    // The reference's `inline S2` case 2 (schedule.hpp:275-314) turns the
    // consumer into mma_ewa: acc + f(a)*b with f(x) = 2x+1 (interp.hpp:367-369).
    // Here f is applied once per element, in place in the landed A slot,
    // between consumer_wait (full) and the MMA (ready): elementwise, so the
    // 128B swizzle of the slot does not matter.
    const int tw = warp - 6;
    RingCursor cr;
    const uint32_t quarter = p.a_stage_bytes / 4;
    for (int tl = 0; tl < my_tiles; ++tl) {
      if (wrap) cr.slot = 0;
      const int uses = E + (wrap ? p.sA - 1 : 0);
      for (int i = 0; i < uses; ++i) {
        const uint32_t slot = cr.slot, par = (cr.phase >> slot) & 1u;
        mbar_wait(smem_u32(&fullA[slot]), par);
        cr.phase ^= 1u << slot;
        if (i < E) {
          const uint32_t base = ringA + slot * p.a_stage_bytes + tw * quarter;
          for (uint32_t off = lane * 16; off < quarter; off += 32 * 16) {
            uint32_t v[4];
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                         : "r"(base + off));
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = pre_op_pair(v[j], p.in_bf16);
            st_shared_v4(base + off, v[0], v[1], v[2], v[3]);
          }
          fence_proxy_async_smem();  // generic-proxy writes -> visible to tcgen05 (async proxy)
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&ready[slot]));
        cr.advance(p.sA);
      }
    }
  } else if (warp < 2 + kEpi) {
    // ======================= epilogue (warps 2-5, or 2-9 with kEpi 8) =======================
    // TMEM -> registers (tcgen05.ld) -> 128B-swizzled smem staging -> TMA
    // bulk-tensor store; two staging buffers per warp so the store of one
    // chunk overlaps the TMEM read of the next.
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const uint32_t stage_base = staging + (warp - 2) * p.stage_bufs * 4096;
    constexpr int kChunkCols = 128 / static_cast<int>(sizeof(OutT));  // 128 B of output per row
    const int nchunks = p.BN / kChunkCols;
    int buf = 0;
    for (int tl = 0; tl < my_tiles; ++tl) {
      const int acc = tl % p.tacc;
      mbar_wait(smem_u32(&tfull[acc]), (tl / p.tacc) & 1);
      tc_fence_after();
      if (tl == 0 && warp == 2 && lane == 0) stamp<kDebug>(p, 5);
      const TileCoord tc = tile_coord(p, static_cast<int>(blockIdx.x) + tl * grid);
      const uint32_t t_addr = tmem_base + acc * p.acc_stride + (static_cast<uint32_t>(q * 32) << 16);
      constexpr int kStep = kEpi / 4;  // warps per TMEM lane quarter
      const int c0 = (warp - 2) / 4;   // this warp's first column chunk
      if (c0 >= nchunks) {             // no chunk for this warp in this tile: release at once
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&tempty[acc]));
      }
      for (int c = c0; c < nchunks; c += kStep) {
        uint32_t w[32];
        epistamp<kDebug>(p, warp, lane, c, 0);
        if constexpr (sizeof(OutT) == 4) {
          tmem_ld_32x32b_x32(t_addr + c * 32, w);
          tmem_wait_ld();
        } else {
          uint32_t r0[32], r1[32];
          tmem_ld_32x32b_x32(t_addr + c * 64, r0);
          tmem_ld_32x32b_x32(t_addr + c * 64 + 32, r1);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            w[i] = pack2<OutT>(r0[2 * i], r0[2 * i + 1]);
            w[16 + i] = pack2<OutT>(r1[2 * i], r1[2 * i + 1]);
          }
        }
        if (c + kStep >= nchunks) {
          // all this warp's TMEM reads of this accumulator done: hand it back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&tempty[acc]));
        }
        epistamp<kDebug>(p, warp, lane, c, 1);
        const uint32_t sbuf = stage_base + buf * 4096;
        if (lane == 0) {  // the store that last read sbuf is done
          if (p.stage_bufs == 2)
            bulk_wait_group_read<1>();
          else
            bulk_wait_group_read<0>();
        }
        __syncwarp();
        epistamp<kDebug>(p, warp, lane, c, 2);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          st_shared_v4(sbuf + lane * 128 + ((j ^ (lane & 7)) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2],
                       w[4 * j + 3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if constexpr (kConv == 3) {
            // warp quarter q holds output rows 2q, 2q+1 of the 8 x 16 pixel block
            const int per_img = p.conv_Pb * p.conv_Qb;
            const int n = tc.mb / per_img;
            const int rem = tc.mb - n * per_img;
            const int pb = rem / p.conv_Qb;
            tma_store_4d(&tmC, sbuf, tc.nb * p.BN + c * kChunkCols, (rem - pb * p.conv_Qb) * 16, pb * 8 + q * 2, n);
          } else {
            tma_store_3d(&tmC, sbuf, tc.nb * p.BN + c * kChunkCols, tc.mb * kTileM + q * 32, tc.b);
          }
          bulk_commit_group();
        }
        epistamp<kDebug>(p, warp, lane, c, 3);
        buf ^= p.stage_bufs - 1;
      }
    }
    if (lane == 0) bulk_wait_group_read<0>();  // smem reads done; grid completion publishes the writes
    __syncwarp();
    if (warp == 2 && lane == 0) stamp<kDebug>(p, 6);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
  if (threadIdx.x == 0) stamp<kDebug>(p, 7);
}

// ---------------------------------------------------------------------------
// cta_group::2 variant: a cluster of two CTAs on one TPC computes a
// 256 x BN output tile with tcgen05.mma.cta_group::2 (M = 256).  Each CTA
// stages its 128 rows of A and half (BN/2) of B's columns per chunk, so the
// per-SM TMA fill per FLOP drops by (128+BN)/(128+BN/2).  Both CTAs' copies
// complete on the leader's full barrier (leader arms it with both CTAs'
// bytes); the leader's single MMA thread consumes the chunk from both shared
// memories and its tcgen05.commit multicasts the release to both CTAs'
// empty barriers — the four primitives of the pass, now spanning a CTA pair.
// Each CTA's TMEM holds its 128 rows x BN columns; the epilogue is per CTA
// and hands the accumulator back on the leader's tmem_empty (8 arrivals).
// Joint A+B ring only (n_stage_A == n_stage_B).
// ---------------------------------------------------------------------------
// stream-K partial hand-off (release / acquire across clusters; the partial
// moves through the async proxy: TMA store by the writer, TMA load by the finisher)
__device__ __forceinline__ int sk_ld_acquire(const int32_t* f) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  return v;
}
__device__ __forceinline__ void sk_red_release_add(int32_t* f, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
__device__ __forceinline__ void sk_fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// kWide: tileN 512 (two N = 256 MMAs per k-step into one 512-column
// accumulator).  A template parameter, not a run-time flag: the per-MMA
// branch of a run-time flag cost the other pair tiles 12-18 % (tools/pair_ab.py).
// kConv: A is an implicit-GEMM conv operand (C % 64 == 0): each CTA's 128
// output pixels per chunk come as one TMA im2col box (one filter tap x 64
// channels), the pair's CTAs taking consecutive 128-pixel halves of the
// 256-pixel tile; B is the filter [K, R*S*C] (K-major).
template <typename OutT, int BK, bool kDebug, bool kSK, bool kWide = false, bool kConv = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsPair, 1)
    alcop_pipelined_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                                     const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmW,
                                     const GemmKParams p) {
  using namespace ptx;
  constexpr int kSteps = BK / 16;
  constexpr int kBoxK = BK >= 64 ? 64 : BK;
  constexpr int kKAtoms = BK / kBoxK;
  constexpr uint32_t kKSbo = BK >= 64 ? 1024u : 512u;
  constexpr uint32_t kKLayout = BK >= 64 ? kLayoutSW128 : kLayoutSW64;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t ringA = smem_u32(smem);
  const uint32_t ringB = ringA + p.sA * p.a_stage_bytes;
  const uint32_t staging = ringB + p.sA * p.b_stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.sA * (p.a_stage_bytes + p.b_stage_bytes) +
                                               4 * kStagingBytesPerWarp * p.stage_bufs);
  uint64_t* full = bars;
  uint64_t* empty = full + p.sA;
  uint64_t* tfull = empty + p.sA;
  uint64_t* tempty = tfull + 2;
  uint64_t* fixbar = tempty + 2;  // stream-K: one per epilogue warp (partial landed)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fixbar + 4);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int half_n = p.BN / 2;
  const bool b_sw64 = (half_n & 63) != 0 && !p.b_pad;  // BN = 192: N-major halves of 96 columns
  constexpr bool wide = kWide;  // one 256 x 512 tile = two N = 256 MMAs per k-step, one TMEM accumulator
  if (threadIdx.x == 0) stamp<kDebug>(p, 0);

  if (warp == 0 && elect_one()) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    prefetch_tmap(&tmC);
    if constexpr (kSK) prefetch_tmap(&tmW);
  }
  if (warp == 1) {
    if (elect_one()) {
      for (int i = 0; i < p.sA; ++i) {
        mbar_init(smem_u32(&full[i]), 1);
        mbar_init(smem_u32(&empty[i]), 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(smem_u32(&tfull[i]), 1);
        mbar_init(smem_u32(&tempty[i]), 8);  // 4 epilogue warps x 2 CTAs
      }
      if constexpr (kSK)
        for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&fixbar[i]), 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc_pair(smem_u32(tmem_slot), p.tmem_cols);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync();  // both CTAs' barriers initialised before any remote arrive / complete_tx
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  grid_dependency_wait();
  grid_launch_dependents();
  if (threadIdx.x == 0) stamp<kDebug>(p, 1);

  const int cluster_id = static_cast<int>(blockIdx.x) >> 1;
  const int nclusters = static_cast<int>(gridDim.x) >> 1;
  const int my_tiles = (p.num_tiles - cluster_id + nclusters - 1) / nclusters;
  const int E = p.E;
  const bool wrap = (p.mode == ALCOP_MODE_WRAP);
  // This cluster's work as segments (k-th segment: tile, chunks [cb, ce)).
  // Whole tiles: tiles cluster_id + k * nclusters.  Stream-K (FUSED only):
  // whole-tile waves as before except the last full wave plus the partial
  // one (R + n tiles, R = tiles mod n), whose chunk stream is split evenly,
  // cluster c taking chunks [c T / n, (c+1) T / n) of T = (R + n) x E —
  // neighbouring clusters stay on neighbouring tiles, so the L2 working set
  // is that of a whole-tile wave.  With >= E chunks per cluster a tile is cut
  // between at most two clusters: the later one (it reaches the cut first, at
  // the start of its range) writes an fp32 partial of the tile's last chunks,
  // the earlier one (at the end of its range) adds it.
  auto for_each_seg = [&](auto&& fn) {
    if constexpr (kSK) {
      const int dp_waves = p.num_tiles / nclusters - 1;
      int k = 0;
      for (; k < dp_waves; ++k) fn(k, cluster_id + k * nclusters, 0, E);
      const int t0 = dp_waves * nclusters;
      const int64_t T = static_cast<int64_t>(p.num_tiles - t0) * E;
      const int64_t e0 = T * (cluster_id + 1) / nclusters;
      int64_t g = T * cluster_id / nclusters;
      for (; g < e0; ++k) {
        const int t = static_cast<int>(g / E);
        const int cb = static_cast<int>(g - static_cast<int64_t>(t) * E);
        const int ce = static_cast<int>(min(static_cast<int64_t>(E), cb + (e0 - g)));
        fn(k, t0 + t, cb, ce);
        g += ce - cb;
      }
    } else {
      for (int k = 0; k < my_tiles; ++k) fn(k, cluster_id + k * nclusters, 0, E);
    }
  };

  if (warp == 0 || warp == 6) {
    if (ROLE_GUARD()) {
      // ======================= producers (both CTAs) =======================
      RingCursor ra;
      TileCoord tc{0, 0, 0};
      int tc_tile = -1;
      [[maybe_unused]] int cv_tile = -1, cv_n = 0, cv_h = 0, cv_w = 0;  // kConv: this CTA's window origin
      const uint32_t a_bytes = p.a_stage_bytes, b_bytes = p.b_stage_bytes;
      const uint32_t pair_bytes = 2 * (a_bytes + b_bytes);
      // Producer issue is split over two warps in FUSED mode: a TMA issue
      // costs the issuing thread ~80 clk and a chunk is 3-4 of them, which
      // bounded the per-chunk time above the 256x256 MMA time (~540 vs 512
      // clk, tools/timeline.py).  Warp 0 commits (arrive.expect_tx of all
      // the chunk's bytes on the leader's full barrier) and loads A; warp 6
      // waits on the same empty barrier and loads B, completing on the same
      // full barrier (its bytes may land before the expect_tx: the phase
      // still needs warp 0's arrival).  kRole: 0 = A + commit, 1 = B, 2 = both.
      auto load = [&](int tile, int chunk, auto role) {
        constexpr int kRole = decltype(role)::value;
        const uint32_t slot = ra.slot;
        const uint32_t par = ((ra.phase >> slot) & 1u) ^ 1u;
        mbar_wait(smem_u32(&empty[slot]), par);  // producer_acquire (own slot, released by the pair's MMA)
        ra.phase ^= 1u << slot;
        if (lane == 0 && warp == 0) chunkstamp<kDebug>(p, 0, ra.count++);
        if (tile != tc_tile) {
          tc_tile = tile;
          tc = tile_coord(p, tile);
        }
        const uint32_t fb_local = smem_u32(&full[slot]);
        const uint32_t fb_leader = mapa_shared(fb_local, 0);
        if constexpr (kConv) {
          if (kRole != 1 && tile != cv_tile) {  // window origin of this CTA's first output pixel
            cv_tile = tile;
            const int m0 = tc.mb * (2 * kTileM) + static_cast<int>(rank) * kTileM;
            const int pq = p.conv_P * p.conv_Q;
            cv_n = m0 / pq;
            const int rem = m0 - cv_n * pq;
            const int pp = rem / p.conv_Q;
            cv_h = pp * p.conv_sh - p.conv_ph;
            cv_w = (rem - pp * p.conv_Q) * p.conv_sw - p.conv_pw;
          }
        }
        ISSUE(if constexpr (kRole != 1) {
                if (leader) mbar_arrive_expect_tx(fb_local, pair_bytes);  // producer_commit (both CTAs' bytes)
                if constexpr (kConv) {
                  const int cb = chunk % p.conv_Cb;
                  const int rs = chunk / p.conv_Cb;
                  const int fs = rs % p.conv_S;
                  tma_load_im2col_4d_pair(ringA + slot * a_bytes, &tmA, fb_leader, cb * 64, cv_w, cv_h, cv_n,
                                          static_cast<uint16_t>(fs), static_cast<uint16_t>(rs / p.conv_S));
                } else if (kKAtoms > 1 && p.a_view) {
                  tma_load_4d_pair(ringA + slot * a_bytes, &tmA, fb_leader, 0,
                                   tc.mb * (2 * kTileM) + static_cast<int>(rank) * kTileM, chunk * kKAtoms, tc.b);
                } else {
#pragma unroll
                  for (int a = 0; a < kKAtoms; ++a) tma_load_3d_pair(
                      ringA + slot * a_bytes + a * (kTileM * 128), &tmA, fb_leader, chunk * BK + a * kBoxK,
                      tc.mb * (2 * kTileM) + static_cast<int>(rank) * kTileM, tc.b);
                }
              }
              const uint32_t dst = ringB + slot * b_bytes; [[maybe_unused]] const int n0 = tc.nb * p.BN + static_cast<int>(rank) * half_n;
              if (kRole == 0) {
              } else if constexpr (wide) {
                // tileN 512: two N = 256 MMAs per k-step; MMA g reads cluster
                // columns [256 g, 256 g + 256), 128 of them from each CTA, so
                // this CTA stages columns 256 g + 128 rank + [0, 128) for g = 0, 1
                const int nw = tc.nb * p.BN + static_cast<int>(rank) * 128;
                if (p.b_mn_major) {
                  for (int a = 0; a < 4; ++a)
                    tma_load_3d_pair(dst + a * (BK * 128), &tmB, fb_leader, nw + (a >> 1) * 256 + (a & 1) * 64,
                                     chunk * BK, tc.b);
                } else {
                  for (int a = 0; a < kKAtoms; ++a)
                    for (int g = 0; g < 2; ++g)
                      tma_load_3d_pair(dst + a * (256 * 128) + g * (128 * kBoxK * 2), &tmB, fb_leader,
                                       chunk * BK + a * kBoxK, nw + g * 256, tc.b);
                }
              } else if (p.b_mn_major && p.b_pad) {
                tma_load_3d_pair(dst, &tmB, fb_leader, n0, chunk * BK, tc.b);
                tma_load_3d_pair(dst + BK * 128, &tmB, fb_leader, n0 + 64, chunk * BK, tc.b);
              } else if (p.b_mn_major && b_sw64) {
                for (int a = 0; a < (half_n >> 5); ++a)  // 32-column SW64 atoms (half_n = 96)
                  tma_load_3d_pair(dst + a * (BK * 64), &tmB, fb_leader, n0 + a * 32, chunk * BK, tc.b);
              } else if (p.b_mn_major) {
                for (int a = 0; a < (half_n >> 6); ++a)
                  tma_load_3d_pair(dst + a * (BK * 128), &tmB, fb_leader, n0 + a * 64, chunk * BK, tc.b);
              } else {
#pragma unroll
                for (int a = 0; a < kKAtoms; ++a)
                  tma_load_3d_pair(dst + a * (half_n * 128), &tmB, fb_leader, chunk * BK + a * kBoxK, n0, tc.b);
              });
        ra.advance(p.sA);
      };
      if (wrap) {
        if (warp == 0) {
          for (int tl = 0; tl < my_tiles; ++tl) {
            ra.slot = 0;
            int c = 0;
            for (int i = 0; i < E + p.sA - 1; ++i) {
              load(cluster_id + tl * nclusters, c, std::integral_constant<int, 2>{});
              c = (c + 1 == E) ? 0 : c + 1;
            }
          }
        }
      } else if (warp == 0) {
        for_each_seg([&](int, int t, int cb, int ce) {
          for (int c = cb; c < ce; ++c) load(t, c, std::integral_constant<int, 0>{});
        });
      } else {
        for_each_seg([&](int, int t, int cb, int ce) {
          for (int c = cb; c < ce; ++c) load(t, c, std::integral_constant<int, 1>{});
        });
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader && ROLE_GUARD()) {
      // ======================= MMA issuer (leader CTA only) =======================
      RingCursor ca;
      const uint64_t adesc0 = make_smem_desc(ringA, 16, kKSbo, kKLayout);
      uint64_t bdesc0;
      uint32_t b_big, b_small;
      if (p.b_mn_major && b_sw64) {
        // N-major B in 32-column SW64 atoms: LBO = next atom along N, SBO =
        // next 8 K rows (512 B); one UMMA_K step = 16 K rows = 1024 B
        bdesc0 = make_smem_desc(ringB, BK * 64, 512, kLayoutSW64);
        b_small = 1024 / 16;
        b_big = 4 * b_small;
      } else if (p.b_mn_major) {
        bdesc0 = make_smem_desc(ringB, BK * 128, 1024, kLayoutSW128);
        b_small = 2048 / 16;
        b_big = 4 * b_small;
      } else {
        bdesc0 = make_smem_desc(ringB, 16, kKSbo, kKLayout);
        b_small = 2;
        b_big = static_cast<uint32_t>(half_n) * 128 / 16;
      }
      // tileN 512: the second MMA's 128 columns of this CTA's B (two 64-column
      // atoms further for N-major B, 128 rows of kBoxK elements further in each
      // K atom for K-major)
      const uint32_t b_group = !wide ? 0u : p.b_mn_major ? 2u * BK * 128u / 16u : 128u * kBoxK * 2u / 16u;
      const uint32_t a_stage16 = p.a_stage_bytes >> 4, b_stage16 = p.b_stage_bytes >> 4;
      const uint32_t idesc = p.idesc;
#ifdef GEMM_TRACE
      // measurement build only (-DGEMM_TRACE): CTA 0's MMA thread, clock64 per chunk
      // (after the full wait, after the chunk's MMAs + commit were issued)
      unsigned long long gtr[96];
      int gtn = 0, gchunk = 0;
#endif
      auto mma_seg = [&](int k, int cb, int ce) {
        const int acc = k % p.tacc;
#ifdef GEMM_TRACE
        if (blockIdx.x == 0 && gtn < 96) gtr[gtn++] = clock64() | (1ull << 62);  // tile start marker
#endif
        mbar_wait(smem_u32(&tempty[acc]), ((k / p.tacc) & 1) ^ 1);  // both CTAs drained it
#ifdef GEMM_TRACE
        if (blockIdx.x == 0 && gtn < 96) gtr[gtn++] = clock64() | (1ull << 61);  // accumulator free
#endif
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * p.acc_stride;
        if (wrap) ca.slot = 0;
        for (int v = cb; v < ce; ++v) {
          const uint32_t slot = ca.slot, par = (ca.phase >> slot) & 1u;
          mbar_wait(smem_u32(&full[slot]), par);  // consumer_wait: both CTAs' halves landed
#ifdef GEMM_TRACE
          if (blockIdx.x == 0 && gtn < 96) gtr[gtn++] = clock64();
#endif
          ca.phase ^= 1u << slot;
          if (lane == 0) chunkstamp<kDebug>(p, 1, ca.count++);
          tc_fence_after();
          if (k == 0 && v == cb && lane == 0) stamp<kDebug>(p, 3);
          const uint64_t ad = adesc0 + slot * a_stage16;
          const uint64_t bd = bdesc0 + slot * b_stage16;
          ISSUE(
#pragma unroll
              for (int u = 0; u < kSteps; ++u) {
                const uint32_t a_off = BK >= 64 ? (u >> 2) * (kTileM * 128 / 16) + (u & 3) * 2 : u * 2;
                const uint32_t b_off = (u >> 2) * b_big + (u & 3) * b_small;
                const uint32_t acc_flag = (v > cb || u > 0) ? 1u : 0u;
                umma_f16_ss_pair(d_tmem, ad + a_off, bd + b_off, idesc, acc_flag);
                if constexpr (wide) umma_f16_ss_pair(d_tmem + 256, ad + a_off, bd + b_group + b_off, idesc, acc_flag);
              } umma_commit_pair_multicast(smem_u32(&empty[slot]), 0x3));  // consumer_release in both CTAs
#ifdef GEMM_TRACE
          if (blockIdx.x == 0 && gtn < 96) gtr[gtn++] = clock64();
#endif
          ca.advance(p.sA);
        }
        ISSUE(umma_commit_pair_multicast(smem_u32(&tfull[acc]), 0x3));
        if (k == my_tiles - 1 && lane == 0) stamp<kDebug>(p, 4);
        if (wrap) {
          // drain the s-1 wrapped tail groups (no MMA): release both CTAs' slots
          for (int d = 0; d < p.sA - 1; ++d) {
            const uint32_t slot = ca.slot, par = (ca.phase >> slot) & 1u;
            mbar_wait(smem_u32(&full[slot]), par);
            ca.phase ^= 1u << slot;
            ISSUE(mbar_arrive(smem_u32(&empty[slot])); mbar_arrive_cluster(mapa_shared(smem_u32(&empty[slot]), 1)));
            ca.advance(p.sA);
          }
        }
      };
      for_each_seg([&](int k, int, int cb, int ce) { mma_seg(k, cb, ce); });
#ifdef GEMM_TRACE
      if (blockIdx.x == 0 && lane == 0)
        for (int i = 0; i < gtn; ++i) printf("T %d %llu\n", i, gtr[i]);
#endif
    }
    __syncwarp();
  } else if (warp < 6) {
    // ======================= epilogue (both CTAs) =======================
    const int q = warp & 3;
    const uint32_t stage_base = staging + (warp - 2) * p.stage_bufs * 4096;
    constexpr int kChunkCols = 128 / static_cast<int>(sizeof(OutT));
    const int nchunks = p.BN / kChunkCols;
    int buf = 0;
    const int row0 = static_cast<int>(rank) * kTileM + q * 32;  // this warp's rows of the cluster's 256
    for_each_seg([&](int k, int t, int cb, int ce) {
      const int acc = k % p.tacc;
      mbar_wait(smem_u32(&tfull[acc]), (k / p.tacc) & 1);
      tc_fence_after();
      if (k == 0 && warp == 2 && lane == 0) stamp<kDebug>(p, 5);
      const TileCoord tc = tile_coord(p, t);
      const uint32_t t_addr = tmem_base + acc * p.acc_stride + (static_cast<uint32_t>(q * 32) << 16);
      const bool writer = kSK && cb > 0;              // the tile's last chunks: fp32 partial out
      const bool finisher = kSK && cb == 0 && ce < E;  // the tile's first chunks: add the partial
      if (writer) {
        // fp32 partial (32-column chunks) into this cluster's workspace slot
        for (int c = 0; c < p.BN / 32; ++c) {
          uint32_t w[32];
          tmem_ld_32x32b_x32(t_addr + c * 32, w);
          tmem_wait_ld();
          if (c == p.BN / 32 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
          }
          const uint32_t sbuf = stage_base + buf * 4096;
          if (lane == 0) {
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
            tma_store_3d(&tmW, sbuf, c * 32, row0, cluster_id);
            bulk_commit_group();
          }
          buf ^= p.stage_bufs - 1;
        }
        // publish: the partial is in global memory before the release
        if (lane == 0) {
          bulk_wait_group<0>();
          sk_fence_proxy_async_global();
          sk_red_release_add(p.sk_flags + cluster_id, 1);
        }
        __syncwarp();
        return;
      }
      uint32_t part = 0;  // finisher: this warp's 32 rows of the partial, staged in the (idle) ring
      if (finisher) {
        part = ringA + static_cast<uint32_t>(q) * static_cast<uint32_t>(p.BN) * 128u;
        int32_t* flag = p.sk_flags + cluster_id + 1;
        if (lane == 0) {
          long long t0 = 0;
          while (sk_ld_acquire(flag) < 8) {  // 4 epilogue warps x 2 CTAs of the writer
            if (t0 == 0) t0 = clock64();
            if (clock64() - t0 > (1ll << 33)) asm volatile("trap;");  // watchdog, as mbar_wait
            __nanosleep(32);
          }
          sk_fence_proxy_async_global();
          mbar_arrive_expect_tx(smem_u32(&fixbar[q]), static_cast<uint32_t>(p.BN) * 128u);
          for (int b = 0; b < p.BN / 32; ++b)
            tma_load_3d(part + b * 4096, &tmW, smem_u32(&fixbar[q]), b * 32, row0, cluster_id + 1);
        }
        __syncwarp();
        mbar_wait(smem_u32(&fixbar[q]), 0);  // one finisher segment per cluster and launch
        if (lane == 0 && atomicAdd(flag, 1) == 15) atomicExch(flag, 0);  // the last reader re-arms the slot
        __syncwarp();
      }
      auto add_part = [&](uint32_t(&r)[32], int box) {
        if (!finisher) return;
        const uint32_t src = part + box * 4096 + lane * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint32_t x0, x1, x2, x3;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                       : "r"(src + ((j ^ (lane & 7)) << 4)));
          r[4 * j] = __float_as_uint(__uint_as_float(r[4 * j]) + __uint_as_float(x0));
          r[4 * j + 1] = __float_as_uint(__uint_as_float(r[4 * j + 1]) + __uint_as_float(x1));
          r[4 * j + 2] = __float_as_uint(__uint_as_float(r[4 * j + 2]) + __uint_as_float(x2));
          r[4 * j + 3] = __float_as_uint(__uint_as_float(r[4 * j + 3]) + __uint_as_float(x3));
        }
      };
      for (int c = 0; c < nchunks; ++c) {
        uint32_t w[32];
        epistamp<kDebug>(p, warp, lane, c, 0);
        if constexpr (sizeof(OutT) == 4) {
          tmem_ld_32x32b_x32(t_addr + c * 32, w);
          tmem_wait_ld();
          if constexpr (kSK) add_part(w, c);
        } else {
          uint32_t r0[32], r1[32];
          tmem_ld_32x32b_x32(t_addr + c * 64, r0);
          tmem_ld_32x32b_x32(t_addr + c * 64 + 32, r1);
          tmem_wait_ld();
          if constexpr (kSK) {
            add_part(r0, 2 * c);
            add_part(r1, 2 * c + 1);
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            w[i] = pack2<OutT>(r0[2 * i], r0[2 * i + 1]);
            w[16 + i] = pack2<OutT>(r1[2 * i], r1[2 * i + 1]);
          }
        }
        if (c == nchunks - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
        }
        epistamp<kDebug>(p, warp, lane, c, 1);
        const uint32_t sbuf = stage_base + buf * 4096;
        if (lane == 0) {
          if (p.stage_bufs == 2)
            bulk_wait_group_read<1>();
          else
            bulk_wait_group_read<0>();
        }
        __syncwarp();
        epistamp<kDebug>(p, warp, lane, c, 2);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          st_shared_v4(sbuf + lane * 128 + ((j ^ (lane & 7)) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2],
                       w[4 * j + 3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&tmC, sbuf, tc.nb * p.BN + c * kChunkCols, tc.mb * (2 * kTileM) + row0, tc.b);
          bulk_commit_group();
        }
        epistamp<kDebug>(p, warp, lane, c, 3);
        buf ^= p.stage_bufs - 1;
      }
    });
    if (lane == 0) bulk_wait_group_read<0>();  // smem reads done; grid completion publishes the writes
    __syncwarp();
    if (warp == 2 && lane == 0) stamp<kDebug>(p, 6);
  }

  tc_fence_before();
  cluster_sync();  // no CTA leaves while its peer may still signal it or read its smem
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, p.tmem_cols);
  }
  if (threadIdx.x == 0) stamp<kDebug>(p, 7);
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_tiled() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// rank-D tiled map with traversal strides (stem conv: overlapping pixel-stride view)
int encode_tiled(CUtensorMap* m, CUtensorMapDataType dt, const void* base, int rank, const cuuint64_t* dims,
                 const cuuint64_t* strides_bytes, const cuuint32_t* box, const cuuint32_t* estr,
                 CUtensorMapSwizzle swz, const char* what) {
  auto enc = get_encode_tiled();
  if (!enc) return set_error(ALCOP_ERR_CUDA, "CudaError", "cuTensorMapEncodeTiled unavailable");
  CUresult r = enc(m, dt, rank, const_cast<void*>(base), dims, strides_bytes, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(ALCOP_ERR_CUDA, "CudaError",
                     std::string("cuTensorMapEncodeTiled failed for ") + what + " (CUresult " + std::to_string(r) + ")");
  return ALCOP_OK;
}

int encode_3d_dt(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
              uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1,
              CUtensorMapSwizzle swz, const char* what) {
  auto enc = get_encode_tiled();
  if (!enc) return set_error(ALCOP_ERR_CUDA, "CudaError", "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(ALCOP_ERR_CUDA, "CudaError",
                     std::string("cuTensorMapEncodeTiled failed for ") + what + " (CUresult " + std::to_string(r) + ")");
  return ALCOP_OK;
}

// Stream-K workspace, one per device, registered by the caller
// (alcop_set_stream_k_workspace): the flags first (fixed place whatever the
// partial size; zero, each launch's finishers re-arm them), then the fp32
// partials (one 256 x BN slot per cluster).  A launch whose problem needs more
// than the registered bytes runs whole tiles.
namespace {
constexpr size_t kSkFlagBytes = 4096;
struct SkWs {
  void* ptr = nullptr;
  size_t bytes = 0;
};
SkWs g_sk_ws[64];
std::mutex g_sk_mu;
}  // namespace

}  // namespace (leave the kernels' anonymous namespace: these two are library-internal API)

size_t sk_bytes_needed(int n_clusters, int BN) {
  return kSkFlagBytes + static_cast<size_t>(n_clusters) * 256 * BN * 4;
}

namespace {

bool sk_workspace(size_t part_bytes, int n, float** part, int32_t** flags) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  if (static_cast<size_t>(n + 1) * sizeof(int32_t) > kSkFlagBytes) return false;
  std::lock_guard<std::mutex> lk(g_sk_mu);
  const SkWs& w = g_sk_ws[dev];
  if (!w.ptr || w.bytes < kSkFlagBytes + part_bytes) return false;
  *flags = static_cast<int32_t*>(w.ptr);
  *part = reinterpret_cast<float*>(static_cast<char*>(w.ptr) + kSkFlagBytes);
  return true;
}

}  // namespace

int set_sk_workspace(void* ptr, int64_t bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64)
    return set_error(ALCOP_ERR_CUDA, "CudaError", "no current CUDA device");
  if (ptr && bytes < static_cast<int64_t>(kSkFlagBytes))
    return set_error(ALCOP_ERR_CONFIG, "Workspace", "stream-K workspace needs at least 4096 bytes");
  if (ptr) {
    cudaError_t e = cudaMemset(ptr, 0, kSkFlagBytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return set_error(ALCOP_ERR_CUDA, "CudaError", cudaGetErrorString(e));
  }
  std::lock_guard<std::mutex> lk(g_sk_mu);
  g_sk_ws[dev].ptr = ptr;
  g_sk_ws[dev].bytes = ptr ? static_cast<size_t>(bytes) : 0;
  return ALCOP_OK;
}

namespace {

template <typename OutT, int BK, bool kJoint, bool kDebug, bool kPreOp = false, int kEpi = 4>
int launch_typed(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const GemmKParams& kp,
                 int grid, int smem, cudaStream_t st) {
  auto kern = alcop_pipelined_gemm_kernel<OutT, BK, kJoint, kDebug, false, kPreOp, kEpi>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_error(ALCOP_ERR_CUDA, "CudaError", cudaGetErrorString(e));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kPreOp ? kThreadsPreOp : (kEpi == 8 ? kThreadsEpi8 : kThreads));
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, kp);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ALCOP_ERR_CUDA, "CudaError", cudaGetErrorString(e));
  return ALCOP_OK;
}

template <typename OutT, int BK, bool kDebug = false, bool kSK = false, bool kWide = false, bool kConv = false>
int launch_pair_t(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const CUtensorMap& tw,
                  const GemmKParams& kp, int grid, int smem, cudaStream_t st) {
  auto kern = alcop_pipelined_gemm_pair_kernel<OutT, BK, kDebug, kSK, kWide, kConv>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_error(ALCOP_ERR_CUDA, "CudaError", cudaGetErrorString(e));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreadsPair);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, tw, kp);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ALCOP_ERR_CUDA, "CudaError", cudaGetErrorString(e));
  return ALCOP_OK;
}

// timeline stamps (alcop_debug_set_stamps) select the instrumented variant;
// kp.sk_flags the stream-K variant (never instrumented)
template <typename OutT, int BK>
int launch_pair(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const CUtensorMap& tw,
                const GemmKParams& kp, int grid, int smem, cudaStream_t st) {
  if (kp.BN == 512) {
    if (kp.sk_flags) return launch_pair_t<OutT, BK, false, true, true>(ta, tb, tc, tw, kp, grid, smem, st);
    return kp.stamps ? launch_pair_t<OutT, BK, true, false, true>(ta, tb, tc, tw, kp, grid, smem, st)
                     : launch_pair_t<OutT, BK, false, false, true>(ta, tb, tc, tw, kp, grid, smem, st);
  }
  if (kp.sk_flags) return launch_pair_t<OutT, BK, false, true>(ta, tb, tc, tw, kp, grid, smem, st);
  return kp.stamps ? launch_pair_t<OutT, BK, true>(ta, tb, tc, tw, kp, grid, smem, st)
                   : launch_pair_t<OutT, BK, false>(ta, tb, tc, tw, kp, grid, smem, st);
}

template <typename OutT, bool kDebug, int kConv>
int launch_typed_conv(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const GemmKParams& kp,
                      int grid, int smem, cudaStream_t st) {
  auto kern = alcop_pipelined_gemm_kernel<OutT, 64, true, kDebug, kConv>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_error(ALCOP_ERR_CUDA, "CudaError", cudaGetErrorString(e));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kDebug ? kThreads : kThreadsSplit);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, kp);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ALCOP_ERR_CUDA, "CudaError", cudaGetErrorString(e));
  return ALCOP_OK;
}

template <typename OutT, int BK>
int launch_variant(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const GemmKParams& kp,
                   int grid, int smem, cudaStream_t st) {
  const bool joint = kp.sA == kp.sB;
  const bool debug = kp.trace != nullptr || kp.stamps != nullptr;
  if (kp.pre_op) {
    if (!joint || debug)
      return set_error(ALCOP_ERR_CONFIG, "Unsupported",
                       "the fused pre-op needs equal A/B stage counts and no debug trace");
    return launch_typed<OutT, BK, true, false, true>(ta, tb, tc, kp, grid, smem, st);
  }
  if (joint) {
    return debug ? launch_typed<OutT, BK, true, true>(ta, tb, tc, kp, grid, smem, st)
                 : (kp.epi_warps == 8 ? launch_typed<OutT, BK, true, false, false, 8>(ta, tb, tc, kp, grid, smem, st)
                                      : launch_typed<OutT, BK, true, false>(ta, tb, tc, kp, grid, smem, st));
  }
  return debug ? launch_typed<OutT, BK, false, true>(ta, tb, tc, kp, grid, smem, st)
               : launch_typed<OutT, BK, false, false>(ta, tb, tc, kp, grid, smem, st);
}

template <typename OutT>
int launch_conv_typed(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const GemmKParams& kp,
                      int grid, int smem, cudaStream_t st) {
  const bool dbg = kp.trace != nullptr || kp.stamps != nullptr;
  if (kp.conv_small_c == 2)
    return dbg ? launch_typed_conv<OutT, true, 3>(ta, tb, tc, kp, grid, smem, st)
               : launch_typed_conv<OutT, false, 3>(ta, tb, tc, kp, grid, smem, st);
  if (kp.conv_small_c)
    return dbg ? launch_typed_conv<OutT, true, 2>(ta, tb, tc, kp, grid, smem, st)
               : launch_typed_conv<OutT, false, 2>(ta, tb, tc, kp, grid, smem, st);
  return dbg ? launch_typed_conv<OutT, true, 1>(ta, tb, tc, kp, grid, smem, st)
             : launch_typed_conv<OutT, false, 1>(ta, tb, tc, kp, grid, smem, st);
}

}  // namespace

// for the chain kernel (chain_sm100.cu)
int encode_tiled_map(CUtensorMap* m, CUtensorMapDataType dt, const void* base, int rank, const cuuint64_t* dims,
                     const cuuint64_t* strides_bytes, const cuuint32_t* box, const cuuint32_t* estr,
                     CUtensorMapSwizzle swz, const char* what) {
  return encode_tiled(m, dt, base, rank, dims, strides_bytes, box, estr, swz, what);
}
bool pdl_enabled() { return g_pdl; }

int device_sm_count() {
  static int sms = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) sms = v;
  });
  return sms;
}

// Tile rows per raster group.  schedule.raster > 0 sets it; 0 picks the group
// that minimises the distinct A-row + B-column panels touched by the tiles in
// flight at once (W = CTAs / cg): G*BM + (W/G)*BN  ->  G = sqrt(W*BN/BM).
static int32_t raster_group(const alcop_schedule& s, int num_m, int num_n, int BM, int BN, int cg) {
  const int ctas = s.num_ctas > 0 ? s.num_ctas : device_sm_count();
  const int W = ctas / cg > 0 ? ctas / cg : 1;
  return raster_group_of(s.raster, W, num_m, num_n, BM, BN);
}

int launch_gemm(const alcop_gemm_desc& w, const alcop_schedule& s, const void* A, const void* B, void* C,
                alcop_event* trace, int64_t trace_cap, void* stream) {
  const int64_t lda = w.lda ? w.lda : w.K;
  const int64_t ldb = w.ldb ? w.ldb : (w.b_layout == ALCOP_B_KN ? w.N : w.K);
  const int64_t ldc = w.ldc ? w.ldc : w.N;
  const int64_t sa = w.stride_a ? w.stride_a : w.M * lda;
  const int64_t sb = w.stride_b ? w.stride_b : (w.b_layout == ALCOP_B_KN ? w.K * ldb : w.N * ldb);
  const int64_t sc = w.stride_c ? w.stride_c : w.M * ldc;
  const CUtensorMapDataType dt =
      w.in_dtype == ALCOP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const int BN = static_cast<int>(s.tileN), BK = static_cast<int>(s.tileK);
  const int cg = s.cta_group == 2 ? 2 : 1;
  const CUtensorMapSwizzle kswz = BK >= 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  const uint32_t kbox = BK >= 64 ? 64 : BK;

  CUtensorMap ta, tb;
  // Atom-stacked views (one TMA instruction per operand per chunk) need the
  // atom dimension to tile the row exactly: a ragged last atom would read
  // across the row end instead of zero-filling.  ALCOP_ATOM_VIEWS=0 disables.
  static const bool views_on = [] {
    const char* e = std::getenv("ALCOP_ATOM_VIEWS");
    return !(e && e[0] == '0');
  }();
  const bool b_pad = pair_b_pad(w, s);
  const int b_atom = (w.b_layout == ALCOP_B_KN && ((BN / cg) & 63) != 0 && !b_pad) ? 32 : 64;  // pair BN 192: SW64 halves
  const bool a_view = views_on && BK > 64 && w.K % 64 == 0 && w.pre_op == 0;
  // B[K,N] on one CTA: the atom-stacked view loads a chunk's BN/64 atoms in one box (the single producer
  // issues 2 TMA instructions per chunk instead of 1 + BN/64)
  const bool b_view = views_on && cg == 1 && w.b_layout == ALCOP_B_KN && w.pre_op == 0 && BN % 64 == 0 &&
                      BN >= 128 && w.N % 64 == 0 && BK >= 64;
  int rc;
  if (a_view) {
    const cuuint64_t dims[4] = {64, static_cast<cuuint64_t>(w.M), static_cast<cuuint64_t>(w.K / 64),
                                static_cast<cuuint64_t>(w.batch)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(lda * 2), 128, static_cast<cuuint64_t>(sa * 2)};
    const cuuint32_t box[4] = {64, kTileM, static_cast<cuuint32_t>(BK / 64), 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    rc = encode_tiled(&ta, dt, A, 4, dims, strides, box, es, CU_TENSOR_MAP_SWIZZLE_128B, "A (atom view)");
  } else {
    rc = encode_3d_dt(&ta, dt, A, w.K, w.M, w.batch, lda * 2, sa * 2, kbox, kTileM, kswz, "A");
  }
  if (rc) return rc;
  if (b_view) {
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(b_atom), static_cast<cuuint64_t>(w.K),
                                static_cast<cuuint64_t>(w.N / b_atom), static_cast<cuuint64_t>(w.batch)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(ldb * 2), static_cast<cuuint64_t>(b_atom * 2),
                                   static_cast<cuuint64_t>(sb * 2)};
    const cuuint32_t box[4] = {static_cast<cuuint32_t>(b_atom), static_cast<cuuint32_t>(BK),
                               static_cast<cuuint32_t>((BN / cg) / b_atom), 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    rc = encode_tiled(&tb, dt, B, 4, dims, strides, box, es,
                      b_atom == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, "B (atom view)");
  } else if (w.b_layout == ALCOP_B_KN && b_atom == 32) {  // pair, BN 192: 32-column SW64 boxes
    rc = encode_3d_dt(&tb, dt, B, w.N, w.K, w.batch, ldb * 2, sb * 2, 32, BK, CU_TENSOR_MAP_SWIZZLE_64B, "B");
  } else if (w.b_layout == ALCOP_B_KN) {
    rc = encode_3d_dt(&tb, dt, B, w.N, w.K, w.batch, ldb * 2, sb * 2, 64, BK, CU_TENSOR_MAP_SWIZZLE_128B, "B");
  } else {
    rc = encode_3d_dt(&tb, dt, B, w.K, w.N, w.batch, ldb * 2, sb * 2, kbox, BN == 512 ? 128 : BN / cg, kswz, "B");
  }
  if (rc) return rc;
  CUtensorMap tc;
  {
    const CUtensorMapDataType odt = w.out_dtype == ALCOP_F32    ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                    : w.out_dtype == ALCOP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                                : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    const int ob = w.out_dtype == ALCOP_F32 ? 4 : 2;
    rc = encode_3d_dt(&tc, odt, C, w.N, w.M, w.batch, ldc * ob, sc * ob, 128 / ob, 32, CU_TENSOR_MAP_SWIZZLE_128B,
                      "C");
    if (rc) return rc;
  }

  GemmKParams kp{};
  kp.M = static_cast<int32_t>(w.M);
  kp.N = static_cast<int32_t>(w.N);
  kp.K = static_cast<int32_t>(w.K);
  kp.batch = static_cast<int32_t>(w.batch);
  kp.BN = BN;
  kp.BK = BK;
  kp.num_m = static_cast<int32_t>((w.M + kTileM * cg - 1) / (kTileM * cg));
  kp.num_n = static_cast<int32_t>((w.N + BN - 1) / BN);
  kp.num_tiles = static_cast<int32_t>(kp.num_m * kp.num_n * w.batch);
  kp.group_m = raster_group(s, kp.num_m, kp.num_n, kTileM * cg, BN, cg);
  kp.E = static_cast<int32_t>((w.K + BK - 1) / BK);
  kp.sA = s.n_stage_smem_A;
  kp.sB = s.n_stage_smem_B;
  kp.tacc = s.n_stage_inner;
  kp.mode = s.mode;
  kp.b_mn_major = w.b_layout == ALCOP_B_KN ? 1 : 0;
  kp.idesc = ptx::make_idesc_f16(w.in_dtype == ALCOP_BF16 ? 1u : 0u, kp.b_mn_major, kTileM * cg,
                                 BN > 256 ? 256 : BN);  // tileN 512 = two N = 256 MMAs
  kp.a_stage_bytes = static_cast<uint32_t>(kTileM * BK * 2);
  kp.b_stage_bytes = static_cast<uint32_t>((b_pad ? (BN / cg + 63) / 64 * 64 : BN / cg) * BK * 2);
  kp.acc_stride = static_cast<uint32_t>(round_up_pow2_cols(BN));
  kp.tmem_cols = static_cast<uint32_t>(round_up_pow2_cols(kp.acc_stride * kp.tacc));
  kp.C = C;
  kp.ldc = ldc;
  kp.stride_c = sc;
  kp.trace = trace;
  kp.trace_cap = static_cast<int32_t>(trace_cap);
  kp.stamps = g_stamps;
  kp.in_bf16 = w.in_dtype == ALCOP_BF16 ? 1 : 0;
  kp.pre_op = w.pre_op;
  kp.b_pad = b_pad ? 1 : 0;
  kp.a_view = a_view ? 1 : 0;
  kp.b_view = b_view ? 1 : 0;

  int sms = device_sm_count();
  if (sms <= 0) return set_error(ALCOP_ERR_CUDA, "CudaError", "no CUDA device");
  int grid = s.num_ctas > 0 ? s.num_ctas : sms;
  kp.epi_warps = cg == 1 ? gemm_epi_warps(w, s) : 4;
  const int smem = static_cast<int>(gemm_smem_bytes_epi(w, s, kp.epi_warps));
  kp.stage_bufs = gemm_staging_bufs_epi(w, s, kp.epi_warps);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (cg == 2) {
    if (w.pre_op) return set_error(ALCOP_ERR_CONFIG, "Unsupported", "the fused pre-op runs with cta_group 1");
    if (trace != nullptr)
      return set_error(ALCOP_ERR_CONFIG, "Unsupported", "the device trace is implemented for cta_group 1");
    grid = (grid / 2) * 2;
    if (grid > 2 * kp.num_tiles) grid = 2 * kp.num_tiles;
    CUtensorMap tw = tc;  // stream-K partials (unused otherwise)
    if (s.stream_k && s.mode == ALCOP_MODE_FUSED && !kp.stamps) {
      // needs >= E chunks per cluster (a tile then spans at most two
      // clusters) and the ring to hold one 256 x BN fp32 partial per CTA
      const int n = grid / 2;
      const bool fits = static_cast<int64_t>(kp.sA) * (kp.a_stage_bytes + kp.b_stage_bytes) >= int64_t(BN) * 512;
      float* part = nullptr;
      int32_t* flags = nullptr;
      if (kp.num_tiles >= n && fits && sk_workspace(static_cast<size_t>(n) * 256 * BN * 4, n, &part, &flags)) {
        rc = encode_3d_dt(&tw, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, part, BN, 256, n, BN * 4, int64_t(256) * BN * 4, 32,
                          32, CU_TENSOR_MAP_SWIZZLE_128B, "stream-K partials");
        if (rc) return rc;
        kp.sk_flags = flags;
      }
    }
    switch (w.out_dtype * 4 + (BK == 32 ? 0 : BK == 64 ? 1 : 2)) {
      case ALCOP_F32 * 4 + 0: return launch_pair<float, 32>(ta, tb, tc, tw, kp, grid, smem, st);
      case ALCOP_F32 * 4 + 1: return launch_pair<float, 64>(ta, tb, tc, tw, kp, grid, smem, st);
      case ALCOP_F32 * 4 + 2: return launch_pair<float, 128>(ta, tb, tc, tw, kp, grid, smem, st);
      case ALCOP_BF16 * 4 + 0: return launch_pair<__nv_bfloat16, 32>(ta, tb, tc, tw, kp, grid, smem, st);
      case ALCOP_BF16 * 4 + 1: return launch_pair<__nv_bfloat16, 64>(ta, tb, tc, tw, kp, grid, smem, st);
      case ALCOP_BF16 * 4 + 2: return launch_pair<__nv_bfloat16, 128>(ta, tb, tc, tw, kp, grid, smem, st);
      case ALCOP_F16 * 4 + 0: return launch_pair<__half, 32>(ta, tb, tc, tw, kp, grid, smem, st);
      case ALCOP_F16 * 4 + 1: return launch_pair<__half, 64>(ta, tb, tc, tw, kp, grid, smem, st);
      case ALCOP_F16 * 4 + 2: return launch_pair<__half, 128>(ta, tb, tc, tw, kp, grid, smem, st);
    }
    return set_error(ALCOP_ERR_CONFIG, "BadDtype", "unsupported output dtype");
  }
  if (grid > kp.num_tiles) grid = kp.num_tiles;
  switch (w.out_dtype * 4 + (BK == 32 ? 0 : BK == 64 ? 1 : 2)) {
    case ALCOP_F32 * 4 + 0: return launch_variant<float, 32>(ta, tb, tc, kp, grid, smem, st);
    case ALCOP_F32 * 4 + 1: return launch_variant<float, 64>(ta, tb, tc, kp, grid, smem, st);
    case ALCOP_F32 * 4 + 2: return launch_variant<float, 128>(ta, tb, tc, kp, grid, smem, st);
    case ALCOP_BF16 * 4 + 0: return launch_variant<__nv_bfloat16, 32>(ta, tb, tc, kp, grid, smem, st);
    case ALCOP_BF16 * 4 + 1: return launch_variant<__nv_bfloat16, 64>(ta, tb, tc, kp, grid, smem, st);
    case ALCOP_BF16 * 4 + 2: return launch_variant<__nv_bfloat16, 128>(ta, tb, tc, kp, grid, smem, st);
    case ALCOP_F16 * 4 + 0: return launch_variant<__half, 32>(ta, tb, tc, kp, grid, smem, st);
    case ALCOP_F16 * 4 + 1: return launch_variant<__half, 64>(ta, tb, tc, kp, grid, smem, st);
    case ALCOP_F16 * 4 + 2: return launch_variant<__half, 128>(ta, tb, tc, kp, grid, smem, st);
  }
  return set_error(ALCOP_ERR_CONFIG, "BadDtype", "unsupported output dtype");
}

PFN_cuTensorMapEncodeIm2col_v12000 get_encode_im2col() {
  static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(ptr);
  });
  return fn;
}

// Implicit-GEMM conv2d (K3): x NHWC, w KRSC, y NPQK.  GEMM view
// M = N*P*Q output pixels, N = K filters, K = R*S*C in the filter's own order.
// A tiles come from the im2col-mode tensor map of x (window origin per
// output pixel, filter-tap offsets, zero fill at the padding), B from w
// viewed as [K, R*S*C] (K-major), C goes to y viewed as [N*P*Q, K].
int launch_conv2d(const alcop_conv_desc& d, const alcop_schedule& s, const void* x, const void* wt, void* y,
                  void* stream) {
  if (d.N < 1 || d.H < 1 || d.W < 1 || d.C < 1 || d.K < 1 || d.R < 1 || d.S < 1 || d.stride_h < 1 ||
      d.stride_w < 1 || d.pad_h < 0 || d.pad_w < 0)
    return set_error(ALCOP_ERR_CONFIG, "BadWorkload", "conv dimensions must be positive, padding >= 0");
  if (d.C == 4) return launch_conv2d_stem_pairs(d, s, x, wt, y, stream);  // stem_sm100.cu
  // C = 64 stride-1 spatial filters with a resident-filter schedule (tileN = K,
  // FUSED): the window mode of the same kernel (the input window loaded once
  // per tile); other schedules run the im2col kernel below
  if ((window_conv_applicable(d) || window_stream_applicable(d)) && validate_stem_pairs(d, s) == ALCOP_OK)
    return launch_conv2d_stem_pairs(d, s, x, wt, y, stream);
  clear_error();
  // A 1x1, stride-1, unpadded conv is a plain GEMM: x viewed as [N*H*W, C],
  // the filter as B[K, C] (K-major), y as [N*H*W, K] — it runs on the GEMM
  // kernels, whose space includes the CTA-pair tiles (the im2col kernel is
  // single-CTA only)
  if (conv_is_gemm(d)) {
    alcop_gemm_desc g{};
    conv_gemm_view(d, &g);
    int rc = validate_gemm(g, s);
    if (rc) return rc;
    return launch_gemm(g, s, x, wt, y, nullptr, 0, stream);
  }
  if (d.C % 8)
    return set_error(ALCOP_ERR_CONFIG, "Unsupported",
                     "implicit-GEMM conv needs C to be a multiple of 8 (pad NHWC channels, e.g. 3 -> 8), or C = 4 "
                     "with stride_w 2 (the stem kernel)");
  const bool small_c = (d.C % 64) != 0;  // 8-channel im2col boxes (no-swizzle core matrices)
  const bool halo = d.x_halo != 0;
  // stem kernel: a filter row's S*C taps are contiguous in the halo-padded input
  const bool stem = halo && d.S * d.C <= 64 && d.stride_w * 16 <= 256 && d.stride_h * 8 <= 256;
  const int64_t Hs = halo ? d.H + 2 * d.pad_h : d.H, Ws = halo ? d.W + 2 * d.pad_w : d.W;  // stored extents
  const int ph = halo ? 0 : d.pad_h, pw = halo ? 0 : d.pad_w;  // padding the im2col map applies
  // 5-D stem view unless disabled (ALCOP_STEM5=0) or the stored height is not a stride multiple
  static const bool stem5_env = [] {
    const char* e = std::getenv("ALCOP_STEM5");
    return !(e && e[0] == '0');
  }();
  const bool stem5 = stem && stem5_env && (Hs % d.stride_h) == 0 && d.stride_w * d.C * 2 % 16 == 0;
  if (d.stride_h > 8 || d.stride_w > 8 || d.pad_h > 127 || d.pad_w > 127 || d.R > 128 || d.S > 128)
    return set_error(ALCOP_ERR_CONFIG, "Unsupported", "stride <= 8 and padding/filter within TMA im2col range");
  if (s.tileK != 64 || s.n_stage_smem_A != s.n_stage_smem_B)
    return set_error(ALCOP_ERR_CONFIG, "BadSchedule", "conv needs tileK 64 and equal A/B stage counts");
  // CTA pairs: the 64-channel im2col path (C % 64 == 0, no halo layout), whole tiles
  const bool pair = s.cta_group == 2;
  if (s.stream_k != 0 || (pair && (small_c || halo)) || (s.cta_group != 1 && !pair))
    return set_error(ALCOP_ERR_CONFIG, "BadSchedule",
                     "the implicit-GEMM conv kernel runs whole tiles, with cta_group 1 or (C % 64 == 0, no halo) 2");
  const int64_t P = (d.H + 2 * d.pad_h - d.R) / d.stride_h + 1;
  const int64_t Q = (d.W + 2 * d.pad_w - d.S) / d.stride_w + 1;
  if (P < 1 || Q < 1) return set_error(ALCOP_ERR_CONFIG, "BadWorkload", "empty output");
  alcop_gemm_desc g{};
  g.M = d.N * P * Q;
  g.N = d.K;
  g.K = stem ? d.R * 64 : d.R * d.S * d.C;
  g.batch = 1;
  g.in_dtype = d.in_dtype;
  g.out_dtype = d.out_dtype;
  g.b_layout = ALCOP_B_NK;
  int rc = validate_gemm(g, s);
  if (rc) return rc;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(wt) | reinterpret_cast<uintptr_t>(y)) & 15)
    return set_error(ALCOP_ERR_CONFIG, "Alignment", "x, w and y must be 16-byte aligned");
  const CUtensorMapDataType dt =
      d.in_dtype == ALCOP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  auto enc = get_encode_im2col();
  if (!enc) return set_error(ALCOP_ERR_CUDA, "CudaError", "cuTensorMapEncodeIm2col unavailable");
  CUtensorMap ta, tb, tc;
  const int BN = static_cast<int>(s.tileN);
  const CUtensorMapDataType odt = d.out_dtype == ALCOP_F32    ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                  : d.out_dtype == ALCOP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                              : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const int ob = d.out_dtype == ALCOP_F32 ? 4 : 2;
  if (stem) {
    // A: {S*C taps of one filter row (elements 56..63 zero-filled), window
    // origin pixel (stride C: overlapping view), row, image}; box 64 x 16 x 8
    // output positions at traversal strides (1, stride_w, stride_h)
    const cuuint32_t one[5] = {1, 1, 1, 1, 1};
    if (stem5) {
      // the strides folded into the view: q steps stride_w pixels, p steps
      // stride_h rows, filter row r = (r / stride_h) p-steps + (r % stride_h) rows
      const cuuint64_t adims[5] = {static_cast<cuuint64_t>(d.S * d.C), static_cast<cuuint64_t>(Q),
                                   static_cast<cuuint64_t>(Hs / d.stride_h), static_cast<cuuint64_t>(d.stride_h),
                                   static_cast<cuuint64_t>(d.N)};
      const cuuint64_t astr[4] = {static_cast<cuuint64_t>(d.stride_w * d.C * 2),
                                  static_cast<cuuint64_t>(d.stride_h * Ws * d.C * 2),
                                  static_cast<cuuint64_t>(Ws * d.C * 2), static_cast<cuuint64_t>(Hs * Ws * d.C * 2)};
      const cuuint32_t abox[5] = {64, 16, 8, 1, 1};
      rc = encode_tiled(&ta, dt, x, 5, adims, astr, abox, one, CU_TENSOR_MAP_SWIZZLE_128B, "x (stem)");
    } else {
      const cuuint64_t adims[4] = {static_cast<cuuint64_t>(d.S * d.C), static_cast<cuuint64_t>(Ws - d.S + 1),
                                   static_cast<cuuint64_t>(Hs), static_cast<cuuint64_t>(d.N)};
      const cuuint64_t astr[3] = {static_cast<cuuint64_t>(d.C * 2), static_cast<cuuint64_t>(Ws * d.C * 2),
                                  static_cast<cuuint64_t>(Hs * Ws * d.C * 2)};
      const cuuint32_t abox[4] = {64, static_cast<cuuint32_t>(16 * d.stride_w),
                                  static_cast<cuuint32_t>(8 * d.stride_h), 1};
      const cuuint32_t aestr[4] = {1, static_cast<cuuint32_t>(d.stride_w), static_cast<cuuint32_t>(d.stride_h), 1};
      rc = encode_tiled(&ta, dt, x, 4, adims, astr, abox, aestr, CU_TENSOR_MAP_SWIZZLE_128B, "x (stem)");
    }
    if (rc) return rc;
    // B: filter row r = S*C contiguous taps of w[k][r][.][.], zero-filled to 64
    const cuuint64_t bdims[3] = {static_cast<cuuint64_t>(d.S * d.C), static_cast<cuuint64_t>(d.R),
                                 static_cast<cuuint64_t>(d.K)};
    const cuuint64_t bstr[2] = {static_cast<cuuint64_t>(d.S * d.C * 2), static_cast<cuuint64_t>(d.R * d.S * d.C * 2)};
    const cuuint32_t bbox[3] = {64, 1, static_cast<cuuint32_t>(BN)};
    rc = encode_tiled(&tb, dt, wt, 3, bdims, bstr, bbox, one, CU_TENSOR_MAP_SWIZZLE_128B, "w (stem)");
    if (rc) return rc;
    // y as {K, Q, P, N}: each epilogue warp stores 2 output rows x 16 columns
    const cuuint64_t cdims[4] = {static_cast<cuuint64_t>(d.K), static_cast<cuuint64_t>(Q), static_cast<cuuint64_t>(P),
                                 static_cast<cuuint64_t>(d.N)};
    const cuuint64_t cstr[3] = {static_cast<cuuint64_t>(d.K * ob), static_cast<cuuint64_t>(Q * d.K * ob),
                                static_cast<cuuint64_t>(P * Q * d.K * ob)};
    const cuuint32_t cbox[4] = {static_cast<cuuint32_t>(128 / ob), 16, 2, 1};
    rc = encode_tiled(&tc, odt, y, 4, cdims, cstr, cbox, one, CU_TENSOR_MAP_SWIZZLE_128B, "y (stem)");
    if (rc) return rc;
  } else {
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(d.C), static_cast<cuuint64_t>(Ws), static_cast<cuuint64_t>(Hs),
                          static_cast<cuuint64_t>(d.N)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(d.C * 2), static_cast<cuuint64_t>(Ws * d.C * 2),
                             static_cast<cuuint64_t>(Hs * Ws * d.C * 2)};
    // bounding box of window origins, per spatial dim in tensor order (W, H)
    int lower[2] = {-pw, -ph};
    int upper[2] = {static_cast<int>(pw - (d.S - 1)), static_cast<int>(ph - (d.R - 1))};
    cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(d.stride_w), static_cast<cuuint32_t>(d.stride_h), 1};
    CUresult r = enc(&ta, dt, 4, const_cast<void*>(x), dims, strides, lower, upper, small_c ? 8 : 64, kTileM, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, small_c ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return set_error(ALCOP_ERR_CUDA, "CudaError", "cuTensorMapEncodeIm2col failed (CUresult " + std::to_string(r) + ")");
    rc = encode_3d_dt(&tb, dt, wt, g.K, g.N, 1, g.K * 2, g.N * g.K * 2, 64, pair ? BN / 2 : BN,
                      CU_TENSOR_MAP_SWIZZLE_128B, "w");
    if (rc) return rc;
    rc = encode_3d_dt(&tc, odt, y, g.N, g.M, 1, g.N * ob, g.M * g.N * ob, 128 / ob, 32, CU_TENSOR_MAP_SWIZZLE_128B,
                      "y");
    if (rc) return rc;
  }

  GemmKParams kp{};
  kp.M = static_cast<int32_t>(g.M);
  kp.N = static_cast<int32_t>(g.N);
  kp.K = static_cast<int32_t>(g.K);
  kp.batch = 1;
  kp.BN = BN;
  kp.BK = 64;
  kp.conv_Pb = static_cast<int32_t>((P + 7) / 8);
  kp.conv_Qb = static_cast<int32_t>((Q + 15) / 16);
  kp.num_m = stem ? static_cast<int32_t>(d.N * kp.conv_Pb * kp.conv_Qb)
                  : static_cast<int32_t>((g.M + kTileM * s.cta_group - 1) / (kTileM * s.cta_group));
  kp.num_n = static_cast<int32_t>((g.N + BN - 1) / BN);
  kp.num_tiles = kp.num_m * kp.num_n;
  kp.group_m = raster_group(s, kp.num_m, kp.num_n, kTileM * s.cta_group, BN, s.cta_group);
  kp.E = static_cast<int32_t>((g.K + 63) / 64);  // small C: the last chunk's taps past R*S meet zero filter rows
                                                 // stem: one chunk per filter row (g.K = R * 64)
  kp.sA = s.n_stage_smem_A;
  kp.sB = s.n_stage_smem_B;
  kp.tacc = s.n_stage_inner;
  kp.mode = s.mode;
  kp.b_mn_major = 0;
  kp.idesc = ptx::make_idesc_f16(d.in_dtype == ALCOP_BF16 ? 1u : 0u, 0u, kTileM * s.cta_group, BN);
  kp.a_stage_bytes = static_cast<uint32_t>(kTileM * 64 * 2);
  kp.b_stage_bytes = static_cast<uint32_t>((pair ? BN / 2 : BN) * 64 * 2);
  kp.acc_stride = static_cast<uint32_t>(round_up_pow2_cols(BN));
  kp.tmem_cols = static_cast<uint32_t>(round_up_pow2_cols(kp.acc_stride * kp.tacc));
  kp.C = y;
  kp.ldc = g.N;
  kp.stride_c = g.M * g.N;
  kp.stamps = g_stamps;
  kp.conv_P = static_cast<int32_t>(P);
  kp.conv_Q = static_cast<int32_t>(Q);
  kp.conv_S = static_cast<int32_t>(d.S);
  kp.conv_Cb = static_cast<int32_t>(small_c ? d.C / 8 : d.C / 64);
  kp.conv_RS = static_cast<int32_t>(d.R * d.S);
  kp.conv_small_c = stem ? 2 : small_c ? 1 : 0;
  kp.conv_stem5 = stem5 ? 1 : 0;
  kp.conv_sh = d.stride_h;
  kp.conv_sw = d.stride_w;
  kp.conv_ph = ph;
  kp.conv_pw = pw;
  const int sms = device_sm_count();
  if (sms <= 0) return set_error(ALCOP_ERR_CUDA, "CudaError", "no CUDA device");
  int grid = s.num_ctas > 0 ? s.num_ctas : sms;
  if (grid > kp.num_tiles) grid = kp.num_tiles;
  const int smem = static_cast<int>(gemm_smem_bytes_epi(g, s, 4));
  kp.stage_bufs = gemm_staging_bufs_epi(g, s, 4);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (pair) {
    if (kp.stamps) return set_error(ALCOP_ERR_CONFIG, "Unsupported", "conv CTA pairs run without timeline stamps");
    grid = ((s.num_ctas > 0 ? s.num_ctas : sms) / 2) * 2;
    if (grid > 2 * kp.num_tiles) grid = 2 * kp.num_tiles;
    kp.epi_warps = 4;
    switch (d.out_dtype) {
      case ALCOP_F32: return launch_pair_t<float, 64, false, false, false, true>(ta, tb, tc, tc, kp, grid, smem, st);
      case ALCOP_BF16:
        return launch_pair_t<__nv_bfloat16, 64, false, false, false, true>(ta, tb, tc, tc, kp, grid, smem, st);
      case ALCOP_F16: return launch_pair_t<__half, 64, false, false, false, true>(ta, tb, tc, tc, kp, grid, smem, st);
    }
    return set_error(ALCOP_ERR_CONFIG, "BadDtype", "unsupported output dtype");
  }
  switch (d.out_dtype) {
    case ALCOP_F32: return launch_conv_typed<float>(ta, tb, tc, kp, grid, smem, st);
    case ALCOP_BF16: return launch_conv_typed<__nv_bfloat16>(ta, tb, tc, kp, grid, smem, st);
    case ALCOP_F16: return launch_conv_typed<__half>(ta, tb, tc, kp, grid, smem, st);
  }
  return set_error(ALCOP_ERR_CONFIG, "BadDtype", "unsupported output dtype");
}

}  // namespace alcop

// Debug-only: route an 8 x uint64 per-CTA globaltimer timeline of the next
// launches into `dev` (device memory, >= 8 * grid entries); NULL turns it off.
extern "C" void alcop_debug_set_stamps(void* dev) { alcop::g_stamps = static_cast<uint64_t*>(dev); }
// Debug-only: programmatic dependent launch on (1, default) / off (0).
extern "C" void alcop_debug_set_pdl(int on) { alcop::g_pdl = on != 0; }
