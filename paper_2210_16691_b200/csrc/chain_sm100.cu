// chain_sm100.cu — several pipelined GEMMs in ONE persistent launch.
//
// The layer's GEMMs (BERT: QKV, O, FFN1, FFN2) run back to back as separate
// launches lose, per launch, the setup, the first fill of the smem ring and
// the epilogue of the last tile (with one tile per CTA nothing overlaps it):
// 4 x 4096x768x768 as four launches take 34 us, as one 16384x768x768 launch
// 21 us (tools/chain_probe.py).  Here the producer/MMA/epilogue pipeline of
// gemm_sm100.cu walks ONE flattened stream of (problem, tile, chunk): the
// smem ring (outer level) and the TMEM accumulator ring (inner level) never
// drain between GEMMs, so the epilogue of GEMM p's last tile overlaps the
// main loop of GEMM p+1's first tile — the paper's holistic pipeline, one
// level up.
//
// Dependencies: with dep[p] set, A of GEMM p row-block mb is read only after
// every tile of GEMM p-1's row-block mb is stored (the chain C_{p-1} -> A_p).
// Tiles are ordered row-block-major (n fastest) so row-blocks complete in
// order; the epilogue publishes a row-block counter after its TMA stores
// complete (cp.async.bulk.wait_group 0, proxy fence, release add) and the
// producer acquires it before the TMA loads (acquire load, proxy fence).
// Every CTA walks the global order, so nothing waits on later work: no
// deadlock with all CTAs resident (grid <= SMs, one CTA per SM).
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
int device_sm_count();
bool pdl_enabled();

namespace {

constexpr int kMaxProblems = ALCOP_CHAIN_MAX;
constexpr int kChainThreads = 192;

struct ChainProblem {
  int32_t num_m, num_n, E, tiles, key0, dep;  // key0: first global tile index (chain_tile)
};

struct ChainKParams {
  int32_t n, total_tiles, max_key, BN, sA, tacc, b_mn_major, stage_bufs, max_mb;
  int32_t bn_cta;     // B columns (rows, K-major) each CTA stages: BN, or BN / 2 on a CTA pair
  uint32_t idesc, a_stage_bytes, b_stage_bytes, acc_stride, tmem_cols;
  int32_t* counters;  // [n][max_mb] row-block completion counters (4 per stored tile and CTA)
  ChainProblem prob[kMaxProblems];
};

struct ChainMaps {
  CUtensorMap a[kMaxProblems], b[kMaxProblems], c[kMaxProblems];
};

template <typename OutT>
__device__ __forceinline__ uint32_t pack2c(uint32_t a, uint32_t b);
template <>
__device__ __forceinline__ uint32_t pack2c<__nv_bfloat16>(uint32_t a, uint32_t b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(a), __uint_as_float(b));
  return *reinterpret_cast<uint32_t*>(&h);
}
template <>
__device__ __forceinline__ uint32_t pack2c<__half>(uint32_t a, uint32_t b) {
  __half2 h = __floats2half2_rn(__uint_as_float(a), __uint_as_float(b));
  return *reinterpret_cast<uint32_t*>(&h);
}

struct ChainTile {
  int p, mb, nb, E;
};

// Scheduling order: the problems one after another, each row-block-major (n
// fastest), CTAs round-robin over the flattened sequence.  (Interleaving a
// dependent problem behind its producer with a two-round lag removes the
// dependency waits but mixes two problems' operands in L2; measured slower,
// tools/chain_step_probe.py.)
__device__ __forceinline__ ChainTile chain_tile(const ChainKParams& k, int t) {
  int p = 0;
#pragma unroll
  for (int i = 1; i < kMaxProblems; ++i)
    if (i < k.n && t >= k.prob[i].key0) p = i;
  const int lt = t - k.prob[p].key0;
  ChainTile c;
  c.p = p;
  c.mb = lt / k.prob[p].num_n;
  c.nb = lt - c.mb * k.prob[p].num_n;
  c.E = k.prob[p].E;
  return c;
}

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int32_t* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// kPair: the chain on CTA pairs (cta_group::2, 256-row tiles): each CTA loads
// its 128 rows of A and half of B's tile columns, both CTAs' copies complete
// on the leader's full barrier, the leader issues M = 256 MMAs and multicasts
// the releases, each CTA drains its own TMEM; the row-block counters count
// 256-row blocks (4 epilogue warps x 2 CTAs per stored tile).
template <typename OutT, int BK, bool kPair = false>
__global__ void __launch_bounds__(kChainThreads, 1)
    alcop_chain_gemm_kernel(const __grid_constant__ ChainMaps maps, const __grid_constant__ ChainKParams p) {
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
                                               4 * 32 * 128 * p.stage_bufs);
  uint64_t* full = bars;
  uint64_t* empty = full + p.sA;
  uint64_t* tfull = empty + p.sA;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const uint32_t rank = kPair ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  constexpr int kRows = kPair ? 2 * kTileM : kTileM;  // output rows per tile
  constexpr int kPubs = kPair ? 8 : 4;                 // counter increments per stored tile
  if (warp == 0 && elect_one()) {
    for (int i = 0; i < p.n; ++i) {
      prefetch_tmap(&maps.a[i]);
      prefetch_tmap(&maps.b[i]);
      prefetch_tmap(&maps.c[i]);
    }
  }
  if (warp == 1) {
    if (elect_one()) {
      for (int i = 0; i < p.sA; ++i) {
        mbar_init(smem_u32(&full[i]), 1);
        mbar_init(smem_u32(&empty[i]), 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(smem_u32(&tfull[i]), 1);
        mbar_init(smem_u32(&tempty[i]), kPair ? 8 : 4);  // 4 epilogue warps (x 2 CTAs)
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
  tc_fence_before();
  if constexpr (kPair)
    cluster_sync();  // both CTAs' barriers initialised before any remote arrive / complete_tx
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  grid_dependency_wait();
  grid_launch_dependents();

  // work units: CTAs, or CTA pairs walking the pair tiles
  const int grid = kPair ? static_cast<int>(gridDim.x) >> 1 : static_cast<int>(gridDim.x);
  const int unit = kPair ? static_cast<int>(blockIdx.x) >> 1 : static_cast<int>(blockIdx.x);
  const int my_tiles = (p.total_tiles - unit + grid - 1) / grid;

  if (warp == 0) {
    // ======================= producer (TMA), one flattened stream =======================
    uint32_t phase = 0;
    int slot = 0;
    const uint32_t bytes = (kPair ? 2u : 1u) * (p.a_stage_bytes + p.b_stage_bytes);  // (both CTAs' halves)
    for (int tl = 0; tl < my_tiles; ++tl) {
      const ChainTile ct = chain_tile(p, unit + tl * grid);
      const CUtensorMap* ta = &maps.a[ct.p];
      const CUtensorMap* tb = &maps.b[ct.p];
      if (p.prob[ct.p].dep) {
        // A row block mb of GEMM p is C row block mb of GEMM p-1: wait for its
        // num_n tiles (4 epilogue warps each), then order the TMA reads after
        const int32_t* cnt = p.counters + (ct.p - 1) * p.max_mb + ct.mb;
        const int target = kPubs * p.prob[ct.p - 1].num_n;
        if (elect_one()) {
          long long t0 = 0;
          while (ld_acquire(cnt) < target) {
            if (t0 == 0) t0 = clock64();
            if (clock64() - t0 > (1ll << 33)) asm volatile("trap;");
            __nanosleep(64);
          }
          fence_proxy_async_global();
        }
        __syncwarp();
      }
      for (int c = 0; c < ct.E; ++c) {
        mbar_wait(smem_u32(&empty[slot]), ((phase >> slot) & 1u) ^ 1u);  // producer_acquire
        phase ^= 1u << slot;
        const uint32_t fb = smem_u32(&full[slot]);
        if (elect_one()) {
          // a CTA pair: this CTA's 128 rows of A and its half of the tile's B
          // columns, completing on the leader's barrier (armed by the leader)
          auto ld = [&](uint32_t dst, const CUtensorMap* m, int c0, int c1) {
            if constexpr (kPair)
              tma_load_3d_pair(dst, m, mapa_shared(fb, 0), c0, c1, 0);
            else
              tma_load_3d(dst, m, fb, c0, c1, 0);
          };
          if (leader) mbar_arrive_expect_tx(fb, bytes);  // producer_commit
          const int row0 = ct.mb * kRows + static_cast<int>(rank) * kTileM;
          const int n0 = ct.nb * p.BN + static_cast<int>(rank) * p.bn_cta;
#pragma unroll
          for (int a = 0; a < kKAtoms; ++a) ld(ringA + slot * p.a_stage_bytes + a * (kTileM * 128), ta, c * BK + a * kBoxK, row0);
          const uint32_t dst = ringB + slot * p.b_stage_bytes;
          if (p.b_mn_major) {
            for (int a = 0; a < (p.bn_cta >> 6); ++a) ld(dst + a * (BK * 128), tb, n0 + a * 64, c * BK);
          } else {
#pragma unroll
            for (int a = 0; a < kKAtoms; ++a) ld(dst + a * (p.bn_cta * 128), tb, c * BK + a * kBoxK, n0);
          }
        }
        __syncwarp();
        slot = (slot + 1 == p.sA) ? 0 : slot + 1;
      }
    }
  } else if (warp == 1 && leader) {
    // ======================= MMA issuer (a CTA pair: the leader's, for both) =======================
    uint32_t phase = 0;
    int slot = 0;
    const uint64_t adesc0 = make_smem_desc(ringA, 16, kKSbo, kKLayout);
    uint64_t bdesc0;
    uint32_t b_big, b_small;
    if (p.b_mn_major) {
      bdesc0 = make_smem_desc(ringB, BK * 128, 1024, kLayoutSW128);
      b_small = 2048 / 16;
      b_big = 4 * b_small;
    } else {
      bdesc0 = make_smem_desc(ringB, 16, kKSbo, kKLayout);
      b_small = 2;
      b_big = static_cast<uint32_t>(p.bn_cta) * 128 / 16;
    }
    const uint32_t a_stage16 = p.a_stage_bytes >> 4, b_stage16 = p.b_stage_bytes >> 4;
    auto commit = [&](uint64_t* bar) {
      if constexpr (kPair)
        umma_commit_pair_multicast(smem_u32(bar), 0x3);  // both CTAs' barriers
      else
        umma_commit(smem_u32(bar));
    };
    for (int tl = 0; tl < my_tiles; ++tl) {
      const int E = chain_tile(p, unit + tl * grid).E;
      const int acc = tl % p.tacc;
      mbar_wait(smem_u32(&tempty[acc]), ((tl / p.tacc) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * p.acc_stride;
      for (int v = 0; v < E; ++v) {
        mbar_wait(smem_u32(&full[slot]), (phase >> slot) & 1u);  // consumer_wait
        phase ^= 1u << slot;
        tc_fence_after();
        const uint64_t ad = adesc0 + slot * a_stage16;
        const uint64_t bd = bdesc0 + slot * b_stage16;
        if (elect_one()) {
#pragma unroll
          for (int u = 0; u < kSteps; ++u) {
            const uint32_t a_off = BK >= 64 ? (u >> 2) * (kTileM * 128 / 16) + (u & 3) * 2 : u * 2;
            const uint32_t b_off = (u >> 2) * b_big + (u & 3) * b_small;
            if constexpr (kPair)
              umma_f16_ss_pair(d_tmem, ad + a_off, bd + b_off, p.idesc, (v > 0 || u > 0) ? 1u : 0u);
            else
              umma_f16_ss(d_tmem, ad + a_off, bd + b_off, p.idesc, (v > 0 || u > 0) ? 1u : 0u);
          }
          commit(&empty[slot]);  // consumer_release
        }
        __syncwarp();
        slot = (slot + 1 == p.sA) ? 0 : slot + 1;
      }
      if (elect_one()) commit(&tfull[acc]);  // accumulator ready
      __syncwarp();
    }
  } else if (warp >= 2) {
    // ======================= epilogue (warps 2-5) =======================
    const int q = warp & 3;
    const uint32_t stage_base = staging + (warp - 2) * p.stage_bufs * 4096;
    constexpr int kChunkCols = 128 / static_cast<int>(sizeof(OutT));
    const int nchunks = p.BN / kChunkCols;
    int buf = 0;
    for (int tl = 0; tl < my_tiles; ++tl) {
      const ChainTile ct = chain_tile(p, unit + tl * grid);
      const CUtensorMap* tcm = &maps.c[ct.p];
      const int acc = tl % p.tacc;
      mbar_wait(smem_u32(&tfull[acc]), (tl / p.tacc) & 1);
      tc_fence_after();
      const uint32_t t_addr = tmem_base + acc * p.acc_stride + (static_cast<uint32_t>(q * 32) << 16);
      for (int c = 0; c < nchunks; ++c) {
        uint32_t w[32];
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
            w[i] = pack2c<OutT>(r0[2 * i], r0[2 * i + 1]);
            w[16 + i] = pack2c<OutT>(r1[2 * i], r1[2 * i + 1]);
          }
        }
        if (c == nchunks - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (kPair)
              mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));  // the leader's barrier
            else
              mbar_arrive(smem_u32(&tempty[acc]));
          }
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
          tma_store_3d(tcm, sbuf, ct.nb * p.BN + c * kChunkCols,
                       ct.mb * kRows + static_cast<int>(rank) * kTileM + q * 32, 0);
          bulk_commit_group();
        }
        buf ^= p.stage_bufs - 1;
      }
      // publish this warp's part of the tile when a later GEMM reads it: the
      // stores must be complete in global memory before the release (the
      // epilogue would idle until the next accumulator anyway)
      if (ct.p + 1 < p.n && p.prob[ct.p + 1].dep) {
        if (lane == 0) {
          bulk_wait_group<0>();
          fence_proxy_async_global();
          red_release_add(p.counters + ct.p * p.max_mb + ct.mb, 1);
        }
        __syncwarp();
      }
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

template <typename OutT, int BK>
int launch_chain_typed(const ChainMaps& maps, const ChainKParams& kp, bool pair, int grid, int smem,
                       cudaStream_t st) {
  auto kern = pair ? alcop_chain_gemm_kernel<OutT, BK, true> : alcop_chain_gemm_kernel<OutT, BK, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_error(ALCOP_ERR_CUDA, "CudaError", cudaGetErrorString(e));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kChainThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;  // CTA pairs (cta_group 2)
  attr[1].val.clusterDim.x = pair ? 2 : 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pair ? 2 : 1;
  e = cudaLaunchKernelEx(&cfg, kern, maps, kp);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ALCOP_ERR_CUDA, "CudaError", cudaGetErrorString(e));
  return ALCOP_OK;
}

}  // namespace

int64_t chain_max_row_blocks(const alcop_chain* ch) {
  int64_t mb = 1;
  for (int i = 0; i < ch->n; ++i) mb = std::max<int64_t>(mb, (ch->desc[i].M + kTileM - 1) / kTileM);
  return mb;
}

int launch_chain(const alcop_chain& ch, const alcop_schedule& s, void* workspace, void* stream) {
  const int BN = static_cast<int>(s.tileN), BK = static_cast<int>(s.tileK);
  const alcop_gemm_desc& w0 = ch.desc[0];
  const CUtensorMapDataType dt =
      w0.in_dtype == ALCOP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const CUtensorMapDataType odt = w0.out_dtype == ALCOP_F32    ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                  : w0.out_dtype == ALCOP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                               : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const int ob = w0.out_dtype == ALCOP_F32 ? 4 : 2;
  const CUtensorMapSwizzle kswz = BK >= 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  const uint32_t kbox = BK >= 64 ? 64 : BK;
  const cuuint32_t es[3] = {1, 1, 1};
  ChainMaps maps;
  ChainKParams kp{};
  const bool pair = s.cta_group == 2;
  const int rows = kTileM * (pair ? 2 : 1);  // output rows per tile
  kp.n = ch.n;
  kp.BN = BN;
  kp.bn_cta = pair ? BN / 2 : BN;
  kp.sA = s.n_stage_smem_A;
  kp.tacc = s.n_stage_inner;
  kp.b_mn_major = w0.b_layout == ALCOP_B_KN ? 1 : 0;
  kp.idesc = ptx::make_idesc_f16(w0.in_dtype == ALCOP_BF16 ? 1u : 0u, kp.b_mn_major, static_cast<uint32_t>(rows), BN);
  kp.a_stage_bytes = static_cast<uint32_t>(kTileM * BK * 2);
  kp.b_stage_bytes = static_cast<uint32_t>(kp.bn_cta * BK * 2);
  kp.acc_stride = static_cast<uint32_t>(round_up_pow2_cols(BN));
  kp.tmem_cols = static_cast<uint32_t>(round_up_pow2_cols(kp.acc_stride * kp.tacc));
  kp.max_mb = static_cast<int32_t>(chain_max_row_blocks(&ch));
  kp.counters = static_cast<int32_t*>(workspace);
  int tiles = 0;
  for (int i = 0; i < ch.n; ++i) {
    const alcop_gemm_desc& w = ch.desc[i];
    const int64_t lda = w.lda ? w.lda : w.K;
    const int64_t ldb = w.ldb ? w.ldb : (w.b_layout == ALCOP_B_KN ? w.N : w.K);
    const int64_t ldc = w.ldc ? w.ldc : w.N;
    int rc;
    {
      const cuuint64_t dims[3] = {static_cast<cuuint64_t>(w.K), static_cast<cuuint64_t>(w.M), 1};
      const cuuint64_t str[2] = {static_cast<cuuint64_t>(lda * 2), static_cast<cuuint64_t>(lda * 2 * w.M)};
      const cuuint32_t box[3] = {kbox, kTileM, 1};
      rc = encode_tiled_map(&maps.a[i], dt, ch.A[i], 3, dims, str, box, es, kswz, "chain A");
    }
    if (rc) return rc;
    if (w.b_layout == ALCOP_B_KN) {
      const cuuint64_t dims[3] = {static_cast<cuuint64_t>(w.N), static_cast<cuuint64_t>(w.K), 1};
      const cuuint64_t str[2] = {static_cast<cuuint64_t>(ldb * 2), static_cast<cuuint64_t>(ldb * 2 * w.K)};
      const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(BK), 1};
      rc = encode_tiled_map(&maps.b[i], dt, ch.B[i], 3, dims, str, box, es, CU_TENSOR_MAP_SWIZZLE_128B, "chain B");
    } else {
      const cuuint64_t dims[3] = {static_cast<cuuint64_t>(w.K), static_cast<cuuint64_t>(w.N), 1};
      const cuuint64_t str[2] = {static_cast<cuuint64_t>(ldb * 2), static_cast<cuuint64_t>(ldb * 2 * w.N)};
      const cuuint32_t box[3] = {kbox, static_cast<cuuint32_t>(kp.bn_cta), 1};
      rc = encode_tiled_map(&maps.b[i], dt, ch.B[i], 3, dims, str, box, es, kswz, "chain B");
    }
    if (rc) return rc;
    {
      const cuuint64_t dims[3] = {static_cast<cuuint64_t>(w.N), static_cast<cuuint64_t>(w.M), 1};
      const cuuint64_t str[2] = {static_cast<cuuint64_t>(ldc * ob), static_cast<cuuint64_t>(ldc * ob * w.M)};
      const cuuint32_t box[3] = {static_cast<cuuint32_t>(128 / ob), 32, 1};
      rc = encode_tiled_map(&maps.c[i], odt, ch.C[i], 3, dims, str, box, es, CU_TENSOR_MAP_SWIZZLE_128B, "chain C");
    }
    if (rc) return rc;
    ChainProblem& pr = kp.prob[i];
    pr.num_m = static_cast<int32_t>((w.M + rows - 1) / rows);
    pr.num_n = static_cast<int32_t>((w.N + BN - 1) / BN);
    pr.E = static_cast<int32_t>((w.K + BK - 1) / BK);
    pr.tiles = pr.num_m * pr.num_n;
    pr.dep = ch.dep[i] ? 1 : 0;
    tiles += pr.tiles;
  }
  kp.total_tiles = tiles;
  // work units: CTAs, or CTA pairs
  int grid = (s.num_ctas > 0 ? s.num_ctas : device_sm_count()) / (pair ? 2 : 1);
  if (grid <= 0) return set_error(ALCOP_ERR_CUDA, "CudaError", "no CUDA device");
  if (grid > tiles) grid = tiles;
  for (int i = 0, begin = 0; i < ch.n; ++i) {  // first global tile of each problem (chain_tile)
    kp.prob[i].key0 = begin;
    begin += kp.prob[i].tiles;
  }
  kp.max_key = tiles;
  alcop_gemm_desc wsm = w0;
  const int smem = static_cast<int>(gemm_smem_bytes_epi(wsm, s, 4));
  kp.stage_bufs = gemm_staging_bufs_epi(wsm, s, 4);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int ctas = grid * (pair ? 2 : 1);
  cudaError_t e = cudaMemsetAsync(workspace, 0, sizeof(int32_t) * kp.max_mb * ch.n, st);
  if (e != cudaSuccess) return set_error(ALCOP_ERR_CUDA, "CudaError", cudaGetErrorString(e));
  switch (w0.out_dtype * 4 + (BK == 32 ? 0 : BK == 64 ? 1 : 2)) {
    case ALCOP_F32 * 4 + 0: return launch_chain_typed<float, 32>(maps, kp, pair, ctas, smem, st);
    case ALCOP_F32 * 4 + 1: return launch_chain_typed<float, 64>(maps, kp, pair, ctas, smem, st);
    case ALCOP_F32 * 4 + 2: return launch_chain_typed<float, 128>(maps, kp, pair, ctas, smem, st);
    case ALCOP_BF16 * 4 + 0: return launch_chain_typed<__nv_bfloat16, 32>(maps, kp, pair, ctas, smem, st);
    case ALCOP_BF16 * 4 + 1: return launch_chain_typed<__nv_bfloat16, 64>(maps, kp, pair, ctas, smem, st);
    case ALCOP_BF16 * 4 + 2: return launch_chain_typed<__nv_bfloat16, 128>(maps, kp, pair, ctas, smem, st);
    case ALCOP_F16 * 4 + 0: return launch_chain_typed<__half, 32>(maps, kp, pair, ctas, smem, st);
    case ALCOP_F16 * 4 + 1: return launch_chain_typed<__half, 64>(maps, kp, pair, ctas, smem, st);
    case ALCOP_F16 * 4 + 2: return launch_chain_typed<__half, 128>(maps, kp, pair, ctas, smem, st);
  }
  return set_error(ALCOP_ERR_CONFIG, "BadDtype", "unsupported output dtype");
}

}  // namespace alcop
