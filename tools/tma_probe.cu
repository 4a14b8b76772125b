// tma_probe.cu — TMA load throughput microbenchmark (measurement tool, not product).
//
// Question it answers: what bounds the L2 -> SM operand fill of the pipelined
// GEMM on B200 — per-SM TMA issue/ingress, or a chip-wide L2 (LTS) cap — and
// is that cap counted in bytes or in box rows (requests)?  Does unicast of
// the same tile to several SMs deduplicate, and does TMA multicast within a
// cluster reduce the cost?
//
// Each CTA runs a producer warp that streams "chunks" (nbox TMA boxes of
// box_rows x box_w bf16 elements) into an s-slot ring, and a consumer warp
// that waits on full[] and releases empty[] immediately (no compute).  The
// data (32 MB bf16 matrix) is L2-resident after warm-up.  CTAs in a share
// group read identical coordinates at the same time; with multicast, a
// cluster of c CTAs shares each chunk, each CTA loads 1/c of the boxes and
// multicasts them to all c CTAs.
//
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lcuda tools/tma_probe.cu -o tools/_bin/tma_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2210_16691_b200/csrc/sm100_ptx.cuh"

using namespace alcop::ptx;

struct Params {
  int box_rows, box_w, nbox, stages, chunks, share, csize, rows, cols, spin, mc;
  long long* cycles;
  long long* trace;  // [3][64] per-chunk clocks of CTA 0 (nullptr = off)
};

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

// non-blocking probe of the phase (no suspend hint): pure spin
__device__ __forceinline__ uint32_t mbar_test_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok;
}
__device__ __forceinline__ void wait_phase(uint32_t bar, uint32_t parity, int spin) {
  if (spin) {
    while (!mbar_test_wait(bar, parity)) {
    }
  } else {
    mbar_wait(bar, parity);
  }
}

__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap tm, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t box_bytes = p.box_rows * p.box_w * 2;
  const uint32_t chunk_bytes = box_bytes * p.nbox;
  const uint32_t ring = smem_u32(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * chunk_bytes);
  uint64_t* empty = full + p.stages;
  const int warp = threadIdx.x >> 5;
  const uint32_t crank = p.csize > 1 ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < p.stages; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), p.csize);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (p.csize > 1) cluster_sync();
  const int group = blockIdx.x / p.share;
  const int nrb = p.rows / (p.box_rows * p.nbox);
  const int ncb = p.cols / p.box_w;
  const int rb = group % nrb;
  long long t0 = clock64();
  if (warp == 0) {
    if (elect_one()) {
      uint32_t phase = 0;
      int slot = 0;
      for (int i = 0; i < p.chunks; ++i) {
        if (p.trace && blockIdx.x == 0 && i < 64) p.trace[192 + i] = clock64() - t0;
        if (!(p.spin == 2 && i < p.stages)) wait_phase(smem_u32(&empty[slot]), ((phase >> slot) & 1u) ^ 1u, p.spin == 1);
        phase ^= 1u << slot;
        if (p.trace && blockIdx.x == 0 && i < 64) p.trace[i] = clock64() - t0;
        const uint32_t fb = smem_u32(&full[slot]);
        mbar_arrive_expect_tx(fb, chunk_bytes);
        if (p.trace && blockIdx.x == 0 && i < 64) p.trace[256 + i] = clock64() - t0;
        const int cb = (i + group) % ncb;
        if (p.csize > 1 && p.mc) {
          for (int b = crank; b < p.nbox; b += p.csize)
            tma_load_2d_mc(ring + slot * chunk_bytes + b * box_bytes, &tm, fb, cb * p.box_w,
                           (rb * p.nbox + b) * p.box_rows, static_cast<uint16_t>((1u << p.csize) - 1));
        } else {
          for (int b = 0; b < p.nbox; ++b)
            tma_load_2d(ring + slot * chunk_bytes + b * box_bytes, &tm, fb, cb * p.box_w,
                        (rb * p.nbox + b) * p.box_rows);
        }
        if (p.trace && blockIdx.x == 0 && i < 64) p.trace[64 + i] = clock64() - t0;
        slot = slot + 1 == p.stages ? 0 : slot + 1;
      }
    }
    __syncwarp();
  } else {
    if (elect_one()) {
      uint32_t phase = 0;
      int slot = 0;
      for (int i = 0; i < p.chunks; ++i) {
        wait_phase(smem_u32(&full[slot]), (phase >> slot) & 1u, p.spin == 1);
        phase ^= 1u << slot;
        if (p.trace && blockIdx.x == 0 && i < 64) p.trace[128 + i] = clock64() - t0;
        if (p.csize > 1) {
          for (uint32_t r = 0; r < static_cast<uint32_t>(p.csize); ++r)
            asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                             mapa_shared(smem_u32(&empty[slot]), r))
                         : "memory");
        } else {
          mbar_arrive(smem_u32(&empty[slot]));
        }
        slot = slot + 1 == p.stages ? 0 : slot + 1;
      }
    }
    __syncwarp();
  }
  __syncthreads();
  if (p.csize > 1) cluster_sync();
  if (threadIdx.x == 0) p.cycles[blockIdx.x] = clock64() - t0;
}


// burst: thread 0 issues nb boxes back-to-back (one mbarrier each, or all on
// barrier 0 when one_bar), then records when each barrier completes
__global__ void __launch_bounds__(32, 1) probe_burst(const __grid_constant__ CUtensorMap tm, int nb, int box_rows,
                                                     int one_bar, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t box_bytes = box_rows * 64 * 2;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + nb * box_bytes);
  if (threadIdx.x != 0) return;
  for (int i = 0; i < nb; ++i) mbar_init(smem_u32(&bars[i]), 1);
  fence_barrier_init();
  long long t0 = clock64();
  if (one_bar) mbar_arrive_expect_tx(smem_u32(&bars[0]), box_bytes * nb);
  for (int i = 0; i < nb; ++i) {
    const uint32_t b = smem_u32(&bars[one_bar ? 0 : i]);
    if (!one_bar) mbar_arrive_expect_tx(b, box_bytes);
    tma_load_2d(smem_u32(smem) + i * box_bytes, &tm, b, (i % 32) * 64, (blockIdx.x * 8 + i / 32) * box_rows);
  }
  long long t1 = clock64();
  for (int i = 0; i < (one_bar ? 1 : nb); ++i) {
    while (!mbar_try_wait(smem_u32(&bars[i]), 0)) {
    }
    out[blockIdx.x * 64 + 1 + i] = clock64() - t0;
  }
  out[blockIdx.x * 64] = t1 - t0;
}


// primitive costs: one thread times N iterations of a primitive on already
// completed / fresh mbarriers (clk per iteration)
__global__ void __launch_bounds__(128, 1) probe_prims(long long* out, int n) {
  __shared__ __align__(8) uint64_t bars[16];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(smem_u32(&bars[i]), 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // (0) try_wait on a phase that is already complete (parity 1 of a fresh barrier)
    long long t0 = clock64();
    uint32_t acc = 0;
    for (int i = 0; i < n; ++i) acc += mbar_try_wait(smem_u32(&bars[i & 15]), 1);
    long long t1 = clock64();
    out[0] = (t1 - t0) / n;
    // (1) mbarrier.arrive (count 1 -> phase flips each time)
    t0 = clock64();
    for (int i = 0; i < n; ++i) mbar_arrive(smem_u32(&bars[i & 15]));
    t1 = clock64();
    out[1] = (t1 - t0) / n;
    // (2) arrive.expect_tx 0 bytes
    t0 = clock64();
    for (int i = 0; i < n; ++i) mbar_arrive_expect_tx(smem_u32(&bars[i & 15]), 0);
    t1 = clock64();
    out[2] = (t1 - t0) / n;
    // (3) arrive + try_wait of the phase it just completed (round trip through the barrier)
    uint32_t ph = 0;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
      mbar_arrive(smem_u32(&bars[0]));
      while (!mbar_try_wait(smem_u32(&bars[0]), ph)) {
      }
      ph ^= 1;
    }
    t1 = clock64();
    out[3] = (t1 - t0) / n;
    out[8] = acc;
  }
  __syncthreads();
  if (warp == 1 && (threadIdx.x & 31) == 0) {
    // (4) tcgen05.commit with nothing in flight -> arrive on a barrier, then wait for it
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bars[1]))
                   : "memory");
      while (!mbar_try_wait(smem_u32(&bars[1]), ph)) {
      }
      ph ^= 1;
    }
    long long t1 = clock64();
    out[4] = (t1 - t0) / n;
    // (6) fence.proxy.async.shared::cta alone
    t0 = clock64();
    for (int i = 0; i < n; ++i) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    t1 = clock64();
    out[6] = (t1 - t0) / n;
    // (7) 8 x st.shared.v4 (one 4 KB staging chunk per warp) + fence.proxy.async
    {
      extern __shared__ uint8_t dyn[];
      const uint32_t base = smem_u32(dyn);
      const int lane = threadIdx.x & 31;
      t0 = clock64();
      for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          st_shared_v4(base + lane * 128 + ((j ^ (lane & 7)) << 4), i, j, i + j, i - j);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      t1 = clock64();
      out[7] = (t1 - t0) / n;
    }
    // (5) tcgen05.commit issue cost alone (no wait), 16 barriers round robin
    t0 = clock64();
    for (int i = 0; i < n; ++i)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bars[2 + (i & 7)]))
                   : "memory");
    t1 = clock64();
    out[5] = (t1 - t0) / n;
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tslot), "r"(32));
  }
}


// issue-rate probe: `nw` warps each issue `per` TMA boxes (16 KB) back to
// back on their own barrier; clk from start to the last issue, per warp
__global__ void __launch_bounds__(128, 1) probe_issue(const __grid_constant__ CUtensorMap tm, int nw, int per,
                                                     long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 12 * 16384);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&bars[i]), 1);
    fence_barrier_init();
  }
  __syncthreads();
  long long t0 = clock64();
  if (warp < nw && (threadIdx.x & 31) == 0) {
    const uint32_t b = smem_u32(&bars[warp]);
    mbar_arrive_expect_tx(b, 16384 * per);
    for (int i = 0; i < per; ++i)
      tma_load_2d(smem_u32(smem) + ((warp * per + i) % 12) * 16384, &tm, b, (i % 32) * 64, (warp * 8 + i / 32) * 128);
    out[warp] = clock64() - t0;
    while (!mbar_try_wait(b, 0)) {
    }
    out[4 + warp] = clock64() - t0;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
}

int main(int argc, char** argv) {
  const int rows = 8192, cols = 2048;
  void* X;
  cudaMalloc(&X, size_t(rows) * cols * 2);
  cudaMemset(X, 1, size_t(rows) * cols * 2);
  long long* cyc;
  cudaMalloc(&cyc, 1024 * sizeof(long long));
  auto enc = encode_fn();
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  // configs: {grid, box_rows, box_w, nbox, stages, share, csize}
  // configs: {grid, box_rows, box_w, nbox, stages, share, csize, spin}
  // configs: {grid, box_rows, box_w, nbox, stages, share, csize, spin, multicast}
  std::vector<std::vector<int>> cfgs = {
  };
  printf("grid box_rows box_w nbox stages share csize | chunkKB  GB/s_total  B/clk_chip  B/clk_SM  rows/clk_chip  clk/chunk\n");
  for (auto& c : cfgs) {
    Params p{};
    int grid = c[0];
    p.box_rows = c[1];
    p.box_w = c[2];
    p.nbox = c[3];
    p.stages = c[4];
    p.share = c[5];
    p.csize = c[6];
    p.spin = c[7];
    p.mc = c[8];
    p.rows = rows;
    p.cols = cols;
    p.chunks = 4000;
    p.cycles = cyc;
    p.trace = cyc + 256;
    CUtensorMap tm;
    cuuint64_t dims[2] = {uint64_t(cols), uint64_t(rows)};
    cuuint64_t strides[1] = {uint64_t(cols) * 2};
    cuuint32_t box[2] = {uint32_t(p.box_w), uint32_t(p.box_rows)};
    cuuint32_t es[2] = {1, 1};
    CUtensorMapSwizzle swz = p.box_w == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                             : p.box_w == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                             : CU_TENSOR_MAP_SWIZZLE_32B;
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, X, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed %d\n", r);
      continue;
    }
    size_t chunk_bytes = size_t(p.box_rows) * p.box_w * 2 * p.nbox;
    size_t smem = 1024 + p.stages * chunk_bytes + 16 * p.stages;
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(64);
    lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = p.csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaError_t le = cudaSuccess;
    for (int w = 0; w < 2; ++w) le = cudaLaunchKernelEx(&lc, probe, tm, p);
    if (le != cudaSuccess) { printf("launch failed: %s\n", cudaGetErrorString(le)); cudaGetLastError(); continue; }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 3;
    for (int w = 0; w < reps; ++w) cudaLaunchKernelEx(&lc, probe, tm, p);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    if (err != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(err));
      return 1;
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> hc(grid);
    cudaMemcpy(hc.data(), cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    long long cmax = 0;
    for (auto v : hc) cmax = v > cmax ? v : cmax;
    double bytes = double(chunk_bytes) * p.chunks * grid;
    double sec = ms * 1e-3 / reps;
    double rows_total = double(p.box_rows) * p.nbox * p.chunks * grid;
    printf("%4d %8d %5d %4d %6d %5d %5d | %7.1f  %10.1f  %10.1f  %8.1f  %12.2f  %9.1f\n", grid, p.box_rows,
           p.box_w, p.nbox, p.stages, p.share, p.csize, chunk_bytes / 1024.0, bytes / sec / 1e9, bytes / cmax,
           bytes / cmax / grid, rows_total / cmax, double(cmax) / p.chunks);
    std::vector<long long> ht(320);
    cudaMemcpy(ht.data(), cyc + 256, 320 * sizeof(long long), cudaMemcpyDeviceToHost);
    const char* nm[5] = {"prod acquired", "prod issued  ", "cons full ok ", "prod pre-wait", "prod expect  "};
    for (int k : {3, 0, 4, 1, 2}) {
      printf("   %s:", nm[k]);
      for (int i = 0; i < 24; ++i) printf(" %lld", ht[k * 64 + i]);
      printf("\n");
    }
  }

  {
    probe_prims<<<1, 128, 8192>>>(cyc, 1024);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> h(16);
    cudaMemcpy(h.data(), cyc, 16 * sizeof(long long), cudaMemcpyDeviceToHost);
    printf("prims (clk/iter): try_wait(done) %lld  arrive %lld  arrive.expect_tx %lld  arrive+wait %lld  "
           "tcgen05.commit+wait %lld  tcgen05.commit issue %lld  fence.proxy.async %lld  8xst.shared.v4+fence %lld  [%s]\n", h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7],
           cudaGetErrorString(e));
  }
  {
    CUtensorMap tm;
    cuuint64_t dims[2] = {uint64_t(cols), uint64_t(rows)};
    cuuint64_t strides[1] = {uint64_t(cols) * 2};
    cuuint32_t box[2] = {64u, 128u};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(probe_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int nw : {1, 2, 4}) {
      const int per = 12 / nw;
      for (int w = 0; w < 3; ++w) probe_issue<<<1, 128, 1024 + 12 * 16384 + 64>>>(tm, nw, per, cyc);
      cudaDeviceSynchronize();
      std::vector<long long> h(8);
      cudaMemcpy(h.data(), cyc, 8 * sizeof(long long), cudaMemcpyDeviceToHost);
      printf("issue: %d warps x %d boxes: last issue at", nw, per);
      for (int i = 0; i < nw; ++i) printf(" %lld", h[i]);
      printf(" clk; all landed at");
      for (int i = 0; i < nw; ++i) printf(" %lld", h[4 + i]);
      printf("\n");
    }
  }
  // ---- burst completion timelines (grid 1 and 148): nb 16 KB boxes (128 rows x 128 B)
  cudaFuncSetAttribute(probe_burst, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int g : {1, 148}) {
    for (int one : {0, 1}) {
      for (int rowsb : {128, 64}) {
        int nb = rowsb == 128 ? 10 : 20;
        CUtensorMap tm;
        cuuint64_t dims[2] = {uint64_t(cols), uint64_t(rows)};
        cuuint64_t strides[1] = {uint64_t(cols) * 2};
        cuuint32_t box[2] = {64u, uint32_t(rowsb)};
        cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        size_t smem = 1024 + nb * rowsb * 128 + 8 * nb;
        for (int w = 0; w < 3; ++w) probe_burst<<<g, 32, smem>>>(tm, nb, rowsb, one, cyc);
        cudaDeviceSynchronize();
        std::vector<long long> h(64);
        cudaMemcpy(h.data(), cyc, 64 * sizeof(long long), cudaMemcpyDeviceToHost);
        printf("burst grid %3d one_bar %d box_rows %3d nb %2d: issue %lld clk; completions:", g, one, rowsb, nb, h[0]);
        for (int i = 0; i < (one ? 1 : nb); ++i) printf(" %lld", h[1 + i]);
        printf("\n");
      }
    }
  }
  return 0;
}
