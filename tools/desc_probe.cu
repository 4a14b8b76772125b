// desc_probe.cu — measurement/semantics probe (not product code): what does
// tcgen05.mma read when a 128B-swizzled K-major A operand's descriptor start
// address is moved by whole 128-byte rows (s rows, s not a multiple of 8),
// with the descriptor's base-offset field = bo?  A window of 144 rows x 64
// bf16 is written into shared memory in the TMA 128B-swizzle pattern
// (16-byte chunk c of row y at chunk c ^ (y & 7), base 1024-aligned), and
// D = A[s : s+128] x B^T (M=128, N=64, K=64) is computed with the shifted
// descriptor.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -shared
// -Xcompiler -fPIC -o tools/_bin/libdesc_probe.so tools/desc_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>

#include "../paper_2210_16691_b200/csrc/sm100_ptx.cuh"

using namespace alcop::ptx;

__global__ void __launch_bounds__(128, 1) desc_probe_kernel(const uint16_t* A, const uint16_t* B, float* D, int shift,
                                                            int bo) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sA = smem_u32(smem);
  const uint32_t sB = sA + 144 * 128;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 144 * 128 + 64 * 128);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // A: 144 rows x 8 chunks of 16 B; B: 64 rows x 8 chunks
  for (int i = tid; i < 144 * 8; i += 128) {
    const int y = i >> 3, c = i & 7;
    const uint4 v = reinterpret_cast<const uint4*>(A)[y * 8 + c];
    const uint32_t dst = sA + y * 128 + ((c ^ (y & 7)) << 4);
    st_shared_v4(dst, v.x, v.y, v.z, v.w);
  }
  for (int i = tid; i < 64 * 8; i += 128) {
    const int y = i >> 3, c = i & 7;
    const uint4 v = reinterpret_cast<const uint4*>(B)[y * 8 + c];
    st_shared_v4(sB + y * 128 + ((c ^ (y & 7)) << 4), v.x, v.y, v.z, v.w);
  }
  fence_proxy_async_smem();
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(smem_u32(bar), 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(smem_u32(tslot), 64);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 0 && elect_one()) {
    const uint32_t idesc = make_idesc_f16(1u, 0u, 128, 64);
    for (int u = 0; u < 4; ++u) {
      uint64_t ad = make_smem_desc(sA + shift * 128 + u * 32, 16, 1024, kLayoutSW128);
      ad |= static_cast<uint64_t>(bo & 7) << 49;
      const uint64_t bd = make_smem_desc(sB + u * 32, 16, 1024, kLayoutSW128);
      umma_f16_ss(tmem, ad, bd, idesc, u > 0 ? 1u : 0u);
    }
    umma_commit(smem_u32(bar));
  }
  __syncwarp();
  mbar_wait(smem_u32(bar), 0);
  tc_fence_after();
  uint32_t r0[32], r1[32];
  const uint32_t t = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  tmem_ld_32x32b_x32(t, r0);
  tmem_ld_32x32b_x32(t + 32, r1);
  tmem_wait_ld();
  const int row = warp * 32 + lane;
  for (int j = 0; j < 32; ++j) {
    D[row * 64 + j] = __uint_as_float(r0[j]);
    D[row * 64 + 32 + j] = __uint_as_float(r1[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 64);
}

extern "C" int desc_probe(const void* A, const void* B, void* D, int shift, int bo) {
  const int smem = 1024 + 144 * 128 + 64 * 128 + 64;
  cudaFuncSetAttribute(desc_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  desc_probe_kernel<<<1, 128, smem>>>(static_cast<const uint16_t*>(A), static_cast<const uint16_t*>(B),
                                       static_cast<float*>(D), shift, bo);
  return static_cast<int>(cudaDeviceSynchronize());
}
