// sharded.cpp — the multi-GPU driver behind the C ABI.
//
// The reference executes the parallel loops of the lowered nest (b, i0, j0)
// one after another (interp.hpp:330-338); on a B200 box those units become
// devices.  Each shard is a contiguous run of rows / batch entries / images
// (granule multiples), its operands already on its device (B or the filter
// replicated), and one host thread per shard enqueues its launch: the host
// work of encoding tensor maps and launching overlaps across devices, and no
// collective touches the compute path.  Errors from a worker thread are
// carried back to the caller's thread-local alcop_last_error().
#include <cuda_runtime.h>

#include <string>
#include <thread>
#include <vector>

#include "alcop_internal.h"

namespace alcop {
namespace {

struct ShardResult {
  int rc = ALCOP_OK;
  std::string error;
};

// contiguous split in granule multiples, earlier shards take the remainder
void split(int64_t total, int32_t rank, int32_t world, int64_t granule, int64_t* start, int64_t* count) {
  const int64_t granules = (total + granule - 1) / granule;
  const int64_t base = granules / world, extra = granules % world;
  const int64_t first = rank * base + (rank < extra ? rank : extra);
  const int64_t n = base + (rank < extra ? 1 : 0);
  const int64_t lo = std::min(total, first * granule), hi = std::min(total, (first + n) * granule);
  *start = lo;
  *count = hi - lo;
}

// Runs fn(shard index) on one thread per shard; the first failure (in shard
// order) becomes the caller's error.
template <typename Fn>
int for_each_shard(int32_t nshards, Fn&& fn) {
  std::vector<ShardResult> res(nshards);
  std::vector<std::thread> pool;
  pool.reserve(nshards);
  for (int32_t i = 0; i < nshards; ++i)
    pool.emplace_back([&, i] {
      res[i].rc = fn(i);
      if (res[i].rc != ALCOP_OK) res[i].error = alcop_last_error();
    });
  for (auto& t : pool) t.join();
  for (int32_t i = 0; i < nshards; ++i)
    if (res[i].rc != ALCOP_OK) {
      const std::string& e = res[i].error;
      const size_t colon = e.find(':');
      return set_error(res[i].rc, colon == std::string::npos ? "ShardError" : e.substr(0, colon),
                       "shard " + std::to_string(i) + ": " + (colon == std::string::npos ? e : e.substr(colon + 2)));
    }
  return ALCOP_OK;
}

int check_shards(int32_t nshards, const alcop_shard* shards) {
  if (nshards < 1 || !shards) return set_error(ALCOP_ERR_CONFIG, "BadShards", "need nshards >= 1 shard records");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
    cudaGetLastError();
    ndev = 0;
  }
  for (int32_t i = 0; i < nshards; ++i)
    if (shards[i].device < 0 || shards[i].device >= ndev)
      return set_error(ALCOP_ERR_CUDA, "CudaError",
                       "shard " + std::to_string(i) + " names device " + std::to_string(shards[i].device) + " of " +
                           std::to_string(ndev));
  return ALCOP_OK;
}

}  // namespace
}  // namespace alcop

using namespace alcop;

extern "C" int alcop_shard_range(int64_t total, int32_t rank, int32_t world, int64_t granule, int64_t* start,
                                 int64_t* count) {
  if (!start || !count) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument");
  if (total < 0 || world < 1 || rank < 0 || rank >= world || granule < 1)
    return set_error(ALCOP_ERR_CONFIG, "BadShards", "need total >= 0, 0 <= rank < world, granule >= 1");
  clear_error();
  split(total, rank, world, granule, start, count);
  return ALCOP_OK;
}

extern "C" int alcop_gemm_sharded(const alcop_gemm_desc* w, const alcop_schedule* s, int32_t nshards,
                                  const alcop_shard* shards, int64_t granule) {
  if (!w) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL descriptor");
  clear_error();
  if (w->lda || w->ldb || w->ldc || w->stride_a || w->stride_b || w->stride_c)
    return set_error(ALCOP_ERR_CONFIG, "BadWorkload", "sharded entry point takes packed tensors only");
  if (granule < 1) return set_error(ALCOP_ERR_CONFIG, "BadShards", "granule must be >= 1");
  int rc = check_shards(nshards, shards);
  if (rc) return rc;
  const bool by_batch = w->batch > 1;
  const int64_t total = by_batch ? w->batch : w->M;
  return for_each_shard(nshards, [&](int32_t i) -> int {
    clear_error();
    int64_t start = 0, count = 0;
    split(total, i, nshards, granule, &start, &count);
    if (count == 0) return ALCOP_OK;
    const alcop_shard& sh = shards[i];
    if (!sh.A || !sh.B || !sh.C) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL operand");
    if (cudaSetDevice(sh.device) != cudaSuccess) return set_error(ALCOP_ERR_CUDA, "CudaError", "cudaSetDevice");
    alcop_gemm_desc sub = *w;
    if (by_batch)
      sub.batch = count;
    else
      sub.M = count;
    alcop_schedule pick;
    if (!s) {
      alcop_hw hw;
      alcop_hw_default_b200(&hw);
      const int prc = alcop_choose_schedule(&sub, &hw, &pick);
      if (prc) return prc;
    }
    return alcop_gemm(&sub, s ? s : &pick, sh.A, sh.B, sh.C, sh.stream);
  });
}

extern "C" int alcop_conv2d_sharded(const alcop_conv_desc* d, const alcop_schedule* s, int32_t nshards,
                                    const alcop_shard* shards) {
  if (!d || !s) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument");
  clear_error();
  int rc = check_shards(nshards, shards);
  if (rc) return rc;
  return for_each_shard(nshards, [&](int32_t i) -> int {
    clear_error();
    int64_t start = 0, count = 0;
    split(d->N, i, nshards, 1, &start, &count);
    if (count == 0) return ALCOP_OK;
    const alcop_shard& sh = shards[i];
    if (!sh.A || !sh.B || !sh.C) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL operand");
    if (cudaSetDevice(sh.device) != cudaSuccess) return set_error(ALCOP_ERR_CUDA, "CudaError", "cudaSetDevice");
    alcop_conv_desc sub = *d;
    sub.N = count;
    return alcop_conv2d(&sub, s, sh.A, sh.B, sh.C, sh.stream);
  });
}
