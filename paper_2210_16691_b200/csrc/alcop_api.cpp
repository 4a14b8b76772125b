// alcop_api.cpp — the C-ABI front end: error reporting, schedule
// validation (the params_valid analogue, perf_model.hpp:129-142, plus the
// pass's LookaheadExceedsOuter rule, pipeline_pass.hpp:305-313), and the
// compute entry points.  No exception crosses the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "alcop_internal.h"

namespace alcop {

namespace {
thread_local std::string g_last_error;
}

struct HostPipe {
  static constexpr int kBlocks = 8;
  bool ready = false;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_start = nullptr, ev_done = nullptr, ev_in[kBlocks] = {}, ev_out[kBlocks] = {};
  // the previous call on this pipe: its kernels' completion (recorded on the
  // caller's stream after its last block) and the host range its D2H writes
  cudaEvent_t ev_kernels = nullptr;
  bool have_prev = false;
  const char* prev_c = nullptr;
  int64_t prev_c_bytes = 0;
  ~HostPipe() {
    if (!ready) return;
    // errors ignored: at process exit the runtime may already be unloading
    for (cudaEvent_t ev : ev_in) cudaEventDestroy(ev);
    for (cudaEvent_t ev : ev_out) cudaEventDestroy(ev);
    cudaEventDestroy(ev_start);
    cudaEventDestroy(ev_done);
    cudaEventDestroy(ev_kernels);
    cudaStreamDestroy(h2d);
    cudaStreamDestroy(d2h);
  }
};

// Smallest A row block the host-buffer pipeline streams (bytes; 0: always 8
// blocks).  A lone synchronous call needs the row-block pipeline to overlap
// its own H2D, MMA and D2H; back-to-back async calls already overlap call
// k+1's H2D with call k's D2H, and there every extra copy costs PCIe rate to
// per-copy setup (BERT-layer e2e step: 8 blocks 1.96 ms, >= 8 MB blocks
// 1.60 ms; tools/e2e_probe.py).  ALCOP_HOST_BLOCK_BYTES overrides both.
int64_t host_block_bytes(bool sync) {
  static const int64_t env = [] {
    const char* e = std::getenv("ALCOP_HOST_BLOCK_BYTES");
    return e ? std::atoll(e) : int64_t(-1);
  }();
  if (env >= 0) return env;
  return sync ? 0 : int64_t(8) << 20;
}

// Copy streams + events of the pipelined host-buffer GEMM, one set per host
// thread and device (the entry point is synchronous, so a thread never has
// two calls in flight on the same set).
HostPipe* host_pipe() {
  thread_local HostPipe pipes[16];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
  HostPipe& hp = pipes[dev];
  if (!hp.ready) {
    bool ok = cudaStreamCreateWithFlags(&hp.h2d, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&hp.d2h, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&hp.ev_start, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&hp.ev_done, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&hp.ev_kernels, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; i < HostPipe::kBlocks && ok; ++i)
      ok = cudaEventCreateWithFlags(&hp.ev_in[i], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&hp.ev_out[i], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) return nullptr;
    hp.ready = true;
  }
  return &hp;
}

int set_error(int code, const std::string& tag, const std::string& msg) {
  g_last_error = tag + ": " + msg;
  return code;
}
void clear_error() { g_last_error.clear(); }

int64_t round_up_pow2_cols(int64_t cols) {
  int64_t c = 32;
  while (c < cols) c <<= 1;
  return c;
}

static int64_t smem_base_cols(const alcop_schedule& s, int64_t b_cols) {
  const int64_t a_stage = kTileM * s.tileK * 2;  // per CTA: 128 rows of A
  const int64_t b_stage = b_cols * s.tileK * 2;
  const int64_t bars = 8 * (3 * s.n_stage_smem_A + 2 * s.n_stage_smem_B + 4) + 16;  // + ready[] (pre-op)
  return 1024 /* alignment slack */ + s.n_stage_smem_A * a_stage + s.n_stage_smem_B * b_stage + bars;
}

// A CTA pair with B[K,N] and 96-column halves (tileN 192) stages each half as
// two 128B-swizzled 64-column atoms (over-fetching 32 columns; gemm_sm100.cu
// b_pad) when that still fits with one epilogue staging buffer per warp, else
// as three 64B-swizzled 32-column atoms (the 7th stage of 256x192 fits only so).
bool pair_b_pad(const alcop_gemm_desc& w, const alcop_schedule& s) {
  const int64_t cg = s.cta_group == 2 ? 2 : 1;
  const int64_t half = s.tileN / cg;
  if (!(cg == 2 && w.b_layout == ALCOP_B_KN && half % 64 != 0)) return false;
  return smem_base_cols(s, (half + 63) / 64 * 64) + 4 * 32 * 128 <= kMaxSmemBytes;
}

static int64_t gemm_smem_base(const alcop_gemm_desc& w, const alcop_schedule& s) {
  const int64_t cg = s.cta_group == 2 ? 2 : 1;
  const int64_t half = s.tileN / cg;  // B columns per CTA
  return smem_base_cols(s, pair_b_pad(w, s) ? (half + 63) / 64 * 64 : half);
}

// Epilogue warps: 8 (two per TMEM lane quarter) when a tile's main loop is at
// most two chunks and the tile has at least two output column chunks — the
// drain then sets the per-tile time (attention QK^T, K = 64); else 4.
int32_t gemm_epi_warps(const alcop_gemm_desc& w, const alcop_schedule& s) {
  const int64_t E = (w.K + s.tileK - 1) / s.tileK;
  const int64_t chunk_cols = w.out_dtype == ALCOP_F32 ? 32 : 64;
  const bool eligible = s.cta_group == 1 && !w.pre_op && s.n_stage_smem_A == s.n_stage_smem_B &&
                        s.mode == ALCOP_MODE_FUSED;
  // only where one staging buffer per warp fits: never needs more shared
  // memory than 4 warps would (4 x 2 buffers), so validity does not change
  return (eligible && E <= 2 && s.tileN / chunk_cols >= 2 && gemm_smem_base(w, s) + 8 * 32 * 128 <= kMaxSmemBytes)
             ? 8
             : 4;
}

// Epilogue TMA-store staging: two 4 KB buffers per epilogue warp (the store of
// one chunk overlaps the TMEM read of the next) when they fit beside the ring,
// else one — shared memory goes to pipeline stages first (one more stage of
// lookahead is worth more than the store overlap).
int32_t gemm_staging_bufs_epi(const alcop_gemm_desc& w, const alcop_schedule& s, int32_t epi) {
  return gemm_smem_base(w, s) + epi * 2 * 32 * 128 <= kMaxSmemBytes ? 2 : 1;
}
int64_t gemm_smem_bytes_epi(const alcop_gemm_desc& w, const alcop_schedule& s, int32_t epi) {
  return gemm_smem_base(w, s) + epi * gemm_staging_bufs_epi(w, s, epi) * 32 * 128;
}
int32_t gemm_staging_bufs(const alcop_gemm_desc& w, const alcop_schedule& s) {
  return gemm_staging_bufs_epi(w, s, gemm_epi_warps(w, s));
}
int64_t gemm_smem_bytes(const alcop_gemm_desc& w, const alcop_schedule& s) {
  return gemm_smem_bytes_epi(w, s, gemm_epi_warps(w, s));
}

static int dtype_bytes(int32_t dt) { return dt == ALCOP_F32 ? 4 : 2; }

int validate_gemm(const alcop_gemm_desc& w, const alcop_schedule& s) {
  if (w.M < 1 || w.N < 1 || w.K < 1 || w.batch < 1)
    return set_error(ALCOP_ERR_CONFIG, "BadWorkload", "M, N, K and batch must be >= 1");
  if (w.M > INT32_MAX || w.N > INT32_MAX || w.K > INT32_MAX)
    return set_error(ALCOP_ERR_CONFIG, "BadWorkload", "M, N, K must fit in int32");
  if (w.in_dtype != ALCOP_F16 && w.in_dtype != ALCOP_BF16)
    return set_error(ALCOP_ERR_CONFIG, "BadDtype", "input dtype must be F16 or BF16 (tcgen05 kind::f16)");
  if (w.out_dtype != ALCOP_F32 && w.out_dtype != ALCOP_F16 && w.out_dtype != ALCOP_BF16)
    return set_error(ALCOP_ERR_CONFIG, "BadDtype", "output dtype must be F32, F16 or BF16");
  if (w.b_layout != ALCOP_B_KN && w.b_layout != ALCOP_B_NK)
    return set_error(ALCOP_ERR_CONFIG, "BadLayout", "b_layout must be KN or NK");
  if (w.pre_op != 0 && w.pre_op != 1)
    return set_error(ALCOP_ERR_CONFIG, "BadWorkload", "pre_op must be 0 or 1 (f(x) = 2x+1)");
  if (w.pre_op && (s.cta_group != 1 || s.n_stage_smem_A != s.n_stage_smem_B))
    return set_error(ALCOP_ERR_CONFIG, "Unsupported", "the fused pre-op needs cta_group 1 and equal stage counts");
  if (s.cta_group != 1 && s.cta_group != 2)
    return set_error(ALCOP_ERR_CONFIG, "BadSchedule", "cta_group must be 1 or 2");
  if (s.tileM != kTileM * s.cta_group)
    return set_error(ALCOP_ERR_CONFIG, "BadTile", "tileM must be 128 x cta_group (UMMA M 128 / 256)");
  if (s.tileN != 64 && s.tileN != 128 && s.tileN != 192 && s.tileN != 256 && s.tileN != 512)
    return set_error(ALCOP_ERR_CONFIG, "BadTile", "tileN must be one of 64, 128, 192, 256 (512: CTA pair)");
  if (s.tileN == 512 && (s.cta_group != 2 || s.n_stage_inner != 1 || s.stream_k != 0))
    return set_error(ALCOP_ERR_CONFIG, "BadTile",
                     "tileN 512 is the CTA-pair 256 x 512 tile: cta_group 2, one TMEM accumulator, whole tiles");
  if (s.cta_group == 2 && s.tileN == 64)
    return set_error(ALCOP_ERR_CONFIG, "BadTile", "cta_group 2 needs tileN 128, 192 or 256");
  if (s.stream_k != 0 && (s.stream_k != 1 || s.cta_group != 2 || s.mode != ALCOP_MODE_FUSED))
    return set_error(ALCOP_ERR_CONFIG, "BadSchedule", "stream_k (0|1) applies to cta_group 2 in FUSED mode");
  if (s.cta_group == 2 && s.n_stage_smem_A != s.n_stage_smem_B)
    return set_error(ALCOP_ERR_CONFIG, "BadStages", "cta_group 2 uses one joint A+B ring: equal stage counts");
  if (s.tileK != 32 && s.tileK != 64 && s.tileK != 128)
    return set_error(ALCOP_ERR_CONFIG, "BadTile", "tileK must be one of 32, 64, 128");
  if (s.raster < 0 || s.num_ctas < 0)
    return set_error(ALCOP_ERR_CONFIG, "BadRaster", "raster group and num_ctas must be >= 0");
  if (s.n_stage_smem_A < 1 || s.n_stage_smem_B < 1 || s.n_stage_smem_A > kMaxStages ||
      s.n_stage_smem_B > kMaxStages)
    return set_error(ALCOP_ERR_CONFIG, "BadStages", "shared-memory stages must be in [1, 16]");
  if (s.n_stage_inner < 1 || s.n_stage_inner > 2)
    return set_error(ALCOP_ERR_CONFIG, "BadStages", "inner (TMEM accumulator) stages must be 1 or 2");
  if (s.mode != ALCOP_MODE_WRAP && s.mode != ALCOP_MODE_FUSED)
    return set_error(ALCOP_ERR_CONFIG, "BadSchedule", "mode must be WRAP or FUSED");
  // The inner pipeline of the reference (A_reg/B_reg, F = tileK/regK k-steps
  // per chunk) may not look further ahead than the outer one covers
  // (LookaheadExceedsOuter, pipeline_pass.hpp:305-313; params_valid,
  // perf_model.hpp:139-140).  On tcgen05 F = tileK/16.
  const int64_t F = s.tileK / 16;
  const int32_t s_outer = std::min(s.n_stage_smem_A, s.n_stage_smem_B);
  if (static_cast<int64_t>(s.n_stage_inner - 1) > static_cast<int64_t>(s_outer - 1) * F && s_outer > 1)
    return set_error(ALCOP_ERR_ANALYSIS, "LookaheadExceedsOuter",
                     "inner pipeline looks ahead further than the outer pipeline covers");
  const int64_t acc_stride = round_up_pow2_cols(s.tileN);
  if (acc_stride * s.n_stage_inner > kTmemCols)
    return set_error(ALCOP_ERR_CONFIG, "TmemCapacity", "n_stage_inner * tileN exceeds 512 TMEM columns");
  const int64_t smem = gemm_smem_bytes(w, s);
  if (smem > kMaxSmemBytes)
    return set_error(ALCOP_ERR_CONFIG, "SmemCapacity",
                     "pipeline ring needs " + std::to_string(smem) + " B shared memory, more than 232448");
  const int64_t lda = w.lda ? w.lda : w.K;
  const int64_t ldb = w.ldb ? w.ldb : (w.b_layout == ALCOP_B_KN ? w.N : w.K);
  const int64_t ldc = w.ldc ? w.ldc : w.N;
  if ((lda * 2) % 16 || (ldb * 2) % 16)
    return set_error(ALCOP_ERR_CONFIG, "Alignment", "A/B row pitch must be a multiple of 16 bytes (TMA)");
  if ((ldc * dtype_bytes(w.out_dtype)) % 16)
    return set_error(ALCOP_ERR_CONFIG, "Alignment", "C row pitch must be a multiple of 16 bytes");
  if (w.stride_a % 8 || w.stride_b % 8 || w.stride_c % 8)
    return set_error(ALCOP_ERR_CONFIG, "Alignment", "batch strides must be multiples of 16 bytes");
  return ALCOP_OK;
}

static int check_ptr_alignment(const void* A, const void* B, const void* C) {
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C)) & 15)
    return set_error(ALCOP_ERR_CONFIG, "Alignment", "A, B and C must be 16-byte aligned");
  return ALCOP_OK;
}

}  // namespace alcop

using namespace alcop;

extern "C" {

const char* alcop_version(void) { return "alcop-b200 0.1.0 (sm_100a)"; }

const char* alcop_last_error(void) { return g_last_error.c_str(); }

void alcop_schedule_default(alcop_schedule* out) {
  if (!out) return;
  std::memset(out, 0, sizeof(*out));
  out->tileM = 128;
  out->tileN = 256;
  out->tileK = 64;
  out->n_stage_smem_A = 4;
  out->n_stage_smem_B = 4;
  out->n_stage_inner = 2;
  out->cta_group = 1;
  out->mode = ALCOP_MODE_FUSED;
}

int alcop_validate(const alcop_gemm_desc* w, const alcop_schedule* s) {
  if (!w || !s) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "descriptor is NULL");
  clear_error();
  return validate_gemm(*w, *s);
}

int64_t alcop_smem_bytes(const alcop_gemm_desc* w, const alcop_schedule* s) {
  if (!w || !s) return -1;
  return gemm_smem_bytes(*w, *s);
}

int alcop_gemm(const alcop_gemm_desc* w, const alcop_schedule* s, const void* A, const void* B, void* C,
               void* stream) {
  if (!w || !s || !A || !B || !C) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument");
  clear_error();
  int rc = validate_gemm(*w, *s);
  if (rc) return rc;
  rc = check_ptr_alignment(A, B, C);
  if (rc) return rc;
  return launch_gemm(*w, *s, A, B, C, nullptr, 0, stream);
}

int alcop_gemm_traced(const alcop_gemm_desc* w, const alcop_schedule* s, const void* A, const void* B, void* C,
                      alcop_event* trace_dev, int64_t events_per_role_cap, void* stream) {
  if (!w || !s || !A || !B || !C || !trace_dev)
    return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument");
  clear_error();
  int rc = validate_gemm(*w, *s);
  if (rc) return rc;
  rc = check_ptr_alignment(A, B, C);
  if (rc) return rc;
  return launch_gemm(*w, *s, A, B, C, trace_dev, events_per_role_cap, stream);
}

int64_t alcop_gemm_workspace_bytes(const alcop_gemm_desc* w) {
  if (!w) return -1;
  auto al = [](int64_t b) { return (b + 255) / 256 * 256; };
  const int64_t ob = w->out_dtype == ALCOP_F32 ? 4 : 2;
  return al(w->batch * w->M * w->K * 2) + al(w->batch * w->K * w->N * 2) + al(w->batch * w->M * w->N * ob);
}

static int gemm_host_impl(const alcop_gemm_desc* w, const alcop_schedule* s, const void* hA, const void* hB,
                          void* hC, void* workspace, void* stream, bool sync) {
  if (!w || !s || !hA || !hB || !hC || !workspace)
    return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument");
  clear_error();
  if (w->lda || w->ldb || w->ldc || w->stride_a || w->stride_b || w->stride_c)
    return set_error(ALCOP_ERR_CONFIG, "BadWorkload", "host-buffer entry point takes packed tensors only");
  int rc = validate_gemm(*w, *s);
  if (rc) return rc;
  auto al = [](int64_t b) { return (b + 255) / 256 * 256; };
  const int64_t ob = w->out_dtype == ALCOP_F32 ? 4 : 2;
  const int64_t bytesA = w->batch * w->M * w->K * 2, bytesB = w->batch * w->K * w->N * 2,
                bytesC = w->batch * w->M * w->N * ob;
  char* dA = static_cast<char*>(workspace);
  char* dB = dA + al(bytesA);
  char* dC = dB + al(bytesB);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // The load-and-use pipeline one level up: A is streamed to the device in
  // row blocks on a copy stream, block i is multiplied on the caller's stream
  // as soon as it lands, and its C rows go back on a second copy stream while
  // block i+1 is multiplied and block i+2 copied in (H2D, compute and D2H
  // overlap; the two copy directions run on separate engines).  B is needed
  // whole by every block and goes first.  Batched / small problems: one block.
  const int64_t tm = s->tileM;
  int nblk = (w->batch == 1 && w->M >= 4 * tm) ? 8 : 1;
  if (nblk > 1) {
    const int64_t target = host_block_bytes(sync);
    if (target > 0) nblk = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(8, bytesA / target)));
  }
  int64_t rows = (w->M + nblk - 1) / nblk;
  rows = (rows + tm - 1) / tm * tm;
  nblk = static_cast<int>((w->M + rows - 1) / rows);
  HostPipe* hp = host_pipe();
  if (!hp) return set_error(ALCOP_ERR_CUDA, "CudaError", "could not create the copy streams");
  cudaError_t e = cudaSuccess;
  // Ordering of this call's H2D copies (they write the workspace and read hA/hB):
  //  * sync: after all earlier work on `stream`;
  //  * async: after the previous call's kernels (they may still read a shared
  //    workspace; everything enqueued on `stream` before them is covered too)
  //    and, when hA or hB overlaps the host range the previous call's D2H
  //    writes (its C feeds this call), after that D2H.  Not after an
  //    unrelated previous D2H: that overlap (H2D of call k+1 with the D2H of
  //    call k on the other copy engine) is the point of the async variant.
  const char* a0 = static_cast<const char*>(hA);
  const char* b0 = static_cast<const char*>(hB);
  auto overlaps = [&](const char* p, int64_t n) {
    return hp->have_prev && p < hp->prev_c + hp->prev_c_bytes && hp->prev_c < p + n;
  };
  if (sync) {
    e = cudaEventRecord(hp->ev_start, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(hp->h2d, hp->ev_start, 0);
  } else if (hp->have_prev) {
    e = cudaStreamWaitEvent(hp->h2d, hp->ev_kernels, 0);
    if (e == cudaSuccess && (overlaps(a0, bytesA) || overlaps(b0, bytesB)))
      e = cudaStreamWaitEvent(hp->h2d, hp->ev_done, 0);
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(dB, hB, bytesB, cudaMemcpyHostToDevice, hp->h2d);
  for (int i = 0; i < nblk && e == cudaSuccess; ++i) {
    const int64_t r0 = i * rows, nr = std::min(rows, w->M - r0);
    const int64_t off = nblk == 1 ? 0 : r0 * w->K * 2, len = nblk == 1 ? bytesA : nr * w->K * 2;
    e = cudaMemcpyAsync(dA + off, static_cast<const char*>(hA) + off, len, cudaMemcpyHostToDevice, hp->h2d);
    if (e == cudaSuccess) e = cudaEventRecord(hp->ev_in[i], hp->h2d);
  }
  for (int i = 0; i < nblk && e == cudaSuccess && rc == ALCOP_OK; ++i) {
    const int64_t r0 = i * rows, nr = std::min(rows, w->M - r0);
    e = cudaStreamWaitEvent(st, hp->ev_in[i], 0);
    if (e != cudaSuccess) break;
    alcop_gemm_desc sub = *w;
    if (nblk > 1) {
      sub.M = nr;
      sub.lda = w->K;
      sub.ldc = w->N;
    }
    rc = launch_gemm(sub, *s, dA + (nblk == 1 ? 0 : r0 * w->K * 2), dB, dC + (nblk == 1 ? 0 : r0 * w->N * ob),
                     nullptr, 0, stream);
    if (rc == ALCOP_OK) e = cudaEventRecord(hp->ev_out[i], st);
  }
  if (rc != ALCOP_OK) {
    cudaStreamSynchronize(hp->h2d);
    return rc;
  }
  if (e == cudaSuccess) e = cudaEventRecord(hp->ev_kernels, st);
  for (int i = 0; i < nblk && e == cudaSuccess; ++i) {
    const int64_t r0 = i * rows, nr = std::min(rows, w->M - r0);
    const int64_t off = nblk == 1 ? 0 : r0 * w->N * ob, len = nblk == 1 ? bytesC : nr * w->N * ob;
    e = cudaStreamWaitEvent(hp->d2h, hp->ev_out[i], 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(static_cast<char*>(hC) + off, dC + off, len, cudaMemcpyDeviceToHost,
                                              hp->d2h);
  }
  if (e == cudaSuccess) e = cudaEventRecord(hp->ev_done, hp->d2h);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, hp->ev_done, 0);  // stream order for the caller
  if (e == cudaSuccess && sync) e = cudaEventSynchronize(hp->ev_done);
  if (e != cudaSuccess) {
    hp->have_prev = false;
    return set_error(ALCOP_ERR_CUDA, "CudaError", cudaGetErrorString(e));
  }
  hp->have_prev = true;
  hp->prev_c = static_cast<const char*>(hC);
  hp->prev_c_bytes = bytesC;
  return ALCOP_OK;
}

int alcop_gemm_host(const alcop_gemm_desc* w, const alcop_schedule* s, const void* hA, const void* hB, void* hC,
                    void* workspace, void* stream) {
  return gemm_host_impl(w, s, hA, hB, hC, workspace, stream, true);
}

int alcop_gemm_host_async(const alcop_gemm_desc* w, const alcop_schedule* s, const void* hA, const void* hB,
                          void* hC, void* workspace, void* stream) {
  return gemm_host_impl(w, s, hA, hB, hC, workspace, stream, false);
}

int64_t alcop_gemm_chain_workspace_bytes(const alcop_chain* ch) {
  if (!ch || ch->n < 1 || ch->n > ALCOP_CHAIN_MAX) return 0;
  return static_cast<int64_t>(sizeof(int32_t)) * ch->n * chain_max_row_blocks(ch);
}

int alcop_gemm_chain(const alcop_chain* ch, const alcop_schedule* s, void* workspace, void* stream) {
  if (!ch || !s || !workspace) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument");
  clear_error();
  if (ch->n < 1 || ch->n > ALCOP_CHAIN_MAX)
    return set_error(ALCOP_ERR_CONFIG, "BadWorkload", "chain length must be 1..ALCOP_CHAIN_MAX");
  if (s->mode != ALCOP_MODE_FUSED || s->n_stage_smem_A != s->n_stage_smem_B || s->stream_k)
    return set_error(ALCOP_ERR_CONFIG, "Unsupported", "the chain runs FUSED, equal A/B stages, whole tiles");
  const alcop_gemm_desc& w0 = ch->desc[0];
  // CTA pairs: each CTA stages half of the tile's B columns — whole 64-column
  // atoms for B[K,N], 16-row groups for B[N,K]
  if (s->cta_group == 2 && (s->tileN % (w0.b_layout == ALCOP_B_KN ? 128 : 32) != 0))
    return set_error(ALCOP_ERR_CONFIG, "Unsupported",
                     "a chain on CTA pairs needs tileN % 128 == 0 (B[K,N]) or tileN % 32 == 0 (B[N,K])");
  for (int i = 0; i < ch->n; ++i) {
    const alcop_gemm_desc& w = ch->desc[i];
    if (!ch->A[i] || !ch->B[i] || !ch->C[i]) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL operand");
    if (w.batch != 1 || w.pre_op || w.stride_a || w.stride_b || w.stride_c)
      return set_error(ALCOP_ERR_CONFIG, "Unsupported", "chain GEMMs are batch 1 without pre-op");
    if (w.in_dtype != w0.in_dtype || w.out_dtype != w0.out_dtype || w.b_layout != w0.b_layout)
      return set_error(ALCOP_ERR_CONFIG, "BadWorkload", "chain GEMMs share dtypes and B layout");
    int rc = validate_gemm(w, *s);
    if (rc) return rc;
    if (ch->dep[i] && (i == 0 || w.M != ch->desc[i - 1].M))
      return set_error(ALCOP_ERR_CONFIG, "BadDependency", "dep[p] needs p > 0 and M_p == M_{p-1}");
  }
  return launch_chain(*ch, *s, workspace, stream);
}

int64_t alcop_stream_k_workspace_bytes(const alcop_gemm_desc* w, const alcop_schedule* s) {
  if (!w || !s || validate_gemm(*w, *s) != ALCOP_OK || s->cta_group != 2) return 0;
  const int sms = device_sm_count() > 0 ? device_sm_count() : 148;
  const int64_t grid = (s->num_ctas > 0 ? s->num_ctas : sms) / 2;
  const int64_t tiles = ((w->M + 255) / 256) * ((w->N + s->tileN - 1) / s->tileN) * w->batch;
  const int n = static_cast<int>(std::min<int64_t>(grid, tiles));
  return static_cast<int64_t>(sk_bytes_needed(n, static_cast<int>(s->tileN)));
}

int alcop_set_stream_k_workspace(void* workspace, int64_t bytes) {
  clear_error();
  return set_sk_workspace(workspace, bytes);
}

int alcop_conv2d(const alcop_conv_desc* d, const alcop_schedule* s, const void* x, const void* wt, void* y,
                 void* stream) {
  if (!d || !s || !x || !wt || !y) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument");
  clear_error();
  return launch_conv2d(*d, *s, x, wt, y, stream);
}

}  // extern "C"
