/*
 * alcop.h — C ABI of the B200-native pipelined load-and-use hot path
 * (ALCOP, arXiv 2210.16691) re-implemented for sm_100a.
 *
 * The reference ("pipec", /root/reference/proj/include/pipec) is a header-only
 * C++20 library with no FFI; its operator surface is the C++ namespace
 * `pipec`.  Every entry point below replaces one reference interface and
 * cites it as file:line relative to /root/reference.  Plain pointers and
 * sizes only: no torch or C++ types cross this boundary, no exceptions
 * cross it, and the library never allocates device memory on a call path
 * (the caller owns buffers and the stream).
 *
 * Return codes follow the reference CLI exit-code map
 * (proj/include/pipec/cli.hpp:23-25) plus ALCOP_ERR_CUDA.  After a non-zero
 * return, alcop_last_error() (thread-local) holds "<RuleTag>: message",
 * reusing the reference rule tags (pipeline_pass.hpp:191-322,
 * schedule.hpp:113-308).
 */
#ifndef ALCOP_H_
#define ALCOP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes: pipec/cli.hpp:23-25 (kOk..kConfig) + CUDA ---------- */
#define ALCOP_OK 0
#define ALCOP_ERR_PARSE 2       /* ParseError        (common.hpp:43)  */
#define ALCOP_ERR_VALIDATE 3    /* ValidationError   (common.hpp:51)  */
#define ALCOP_ERR_ANALYSIS 4    /* AnalysisError/InterpError (common.hpp:57,67) */
#define ALCOP_ERR_EQUIVALENCE 5 /* equivalence failure (cli.hpp:296-298) */
#define ALCOP_ERR_CONFIG 6      /* ConfigError       (common.hpp:63)  */
#define ALCOP_ERR_CUDA 7        /* CUDA runtime / launch failure (new) */

/* ---- element types.  The reference has names only (f16 = 2 bytes,
 * schedule.hpp:341-349); bf16 is added because B200 computes in it. ----- */
typedef enum {
  ALCOP_F16 = 0,
  ALCOP_BF16 = 1,
  ALCOP_F32 = 2
} alcop_dtype;

/* B operand layout.  The reference lowers B as [K,N] row-major
 * (schedule.hpp:389) = MN-major for tcgen05; NK is the K-major variant. */
typedef enum {
  ALCOP_B_KN = 0,
  ALCOP_B_NK = 1
} alcop_b_layout;

/* Pipeline emission mode.
 *  WRAP  : bit-faithful to the pass output (pipeline_pass.hpp:482-552,
 *          622-748): per output tile an n_stage-1 chunk prologue, steady
 *          loads of chunk (v+s-1)%E into slot (v+s-1)%s, consumer slot v%s,
 *          and s-1 drain wait/release pairs after the k loop.
 *  FUSED : the paper's holistic pipeline applied to the persistent tile
 *          loop: lookahead crosses into the next tile's chunks, so no
 *          redundant wrapped loads and no per-tile drains. */
typedef enum {
  ALCOP_MODE_WRAP = 0,
  ALCOP_MODE_FUSED = 1
} alcop_mode;

/* Problem descriptor.  Mirrors pipec::WorkloadDesc (schedule.hpp:15-19)
 * plus the layout facts the reference fixes implicitly (row-major A[b,M,K],
 * B[b,K,N], C[b,M,N], schedule.hpp:388-390).  Leading dims / batch strides
 * are in elements; 0 means packed. */
typedef struct {
  int64_t M, N, K, batch;
  int32_t in_dtype;  /* alcop_dtype: F16 or BF16 */
  int32_t out_dtype; /* alcop_dtype: F32, F16 or BF16 */
  int32_t b_layout;  /* alcop_b_layout */
  int32_t pre_op;    /* 0, or 1 = gemm_schedule(w, preOp=true): the mma reads f(A) = 2A+1
                        (the reference's "ew" tag, interp.hpp:363, schedule.hpp:73-86) */
  int64_t lda, ldb, ldc;
  int64_t stride_a, stride_b, stride_c;
} alcop_gemm_desc;

/* Schedule.  Mirrors the per-buffer pipelining hints (BufferDecl::
 * pipelineStages, ir.hpp:12-26; mark_pipeline, schedule.hpp:258-268), the
 * tile splits (tile, schedule.hpp:141-193) and perf::ScheduleParams
 * (perf_model.hpp:32-38).  n_stage 1 = "no hint" (not pipelined): the
 * reference cannot express it (stages >= 2, schedule.hpp:261), here it is
 * the in-run baseline variant (one slot: load -> wait -> use -> release). */
typedef struct {
  int64_t tileM, tileN, tileK; /* tile; tileM = 128 x cta_group; tileN 64..256 (512: pair, 1 accumulator) */
  int32_t n_stage_smem_A;      /* A_shared ring depth (outer level)     */
  int32_t n_stage_smem_B;      /* B_shared ring depth (outer level)     */
  int32_t n_stage_inner;       /* A_reg/B_reg level -> TMEM accumulator buffers (1|2) */
  int32_t cta_group;           /* 1, or 2 = CTA pair (tcgen05 cta_group::2, tileM 256) */
  int32_t mode;                /* alcop_mode                             */
  int32_t num_ctas;            /* persistent grid; 0 = #SMs              */
  int32_t raster;              /* tile rows per raster group; 0 = auto  */
  int32_t stream_k;            /* CTA pair, FUSED: 1 = split the output tiles' chunk stream
                                  evenly over the clusters (a tile cut between two clusters
                                  is finished from an fp32 partial); the partials live in the
                                  device's stream-K workspace (alcop_set_stream_k_workspace), so
                                  stream_k launches must not run concurrently on two streams;
                                  without a large enough workspace the launch runs whole
                                  tiles.  0 = whole tiles per cluster */
} alcop_schedule;

/* ---- several GEMMs in one persistent launch (new; no reference form) ------
 * The GEMMs run as ONE flattened (problem, tile, chunk) stream through the
 * same smem ring and TMEM accumulator ring, so nothing drains between them
 * (the holistic pipeline one level up: the last tile's epilogue of GEMM p
 * overlaps GEMM p+1's main loop).  dep[p] = 1: row block mb (one tile row) of
 * A_p is read only after every tile of row block mb of C_{p-1} is stored
 * (requires M_p == M_{p-1}); dep[0] must be 0.  All GEMMs share the schedule
 * (FUSED, equal A/B stages; cta_group 1, or 2 = CTA pairs with 256-row
 * blocks and tileN % 128 == 0 for B[K,N], % 32 for B[N,K]), dtypes and B
 * layout; batch 1.
 * workspace: device memory of alcop_gemm_chain_workspace_bytes() bytes
 * (row-block counters, zeroed on `stream` by the call). */
#define ALCOP_CHAIN_MAX 4
typedef struct {
  int32_t n; /* 1..ALCOP_CHAIN_MAX */
  int32_t dep[ALCOP_CHAIN_MAX];
  alcop_gemm_desc desc[ALCOP_CHAIN_MAX];
  const void* A[ALCOP_CHAIN_MAX];
  const void* B[ALCOP_CHAIN_MAX];
  void* C[ALCOP_CHAIN_MAX];
} alcop_chain;
int64_t alcop_gemm_chain_workspace_bytes(const alcop_chain* ch);
int alcop_gemm_chain(const alcop_chain* ch, const alcop_schedule* s, void* workspace, void* stream);

/* Implicit-GEMM conv2d descriptor (no reference form: SPEC.md:218).
 * x: NHWC, w: KRSC, y: NPQK. */
typedef struct {
  int64_t N, H, W, C, K, R, S;
  int32_t stride_h, stride_w, pad_h, pad_w;
  int32_t in_dtype, out_dtype;
  int32_t x_halo;   /* 1: x is stored [N][H+2pad_h][W+2pad_w][C] with its zero
                       padding halo (a network-input layout); enables the stem
                       kernel (one TMA box per filter row) when S*C <= 64 */
  int32_t reserved0;
} alcop_conv_desc;

/* Hardware spec for the analytical model (perf::HardwareSpec,
 * perf_model.hpp:14-30), B200 defaults via alcop_hw_default_b200(). */
typedef struct {
  int32_t numSM;
  double throughputSM; /* FLOP / cycle / SM (dense f16/bf16) */
  double bwLLC;        /* bytes / cycle, device-wide L2 -> SM */
  double bwDRAM;       /* bytes / cycle */
  double bwDRAMWrite;  /* bytes / cycle */
  double latLLCRead, latDRAMRead, latDRAMWrite; /* cycles */
  double bwSmem, latSmem;
  int64_t smemPerSM, regsPerSM;
  int32_t maxThreadblkPerSM, maxWarpsPerSM, utilKneeWarps;
  int32_t tmemColsPerSM; /* 512 (new: TMEM capacity) */
  double clockGHz;       /* cycles -> seconds */
  /* B200 additions (calibrated, tools/fit_model.py on profiles/sweep_r01.json) */
  double tIssue;         /* per-chunk producer/MMA issue floor, cycles */
  double tIssuePerBox;   /* + cycles per TMA box of the chunk */
  double tLaunch;        /* kernel launch + setup, cycles */
  double tTile;          /* per output tile fixed cost, cycles */
  double overlapDRAM;    /* soft-max weight between the SM pipeline and HBM time */
  double tPair;          /* fixed extra cycles of a cta_group::2 (CTA-pair) launch */
  /* Power-capped regime (new; tools/fit_power.py on profiles/power_r02.json):
   * under sustained load the B200 holds its ~1 kW cap by lowering the SM
   * clock, so a long kernel takes at least energy / power =
   * tCapFlop * FLOPs + tCapL2Byte * (L2 -> SM bytes) + tCapDramByte * (DRAM bytes). */
  double tCapFlop;          /* seconds per FLOP at the cap */
  double tCapL2Byte;        /* seconds per L2 -> shared-memory (TMA) byte at the cap */
  double tCapDramByte;      /* seconds per HBM byte at the cap */
  double dramReusePair;     /* DRAM bytes / ideal grouped-raster bytes, CTA pairs, K <= 8192 */
  double dramReusePairPerK; /* + per reduction element above 8192 (pairs drift apart over long K) */
} alcop_hw;

/* perf::LatencyBreakdown (perf_model.hpp:40-47); field names follow
 * json_io.hpp:95-114. */
typedef struct {
  double tKernel, tThreadblk, tInit, tMainLoop, tEpilogue;
  double tSmemLoad, tRegLoad, tSmemUse, tCompute;
  int64_t nThreadblkBatch, nThreadblkPerSM, nThreadblkPerBatch;
  int64_t nSmemLoop, nRegLoop;
  int64_t bytesOneSmemLoop, bytesWorkset, bytesOutputTile;
  int64_t flopsOneRegLoop;
  double seconds; /* tKernel / clock (new) */
  /* new: traffic and the power-capped bound */
  double bytesL2;  /* L2 -> shared-memory TMA bytes of the whole launch (exact) */
  double bytesDram; /* estimated HBM bytes (grouped raster, L2 reuse) */
  double tPower;   /* energy / power-cap bound, cycles; tKernel = max(latency model, tPower) */
} alcop_breakdown;

/* One pipeline bookkeeping event (host enumerator and device trace).
 * kind: 0 producer_acquire+commit (a load), 1 consumer_wait,
 *       2 consumer_release.  buf: 0 = A_shared, 1 = B_shared.
 * Counters follow interp.hpp:87-94 / TraceEvent (interp.hpp:20-26). */
typedef struct {
  int32_t kind, buf, tile, slot, chunk, parity;
  int32_t acquired, committed, waited, released;
} alcop_event;

/* ---- library ---------------------------------------------------------- */
const char* alcop_version(void);
/* thread-local "<RuleTag>: message" of the last failing call */
const char* alcop_last_error(void);

/* ---- schedule surface ------------------------------------------------- */
void alcop_schedule_default(alcop_schedule* out);

/* Applies a reference schedule script (apply_script, schedule.hpp:590-646:
 * `cache_read`, `tile C i0=.. i1=.. j0=.. j1=.. ko=.. ki=..`, `pipeline
 * <buf> <n>`, `inline S2`) to gemm_schedule(w) (schedule.hpp:73-86) with the
 * reference eligibility rules (check_eligibility, schedule.hpp:198-254) and
 * rule tags, and maps the result to an alcop_schedule.  Buffers left without
 * a hint get n_stage 1.  `warnings` (may be NULL) receives the
 * SyncPositionConflict refusal text (schedule.hpp:625-637). */
int alcop_parse_schedule_script(const alcop_gemm_desc* w, const char* script, alcop_schedule* out,
                                char* warnings, size_t warnings_len);

/* params_valid analogue (perf_model.hpp:129-142) for the B200 kernel:
 * tile shape, stage counts vs 227 KB shared memory, TMEM columns,
 * LookaheadExceedsOuter (pipeline_pass.hpp:305-313), alignment. */
int alcop_validate(const alcop_gemm_desc* w, const alcop_schedule* s);
/* dynamic shared memory bytes the kernel will request for (w, s) */
int64_t alcop_smem_bytes(const alcop_gemm_desc* w, const alcop_schedule* s);

/* ---- host bookkeeping enumerator (pipeline_pass.hpp:482-748 index
 * algebra + interp.hpp:375-418 counters): the event sequence one CTA
 * executes for `num_tiles` output tiles of E = ceil(K/tileK) chunks.
 * role 0 = producer events, role 1 = consumer events.  Writes at most
 * `cap` events, sets *count to the full length. */
int alcop_enumerate_pipeline(int64_t num_tiles, int64_t E, int32_t sA, int32_t sB, int32_t mode,
                             int32_t role, alcop_event* out, int64_t cap, int64_t* count);

/* ---- reference IR front end ---------------------
 * Parses a program in the reference's textual IR (the
 * `pipec schedule` output = lower() with `stages` hints, schedule.hpp:357-584),
 * recognises the lowered GEMM / batched-GEMM nest and returns the problem and
 * schedule that run it on B200 (mode WRAP = the pass's own emission, f16 in,
 * f32 out = the interpreter's exact sums).  Parse errors -> ALCOP_ERR_PARSE
 * ("ParseError: ... (line L, col C)", parser.hpp:22-454); an already
 * transformed program -> ALCOP_ERR_ANALYSIS "AlreadySynchronized"
 * (pipeline_pass.hpp:191-196).  `info` (may be NULL) receives a summary. */
int alcop_ir_to_gemm(const char* ir_text, alcop_gemm_desc* desc, alcop_schedule* sched, char* info,
                     size_t info_len);

/* ---- compute entry points (device pointers, caller-owned stream) ------ */
/* Pipelined matmul: gemm_schedule -> lower -> transform -> run
 * (schedule.hpp:73,357; pipeline_pass.hpp:753; interp.hpp:440) as one
 * sm_100a kernel launch.  batch > 1 is the batched GEMM (schedule.hpp:384-390). */
int alcop_gemm(const alcop_gemm_desc* w, const alcop_schedule* s, const void* A, const void* B, void* C,
               void* stream);

/* Same launch with the device debug trace: each CTA's producer and MMA
 * threads log their events.  trace must hold
 * num_ctas * 2 * events_per_role_cap alcop_event records. */
int alcop_gemm_traced(const alcop_gemm_desc* w, const alcop_schedule* s, const void* A, const void* B,
                      void* C, alcop_event* trace_dev, int64_t events_per_role_cap, void* stream);

/* End-to-end call with HOST buffers: H2D of A,B (pinned host recommended),
 * the kernel, D2H of C, all on `stream`; `workspace` is caller-owned device
 * memory of at least alcop_gemm_workspace_bytes(w) bytes. Synchronous. */
int64_t alcop_gemm_workspace_bytes(const alcop_gemm_desc* w);
int alcop_gemm_host(const alcop_gemm_desc* w, const alcop_schedule* s, const void* hA, const void* hB,
                    void* hC, void* workspace, void* stream);

/* Stream-ordered variant (returns before the copies finish): A's row blocks go
 * up on an internal copy stream, each block is multiplied on `stream` as it
 * lands, C's blocks come back on a second copy stream; `stream` is made to
 * wait for the last D2H, so C is valid after cudaStreamSynchronize(stream).
 * Consecutive calls overlap (the H2D of call k+1 with the D2H of call k) when
 * each call in flight has its own workspace and host buffers.
 * Ordering: a call's H2D copies start after the previous call's kernels on this
 * host thread and device (so a shared workspace is safe, as is all work enqueued
 * on `stream` before them) and, when hA or hB overlaps the previous call's hC,
 * after that call's D2H (a chain where C_k is A_{k+1}).  Host inputs written by
 * OTHER work (the caller's own copies, another thread) must be complete on the
 * host before the call. */
int alcop_gemm_host_async(const alcop_gemm_desc* w, const alcop_schedule* s, const void* hA, const void* hB,
                          void* hC, void* workspace, void* stream);

/* Stream-K workspace of the current device (caller-owned device memory; the
 * library never allocates it): fp32 partials + hand-off flags.  bytes =
 * alcop_stream_k_workspace_bytes(w, s) covers that problem/schedule; the call
 * zeroes the flags (cudaMemset on the legacy stream, synchronised).  NULL
 * unregisters.  Register before capturing stream_k launches in a graph. */
int64_t alcop_stream_k_workspace_bytes(const alcop_gemm_desc* w, const alcop_schedule* s);
int alcop_set_stream_k_workspace(void* workspace, int64_t bytes);

/* Implicit-GEMM conv2d (new; the reference excludes it).
 * Kernel by shape and schedule (all pipelined, all on sm_100a; no fallback):
 *  - C == 4, stride_w == 2 (e.g. ResNet-50 conv1 with the 3 channels padded to
 *    4): the resident-filter kernel in pixel-pair mode; W % 16 == 0,
 *    K % 16 == 0, K <= 256, K * out bytes % 128 == 0; schedule tileM 128,
 *    tileN == K, tileK 64, FUSED, cta_group 1, n_stage = window ring depth,
 *    n_stage_inner = TMEM accumulators (1..8, n_stage_inner * K <= 512);
 *  - C == 64, stride 1, spatial filter whose K x R x S x 64 filter fits
 *    (<= 80 KB), with such a resident-filter schedule: window mode of the same
 *    kernel (the tile's input window loaded once, taps = shifted descriptors);
 *  - C % 64 == 0, C > 64, K <= 128, stride 1, spatial filter, with a schedule
 *    that validates there (tileN == K, tileK 64 or 64 x S = taps per filter
 *    chunk, n_stage_smem_A = window ring 1..4, n_stage_smem_B = filter ring,
 *    n_stage_inner 1..2): window mode with the filter streamed through its
 *    own ring;
 *    both window modes also run on CTA pairs (cta_group 2, tileM 256,
 *    K % 32 == 0): a 256-pixel tile = the two CTAs' windows, each CTA staging
 *    half of the filter rows;
 *  - 1x1, stride 1, no padding: the GEMM kernels ([N*H*W, C] x [K, C]^T),
 *    any GEMM schedule incl. CTA pairs;
 *  - otherwise C % 8 == 0: the implicit-GEMM kernel with TMA im2col loads
 *    (tileK 64, equal A/B stages, whole tiles; cta_group 2 = CTA pairs when
 *    C % 64 == 0 and x is not in the halo layout, each CTA a 128-pixel half
 *    of the 256-pixel tile). */
int alcop_conv2d(const alcop_conv_desc* d, const alcop_schedule* s, const void* x, const void* w, void* y,
                 void* stream);

/* ---- multi-GPU driver (new: the reference runs its parallel
 * b / i0 / j0 loops sequentially, interp.hpp:330-338) --------------------
 * The units that shard — rows of A and C (M-sharded GEMM, B replicated),
 * batch entries (batched GEMM) or images (conv, filter replicated) — split
 * contiguously over `nshards` in multiples of `granule` (earlier shards take
 * the remainder granules); no collective on the compute path.  One host
 * thread per shard sets its device and enqueues that shard's launch on its
 * stream; the call returns when every shard is enqueued (stream-ordered per
 * device; synchronise each shard's stream for the results).  Several shards
 * may name the same device (distinct streams run concurrently). */
typedef struct {
  int32_t device;  /* CUDA device ordinal */
  void* stream;    /* that device's stream (NULL: its legacy default stream) */
  const void* A;   /* GEMM: this shard's rows (or batch entries) of A; conv: its images of x */
  const void* B;   /* the replica of B (conv: of the filter) on `device` */
  void* C;         /* this shard's rows / batch entries of C (conv: its images of y) */
} alcop_shard;

/* [*start, *start + *count): shard `rank` of `total` units over `world`
 * shards in `granule` multiples (bench.py and paper_2210_16691_b200/sharded.py
 * use the same split). */
int alcop_shard_range(int64_t total, int32_t rank, int32_t world, int64_t granule, int64_t* start,
                      int64_t* count);
/* Sharded GEMM: batch == 1 shards M (granule >= 1 rows; 256 = one CTA-pair tile
 * row), batch > 1 shards the batch.  s == NULL: the model's pick per shard
 * shape (alcop_choose_schedule with the B200 defaults); empty shards launch
 * nothing.  Packed tensors only (no lda/ldb/ldc, no batch strides). */
int alcop_gemm_sharded(const alcop_gemm_desc* w, const alcop_schedule* s, int32_t nshards,
                       const alcop_shard* shards, int64_t granule);
/* Batch-sharded implicit-GEMM conv2d (images split one by one). */
int alcop_conv2d_sharded(const alcop_conv_desc* d, const alcop_schedule* s, int32_t nshards,
                         const alcop_shard* shards);

/* ---- analytical model (perf_model.hpp:157-187, tuner.hpp:68-80) -------- */
void alcop_hw_default_b200(alcop_hw* hw);
void alcop_hw_default_a100_reference(alcop_hw* hw); /* perf_model.hpp:14-30 defaults */
int alcop_predict(const alcop_gemm_desc* w, const alcop_schedule* s, const alcop_hw* hw,
                  alcop_breakdown* out);
int alcop_choose_schedule(const alcop_gemm_desc* w, const alcop_hw* hw, alcop_schedule* out);
/* The same for a conv, over the space of the kernel alcop_conv2d runs it on
 * (see there): the resident-filter kernel's ring depth x accumulators (its
 * own per-tile model: MMA, window fill, the SM's share of the HBM stream,
 * pipeline_latency over the windows), the GEMM space for 1x1 stride-1 convs,
 * else the implicit-GEMM kernel's space (tileK 64, equal stages; CTA pairs
 * when C % 64 == 0) ranked on the conv's GEMM view; the window modes'
 * space includes CTA pairs. */
int alcop_choose_conv_schedule(const alcop_conv_desc* d, const alcop_hw* hw, alcop_schedule* out);

/* One measured candidate of the model-assisted tuner. */
typedef struct {
  alcop_schedule schedule;
  double predicted_s; /* alcop_predict seconds */
  double measured_s;  /* CUDA-event time per launch */
} alcop_tune_trial;

/* Model-assisted tuning on real B200 timings (tuner.hpp:363-531, the
 * AnalyticalOnly method of tuner.hpp:407-413 with measure_ground_truth,
 * pipe_sim.hpp:195-239, replaced by the GPU): enumerate the B200 space,
 * rank by alcop_predict, time the top `budget` schedules on the caller's
 * buffers (steady-state CUDA-graph timing over rotating copies > 2x L2,
 * placed in the caller's `workspace` of alcop_tune_workspace_bytes(w)),
 * return the fastest in *best.  Whole-tile schedules only: stream_k is an
 * explicit opt-in (its workspace is shared per device). 
 * `trials` (may be NULL) receives up to `trials_cap` measured candidates in
 * rank order; *n_trials their count. */
int alcop_tune(const alcop_gemm_desc* w, const alcop_hw* hw, int32_t budget, const void* A, const void* B, void* C,
               void* workspace, int64_t workspace_bytes, void* stream, alcop_schedule* best,
               alcop_tune_trial* trials, int32_t trials_cap, int32_t* n_trials);
/* Device bytes alcop_tune needs for its rotating operand copies (> 2 x L2). */
int64_t alcop_tune_workspace_bytes(const alcop_gemm_desc* w);

/* ---- event-level pipeline simulation (pipe_sim.hpp:16-167) ------------ */
/* SimConfig (pipe_sim.hpp:16-22): nMplx workers share one compute unit, each
 * with nPipe chunk slots; loads take tLoad, uses tUse (serialised). */
typedef struct {
  double tLoad, tUse;
  int64_t nLoop;
  int32_t nPipe, nMplx;
} alcop_sim_config;

/* SimResult (pipe_sim.hpp:43-49) + comparable_worker_latency (:129-133). */
typedef struct {
  double makespan, firstComputeStart, busy, idleFraction;
  double comparable; /* per-worker latency comparable with the closed form */
} alcop_sim_result;

/* SimEvent (pipe_sim.hpp:24-40): kind 0 loadIssue, 1 loadDone,
 * 2 computeStart, 3 computeEnd. */
typedef struct {
  double time;
  int32_t worker, kind;
  int64_t iteration;
} alcop_sim_event;

/* simulate_pipeline (pipe_sim.hpp:55-127).  trace (may be NULL) receives up
 * to trace_cap events sorted by time (stable); *n_events = the full count.
 * Counts < 1 or negative times -> ALCOP_ERR_CONFIG "BadSimConfig". */
int alcop_simulate_pipeline(const alcop_sim_config* cfg, alcop_sim_result* out, alcop_sim_event* trace,
                            int64_t trace_cap, int64_t* n_events);
/* simulate_two_level (pipe_sim.hpp:138-167): fused != 0 lets inner loads run
 * ahead across outer chunks, 0 restarts the inner pipeline per outer chunk. */
int alcop_simulate_two_level(const alcop_sim_config* outer, const alcop_sim_config* inner, int32_t fused,
                             double* makespan);

/* B200 two-level kernel simulation (the event-level analogue of
 * alcop_predict, as measure_ground_truth is of perf::predict,
 * pipe_sim.hpp:195-239): per persistent CTA (pair), the outer level is the
 * n_stage smem ring (FUSED: loads run ahead across tiles; WRAP: the ring
 * restarts per tile with s-1 drained wrap loads), the inner level is the
 * n_stage_inner TMEM accumulator ring between the MMA issuer and the
 * epilogue.  Chunk load/use and epilogue times come from alcop_predict. */
typedef struct {
  double tKernel;     /* cycles */
  double seconds;
  double tBody;       /* first load -> last epilogue end, one CTA (pair) */
  double mmaBusy;     /* cycles the MMA issuer is busy */
  double mmaIdleFraction;
  double tMainLoopTile, tEpilogueTile, tLoadChunk, tUseChunk;
  int64_t tilesPerUnit, loads;
} alcop_sim_kernel;
int alcop_simulate_kernel(const alcop_gemm_desc* w, const alcop_schedule* s, const alcop_hw* hw,
                          alcop_sim_kernel* out);

#ifdef __cplusplus
}
#endif
#endif /* ALCOP_H_ */
