/*
 * alcop_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C restatement of the reference (/root/reference, "pipec") for the
 * pipelined load-and-use path, built into oracle/liboracle.so and driven from
 * tests/ through ctypes.  Each function cites the reference it restates.
 * Pinned against the reference itself (oracle/_ref/ref_driver, built from the
 * reference headers) through the golden fixtures in tests/golden/.
 *
 *  1. SplitMix64 / random_tensor        common.hpp:74-97, cli.hpp:41-46
 *  2. fp16 / bf16 <-> fp32 (RNE)         (IEEE 754 binary16, bfloat16)
 *  3. GEMM / BMM with fp32 accumulation  schedule.hpp:543-572 (mma nest) over
 *     fp16/bf16 inputs; int64 GEMM      interp.hpp:364-366 (integer mma)
 *  4. direct conv2d NHWC x KRSC          (no reference form)
 *  4b. sampled exact GEMM rows / columns and conv output pixels at benchmark
 *     scale (check_equivalence, interp.hpp:469-509, on samples)
 *  5. pipeline index algebra             pipeline_pass.hpp:482-552, 622-748
 *  6. interpreter group counters         interp.hpp:375-418 (+ the two-level
 *     drain leak of pipeline_pass.hpp:340-347,732-742 and its fix)
 *  7. analytical model                   perf_model.hpp:53-187
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- 1 */
static uint64_t sm_next(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

void oracle_random_tensor(int64_t count, uint64_t seed, int64_t lo, int64_t hi, int64_t* out) {
  uint64_t st = seed;
  uint64_t n = (uint64_t)(hi - lo + 1);
  for (int64_t i = 0; i < count; ++i) out[i] = lo + (int64_t)(sm_next(&st) % n);
}

/* ---------------------------------------------------------------- 2 */
static float half_to_float(uint16_t h) {
  uint32_t sign = (uint32_t)(h >> 15) << 31, exp = (h >> 10) & 0x1f, man = h & 0x3ff, bits;
  if (exp == 0) {
    if (man == 0) {
      bits = sign;
    } else { /* subnormal */
      int e = -1;
      do {
        ++e;
        man <<= 1;
      } while (!(man & 0x400));
      bits = sign | (uint32_t)(127 - 15 - e) << 23 | (man & 0x3ff) << 13;
    }
  } else if (exp == 31) {
    bits = sign | 0x7f800000u | man << 13;
  } else {
    bits = sign | (exp - 15 + 127) << 23 | man << 13;
  }
  float f;
  memcpy(&f, &bits, 4);
  return f;
}

static uint16_t float_to_half(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000;
  int32_t exp = (int32_t)((x >> 23) & 0xff);
  uint32_t man = x & 0x7fffff;
  if (exp == 255) return (uint16_t)(sign | 0x7c00 | (man ? 0x200 : 0));
  int32_t e = exp - 127 + 15;
  if (e >= 31) return (uint16_t)(sign | 0x7c00);
  if (e <= 0) {
    if (e < -10) return (uint16_t)sign;
    man |= 0x800000;
    uint32_t shift = (uint32_t)(14 - e);
    uint32_t h = man >> shift;
    uint32_t rem = man & ((1u << shift) - 1), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (h & 1))) ++h;
    return (uint16_t)(sign | h);
  }
  uint32_t h = (uint32_t)e << 10 | (man >> 13);
  uint32_t rem = man & 0x1fff;
  if (rem > 0x1000 || (rem == 0x1000 && (h & 1))) ++h;
  return (uint16_t)(sign | h);
}

static float bf16_to_float(uint16_t b) {
  uint32_t bits = (uint32_t)b << 16;
  float f;
  memcpy(&f, &bits, 4);
  return f;
}

static uint16_t float_to_bf16(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  if ((x & 0x7f800000u) == 0x7f800000u && (x & 0x7fffff)) return (uint16_t)((x >> 16) | 0x40);
  uint32_t lsb = (x >> 16) & 1;
  x += 0x7fff + lsb;
  return (uint16_t)(x >> 16);
}

/* dtype codes follow include/alcop.h: 0 f16, 1 bf16, 2 f32 */
static float load_elem(const void* p, int dt, int64_t i) {
  if (dt == 2) return ((const float*)p)[i];
  uint16_t v = ((const uint16_t*)p)[i];
  return dt == 1 ? bf16_to_float(v) : half_to_float(v);
}

static void store_elem(void* p, int dt, int64_t i, float v) {
  if (dt == 2)
    ((float*)p)[i] = v;
  else
    ((uint16_t*)p)[i] = dt == 1 ? float_to_bf16(v) : float_to_half(v);
}

void oracle_convert(const void* src, int src_dt, void* dst, int dst_dt, int64_t n) {
  for (int64_t i = 0; i < n; ++i) store_elem(dst, dst_dt, i, load_elem(src, src_dt, i));
}

/* ---------------------------------------------------------------- 3 */
/* C[b,m,n] = sum_k A[b,m,k] * B[b,k,n] (b_layout 0, the reference layout
 * schedule.hpp:388-390) or B[b,n,k] (b_layout 1); fp32 accumulation in k
 * order, like the C_reg f32 accumulator of the lowered nest (schedule.hpp:440,
 * 543-546). */
void oracle_gemm(int64_t M, int64_t N, int64_t K, int64_t batch, const void* A, const void* B, void* C, int in_dt,
                 int out_dt, int b_layout) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t m = 0; m < M; ++m) {
      float* row = (float*)malloc(sizeof(float) * (size_t)N);
      for (int64_t n = 0; n < N; ++n) row[n] = 0.f;
      for (int64_t k = 0; k < K; ++k) {
        float a = load_elem(A, in_dt, (b * M + m) * K + k);
        if (b_layout == 0) {
          for (int64_t n = 0; n < N; ++n) row[n] += a * load_elem(B, in_dt, (b * K + k) * N + n);
        } else {
          for (int64_t n = 0; n < N; ++n) row[n] += a * load_elem(B, in_dt, (b * N + n) * K + k);
        }
      }
      for (int64_t n = 0; n < N; ++n) store_elem(C, out_dt, (b * M + m) * N + n, row[n]);
      free(row);
    }
}

/* the interpreter's integer mma (interp.hpp:364-366): exact int64 */
void oracle_gemm_i64(int64_t M, int64_t N, int64_t K, int64_t batch, const int64_t* A, const int64_t* B,
                     int64_t* C) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t m = 0; m < M; ++m)
      for (int64_t n = 0; n < N; ++n) {
        int64_t acc = 0;
        for (int64_t k = 0; k < K; ++k) acc += A[(b * M + m) * K + k] * B[(b * K + k) * N + n];
        C[(b * M + m) * N + n] = acc;
      }
}

/* ---------------------------------------------------------------- 4 */
void oracle_conv2d(int64_t N, int64_t H, int64_t W, int64_t Cin, int64_t Kout, int64_t R, int64_t S, int sh, int sw,
                   int ph, int pw, const void* x, const void* w, void* y, int in_dt, int out_dt) {
  const int64_t P = (H + 2 * ph - R) / sh + 1, Q = (W + 2 * pw - S) / sw + 1;
#pragma omp parallel for collapse(3) schedule(static)
  for (int64_t n = 0; n < N; ++n)
    for (int64_t p = 0; p < P; ++p)
      for (int64_t q = 0; q < Q; ++q)
        for (int64_t k = 0; k < Kout; ++k) {
          float acc = 0.f;
          for (int64_t r = 0; r < R; ++r) {
            const int64_t h = p * sh - ph + r;
            if (h < 0 || h >= H) continue;
            for (int64_t s = 0; s < S; ++s) {
              const int64_t ww = q * sw - pw + s;
              if (ww < 0 || ww >= W) continue;
              for (int64_t c = 0; c < Cin; ++c)
                acc += load_elem(x, in_dt, ((n * H + h) * W + ww) * Cin + c) *
                       load_elem(w, in_dt, ((k * R + r) * S + s) * Cin + c);
            }
          }
          store_elem(y, out_dt, ((n * P + p) * Q + q) * Kout + k, acc);
        }
}

/* ---------------------------------------------------------------- 4b */
/* Sampled exact checks at benchmark scale (the reference's check_equivalence,
 * interp.hpp:469-509, compares every transformed program against the
 * untransformed one; at 16384^3 the checker evaluates sampled rows, columns
 * and output pixels instead of the whole product).
 *
 * Inputs are the reference's D-int draws (SplitMix64 range(-8,8),
 * cli.hpp:41-46) stored as int8.  Every partial sum is bounded by 64*K
 * (< 2^31 for K < 2^25), so int32 accumulation is the interpreter's int64 mma
 * (interp.hpp:364-366) exactly; results are widened to int64. */

/* the same draws as oracle_random_tensor, element-parallel (SplitMix64 is a
 * counter generator: draw i is mix(seed + (i+1)*gamma)) */
void oracle_random_i8(int64_t count, uint64_t seed, int64_t lo, int64_t hi, int8_t* out) {
  const uint64_t n = (uint64_t)(hi - lo + 1);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) {
    uint64_t z = seed + (uint64_t)(i + 1) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    out[i] = (int8_t)(lo + (int64_t)(z % n));
  }
}

/* C rows `rows[i]` (global row = b*M + m) of C = A @ B:
 * A [batch,M,K] int8, B [batch,K,N] (b_layout 0) or [batch,N,K] (1) int8;
 * out [nrows, N] int64.  Parallel over (row, column block); each thread
 * streams the rows of B once per row block. */
void oracle_gemm_rows_i8(int64_t M, int64_t N, int64_t K, int64_t batch, const int8_t* A, const int8_t* B,
                         int b_layout, int64_t nrows, const int64_t* rows, int64_t* out) {
  const int64_t JB = 2048;
  const int64_t nj = (N + JB - 1) / JB;
  (void)batch;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int64_t i = 0; i < nrows; ++i)
    for (int64_t jb = 0; jb < nj; ++jb) {
      const int64_t r = rows[i], b = r / M;
      const int8_t* a = A + r * K;
      const int64_t j0 = jb * JB, j1 = j0 + JB < N ? j0 + JB : N;
      int32_t acc[2048];
      for (int64_t j = 0; j < j1 - j0; ++j) acc[j] = 0;
      if (b_layout == 0) {
        const int8_t* bb = B + b * K * N;
        for (int64_t k = 0; k < K; ++k) {
          const int32_t av = a[k];
          const int8_t* brow = bb + k * N + j0;
          for (int64_t j = 0; j < j1 - j0; ++j) acc[j] += av * (int32_t)brow[j];
        }
      } else {
        const int8_t* bb = B + b * N * K;
        for (int64_t j = 0; j < j1 - j0; ++j) {
          const int8_t* bcol = bb + (j0 + j) * K;
          int32_t s = 0;
          for (int64_t k = 0; k < K; ++k) s += (int32_t)a[k] * (int32_t)bcol[k];
          acc[j] = s;
        }
      }
      for (int64_t j = 0; j < j1 - j0; ++j) out[i * N + j0 + j] = acc[j];
    }
}

/* C columns `cols[j]` of every row of every batch: out [batch*M, ncols] int64 */
void oracle_gemm_cols_i8(int64_t M, int64_t N, int64_t K, int64_t batch, const int8_t* A, const int8_t* B,
                         int b_layout, int64_t ncols, const int64_t* cols, int64_t* out) {
  for (int64_t b = 0; b < batch; ++b) {
    /* gather the sampled columns of B_b as [K, ncols] int32 */
    int32_t* bp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(K * ncols));
    for (int64_t k = 0; k < K; ++k)
      for (int64_t j = 0; j < ncols; ++j)
        bp[k * ncols + j] = b_layout == 0 ? B[(b * K + k) * N + cols[j]] : B[(b * N + cols[j]) * K + k];
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
      int32_t* acc = (int32_t*)calloc((size_t)ncols, sizeof(int32_t));
      const int8_t* a = A + (b * M + m) * K;
      for (int64_t k = 0; k < K; ++k) {
        const int32_t av = a[k];
        const int32_t* br = bp + k * ncols;
        for (int64_t j = 0; j < ncols; ++j) acc[j] += av * br[j];
      }
      for (int64_t j = 0; j < ncols; ++j) out[(b * M + m) * ncols + j] = acc[j];
      free(acc);
    }
    free(bp);
  }
}

/* direct conv2d (as oracle_conv2d) at output pixels pts[i] = (n, p, q), all K
 * channels: x NHWC int8, w KRSC int8, out [npts, K] int64 */
void oracle_conv2d_points_i8(int64_t N, int64_t H, int64_t W, int64_t Cin, int64_t Kout, int64_t R, int64_t S,
                             int sh, int sw, int ph, int pw, const int8_t* x, const int8_t* w, int64_t npts,
                             const int64_t* pts, int64_t* out) {
  (void)N;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t i = 0; i < npts; ++i) {
    const int64_t n = pts[3 * i], p = pts[3 * i + 1], q = pts[3 * i + 2];
    for (int64_t k = 0; k < Kout; ++k) {
      int32_t acc = 0;
      for (int64_t r = 0; r < R; ++r) {
        const int64_t h = p * sh - ph + r;
        if (h < 0 || h >= H) continue;
        for (int64_t s = 0; s < S; ++s) {
          const int64_t ww = q * sw - pw + s;
          if (ww < 0 || ww >= W) continue;
          const int8_t* xp = x + ((n * H + h) * W + ww) * Cin;
          const int8_t* wp = w + ((k * R + r) * S + s) * Cin;
          for (int64_t c = 0; c < Cin; ++c) acc += (int32_t)xp[c] * (int32_t)wp[c];
        }
      }
      out[i * Kout + k] = acc;
    }
  }
}

/* ---------------------------------------------------------------- 5 */
/* floor-mod with non-negative remainder (expr.hpp:56-62) */
static int64_t fmod_i(int64_t a, int64_t b) {
  int64_t r = a % b;
  return r < 0 ? r + b : r;
}
static int64_t fdiv_i(int64_t a, int64_t b) { return (a - fmod_i(a, b)) / b; }

/* Root pipeline over v (extent E, stages s), pipeline_pass.hpp:501-509 and
 * the prologue clones v := c-(s-1) of pipeline_pass.hpp:647-656.
 * Fills (s-1)+E producer (slot, chunk) pairs and E consumer slots. */
void oracle_root_schedule(int64_t E, int64_t s, int64_t* prod_slot, int64_t* prod_chunk, int64_t* cons_slot) {
  int64_t i = 0;
  for (int64_t c = 0; c < s - 1; ++c, ++i) {
    int64_t v = c - (s - 1);
    prod_slot[i] = fmod_i(v + s - 1, s);
    prod_chunk[i] = fmod_i(v + s - 1, E);
  }
  for (int64_t v = 0; v < E; ++v, ++i) {
    prod_slot[i] = fmod_i(v + s - 1, s);
    prod_chunk[i] = fmod_i(v + s - 1, E);
    cons_slot[v] = fmod_i(v, s);
  }
}

/* Nested pipeline over u (extent F, stages t) under parent v (extent E,
 * stages s), pipeline_pass.hpp:510-527 (+ consumer 489-492): for each (v,u)
 * the inner producer's dst slot, source outer slot, source inner offset and
 * source outer chunk; the consumer slot.  Prologue (657-676): at v==0, m in
 * [0,t-1) with u := m-(t-1). Arrays hold (t-1) prologue rows then E*F rows. */
void oracle_nested_schedule(int64_t E, int64_t F, int64_t s, int64_t t, int64_t* dst_slot, int64_t* src_slot,
                            int64_t* src_u, int64_t* src_v, int64_t* cons_slot) {
  int64_t i = 0;
  for (int64_t m = 0; m < t - 1; ++m, ++i) {
    int64_t v = 0, u = m - (t - 1);
    int64_t g = v * F + u + t - 1;
    dst_slot[i] = fmod_i(g, t);
    src_slot[i] = fmod_i(fdiv_i(g, F), s);
    src_u[i] = fmod_i(g, F);
    src_v[i] = fmod_i(fdiv_i(g, F), E);
  }
  for (int64_t v = 0; v < E; ++v)
    for (int64_t u = 0; u < F; ++u, ++i) {
      int64_t g = v * F + u + t - 1;
      dst_slot[i] = fmod_i(g, t);
      src_slot[i] = fmod_i(fdiv_i(g, F), s);
      src_u[i] = fmod_i(g, F);
      src_v[i] = fmod_i(fdiv_i(g, F), E);
      cons_slot[v * F + u] = fmod_i(v * F + u, t);
    }
}

/* ---------------------------------------------------------------- 6 */
/* Sync event stream of the transformed GEMM nest, with the interpreter's
 * group counters after each event (interp.hpp:375-418, TraceEvent
 * interp.hpp:20-26).  Groups: 0 A_shared, 1 A_reg, 2 B_shared, 3 B_reg
 * (plan order, pipeline_pass.hpp:349-365).  stages 0 = not pipelined.
 * Event record: {kind (0 acquire,1 commit,2 wait,3 release), group,
 * acquired, committed, waited, released, inflight}.
 * leak_fix = 1 appends dmax x consumer_release <parent> after the root
 * drains (the validated fix for pipeline_pass.hpp:340-347/732-742). */
typedef struct {
  int64_t acq, com, wai, rel;
} grp_t;

typedef struct {
  int64_t* out;
  int64_t cap, n;
  grp_t g[4];
} emit_t;

static void ev(emit_t* e, int kind, int grp) {
  grp_t* g = &e->g[grp];
  if (kind == 0) g->acq++;
  if (kind == 1) g->com++;
  if (kind == 2) g->wai++;
  if (kind == 3) g->rel++;
  if (e->n < e->cap) {
    int64_t* r = e->out + e->n * 7;
    r[0] = kind;
    r[1] = grp;
    r[2] = g->acq;
    r[3] = g->com;
    r[4] = g->wai;
    r[5] = g->rel;
    r[6] = g->com - g->rel;
  }
  e->n++;
}

int64_t oracle_sync_trace(int64_t tiles, int64_t E, int64_t F, int64_t sA, int64_t sB, int64_t tA, int64_t tB,
                          int leak_fix, int64_t* out, int64_t cap) {
  /* restated shapes: per side either no register hint, or both levels hinted */
  if ((tA >= 2 && sA < 2) || (tB >= 2 && sB < 2)) return -1;
  emit_t e;
  memset(&e, 0, sizeof e);
  e.out = out;
  e.cap = cap;
  const int64_t s[2] = {sA, sB}, t[2] = {tA, tB};
  /* predicateWaits = ceil((t-1)/F) when nested (pipeline_pass.hpp:313) */
  int64_t pw[2], drainRoot[2], drainChild[2];
  for (int x = 0; x < 2; ++x) {
    int nested = s[x] >= 2 && t[x] >= 2;
    pw[x] = nested ? (t[x] - 1 + F - 1) / F : 0;
    drainRoot[x] = s[x] >= 2 ? s[x] - 1 - pw[x] : 0; /* dmax over its child */
    drainChild[x] = t[x] >= 2 ? t[x] - 1 : 0;
  }
  for (int64_t tile = 0; tile < tiles; ++tile) {
    /* root prologues before the ko loop, A then B (pipeline_pass.hpp:647-656) */
    for (int x = 0; x < 2; ++x)
      if (s[x] >= 2)
        for (int64_t c = 0; c < s[x] - 1; ++c) {
          ev(&e, 0, 2 * x);
          ev(&e, 1, 2 * x);
        }
    for (int64_t v = 0; v < E; ++v) {
      if (v == 0)
        for (int x = 0; x < 2; ++x)
          if (s[x] >= 2 && t[x] >= 2) { /* predicated inner prologue, head of ko body */
            for (int64_t w = 0; w < pw[x]; ++w) ev(&e, 2, 2 * x);
            for (int64_t m = 0; m < t[x] - 1; ++m) {
              ev(&e, 0, 2 * x + 1);
              ev(&e, 1, 2 * x + 1);
            }
          }
      for (int x = 0; x < 2; ++x)
        if (s[x] >= 2) {
          ev(&e, 0, 2 * x);
          ev(&e, 1, 2 * x);
        }
      for (int x = 0; x < 2; ++x)
        if (s[x] >= 2) ev(&e, 2, 2 * x);
      for (int64_t u = 0; u < F; ++u) {
        for (int x = 0; x < 2; ++x)
          if (t[x] >= 2) {
            ev(&e, 0, 2 * x + 1);
            ev(&e, 1, 2 * x + 1);
          }
        for (int x = 0; x < 2; ++x)
          if (t[x] >= 2) ev(&e, 2, 2 * x + 1);
        for (int x = 0; x < 2; ++x)
          if (t[x] >= 2) ev(&e, 3, 2 * x + 1);
      }
      for (int x = 0; x < 2; ++x)
        if (s[x] >= 2) ev(&e, 3, 2 * x);
    }
    /* drains after the root loop, plan order A_shared, A_reg, B_shared, B_reg
     * (pipeline_pass.hpp:732-742) */
    for (int x = 0; x < 2; ++x) {
      if (s[x] >= 2) {
        for (int64_t d = 0; d < drainRoot[x]; ++d) {
          ev(&e, 2, 2 * x);
          ev(&e, 3, 2 * x);
        }
        if (t[x] >= 2)
          for (int64_t d = 0; d < drainChild[x]; ++d) {
            ev(&e, 2, 2 * x + 1);
            ev(&e, 3, 2 * x + 1);
          }
        if (leak_fix)
          for (int64_t d = 0; d < pw[x]; ++d) ev(&e, 3, 2 * x);
      }
    }
  }
  return e.n;
}

/* ---------------------------------------------------------------- 7 */
/* perf_model.hpp:14-30 field order */
typedef struct {
  int numSM;
  double throughputSM, bwLLC, bwDRAM, bwDRAMWrite, latLLCRead, latDRAMRead, latDRAMWrite, bwSmem, latSmem;
  int64_t smemPerSM, regsPerSM;
  int maxThreadblkPerSM, maxWarpsPerSM, utilKneeWarps;
} oracle_hw;

void oracle_hw_default(oracle_hw* h) {
  h->numSM = 108;
  h->throughputSM = 1024;
  h->bwLLC = 512;
  h->bwDRAM = 64;
  h->bwDRAMWrite = 32;
  h->latLLCRead = 200;
  h->latDRAMRead = 400;
  h->latDRAMWrite = 400;
  h->bwSmem = 128;
  h->latSmem = 25;
  h->smemPerSM = 163840;
  h->regsPerSM = 262144;
  h->maxThreadblkPerSM = 32;
  h->maxWarpsPerSM = 64;
  h->utilKneeWarps = 8;
}

double oracle_pipeline_latency(double tLoad, double tUse, int64_t nLoop, int nPipe, int nMplx) {
  if (tLoad <= ((double)nPipe * nMplx - 1) * tUse) return tUse * (double)nLoop;
  return (tLoad + tUse) * (double)nLoop / nPipe;
}

static double util_(int nWarp, int64_t nTb, const oracle_hw* h) {
  double w = (double)nWarp * (double)nTb;
  double u = w / h->utilKneeWarps;
  return u < 1.0 ? u : 1.0;
}

double oracle_compute_latency(int64_t flops, const oracle_hw* h, int nWarp, int64_t nTb) {
  if (flops == 0) return 0;
  return (double)flops / (h->throughputSM * util_(nWarp, nTb, h));
}

double oracle_smem_load_latency(int64_t bytes, int64_t workset, int64_t nTbPerBatch, const oracle_hw* h) {
  double llc = h->latLLCRead + (double)bytes * (double)nTbPerBatch / h->bwLLC;
  double dram = h->latDRAMRead + (double)workset / h->bwDRAM;
  return llc > dram ? llc : dram;
}

double oracle_epilogue_latency(int64_t bytes, int64_t nTbPerBatch, const oracle_hw* h) {
  return h->latDRAMWrite + (double)bytes * (double)nTbPerBatch / h->bwDRAMWrite;
}

/* predict(): out[0..10] = tKernel tThreadblk tInit tMainLoop tEpilogue
 * tSmemLoad tRegLoad tSmemUse tCompute nThreadblkBatch nThreadblkPerSM.
 * p = {M,N,K,batch,tileM,tileN,tileK,regTileM,regTileN,regTileK,
 *      nSmemPipeStage,nRegPipeStage,nWarpPerThreadblk}; elemBytes = 2.
 * Returns 0, or -1 when params_valid fails / no threadblock fits. */
int oracle_predict(const int64_t* p, const oracle_hw* h, double* out) {
  const int64_t M = p[0], N = p[1], K = p[2], batch = p[3], tM = p[4], tN = p[5], tK = p[6], rM = p[7], rN = p[8],
                rK = p[9];
  const int sS = (int)p[10], sR = (int)p[11], nW = (int)p[12];
  const int64_t eb = 2;
  /* params_valid, perf_model.hpp:129-142 */
  if (tM < 1 || tN < 1 || tK < 1 || rM < 1 || rN < 1 || rK < 1 || nW < 1) return -1;
  if (sS < 2 || sR < 2) return -1;
  if (M % tM || N % tN || K % tK) return -1;
  if (tM % rM || tN % rN || tK % rK) return -1;
  if ((int64_t)nW * rM * rN != tM * tN) return -1;
  if ((int64_t)(sR - 1) > (int64_t)(sS - 1) * (tK / rK)) return -1;
  /* occupancy, perf_model.hpp:110-127 */
  int64_t smem = (tM * tK + tK * tN) * eb * sS;
  int64_t regs = ((rM * rK + rK * rN) * eb * sR + rM * rN * 4) * nW;
  int64_t bySmem = h->smemPerSM / (smem > 1 ? smem : 1);
  int64_t byReg = h->regsPerSM / (regs > 1 ? regs : 1);
  int64_t byWarps = h->maxWarpsPerSM / (nW > 1 ? nW : 1);
  int64_t tbPerSM = h->maxThreadblkPerSM;
  if (bySmem < tbPerSM) tbPerSM = bySmem;
  if (byReg < tbPerSM) tbPerSM = byReg;
  if (byWarps < tbPerSM) tbPerSM = byWarps;
  if (tbPerSM < 1) return -1;
  int64_t total = (M / tM) * (N / tN) * batch;
  int64_t perBatch = tbPerSM * h->numSM;
  int64_t nBatch = (total + perBatch - 1) / perBatch;
  /* predict, perf_model.hpp:157-187 */
  int64_t nSmemLoop = K / tK, nRegLoop = tK / rK;
  int64_t flopsOne = 2 * rM * rN * rK;
  int64_t bytesOne = (tM + tN) * tK * eb;
  int64_t nJ = N / tN;
  int64_t rows = (perBatch + nJ - 1) / nJ;
  int64_t cols = perBatch < nJ ? perBatch : nJ;
  int64_t workset = rows * tM * tK * eb + cols * tK * tN * eb;
  int64_t outTile = tM * tN * eb;
  double tCompute = oracle_compute_latency(flopsOne, h, nW, tbPerSM);
  double tRegLoad = h->latSmem + (double)((rM * rK + rK * rN) * eb) / h->bwSmem;
  double tSmemLoad = oracle_smem_load_latency(bytesOne, workset, perBatch, h);
  double tSmemUse = oracle_pipeline_latency(tRegLoad, tCompute, nRegLoop, sR, nW);
  double tMain = oracle_pipeline_latency(tSmemLoad, tSmemUse, nSmemLoop, sS, (int)tbPerSM);
  double tInit = tSmemLoad + tRegLoad;
  double tEpi = oracle_epilogue_latency(outTile, perBatch, h);
  double tTb = tInit + tMain + tEpi;
  out[0] = tTb * (double)nBatch;
  out[1] = tTb;
  out[2] = tInit;
  out[3] = tMain;
  out[4] = tEpi;
  out[5] = tSmemLoad;
  out[6] = tRegLoad;
  out[7] = tSmemUse;
  out[8] = tCompute;
  out[9] = (double)nBatch;
  out[10] = (double)tbPerSM;
  return 0;
}
