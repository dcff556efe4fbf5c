/*
 * dlx_oracle.c — plain-C restatement of the DiLoCoX outer-sync path.
 *
 * TEST INFRASTRUCTURE ONLY (see dlx_oracle.h). This is the CPU checker the CUDA path is
 * compared against; it is never linked into or called by the product library.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the reference
 * itself (oracle/_ref/libdlxref.so, compiled from /root/reference by oracle/Makefile) and
 * against the committed golden vectors in tests/golden/ (generated from the reference by
 * tests/golden/gen_golden.py). Bit-exact except orc_singular_values, which uses cyclic
 * Jacobi instead of the reference's Householder+QL (agreement ~1e-12 relative; the
 * derived effective ranks are equal except at exact tau ties).
 *
 * Citations are to /root/reference/proj/core/{include/dilocox,src}/ file:line.
 * Build: -ffp-contract=off (proj/CMakeLists.txt:15): every float op rounds separately.
 */
#include "dlx_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* orc_last_error(void) { return g_err; }
const char* orc_backend(void) { return "restatement"; }

/* ---------------------------------------------------------------- RNG (rng.hpp:11-66) */

static const uint64_t GOLDEN = 0x9e3779b97f4a7c15ull;

/* splitmix64 finaliser; rng.hpp:23-28 (mix) and :30-35 (next_u64 after the increment) */
static uint64_t fmix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static uint64_t mix64(uint64_t z) { return fmix(z + GOLDEN); }

uint64_t orc_stream_init(uint64_t seed, uint64_t stream_id) { /* rng.hpp:13-16 */
  uint64_t s = mix64(seed ^ GOLDEN);
  return mix64(s ^ mix64(stream_id + 0xbf58476d1ce4e5b9ull));
}

uint64_t orc_stream_key(const uint64_t* parts, int n) { /* rng.hpp:63-66 */
  uint64_t h = 0x100000001b3ull;
  for (int i = 0; i < n; ++i) h = mix64(h ^ mix64(parts[i]));
  return h;
}

uint64_t orc_next_u64(uint64_t* st) { /* rng.hpp:25-31: counter += gamma, finalise */
  *st += GOLDEN;
  return fmix(*st);
}

static float unit_f(uint64_t* st) { /* rng.hpp:37: top 24 bits */
  return (float)(orc_next_u64(st) >> 40) * 0x1.0p-24f;
}
static double unit_d(uint64_t* st) { /* rng.hpp:34 */
  return (double)(orc_next_u64(st) >> 11) * 0x1.0p-53;
}

void orc_uniform(uint64_t* st, int64_t n, float lo, float hi, float* out) {
  /* Tensor::uniform tensor.cpp:43-47 -> RngStream::uniform rng.hpp:39 */
  const float span = hi - lo;
  for (int64_t i = 0; i < n; ++i) {
    const float u = unit_f(st);
    const float t = span * u;
    out[i] = lo + t;
  }
}

void orc_gaussian(uint64_t* st, int64_t n, float* out) {
  /* Tensor::gaussian tensor.cpp:49-53 -> RngStream::normal rng.hpp:52-56 (Irwin-Hall 12) */
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int k = 0; k < 12; ++k) s += unit_d(st);
    out[i] = (float)(s - 6.0);
  }
}

/* ------------------------------------------------------- GEMMs (tensor.cpp:67-155) */
/* Each output accumulates float products in double over ascending k, cast once. */

int orc_matmul(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c) {
  /* tensor.cpp:70-96: C[m,n] = A[m,k] B[k,n] */
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int64_t p = 0; p < k; ++p) acc += (double)a[i * k + p] * (double)b[p * n + j];
      c[i * n + j] = (float)acc;
    }
  return 0;
}

int orc_matmul_tn(int64_t k, int64_t m, int64_t n, const float* a, const float* b, float* c) {
  /* tensor.cpp:98-131: C[m,n] = A[k,m]^T B[k,n] */
  double* acc = calloc((size_t)(m * n), sizeof(double));
  if (!acc) return fail(9, "oom");
  for (int64_t p = 0; p < k; ++p)
    for (int64_t i = 0; i < m; ++i) {
      const double av = (double)a[p * m + i];
      for (int64_t j = 0; j < n; ++j) acc[i * n + j] += av * (double)b[p * n + j];
    }
  for (int64_t i = 0; i < m * n; ++i) c[i] = (float)acc[i];
  free(acc);
  return 0;
}

int orc_matmul_nt(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c) {
  /* tensor.cpp:133-155: C[m,n] = A[m,k] B[n,k]^T */
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int64_t p = 0; p < k; ++p) acc += (double)a[i * k + p] * (double)b[j * k + p];
      c[i * n + j] = (float)acc;
    }
  return 0;
}

/* ------------------------------------------- orthonormalisation (tensor.cpp:174-227) */
/* Modified Gram-Schmidt, two passes per column, fp64 column-major scratch. A column
 * whose residual norm is <= 1e-7 * max(1, largest input column norm) is replaced by
 * uniform(-1,1) draws from RngStream(0x5eedc01, stream_key({n, r, j, attempt})). */
int orc_orthonormalize(int64_t n, int64_t r, const float* in, float* out, int* replaced) {
  if (n < r) return fail(2, "orthonormalize: need rows >= cols");
  double* col = malloc(sizeof(double) * (size_t)(n * r));
  float* tmp = malloc(sizeof(float) * (size_t)n);
  if (!col || !tmp) return fail(9, "oom");
  double big = 0.0;
  for (int64_t j = 0; j < r; ++j) {
    double ss = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double v = (double)in[i * r + j];
      col[j * n + i] = v;
      ss += v * v;
    }
    const double nrm = sqrt(ss);
    if (nrm > big) big = nrm;
  }
  const double tol = 1e-7 * (big > 1.0 ? big : 1.0);
  int nrep = 0;
  for (int64_t j = 0; j < r; ++j) {
    double* cj = col + j * n;
    for (int attempt = 0;; ++attempt) {
      for (int pass = 0; pass < 2; ++pass)
        for (int64_t p = 0; p < j; ++p) {
          const double* cp = col + p * n;
          double dot = 0.0;
          for (int64_t i = 0; i < n; ++i) dot += cj[i] * cp[i];
          for (int64_t i = 0; i < n; ++i) cj[i] -= dot * cp[i];
        }
      double ss = 0.0;
      for (int64_t i = 0; i < n; ++i) ss += cj[i] * cj[i];
      const double nrm = sqrt(ss);
      if (nrm > tol) {
        const double inv = 1.0 / nrm;
        for (int64_t i = 0; i < n; ++i) cj[i] *= inv;
        break;
      }
      const uint64_t key[4] = {(uint64_t)n, (uint64_t)r, (uint64_t)j, (uint64_t)attempt};
      uint64_t st = orc_stream_init(0x5eedc01u, orc_stream_key(key, 4));
      orc_uniform(&st, n, -1.0f, 1.0f, tmp);
      for (int64_t i = 0; i < n; ++i) cj[i] = (double)tmp[i];
      if (attempt == 0) ++nrep;
    }
  }
  for (int64_t j = 0; j < r; ++j)
    for (int64_t i = 0; i < n; ++i) out[i * r + j] = (float)col[j * n + i];
  if (replaced) *replaced = nrep;
  free(col);
  free(tmp);
  return 0;
}

/* --------------------------------------------------------- singular values (Jacobi) */
/* Reference: Gram on the shorter side (tensor.cpp:330-353), Householder + implicit QL
 * (:234-321), sorted descending, sqrt(max(0, .)). Restated with cyclic Jacobi on the
 * same fp64 Gram. */
static void jacobi_eigvals(double* A, int n, double* w) {
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < n; ++i) {
      diag += A[i * n + i] * A[i * n + i];
      for (int j = i + 1; j < n; ++j) off += A[i * n + j] * A[i * n + j];
    }
    if (off <= 1e-30 * diag || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p * n + q];
        if (apq == 0.0) continue;
        const double app = A[p * n + p], aqq = A[q * n + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A[k * n + p], akq = A[k * n + q];
          A[k * n + p] = c * akp - s * akq;
          A[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A[p * n + k], aqk = A[q * n + k];
          A[p * n + k] = c * apk - s * aqk;
          A[q * n + k] = s * apk + c * aqk;
        }
      }
  }
  for (int i = 0; i < n; ++i) w[i] = A[i * n + i];
}

static int cmp_desc(const void* x, const void* y) {
  const double a = *(const double*)x, b = *(const double*)y;
  return (a < b) - (a > b);
}

int orc_singular_values(int64_t a, int64_t b, const float* m, double* sv) {
  const int n = (int)(a < b ? a : b);
  double* g = calloc((size_t)n * (size_t)n, sizeof(double));
  if (!g) return fail(9, "oom");
  if (a <= b) {
    for (int64_t i = 0; i < a; ++i)
      for (int64_t j = 0; j <= i; ++j) {
        double s = 0.0;
        for (int64_t k = 0; k < b; ++k) s += (double)m[i * b + k] * (double)m[j * b + k];
        g[i * n + j] = g[j * n + i] = s;
      }
  } else {
    for (int64_t p = 0; p < a; ++p)
      for (int64_t i = 0; i < b; ++i) {
        const double v = (double)m[p * b + i];
        for (int64_t j = 0; j <= i; ++j) g[i * n + j] += v * (double)m[p * b + j];
      }
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) g[i * n + j] = g[j * n + i];
  }
  jacobi_eigvals(g, n, sv);
  qsort(sv, (size_t)n, sizeof(double), cmp_desc);
  for (int i = 0; i < n; ++i) sv[i] = sqrt(sv[i] > 0.0 ? sv[i] : 0.0);
  free(g);
  return 0;
}

/* -------------------------------------------------------------- low rank (compress.cpp:56-78) */

static float* orth_alloc(int64_t n, int64_t r, const float* in) {
  float* o = malloc(sizeof(float) * (size_t)(n * r));
  if (o) orc_orthonormalize(n, r, in, o, NULL);
  return o;
}

int orc_lowrank_approx(int64_t a, int64_t b, const float* m, int r, const float* warm_q,
                       int iters, uint64_t* st, float* p_out, float* q_out) {
  if (r < 1 || r > (a < b ? a : b)) return fail(1, "lowrank_approx: rank out of range");
  if (iters < 1) return fail(1, "lowrank_approx: iters must be >= 1");
  float* q = malloc(sizeof(float) * (size_t)(b * r));
  float* y = malloc(sizeof(float) * (size_t)((a > b ? a : b) * r));
  if (!q || !y) return fail(9, "oom");
  if (warm_q) {
    memcpy(q, warm_q, sizeof(float) * (size_t)(b * r));
  } else { /* cold start: b x r uniform(-1,1) from the shared stream, row-major */
    orc_uniform(st, b * r, -1.0f, 1.0f, y);
    orc_orthonormalize(b, r, y, q, NULL);
  }
  for (int it = 0; it < iters; ++it) {
    orc_matmul(a, b, r, m, q, y); /* Y = M Q */
    float* p = orth_alloc(a, r, y);
    orc_matmul_tn(a, b, r, m, p, y); /* Z = M^T P */
    orc_orthonormalize(b, r, y, q, NULL);
    free(p);
  }
  orc_matmul(a, b, r, m, q, p_out); /* P = M Q carries the magnitudes */
  memcpy(q_out, q, sizeof(float) * (size_t)(b * r));
  free(q);
  free(y);
  return 0;
}

/* ------------------------------------------------------------ quantise (compress.cpp:24-54) */

int orc_quantize(const float* x, int64_t n, int qbits, int rounding, uint64_t* st,
                 int8_t* codes, float* scale) {
  if (qbits < 2 || qbits > 8) return fail(1, "quantization bits must be in [2, 8]");
  float mx = 0.0f;
  for (int64_t i = 0; i < n; ++i) {
    const float ax = fabsf(x[i]);
    mx = mx < ax ? ax : mx;
  }
  if (n > 0) memset(codes, 0, (size_t)n);
  *scale = 0.0f;
  if (mx == 0.0f) return 0; /* all-zero chunk: scale 0, codes 0, no draws */
  const int L = (1 << (qbits - 1)) - 1;
  const float s = mx / (float)L;
  const float inv = 1.0f / s;
  *scale = s;
  for (int64_t i = 0; i < n; ++i) {
    const float y = x[i] * inv;
    int c;
    if (rounding != 0) {
      c = (int)lrintf(y); /* round half to even */
    } else {
      const float fl = floorf(y);
      const float frac = y - fl;
      c = (int)fl + (unit_f(st) < frac ? 1 : 0);
    }
    if (c < -L) c = -L;
    if (c > L) c = L;
    codes[i] = (int8_t)c;
  }
  return 0;
}

/* ------------------------------------------------------------------ tables / payload */

static int64_t numel(const int* ndim, const int64_t* dims, int i) {
  return ndim[i] == 2 ? dims[2 * i] * dims[2 * i + 1] : dims[2 * i];
}
static int reff(const int* ndim, const int64_t* dims, int i, int rank) {
  if (ndim[i] != 2) return 0;
  int64_t m = dims[2 * i] < dims[2 * i + 1] ? dims[2 * i] : dims[2 * i + 1];
  return (int)(rank < m ? rank : m);
}

int64_t orc_codes_count(int nt, const int* ndim, const int64_t* dims, const int* ranks) {
  int64_t c = 0;
  for (int i = 0; i < nt; ++i)
    c += ndim[i] == 2 ? (dims[2 * i] + dims[2 * i + 1]) * ranks[i] : dims[2 * i];
  return c;
}
int64_t orc_scales_count(int nt, const int* ndim, const int64_t* dims, const int* ranks) {
  (void)dims;
  int64_t c = 0;
  for (int i = 0; i < nt; ++i) c += ndim[i] == 2 ? 2 * ranks[i] : 1;
  return c;
}
int64_t orc_qfactor_count(int nt, const int* ndim, const int64_t* dims, const int* ranks) {
  int64_t c = 0;
  for (int i = 0; i < nt; ++i)
    if (ndim[i] == 2) c += dims[2 * i + 1] * ranks[i];
  return c;
}

uint64_t orc_payload_bits(int nt, const int* ndim, const int64_t* dims, const int* ranks,
                          int qbits) { /* compress.cpp:92-114 */
  uint64_t bits = 0;
  for (int i = 0; i < nt; ++i) {
    if (ndim[i] == 2)
      bits += (uint64_t)(dims[2 * i] + dims[2 * i + 1]) * (uint64_t)ranks[i] * (uint64_t)qbits +
              64ull * (uint64_t)ranks[i];
    else
      bits += (uint64_t)dims[2 * i] * (uint64_t)qbits + 32ull;
  }
  return bits;
}

/* Per-column quantisation of an n x r row-major factor; codes column-major
 * (compress.cpp:119-131). */
static void quantize_factor(const float* f, int64_t n, int r, int qbits, int rounding,
                            uint64_t* st, int8_t* codes, float* scales, float* colbuf) {
  for (int j = 0; j < r; ++j) {
    for (int64_t i = 0; i < n; ++i) colbuf[i] = f[i * r + j];
    orc_quantize(colbuf, n, qbits, rounding, st, codes + (int64_t)j * n, scales + j);
  }
}

int orc_compress(int nt, const int* ndim, const int64_t* dims, const float* data, int rank,
                 int qbits, int rounding, int iters, int warm_rank, const float* warm_q,
                 uint64_t* st, int8_t* codes, float* scales, float* q_out, int* ranks,
                 uint64_t* payload_bits) {
  /* compress.cpp:146-183 */
  if (qbits < 2 || qbits > 8) return fail(1, "quantization bits must be in [2, 8]");
  if (rank < 1) return fail(1, "compress: rank must be >= 1");
  int64_t off = 0, co = 0, so = 0, qo = 0, wo = 0;
  for (int i = 0; i < nt; ++i) {
    const int64_t n = numel(ndim, dims, i);
    const float* t = data + off;
    if (ndim[i] == 2) {
      const int64_t a = dims[2 * i], b = dims[2 * i + 1];
      const int r = reff(ndim, dims, i, rank);
      const int64_t wr = warm_rank > 0 ? reff(ndim, dims, i, warm_rank) : 0;
      /* warm start only if the operating rank is unchanged (compress.cpp:161) and the
       * factor is b x r (compress.cpp:64) */
      const float* wq = (warm_q && warm_rank == rank && wr == r) ? warm_q + wo : NULL;
      float* p = malloc(sizeof(float) * (size_t)(a * r));
      float* q = malloc(sizeof(float) * (size_t)(b * r));
      float* colbuf = malloc(sizeof(float) * (size_t)(a > b ? a : b));
      if (!p || !q || !colbuf) return fail(9, "oom");
      int rc = orc_lowrank_approx(a, b, t, r, wq, iters, st, p, q);
      if (rc) return rc;
      quantize_factor(p, a, r, qbits, rounding, st, codes + co, scales + so, colbuf);
      quantize_factor(q, b, r, qbits, rounding, st, codes + co + a * r, scales + so + r, colbuf);
      if (q_out) memcpy(q_out + qo, q, sizeof(float) * (size_t)(b * r));
      if (ranks) ranks[i] = r;
      co += (a + b) * r;
      so += 2 * r;
      qo += b * r;
      wo += b * wr;
      free(p);
      free(q);
      free(colbuf);
    } else if (ndim[i] == 1) {
      orc_quantize(t, n, qbits, rounding, st, codes + co, scales + so);
      if (ranks) ranks[i] = 0;
      co += n;
      so += 1;
    } else {
      return fail(2, "compress: only 1-D and 2-D tensors are supported");
    }
    off += n;
  }
  if (payload_bits) {
    int* rr = malloc(sizeof(int) * (size_t)nt);
    for (int i = 0; i < nt; ++i) rr[i] = reff(ndim, dims, i, rank);
    *payload_bits = orc_payload_bits(nt, ndim, dims, rr, qbits);
    free(rr);
  }
  return 0;
}

/* ------------------------------------------------ decompress / average (compress.cpp:201-238) */

static void decompress_tensor(int64_t a, int64_t b, int r, const int8_t* codes,
                              const float* scales, float* out) {
  /* dequantize_columns (compress.cpp:133-142) then matmul_nt (tensor.cpp:133-155) */
  float* P = malloc(sizeof(float) * (size_t)(a * r));
  float* Q = malloc(sizeof(float) * (size_t)(b * r));
  for (int j = 0; j < r; ++j) {
    for (int64_t i = 0; i < a; ++i) P[i * r + j] = (float)codes[j * a + i] * scales[j];
    for (int64_t i = 0; i < b; ++i) Q[i * r + j] = (float)codes[a * r + j * b + i] * scales[r + j];
  }
  orc_matmul_nt(a, r, b, P, Q, out);
  free(P);
  free(Q);
}

int orc_decompress(int nt, const int* ndim, const int64_t* dims, const int* ranks,
                   const int8_t* codes, const float* scales, float* out) {
  int64_t off = 0, co = 0, so = 0;
  for (int i = 0; i < nt; ++i) {
    const int64_t n = numel(ndim, dims, i);
    if (ndim[i] == 2) {
      const int64_t a = dims[2 * i], b = dims[2 * i + 1];
      decompress_tensor(a, b, ranks[i], codes + co, scales + so, out + off);
      co += (a + b) * ranks[i];
      so += 2 * ranks[i];
    } else {
      for (int64_t k = 0; k < n; ++k) out[off + k] = (float)codes[co + k] * scales[so];
      co += n;
      so += 1;
    }
    off += n;
  }
  return 0;
}

static int64_t total_numel(int nt, const int* ndim, const int64_t* dims) {
  int64_t n = 0;
  for (int i = 0; i < nt; ++i) n += numel(ndim, dims, i);
  return n;
}

int orc_allreduce_avg(int D, int nt, const int* ndim, const int64_t* dims, const int* ranks,
                      const int8_t* const* codes, const float* const* scales, float* out) {
  /* collective.cpp:17-46: double sum in worker order, times 1/D, cast once */
  if (D < 1) return fail(1, "allreduce_avg: no payloads");
  const int64_t n = total_numel(nt, ndim, dims);
  double* acc = malloc(sizeof(double) * (size_t)n);
  float* dec = malloc(sizeof(float) * (size_t)n);
  if (!acc || !dec) return fail(9, "oom");
  for (int w = 0; w < D; ++w) {
    orc_decompress(nt, ndim, dims, ranks, codes[w], scales[w], dec);
    for (int64_t k = 0; k < n; ++k) acc[k] = (w == 0 ? 0.0 : acc[k]) + (double)dec[k];
  }
  const double inv = 1.0 / (double)D;
  for (int64_t k = 0; k < n; ++k) out[k] = (float)(acc[k] * inv);
  free(acc);
  free(dec);
  return 0;
}

int orc_measure_error(int nt, const int* ndim, const int64_t* dims, const float* delta,
                      const int* ranks, const int8_t* codes, const float* scales, double* err) {
  /* compress.cpp:246-262 */
  const int64_t n = total_numel(nt, ndim, dims);
  float* rec = malloc(sizeof(float) * (size_t)n);
  if (!rec) return fail(9, "oom");
  orc_decompress(nt, ndim, dims, ranks, codes, scales, rec);
  double num = 0.0, den = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    const double d = (double)rec[k] - (double)delta[k];
    num += d * d;
    den += (double)delta[k] * (double)delta[k];
  }
  *err = den == 0.0 ? 0.0 : num / den;
  free(rec);
  return 0;
}

/* ------------------------------------------------------------- Nesterov (optim.cpp:56-78) */

/* ----------------------------------------------------------------- adamw (optim.cpp:15-47) */

int orc_adamw_step(int64_t n, float lr, float beta1, float beta2, float eps, float weight_decay,
                   int64_t warmup_steps, int64_t* step, float* p, const float* g, float* m,
                   float* v) {
  *step += 1;
  const float bc1 = 1.0f - powf(beta1, (float)(*step));
  const float bc2 = 1.0f - powf(beta2, (float)(*step));
  float lr_t = lr;
  if (warmup_steps > 0 && *step < warmup_steps) lr_t = lr * (float)(*step) / (float)warmup_steps;
  const float inv_bc1 = 1.0f / bc1;
  const float inv_bc2 = 1.0f / bc2;
  float probe = 0.0f;
  for (int64_t k = 0; k < n; ++k) {
    const float gk = g[k];
    probe += gk * 0.0f;
    const float m1 = beta1 * m[k];
    const float m2 = (1.0f - beta1) * gk;
    m[k] = m1 + m2;
    const float v1 = beta2 * v[k];
    const float v2 = ((1.0f - beta2) * gk) * gk;
    v[k] = v1 + v2;
    const float mhat = m[k] * inv_bc1;
    const float vhat = v[k] * inv_bc2;
    const float den = sqrtf(vhat) + eps;
    const float upd = mhat / den + weight_decay * p[k];
    p[k] = p[k] - lr_t * upd;
  }
  if (!isfinite(probe)) return fail(4, "adamw_step: non-finite gradient");
  return 0;
}

int orc_nesterov(int64_t n, float gamma, float beta, int classical, float* anchor, float* v,
                 const float* delta) {
  for (int64_t k = 0; k < n; ++k) {
    const float bv = beta * v[k];
    v[k] = bv + delta[k];
    if (classical) {
      const float step = gamma * v[k];
      anchor[k] = anchor[k] - step;
    } else {
      const float look = beta * v[k];
      const float dir = delta[k] + look;
      const float step = gamma * dir;
      anchor[k] = anchor[k] - step;
    }
  }
  return 0;
}

/* -------------------------------------------------------- effective rank (compress.cpp:306-344) */

int orc_effective_rank(int nt, const int* ndim, const int64_t* dims, const float* data,
                       double tau, int r_max, int* per_tensor, int* aggregate, int* all_zero) {
  if (!(tau > 0.0) || !(tau < 1.0)) return fail(1, "effective_rank: need 0 < tau < 1");
  if (r_max < 1) return fail(1, "effective_rank: need r_max >= 1");
  double weighted = 0.0, energy = 0.0;
  int64_t weight = 0, off = 0;
  int slot = 0;
  for (int i = 0; i < nt; ++i) {
    const int64_t n = numel(ndim, dims, i);
    if (ndim[i] == 2) {
      const int64_t a = dims[2 * i], b = dims[2 * i + 1];
      const int d = (int)(a < b ? a : b);
      double* sv = malloc(sizeof(double) * (size_t)d);
      orc_singular_values(a, b, data + off, sv);
      double total = 0.0;
      for (int j = 0; j < d; ++j) total += sv[j] * sv[j];
      energy += total;
      int k = 1;
      if (total > 0.0) {
        double prefix = 0.0;
        for (int j = 0; j < d; ++j) {
          prefix += sv[j] * sv[j];
          k = j + 1;
          if (prefix >= tau * total) break;
        }
      }
      if (per_tensor) per_tensor[slot] = k;
      ++slot;
      weighted += (double)n * (double)k;
      weight += n;
      free(sv);
    }
    off += n;
  }
  *all_zero = 0;
  if (weight == 0 || energy == 0.0) {
    *aggregate = 1;
    *all_zero = energy == 0.0;
    return 0;
  }
  int agg = (int)ceil(weighted / (double)weight);
  *aggregate = agg < 1 ? 1 : (agg > r_max ? r_max : agg);
  return 0;
}

/* ------------------------------------------------------ controller (engine.cpp:294-308) */

int orc_adapt_compression(const int* window, int len, int r1, int H1, int c, int h_min,
                          int* r_out, int* h_out) {
  if (r1 < 1 || H1 < 1 || c < 1) return fail(1, "adapt_compression: bad parameters");
  if (h_min < 1) return fail(1, "adapt_compression: H_min must be >= 1");
  if (len < c) {
    *r_out = r1;
    *h_out = H1;
    return 0;
  }
  double sum = 0.0;
  for (int i = len - c; i < len; ++i) sum += (double)window[i];
  int r = (int)ceil(sum / (double)c);
  r = r < 1 ? 1 : (r > r1 ? r1 : r);
  const double alpha = (double)(r1 - r) / (double)r1;
  int h = (int)llround((double)H1 * alpha);
  h = h < h_min ? h_min : (h > H1 ? H1 : h);
  *r_out = r;
  *h_out = h;
  return 0;
}

double orc_omega_bound(int r, int d, int q) { /* compress.cpp:240-244 */
  if (r < 1 || r > d || q < 0) return -1.0;
  return 1.0 - ((double)r / (double)d) * pow(2.0, -q);
}

/* -------------------------------------------------------- wire format (compress.cpp:350-426) */

typedef struct {
  uint8_t* p;
  int64_t n, cap;
} wbuf;

static void put8(wbuf* w, uint8_t v) {
  if (w->p && w->n < w->cap) w->p[w->n] = v;
  w->n++;
}
static void put_le(wbuf* w, uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) put8(w, (uint8_t)(v >> (8 * i)));
}
static void put_codes(wbuf* w, const int8_t* c, int64_t n, int q) {
  /* q-bit two's complement, LSB first, final partial byte flushed (compress.cpp:352-367) */
  uint32_t acc = 0;
  int nb = 0;
  const uint32_t mask = (1u << q) - 1u;
  for (int64_t i = 0; i < n; ++i) {
    acc |= ((uint32_t)(uint8_t)c[i] & mask) << nb;
    nb += q;
    while (nb >= 8) {
      put8(w, (uint8_t)acc);
      acc >>= 8;
      nb -= 8;
    }
  }
  if (nb > 0) put8(w, (uint8_t)acc);
}
static void put_f32(wbuf* w, float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  put_le(w, u, 4);
}

int64_t orc_serialize(int nt, const int* ndim, const int64_t* dims, const int* ranks, int rank,
                      int qbits, const int8_t* codes, const float* scales, uint8_t* out,
                      int64_t cap) {
  wbuf w = {out, 0, out ? cap : 0};
  put_le(&w, 0x43584c44u, 4); /* "DLXC" */
  put_le(&w, 1u, 4);
  put_le(&w, (uint32_t)rank, 4);
  put_le(&w, (uint32_t)qbits, 4);
  put_le(&w, (uint32_t)nt, 4);
  int64_t co = 0, so = 0;
  char name[32];
  for (int i = 0; i < nt; ++i) {
    const int len = snprintf(name, sizeof name, "t%d", i);
    put_le(&w, (uint16_t)len, 2);
    for (int k = 0; k < len; ++k) put8(&w, (uint8_t)name[k]);
    put8(&w, ndim[i] == 2 ? 0 : 1); /* PayloadKind LowRankQuant / DenseQuant */
    put8(&w, (uint8_t)ndim[i]);
    for (int d = 0; d < ndim[i]; ++d) put_le(&w, (uint64_t)dims[2 * i + d], 8);
    put_le(&w, (uint32_t)ranks[i], 4);
    put_le(&w, (uint32_t)qbits, 4);
    if (ndim[i] == 2) {
      const int64_t a = dims[2 * i], b = dims[2 * i + 1];
      const int r = ranks[i];
      put_codes(&w, codes + co, a * r, qbits);
      put_codes(&w, codes + co + a * r, b * r, qbits);
      for (int j = 0; j < 2 * r; ++j) put_f32(&w, scales[so + j]);
      co += (a + b) * r;
      so += 2 * r;
    } else {
      put_codes(&w, codes + co, dims[2 * i], qbits);
      put_f32(&w, scales[so]);
      co += dims[2 * i];
      so += 1;
    }
  }
  return w.n;
}

/* ----------------------------------------------------- one overlapped round (engine.cpp:458-509) */

typedef struct {
  int w, nt;
  const int* ndim;
  const int64_t* dims;
  const float* data;
  int rank, qbits, rounding, iters, warm_rank;
  const float* warm_q;
  uint64_t state;
  int8_t* codes;
  float* scales;
  float* q_out;
  int* ranks;
  int rc;
} cjob;

static void* cjob_run(void* arg) {
  cjob* j = (cjob*)arg;
  j->rc = orc_compress(j->nt, j->ndim, j->dims, j->data, j->rank, j->qbits, j->rounding,
                       j->iters, j->warm_rank, j->warm_q, &j->state, j->codes, j->scales,
                       j->q_out, j->ranks, NULL);
  return NULL;
}

int orc_outer_round(int D, int nt, const int* ndim, const int64_t* dims, uint64_t seed,
                    int64_t round_index, int rank, int qbits, int rounding, int iters,
                    int adaptive, double tau, int r1, float gamma, float beta, int classical,
                    int threads, float* anchor, float* velocity, float* pending,
                    const float* local, int* warm_rank, float* warm_q, int* r_prime,
                    double* comp_error, uint64_t* payload_bits, double* err_norm0,
                    double* max_delta_norm) {
  const int64_t n = total_numel(nt, ndim, dims);
  int* ranks = malloc(sizeof(int) * (size_t)nt);
  for (int i = 0; i < nt; ++i) ranks[i] = reff(ndim, dims, i, rank);
  const int64_t nc = orc_codes_count(nt, ndim, dims, ranks);
  const int64_t ns = orc_scales_count(nt, ndim, dims, ranks);
  const int64_t nq = orc_qfactor_count(nt, ndim, dims, ranks);
  cjob* jobs = calloc((size_t)D, sizeof(cjob));
  int8_t** cp = malloc(sizeof(int8_t*) * (size_t)D);
  float** sp = malloc(sizeof(float*) * (size_t)D);
  const uint64_t key[2] = {0xc09c, (uint64_t)round_index};
  const uint64_t st0 = orc_stream_init(seed, orc_stream_key(key, 2)); /* engine.cpp:226 */
  for (int w = 0; w < D; ++w) {
    cjob* j = &jobs[w];
    j->w = w;
    j->nt = nt;
    j->ndim = ndim;
    j->dims = dims;
    j->data = pending + (int64_t)w * n;
    j->rank = rank;
    j->qbits = qbits;
    j->rounding = rounding;
    j->iters = iters;
    j->warm_rank = *warm_rank;
    j->warm_q = warm_q;
    j->state = st0;
    j->codes = cp[w] = malloc((size_t)nc);
    j->scales = sp[w] = malloc(sizeof(float) * (size_t)ns);
    j->q_out = w == 0 ? malloc(sizeof(float) * (size_t)(nq > 0 ? nq : 1)) : NULL;
    j->ranks = NULL;
  }
  /* compress fan-out over workers (parallel_over, engine.cpp:135-156) */
  int nthr = threads < 1 ? 1 : (threads > D ? D : threads);
  for (int base = 0; base < D; base += nthr) {
    pthread_t th[64];
    int cnt = 0;
    for (int w = base; w < D && w < base + nthr && cnt < 64; ++w, ++cnt)
      pthread_create(&th[cnt], NULL, cjob_run, &jobs[w]);
    for (int k = 0; k < cnt; ++k) pthread_join(th[k], NULL);
  }
  int rc = 0;
  for (int w = 0; w < D; ++w)
    if (jobs[w].rc) rc = jobs[w].rc;
  if (!rc) {
    float* avg = malloc(sizeof(float) * (size_t)n);
    orc_allreduce_avg(D, nt, ndim, dims, ranks, (const int8_t* const*)cp,
                      (const float* const*)sp, avg);
    orc_measure_error(nt, ndim, dims, pending, ranks, cp[0], sp[0], comp_error);
    *payload_bits = orc_payload_bits(nt, ndim, dims, ranks, qbits);
    *r_prime = 0;
    if (adaptive) {
      int all_zero = 0;
      orc_effective_rank(nt, ndim, dims, avg, tau, r1, NULL, r_prime, &all_zero);
    }
    /* e_w = delta_w - avg; delta_w <- (anchor - local_w) + e_w (engine.cpp:254-257, 266-276) */
    double maxn = 0.0;
    for (int w = 0; w < D; ++w) {
      float* pd = pending + (int64_t)w * n;
      const float* lw = local + (int64_t)w * n;
      /* ps_l2_norm sums per-tensor Frobenius norms (params.cpp:83-87) */
      double ss = 0.0, es = 0.0;
      int64_t k = 0;
      for (int i = 0; i < nt; ++i) {
        double ts = 0.0, te = 0.0;
        const int64_t end = k + numel(ndim, dims, i);
        for (; k < end; ++k) {
          const float e = pd[k] - avg[k];
          const float d0 = anchor[k] - lw[k];
          const float d = d0 + e;
          te += (double)e * (double)e;
          ts += (double)d * (double)d;
          pd[k] = d;
        }
        ss += ts;
        es += te;
      }
      if (w == 0) *err_norm0 = sqrt(es);
      const double nn = sqrt(ss);
      if (nn > maxn) maxn = nn;
    }
    *max_delta_norm = maxn;
    orc_nesterov(n, gamma, beta, classical, anchor, velocity, avg); /* engine.cpp:495 */
    *warm_rank = rank;                                              /* engine.cpp:498-501 */
    memcpy(warm_q, jobs[0].q_out, sizeof(float) * (size_t)nq);
    free(avg);
  }
  for (int w = 0; w < D; ++w) {
    free(cp[w]);
    free(sp[w]);
    free(jobs[w].q_out);
  }
  free(cp);
  free(sp);
  free(jobs);
  free(ranks);
  return rc;
}
