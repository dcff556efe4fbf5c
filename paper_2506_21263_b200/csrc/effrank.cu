// effrank.cu — adaptive-rank measurement (effective_rank compress.cpp:306-344) in factor
// space.
//
// The reference runs a dense fp64 SVD of every averaged Delta (Gram + Householder + QL,
// tensor.cpp:325-361): 179 s per OPT-1.3B layer on a CPU core. Delta = (1/D) A B^T with
// A = [P_1 .. P_D] (a x K), B = [Q_1 .. Q_D] (b x K), K = D r, so its nonzero squared
// singular values are the eigenvalues of (1/D^2) L^T (A^T A) L where B^T B = L L^T. The
// per-tensor work is two fp64 Gram matrices (tall-skinny, batched) and one K x K symmetric
// eigenproblem (cyclic parallel Jacobi, one CTA per tensor). r' can differ from the dense
// reference only where the prefix energy lands within rounding of tau (ties).
#include <cuda_bf16.h>
#include <cstdlib>
#include <cstdio>

#include "dlx_internal.cuh"
#include "ptx.cuh"

namespace dlx {

// ------------------------------------------------------------------ code Grams
// The factor Grams come straight from the packed codes: C^T C over the gathered codes of one
// side of one tensor is an integer matrix (|c| <= 2^(q-1)), so it can be formed exactly on
// tensor cores from the codes themselves — no dequantised factor copies, no fp32 Gram sweep.
// G = diag(s) C^T C diag(s) with the column scales is formed inside k_effrank. (An fp64 DMMA
// variant for K <= 64 from round 1 was no longer launched — every K goes through the bf16
// kernel below, equally exact — and has been removed.)
constexpr int kCgChunk = 1024;  // rows per code-Gram block

struct CodeGramJob : PlanExt {
  std::vector<int4> chunks;  // (t2 slot, side, row0, row1)
  int4* d = nullptr;
};

// K up to 256: the integer Gram on the bf16 tensor cores (mma.sync m16n8k16, fp32
// accumulate). Codes are exact in bf16 and every per-chunk partial sum is an integer below
// 1024 * 127^2 < 2^24, so the fp32 accumulation is exact; chunk sums are added as fp64 (exact,
// order-independent). Block = (1024-row chunk of one factor side, group of 32x32 output
// tiles of the upper block triangle); 64 rows are decoded per pass into Ct[k][row] (bf16).
constexpr int kCgmRows = 64;
constexpr int kCgmLd = kCgmRows + 8;  // bf16 row stride of Ct: conflict-free ldmatrix
constexpr int kCgmTilesPerWarp = 2;
constexpr int kCgmWarps = 8;

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(su32(p)));
}
__device__ __forceinline__ void ldsm_x2(uint32_t (&r)[2], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
               : "=r"(r[0]), "=r"(r[1])
               : "r"(su32(p)));
}
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4],
                                               const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__global__ void __launch_bounds__(256) k_code_gram_mma(const DevT2* __restrict__ T,
                                                       const int4* __restrict__ chunks,
                                                       const uint8_t* __restrict__ gathered,
                                                       int64_t pay_bytes, int qbits, int D,
                                                       int kst, double* __restrict__ G) {
  __shared__ __align__(16) __nv_bfloat16 Ct[256 * kCgmLd];
  const int4 ch = chunks[blockIdx.x];
  const DevT2& t = T[ch.x];
  const int side = ch.y, r = t.r, K = D * r;
  const int64_t n = side == 0 ? t.a : t.b;
  const int KP = (K + 31) / 32 * 32;  // padded to whole 32x32 tiles
  const int nt32 = KP / 32, ntiles = nt32 * (nt32 + 1) / 2;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tile0 = blockIdx.y * kCgmWarps * kCgmTilesPerWarp;
  if (tile0 >= ntiles) return;  // uniform
  // decode tasks: (column k, 8-row group) -> one <= 64-bit field of 8 codes
  const uint32_t* words = reinterpret_cast<const uint32_t*>(gathered);
  const int64_t nwords = D * pay_bytes / 4;
  const uint32_t mask = (1u << qbits) - 1u;
  const int sh = 32 - qbits;
  const int64_t rend = min((int64_t)ch.w, n);
  // this warp's output tiles (ti <= tj in 32-blocks)
  int tI[kCgmTilesPerWarp], tJ[kCgmTilesPerWarp];
  bool tv[kCgmTilesPerWarp];
#pragma unroll
  for (int u = 0; u < kCgmTilesPerWarp; ++u) {
    const int id = tile0 + warp + kCgmWarps * u;
    tv[u] = id < ntiles;
    int bi = 0, rem = tv[u] ? id : 0;
    while (rem >= nt32 - bi) {
      rem -= nt32 - bi;
      ++bi;
    }
    tI[u] = bi;
    tJ[u] = bi + rem;
  }
  float acc[kCgmTilesPerWarp][2][4][4];
#pragma unroll
  for (int u = 0; u < kCgmTilesPerWarp; ++u)
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[u][a][b][c] = 0.f;
  const int ntask = KP * (kCgmRows / 8);
  for (int64_t row0 = ch.z; row0 < ch.w; row0 += kCgmRows) {
    __syncthreads();
    for (int task = threadIdx.x; task < ntask; task += 256) {
      const int k = task / (kCgmRows / 8), tg = task % (kCgmRows / 8);
      const int64_t rowg = row0 + 8 * tg;
      uint32_t packed[4] = {0u, 0u, 0u, 0u};
      if (k < K && rowg < rend) {
        const int w = k / r, j = k % r;
        const int64_t bit = ((w * pay_bytes + (side == 0 ? t.seg_pc : t.seg_qc)) * 8 +
                             (int64_t)j * n * qbits) + rowg * qbits;
        const int64_t wi = bit >> 5;
        const uint32_t w0 = words[wi];
        const uint32_t w1 = wi + 1 < nwords ? words[wi + 1] : 0u;
        const uint32_t w2 = wi + 2 < nwords ? words[wi + 2] : 0u;
        const int s = static_cast<int>(bit & 31);
        const uint64_t lo = static_cast<uint64_t>(w0) | (static_cast<uint64_t>(w1) << 32);
        const uint64_t v = (lo >> s) | (s ? (static_cast<uint64_t>(w2) << (64 - s)) : 0ull);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          int c = static_cast<int>((static_cast<uint32_t>(v >> (i * qbits)) & mask) << sh) >> sh;
          if (rowg + i >= rend) c = 0;
          const uint32_t hb = __bfloat16_as_ushort(__int2bfloat16_rn(c));
          packed[i / 2] |= hb << (16 * (i % 2));
        }
      }
      *reinterpret_cast<uint4*>(&Ct[k * kCgmLd + 8 * tg]) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kCgmTilesPerWarp; ++u) {
      if (!tv[u]) continue;
      const int i0 = 32 * tI[u], j0 = 32 * tJ[u];
#pragma unroll
      for (int k0 = 0; k0 < kCgmRows; k0 += 16) {
        uint32_t af[2][4], bf[4][2];
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          const int rr_ = i0 + 16 * a + (lane % 8) + 8 * ((lane / 8) % 2);
          const int cc = k0 + 8 * (lane / 16);
          ldsm_x4(af[a], &Ct[rr_ * kCgmLd + cc]);
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int rr_ = j0 + 8 * b + (lane % 8);
          const int cc = k0 + 8 * ((lane / 8) % 2);
          ldsm_x2(bf[b], &Ct[rr_ * kCgmLd + cc]);
        }
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) mma_bf16_16816(acc[u][a][b], af[a], bf[b]);
      }
    }
  }
  // accumulator fragment (m16n8): c0,c1 at row g, cols 2q, 2q+1; c2,c3 at row g + 8
  double* g = G + ((int64_t)ch.x * 2 + side) * kst * kst;
#pragma unroll
  for (int u = 0; u < kCgmTilesPerWarp; ++u) {
    if (!tv[u]) continue;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int i = 32 * tI[u] + 16 * a + lane / 4 + 8 * (c / 2);
          const int j = 32 * tJ[u] + 8 * b + 2 * (lane % 4) + (c % 2);
          const float v = acc[u][a][b][c];
          if (i < K && j < K && i <= j && v != 0.f) atomicAdd(&g[i * kst + j], static_cast<double>(v));
        }
  }
}

// ------------------------------------------------------------------ eigenproblem
// Per tensor: G_B = L L^T (semidefinite Cholesky), M = L^T G_A L (K x K, K = D r), Householder
// tridiagonalisation, eigenvalues by Sturm-count multisection, prefix energy. Working set:
// L, G_A L and M all in shared memory for n <= 64; M alone in shared memory for n <= 128 (L
// and G_A L in the global work buffer, L2-resident); everything in the work buffer above.
// Grams come either as fp64 matrices (GA, GB; row stride rr) or as integer code Grams (GI,
// upper triangle, stride rr) scaled by the payload's column scales.
__device__ long long g_er_prof[16];
// K above which k_effrank_big runs (dlx_set_option). 96: tools/er_bigfrom.py on B200 —
// K = 128: blocked 0.82 vs 1.11 ms (Llama-7B layer, r = 128), 1.08 vs 1.12 ms (OPT-1.3B,
// D = 4); K = 96 on OPT-1.3B (D = 3): 0.76 vs 0.71 ms, so the unblocked kernel keeps K <= 96
int& option_effrank_big_from() {
  static int v = 96;
  return v;
}  // experiments (DLX_ER_PROF): phase cycles of block 0
constexpr int kErAllSmem = 64;   // n <= 64: L, G_A L, M staged in shared memory
constexpr int kErMSmem = 128;    // n <= 128: M staged in shared memory
constexpr int kErMaxN = 256;     // tridiagonal scratch size
constexpr int kErSwitch = 160;   // global mode: trailing block moves to smem at this size

// Steps k in [k0, k1) of the one-stage Householder tridiagonalisation (P = I - v v^T / H,
// A <- P A P) of the n x n symmetric matrix M (row stride ldm); sh = shared (H, alpha, K).
__device__ __noinline__ void hh_steps(double* M, int ldm, int n, int k0, int k1, double* V,
                                      double* Pv, double* sh) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int k = k0; k < k1; ++k) {
    if (tid < 32) {
      double ss = 0.0;
      for (int i = k + 1 + tid; i < n; i += 32) {
        const double x = M[i * ldm + k];
        ss += x * x;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (tid == 0) {
        const double x0 = M[(k + 1) * ldm + k];
        const double nrm = sqrt(ss);
        if (!(ss - x0 * x0 > 1e-300 * ss) || nrm == 0.0) {
          sh[0] = 0.0;  // column already reduced
          sh[1] = x0;
        } else {
          const double alpha = x0 > 0.0 ? -nrm : nrm;
          sh[1] = alpha;
          sh[0] = ss - x0 * alpha;  // ||v||^2 / 2
        }
      }
    }
    __syncthreads();
    const double H = sh[0];
    if (H == 0.0) {  // uniform
      __syncthreads();
      continue;
    }
    for (int i = k + 1 + tid; i < n; i += nt) V[i] = i == k + 1 ? M[i * ldm + k] - sh[1] : M[i * ldm + k];
    __syncthreads();
    {
      const int part = tid % 4, rows_per = nt / 4;
      const int passes = (n - k - 1 + rows_per - 1) / rows_per;  // uniform: all lanes shuffle
      for (int ps = 0; ps < passes; ++ps) {
        const int row = k + 1 + tid / 4 + ps * rows_per;
        double acc = 0.0;
        if (row < n)
          for (int j = k + 1 + part; j < n; j += 4) acc = fma(M[row * ldm + j], V[j], acc);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        if (row < n && part == 0) Pv[row] = acc / H;
      }
    }
    __syncthreads();
    if (tid < 32) {
      double acc = 0.0;
      for (int i = k + 1 + tid; i < n; i += 32) acc = fma(V[i], Pv[i], acc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (tid == 0) sh[2] = acc / (2.0 * H);
    }
    __syncthreads();
    const double Kc = sh[2];
    for (int i = k + 1 + tid / 32; i < n; i += nt / 32) {
      const double vi = V[i], wi = Pv[i] - Kc * vi;
      for (int j = k + 1 + tid % 32; j < n; j += 32) {
        const double wj = Pv[j] - Kc * V[j];
        M[i * ldm + j] -= vi * wj + wi * V[j];
      }
    }
    if (tid == 0) M[(k + 1) * ldm + k] = sh[1];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(512) k_effrank(const DevT2* __restrict__ T, int D, int rr,
                                                 const double* __restrict__ GA,
                                                 const double* __restrict__ GB,
                                                 const double* __restrict__ GI,
                                                 const uint8_t* __restrict__ gathered,
                                                 int64_t pay_bytes, int sdim, int mdim,
                                                 double* __restrict__ work, double tau,
                                                 int* __restrict__ per,
                                                 double* __restrict__ energy, int shard,
                                                 int nshards) {
  extern __shared__ double er_sm[];
  __shared__ double tri[4 * kErMaxN];  // V | A v / H | diagonal | squared off-diagonal
  __shared__ double s_tot;
  __shared__ int s_k;
  const int e = shard + blockIdx.x * nshards;  // this shard's tensors: e % nshards == shard
  const DevT2& t = T[e];
  const int K = D * t.r;
  const int n2 = K + (K & 1);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t mat = (int64_t)rr * rr;
  double* gw = work + 3 * (int64_t)blockIdx.x * mat;
  // G_A / G_B entries from the integer code Grams (scaled) or the fp64 Grams
  auto gram = [&](int which, int i, int k) -> double {
    if (GI) {
      const int lo = min(i, k), hi = max(i, k);
      const double* gi = GI + (int64_t)e * 2 * mat + (which ? mat : 0);
      const int wi = i / t.r, ji = i % t.r, wk = k / t.r, jk = k % t.r;
      const int64_t so = which ? t.seg_qs : t.seg_ps;
      const double si = *reinterpret_cast<const float*>(gathered + wi * pay_bytes + so + 4 * ji);
      const double sk = *reinterpret_cast<const float*>(gathered + wk * pay_bytes + so + 4 * jk);
      return gi[lo * rr + hi] * si * sk;
    }
    return (which ? GB : GA)[e * mat + i * rr + k];
  };
  // working set: all three in shared memory (n <= sdim); the Cholesky and M in shared memory
  // one after the other with L and G_A L in the work buffer (n <= mdim); else all global
  const bool all_s = n2 <= sdim, mid_s = !all_s && n2 <= mdim;
  double *Lm, *Tm, *M;
  int ldl, ldm;
  if (all_s) {
    ldl = ldm = sdim + 1;
    Lm = er_sm;
    Tm = er_sm + (int64_t)sdim * ldl;
    M = er_sm + 2 * (int64_t)sdim * ldl;
  } else if (mid_s) {
    ldl = mdim + 1;  // Cholesky staged in shared memory first
    ldm = mdim + 1;
    Lm = er_sm;
    Tm = gw + mat;
    M = er_sm;
  } else {
    ldl = ldm = rr;
    Lm = gw;
    Tm = gw + mat;
    M = gw + 2 * mat;
  }
  long long pt0 = clock64();
#define ER_MARK(i) do { if (blockIdx.x == 0 && tid == 0) { const long long c = clock64(); g_er_prof[i] = c - pt0; pt0 = c; } } while (0)
  // 0. stage G_B -> Lm (lower), G_A -> GAs (M itself, or the work buffer in the mid mode)
  double* GAs = mid_s ? gw + 2 * mat : M;
  const int ldg = mid_s ? rr : ldm;
  for (int idx = tid; idx < K * K; idx += nt) {
    const int i = idx / K, k = idx % K;
    if (k <= i) Lm[i * ldl + k] = gram(1, i, k);
    GAs[i * ldg + k] = gram(0, i, k);
  }
  __syncthreads();
  ER_MARK(0);
  // 1. semidefinite Cholesky of G_B (lower), columns with vanishing pivot dropped
  double dmax = 0.0;
  for (int j = 0; j < K; ++j) dmax = fmax(dmax, Lm[j * ldl + j]);
  const double floor_piv = 1e-14 * dmax;
  for (int j = 0; j < K; ++j) {
    __shared__ double s_ljj, s_inv;
    if (tid == 0) {  // one sqrt / division per step, broadcast
      const double d = Lm[j * ldl + j];
      const bool keep = d > floor_piv && d > 0.0;
      s_ljj = keep ? sqrt(d) : 0.0;
      s_inv = keep ? 1.0 / s_ljj : 0.0;
    }
    __syncthreads();
    const double ljj = s_ljj, inv = s_inv;
    for (int i = j + 1 + tid; i < K; i += nt) Lm[i * ldl + j] *= inv;
    if (tid == 0) Lm[j * ldl + j] = ljj;
    __syncthreads();
    // trailing lower-triangle update: warp per row, lanes over columns
    for (int i = j + 1 + tid / 32; i < K; i += nt / 32) {
      const double lij = Lm[i * ldl + j];
      for (int k = j + 1 + tid % 32; k <= i; k += 32) Lm[i * ldl + k] -= lij * Lm[k * ldl + j];
    }
    __syncthreads();
  }
  if (mid_s) {  // move L to the work buffer; shared memory is needed for M next
    for (int idx = tid; idx < K * K; idx += nt) {
      const int i = idx / K, k = idx % K;
      gw[i * rr + k] = k <= i ? Lm[i * ldl + k] : 0.0;
    }
    __syncthreads();
    Lm = gw;
    ldl = rr;
  } else {
    for (int idx = tid; idx < K * K; idx += nt) {  // zero the strict upper part
      const int i = idx / K, k = idx % K;
      if (k > i) Lm[i * ldl + k] = 0.0;
    }
  }
  __syncthreads();
  ER_MARK(1);
  // 2. Tm = G_A L ; M = L^T Tm (symmetrised), on the fp64 tensor cores: warp = 8x8 output
  // block, DMMA m8n8k4 over the triangular K range (operands zero-padded to whole blocks)
  const int nw = nt / 32, lane = tid % 32;
  const int KB = (K + 7) / 8;
  auto ldz = [](const double* X, int ld, int r, int c, int lim) -> double {
    return (r < lim && c < lim) ? X[r * ld + c] : 0.0;
  };
  for (int blk = tid / 32; blk < KB * KB; blk += nw) {
    const int bi = blk / KB, bj = blk % KB;
    double acc[2] = {0.0, 0.0};
    for (int k0 = 8 * bj; k0 < K; k0 += 4)  // L[k][j] = 0 for k < j
      dmma_8x8x4(acc, ldz(GAs, ldg, 8 * bi + lane / 4, k0 + lane % 4, K),
                 ldz(Lm, ldl, k0 + lane % 4, 8 * bj + lane / 4, K));
    const int i = 8 * bi + lane / 4;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = 8 * bj + 2 * (lane % 4) + q;
      if (i < K && j < K) Tm[i * ldl + j] = acc[q];
    }
  }
  __syncthreads();
  const int NB2 = (n2 + 7) / 8;
  for (int blk = tid / 32; blk < NB2 * NB2; blk += nw) {
    const int bi = blk / NB2, bj = blk % NB2;
    double acc[2] = {0.0, 0.0};
    for (int k0 = 8 * bi; k0 < K; k0 += 4)  // L[k][i] = 0 for k < i
      dmma_8x8x4(acc, ldz(Lm, ldl, k0 + lane % 4, 8 * bi + lane / 4, K),
                 ldz(Tm, ldl, k0 + lane % 4, 8 * bj + lane / 4, K));
    const int i = 8 * bi + lane / 4;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = 8 * bj + 2 * (lane % 4) + q;
      if (i < n2 && j < n2) M[i * ldm + j] = (i < K && j < K) ? acc[q] : 0.0;
    }
  }
  __syncthreads();
  for (int idx = tid; idx < n2 * n2; idx += nt) {
    const int i = idx / n2, j = idx % n2;
    if (j > i) {
      const double v = 0.5 * (M[i * ldm + j] + M[j * ldm + i]);
      M[i * ldm + j] = v;
      M[j * ldm + i] = v;
    }
  }
  __syncthreads();
  ER_MARK(2);
  // 3a. Householder tridiagonalisation. In the global-memory mode the trailing block moves
  // into shared memory once it fits (kErSwitch rows) and is copied back afterwards.
  double* V = tri;
  double* Pv = tri + kErMaxN;
  const int n = n2;
  __shared__ double s_hak[3];
  {
    const int k_end = max(n - 2, 0);
    const int k_sw = (all_s || mid_s) ? k_end : max(0, min(k_end, n - kErSwitch));
    hh_steps(M, ldm, n, 0, k_sw, V, Pv, s_hak);
    if (k_sw < k_end) {
      const int ls = kErSwitch + 1;
      for (int i = k_sw + tid / 32; i < n; i += nt / 32)
        for (int j = k_sw + tid % 32; j < n; j += 32) er_sm[(i - k_sw) * ls + (j - k_sw)] = M[i * ldm + j];
      __syncthreads();
      hh_steps(er_sm - (int64_t)k_sw * ls - k_sw, ls, n, k_sw, k_end, V, Pv, s_hak);
      for (int i = k_sw + tid / 32; i < n; i += nt / 32)
        for (int j = k_sw + tid % 32; j < n; j += 32) M[i * ldm + j] = er_sm[(i - k_sw) * ls + (j - k_sw)];
      __syncthreads();
    }
  }
  ER_MARK(3);
  // 3b. eigenvalues of the tridiagonal (d, e) by multisection on Sturm counts: a group of G
  // lanes per eigenvalue evaluates G interior points per step (log2(G+1) bits per step)
  double* Dg = tri + 2 * kErMaxN;
  double* E2 = tri + 3 * kErMaxN;
  for (int i = tid; i < n; i += nt) {
    Dg[i] = M[i * ldm + i];
    E2[i] = i + 1 < n ? M[(i + 1) * ldm + i] * M[(i + 1) * ldm + i] : 0.0;
  }
  __syncthreads();
  double lo = 0.0, hi = 0.0, amax = 0.0;
  for (int i = 0; i < n; ++i) {  // Gershgorin (every thread, uniform)
    const double r0 = i > 0 ? sqrt(E2[i - 1]) : 0.0, r1 = i + 1 < n ? sqrt(E2[i]) : 0.0;
    lo = fmin(lo, Dg[i] - r0 - r1);
    hi = fmax(hi, Dg[i] + r0 + r1);
    amax = fmax(amax, fabs(Dg[i]) + r0 + r1);
  }
  hi += 1e-14 * amax + 1e-300;
  lo -= 1e-14 * amax + 1e-300;
  double* ev = V;  // eigenvalues, descending (V is free now)
  int G = 1;
  while (G * 2 <= 32 && G * 2 * n <= nt) G *= 2;
  const int iters = G >= 16 ? 12 : G >= 8 ? 15 : G >= 4 ? 20 : G >= 2 ? 29 : 50;
  const int lanes = (nt / G) * G;  // threads in whole groups
  for (int base_idx = 0; base_idx < n; base_idx += nt / G) {
    const int idx = base_idx + tid / G, l = tid % G;
    double blo = lo, bhi = hi;
    const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << ((tid % 32) / G * G);
    for (int it = 0; it < iters; ++it) {
      const double sig = blo + (bhi - blo) * (double)(l + 1) / (double)(G + 1);
      // Sturm count = sign changes of the characteristic-polynomial sequence
      // p_j = (d_j - sig) p_{j-1} - e_{j-1}^2 p_{j-2} (division-free; exact power-of-two
      // rescaling keeps it in range; a zero takes the sign opposite to its predecessor, as
      // the LDL^T recurrence with a -pivmin pivot does)
      int c = 0;
      {
        double pm = 1.0, p = Dg[0] - sig;
        bool neg_prev = false;  // sign of p_0 = +
        bool neg = p < 0.0 || p == 0.0;
        c += neg != neg_prev;
        neg_prev = neg;
        for (int j = 1; j < n; ++j) {
          const double pn = fma(Dg[j] - sig, p, -E2[j - 1] * pm);
          neg = pn == 0.0 ? !neg_prev : pn < 0.0;
          c += neg != neg_prev;
          neg_prev = neg;
          pm = p;
          p = pn;
          const double ap = fabs(p) + fabs(pm);
          if (ap > 0x1p+600) {
            p = scalbn(p, -600);
            pm = scalbn(pm, -600);
          } else if (ap < 0x1p-600) {
            p = scalbn(p, 600);
            pm = scalbn(pm, 600);
          }
        }
      }
      const unsigned below = __ballot_sync(0xffffffffu, c <= idx) & gmask;
      const int L = __popc(below);
      const int base = (tid % 32) / G * G;
      const double s_lo = __shfl_sync(0xffffffffu, sig, base + max(L - 1, 0));
      const double s_hi = __shfl_sync(0xffffffffu, sig, base + min(L, G - 1));
      if (L > 0) blo = s_lo;
      if (L < G) bhi = s_hi;
    }
    // (an all-zero M — an all-zero exchange — has exactly zero eigenvalues: without the
    // guard the bisection midpoint of the [-1e-300, 1e-300] bracket leaves a denormal-size
    // energy and the reduce would not flag the round all-zero)
    if (l == 0 && idx < n && tid < lanes)
      ev[n - 1 - idx] = amax > 0.0 ? fmax(0.5 * (blo + bhi), 0.0) : 0.0;
  }
  __syncthreads();
  ER_MARK(4);
  // 4. prefix energy
  if (tid == 0) {
    double tot = 0.0;
    for (int i = 0; i < n; ++i) tot += ev[i];
    int k = 1;
    if (tot > 0.0) {
      double pre = 0.0;
      for (int i = 0; i < n; ++i) {
        pre += ev[i];
        k = i + 1;
        if (pre >= tau * tot) break;
      }
    }
    s_k = k;
    s_tot = tot / ((double)D * (double)D);
  }
  __syncthreads();
  if (tid == 0) {
    per[e] = s_k;
    energy[e] = s_tot;
  }
}

// ------------------------------------------------------------------ eigenproblem, K > 128
// One CTA per tensor; the K x K working matrices (K <= 256, fp64: up to 512 KB each) live in
// the global work buffer (L2-resident) with shared-memory staging:
//  1. semidefinite Cholesky of G_B, blocked (32-column panels factored in shared memory,
//     trailing SYRK update on the fp64 tensor cores);
//  2. T = G_A L and the lower triangle of M = L^T T as 64 x 64 output tiles over 32-wide
//     K panels staged in shared memory (DMMA m8n8k4);
//  3. Householder tridiagonalisation of M in packed lower storage with the rank-2 update of
//     step k-1 fused into the matrix-vector product of step k (one read and one write of the
//     trailing triangle per step); the trailing triangle moves into shared memory once it
//     fits (m <= kEbSmemM);
//  4. Sturm-count multisection with certified early exit: iterate until the eigenvalue
//     intervals decide r' (smallest k whose prefix energy reaches tau of the total) — the
//     same k as fully converged eigenvalues except at ties; energy = trace(M).
constexpr int kEbThreads = 512;
constexpr int kEbWarps = kEbThreads / 32;
constexpr int kEbVec = 256;                       // vector scratch length (K <= 256)
constexpr int kEbPld = 33;                        // Cholesky panel row stride (doubles)
constexpr int kEbTA = 36, kEbTB = 68;             // product tile strides (conflict-free DMMA)
// dynamic shared memory: 8 vectors | column partials [16][256] | region (panel/tiles/packed M)
constexpr int kEbRegion = (227 * 1024) / 8 - 8 * kEbVec - kEbWarps * kEbVec - 160;  // 1 KB static
constexpr size_t kEbSmem = sizeof(double) * (8 * kEbVec + kEbWarps * kEbVec + kEbRegion);

__device__ __forceinline__ int64_t pk(int i, int j, int o) {  // packed lower, origin o
  const int64_t a = i - o;
  return a * (a + 1) / 2 + (j - o);
}

__device__ double eb_block_reduce(double v, double* red, bool is_max) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, u) : v + u;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = red[0];
  for (int i = 1; i < kEbWarps; ++i) s = is_max ? fmax(s, red[i]) : s + red[i];
  return s;
}

// Y[i0.., j0..] (64 x 64 tile) = sum over K panels [kbeg, K) of A(i, k) B(k, j), with
// A(i, k) = TA ? X[k * K + i] : X[i * K + k] and B(k, j) = Y[k * K + j]; 16 warps x four 8x8
// blocks (one block row per warp pair). Returns the accumulators.
template <bool TA>
__device__ __forceinline__ void eb_tile(const double* X, const double* Yv, int K, int i0, int j0,
                                        int kbeg, double* As, double* Bs, double (&acc)[4][2]) {
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int bi = warp / 2, bj0 = 4 * (warp % 2);
#pragma unroll
  for (int u = 0; u < 4; ++u) acc[u][0] = acc[u][1] = 0.0;
  for (int k0 = kbeg; k0 < K; k0 += 32) {
    for (int idx = tid; idx < 64 * 32; idx += kEbThreads) {
      if (TA) {  // As[i][k] = X[(k0 + k) * K + i0 + i]: read rows of X coalesced over i
        const int k = idx / 64, i = idx % 64;
        const int gi = i0 + i, gk = k0 + k;
        As[i * kEbTA + k] = (gi < K && gk < K) ? X[(int64_t)gk * K + gi] : 0.0;
      } else {
        const int i = idx / 32, k = idx % 32;
        const int gi = i0 + i, gk = k0 + k;
        As[i * kEbTA + k] = (gi < K && gk < K) ? X[(int64_t)gi * K + gk] : 0.0;
      }
      const int k = idx / 64, j = idx % 64;
      const int gk = k0 + k, gj = j0 + j;
      Bs[k * kEbTB + j] = (gk < K && gj < K) ? Yv[(int64_t)gk * K + gj] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 32; kk += 4) {
      const double a = As[(8 * bi + lane / 4) * kEbTA + kk + lane % 4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        dmma_8x8x4(acc[u], a, Bs[(kk + lane % 4) * kEbTB + 8 * (bj0 + u) + lane / 4]);
    }
    __syncthreads();
  }
}

// Fused pass of one tridiagonalisation step over the trailing triangle rows/cols [c0, n):
// a = stored - (v' w'^T + w' v'^T) (step k-1), stored back; Prow[i] = sum_{j<=i} a_ij v_j and
// the lane's column partials cp[q] (column c0 + lane + 32 q) += a_ij v_i for j < i. R = 16 / Q
// rows per batch: their loads are issued together and their row reductions interleave.
template <int Q>
__device__ __forceinline__ void eb_pass(double* M, int org, int n, int c0, int warp, int lane,
                                        const double* Vp, const double* Wp, const double* Vr,
                                        double v1, bool reduced, double* Prow,
                                        double (&cp)[8]) {
  constexpr int R = 16 / Q;
  double wj[Q], vpj[Q], vnj[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int j = c0 + lane + 32 * q;
    const bool ok = j < n;
    wj[q] = ok ? Wp[j] : 0.0;
    vpj[q] = ok ? Vp[j] : 0.0;
    vnj[q] = (!ok || reduced) ? 0.0 : (j == c0 ? v1 : Vr[j]);
  }
  for (int i0 = c0 + warp; i0 < n; i0 += kEbWarps * R) {
    double x[R][Q];
    double* rowp[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = i0 + kEbWarps * r;
      rowp[r] = M + pk(i < n ? i : c0, c0, org);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int j = c0 + lane + 32 * q;
        x[r][q] = (i < n && j <= i) ? rowp[r][lane + 32 * q] : 0.0;
      }
    }
    double rs[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = i0 + kEbWarps * r;
      rs[r] = 0.0;
      if (i < n) {
        const double vpi = Vp[i], wpi = Wp[i];
        const double vni = reduced ? 0.0 : (i == c0 ? v1 : Vr[i]);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int j = c0 + lane + 32 * q;
          if (j <= i) {
            const double a = x[r][q] - (vpi * wj[q] + wpi * vpj[q]);
            rowp[r][lane + 32 * q] = a;
            rs[r] = fma(a, vnj[q], rs[r]);
            if (j < i) cp[q] = fma(a, vni, cp[q]);
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int r = 0; r < R; ++r) rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], o);
    if (lane == 0)
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (i0 + kEbWarps * r < n) Prow[i0 + kEbWarps * r] = rs[r];
  }
}

__global__ void __launch_bounds__(kEbThreads) k_effrank_big(
    const DevT2* __restrict__ T, int D, int rr, const double* __restrict__ GI,
    const uint8_t* __restrict__ gathered, int64_t pay_bytes, double* __restrict__ work,
    double tau, int* __restrict__ per, double* __restrict__ energy, int shard, int nshards) {
  extern __shared__ double eb_sm[];
  __shared__ double red[kEbWarps];
  __shared__ double s_b[4];
  __shared__ int s_i[2];
  const int e = shard + blockIdx.x * nshards;
  const DevT2& t = T[e];
  const int K = D * t.r;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int64_t mat = (int64_t)rr * rr;
  double* gL = work + 3 * (int64_t)blockIdx.x * mat;  // L (lower), stride K
  double* gA = gL + mat;                              // G_A, later packed M
  double* gT = gA + mat;                              // G_A L
  double* sA = eb_sm;                                 // P-side column scales
  double* sB = sA + kEbVec;                           // Q-side column scales
  double* Vp = sB + kEbVec;                           // v, w of the previous step
  double* Wp = Vp + kEbVec;
  double* Vn = Wp + kEbVec;                           // column k, parity k & 1 (with Pn)
  double* Pn = Vn + kEbVec;
  double* Dg = Pn + kEbVec;                           // tridiagonal: diagonal
  double* E2 = Dg + kEbVec;                           // squared off-diagonal
  double* colp = E2 + kEbVec;                         // [16][256] column partials
  double* R = colp + kEbWarps * kEbVec;               // region
  long long pt0 = clock64();
#define EB_MARK(i) do { if (blockIdx.x == 0 && tid == 0) { const long long c = clock64(); g_er_prof[i] = c - pt0; pt0 = c; } } while (0)
  // ---- 0. scales, G_B -> gL (lower), G_A -> gA
  for (int i = tid; i < K; i += kEbThreads) {
    const int w = i / t.r, j = i % t.r;
    sA[i] = *reinterpret_cast<const float*>(gathered + w * pay_bytes + t.seg_ps + 4 * j);
    sB[i] = *reinterpret_cast<const float*>(gathered + w * pay_bytes + t.seg_qs + 4 * j);
  }
  __syncthreads();
  const double* giA = GI + (int64_t)e * 2 * mat;
  const double* giB = giA + mat;
  double dloc = 0.0;
  for (int idx = tid; idx < K * K; idx += kEbThreads) {
    const int i = idx / K, k = idx % K;
    const int lo = min(i, k), hi = max(i, k);
    gA[idx] = giA[lo * rr + hi] * sA[i] * sA[k];
    const double b = giB[lo * rr + hi] * sB[i] * sB[k];
    gL[idx] = k <= i ? b : 0.0;
    if (i == k) dloc = fmax(dloc, b);
  }
  const double floor_piv = 1e-14 * eb_block_reduce(dloc, red, true);
  __syncthreads();
  EB_MARK(0);
  // ---- 1. blocked semidefinite Cholesky (columns with a vanishing pivot are dropped)
  for (int p0 = 0; p0 < K; p0 += 32) {
    const int pw = min(32, K - p0), rows = K - p0;
    double* Pm = R;  // [rows][kEbPld]
    for (int idx = tid; idx < rows * 32; idx += kEbThreads) {
      const int r = idx / 32, c = idx % 32;
      if (c < pw) Pm[r * kEbPld + c] = gL[(int64_t)(p0 + r) * K + p0 + c];
    }
    __syncthreads();
    for (int j = 0; j < pw; ++j) {
      if (tid == 0) {
        const double d = Pm[j * kEbPld + j];
        const bool keep = d > floor_piv && d > 0.0;
        s_b[0] = keep ? sqrt(d) : 0.0;
        s_b[1] = keep ? 1.0 / s_b[0] : 0.0;
      }
      __syncthreads();
      const double inv = s_b[1];
      for (int r = j + 1 + tid; r < rows; r += kEbThreads) Pm[r * kEbPld + j] *= inv;
      if (tid == 0) Pm[j * kEbPld + j] = s_b[0];
      __syncthreads();
      const int nc = pw - j - 1;
      if (nc > 0)
        for (int idx = tid; idx < (rows - j - 1) * nc; idx += kEbThreads) {
          const int r = j + 1 + idx / nc, c = j + 1 + idx % nc;
          if (r >= c) Pm[r * kEbPld + c] -= Pm[r * kEbPld + j] * Pm[c * kEbPld + j];
        }
      __syncthreads();
    }
    for (int idx = tid; idx < rows * 32; idx += kEbThreads) {
      const int r = idx / 32, c = idx % 32;
      if (c < pw) gL[(int64_t)(p0 + r) * K + p0 + c] = r >= c ? Pm[r * kEbPld + c] : 0.0;
    }
    // trailing SYRK (lower 8x8 blocks): L[i][k] -= sum_j Pm[i][j] Pm[k][j]
    const int mt = K - p0 - pw, nb = (mt + 7) / 8;
    for (int blk = warp; blk < nb * (nb + 1) / 2; blk += kEbWarps) {
      int bi = 0, rem = blk;
      while (rem > bi) {
        rem -= bi + 1;
        ++bi;
      }
      const int bj = rem;
      double acc[2] = {0.0, 0.0};
      const int ra = pw + 8 * bi + lane / 4, rb = pw + 8 * bj + lane / 4;
      for (int k0 = 0; k0 < pw; k0 += 4) {
        const int kc = k0 + lane % 4;
        const double a = (ra < rows && kc < pw) ? Pm[ra * kEbPld + kc] : 0.0;
        const double b = (rb < rows && kc < pw) ? Pm[rb * kEbPld + kc] : 0.0;
        dmma_8x8x4(acc, a, b);
      }
      const int i = p0 + pw + 8 * bi + lane / 4;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int j = p0 + pw + 8 * bj + 2 * (lane % 4) + q;
        if (i < K && j <= i) gL[(int64_t)i * K + j] -= acc[q];
      }
    }
    __syncthreads();
  }
  EB_MARK(1);
  // ---- 2. T = G_A L (L[k][j] = 0 for k < j), then lower(M) = lower(L^T T) packed into gA
  {
    double* As = R;
    double* Bs = R + 64 * kEbTA;
    const int nt64 = (K + 63) / 64;
    for (int tile = 0; tile < nt64 * nt64; ++tile) {
      const int ti = tile / nt64, tj = tile % nt64;
      double acc[4][2];
      eb_tile<false>(gA, gL, K, 64 * ti, 64 * tj, 64 * tj, As, Bs, acc);
      const int i = 64 * ti + 8 * (warp / 2) + lane / 4;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int j = 64 * tj + 8 * (4 * (warp % 2) + u) + 2 * (lane % 4) + q;
          if (i < K && j < K) gT[(int64_t)i * K + j] = acc[u][q];
        }
    }
    __syncthreads();
    for (int ti = 0; ti < nt64; ++ti)
      for (int tj = 0; tj <= ti; ++tj) {
        double acc[4][2];
        eb_tile<true>(gL, gT, K, 64 * ti, 64 * tj, 64 * ti, As, Bs, acc);
        const int i = 64 * ti + 8 * (warp / 2) + lane / 4;
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int j = 64 * tj + 8 * (4 * (warp % 2) + u) + 2 * (lane % 4) + q;
            if (i < K && j <= i) gA[pk(i, j, 0)] = acc[u][q];
          }
      }
    __syncthreads();
  }
  EB_MARK(2);
  // ---- 3. tridiagonalisation, packed lower storage, update of step k-1 fused into step k.
  // Three block barriers per step: column reduction, fused pass, dot reduction. v of step k
  // is the column itself except at k+1 (vget), so it needs no barrier of its own.
  const int n = K;
  double* Mg = gA;
  double* M = Mg;
  int org = 0;
  bool in_smem = false;
  double* Vr2 = Vn;   // raw column k (= v but at k+1), two parity buffers: Vn | Pn
  double* Prow = sA;  // row sums (the scales are dead after staging)
  for (int i = tid; i < kEbVec; i += kEbThreads) {
    Vp[i] = 0.0;
    Wp[i] = 0.0;
  }
  double trace_loc = 0.0;
  double vk = 0.0, wk = 0.0;  // v, w of step k-1 at index k (carried in registers)
  __shared__ double redA[2][kEbWarps], redB[2][kEbWarps];
  __syncthreads();
  for (int k = 0; k + 1 < n; ++k) {
    const int m = n - k;
    if (!in_smem && (int64_t)m * (m + 1) / 2 <= kEbRegion) {
      for (int i = k + warp; i < n; i += kEbWarps)
        for (int j = k + lane; j <= i; j += 32) R[pk(i, j, k)] = Mg[pk(i, j, 0)];
      __syncthreads();
      M = R;
      org = k;
      in_smem = true;
    }
    double* Vr = Vr2 + (k & 1) * kEbVec;
    // A. column k of A^(k) = stored column - (v w^T + w v^T) of step k-1
    const int ic = k + tid;
    double x = 0.0;
    if (ic < n) {
      x = M[pk(ic, k, org)] - (Vp[ic] * wk + Wp[ic] * vk);
      Vr[ic] = x;
    }
    double ssp = (ic > k && ic < n) ? x * x : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ssp += __shfl_xor_sync(0xffffffffu, ssp, o);
    if (lane == 0) redA[k & 1][warp] = ssp;
    __syncthreads();  // #1
    double ss = 0.0;
#pragma unroll
    for (int w = 0; w < kEbWarps; ++w) ss += redA[k & 1][w];
    const double x0 = Vr[k + 1];
    const double nrm = sqrt(ss);
    const bool reduced = !(ss - x0 * x0 > 1e-300 * ss) || nrm == 0.0;
    const double alpha = reduced ? x0 : (x0 > 0.0 ? -nrm : nrm);
    const double H = reduced ? 0.0 : ss - x0 * alpha;  // ||v||^2 / 2
    const double v1 = reduced ? 0.0 : x0 - alpha;
    if (tid == 0) {
      Dg[k] = Vr[k];
      E2[k] = alpha * alpha;
      trace_loc += Vr[k];
    }
    // B. fused pass over the trailing triangle [k+1, n): apply step k-1, accumulate A^(k) v
    const int c0 = k + 1, nc = n - c0;
    double cp[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) cp[q] = 0.0;
    if (nc > 128)
      eb_pass<8>(M, org, n, c0, warp, lane, Vp, Wp, Vr, v1, reduced, Prow, cp);
    else
      eb_pass<4>(M, org, n, c0, warp, lane, Vp, Wp, Vr, v1, reduced, Prow, cp);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (32 * q < nc) colp[warp * kEbVec + lane + 32 * q] = cp[q];
    __syncthreads();  // #3
    // C. p / H, v . p, and w = p / H - K v
    const auto vget = [&](int j) { return reduced ? 0.0 : (j == c0 ? v1 : Vr[j]); };
    double p_own = 0.0, dot = 0.0;
    if (tid < nc) {
      double p = Prow[c0 + tid];
      for (int w = 0; w < kEbWarps; ++w) p += colp[w * kEbVec + tid];
      p_own = H != 0.0 ? p / H : 0.0;
      dot = vget(c0 + tid) * p_own;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) redB[k & 1][warp] = dot;
    double pc0 = Prow[c0];  // p at c0, needed by every thread next step (w at index k+1)
    for (int w = 0; w < kEbWarps; ++w) pc0 += colp[w * kEbVec];
    pc0 = H != 0.0 ? pc0 / H : 0.0;
    __syncthreads();  // #4
    double dsum = 0.0;
#pragma unroll
    for (int w = 0; w < kEbWarps; ++w) dsum += redB[k & 1][w];
    const double Kc = H != 0.0 ? dsum / (2.0 * H) : 0.0;
    if (tid < nc) {
      const double v = vget(c0 + tid);
      Vp[c0 + tid] = v;
      Wp[c0 + tid] = p_own - Kc * v;
    }
    vk = v1;
    wk = pc0 - Kc * v1;
  }
  if (tid == 0) {
    const double a = M[pk(n - 1, n - 1, org)] - 2.0 * vk * wk;
    Dg[n - 1] = a;
    E2[n - 1] = 0.0;
    trace_loc += a;
  }
  const double trace = eb_block_reduce(trace_loc, red, false);
  __syncthreads();
  EB_MARK(3);
  // ---- 4. eigenvalues by Sturm multisection, stopped once the intervals decide r'
  double lo = 0.0, hi = 0.0, amax = 0.0;
  for (int i = 0; i < n; ++i) {  // Gershgorin (every thread, uniform)
    const double r0 = i > 0 ? sqrt(E2[i - 1]) : 0.0, r1 = i + 1 < n ? sqrt(E2[i]) : 0.0;
    lo = fmin(lo, Dg[i] - r0 - r1);
    hi = fmax(hi, Dg[i] + r0 + r1);
    amax = fmax(amax, fabs(Dg[i]) + r0 + r1);
  }
  hi += 1e-14 * amax + 1e-300;
  lo -= 1e-14 * amax + 1e-300;
  double* ilo = Vp;  // per eigenvalue (descending order) interval
  double* ihi = Wp;
  const int G = 2;   // lanes per eigenvalue: n <= 256 eigenvalues per pass
  const int idx = tid / G, l = tid % G;
  double blo = lo, bhi = hi;
  const unsigned gmask = 3u << ((tid % 32) / G * G);
  int kres = 1;
  constexpr int kMaxIt = 34;  // 3^34 > 2^53: fully converged
  const int idc = min(idx, n - 1);  // lanes past n repeat the last eigenvalue (uniform warps)
  for (int it = 0; it < kMaxIt; ++it) {
    {
      const double sig = blo + (bhi - blo) * (double)(l + 1) / (double)(G + 1);
      int c = 0;
      double pm = 1.0, p = Dg[0] - sig;
      bool neg_prev = false;
      bool neg = p < 0.0 || p == 0.0;
      c += neg != neg_prev;
      neg_prev = neg;
      for (int j = 1; j < n; ++j) {
        const double pn = fma(Dg[j] - sig, p, -E2[j - 1] * pm);
        neg = pn == 0.0 ? !neg_prev : pn < 0.0;
        c += neg != neg_prev;
        neg_prev = neg;
        pm = p;
        p = pn;
        const double ap = fabs(p) + fabs(pm);
        if (ap > 0x1p+600) {
          p = scalbn(p, -600);
          pm = scalbn(pm, -600);
        } else if (ap < 0x1p-600) {
          p = scalbn(p, 600);
          pm = scalbn(pm, 600);
        }
      }
      const unsigned below = __ballot_sync(0xffffffffu, c <= idc) & gmask;
      const int L = __popc(below);
      const int base = (tid % 32) / G * G;
      const double s_lo = __shfl_sync(0xffffffffu, sig, base + max(L - 1, 0));
      const double s_hi = __shfl_sync(0xffffffffu, sig, base + min(L, G - 1));
      if (L > 0) blo = s_lo;
      if (L < G) bhi = s_hi;
      if (l == 0 && idx < n) {
        ilo[n - 1 - idx] = fmax(blo, 0.0);
        ihi[n - 1 - idx] = fmax(bhi, 0.0);
      }
    }
    __syncthreads();
    if ((it >= 6 || it == kMaxIt - 1) && warp == 0) {
      // prefix sums of lo / hi / mid over the descending eigenvalues (8 per lane + warp scan)
      double a_lo[8], a_hi[8];
      double slo = 0.0, shi = 0.0, smid = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int i = 8 * lane + q;
        a_lo[q] = i < n ? ilo[i] : 0.0;
        a_hi[q] = i < n ? ihi[i] : 0.0;
        slo += a_lo[q];
        shi += a_hi[q];
        smid += 0.5 * (a_lo[q] + a_hi[q]);
      }
      double plo = slo, phi = shi, pmid = smid;  // inclusive scans
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double u0 = __shfl_up_sync(0xffffffffu, plo, o);
        const double u1 = __shfl_up_sync(0xffffffffu, phi, o);
        const double u2 = __shfl_up_sync(0xffffffffu, pmid, o);
        if (lane >= o) {
          plo += u0;
          phi += u1;
          pmid += u2;
        }
      }
      const double tlo = __shfl_sync(0xffffffffu, plo, 31);
      const double thi = __shfl_sync(0xffffffffu, phi, 31);
      const double tmid = __shfl_sync(0xffffffffu, pmid, 31);
      // candidate k from the midpoints: first i with prefix_mid >= tau * total_mid
      double elo = plo - slo, ehi = phi - shi, emid = pmid - smid;  // exclusive
      int kc = 1 << 30;
      bool ok = true;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int i = 8 * lane + q;
        const double mid = 0.5 * (a_lo[q] + a_hi[q]);
        if (i < n && kc == (1 << 30) && emid + mid >= tau * tmid) {
          kc = i;
          // certified: (1 - tau) prefix_{<i} < tau suffix_{>=i} and
          //            (1 - tau) prefix_{<=i} >= tau suffix_{>i}
          const double pre_hi = ehi, suf_lo = tlo - elo;
          const double pre_lo = elo + a_lo[q], suf_hi = thi - ehi - a_hi[q];
          ok = (1.0 - tau) * pre_hi < tau * suf_lo && (1.0 - tau) * pre_lo >= tau * suf_hi;
        }
        elo += a_lo[q];
        ehi += a_hi[q];
        emid += mid;
      }
      // first lane holding the candidate decides
      const unsigned has = __ballot_sync(0xffffffffu, kc != (1 << 30));
      const int src = has ? __ffs(has) - 1 : 0;
      const int kfin = __shfl_sync(0xffffffffu, kc, src);
      const bool okf = __shfl_sync(0xffffffffu, ok, src);
      if (lane == 0) {
        const bool zero = !(trace > 0.0);
        s_i[0] = zero ? 1 : (has ? kfin + 1 : n);
        s_i[1] = zero || (has && okf) || it == kMaxIt - 1;
      }
    }
    __syncthreads();
    if ((it >= 6 || it == kMaxIt - 1) && s_i[1]) break;
  }
  kres = s_i[0];
  EB_MARK(4);
  if (tid == 0) {
    per[e] = kres;
    energy[e] = fmax(trace, 0.0) / ((double)D * (double)D);
  }
#undef EB_MARK
}

static void launch_effrank(const Plan& P, int D, int rr, const double* GA, const double* GB,
                           const double* GI, const uint8_t* gathered, double* W, double tau,
                           int* d_per, double* d_energy, int shard, int nshards,
                           cudaStream_t s) {
  smem_optin(reinterpret_cast<const void*>(k_effrank),
             static_cast<int>(sizeof(double) * kErSwitch * (kErSwitch + 1)));
  int n2max = 0;
  for (const DevT2& t : P.t2) n2max = std::max(n2max, D * t.r + ((D * t.r) & 1));
  if (n2max > kErMaxN) raise(DLX_ERR_VALIDATION, "effective_rank: D * rank above 256 unsupported");
  const int ne = static_cast<int>(P.t2.size());
  const int nb = (ne - shard + nshards - 1) / nshards;
  if (nb <= 0) return;
  if (GI && n2max > option_effrank_big_from()) {
    smem_optin(reinterpret_cast<const void*>(k_effrank_big), static_cast<int>(kEbSmem));
    k_effrank_big<<<nb, kEbThreads, kEbSmem, s>>>(P.d_t2, D, rr, GI, gathered, P.payload_bytes,
                                                  W, tau, d_per, d_energy, shard, nshards);
    DLX_LAUNCHED();
    if (getenv("DLX_ER_PROF")) {
      long long h[8];
      DLX_CUDA(cudaStreamSynchronize(s));
      DLX_CUDA(cudaMemcpyFromSymbol(h, g_er_prof, sizeof(h)));
      long long z[16] = {};
      DLX_CUDA(cudaMemcpyFromSymbol(h, g_er_prof, sizeof(h)));
      long long hh[16];
      DLX_CUDA(cudaMemcpyFromSymbol(hh, g_er_prof, sizeof(hh)));
      DLX_CUDA(cudaMemcpyToSymbol(g_er_prof, z, sizeof(z)));
      fprintf(stderr, "[k_effrank_big n=%d] cycles: stage %lld chol %lld products %lld tridiag %lld sturm %lld\n",
              n2max, h[0], h[1], h[2], h[3], h[4]);
      (void)hh;
    }
    return;
  }
  int sdim = 0, mdim = 0;
  size_t smem = 0;
  if (n2max <= kErAllSmem) {
    sdim = n2max;
    smem = 3 * static_cast<size_t>(sdim) * (sdim + 1) * sizeof(double);
  } else if (n2max <= kErMSmem) {
    mdim = n2max;
    smem = static_cast<size_t>(mdim) * (mdim + 1) * sizeof(double);
  } else {
    smem = static_cast<size_t>(kErSwitch) * (kErSwitch + 1) * sizeof(double);
  }
  const int threads = n2max <= 64 ? 256 : 512;
  k_effrank<<<nb, threads, smem, s>>>(P.d_t2, D, rr, GA, GB, GI, gathered, P.payload_bytes,
                                      sdim, mdim, W, tau, d_per, d_energy, shard, nshards);
  DLX_LAUNCHED();
  if (getenv("DLX_ER_PROF")) {
    long long h[8];
    DLX_CUDA(cudaStreamSynchronize(s));
    DLX_CUDA(cudaMemcpyFromSymbol(h, g_er_prof, sizeof(h)));
    fprintf(stderr, "[k_effrank n=%d] cycles: stage %lld chol %lld products %lld tridiag %lld sturm %lld\n",
            n2max, h[0], h[1], h[2], h[3], h[4]);
  }
}

void effective_rank_factors(dlx_ctx* ctx, const Plan& P, int D, const uint8_t* gathered,
                            double tau, int* d_per, double* d_energy, int shard, int nshards,
                            cudaStream_t s) {
  HostProf hp_("effective_rank_factors");
  if (P.t2.empty()) return;
  if (nshards < 1 || shard < 0 || shard >= nshards)
    raise(DLX_ERR_VALIDATION, "effective_rank: need 0 <= shard < nshards");
  if (nshards > 1) {  // tensors of other shards report (0, 0)
    DLX_CUDA(cudaMemsetAsync(d_per, 0, sizeof(int) * P.t2.size(), s));
    DLX_CUDA(cudaMemsetAsync(d_energy, 0, sizeof(double) * P.t2.size(), s));
  }
  int K = 0;
  for (const DevT2& t : P.t2) K = std::max(K, D * t.r);
  if (K > kErMaxN) raise(DLX_ERR_VALIDATION, "effective_rank: D * rank above 256 unsupported");
  const int64_t mat = static_cast<int64_t>(K) * K;
  const size_t ne = P.t2.size();
  const int nown = (static_cast<int>(ne) - shard + nshards - 1) / nshards;
  if (nown <= 0) return;
  auto* W = static_cast<double*>(ctx->scratch("er_W", sizeof(double) * mat * nown * 3));
  // integer code Grams straight from the gathered payloads
  bool fresh = false;
  CodeGramJob& J = plan_ext<CodeGramJob>(
      P, "code_gram/" + std::to_string(shard) + "/" + std::to_string(nshards), &fresh);
  if (fresh) {
    for (size_t k = shard; k < ne; k += static_cast<size_t>(nshards))
      for (int side = 0; side < 2; ++side) {
        const int64_t n = side == 0 ? P.t2[k].a : P.t2[k].b;
        for (int64_t r0 = 0; r0 < n; r0 += kCgChunk)
          J.chunks.push_back(make_int4(static_cast<int>(k), side, static_cast<int>(r0),
                                       static_cast<int>(std::min(n, r0 + kCgChunk))));
      }
    J.d = plan_upload(P, J.chunks);
  }
  auto* GI = static_cast<double*>(ctx->scratch("er_GI", sizeof(double) * mat * ne * 2));
  DLX_CUDA(cudaMemsetAsync(GI, 0, sizeof(double) * mat * ne * 2, s));
  if (J.chunks.empty()) return;
  {
    const int nt32 = (K + 31) / 32;
    const int gy = (nt32 * (nt32 + 1) / 2 + kCgmWarps * kCgmTilesPerWarp - 1) /
                   (kCgmWarps * kCgmTilesPerWarp);
    k_code_gram_mma<<<dim3(J.chunks.size(), gy), 256, 0, s>>>(P.d_t2, J.d, gathered,
                                                              P.payload_bytes, P.qbits, D, K, GI);
    DLX_LAUNCHED();
  }
  launch_effrank(P, D, K, nullptr, nullptr, GI, gathered,
                 W, tau, d_per, d_energy, shard, nshards, s);
}

}  // namespace dlx
