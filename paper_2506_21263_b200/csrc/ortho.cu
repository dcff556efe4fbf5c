// ortho.cu — batched orthonormalisation of the power-iteration factors
// (orthonormalize tensor.cpp:174-227).
//
// B200 design: all factors of one side (every P, or every Q) are orthonormalised in one
// pass of four launches instead of a column-serial MGS per tensor:
//   Gram (fp64, row-split, deterministic) -> Cholesky + R^-1 (one CTA per factor)
//   -> apply Y R^-1 (fp64 accumulate)  — twice (CholQR2, equal to MGS2 up to rounding).
// Cholesky + R^-1: r <= 32 one warp in registers (warp_chol_inv); 32 < r <= 128 blocked,
// 32-wide panels (k_cholblk: warp_chol_inv on the diagonal blocks, DMMA for the panel rows,
// trailing updates and the off-diagonal blocks of R^-1); above, k_chol in global memory.
// A factor whose Cholesky pivot falls within 10x of the reference's dependence tolerance
// (1e-7 * max(1, largest column norm)) is left untouched by CholQR2 and re-done by an exact
// MGS2 kernel with the reference's seeded column replacement (RngStream(0x5eedc01,
// stream_key({n, r, j, attempt}))). That path only triggers on (near) rank-deficient
// inputs such as all-zero tensors.
#include <cstdlib>

#include "dlx_internal.cuh"
#include "ptx.cuh"

namespace dlx {

// ------------------------------------------------------------------ job tables
struct GramJob : PlanExt {
  std::vector<DevMat> mats;
  DevMat* d_mats = nullptr;
  std::vector<int4> splits;  // (entry, row0, row1, part index)
  int4* d_splits = nullptr;
  std::vector<int4> apply;   // (entry, row0, col block, -)
  int4* d_apply = nullptr;
  std::vector<int> part0;    // per entry: first part index
  int* d_part0 = nullptr;
  std::vector<int> nparts;   // per entry
  int* d_nparts = nullptr;
  int rmax = 0;
  int total_parts = 0;
};

static void make_job(const Plan& P, GramJob* J, const std::vector<DevMat>& mats) {
  J->mats = mats;
  for (size_t e = 0; e < mats.size(); ++e) {
    const DevMat& m = mats[e];
    J->rmax = std::max(J->rmax, m.r);
    static const int64_t split_rows = [] {  // experiments: DLX_GRAM_SPLIT
      const char* e = getenv("DLX_GRAM_SPLIT");
      return static_cast<int64_t>(e ? atoi(e) : 512);
    }();
    // at most kMaxParts row splits per factor: the Cholesky kernels fold an entry's partials
    // in one CTA, so the longest factor (the 50272-row embedding: ~100 splits of 512 rows)
    // set the whole launch's duration
    constexpr int64_t kMaxParts = 32;
    const int64_t ns = std::max<int64_t>(1, std::min(kMaxParts, ceil_div(m.n, split_rows)));
    const int64_t rows = round_up(ceil_div(m.n, ns), 32);
    J->part0.push_back(J->total_parts);
    int cnt = 0;
    for (int64_t r0 = 0; r0 < m.n; r0 += rows, ++cnt)
      J->splits.push_back(make_int4(static_cast<int>(e), static_cast<int>(r0),
                                    static_cast<int>(std::min(m.n, r0 + rows)),
                                    J->total_parts + cnt));
    J->nparts.push_back(cnt);
    J->total_parts += cnt;
    for (int64_t r0 = 0; r0 < m.n; r0 += 128)
      J->apply.push_back(make_int4(static_cast<int>(e), static_cast<int>(r0), 0, 0));
  }
  J->d_mats = plan_upload(P, J->mats);
  J->d_splits = plan_upload(P, J->splits);
  J->d_apply = plan_upload(P, J->apply);
  J->d_part0 = plan_upload(P, J->part0);
  J->d_nparts = plan_upload(P, J->nparts);
}

static GramJob& job_for(const Plan& P, const std::string& key,
                        const std::vector<DevMat>& mats) {
  bool fresh = false;
  GramJob& J = plan_ext<GramJob>(P, "gram:" + key, &fresh);
  if (fresh) make_job(P, &J, mats);
  return J;
}

// ------------------------------------------------------------------ deterministic reduce
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32, nw = blockDim.x / 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += red[i];  // fixed order
  return s;
}

// ------------------------------------------------------------------ Gram (fp64)
// partial[p][j*rr + k] = sum over rows of the split of Y[row, j] * Y[row, k] for the
// 4x4 block of (j, k) owned by a thread (upper block triangle only).
constexpr int kGramRows = 32;

__global__ void __launch_bounds__(256) k_gram(const DevMat* __restrict__ mats,
                                              const int4* __restrict__ splits,
                                              const float* __restrict__ buf, int rr,
                                              double* __restrict__ partial,
                                              const int* __restrict__ only) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int4 sp = splits[blockIdx.x];
  if (only && !only[sp.x]) return;  // entry not selected for this pass
  const DevMat m = mats[sp.x];
  const int nb = (m.r + 3) / 4, nblk = nb * (nb + 1) / 2;
  float* Ys = reinterpret_cast<float*>(smem_raw);  // [rpad][kGramRows + 1] (padded: no bank conflicts)
  const int rpad = nb * 4;
  // thread -> (block, group); block index across grid.y passes when nblk > 256
  const int groups = nblk >= 256 ? 1 : 256 / nblk;
  const int blk = nblk >= 256 ? threadIdx.x + 256 * blockIdx.y : threadIdx.x % nblk;
  const int grp = nblk >= 256 ? 0 : threadIdx.x / nblk;
  const bool active = blk < nblk && grp < groups;
  if (nblk < 256 && blockIdx.y > 0) return;  // uniform per CTA
  int jb = 0, kb = 0;
  if (active) {  // unrank blk -> (jb <= kb), row-major over the upper block triangle
    int rem = blk;
    jb = 0;
    while (rem >= nb - jb) {
      rem -= nb - jb;
      ++jb;
    }
    kb = jb + rem;
  }
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  const float* Y = buf + m.off;
  for (int r0 = sp.y; r0 < sp.z; r0 += kGramRows) {
    __syncthreads();
    for (int e = threadIdx.x; e < rpad * kGramRows; e += 256) {
      const int c = e / kGramRows, rr0 = e % kGramRows;
      const int row = r0 + rr0;
      Ys[c * (kGramRows + 1) + rr0] = (c < m.r && row < sp.z) ? Y[(int64_t)c * m.ld + row] : 0.f;
    }
    __syncthreads();
    if (active) {
      for (int rr0 = grp; rr0 < kGramRows; rr0 += groups) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          a[i] = (double)Ys[(jb * 4 + i) * (kGramRows + 1) + rr0];
          b[i] = (double)Ys[(kb * 4 + i) * (kGramRows + 1) + rr0];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
    }
  }
  // reduce groups in fixed order through shared memory
  __syncthreads();
  double* red = reinterpret_cast<double*>(smem_raw);
  if (groups > 1) {
    if (active)
#pragma unroll
      for (int i = 0; i < 16; ++i) red[(grp * nblk + blk) * 16 + i] = acc[i / 4][i % 4];
    __syncthreads();
    if (active && grp == 0) {
      for (int g = 1; g < groups; ++g)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i / 4][i % 4] += red[(g * nblk + blk) * 16 + i];
    }
  }
  if (active && grp == 0) {
    double* out = partial + (int64_t)sp.w * rr * rr;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int gj = jb * 4 + i, gk = kb * 4 + j;
        if (gj < m.r && gk < m.r) out[gj * rr + gk] = acc[i][j];
      }
  }
}

// r <= 32 fast path on the fp64 tensor cores (mma.sync m8n8k4 f64, DMMA): 64-row tiles of
// Y staged once as fp64 in shared memory, next tile prefetched into registers; warp w owns
// one 8x8 block (ci <= cj) of the upper block triangle of G = Y^T Y and accumulates it over
// every 4-row k step (A = Y^T block, B = Y block: the same fragment shape).
constexpr int kGdRows = 64;
constexpr int kGdLd = kGdRows + 4;  // [col][row] stride: conflict-free fragment loads


template <int TSH>  // tile rows 64 << TSH: 2 for r <= 8, 1 for r <= 16, 0 above
__global__ void __launch_bounds__(320) k_gram_dmma(const DevMat* __restrict__ mats,
                                                   const int4* __restrict__ splits,
                                                   const float* __restrict__ buf, int rr,
                                                   double* __restrict__ partial,
                                                   const int* __restrict__ only) {
  __shared__ double Ys[32 * kGdLd];
  const int4 sp = splits[blockIdx.x];
  if (only && !only[sp.x]) return;
  const DevMat m = mats[sp.x];
  const int nb = (m.r + 7) / 8, nblk = nb * (nb + 1) / 2;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // fewer columns -> taller tiles in the same shared memory (8 cols x 256 rows, 16 x 128,
  // 32 x 64), and the 10 warps split each tile's k steps between `nsl` slices of every 8x8
  // block (summed in a fixed order at the end): at the low ranks the adaptive schedule
  // reaches, one to three blocks otherwise left most warps idle behind two barriers per
  // 64 rows
  constexpr int TR = kGdRows << TSH, LD = TR + 4;
  const int nsl = TSH == 0 ? 1 : 10 / nblk;
  const int blk = warp % nblk, slice = warp / nblk;
  int ci = 0, cj = 0;
  {
    int rem = blk;
    while (ci < nb && rem >= nb - ci) {
      rem -= nb - ci;
      ++ci;
    }
    cj = ci + rem;
  }
  const bool active = slice < nsl;
  double acc[2] = {0.0, 0.0}, acc2[2] = {0.0, 0.0};  // two independent DMMA chains
  const float* Y = buf + m.off;
  const int cols = nb * 8;
  const int per = (cols * TR + 319) / 320;  // staged elements per thread (<= 7)
  float pre[7];
  auto fetch = [&](int r0) {
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      const int e = threadIdx.x + 320 * i;
      const int c = e >> (6 + TSH), rl = e & (TR - 1);
      const int row = r0 + rl;
      pre[i] = (i < per && c < m.r && row < sp.z) ? __ldg(&Y[(int64_t)c * m.ld + row]) : 0.f;
    }
  };
  fetch(sp.y);
  for (int r0 = sp.y; r0 < sp.z; r0 += TR) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      const int e = threadIdx.x + 320 * i;
      if (i < per && e < cols * TR) Ys[(e >> (6 + TSH)) * LD + (e & (TR - 1))] = (double)pre[i];
    }
    __syncthreads();
    if (r0 + TR < sp.z) fetch(r0 + TR);
    if (active) {
      const double* pa = Ys + (ci * 8 + lane / 4) * LD + lane % 4;
      const double* pb = Ys + (cj * 8 + lane / 4) * LD + lane % 4;
      if (TSH == 0) {  // nb >= 3: 64-row tiles, one slice, constant offsets
#pragma unroll 4
        for (int k = 0; k < kGdRows; k += 8) {
          dmma_8x8x4(acc, pa[k], pb[k]);
          dmma_8x8x4(acc2, pa[k + 4], pb[k + 4]);
        }
      } else {
        const int step = 4 * nsl;
        int k = 4 * slice;
        for (; k + step < TR; k += 2 * step) {
          dmma_8x8x4(acc, pa[k], pb[k]);
          dmma_8x8x4(acc2, pa[k + step], pb[k + step]);
        }
        if (k < TR) dmma_8x8x4(acc, pa[k], pb[k]);
      }
    }
  }
  // slices of a block summed in slice order (deterministic)
  double* red = Ys;  // [slice][blk][lane][2]
  if (TSH > 0) {
    __syncthreads();
    if (active && slice > 0) {
      red[((slice * nblk + blk) * 32 + lane) * 2] = acc[0] + acc2[0];
      red[((slice * nblk + blk) * 32 + lane) * 2 + 1] = acc[1] + acc2[1];
    }
    __syncthreads();
  }
  if (active && slice == 0) {
    acc[0] += acc2[0];
    acc[1] += acc2[1];
    for (int sl = 1; sl < nsl; ++sl) {
      acc[0] += red[((sl * nblk + blk) * 32 + lane) * 2];
      acc[1] += red[((sl * nblk + blk) * 32 + lane) * 2 + 1];
    }
    double* out = partial + (int64_t)sp.w * rr * rr;
    const int gj = ci * 8 + lane / 4;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int gk = cj * 8 + 2 * (lane % 4) + q;
      if (gj < m.r && gk < m.r && gj <= gk) out[gj * rr + gk] = acc[q];
    }
  }
}

// 32 < r <= 128 on DMMA: 32-row slabs of Y staged as fp64 ([col][row]); warp w owns the 8x8
// blocks w, w + 8, w + 16, ... of the upper block triangle of G = Y^T Y (up to 17 blocks at
// r = 128), one accumulator pair each — independent chains, so the DMMA pipe stays busy.
constexpr int kGbRows = 32;
constexpr int kGbLd = kGbRows + 4;

template <int NB>
__global__ void __launch_bounds__(256) k_gram_dmma_big(const DevMat* __restrict__ mats,
                                                       const int4* __restrict__ splits,
                                                       const float* __restrict__ buf, int rr,
                                                       double* __restrict__ partial,
                                                       const int* __restrict__ only) {
  constexpr int kMaxB = (NB * (NB + 1) / 2 + 7) / 8;  // blocks per warp
  constexpr int kPer = NB * 8 * kGbRows / 256;         // staged elements per thread
  __shared__ double Ys[NB * 8 * kGbLd];
  const int4 sp = splits[blockIdx.x];
  if (only && !only[sp.x]) return;
  const DevMat m = mats[sp.x];
  const int nb = (m.r + 7) / 8, nblk = nb * (nb + 1) / 2;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int ci[kMaxB], cj[kMaxB];
#pragma unroll
  for (int q = 0; q < kMaxB; ++q) {
    int rem = warp + 8 * q, a = 0;
    while (a < nb && rem >= nb - a) {
      rem -= nb - a;
      ++a;
    }
    ci[q] = a;
    cj[q] = a + rem;
  }
  double acc[kMaxB][2];
#pragma unroll
  for (int q = 0; q < kMaxB; ++q) acc[q][0] = acc[q][1] = 0.0;
  const float* Y = buf + m.off;
  float pre[kPer];
  auto fetch = [&](int r0) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = threadIdx.x + 256 * u;
      const int c = e / kGbRows, rl = e % kGbRows;
      const int row = r0 + rl;
      pre[u] = (c < m.r && row < sp.z) ? __ldg(&Y[(int64_t)c * m.ld + row]) : 0.f;
    }
  };
  fetch(sp.y);
  for (int r0 = sp.y; r0 < sp.z; r0 += kGbRows) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = threadIdx.x + 256 * u;
      Ys[(e / kGbRows) * kGbLd + e % kGbRows] = (double)pre[u];
    }
    __syncthreads();
    if (r0 + kGbRows < sp.z) fetch(r0 + kGbRows);
#pragma unroll
    for (int k = 0; k < kGbRows; k += 4) {
#pragma unroll
      for (int q = 0; q < kMaxB; ++q) {
        if (warp + 8 * q < nblk) {
          const double a = Ys[(ci[q] * 8 + lane / 4) * kGbLd + lane % 4 + k];
          const double b = Ys[(cj[q] * 8 + lane / 4) * kGbLd + lane % 4 + k];
          dmma_8x8x4(acc[q], a, b);
        }
      }
    }
  }
  double* out = partial + (int64_t)sp.w * rr * rr;
#pragma unroll
  for (int q = 0; q < kMaxB; ++q) {
    if (warp + 8 * q >= nblk) continue;
    const int gj = ci[q] * 8 + lane / 4;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gk = cj[q] * 8 + 2 * (lane % 4) + h;
      if (gj < m.r && gk < m.r && gj <= gk) out[gj * rr + gk] = acc[q][h];
    }
  }
}

static size_t gram_smem(int rmax) {
  const int rpad = (rmax + 3) / 4 * 4;
  return std::max<size_t>(sizeof(float) * rpad * (kGramRows + 1), sizeof(double) * 16 * 256);
}

static void launch_gram(const GramJob& J, const float* buf, double* partial, cudaStream_t s,
                        const int* only = nullptr) {
  if (J.rmax <= 32) {
    if (J.rmax <= 8)
      k_gram_dmma<2><<<J.splits.size(), 320, 0, s>>>(J.d_mats, J.d_splits, buf, J.rmax, partial, only);
    else if (J.rmax <= 16)
      k_gram_dmma<1><<<J.splits.size(), 320, 0, s>>>(J.d_mats, J.d_splits, buf, J.rmax, partial, only);
    else
      k_gram_dmma<0><<<J.splits.size(), 320, 0, s>>>(J.d_mats, J.d_splits, buf, J.rmax, partial, only);
    DLX_LAUNCHED();
    return;
  }
  if (J.rmax <= 64) {
    k_gram_dmma_big<8><<<J.splits.size(), 256, 0, s>>>(J.d_mats, J.d_splits, buf, J.rmax, partial,
                                                       only);
    DLX_LAUNCHED();
    return;
  }

  const int nb = (J.rmax + 3) / 4, nblk = nb * (nb + 1) / 2;
  const int gy = nblk >= 256 ? (nblk + 255) / 256 : 1;
  const size_t sm = gram_smem(J.rmax);
  smem_optin(reinterpret_cast<const void*>(k_gram), 64 * 1024);
  k_gram<<<dim3(J.splits.size(), gy), 256, sm, s>>>(J.d_mats, J.d_splits, buf, J.rmax, partial,
                                                     only);
  DLX_LAUNCHED();
}

// ------------------------------------------------------------------ Cholesky + R^-1
// G = sum_p partial[p] (fixed order); upper Cholesky G = R^T R; Rinv = R^-1 (upper).
// flags[e] = 1 if a pivot is within 10x of the reference dependence tolerance (exact MGS2
// fallback). need2[e] = 1 if the factor is ill-conditioned enough that a second CholQR pass
// is needed (cond_F(R) > 2e3): with an fp64 Gram of fp32 data, fp64 Cholesky and fp64 apply,
// one pass is already orthonormal to fp32 precision below that. Matrices live in shared
// memory for r <= 64, in the global work buffer otherwise.
__global__ void __launch_bounds__(256) k_chol(const DevMat* __restrict__ mats,
                                              const int* __restrict__ part0,
                                              const int* __restrict__ nparts, int rr,
                                              const double* __restrict__ partial,
                                              double* __restrict__ work,
                                              double* __restrict__ rinv,
                                              int* __restrict__ flags,
                                              int* __restrict__ need2,
                                              const int* __restrict__ only) {
  extern __shared__ __align__(16) unsigned char chol_smem[];
  __shared__ int s_flag;
  __shared__ double s_thr, red[8];
  const int e = blockIdx.x;
  if (only && !only[e]) {
    if (threadIdx.x == 0) {
      flags[e] = 0;
      if (need2) need2[e] = 0;
    }
    return;
  }
  const DevMat m = mats[e];
  const int r = m.r;
  const bool in_smem = rr <= 64;  // launch-uniform: dynamic smem is sized for rr
  const int ld = in_smem ? r : rr;
  double* W = in_smem ? reinterpret_cast<double*>(chol_smem) : work + (int64_t)e * rr * rr;
  double* X = in_smem ? W + r * r : rinv + (int64_t)e * rr * rr;
  const double* src = partial + (int64_t)part0[e] * rr * rr;
  const int np = nparts[e];
  for (int idx = threadIdx.x; idx < r * r; idx += blockDim.x) {
    const int j = idx / r, k = idx % r;
    if (k < j) continue;
    double g = 0.0;
    for (int p = 0; p < np; ++p) g += src[(int64_t)p * rr * rr + j * rr + k];
    W[j * ld + k] = g;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int j = 0; j < r; ++j) mx = fmax(mx, W[j * ld + j]);
    const double big = sqrt(mx);
    const double tol = 1e-7 * fmax(1.0, big);
    s_thr = (10.0 * tol) * (10.0 * tol);
    s_flag = 0;
  }
  __syncthreads();
  for (int j = 0; j < r; ++j) {
    if (threadIdx.x == 0) {
      const double d = W[j * ld + j];
      if (!(d > s_thr)) s_flag = 1;
    }
    __syncthreads();
    if (s_flag) break;
    const double rjj = sqrt(W[j * ld + j]);
    const double inv = 1.0 / rjj;
    __syncthreads();
    for (int k = j + 1 + threadIdx.x; k < r; k += blockDim.x) W[j * ld + k] *= inv;
    if (threadIdx.x == 0) W[j * ld + j] = rjj;
    __syncthreads();
    const int rem = r - j - 1;
    for (int idx = threadIdx.x; idx < rem * rem; idx += blockDim.x) {
      const int i = j + 1 + idx / rem, k = j + 1 + idx % rem;
      if (k < i) continue;
      W[i * ld + k] -= W[j * ld + i] * W[j * ld + k];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) flags[e] = s_flag;
  if (s_flag) {
    if (need2 && threadIdx.x == 0) need2[e] = 0;
    return;
  }
  // upper-triangular inverse, one column per thread (back substitution)
  double xf = 0.0, rf = 0.0;
  for (int c = threadIdx.x; c < r; c += blockDim.x) {
    X[c * ld + c] = 1.0 / W[c * ld + c];
    for (int i = c - 1; i >= 0; --i) {
      double sum = 0.0;
      for (int k = i + 1; k <= c; ++k) sum += W[i * ld + k] * X[k * ld + c];
      X[i * ld + c] = -sum / W[i * ld + i];
    }
    for (int i = c + 1; i < r; ++i) X[i * ld + c] = 0.0;
    for (int i = 0; i <= c; ++i) {
      xf += X[i * ld + c] * X[i * ld + c];
      rf += W[i * ld + c] * W[i * ld + c];
    }
  }
  if (need2) {
    double v[2] = {xf, rf};
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
    }
    if ((threadIdx.x & 31) == 0) {
      red[threadIdx.x / 32] = v[0];
    }
    __syncthreads();
    double xs = 0.0;
    for (int i = 0; i < 8; ++i) xs += red[i];
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = v[1];
    __syncthreads();
    double rs = 0.0;
    for (int i = 0; i < 8; ++i) rs += red[i];
    if (threadIdx.x == 0) need2[e] = (sqrt(xs) * sqrt(rs) > 2e3) ? 1 : 0;
  }
  if (in_smem) {
    __syncthreads();
    double* G = rinv + (int64_t)e * rr * rr;
    for (int idx = threadIdx.x; idx < r * r; idx += blockDim.x) G[(idx / r) * rr + idx % r] = X[idx];
  }
}

// (A register-tiled variant — 4 x 8 tiles per thread, pivot rows broadcast through shared
// memory — measured slower on the Llama-7B layer: r = 64 120 vs 70 us, r = 128 258 vs 219 us
// per call.)
// 32 < r <= 128: the whole factorisation in shared memory (r x (r + 1) doubles <= 132 KB):
// fold, right-looking Cholesky with the trailing update spread over 4 row groups x r
// columns, then R^-1 IN PLACE (upper triangular inversion column by column, the dot
// products of column j split over 4 lanes each) — no global round trips inside the O(r^3)
// loops. Same pivot test / flags / need2 as k_chol.
constexpr int kChol128Threads = 512;

__global__ void __launch_bounds__(kChol128Threads) k_chol128(const DevMat* __restrict__ mats,
                                                           const int* __restrict__ part0,
                                                           const int* __restrict__ nparts,
                                                           int rr,
                                                           const double* __restrict__ partial,
                                                           double* __restrict__ rinv,
                                                           int* __restrict__ flags,
                                                           int* __restrict__ need2,
                                                           const int* __restrict__ only) {
  extern __shared__ __align__(16) double Wc[];  // [r][r + 1], upper triangle used
  __shared__ double tmp[128];
  __shared__ double red[2][kChol128Threads / 32];
  const int e = blockIdx.x, tid = threadIdx.x;
  if (only && !only[e]) {
    if (tid == 0) {
      flags[e] = 0;
      if (need2) need2[e] = 0;
    }
    return;
  }
  const DevMat m = mats[e];
  const int r = m.r, ld = r + 1;
  const double* src = partial + (int64_t)part0[e] * rr * rr;
  const int np = nparts[e];
  const int64_t st = (int64_t)rr * rr;
  for (int idx = tid; idx < r * r; idx += kChol128Threads) {
    const int j = idx / r, k = idx % r;
    if (k < j) continue;
    const double* sp = src + j * rr + k;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    int p = 0;
    for (; p + 4 <= np; p += 4)
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] += sp[(p + u) * st];
    for (; p < np; ++p) a[p & 3] += sp[p * st];
    Wc[j * ld + k] = (a[0] + a[1]) + (a[2] + a[3]);
  }
  __syncthreads();
  double mx = 0.0;
  for (int j = 0; j < r; ++j) mx = fmax(mx, Wc[j * ld + j]);
  const double tol = 1e-7 * fmax(1.0, sqrt(mx));
  const double thr = (10.0 * tol) * (10.0 * tol);
  const int g = tid / 128, c = tid % 128;  // trailing update: row group g, column c
  int flag = 0;
  for (int j = 0; j < r; ++j) {
    const double d = Wc[j * ld + j];
    if (!(d > thr)) {  // every thread read the same pivot: uniform exit
      flag = 1;
      break;
    }
    const double rjj = sqrt(d), inv = 1.0 / rjj;
    __syncthreads();  // the pivot has been read everywhere
    for (int k = j + 1 + tid; k < r; k += kChol128Threads) Wc[j * ld + k] *= inv;
    if (tid == 0) Wc[j * ld + j] = rjj;
    __syncthreads();
    const int k = j + 1 + c;
    if (k < r) {
      const double rjk = Wc[j * ld + k];
      for (int i = j + 1 + g; i <= k; i += 4) Wc[i * ld + k] = fma(-Wc[j * ld + i], rjk, Wc[i * ld + k]);
    }
    __syncthreads();
  }
  if (tid == 0) flags[e] = flag;
  if (flag) {
    if (need2 && tid == 0) need2[e] = 0;
    return;
  }
  // ||R||_F^2 before the inversion overwrites R
  double rf = 0.0;
  for (int idx = tid; idx < r * r; idx += kChol128Threads) {
    const int i = idx / r, k = idx % r;
    if (k >= i) rf += Wc[i * ld + k] * Wc[i * ld + k];
  }
  __syncthreads();
  // R^-1 in place (upper): column j = -(inv(R[0:j,0:j]) R[0:j, j]) / R[j][j]
  for (int j = 0; j < r; ++j) {
    const double djj = 1.0 / Wc[j * ld + j];
    const int i = tid >> 2, q = tid & 3;  // row i, lane q of its 4-lane dot product
    double s = 0.0;
    if (i < j)
      for (int k = i + q; k < j; k += 4) s = fma(Wc[i * ld + k], Wc[k * ld + j], s);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (i < j && q == 0) tmp[i] = s;
    __syncthreads();
    for (int ii = tid; ii < j; ii += kChol128Threads) Wc[ii * ld + j] = -tmp[ii] * djj;
    if (tid == 0) Wc[j * ld + j] = djj;
    __syncthreads();
  }
  double xf = 0.0;
  double* X = rinv + (int64_t)e * rr * rr;
  for (int idx = tid; idx < r * r; idx += kChol128Threads) {
    const int i = idx / r, k = idx % r;
    const double v = k >= i ? Wc[i * ld + k] : 0.0;
    xf += v * v;
    X[i * rr + k] = v;
  }
  if (need2) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      xf += __shfl_xor_sync(0xffffffffu, xf, o);
      rf += __shfl_xor_sync(0xffffffffu, rf, o);
    }
    if ((tid & 31) == 0) {
      red[0][tid / 32] = xf;
      red[1][tid / 32] = rf;
    }
    __syncthreads();
    if (tid == 0) {
      double xs = 0.0, rs = 0.0;
      for (int w = 0; w < kChol128Threads / 32; ++w) {
        xs += red[0][w];
        rs += red[1][w];
      }
      need2[e] = (sqrt(xs) * sqrt(rs) > 2e3) ? 1 : 0;
    }
  }
}

// max of the first r diagonal entries of a shared-memory matrix, lane-parallel + warp
// reduction (every lane of the calling warp gets it)
__device__ __forceinline__ double warp_diag_max(const double* A, int ld, int r) {
  double mx = 0.0;
  for (int j = threadIdx.x & 31; j < r; j += 32) mx = fmax(mx, A[j * ld + j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  return mx;
}

// Branch-free fp64 1/sqrt: MUFU seed + two Newton steps (same result as the library rsqrt
// to 1 ulp on tools/micro/chol_micro.cu; one step leaves 1e-13). The library rsqrt carries a
// special-case branch, which splits the basic block and keeps the scheduler from overlapping
// the next pivot's square root with the current trailing update.
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double h = 0.5 * d;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

// Shared-memory scratch of one warp_chol_inv<RR>: the current pivot row of R (double-
// buffered; lane c stores R[j][c] at 32 + c - j - 1, so R[j][j+1 ..] starts on an aligned
// index) and the columns of R reversed (ct[k][d + 1] = R[k - d][k], zeros for k - d < 0).
template <int RR>
struct CholScratch {
  static constexpr int LC = 2 * RR + 2;  // ct row stride (doubles; rows 16-B aligned)
  double row[2][128];
  double ct[RR * LC];
};

// One warp factors the RR x RR (RR <= 32) symmetric block whose upper triangle sits in
// shared memory at G (row stride ldg) as G = R^T R and inverts R. Lane c owns column c; the
// step loops are ROLLED with a register window that shifts by one row per step (position
// i = row j + i), so every register index stays static (fully unrolled, the factorisation +
// inversion was ~10k instructions run by ONE warp per SM: instruction-cache misses were
// half of its time). tools/micro/chol_micro.cu (B200, one 32 x 32 factor + inverse per SM):
// unrolled with shuffles 33 us, rolled with shuffles 16.9 us, this 7.4 us.
//   factor: row j of R goes through shared memory and is read back with 16-B broadcast
//           loads; the next pivot is updated first and its rsqrt issued before the rest of
//           the trailing update (lookahead: the two dependent chains overlap); the updates
//           are unconditional — the strictly-lower entries (and rows past RR) they also touch
//           are never read;
//   invert: right-looking back substitution from the bottom — once x_k = R^-1[k][c] is known
//           every partial sum of the rows above takes its fma, column k of R read with 16-B
//           loads from ct, so the dependent chain is two ops per step;
//           put(k, x_k) receives row k of column c.
// rf / xf: this lane's ||R[:,c]||^2 / ||R^-1[:,c]||^2 for columns c < r; dinv[j] = 1/R[j][j].
// Returns the (warp-uniform) pivot failure (some pivot <= thr).
template <int RR, typename Put>
__device__ __forceinline__ bool warp_chol_inv(const double* G, int ldg, int r, double thr,
                                              double* dinv, CholScratch<RR>& sc, Put put,
                                              double& rf, double& xf) {
  constexpr int LC = CholScratch<RR>::LC;
  const int c = threadIdx.x & 31;
  const bool own = c < RR;
  double w[RR];  // w[i] = W[j + i][c]
#pragma unroll
  for (int i = 0; i < RR; ++i) w[i] = (i <= c && own) ? G[i * ldg + c] : 0.0;
  for (int i = c; i < RR * LC; i += 32) sc.ct[i] = 0.0;
  for (int i = c; i < 256; i += 32) sc.row[0][i] = 0.0;
  bool bad = false;
  rf = 0.0;
  __syncwarp();
  double d = __shfl_sync(0xffffffffu, w[0], 0);
  double inv = rsqrt_nr(d);
#pragma unroll 1
  for (int j = 0; j < RR; ++j) {
    bad |= !(d > thr);
    const double rj = c == j ? d * inv : w[0] * inv;  // R[j][c] for c >= j
    if (c == j) dinv[j] = inv;
    double* row = sc.row[j & 1];
    if (own) row[32 + c - j - 1] = rj;  // row[32 + i - 1] = R[j][j + i]
    if (own && c >= j) {
      sc.ct[c * LC + (c - j) + 1] = rj;
      if (c < r) rf = fma(rj, rj, rf);
    }
    __syncwarp();
    double rv[RR];
    const double2* rp = reinterpret_cast<const double2*>(row + 32);
#pragma unroll
    for (int i = 0; i < RR / 2; ++i) {
      const double2 t = rp[i];
      rv[2 * i] = t.x;
      rv[2 * i + 1] = t.y;
    }
    w[0] = fma(-rv[0], rj, w[1]);
    const double dn = __shfl_sync(0xffffffffu, w[0], (j + 1) & 31);
    const double invn = rsqrt_nr(dn);
#pragma unroll
    for (int i = 2; i < RR; ++i) w[i - 1] = fma(-rv[i - 1], rj, w[i]);  // W[j+i][c] -= R[j][j+i] R[j][c]
    w[RR - 1] = 0.0;
    d = dn;
    inv = invn;
  }
  if (__any_sync(0xffffffffu, bad)) return true;
  __syncwarp();  // ct and dinv visible to the whole warp
  double sacc[RR];  // sacc[i] = partial sum of row k - i
#pragma unroll
  for (int i = 0; i < RR; ++i) sacc[i] = 0.0;
  xf = 0.0;
#pragma unroll 1
  for (int k = RR - 1; k >= 0; --k) {
    const double xk = ((k == c ? 1.0 : 0.0) - sacc[0]) * dinv[k];
    put(k, xk);
    if (c < r) xf = fma(xk, xk, xf);
    double cv[RR];  // cv[i - 1] = R[k - i][k]
    const double2* cp = reinterpret_cast<const double2*>(sc.ct + k * LC + 2);
#pragma unroll
    for (int i = 0; i < RR / 2; ++i) {
      const double2 t = cp[i];
      cv[2 * i] = t.x;
      cv[2 * i + 1] = t.y;
    }
#pragma unroll
    for (int i = 1; i < RR; ++i) sacc[i - 1] = fma(cv[i - 1], xk, sacc[i]);
    sacc[RR - 1] = 0.0;
  }
  return false;
}

// r <= 32 fast path: the partial Grams are folded by the whole CTA, then one warp factors
// and inverts (warp_chol_inv). Same pivot test / flags / need2 as k_chol.
template <int RR>
__global__ void __launch_bounds__(256) k_chol32(const DevMat* __restrict__ mats,
                                                const int* __restrict__ part0,
                                                const int* __restrict__ nparts, int rr,
                                                const double* __restrict__ partial,
                                                double* __restrict__ rinv,
                                                int* __restrict__ flags,
                                                int* __restrict__ need2,
                                                const int* __restrict__ only) {
  __shared__ double G[RR][RR + 1];
  __shared__ double dinv[RR];
  __shared__ __align__(16) CholScratch<RR> scr;
  const int e = blockIdx.x;
  if (only && !only[e]) {
    if (threadIdx.x == 0) {
      flags[e] = 0;
      if (need2) need2[e] = 0;
    }
    return;
  }
  const DevMat m = mats[e];
  const int r = m.r;
  const double* src = partial + (int64_t)part0[e] * rr * rr;
  const int np = nparts[e];
  // fold; columns >= r are padded with the identity so the factorisation below runs all RR
  // (8 / 16 / 32, the rank rounded up) steps without data-dependent branches. The kernel
  // lasts as long as its slowest entry — the one with the most row-split partials (~100 for
  // the 50272-row embedding) — so every thread keeps kU elements x 8 partials of loads in
  // flight per step (unconditional loads at clamped addresses, masked in the fma).
  constexpr int kU = (RR * RR + 255) / 256;
  {
    const int64_t st = (int64_t)rr * rr;
    int off[kU];
    double msk[kU], acc[kU][2];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int idx = threadIdx.x + 256 * u;
      const int j = idx / RR, k = idx % RR;
      const bool live = idx < RR * RR && j < r && k < r && k >= j;
      off[u] = live ? j * rr + k : 0;
      msk[u] = live ? 1.0 : 0.0;
      acc[u][0] = acc[u][1] = 0.0;
    }
    int p = 0;
    for (; p + 8 <= np; p += 8) {
      double v[kU][8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u][q] = __ldg(src + (p + q) * st + off[u]);
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[u][q & 1] = fma(msk[u], v[u][q], acc[u][q & 1]);
    }
    for (; p < np; ++p)
#pragma unroll
      for (int u = 0; u < kU; ++u) acc[u][0] = fma(msk[u], __ldg(src + p * st + off[u]), acc[u][0]);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int idx = threadIdx.x + 256 * u;
      const int j = idx / RR, k = idx % RR;
      if (idx < RR * RR) G[j][k] = (j == k && j >= r) ? 1.0 : acc[u][0] + acc[u][1];
    }
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int c = threadIdx.x;  // lanes >= RR idle along (their columns stay zero)
  const double mx = warp_diag_max(&G[0][0], RR + 1, r);
  const double tol = 1e-7 * fmax(1.0, sqrt(mx));
  const double thr = (10.0 * tol) * (10.0 * tol);
  double rf = 0.0, xf = 0.0;
  double* X = rinv + (int64_t)e * rr * rr;
  const int flag = warp_chol_inv<RR>(&G[0][0], RR + 1, r, thr, dinv, scr,
                                     [&](int k, double v) {
                                       if (k < r && c < r) X[k * rr + c] = v;
                                     },
                                     rf, xf)
                       ? 1
                       : 0;
  if (c == 0) flags[e] = flag;
  if (flag) {
    if (need2 && c == 0) need2[e] = 0;
    return;
  }
  if (need2) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      xf += __shfl_xor_sync(0xffffffffu, xf, o);
      rf += __shfl_xor_sync(0xffffffffu, rf, o);
    }
    if (c == 0) need2[e] = (sqrt(xf) * sqrt(rf) > 2e3) ? 1 : 0;
  }
}

// 32 < r <= 128, blocked (RR = 32 NB, the rank padded with the identity): the whole
// factorisation in shared memory, 32-wide panels. Per panel p: one warp factors and inverts
// the diagonal block (warp_chol_inv), the CTA forms the panel row R_pq = R_pp^-T W_pq and
// the trailing update W_qq' -= R_pq^T R_pq' on the fp64 tensor cores (DMMA m8n8k4); then
// R^-1 block row by block row from the bottom, X_ij = -R_ii^-1 sum_{k=i+1..j} R_ik X_kj
// (DMMA). The serial part is NB warp factorisations instead of r barrier-separated steps.
constexpr int kCholBlkThreads = 256;

__host__ __device__ constexpr size_t cholblk_smem(int NB) {
  return sizeof(double) * (static_cast<size_t>(32 * NB) * (32 * NB + 1) + 2 * NB * 32 * 33) +
         sizeof(CholScratch<32>);
}

// D (8x8 tile at row m0, col n0 of a 32-row block product) = sum over k < kn of A[m][k] B[k][n]
// for A, B given as element accessors; fragments of dmma_8x8x4.
template <typename FA, typename FB>
__device__ __forceinline__ void dmma_tile(double (&d)[2], int kn, FA fa, FB fb) {
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < kn; k += 4) dmma_8x8x4(d, fa(lane >> 2, k + (lane & 3)), fb(k + (lane & 3), lane >> 2));
}

// two independent tiles interleaved (two DMMA chains in flight per warp); `two` is
// warp-uniform
template <typename FA0, typename FB0, typename FA1, typename FB1>
__device__ __forceinline__ void dmma_tile2(double (&d0)[2], double (&d1)[2], int kn, bool two,
                                           FA0 fa0, FB0 fb0, FA1 fa1, FB1 fb1) {
  const int lane = threadIdx.x & 31, m = lane >> 2;
  for (int k = 0; k < kn; k += 4) {
    const int ka = k + (lane & 3);
    dmma_8x8x4(d0, fa0(m, ka), fb0(ka, m));
    if (two) dmma_8x8x4(d1, fa1(m, ka), fb1(ka, m));
  }
}

// warp 0's share of a panel: factor + invert the diagonal block, R_pp^-1 into Xo. (Kept out of
// line: inlined into the panel loop, the register arrays of warp_chol_inv were demoted to
// local memory.)
template <int LD, int XL>
__device__ __noinline__ double diag_block(const double* G, int r, double thr, double* dinv,
                                         CholScratch<32>& sc, double* Xo, int* flag) {
  const int lane = threadIdx.x & 31;
  double rfp = 0.0, xfp = 0.0;
  const bool bad = warp_chol_inv<32>(G, LD, r, thr, dinv, sc,
                                     [&](int k, double v) { Xo[k * XL + lane] = v; }, rfp, xfp);
  if (lane == 0) *flag = bad ? 1 : 0;
  return bad ? 0.0 : rfp;
}

template <int NB>
__global__ void __launch_bounds__(kCholBlkThreads, 1) k_cholblk(const DevMat* __restrict__ mats,
                                                             const int* __restrict__ part0,
                                                             const int* __restrict__ nparts,
                                                             int rr,
                                                             const double* __restrict__ partial,
                                                             double* __restrict__ rinv,
                                                             int* __restrict__ flags,
                                                             int* __restrict__ need2,
                                                             const int* __restrict__ only) {
  constexpr int RR = 32 * NB, LD = RR + 1, XL = 33;
  constexpr int NW = kCholBlkThreads / 32;
  extern __shared__ __align__(16) double cb_smem[];
  double* W = cb_smem;              // [RR][LD]: G, then R (upper), then R^-1 off the diagonal
  double* Xd = W + RR * LD;         // [NB][32][XL]: R_pp^-1
  double* Tb = Xd + NB * 32 * XL;   // [NB][32][XL]: block-row temporaries
  auto* scr = reinterpret_cast<CholScratch<32>*>(Tb + NB * 32 * XL);  // warp 0's scratch
  __shared__ double dinv[32];
  __shared__ double red[2][NW];
  __shared__ int s_flag;
  const int e = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (only && !only[e]) {
    if (tid == 0) {
      flags[e] = 0;
      if (need2) need2[e] = 0;
    }
    return;
  }
  const DevMat m = mats[e];
  const int r = m.r;
  const double* src = partial + (int64_t)part0[e] * rr * rr;
  const int np = nparts[e];
  const int64_t st = (int64_t)rr * rr;
  // fold: 16 elements per thread per pass, the partials outermost (16 independent loads in
  // flight per step); identity padding past r
  constexpr int kU = 16;
  for (int base = 0; base < RR * RR; base += kU * kCholBlkThreads) {
    double acc[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) acc[u] = 0.0;
    // element offsets (clamped to a valid address where the element is not folded) and
    // masks computed once: the loads are unconditional, so all kU of a step issue together
    int off[kU];
    double msk[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int idx = base + u * kCholBlkThreads + tid;
      const int j = idx / RR, k = idx % RR;
      const bool live = idx < RR * RR && j < r && k < r && k >= j;
      off[u] = live ? j * rr + k : 0;
      msk[u] = live ? 1.0 : 0.0;
    }
    for (int p = 0; p < np; ++p) {
      const double* sp = src + p * st;
#pragma unroll
      for (int u = 0; u < kU; ++u) acc[u] = fma(msk[u], __ldg(sp + off[u]), acc[u]);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int idx = base + u * kCholBlkThreads + tid;
      const int j = idx / RR, k = idx % RR;
      if (idx < RR * RR) W[j * LD + k] = (j == k && j >= r) ? 1.0 : acc[u];
    }
  }
  __syncthreads();
  const double mx = warp_diag_max(W, LD, r);
  const double tol = 1e-7 * fmax(1.0, sqrt(mx));
  const double thr = (10.0 * tol) * (10.0 * tol);
  double rf = 0.0;  // ||R||_F^2 (columns < r), lane-partial
#pragma unroll 1
  for (int p = 0; p < NB; ++p) {
    const int o = 32 * p;
    if (warp == 0) {
      const double rfp = diag_block<LD, XL>(W + o * LD + o, r - o, thr, dinv, *scr,
                                            Xd + p * 32 * XL, &s_flag);
      rf += rfp;
    }
    __syncthreads();
    if (s_flag) {
      if (tid == 0) {
        flags[e] = 1;
        if (need2) need2[e] = 0;
      }
      return;
    }
    if (p == NB - 1) break;
    const int q0 = o + 32, nq = RR - q0;  // trailing columns
    // panel row: R[o+i][q0+n] = sum_k Xd[p][k][i] W[o+k][q0+n]   (k <= i); its squares
    // (columns < r) join ||R||_F^2 here, before the inversion overwrites these blocks
    {
      constexpr int kSlots = 2 * (NB - 1);  // >= ceil(16 (NB - 1) / NW) tiles per warp
      const int ntn = nq / 8, ntiles = 4 * ntn;
      double dres[kSlots][2];
#pragma unroll
      for (int it = 0; it < kSlots; ++it) {
        const int t = warp + it * NW;
        dres[it][0] = dres[it][1] = 0.0;
        if (t < ntiles) {
          const int ti = t / ntn, tj = t % ntn;
          const double* xa = Xd + p * 32 * XL;
          dmma_tile(dres[it], 8 * ti + 8,
                    [&](int mm, int k) { return xa[k * XL + 8 * ti + mm]; },
                    [&](int k, int n) { return W[(o + k) * LD + q0 + 8 * tj + n]; });
        }
      }
      __syncthreads();
#pragma unroll
      for (int it = 0; it < kSlots; ++it) {
        const int t = warp + it * NW;
        if (t < ntiles) {
          const int ti = t / ntn, tj = t % ntn;
          const int col = q0 + 8 * tj + 2 * (lane & 3);
          double* dst = W + (o + 8 * ti + (lane >> 2)) * LD + col;
          dst[0] = dres[it][0];
          dst[1] = dres[it][1];
          if (col < r) rf = fma(dres[it][0], dres[it][0], rf);
          if (col + 1 < r) rf = fma(dres[it][1], dres[it][1], rf);
        }
      }
      __syncthreads();
    }
    // trailing update (upper tile triangle): W[a][b] -= sum_k R[o+k][a] R[o+k][b]
    {
      const int mt = nq / 8, ntiles = mt * (mt + 1) / 2;
      auto unrank = [&](int t, int& ti, int& tj) {
        int rem = t;
        ti = 0;
        while (rem >= mt - ti) {
          rem -= mt - ti;
          ++ti;
        }
        tj = ti + rem;
      };
      for (int t = warp; t < ntiles; t += 2 * NW) {
        const int t2 = t + NW;
        const bool two = t2 < ntiles;
        int ti, tj, ti2 = 0, tj2 = 0;
        unrank(t, ti, tj);
        if (two) unrank(t2, ti2, tj2);
        double d[2] = {0.0, 0.0}, d2[2] = {0.0, 0.0};
        dmma_tile2(d, d2, 32, two,
                   [&](int mm, int k) { return W[(o + k) * LD + q0 + 8 * ti + mm]; },
                   [&](int k, int n) { return W[(o + k) * LD + q0 + 8 * tj + n]; },
                   [&](int mm, int k) { return W[(o + k) * LD + q0 + 8 * ti2 + mm]; },
                   [&](int k, int n) { return W[(o + k) * LD + q0 + 8 * tj2 + n]; });
        double* dst = W + (q0 + 8 * ti + (lane >> 2)) * LD + q0 + 8 * tj + 2 * (lane & 3);
        dst[0] -= d[0];
        dst[1] -= d[1];
        if (two) {
          double* dst2 = W + (q0 + 8 * ti2 + (lane >> 2)) * LD + q0 + 8 * tj2 + 2 * (lane & 3);
          dst2[0] -= d2[0];
          dst2[1] -= d2[1];
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0) flags[e] = 0;
  // R^-1 off the diagonal, block rows from the bottom; X_kj (k > i) already sits in W
#pragma unroll 1
  for (int i = NB - 2; i >= 0; --i) {
    const int nj = NB - 1 - i;  // blocks j = i+1 .. NB-1
    // T_j = sum_{k=i+1..j} R_ik X_kj
    for (int t = warp; t < nj * 16; t += NW) {
      const int jb = i + 1 + t / 16, ti = (t % 16) / 4, tj = t % 4;
      double d[2] = {0.0, 0.0};
      for (int kb = i + 1; kb <= jb; ++kb) {
        const double* xb = kb == jb ? Xd + jb * 32 * XL : nullptr;
        dmma_tile(d, 32,
                  [&](int mm, int k) { return W[(32 * i + 8 * ti + mm) * LD + 32 * kb + k]; },
                  [&](int k, int n) {
                    return xb ? xb[k * XL + 8 * tj + n] : W[(32 * kb + k) * LD + 32 * jb + 8 * tj + n];
                  });
      }
      double* dst = Tb + (jb * 32 + 8 * ti + (lane >> 2)) * XL + 8 * tj + 2 * (lane & 3);
      dst[0] = d[0];
      dst[1] = d[1];
    }
    __syncthreads();
    // X_ij = -R_ii^-1 T_j  (R_ii^-1 upper: k >= row)
    const double* xa = Xd + i * 32 * XL;
    for (int t = warp; t < nj * 16; t += 2 * NW) {
      const int t2 = t + NW;
      const bool two = t2 < nj * 16;
      const int jb = i + 1 + t / 16, ti = (t % 16) / 4, tj = t % 4;
      const int jb2 = two ? i + 1 + t2 / 16 : jb, ti2 = (t2 % 16) / 4, tj2 = t2 % 4;
      const double* tb = Tb + jb * 32 * XL;
      const double* tb2 = Tb + jb2 * 32 * XL;
      double d[2] = {0.0, 0.0}, d2[2] = {0.0, 0.0};
      dmma_tile2(d, d2, 32, two,
                 [&](int mm, int k) { return xa[(8 * ti + mm) * XL + k]; },
                 [&](int k, int n) { return tb[k * XL + 8 * tj + n]; },
                 [&](int mm, int k) { return xa[(8 * ti2 + mm) * XL + k]; },
                 [&](int k, int n) { return tb2[k * XL + 8 * tj2 + n]; });
      double* dst = W + (32 * i + 8 * ti + (lane >> 2)) * LD + 32 * jb + 8 * tj + 2 * (lane & 3);
      dst[0] = -d[0];
      dst[1] = -d[1];
      if (two) {
        double* dst2 = W + (32 * i + 8 * ti2 + (lane >> 2)) * LD + 32 * jb2 + 8 * tj2 + 2 * (lane & 3);
        dst2[0] = -d2[0];
        dst2[1] = -d2[1];
      }
    }
    __syncthreads();
  }
  double xf = 0.0;
  double* X = rinv + (int64_t)e * rr * rr;
  for (int i = warp; i < r; i += NW)  // row i, lanes over columns (no runtime divisions)
    for (int k = lane; k < r; k += 32) {
      double v = 0.0;
      if (k >= i) v = (i >> 5) == (k >> 5) ? Xd[((i >> 5) * 32 + (i & 31)) * XL + (k & 31)] : W[i * LD + k];
      xf = fma(v, v, xf);
      X[i * rr + k] = v;
    }
  if (need2) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      xf += __shfl_xor_sync(0xffffffffu, xf, o);
      rf += __shfl_xor_sync(0xffffffffu, rf, o);
    }
    if (lane == 0) {
      red[0][warp] = xf;
      red[1][warp] = rf;
    }
    __syncthreads();
    if (tid == 0) {
      double xs = 0.0, rs = 0.0;
      for (int w = 0; w < NW; ++w) {
        xs += red[0][w];
        rs += red[1][w];
      }
      need2[e] = (sqrt(xs) * sqrt(rs) > 2e3) ? 1 : 0;
    }
  }
}

// ------------------------------------------------------------------ apply: Y <- Y R^-1
// One CTA per 128-row tile of a factor, all columns: the tile is staged in shared memory
// first, so the update is in place. fp64 accumulation, R^-1 upper triangular.
__global__ void __launch_bounds__(128) k_apply(const DevMat* __restrict__ mats,
                                               const int4* __restrict__ jobs, int rr,
                                               const double* __restrict__ rinv,
                                               const int* __restrict__ skip,
                                               const int* __restrict__ only,
                                               float* __restrict__ buf) {
  extern __shared__ __align__(16) unsigned char ap_smem[];
  const int4 jb = jobs[blockIdx.x];
  if (skip[jb.x] || (only && !only[jb.x])) return;
  const DevMat m = mats[jb.x];
  const int r = m.r;
  double* Rs = reinterpret_cast<double*>(ap_smem);  // [32][33]
  float* Ys = reinterpret_cast<float*>(Rs + 32 * 33);  // [r][129]
  const int64_t row = jb.y + threadIdx.x;
  const bool live = row < m.n;
  float* Y = buf + m.off;
  const double* X = rinv + (int64_t)jb.x * rr * rr;
  for (int idx = threadIdx.x; idx < r * 128; idx += 128) {
    const int c = idx / 128, i = idx % 128;
    Ys[c * 129 + i] = (jb.y + i < m.n) ? Y[(int64_t)c * m.ld + jb.y + i] : 0.f;
  }
  __syncthreads();
  for (int cb = 0; cb * 32 < r; ++cb) {
    double acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0;
    for (int kb = 0; kb <= cb; ++kb) {
      __syncthreads();
      for (int idx = threadIdx.x; idx < 32 * 32; idx += 128) {
        const int k = kb * 32 + idx / 32, j = cb * 32 + idx % 32;
        Rs[(idx / 32) * 33 + idx % 32] = (k < r && j < r) ? X[k * rr + j] : 0.0;
      }
      __syncthreads();
      const int kmax = min(32, r - kb * 32);
      for (int k = 0; k < kmax; ++k) {
        const double y = (double)Ys[(kb * 32 + k) * 129 + threadIdx.x];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = fma(y, Rs[k * 33 + j], acc[j]);
      }
    }
    if (live) {
      const int jmax = min(32, r - cb * 32);
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < jmax) Y[(int64_t)(cb * 32 + j) * m.ld + row] = (float)acc[j];
    }
  }
}

// r <= 16: SIMT fp64, lane = row. One CTA per 128-row job: the job's rows load their r
// columns (coalesced: 128 B per column per warp), out[j] = sum_{k <= j} y[k] X[k][j] with X
// broadcast from shared memory (16-B loads), each output column stored coalesced. At these
// ranks the DMMA tile (fixed 32-wide staging, 2 of 4 column blocks live) was half idle:
// tools/micro/apply_micro.cu on the OPT-1.3B P side at r = 16, 45 us (DMMA) vs 23 us.
template <int RR>
__global__ void __launch_bounds__(128) k_apply_simt(const DevMat* __restrict__ mats,
                                                    const int4* __restrict__ jobs, int rr,
                                                    const double* __restrict__ rinv,
                                                    const int* __restrict__ skip,
                                                    const int* __restrict__ only,
                                                    float* __restrict__ buf) {
  __shared__ __align__(16) double Xs[RR * RR];  // [k][j], upper, zeros elsewhere
  const int4 jb = jobs[blockIdx.x];
  if (skip[jb.x] || (only && !only[jb.x])) return;
  const DevMat m = mats[jb.x];
  const int r = m.r;
  const double* X = rinv + (int64_t)jb.x * rr * rr;
  for (int idx = threadIdx.x; idx < RR * RR; idx += 128) {
    const int k = idx / RR, c = idx % RR;
    Xs[idx] = (k < r && c < r && k <= c) ? X[k * rr + c] : 0.0;
  }
  const int64_t row = jb.y + threadIdx.x;
  const bool live = row < m.n;
  float* Y = buf + m.off;
  float v[RR];
#pragma unroll
  for (int k = 0; k < RR; ++k) v[k] = (k < r && live) ? Y[(int64_t)k * m.ld + row] : 0.f;
  __syncthreads();
  double o[RR];
#pragma unroll
  for (int j = 0; j < RR; ++j) o[j] = 0.0;
#pragma unroll
  for (int k = 0; k < RR; ++k) {
    const double y = (double)v[k];
    const double2* xr = reinterpret_cast<const double2*>(Xs + k * RR);
#pragma unroll
    for (int j2 = 0; j2 < RR / 2; ++j2) {
      if (2 * j2 + 1 < k) continue;  // X[k][j] = 0 for j < k
      const double2 x = xr[j2];
      o[2 * j2] = fma(y, x.x, o[2 * j2]);
      o[2 * j2 + 1] = fma(y, x.y, o[2 * j2 + 1]);
    }
  }
  if (live) {
#pragma unroll
    for (int j = 0; j < RR; ++j)
      if (j < r) Y[(int64_t)j * m.ld + row] = (float)o[j];
  }
}

// r <= 32 fast path on DMMA: Y <- Y R^-1 for one 128-row tile. The tile (fp64, [row][k])
// and R^-1 (upper, zero-padded) are staged in shared memory; warp w owns rows
// [32 w, 32 w + 32) = four 8-row blocks, and column block cj only needs the k steps
// k < 8 (cj + 1) (triangular).
constexpr int kAdLdY = 36;  // [row][k] stride: conflict-free A fragments
constexpr int kAdLdR = 40;  // [k][col] stride: conflict-free B fragments

__global__ void __launch_bounds__(128) k_apply_dmma(const DevMat* __restrict__ mats,
                                                    const int4* __restrict__ jobs, int njobs,
                                                    int per_cta, int rr,
                                                    const double* __restrict__ rinv,
                                                    const int* __restrict__ skip,
                                                    const int* __restrict__ only,
                                                    float* __restrict__ buf) {
  // A run of consecutive 128-row tiles per CTA: the next tile's rows are loaded into
  // registers while the current one is multiplied; R^-1 is restaged only when the tile
  // run crosses into another factor.
  __shared__ __align__(16) double Ys[128 * kAdLdY];
  __shared__ double Rs[32 * kAdLdR];
  const int j0 = blockIdx.x * per_cta, j1 = min(njobs, j0 + per_cta);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  auto live_job = [&](int j) {
    const int e = jobs[j].x;
    return !skip[e] && !(only && !only[e]);
  };
  float v[32];
  auto fetch = [&](int j) {
    const int4 jb = jobs[j];
    const DevMat& m = mats[jb.x];
    const int64_t row = jb.y + threadIdx.x;
    const bool live = row < m.n;
    const float* Y = buf + m.off;
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = (k < m.r && live) ? Y[(int64_t)k * m.ld + row] : 0.f;
  };
  int cur = -1;
  int j = j0;
  while (j < j1 && !live_job(j)) ++j;
  if (j < j1) fetch(j);
  while (j < j1) {
    const int4 jb = jobs[j];
    const DevMat m = mats[jb.x];
    const int r = m.r, nb = (r + 7) / 8;
    __syncthreads();  // previous tile's fragments consumed
    if (jb.x != cur) {
      const double* X = rinv + (int64_t)jb.x * rr * rr;
      for (int idx = threadIdx.x; idx < 32 * 32; idx += 128) {
        const int k = idx / 32, c = idx % 32;
        Rs[k * kAdLdR + c] = (k < r && c < r && k <= c) ? X[k * rr + c] : 0.0;
      }
      cur = jb.x;
    }
    {
      double* dst = Ys + threadIdx.x * kAdLdY;
#pragma unroll
      for (int k = 0; k < 32; k += 2) *reinterpret_cast<double2*>(dst + k) = make_double2(v[k], v[k + 1]);
    }
    __syncthreads();
    int jn = j + 1;
    while (jn < j1 && !live_job(jn)) ++jn;
    if (jn < j1) fetch(jn);
    float* Y = buf + m.off;
#pragma unroll
    for (int rb = 0; rb < 4; ++rb) {
      const int rl = warp * 32 + rb * 8;  // first tile row of this 8-row block
      const double* pa = Ys + (rl + lane / 4) * kAdLdY + lane % 4;
      // the four column blocks as independent DMMA chains (block cj needs k < 8 (cj + 1))
      double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      const double* pb = Rs + (lane % 4) * kAdLdR + lane / 4;
#pragma unroll
      for (int k = 0; k < 32; k += 4) {
        const double a = pa[k];
#pragma unroll
        for (int cj = 0; cj < 4; ++cj)
          if (cj < nb && k < 8 * (cj + 1)) dmma_8x8x4(acc[cj], a, pb[k * kAdLdR + cj * 8]);
      }
      const int64_t row = jb.y + rl + lane / 4;
      if (row < m.n) {
#pragma unroll
        for (int cj = 0; cj < 4; ++cj)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int col = cj * 8 + 2 * (lane % 4) + q;
            if (cj < nb && col < r) Y[(int64_t)col * m.ld + row] = (float)acc[cj][q];
          }
      }
    }
    j = jn;
  }
}

// 32 < r <= 128 on DMMA: Y <- Y R^-1 for one 128-row job in two 64-row halves. R^-1 (upper,
// zero-padded) is staged once per factor in shared memory; warp w owns the 8-row block w of
// the half and every 8-column block of the output (NB independent accumulator pairs), and
// column block cj only takes the k steps k < 8 (cj + 1) (triangular).
template <int NB>
__global__ void __launch_bounds__(256) k_apply_dmma_big(const DevMat* __restrict__ mats,
                                                        const int4* __restrict__ jobs, int njobs,
                                                        int per_cta, int rr,
                                                        const double* __restrict__ rinv,
                                                        const int* __restrict__ skip,
                                                        const int* __restrict__ only,
                                                        float* __restrict__ buf) {
  constexpr int C = NB * 8;       // padded columns
  constexpr int LY = C + 4;       // [row][k] stride
  constexpr int LR = C + 8;       // [k][col] stride
  extern __shared__ __align__(16) double ad_smem[];
  double* Ys = ad_smem;           // [64][LY]
  double* Rs = Ys + 64 * LY;      // [C][LR]
  const int j0 = blockIdx.x * per_cta, j1 = min(njobs, j0 + per_cta);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int cur = -1;
  for (int j = j0; j < j1; ++j) {
    const int4 jb = jobs[j];
    const int e = jb.x;
    if (skip[e] || (only && !only[e])) continue;
    const DevMat m = mats[e];
    const int r = m.r, nb = (r + 7) / 8;
    float* Y = buf + m.off;
    if (e != cur) {
      __syncthreads();
      const double* X = rinv + (int64_t)e * rr * rr;
      for (int idx = threadIdx.x; idx < C * C; idx += 256) {
        const int k = idx / C, c = idx % C;
        Rs[k * LR + c] = (k < r && c < r && k <= c) ? X[k * rr + c] : 0.0;
      }
      cur = e;
    }
    for (int h = 0; h < 2; ++h) {
      const int64_t row0 = jb.y + 64 * h;
      __syncthreads();  // Rs staged / the previous half's Ys consumed
      for (int idx = threadIdx.x; idx < 64 * C; idx += 256) {
        const int k = idx / 64, rl = idx % 64;  // coalesced over rows of a column
        const int64_t row = row0 + rl;
        Ys[rl * LY + k] = (k < r && row < m.n) ? (double)Y[(int64_t)k * m.ld + row] : 0.0;
      }
      __syncthreads();
      double acc[NB][2];
#pragma unroll
      for (int cj = 0; cj < NB; ++cj) acc[cj][0] = acc[cj][1] = 0.0;
      const double* pa = Ys + (warp * 8 + lane / 4) * LY + lane % 4;
      const double* pb = Rs + (lane % 4) * LR + lane / 4;
      for (int k = 0; k < 8 * nb; k += 4) {
        const double a = pa[k];
#pragma unroll
        for (int cj = 0; cj < NB; ++cj)
          if (cj < nb && k < 8 * (cj + 1)) dmma_8x8x4(acc[cj], a, pb[k * LR + cj * 8]);
      }
      __syncthreads();  // every warp read its Ys rows before the in-place stores below
      const int64_t row = row0 + warp * 8 + lane / 4;
      if (row < m.n) {
#pragma unroll
        for (int cj = 0; cj < NB; ++cj)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int col = cj * 8 + 2 * (lane % 4) + q;
            if (cj < nb && col < r) Y[(int64_t)col * m.ld + row] = (float)acc[cj][q];
          }
      }
    }
  }
}

// ------------------------------------------------------------------ exact MGS2 fallback
__global__ void __launch_bounds__(1024) k_mgs_fallback(const DevMat* __restrict__ mats,
                                                       const int* __restrict__ flags,
                                                       float* __restrict__ buf,
                                                       double* __restrict__ scratch) {
  __shared__ double red[32];
  const int e = blockIdx.x;
  if (!flags[e]) return;
  const DevMat m = mats[e];
  const int64_t n = m.n;
  const int r = m.r;
  float* Yf = buf + m.off;
  double* Yd = scratch + m.off;  // same indexing as the float buffer
  double big = 0.0;
  for (int j = 0; j < r; ++j) {
    double ss = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const double v = (double)Yf[j * m.ld + i];
      Yd[j * m.ld + i] = v;
      ss += v * v;
    }
    big = fmax(big, sqrt(block_sum(ss, red)));
  }
  const double tol = 1e-7 * fmax(1.0, big);
  for (int j = 0; j < r; ++j) {
    double* cj = Yd + (int64_t)j * m.ld;
    for (int attempt = 0; attempt < 1000; ++attempt) {
      for (int pass = 0; pass < 2; ++pass)
        for (int p = 0; p < j; ++p) {
          const double* cp = Yd + (int64_t)p * m.ld;
          double d = 0.0;
          for (int64_t i = threadIdx.x; i < n; i += blockDim.x) d += cj[i] * cp[i];
          const double dot = block_sum(d, red);
          for (int64_t i = threadIdx.x; i < n; i += blockDim.x) cj[i] -= dot * cp[i];
          __syncthreads();
        }
      double ss = 0.0;
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) ss += cj[i] * cj[i];
      const double nrm = sqrt(block_sum(ss, red));
      if (nrm > tol) {
        const double inv = 1.0 / nrm;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) cj[i] *= inv;
        __syncthreads();
        break;
      }
      const uint64_t st = stream_init(0x5eedc01ull, stream_key4((uint64_t)n, (uint64_t)r,
                                                                 (uint64_t)j, (uint64_t)attempt));
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        cj[i] = (double)__fadd_rn(-1.0f, __fmul_rn(2.0f, unit_f(draw_at(st, i + 1))));
      __syncthreads();
    }
  }
  for (int j = 0; j < r; ++j)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) Yf[j * m.ld + i] = (float)Yd[j * m.ld + i];
}

// ------------------------------------------------------------------ driver
static size_t apply_smem(int rmax) { return 32 * 33 * sizeof(double) + sizeof(float) * rmax * 129; }

// k_apply_dmma_big measured slower than the SIMT k_apply on the Llama-7B layer (r = 64: 212
// vs 165 us, r = 128: 492 vs 408 us per call); kept for experiments (DLX_APPLY_DMMA=1)
static bool apply_dmma_big_enabled() {
  static const bool on = [] {
    const char* e = getenv("DLX_APPLY_DMMA");
    return e && e[0] == '1';
  }();
  return on;
}

static void launch_apply(const GramJob& J, int rr, const double* rinv, const int* skip,
                         const int* only, float* buf, size_t asm_, cudaStream_t s) {
  if (rr <= 16) {
    const int nj = static_cast<int>(J.apply.size());
    if (rr <= 8)
      k_apply_simt<8><<<nj, 128, 0, s>>>(J.d_mats, J.d_apply, rr, rinv, skip, only, buf);
    else
      k_apply_simt<16><<<nj, 128, 0, s>>>(J.d_mats, J.d_apply, rr, rinv, skip, only, buf);
  } else if (rr <= 32) {
    const int nj = static_cast<int>(J.apply.size());
    const int per = std::max(1, (nj + 4 * 148 - 1) / (4 * 148));
    k_apply_dmma<<<(nj + per - 1) / per, 128, 0, s>>>(J.d_mats, J.d_apply, nj, per, rr, rinv, skip,
                                                      only, buf);
  }
  else if (rr <= 128 && apply_dmma_big_enabled()) {
    const int nj = static_cast<int>(J.apply.size());
    const int per = std::max(1, (nj + 148 - 1) / 148);
    if (rr <= 64) {
      const int sm = static_cast<int>(sizeof(double) * (64 * 68 + 64 * 72));
      smem_optin(reinterpret_cast<const void*>(k_apply_dmma_big<8>), sm);
      k_apply_dmma_big<8><<<(nj + per - 1) / per, 256, sm, s>>>(J.d_mats, J.d_apply, nj, per, rr,
                                                               rinv, skip, only, buf);
    } else {
      const int sm = static_cast<int>(sizeof(double) * (64 * 132 + 128 * 136));
      smem_optin(reinterpret_cast<const void*>(k_apply_dmma_big<16>), sm);
      k_apply_dmma_big<16><<<(nj + per - 1) / per, 256, sm, s>>>(J.d_mats, J.d_apply, nj, per, rr,
                                                                rinv, skip, only, buf);
    }
  } else {
    k_apply<<<J.apply.size(), 128, asm_, s>>>(J.d_mats, J.d_apply, rr, rinv, skip, only, buf);
  }
  DLX_LAUNCHED();
}

// dlx_set_option("cholqr_blocked", 0) selects the unblocked shared-memory k_chol128 for
// 32 < r <= 128 (A/B measurements and cross-checks)
bool& option_cholblk() {
  static bool on = true;
  return on;
}

static void launch_chol(const GramJob& J, int rr, const double* partial, double* work,
                        double* rinv, int* flags, int* need2, const int* only, size_t csm,
                        cudaStream_t s) {
  const int ne = static_cast<int>(J.mats.size());
  if (rr <= 32) {
    // the fixed-size factorisation shrinks with the rank (the adaptive schedule drives r_t
    // to a few columns): 8 / 16 / 32 steps
    if (rr <= 8)
      k_chol32<8><<<ne, 256, 0, s>>>(J.d_mats, J.d_part0, J.d_nparts, rr, partial, rinv, flags,
                                     need2, only);
    else if (rr <= 16)
      k_chol32<16><<<ne, 256, 0, s>>>(J.d_mats, J.d_part0, J.d_nparts, rr, partial, rinv, flags,
                                      need2, only);
    else
      k_chol32<32><<<ne, 256, 0, s>>>(J.d_mats, J.d_part0, J.d_nparts, rr, partial, rinv, flags,
                                      need2, only);
  } else if (rr <= 128 && option_cholblk()) {
    auto go = [&](auto kern, int nb) {
      const int smem = static_cast<int>(cholblk_smem(nb));
      smem_optin(reinterpret_cast<const void*>(kern), smem);
      kern<<<ne, kCholBlkThreads, smem, s>>>(J.d_mats, J.d_part0, J.d_nparts, rr, partial, rinv,
                                             flags, need2, only);
    };
    if (rr <= 64)
      go(k_cholblk<2>, 2);
    else if (rr <= 96)
      go(k_cholblk<3>, 3);
    else
      go(k_cholblk<4>, 4);
  } else if (rr <= 128) {
    const int smem = static_cast<int>(sizeof(double) * rr * (rr + 1));
    smem_optin(reinterpret_cast<const void*>(k_chol128), smem);
    k_chol128<<<ne, kChol128Threads, smem, s>>>(J.d_mats, J.d_part0, J.d_nparts, rr, partial,
                                                rinv, flags, need2, only);
  } else
    k_chol<<<ne, 256, csm, s>>>(J.d_mats, J.d_part0, J.d_nparts, rr, partial, work, rinv, flags,
                                need2, only);
  DLX_LAUNCHED();
}

static void cholqr2(dlx_ctx* ctx, GramJob& J, float* buf, float* /*tmp*/, const std::string& tag,
                    int64_t buf_elems, cudaStream_t s) {
  const int rr = J.rmax;
  const size_t ne = J.mats.size();
  auto* partial = static_cast<double*>(ctx->scratch("gram_part", sizeof(double) * J.total_parts * rr * rr));
  auto* work = static_cast<double*>(ctx->scratch("chol_work", sizeof(double) * ne * rr * rr));
  auto* rinv = static_cast<double*>(ctx->scratch("chol_rinv", sizeof(double) * ne * rr * rr));
  auto* flags1 = static_cast<int*>(ctx->scratch("ortho_flags1" + tag, sizeof(int) * ne));
  auto* need2 = static_cast<int*>(ctx->scratch("ortho_need2" + tag, sizeof(int) * ne));
  auto* flags2 = static_cast<int*>(ctx->scratch("ortho_flags2" + tag, sizeof(int) * ne));
  smem_optin(reinterpret_cast<const void*>(k_apply), 160 * 1024);
  smem_optin(reinterpret_cast<const void*>(k_chol), 80 * 1024);
  const size_t csm = rr <= 64 ? 2 * sizeof(double) * rr * rr : 0;
  const size_t asm_ = apply_smem(rr);
  // pass 1 (every factor), in place
  launch_gram(J, buf, partial, s);
  launch_chol(J, rr, partial, work, rinv, flags1, need2, nullptr, csm, s);
  launch_apply(J, rr, rinv, flags1, nullptr, buf, asm_, s);
  // pass 2 only for factors whose conditioning needs it (need2), in place
  launch_gram(J, buf, partial, s, need2);
  launch_chol(J, rr, partial, work, rinv, flags2, nullptr, need2, csm, s);
  launch_apply(J, rr, rinv, flags2, need2, buf, asm_, s);
  // exact MGS2 for flagged entries (pass-1 flags: buf still holds their input)
  auto* dscr = static_cast<double*>(ctx->scratch("mgs_scratch", sizeof(double) * buf_elems));
  k_mgs_fallback<<<ne, 1024, 0, s>>>(J.d_mats, flags1, buf, dscr);
  DLX_LAUNCHED();
}

void orthonormalize_batched(dlx_ctx* ctx, const Plan& P, int side, float* buf, float* tmp,
                            cudaStream_t s) {
  HostProf hp_("orthonormalize_batched");
  if (P.mats[side].empty()) return;
  GramJob& J = job_for(P, side == 0 ? "P" : "Q", P.mats[side]);
  cholqr2(ctx, J, buf, tmp, side == 0 ? "P" : "Q", side == 0 ? P.pelems : P.qelems, s);
}

}  // namespace dlx
