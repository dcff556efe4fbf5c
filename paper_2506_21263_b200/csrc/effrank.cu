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
#include "dlx_internal.cuh"

namespace dlx {

void gram_batched(dlx_ctx* ctx, const Plan& P, const std::string& key,
                  const std::vector<DevMat>& mats, const float* buf, double* out,
                  cudaStream_t s);

__device__ double er_block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

__global__ void __launch_bounds__(256) k_effrank(const DevT2* __restrict__ T, int D, int rr,
                                                 const double* __restrict__ GA,
                                                 const double* __restrict__ GB,
                                                 double* __restrict__ work, double tau,
                                                 int* __restrict__ per,
                                                 double* __restrict__ energy) {
  __shared__ double red[32];
  __shared__ double cs[1024], sn[1024];
  __shared__ int pp[1024], qq[1024];
  __shared__ int s_k;
  __shared__ double s_tot;
  const int e = blockIdx.x;
  const int K = D * T[e].r;
  const int n2 = K + (K & 1);
  const int64_t mat = (int64_t)rr * rr;
  const double* Ga = GA + e * mat;
  double* Lm = work + (3 * e + 0) * mat;  // L (lower), from G_B
  double* Tm = work + (3 * e + 1) * mat;  // G_A L
  double* M = work + (3 * e + 2) * mat;   // L^T G_A L  (n2 x n2, row stride rr)
  // 1. semidefinite Cholesky of G_B (lower), columns with vanishing pivot dropped
  for (int idx = threadIdx.x; idx < K * K; idx += blockDim.x)
    Lm[(idx / K) * rr + idx % K] = GB[e * mat + (idx / K) * rr + idx % K];
  __syncthreads();
  double dmax = 0.0;
  for (int j = 0; j < K; ++j) dmax = fmax(dmax, Lm[j * rr + j]);
  const double floor_piv = 1e-14 * dmax;
  for (int j = 0; j < K; ++j) {
    const double d = Lm[j * rr + j];
    const bool keep = d > floor_piv && d > 0.0;
    const double ljj = keep ? sqrt(d) : 0.0;
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < K; i += blockDim.x)
      Lm[i * rr + j] = keep ? Lm[i * rr + j] / ljj : 0.0;
    if (threadIdx.x == 0) Lm[j * rr + j] = ljj;
    __syncthreads();
    const int rem = K - j - 1;
    for (int idx = threadIdx.x; idx < rem * rem; idx += blockDim.x) {
      const int i = j + 1 + idx / rem, k = j + 1 + idx % rem;
      if (k > i) continue;
      Lm[i * rr + k] -= Lm[i * rr + j] * Lm[k * rr + j];
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < K * K; idx += blockDim.x) {  // zero the strict upper part
    const int i = idx / K, k = idx % K;
    if (k > i) Lm[i * rr + k] = 0.0;
  }
  __syncthreads();
  // 2. Tm = G_A L ; M = L^T Tm
  for (int idx = threadIdx.x; idx < K * K; idx += blockDim.x) {
    const int i = idx / K, j = idx % K;
    double s = 0.0;
    for (int k = j; k < K; ++k) s = fma(Ga[i * rr + k], Lm[k * rr + j], s);
    Tm[i * rr + j] = s;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n2 * n2; idx += blockDim.x) {
    const int i = idx / n2, j = idx % n2;
    double s = 0.0;
    if (i < K && j < K)
      for (int k = i; k < K; ++k) s = fma(Lm[k * rr + i], Tm[k * rr + j], s);
    M[i * rr + j] = s;
  }
  __syncthreads();
  // symmetrise (rounding) and 3. parallel cyclic Jacobi (round-robin pairing)
  for (int idx = threadIdx.x; idx < n2 * n2; idx += blockDim.x) {
    const int i = idx / n2, j = idx % n2;
    if (j > i) {
      const double v = 0.5 * (M[i * rr + j] + M[j * rr + i]);
      M[i * rr + j] = v;
      M[j * rr + i] = v;
    }
  }
  __syncthreads();
  const int half = n2 / 2;
  for (int sweep = 0; sweep < 40 && n2 > 1; ++sweep) {
    double off = 0.0, dg = 0.0;
    for (int idx = threadIdx.x; idx < n2 * n2; idx += blockDim.x) {
      const int i = idx / n2, j = idx % n2;
      const double v = M[i * rr + j];
      if (i == j) dg += v * v; else off += v * v;
    }
    off = er_block_sum(off, red);
    dg = er_block_sum(dg, red);
    if (off <= 1e-30 * dg || off == 0.0) break;
    for (int rd = 0; rd < n2 - 1; ++rd) {
      for (int i = threadIdx.x; i < half; i += blockDim.x) {
        int a = (rd + i) % (n2 - 1);
        int b = i == 0 ? n2 - 1 : (rd - i + n2 - 1) % (n2 - 1);
        const int p = min(a, b), q = max(a, b);
        const double apq = M[p * rr + q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0) {
          const double theta = (M[q * rr + q] - M[p * rr + p]) / (2.0 * apq);
          const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          c = 1.0 / sqrt(t * t + 1.0);
          s = t * c;
        }
        cs[i] = c;
        sn[i] = s;
        pp[i] = p;
        qq[i] = q;
      }
      __syncthreads();
      for (int idx = threadIdx.x; idx < half * n2; idx += blockDim.x) {  // rows
        const int i = idx / n2, k = idx % n2;
        const int p = pp[i], q = qq[i];
        const double c = cs[i], s = sn[i];
        const double ap = M[p * rr + k], aq = M[q * rr + k];
        M[p * rr + k] = c * ap - s * aq;
        M[q * rr + k] = s * ap + c * aq;
      }
      __syncthreads();
      for (int idx = threadIdx.x; idx < half * n2; idx += blockDim.x) {  // columns
        const int i = idx / n2, k = idx % n2;
        const int p = pp[i], q = qq[i];
        const double c = cs[i], s = sn[i];
        const double ap = M[k * rr + p], aq = M[k * rr + q];
        M[k * rr + p] = c * ap - s * aq;
        M[k * rr + q] = s * ap + c * aq;
      }
      __syncthreads();
    }
  }
  // 4. eigenvalues (clamped >= 0) sorted descending by rank counting; prefix energy
  double* ev = Tm;  // reuse: ev[rank] = value
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    const double v = fmax(M[i * rr + i], 0.0);
    int rank = 0;
    for (int j = 0; j < n2; ++j) {
      const double w = fmax(M[j * rr + j], 0.0);
      rank += (w > v) || (w == v && j < i);
    }
    ev[rank] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int i = 0; i < n2; ++i) tot += ev[i];
    int k = 1;
    if (tot > 0.0) {
      double pre = 0.0;
      for (int i = 0; i < n2; ++i) {
        pre += ev[i];
        k = i + 1;
        if (pre >= tau * tot) break;
      }
    }
    s_k = k;
    s_tot = tot / ((double)D * (double)D);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    per[e] = s_k;
    energy[e] = s_tot;
  }
}

void effective_rank_factors(dlx_ctx* ctx, const Plan& P, int D, const uint8_t* gathered,
                            double tau, int* d_per, double* d_energy, cudaStream_t s) {
  if (P.t2.empty()) return;
  float* phat = static_cast<float*>(ctx->scratch("er_phat", sizeof(float) * P.pelems * D));
  float* qhat = static_cast<float*>(ctx->scratch("er_qhat", sizeof(float) * P.qelems * D));
  dequant_factors(P, D, gathered, P.payload_bytes, phat, qhat, 0, s);
  std::vector<DevMat> A, B;
  int K = 0;
  for (size_t k = 0; k < P.t2.size(); ++k) {
    const DevT2& t = P.t2[k];
    A.push_back(DevMat{D * t.poff, t.a, t.lda, D * t.r, static_cast<int>(k)});
    B.push_back(DevMat{D * t.qoff, t.b, t.ldb, D * t.r, static_cast<int>(k)});
    K = std::max(K, D * t.r);
  }
  if (K > 2048) raise(DLX_ERR_VALIDATION, "effective_rank: D * rank above 2048 unsupported");
  const int64_t mat = static_cast<int64_t>(K) * K;
  const size_t ne = P.t2.size();
  auto* GA = static_cast<double*>(ctx->scratch("er_GA", sizeof(double) * mat * ne));
  auto* GB = static_cast<double*>(ctx->scratch("er_GB", sizeof(double) * mat * ne));
  auto* W = static_cast<double*>(ctx->scratch("er_W", sizeof(double) * mat * ne * 3));
  const std::string tag = std::to_string(D);
  gram_batched(ctx, P, "erA" + tag, A, phat, GA, s);
  gram_batched(ctx, P, "erB" + tag, B, qhat, GB, s);
  k_effrank<<<ne, 256, 0, s>>>(P.d_t2, D, K, GA, GB, W, tau, d_per, d_energy);
  DLX_LAUNCHED();
}

}  // namespace dlx
