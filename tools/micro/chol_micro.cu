// Microbenchmark: one warp factors + inverts a 32x32 SPD block (the serial core of
// k_chol32 / k_cholblk), 148 CTAs x 1 warp, variants timed with CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chol_micro chol_micro.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int RR = 32, LDG = RR + 1;

// V0: rolled, pivot row broadcast with shuffles; back substitution reads column k of R
__device__ void v0(double* G, double* dinv, double* X) {
  const int c = threadIdx.x & 31;
  double w[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) w[i] = (i <= c) ? G[i * LDG + c] : 0.0;
#pragma unroll 1
  for (int j = 0; j < RR; ++j) {
    const double d = __shfl_sync(0xffffffffu, w[0], j);
    const double inv = rsqrt(d);
    const double rj = c == j ? d * inv : w[0] * inv;
    if (c == j) dinv[j] = inv;
    G[j * LDG + c] = rj;
#pragma unroll
    for (int i = 1; i < RR; ++i) {
      const double rji = __shfl_sync(0xffffffffu, rj, (j + i) & 31);
      w[i - 1] = (j + i <= c) ? fma(-rji, rj, w[i]) : w[i];
    }
    w[RR - 1] = 0.0;
  }
  __syncwarp();
  double s[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) s[i] = 0.0;
#pragma unroll 1
  for (int k = RR - 1; k >= 0; --k) {
    const double xk = ((k == c ? 1.0 : 0.0) - s[0]) * dinv[k];
    X[k * RR + c] = xk;
#pragma unroll
    for (int i = 1; i < RR; ++i) {
      const int row = k - i < 0 ? 0 : k - i;
      s[i - 1] = fma(G[row * LDG + k], xk, s[i]);
    }
    s[RR - 1] = 0.0;
  }
}

// V1: rolled; pivot row j of R goes through shared memory (broadcast loads, no shuffles);
// R^T kept with 32 zeros in front of each row so the back substitution reads column k of R
// as one contiguous, clamp-free run (vector loads)
constexpr int LT = 2 * RR + 2;  // Rt row stride (doubles), 16-B aligned rows
__device__ void v1(double* G, double* dinv, double* X, double* Rrow, double* Rt) {
  const int c = threadIdx.x & 31;
  double w[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) w[i] = (i <= c) ? G[i * LDG + c] : 0.0;
  for (int i = c; i < RR * LT; i += 32) Rt[i] = 0.0;
#pragma unroll 1
  for (int j = 0; j < RR; ++j) {
    const double d = __shfl_sync(0xffffffffu, w[0], j);
    const double inv = rsqrt(d);
    const double rj = c == j ? d * inv : w[0] * inv;
    if (c == j) dinv[j] = inv;
    Rrow[(j & 1) * 64 + 32 + c] = rj;      // double-buffered row, 32 zeros in front
    Rt[c * LT + RR + j] = rj;               // R^T[c][j]
    __syncwarp();
    const double* rr = Rrow + (j & 1) * 64 + 32 + j;  // rr[i] = R[j][j + i]
#pragma unroll
    for (int i = 1; i < RR; ++i) {
      const double rji = (j + i < RR) ? rr[i] : 0.0;
      w[i - 1] = (j + i <= c) ? fma(-rji, rj, w[i]) : w[i];
    }
    w[RR - 1] = 0.0;
  }
  __syncwarp();
  double s[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) s[i] = 0.0;
#pragma unroll 1
  for (int k = RR - 1; k >= 0; --k) {
    const double xk = ((k == c ? 1.0 : 0.0) - s[0]) * dinv[k];
    X[k * RR + c] = xk;
    const double* col = Rt + k * LT + RR + k;  // col[-i] = R[k - i][k] (0 for k - i < 0)
#pragma unroll
    for (int i = 1; i < RR; ++i) s[i - 1] = fma(col[-i], xk, s[i]);
    s[RR - 1] = 0.0;
  }
}

// V2: fully unrolled, sqrt + divide, dot-product back substitution (round-1 k_chol32)
__device__ void v2(double* G, double* dinv, double* X) {
  const int c = threadIdx.x & 31;
  double w[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) w[i] = (i <= c) ? G[i * LDG + c] : 0.0;
#pragma unroll
  for (int j = 0; j < RR; ++j) {
    const double d = __shfl_sync(0xffffffffu, w[j], j);
    const double rjj = sqrt(d), inv = 1.0 / rjj;
    if (c == j) { w[j] = rjj; dinv[j] = inv; }
    if (c > j) w[j] *= inv;
#pragma unroll
    for (int i = j + 1; i < RR; ++i) {
      const double rji = __shfl_sync(0xffffffffu, w[j], i);
      if (i <= c) w[i] = fma(-rji, w[j], w[i]);
    }
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < RR; ++i) G[i * LDG + c] = (i <= c) ? w[i] : 0.0;
  __syncwarp();
  double x[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) x[i] = (i == c) ? dinv[c] : 0.0;
#pragma unroll
  for (int i = RR - 2; i >= 0; --i) {
    double sum = 0.0;
#pragma unroll
    for (int k = i + 1; k < RR; ++k) sum = fma(G[i * LDG + k], x[k], sum);
    if (i < c) x[i] = -sum * dinv[i];
  }
#pragma unroll
  for (int i = 0; i < RR; ++i) X[i * RR + c] = x[i];
}


// branch-free fp64 rsqrt: MUFU seed + three Newton steps (no special-case paths, so the
// scheduler can interleave it with independent work of the same basic block)
template <int NR = 3>
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double h = 0.5 * d;
#pragma unroll
  for (int i = 0; i < NR; ++i) y = y * fma(-h * y, y, 1.5);
  return y;
}

// V3: V1 with rsqrt_nr
__device__ void v3(double* G, double* dinv, double* X, double* Rrow, double* Rt) {
  const int c = threadIdx.x & 31;
  double w[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) w[i] = (i <= c) ? G[i * LDG + c] : 0.0;
  for (int i = c; i < RR * LT; i += 32) Rt[i] = 0.0;
#pragma unroll 1
  for (int j = 0; j < RR; ++j) {
    const double d = __shfl_sync(0xffffffffu, w[0], j);
    const double inv = rsqrt_nr(d);
    const double rj = c == j ? d * inv : w[0] * inv;
    if (c == j) dinv[j] = inv;
    Rrow[(j & 1) * 64 + 32 + c] = rj;
    Rt[c * LT + RR + j] = rj;
    __syncwarp();
    const double* rr = Rrow + (j & 1) * 64 + 32 + j;
#pragma unroll
    for (int i = 1; i < RR; ++i) {
      const double rji = (j + i < RR) ? rr[i] : 0.0;
      w[i - 1] = (j + i <= c) ? fma(-rji, rj, w[i]) : w[i];
    }
    w[RR - 1] = 0.0;
  }
  __syncwarp();
  double s[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) s[i] = 0.0;
#pragma unroll 1
  for (int k = RR - 1; k >= 0; --k) {
    const double xk = ((k == c ? 1.0 : 0.0) - s[0]) * dinv[k];
    X[k * RR + c] = xk;
    const double* col = Rt + k * LT + RR + k;
#pragma unroll
    for (int i = 1; i < RR; ++i) s[i - 1] = fma(col[-i], xk, s[i]);
    s[RR - 1] = 0.0;
  }
}

// V4: V3 + lookahead — the next pivot is updated first, shuffled and its rsqrt issued before
// the rest of the trailing update (same basic block: the chains overlap)
__device__ void v4(double* G, double* dinv, double* X, double* Rrow, double* Rt) {
  const int c = threadIdx.x & 31;
  double w[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) w[i] = (i <= c) ? G[i * LDG + c] : 0.0;
  for (int i = c; i < RR * LT; i += 32) Rt[i] = 0.0;
  double d = __shfl_sync(0xffffffffu, w[0], 0);
  double inv = rsqrt_nr(d);
#pragma unroll 1
  for (int j = 0; j < RR; ++j) {
    const double rj = c == j ? d * inv : w[0] * inv;
    if (c == j) dinv[j] = inv;
    Rrow[(j & 1) * 64 + 32 + c] = rj;
    Rt[c * LT + RR + j] = rj;
    __syncwarp();
    const double* rr = Rrow + (j & 1) * 64 + 32 + j;
    const double r1 = (j + 1 < RR) ? rr[1] : 0.0;
    w[0] = (j + 1 <= c) ? fma(-r1, rj, w[1]) : w[1];
    const double dn = __shfl_sync(0xffffffffu, w[0], (j + 1) & 31);
    const double invn = rsqrt_nr(dn);
#pragma unroll
    for (int i = 2; i < RR; ++i) {
      const double rji = (j + i < RR) ? rr[i] : 0.0;
      w[i - 1] = (j + i <= c) ? fma(-rji, rj, w[i]) : w[i];
    }
    w[RR - 1] = 0.0;
    d = dn;
    inv = invn;
  }
  __syncwarp();
  double s[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) s[i] = 0.0;
#pragma unroll 1
  for (int k = RR - 1; k >= 0; --k) {
    const double xk = ((k == c ? 1.0 : 0.0) - s[0]) * dinv[k];
    X[k * RR + c] = xk;
    const double* col = Rt + k * LT + RR + k;
#pragma unroll
    for (int i = 1; i < RR; ++i) s[i - 1] = fma(col[-i], xk, s[i]);
    s[RR - 1] = 0.0;
  }
}


// V5: V4 with unconditional loads (row buffer zero past the block) and unconditional
// trailing fmas (the strictly-lower entries they touch are never read)
__device__ void v5(double* G, double* dinv, double* X, double* Rrow, double* Rt) {
  const int c = threadIdx.x & 31;
  double w[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) w[i] = (i <= c) ? G[i * LDG + c] : 0.0;
  for (int i = c; i < RR * LT; i += 32) Rt[i] = 0.0;
  for (int i = c; i < 256; i += 32) Rrow[i] = 0.0;
  __syncwarp();
  double d = __shfl_sync(0xffffffffu, w[0], 0);
  double inv = rsqrt_nr(d);
#pragma unroll 1
  for (int j = 0; j < RR; ++j) {
    const double rj = c == j ? d * inv : w[0] * inv;
    if (c == j) dinv[j] = inv;
    Rrow[(j & 1) * 128 + 32 + c] = rj;
    Rt[c * LT + RR + j] = rj;
    __syncwarp();
    const double* rr = Rrow + (j & 1) * 128 + 32 + j;
    w[0] = fma(-rr[1], rj, w[1]);
    const double dn = __shfl_sync(0xffffffffu, w[0], (j + 1) & 31);
    const double invn = rsqrt_nr(dn);
#pragma unroll
    for (int i = 2; i < RR; ++i) w[i - 1] = fma(-rr[i], rj, w[i]);
    w[RR - 1] = 0.0;
    d = dn;
    inv = invn;
  }
  __syncwarp();
  double s[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) s[i] = 0.0;
#pragma unroll 1
  for (int k = RR - 1; k >= 0; --k) {
    const double xk = ((k == c ? 1.0 : 0.0) - s[0]) * dinv[k];
    X[k * RR + c] = xk;
    const double* col = Rt + k * LT + RR + k;
#pragma unroll
    for (int i = 1; i < RR; ++i) s[i - 1] = fma(col[-i], xk, s[i]);
    s[RR - 1] = 0.0;
  }
}


// V6: V5 with 16-B vector loads: the pivot row is written shifted by the step (lane c stores
// R[j][c] at 32 + c - j - 1, so R[j][j+1..j+31] starts on an aligned index), and column k of
// R is kept reversed per row of Ct (Ct[k][d + 1] = R[k - d][k]) so the back substitution reads
// it from an aligned index too
constexpr int LC = 2 * RR + 2;
template <int NR>
__device__ void v6(double* G, double* dinv, double* X, double* Rrow, double* Ct) {
  const int c = threadIdx.x & 31;
  double w[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) w[i] = (i <= c) ? G[i * LDG + c] : 0.0;
  for (int i = c; i < RR * LC; i += 32) Ct[i] = 0.0;
  __syncwarp();
  double d = __shfl_sync(0xffffffffu, w[0], 0);
  double inv = rsqrt_nr<NR>(d);
#pragma unroll 1
  for (int j = 0; j < RR; ++j) {
    const double rj = c == j ? d * inv : w[0] * inv;
    if (c == j) dinv[j] = inv;
    double* row = Rrow + (j & 1) * 128;
    row[32 + c - j - 1] = rj;                 // row[32 + i - 1] = R[j][j + i]
    if (c >= j) Ct[c * LC + (c - j) + 1] = rj;  // Ct[c][d + 1] = R[c - d][c]
    __syncwarp();
    const double2* rv = reinterpret_cast<const double2*>(row + 32);
    double rrv[RR];
#pragma unroll
    for (int i = 0; i < RR / 2; ++i) {
      const double2 t = rv[i];
      rrv[2 * i] = t.x;
      rrv[2 * i + 1] = t.y;
    }
    w[0] = fma(-rrv[0], rj, w[1]);
    const double dn = __shfl_sync(0xffffffffu, w[0], (j + 1) & 31);
    const double invn = rsqrt_nr<NR>(dn);
#pragma unroll
    for (int i = 2; i < RR; ++i) w[i - 1] = fma(-rrv[i - 1], rj, w[i]);
    w[RR - 1] = 0.0;
    d = dn;
    inv = invn;
  }
  __syncwarp();
  double s[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) s[i] = 0.0;
#pragma unroll 1
  for (int k = RR - 1; k >= 0; --k) {
    const double xk = ((k == c ? 1.0 : 0.0) - s[0]) * dinv[k];
    X[k * RR + c] = xk;
    const double2* cv = reinterpret_cast<const double2*>(Ct + k * LC + 2);  // d = 1, 2, ...
    double cc[RR];
#pragma unroll
    for (int i = 0; i < RR / 2; ++i) {
      const double2 t = cv[i];
      cc[2 * i] = t.x;
      cc[2 * i + 1] = t.y;
    }
#pragma unroll
    for (int i = 1; i < RR; ++i) s[i - 1] = fma(cc[i - 1], xk, s[i]);
    s[RR - 1] = 0.0;
  }
}

template <int V>
__global__ void __launch_bounds__(32) kern(const double* A, double* out, int reps) {
  __shared__ double G[RR * LDG];
  __shared__ double dinv[RR];
  __shared__ __align__(16) double Rrow[256];
  __shared__ __align__(16) double Rt[RR * LC];
  const int c = threadIdx.x;
  for (int rep = 0; rep < reps; ++rep) {
    for (int i = 0; i < RR; ++i) G[i * LDG + c] = A[i * RR + c];
    __syncwarp();
    double* X = out + (size_t)blockIdx.x * RR * RR;
    if (V == 0) v0(G, dinv, X);
    if (V == 1) v1(G, dinv, X, Rrow, Rt);
    if (V == 2) v2(G, dinv, X);
    if (V == 3) v3(G, dinv, X, Rrow, Rt);
    if (V == 4) v4(G, dinv, X, Rrow, Rt);
    if (V == 5) v5(G, dinv, X, Rrow, Rt);
    if (V == 6) v6<3>(G, dinv, X, Rrow, Rt);
    if (V == 7) v6<2>(G, dinv, X, Rrow, Rt);
    if (V == 8) v6<1>(G, dinv, X, Rrow, Rt);
    __syncwarp();
  }
}

int main() {
  std::vector<double> a(RR * RR), g(RR * RR);
  srand(1);
  for (auto& x : a) x = rand() / (double)RAND_MAX - 0.5;
  for (int i = 0; i < RR; ++i)
    for (int j = 0; j < RR; ++j) {
      double s = (i == j) ? 4.0 : 0.0;
      for (int k = 0; k < RR; ++k) s += a[k * RR + i] * a[k * RR + j];
      g[i * RR + j] = s;
    }
  double *dA, *dO;
  cudaMalloc(&dA, sizeof(double) * RR * RR);
  cudaMalloc(&dO, sizeof(double) * RR * RR * 148 * 9);
  cudaMemcpy(dA, g.data(), sizeof(double) * RR * RR, cudaMemcpyHostToDevice);
  std::vector<double> res[9];
  const int reps = 10;
  for (int v = 0; v < 9; ++v) {
    auto launch = [&] {
      if (v == 0) kern<0><<<148, 32>>>(dA, dO + v * RR * RR * 148, reps);
      if (v == 1) kern<1><<<148, 32>>>(dA, dO + v * RR * RR * 148, reps);
      if (v == 2) kern<2><<<148, 32>>>(dA, dO + v * RR * RR * 148, reps);
      if (v == 3) kern<3><<<148, 32>>>(dA, dO + v * RR * RR * 148, reps);
      if (v == 4) kern<4><<<148, 32>>>(dA, dO + v * RR * RR * 148, reps);
      if (v == 5) kern<5><<<148, 32>>>(dA, dO + v * RR * RR * 148, reps);
      if (v == 6) kern<6><<<148, 32>>>(dA, dO + v * RR * RR * 148, reps);
      if (v == 7) kern<7><<<148, 32>>>(dA, dO + v * RR * RR * 148, reps);
      if (v == 8) kern<8><<<148, 32>>>(dA, dO + v * RR * RR * 148, reps);
    };
    launch();
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    res[v].resize(RR * RR);
    cudaMemcpy(res[v].data(), dO + v * RR * RR * 148, sizeof(double) * RR * RR, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < RR * RR; ++i) err = fmax(err, fabs(res[v][i] - res[0][i]));
    printf("variant %d: %.2f us per factor+inverse (max |X - X_v0| = %.3g) %s\n", v,
           ms * 1000.0 / (10 * reps), err, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
