// Microbenchmark: CholQR apply Y <- Y R^-1 (r <= 32) over the OPT-1.3B P-side factor set
// (146 column-major factors, 494690 rows), variants timed with CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o apply_micro apply_micro.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

struct DevMat { long long off, n, ld; int r, slot; };

__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

// ---- V0: the library's k_apply_dmma (round-2 state)
constexpr int kAdLdY = 36, kAdLdR = 40;
__global__ void __launch_bounds__(128) v0(const DevMat* mats, const int4* jobs, int njobs, int per_cta,
                                         int rr, const double* rinv, float* buf) {
  __shared__ __align__(16) double Ys[128 * kAdLdY];
  __shared__ double Rs[32 * kAdLdR];
  const int j0 = blockIdx.x * per_cta, j1 = min(njobs, j0 + per_cta);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float v[32];
  auto fetch = [&](int j) {
    const int4 jb = jobs[j];
    const DevMat& m = mats[jb.x];
    const long long row = jb.y + threadIdx.x;
    const bool live = row < m.n;
    const float* Y = buf + m.off;
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = (k < m.r && live) ? Y[(long long)k * m.ld + row] : 0.f;
  };
  int cur = -1;
  int j = j0;
  if (j < j1) fetch(j);
  while (j < j1) {
    const int4 jb = jobs[j];
    const DevMat m = mats[jb.x];
    const int r = m.r, nb = (r + 7) / 8;
    __syncthreads();
    if (jb.x != cur) {
      const double* X = rinv + (long long)jb.x * rr * rr;
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
    if (jn < j1) fetch(jn);
    float* Y = buf + m.off;
#pragma unroll
    for (int rb = 0; rb < 4; ++rb) {
      const int rl = warp * 32 + rb * 8;
      const double* pa = Ys + (rl + lane / 4) * kAdLdY + lane % 4;
      double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      const double* pb = Rs + (lane % 4) * kAdLdR + lane / 4;
#pragma unroll
      for (int k = 0; k < 32; k += 4) {
        const double a = pa[k];
#pragma unroll
        for (int cj = 0; cj < 4; ++cj)
          if (cj < nb && k < 8 * (cj + 1)) dmma_8x8x4(acc[cj], a, pb[k * kAdLdR + cj * 8]);
      }
      const long long row = jb.y + rl + lane / 4;
      if (row < m.n) {
#pragma unroll
        for (int cj = 0; cj < 4; ++cj)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int col = cj * 8 + 2 * (lane % 4) + q;
            if (cj < nb && col < r) Y[(long long)col * m.ld + row] = (float)acc[cj][q];
          }
      }
    }
    j = jn;
  }
}

// ---- V1: SIMT, lane = row: each warp takes 32 rows of a tile, loads its r columns
// (coalesced 128 B per column), forms out[j] = sum_{k <= j} y[k] X[k][j] in fp64 with X broadcast
// from shared memory, stores each output column coalesced. CTA = 8 warps = one 256-row job;
// X staged once per CTA.
template <int RR>
__global__ void __launch_bounds__(256) v1(const DevMat* mats, const int4* jobs, int njobs, int rr,
                                         const double* rinv, float* buf) {
  __shared__ __align__(16) double Xs[RR * RR];  // [k][j], upper, zeros elsewhere
  const int4 jb = jobs[blockIdx.x];
  const DevMat m = mats[jb.x];
  const int r = m.r;
  const double* X = rinv + (long long)jb.x * rr * rr;
  for (int idx = threadIdx.x; idx < RR * RR; idx += 256) {
    const int k = idx / RR, c = idx % RR;
    Xs[idx] = (k < r && c < r && k <= c) ? X[k * rr + c] : 0.0;
  }
  const long long row = jb.y + threadIdx.x;
  const bool live = row < m.n;
  float* Y = buf + m.off;
  float v[RR];
#pragma unroll
  for (int k = 0; k < RR; ++k) v[k] = (k < r && live) ? Y[(long long)k * m.ld + row] : 0.f;
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
      if (j < r) Y[(long long)j * m.ld + row] = (float)o[j];
  }
}


// ---- V2 (RR = 32): two threads per row, output columns split by parity (balanced triangular
// work: 256 / 272 fmas); X staged permuted, Xp[p][k][i] = X[k][2i + p], so each thread's
// row of X is one contiguous 16-double run (LDS.128). CTA = 512 threads = 256 rows.
__global__ void __launch_bounds__(512) v2(const DevMat* mats, const int4* jobs, int njobs, int rr,
                                         const double* rinv, float* buf) {
  __shared__ __align__(16) double Xp[2 * 32 * 16];
  const int4 jb = jobs[blockIdx.x];
  const DevMat m = mats[jb.x];
  const int r = m.r;
  const double* X = rinv + (long long)jb.x * rr * rr;
  for (int idx = threadIdx.x; idx < 2 * 32 * 16; idx += 512) {
    const int p = idx / 512, k = (idx / 16) % 32, i = idx % 16, c = 2 * i + p;
    Xp[idx] = (k < r && c < r && k <= c) ? X[k * rr + c] : 0.0;
  }
  const int p = threadIdx.x / 256;
  const long long row = jb.y + (threadIdx.x % 256);
  const bool live = row < m.n;
  float* Y = buf + m.off;
  float v[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = (k < r && live) ? Y[(long long)k * m.ld + row] : 0.f;
  __syncthreads();
  double o[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i] = 0.0;
  const double* xb = Xp + p * 32 * 16;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double y = (double)v[k];
    const double2* xr = reinterpret_cast<const double2*>(xb + k * 16);
#pragma unroll
    for (int i2 = 0; i2 < 8; ++i2) {
      if (4 * i2 + 3 < k) continue;  // columns 2i+p < k are zero
      const double2 x = xr[i2];
      o[2 * i2] = fma(y, x.x, o[2 * i2]);
      o[2 * i2 + 1] = fma(y, x.y, o[2 * i2 + 1]);
    }
  }
  __syncthreads();  // both halves of the row have read it before either stores (in place)
  if (live) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (2 * i + p < r) Y[(long long)(2 * i + p) * m.ld + row] = (float)o[i];
  }
}


// ---- V3 (r <= 32): DMMA with the A fragments loaded straight from global memory (fp32 ->
// fp64 in registers), no shared-memory staging of Y and no block barriers per tile: each warp
// owns 32-row slices; R^-1 staged once per CTA (one factor per CTA-run of jobs as V0).
__global__ void __launch_bounds__(128) v3(const DevMat* mats, const int4* jobs, int njobs, int per_cta,
                                         int rr, const double* rinv, float* buf) {
  __shared__ double Rs[32 * kAdLdR];
  const int j0 = blockIdx.x * per_cta, j1 = min(njobs, j0 + per_cta);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int cur = -1;
  for (int j = j0; j < j1; ++j) {
    const int4 jb = jobs[j];
    const DevMat m = mats[jb.x];
    const int r = m.r, nb = (r + 7) / 8;
    if (jb.x != cur) {
      __syncthreads();
      const double* X = rinv + (long long)jb.x * rr * rr;
      for (int idx = threadIdx.x; idx < 32 * 32; idx += 128) {
        const int k = idx / 32, c = idx % 32;
        Rs[k * kAdLdR + c] = (k < r && c < r && k <= c) ? X[k * rr + c] : 0.0;
      }
      __syncthreads();
      cur = jb.x;
    }
    float* Y = buf + m.off;
    const double* pb = Rs + (lane % 4) * kAdLdR + lane / 4;
#pragma unroll
    for (int rb = 0; rb < 4; ++rb) {
      const long long row = jb.y + warp * 32 + rb * 8 + lane / 4;
      const bool live = row < m.n;
      // this lane's A elements: Y[row][k + lane%4] for the 8 k-steps
      float a[8];
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int col = 4 * ks + lane % 4;
        a[ks] = (live && col < r) ? Y[(long long)col * m.ld + row] : 0.f;
      }
      double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int k = 4 * ks;
        const double ad = (double)a[ks];
#pragma unroll
        for (int cj = 0; cj < 4; ++cj)
          if (cj < nb && k < 8 * (cj + 1)) dmma_8x8x4(acc[cj], ad, pb[k * kAdLdR + cj * 8]);
      }
      __syncwarp();  // every lane has read its rows before the in-place stores (same warp)
      if (live) {
#pragma unroll
        for (int cj = 0; cj < 4; ++cj)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int col = cj * 8 + 2 * (lane % 4) + q;
            if (cj < nb && col < r) Y[(long long)col * m.ld + row] = (float)acc[cj][q];
          }
      }
    }
  }
}


__global__ void __launch_bounds__(128) v4(const DevMat* mats, const int4* jobs, int njobs, int per_cta,
                                         int rr, const double* rinv, float* buf) {
  __shared__ double Rs[32 * kAdLdR];
  const int j0 = blockIdx.x * per_cta, j1 = min(njobs, j0 + per_cta);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int cur = -1;
  for (int j = j0; j < j1; ++j) {
    const int4 jb = jobs[j];
    const DevMat m = mats[jb.x];
    const int r = m.r, nb = (r + 7) / 8;
    if (jb.x != cur) {
      __syncthreads();
      const double* X = rinv + (long long)jb.x * rr * rr;
      for (int idx = threadIdx.x; idx < 32 * 32; idx += 128) {
        const int k = idx / 32, c = idx % 32;
        Rs[k * kAdLdR + c] = (k < r && c < r && k <= c) ? X[k * rr + c] : 0.0;
      }
      __syncthreads();
      cur = jb.x;
    }
    float* Y = buf + m.off;
    const double* pb = Rs + (lane % 4) * kAdLdR + lane / 4;
    float a[4][8];
#pragma unroll
    for (int rb = 0; rb < 4; ++rb) {
      const long long row = jb.y + warp * 32 + rb * 8 + lane / 4;
      const bool live = row < m.n;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int col = 4 * ks + lane % 4;
        a[rb][ks] = (live && col < r) ? Y[(long long)col * m.ld + row] : 0.f;
      }
    }
    __syncwarp();
#pragma unroll
    for (int rb = 0; rb < 4; ++rb) {
      const long long row = jb.y + warp * 32 + rb * 8 + lane / 4;
      double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int k = 4 * ks;
        const double ad = (double)a[rb][ks];
#pragma unroll
        for (int cj = 0; cj < 4; ++cj)
          if (cj < nb && k < 8 * (cj + 1)) dmma_8x8x4(acc[cj], ad, pb[k * kAdLdR + cj * 8]);
      }
      if (row < m.n) {
#pragma unroll
        for (int cj = 0; cj < 4; ++cj)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int col = cj * 8 + 2 * (lane % 4) + q;
            if (cj < nb && col < r) Y[(long long)col * m.ld + row] = (float)acc[cj][q];
          }
      }
    }
  }
}

int main() {
  // OPT-1.3B P side: embed 50272, pos 2050, 24 x (q,k,v,o 2048; fc1 8192; fc2 2048)
  std::vector<long long> ns = {50272, 2050};
  for (int l = 0; l < 24; ++l) { for (int i = 0; i < 4; ++i) ns.push_back(2048); ns.push_back(8192); ns.push_back(2048); }
  for (int R : {32, 16}) {
    std::vector<DevMat> mats;
    long long off = 0;
    for (size_t e = 0; e < ns.size(); ++e) { mats.push_back({off, ns[e], ns[e], R, (int)e}); off += ns[e] * R; }
    const long long total = off;
    std::vector<float> h(total);
    srand(3);
    for (auto& x : h) x = rand() / (float)RAND_MAX - 0.5f;
    const int ne = mats.size();
    std::vector<double> X(ne * 32 * 32, 0.0);
    for (int e = 0; e < ne; ++e)
      for (int k = 0; k < R; ++k)
        for (int c = k; c < R; ++c) X[e * 1024 + k * 32 + c] = (k == c) ? 1.0 + 0.01 * k : 0.01 * ((k * 7 + c * 3) % 11 - 5);
    std::vector<int4> jobs128, jobs256;
    for (int e = 0; e < ne; ++e) {
      for (long long r0 = 0; r0 < mats[e].n; r0 += 128) jobs128.push_back(make_int4(e, (int)r0, 0, 0));
      for (long long r0 = 0; r0 < mats[e].n; r0 += 256) jobs256.push_back(make_int4(e, (int)r0, 0, 0));
    }
    DevMat* dm; int4 *dj128, *dj256; double* dX; float *dY0, *dY;
    cudaMalloc(&dm, sizeof(DevMat) * ne); cudaMemcpy(dm, mats.data(), sizeof(DevMat) * ne, cudaMemcpyHostToDevice);
    cudaMalloc(&dj128, sizeof(int4) * jobs128.size()); cudaMemcpy(dj128, jobs128.data(), sizeof(int4) * jobs128.size(), cudaMemcpyHostToDevice);
    cudaMalloc(&dj256, sizeof(int4) * jobs256.size()); cudaMemcpy(dj256, jobs256.data(), sizeof(int4) * jobs256.size(), cudaMemcpyHostToDevice);
    cudaMalloc(&dX, sizeof(double) * X.size()); cudaMemcpy(dX, X.data(), sizeof(double) * X.size(), cudaMemcpyHostToDevice);
    cudaMalloc(&dY0, sizeof(float) * total); cudaMemcpy(dY0, h.data(), sizeof(float) * total, cudaMemcpyHostToDevice);
    cudaMalloc(&dY, sizeof(float) * total);
    std::vector<float> ref;
    for (int v = 0; v < 12; ++v) {
      auto launch = [&] {
        if (v == 0 || (v >= 3 && v <= 6)) {
          const int nj = jobs128.size();
          int per = std::max(1, (nj + 4 * 148 - 1) / (4 * 148));
          if (v == 3) per = 1;
          if (v == 4) per = 2;
          if (v == 5) per = 4;
          if (v == 6) per = 12;
          v0<<<(nj + per - 1) / per, 128>>>(dm, dj128, nj, per, 32, dX, dY);
        } else if (v >= 7 && v <= 9) {
          const int nj = jobs128.size();
          const int per = v == 7 ? std::max(1, (nj + 4 * 148 - 1) / (4 * 148)) : (v == 8 ? 2 : 1);
          v3<<<(nj + per - 1) / per, 128>>>(dm, dj128, nj, per, 32, dX, dY);
        } else if (v >= 10) {
          const int nj = jobs128.size();
          const int per = v == 10 ? 1 : 2;
          v4<<<(nj + per - 1) / per, 128>>>(dm, dj128, nj, per, 32, dX, dY);
        } else if (v == 2) {
          v2<<<jobs256.size(), 512>>>(dm, dj256, jobs256.size(), 32, dX, dY);
        } else if (R == 32) {
          v1<32><<<jobs256.size(), 256>>>(dm, dj256, jobs256.size(), 32, dX, dY);
        } else {
          v1<16><<<jobs256.size(), 256>>>(dm, dj256, jobs256.size(), 32, dX, dY);
        }
      };
      float best = 1e9;
      for (int it = 0; it < 6; ++it) {
        cudaMemcpy(dY, dY0, sizeof(float) * total, cudaMemcpyDeviceToDevice);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (it > 0) best = fminf(best, ms);
      }
      std::vector<float> out(total);
      cudaMemcpy(out.data(), dY, sizeof(float) * total, cudaMemcpyDeviceToHost);
      double md = 0; long long ndiff = 0;
      if (v == 0) ref = out; else for (long long i = 0; i < total; ++i) { double d = fabs(out[i] - ref[i]); if (d > 0) ++ndiff; md = fmax(md, d); }
      printf("r=%d variant %d: %.2f us  (vs v0: max |diff| %.3g, %lld differing)  %s\n", R, v, best * 1000, md, ndiff,
             cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(dm); cudaFree(dj128); cudaFree(dj256); cudaFree(dX); cudaFree(dY0); cudaFree(dY);
  }
  return 0;
}
