// Microbenchmark: CholQR apply Y <- Y R^-1 at 32 < r <= 64 over the OPT-1.3B P-side factor
// set: the library's SIMT k_apply (one smem load per fma) vs a SIMT variant with R^-1 staged
// once and read with 16-B broadcast loads, triangle-aware.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o apply64_micro apply64_micro.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

struct DevMat { long long off, n, ld; int r, slot; };

__global__ void __launch_bounds__(128) k_apply(const DevMat* __restrict__ mats,
                                               const int4* __restrict__ jobs, int rr,
                                               const double* __restrict__ rinv,
                                               float* __restrict__ buf) {
  extern __shared__ __align__(16) unsigned char ap_smem[];
  const int4 jb = jobs[blockIdx.x];
  const DevMat m = mats[jb.x];
  const int r = m.r;
  double* Rs = reinterpret_cast<double*>(ap_smem);
  float* Ys = reinterpret_cast<float*>(Rs + 32 * 33);
  const long long row = jb.y + threadIdx.x;
  const bool live = row < m.n;
  float* Y = buf + m.off;
  const double* X = rinv + (long long)jb.x * rr * rr;
  for (int idx = threadIdx.x; idx < r * 128; idx += 128) {
    const int c = idx / 128, i = idx % 128;
    Ys[c * 129 + i] = (jb.y + i < m.n) ? Y[(long long)c * m.ld + jb.y + i] : 0.f;
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
        if (j < jmax) Y[(long long)(cb * 32 + j) * m.ld + row] = (float)acc[j];
    }
  }
}

// New: X (RR x RR upper) staged once per CTA (row-major, 16-B aligned rows); each thread one
// row with its RR inputs in registers; outputs in 32-column passes, X read as double2.
template <int RR>
__global__ void __launch_bounds__(128) k_apply_x(const DevMat* __restrict__ mats,
                                                 const int4* __restrict__ jobs, int rr,
                                                 const double* __restrict__ rinv,
                                                 float* __restrict__ buf) {
  __shared__ __align__(16) double Xs[RR * RR];
  const int4 jb = jobs[blockIdx.x];
  const DevMat m = mats[jb.x];
  const int r = m.r;
  const double* X = rinv + (long long)jb.x * rr * rr;
  for (int idx = threadIdx.x; idx < RR * RR; idx += 128) {
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
#pragma unroll
  for (int cb = 0; cb < RR / 32; ++cb) {
    double acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0;
#pragma unroll
    for (int k = 0; k < 32 * (cb + 1); ++k) {
      const double y = (double)v[k];
      const double2* xr = reinterpret_cast<const double2*>(Xs + k * RR + 32 * cb);
#pragma unroll
      for (int j2 = 0; j2 < 16; ++j2) {
        if (32 * cb + 2 * j2 + 1 < k) continue;  // X[k][j] = 0 for j < k
        const double2 x = xr[j2];
        acc[2 * j2] = fma(y, x.x, acc[2 * j2]);
        acc[2 * j2 + 1] = fma(y, x.y, acc[2 * j2 + 1]);
      }
    }
    if (live) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (32 * cb + j < r) Y[(long long)(32 * cb + j) * m.ld + row] = (float)acc[j];
    }
  }
}


// Variant 2: Y tile in shared memory ([col][row], as k_apply), X staged once (row-major),
// per k: one y load + 16 double2 X loads for 32 fmas.
template <int RR>
__global__ void __launch_bounds__(128) k_apply_y(const DevMat* __restrict__ mats,
                                                 const int4* __restrict__ jobs, int rr,
                                                 const double* __restrict__ rinv,
                                                 float* __restrict__ buf) {
  extern __shared__ __align__(16) unsigned char sm2[];
  double* Xs = reinterpret_cast<double*>(sm2);           // [RR][RR]
  float* Ys = reinterpret_cast<float*>(Xs + RR * RR);     // [RR][129]
  const int4 jb = jobs[blockIdx.x];
  const DevMat m = mats[jb.x];
  const int r = m.r;
  const double* X = rinv + (long long)jb.x * rr * rr;
  for (int idx = threadIdx.x; idx < RR * RR; idx += 128) {
    const int k = idx / RR, c = idx % RR;
    Xs[idx] = (k < r && c < r && k <= c) ? X[k * rr + c] : 0.0;
  }
  float* Y = buf + m.off;
  for (int idx = threadIdx.x; idx < r * 128; idx += 128) {
    const int c = idx / 128, i = idx % 128;
    Ys[c * 129 + i] = (jb.y + i < m.n) ? Y[(long long)c * m.ld + jb.y + i] : 0.f;
  }
  __syncthreads();
  const long long row = jb.y + threadIdx.x;
  const bool live = row < m.n;
#pragma unroll 1
  for (int cb = 0; cb < RR / 32; ++cb) {
    if (32 * cb >= r) break;
    double acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0;
    const int kmax = min(r, 32 * (cb + 1));
    for (int k = 0; k < kmax; ++k) {
      const double y = (double)Ys[k * 129 + threadIdx.x];
      const double2* xr = reinterpret_cast<const double2*>(Xs + k * RR + 32 * cb);
#pragma unroll
      for (int j2 = 0; j2 < 16; ++j2) {
        const double2 x = xr[j2];
        acc[2 * j2] = fma(y, x.x, acc[2 * j2]);
        acc[2 * j2 + 1] = fma(y, x.y, acc[2 * j2 + 1]);
      }
    }
    if (live) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (32 * cb + j < r) Y[(long long)(32 * cb + j) * m.ld + row] = (float)acc[j];
    }
  }
}

int main() {
  std::vector<long long> ns = {50272, 2050};
  for (int l = 0; l < 24; ++l) { for (int i = 0; i < 4; ++i) ns.push_back(2048); ns.push_back(8192); ns.push_back(2048); }
  const int RR = 64;
  for (int R : {64, 48}) {
    std::vector<DevMat> mats;
    long long off = 0;
    for (size_t e = 0; e < ns.size(); ++e) { mats.push_back({off, ns[e], ns[e], R, (int)e}); off += ns[e] * R; }
    const long long total = off;
    std::vector<float> h(total);
    srand(3);
    for (auto& x : h) x = rand() / (float)RAND_MAX - 0.5f;
    const int ne = mats.size();
    std::vector<double> X((size_t)ne * RR * RR, 0.0);
    for (int e = 0; e < ne; ++e)
      for (int k = 0; k < R; ++k)
        for (int c = k; c < R; ++c) X[(size_t)e * RR * RR + k * RR + c] = (k == c) ? 1.0 + 0.01 * k : 0.01 * ((k * 7 + c * 3) % 11 - 5);
    std::vector<int4> jobs;
    for (int e = 0; e < ne; ++e)
      for (long long r0 = 0; r0 < mats[e].n; r0 += 128) jobs.push_back(make_int4(e, (int)r0, 0, 0));
    DevMat* dm; int4* dj; double* dX; float *dY0, *dY;
    cudaMalloc(&dm, sizeof(DevMat) * ne); cudaMemcpy(dm, mats.data(), sizeof(DevMat) * ne, cudaMemcpyHostToDevice);
    cudaMalloc(&dj, sizeof(int4) * jobs.size()); cudaMemcpy(dj, jobs.data(), sizeof(int4) * jobs.size(), cudaMemcpyHostToDevice);
    cudaMalloc(&dX, sizeof(double) * X.size()); cudaMemcpy(dX, X.data(), sizeof(double) * X.size(), cudaMemcpyHostToDevice);
    cudaMalloc(&dY0, sizeof(float) * total); cudaMemcpy(dY0, h.data(), sizeof(float) * total, cudaMemcpyHostToDevice);
    cudaMalloc(&dY, sizeof(float) * total);
    const size_t sm = 32 * 33 * sizeof(double) + sizeof(float) * R * 129;
    cudaFuncSetAttribute(k_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    std::vector<float> ref;
    cudaFuncSetAttribute(k_apply_y<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int v = 0; v < 3; ++v) {
      float best = 1e9;
      for (int it = 0; it < 6; ++it) {
        cudaMemcpy(dY, dY0, sizeof(float) * total, cudaMemcpyDeviceToDevice);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        if (v == 0) k_apply<<<jobs.size(), 128, sm>>>(dm, dj, RR, dX, dY);
        else if (v == 1) k_apply_x<64><<<jobs.size(), 128>>>(dm, dj, RR, dX, dY);
        else k_apply_y<64><<<jobs.size(), 128, sizeof(double) * 64 * 64 + sizeof(float) * 64 * 129>>>(dm, dj, RR, dX, dY);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (it > 0) best = fminf(best, ms);
      }
      std::vector<float> out(total);
      cudaMemcpy(out.data(), dY, sizeof(float) * total, cudaMemcpyDeviceToHost);
      double md = 0; long long nd = 0;
      if (v == 0) ref = out; else for (long long i = 0; i < total; ++i) { double d = fabs(out[i] - ref[i]); if (d > 0) ++nd; md = fmax(md, d); }
      printf("r=%d variant %d: %.2f us (vs v0 max |diff| %.3g, %lld differ) %s\n", R, v, best * 1000, md, nd, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(dm); cudaFree(dj); cudaFree(dX); cudaFree(dY0); cudaFree(dY);
  }
  return 0;
}
