// tma_rw.cu — microbenchmark: HBM throughput of the fused outer update's access mix
// (4 streams read, 3 written back in place, TMA both ways) without any compute, as a
// function of tile width and stage count. Experiments only.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_rw.cu -o /tmp/tma_rw -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2506_21263_b200/csrc/ptx.cuh"

using namespace dlx;

struct Maps {
  CUtensorMap m[4];
};

__global__ void __launch_bounds__(128, 1) k_rw(const Maps* maps, int rows, int cols, int bw,
                                               int nst, int nwrite, int* ctr, int band_mode) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t box = 128 * bw * 4;
  const uint32_t stage = 4 * box;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + nst * stage);
  uint64_t* empty = full + nst;
  int* tinfo = reinterpret_cast<int*>(empty + nst);
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int tiles_per_band = cols / bw, nbands = rows / 128;
  const int ntiles = tiles_per_band * nbands;
  if (threadIdx.x < 32) {
    int s = 0;
    uint32_t ph = 0;
    int bt = 0, bend = 0;  // band mode: tiles of the claimed band
    for (;;) {
      int t = 0;
      if (band_mode) {
        if (bt == bend) {
          int b = 0;
          if (threadIdx.x == 0) b = atomicAdd(ctr, 1);
          b = __shfl_sync(0xffffffffu, b, 0);
          bt = b * tiles_per_band;
          bend = bt + tiles_per_band;
          if (b >= nbands) bt = bend = ntiles;
        }
        t = bt < ntiles ? bt++ : ntiles;
      } else {
        if (threadIdx.x == 0) t = atomicAdd(ctr, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
      }
      mbar_wait(&empty[s], ph ^ 1);
      if (threadIdx.x == 0) {
        tinfo[s] = t < ntiles ? t : -1;
        if (t < ntiles) {
          const int band = t / tiles_per_band, n0 = (t % tiles_per_band) * bw;
          mbar_expect_tx(&full[s], stage);
          for (int q = 0; q < 4; ++q) tma_load_2d(sm + s * stage + q * box, &maps->m[q], &full[s], n0, band * 128);
        } else {
          mbar_arrive(&full[s]);
        }
      }
      __syncwarp();
      if (++s == nst) {
        s = 0;
        ph ^= 1;
      }
      if (t >= ntiles) break;
    }
  } else if (threadIdx.x == 32) {
    int s = 0;
    uint32_t ph = 0;
    for (;;) {
      mbar_wait(&full[s], ph);
      const int t = tinfo[s];
      if (t < 0) break;
      const int band = t / tiles_per_band, n0 = (t % tiles_per_band) * bw;
      for (int q = 0; q < nwrite; ++q) tma_store_2d(&maps->m[q], sm + s * stage + q * box, n0, band * 128);
      bulk_commit();
      bulk_wait_read0();
      mbar_arrive(&empty[s]);
      if (++s == nst) {
        s = 0;
        ph ^= 1;
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const int rows = 16384, cols = 8192;  // 512 MiB per array, 4 arrays
  std::vector<float*> a(4);
  for (auto& p : a) {
    cudaMalloc(&p, (size_t)rows * cols * 4);
    cudaMemset(p, 0, (size_t)rows * cols * 4);
  }
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
  Maps* dm;
  cudaMalloc(&dm, sizeof(Maps));
  int* ctr;
  cudaMalloc(&ctr, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_rw, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  struct Cfg { int bw, nst, nwrite, band; };
  std::vector<Cfg> cfgs = {{32, 2, 3, 0}, {32, 2, 3, 1}, {32, 3, 3, 1}, {16, 5, 3, 0}, {16, 5, 3, 1},
                           {32, 3, 0, 0}, {32, 3, 0, 1}};
  for (auto c : cfgs) {
    Maps h;
    for (int q = 0; q < 4; ++q) {
      const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
      const cuuint64_t str[1] = {(cuuint64_t)cols * 4};
      const cuuint32_t box[2] = {(cuuint32_t)c.bw, 128};
      const cuuint32_t es[2] = {1, 1};
      enc(&h.m[q], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a[q], dims, str, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE,
          c.bw == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : c.bw == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    cudaMemcpy(dm, &h, sizeof(h), cudaMemcpyHostToDevice);
    const int smem = c.nst * 4 * 128 * c.bw * 4 + 1024 + 64 * c.nst;
    float best = 1e30f;
    for (int it = 0; it < 6; ++it) {
      cudaMemset(ctr, 0, 4);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k_rw<<<sms, 128, smem>>>(dm, rows, cols, c.bw, c.nst, c.nwrite, ctr, c.band);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it > 0 && ms < best) best = ms;
    }
    const double bytes = (double)rows * cols * 4 * (4 + c.nwrite);
    printf("bw=%2d nst=%d writes=%d band_per_cta=%d: %.3f ms  %.1f GB/s  err=%s\n", c.bw, c.nst, c.nwrite, c.band, best,
           bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
