// tma_bw.cu — microbenchmark: HBM read bandwidth of a persistent TMA-streaming kernel as a
// function of the box shape (rows x bytes-per-row) and boxes per stage. Experiments only.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_bw.cu -o /tmp/tma_bw -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2506_21263_b200/csrc/ptx.cuh"

using namespace dlx;

__global__ void __launch_bounds__(128, 1) k_stream(const CUtensorMap* map, int rows_total,
                                                   int cols_total, int box_c, int box_r,
                                                   int per_stage, int stages, int touch) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int stage_bytes = box_c * box_r * 4 * per_stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * stage_bytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 96);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // tiles: row blocks of box_r rows, each swept along columns in steps of box_c*per_stage
  const int rblocks = rows_total / box_r;
  const int csteps = cols_total / (box_c * per_stage);
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      uint32_t it = 0;
      for (int rb = blockIdx.x; rb < rblocks; rb += gridDim.x)
        for (int cs = 0; cs < csteps; ++cs, ++it) {
          const int s = it % stages;
          mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
          mbar_expect_tx(&full[s], stage_bytes);
          for (int q = 0; q < per_stage; ++q)
            tma_load_2d(sm + s * stage_bytes + q * box_c * box_r * 4, map, &full[s],
                        (cs * per_stage + q) * box_c, rb * box_r);
        }
    }
    return;
  }
  uint32_t it = 0;
  float acc = 0.f;
  for (int rb = blockIdx.x; rb < rblocks; rb += gridDim.x)
    for (int cs = 0; cs < csteps; ++cs, ++it) {
      const int s = it % stages;
      mbar_wait(&full[s], (it / stages) & 1);
      if (touch) {
        const float4* p = reinterpret_cast<const float4*>(sm + s * stage_bytes);
        for (int i = threadIdx.x - 32; i < stage_bytes / 16; i += 96) {
          float4 v = p[i];
          acc += v.x + v.y + v.z + v.w;
        }
      }
      mbar_arrive(&empty[s]);
    }
  if (acc == 12345.f) printf("x");
}

int main() {
  const int rows = 65536, cols = 8192;  // 2 GiB fp32
  float* d;
  cudaMalloc(&d, (size_t)rows * cols * 4);
  cudaMemset(d, 0, (size_t)rows * cols * 4);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap* dmap;
  cudaMalloc(&dmap, sizeof(CUtensorMap));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct Cfg { int bc, br, per, stages, swz; };
  std::vector<Cfg> cfgs = {{32, 128, 1, 8, 1}, {32, 128, 2, 5, 1}, {32, 128, 4, 3, 1},
                           {32, 64, 4, 5, 1},  {64, 64, 1, 8, 0},  {128, 32, 1, 8, 0},
                           {128, 16, 1, 8, 0}, {256, 16, 1, 6, 0}, {256, 32, 1, 3, 0},
                           {32, 256, 1, 4, 1}};
  for (int touch = 0; touch < 2; ++touch)
    for (auto c : cfgs) {
      CUtensorMap m;
      const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
      const cuuint64_t str[1] = {(cuuint64_t)cols * 4};
      const cuuint32_t box[2] = {(cuuint32_t)c.bc, (cuuint32_t)c.br};
      const cuuint32_t es[2] = {1, 1};
      CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE,
                       c.swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("encode failed %d for %dx%d\n", (int)r, c.bc, c.br);
        continue;
      }
      cudaMemcpy(dmap, &m, sizeof(m), cudaMemcpyHostToDevice);
      const int smem = c.stages * c.bc * c.br * 4 * c.per + 1024;
      cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      for (int w = 0; w < 2; ++w)
        k_stream<<<sms, 128, smem>>>(dmap, rows, cols, c.bc, c.br, c.per, c.stages, touch);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      const int n = 5;
      for (int w = 0; w < n; ++w)
        k_stream<<<sms, 128, smem>>>(dmap, rows, cols, c.bc, c.br, c.per, c.stages, touch);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= n;
      printf("touch=%d box %3d cols x %3d rows x%d/stage, %d stages (%3d KB in flight/SM): %7.1f GB/s  err=%s\n",
             touch, c.bc, c.br, c.per, c.stages, c.stages * c.bc * c.br * 4 * c.per / 1024,
             (double)rows * cols * 4 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
