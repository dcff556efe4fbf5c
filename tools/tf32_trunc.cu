// tf32_trunc.cu — does tcgen05.mma.kind::tf32 truncate or round fp32 operands? (experiment)
// D[m][n] = sum_k A[m][k] B[n][k] with A[m][0] = v_m, B[n][0] = 1, everything else 0.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2506_21263_b200/csrc/ptx.cuh"
using namespace dlx;

__global__ void k(const float* v, float* out) {
  __shared__ __align__(1024) uint8_t sm[128 * 128 + 32 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  float* A = reinterpret_cast<float*>(sm);
  float* B = reinterpret_cast<float*>(sm + 128 * 128);
  for (int i = threadIdx.x; i < 128 * 32 + 32 * 32; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  __syncthreads();
  const int m = threadIdx.x;
  A[m * 32 + (m & 7) * 4] = v[m];              // k = 0 of row m (SW128: chunk 0 at chunk m%8)
  if (m < 32) B[m * 32 + (m & 7) * 4] = 1.0f;  // k = 0 of row n = m
  fence_async_smem();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    mma_tf32(tmem, sdesc(su32(A), 16, 1024), sdesc(su32(B), 16, 1024), idesc_tf32(32, false, false), 0u);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float d[16];
  const uint32_t lane_base = static_cast<uint32_t>((threadIdx.x / 32) * 32) << 16;
  tmem_ld16(tmem + lane_base, d);
  out[m] = d[0];
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}

int main() {
  float h[128], o[128];
  for (int i = 0; i < 128; ++i) {
    // 1 + mantissa pattern in the 13 dropped bits: bit 12 (half ulp) and below
    const uint32_t bits = 0x3F800000u | (uint32_t)(i * 64 + (i % 3)) ;
    memcpy(&h[i], &bits, 4);
  }
  float *dv, *dout;
  cudaMalloc(&dv, 512); cudaMalloc(&dout, 512);
  cudaMemcpy(dv, h, 512, cudaMemcpyHostToDevice);
  k<<<1, 128>>>(dv, dout);
  cudaMemcpy(o, dout, 512, cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  int trunc = 0, rn = 0, other = 0;
  for (int i = 0; i < 128; ++i) {
    uint32_t b; memcpy(&b, &h[i], 4);
    const uint32_t t = b & 0xFFFFE000u;
    uint32_t r = b + 0x1000u; r &= 0xFFFFE000u;  // round half up (approx RN)
    uint32_t ob; memcpy(&ob, &o[i], 4);
    if (ob == t) ++trunc; else if (ob == r) ++rn; else ++other;
    if (i < 6 || (i % 32) == 0) printf("in=%08x out=%08x trunc=%08x rn=%08x\n", b, ob, t, r);
  }
  printf("trunc-match=%d rn-match=%d other=%d\n", trunc, rn, other);
}
