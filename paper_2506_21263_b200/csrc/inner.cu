// inner.cu — the inner optimiser step that overlaps the outer synchronisation
// (SURVEY §8f row 2): bias-corrected AdamW with decoupled weight decay, adamw_step
// (optim.cpp:15-47), one fused elementwise pass over the parameter slab (4 reads, 3 writes:
// 28 B/param). Bit-exact with the reference: the step-dependent scalars (bias corrections,
// warm-up learning rate) are computed on the host exactly as optim.cpp does, every device
// operation rounds separately (-ffp-contract=off in the reference build).
#include <cmath>

#include "dlx_internal.cuh"

namespace dlx {

__global__ void __launch_bounds__(256) k_adamw(int64_t n, float lr, float beta1, float beta2,
                                               float om1, float om2, float eps, float wd,
                                               float inv_bc1, float inv_bc2, float* __restrict__ p,
                                               const float* __restrict__ g,
                                               float* __restrict__ m, float* __restrict__ v,
                                               int* __restrict__ nonfinite) {
  int bad = 0;
  auto one = [&](float& pk, float gk, float& mk, float& vk) {
    bad |= !isfinite(gk);  // the reference's probe += g * 0 (NaN / Inf poison it)
    mk = __fadd_rn(__fmul_rn(beta1, mk), __fmul_rn(om1, gk));
    vk = __fadd_rn(__fmul_rn(beta2, vk), __fmul_rn(__fmul_rn(om2, gk), gk));
    const float mhat = __fmul_rn(mk, inv_bc1);
    const float vhat = __fmul_rn(vk, inv_bc2);
    const float den = __fadd_rn(__fsqrt_rn(vhat), eps);
    const float upd = __fadd_rn(__fdiv_rn(mhat, den), __fmul_rn(wd, pk));
    pk = __fsub_rn(pk, __fmul_rn(lr, upd));
  };
  const int64_t n4 = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 pp = reinterpret_cast<float4*>(p)[i];
    const float4 gg = __ldcs(reinterpret_cast<const float4*>(g) + i);
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    one(pp.x, gg.x, mm.x, vv.x);
    one(pp.y, gg.y, mm.y, vv.y);
    one(pp.z, gg.z, mm.z, vv.z);
    one(pp.w, gg.w, mm.w, vv.w);
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    one(p[i], g[i], m[i], v[i]);
  if (bad && nonfinite) atomicOr(nonfinite, 1);
}

void launch_adamw(int64_t n, float lr, float beta1, float beta2, float eps, float wd,
                  int64_t warmup_steps, int64_t step, float* p, const float* g, float* m,
                  float* v, int* nonfinite, cudaStream_t s) {
  // optim.cpp:21-27, host-side (same libm as the reference)
  const float bc1 = 1.0f - std::pow(beta1, static_cast<float>(step));
  const float bc2 = 1.0f - std::pow(beta2, static_cast<float>(step));
  float lr_t = lr;
  if (warmup_steps > 0 && step < warmup_steps)
    lr_t = lr * static_cast<float>(step) / static_cast<float>(warmup_steps);
  const float inv_bc1 = 1.0f / bc1;
  const float inv_bc2 = 1.0f / bc2;
  const float om1 = 1.0f - beta1, om2 = 1.0f - beta2;
  if (((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g) |
        reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) != 0)
    raise(DLX_ERR_VALIDATION, "adamw_step: buffers must be 16-byte aligned");
  int dev = 0, sms = 0;
  DLX_CUDA(cudaGetDevice(&dev));
  DLX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  KernelTimer timer("k_adamw", 28.0 * n, s);
  k_adamw<<<sms * 8, 256, 0, s>>>(n, lr_t, beta1, beta2, om1, om2, eps, wd, inv_bc1, inv_bc2, p, g,
                                  m, v, nonfinite);
  DLX_LAUNCHED();
}

}  // namespace dlx
