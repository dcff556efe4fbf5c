// epilogue.cuh — one element of the fused outer update, with the reference's rounding order
// (engine.cpp:254-276, optim.cpp:56-78; -ffp-contract=off: every op rounds separately).
#pragma once
#include "dlx_internal.cuh"

namespace dlx {

struct EpiOut {
  float pend, anchor, v, e;
};

// One element of the fused epilogue given Delta (all roundings explicit).
__device__ __forceinline__ EpiOut epilogue(float delta, float pend, float anchor, float local,
                                           float v, int mode, float gamma, float beta,
                                           int classical) {
  EpiOut o;
  if (mode == DLX_MODE_OVERLAPPED) {
    o.e = __fsub_rn(pend, delta);
    o.pend = __fadd_rn(__fsub_rn(anchor, local), o.e);
  } else {
    o.e = __fsub_rn(pend, delta);
    o.pend = o.e;
  }
  o.v = __fadd_rn(__fmul_rn(beta, v), delta);
  if (classical) {
    o.anchor = __fsub_rn(anchor, __fmul_rn(gamma, o.v));
  } else {
    o.anchor = __fsub_rn(anchor, __fmul_rn(gamma, __fadd_rn(delta, __fmul_rn(beta, o.v))));
  }
  return o;
}

}  // namespace dlx
