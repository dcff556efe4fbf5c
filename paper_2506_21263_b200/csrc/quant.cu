// quant.cu — per-column q-bit quantisation with counter-addressed stochastic rounding and
// in-kernel bit packing (quantize compress.cpp:24-49, quantize_columns :119-131,
// pack_codes :352-367), plus the gathered-payload dequantiser (dequantize_columns
// :133-142) for the reconstruction and the effective rank.
//
// Bit-exactness recipe (given identical fp32 inputs): maxabs is order independent;
// scale = max / L and inv = 1 / scale with IEEE division; y = x * inv (one rounding);
// nearest = round-half-even (lrintf); stochastic = floor(y) + (u < y - floor(y)) with u the
// top 24 bits of draw k of the shared splitmix stream. Draw k is addressed directly:
// k = 1 + (draws consumed by all earlier chunks, including cold-start inits) + index in
// chunk, found by an exclusive scan over the chunk table. All-zero chunks draw nothing.
#include "dlx_internal.cuh"

namespace dlx {

__device__ __forceinline__ const float* buf_ptr(int buf, const float* p, const float* q,
                                                const float* slab) {
  return buf == 0 ? p : (buf == 1 ? q : slab);
}

// ------------------------------------------------------------------ 1. chunk max|x|
__global__ void __launch_bounds__(256) k_chunk_max(const DevChunk* __restrict__ chunks,
                                                   const float* __restrict__ p,
                                                   const float* __restrict__ q,
                                                   const float* __restrict__ slab,
                                                   float* __restrict__ cmax) {
  __shared__ float red[8];
  const DevChunk c = chunks[blockIdx.x];
  const float* src = buf_ptr(c.buf, p, q, slab) + c.src;
  float m = 0.f;
  // 16-B loads where the chunk start is 16-B aligned (factor columns start on 32-float rows,
  // tensors on 256-B offsets), 4 in flight per thread: the long pole is the embedding's
  // 50272-row columns, one CTA each
  int64_t head = 0;
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const int64_t nv = c.len / 4;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    int64_t i = threadIdx.x;
    for (; i + 3 * 256 < nv; i += 4 * 256) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(s4 + i + u * 256);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        m = fmaxf(m, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
    }
    for (; i < nv; i += 256) {
      const float4 v = __ldg(s4 + i);
      m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
    head = 4 * nv;
  }
  for (int64_t i = head + threadIdx.x; i < c.len; i += blockDim.x) m = fmaxf(m, fabsf(src[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float r = red[0];
    for (int i = 1; i < 8; ++i) r = fmaxf(r, red[i]);
    cmax[blockIdx.x] = r;
  }
}

// ------------------------------------------------------------------ 2. scan + scales
// Single CTA. base[c] = draw offset of the chunk's first element (0-based count of draws
// consumed before it). Also writes the fp32 scales into the payload, inv[c], the total
// draw count, and checks the speculative cold-start bases.
__global__ void __launch_bounds__(1024) k_chunk_scan(const DevChunk* __restrict__ chunks, int n,
                                                     const float* __restrict__ cmax, int levels,
                                                     int stochastic, int cold,
                                                     const int64_t* __restrict__ spec,
                                                     int64_t* __restrict__ base,
                                                     float* __restrict__ inv,
                                                     uint8_t* __restrict__ payload,
                                                     uint64_t* __restrict__ total,
                                                     int* __restrict__ mismatch,
                                                     int64_t* __restrict__ cold_actual) {
  __shared__ int64_t warp_tot[32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // the next 1024 chunks are loaded while the current ones are scanned (one exposed load
  // latency per launch instead of one per 1024 chunks)
  DevChunk nch{};
  float nmx = 0.f;
  if (threadIdx.x < n) {
    nch = chunks[threadIdx.x];
    nmx = cmax[threadIdx.x];
  }
  for (int t0 = 0; t0 < n; t0 += 1024) {
    const int c = t0 + threadIdx.x;
    const DevChunk ch = nch;
    const float mx = nmx;
    if (c + 1024 < n) {
      nch = chunks[c + 1024];
      nmx = cmax[c + 1024];
    }
    int64_t extra = 0, own = 0;
    if (c < n) {
      extra = cold ? ch.extra : 0;
      own = (stochastic && mx != 0.f) ? ch.len : 0;
    }
    const int64_t v = extra + own;
    // inclusive warp scan
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int64_t w = warp_tot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_tot[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int64_t before = carry + (wid > 0 ? warp_tot[wid - 1] : 0) + (x - v);  // exclusive
    if (c < n) {
      base[c] = before + extra;
      float sc = 0.f, iv = 0.f;
      if (mx != 0.f) {
        sc = __fdiv_rn(mx, (float)levels);
        iv = __fdiv_rn(1.0f, sc);
      }
      inv[c] = iv;
      *reinterpret_cast<float*>(payload + ch.scale_dst) = sc;
      if (cold && ch.extra > 0 && ch.tensor >= 0) {
        cold_actual[ch.tensor] = before;
        if (spec && spec[ch.tensor] != before) atomicOr(mismatch, 1);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_tot[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = static_cast<uint64_t>(carry);
}

// ------------------------------------------------------------------ 3. quantise + pack
__global__ void __launch_bounds__(256) k_quant_pack(const DevStream* __restrict__ streams,
                                                    int nstreams, int64_t ngroups,
                                                    const int64_t* __restrict__ base,
                                                    const float* __restrict__ inv,
                                                    const float* __restrict__ cmax,
                                                    const float* __restrict__ p,
                                                    const float* __restrict__ q,
                                                    const float* __restrict__ slab, int qbits,
                                                    int stochastic, uint64_t s0,
                                                    const uint64_t* __restrict__ s0p,
                                                    uint8_t* __restrict__ payload) {
  if (s0p) s0 = *s0p;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  // the stream of the block's first group: one binary search per block (not a chain of
  // dependent global loads per thread), then a short forward walk per thread
  __shared__ int s_first;
  if (threadIdx.x == 0) {
    const int64_t g0 = blockIdx.x * (int64_t)blockDim.x;
    int lo = 0, hi = nstreams - 1;  // last stream with group0 <= g0
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (streams[mid].group0 <= g0) lo = mid; else hi = mid - 1;
    }
    s_first = lo;
  }
  __syncthreads();
  if (g >= ngroups) return;
  int lo = s_first;
  while (lo + 1 < nstreams && streams[lo + 1].group0 <= g) ++lo;
  const DevStream st = streams[lo];
  const int64_t lg = g - st.group0;
  const int64_t total = st.col_len * st.ncols;
  const float* src = buf_ptr(st.buf, p, q, slab) + st.src;
  const int L = (1 << (qbits - 1)) - 1;
  const uint64_t mask = (1ull << qbits) - 1ull;
  uint64_t bits = 0;
  int valid = 0;
  // (column, row) of the group's first code: one 32-bit division per group, then stepped
  const uint32_t clen = static_cast<uint32_t>(st.col_len);
  const uint32_t idx0 = static_cast<uint32_t>(lg * 8);
  uint32_t colw = idx0 / clen, roww = idx0 - colw * clen;
  const float* gsrc = src + static_cast<int64_t>(colw) * st.ld + roww;
  if (roww + 8 <= clen && (reinterpret_cast<uintptr_t>(gsrc) & 15) == 0) {
    // the whole group in one column, 16-B aligned: two vector loads, one chunk's constants
    const int64_t c = st.chunk0 + colw;
    const float mx = cmax[c];
    if (mx != 0.f) {
      const float iv = inv[c];
      const float4 v0 = *reinterpret_cast<const float4*>(gsrc);
      const float4 v1 = *reinterpret_cast<const float4*>(gsrc + 4);
      const float xs[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
      // counter of the group's first draw; the next ones are +gamma each (no 64-bit multiply
      // per element: the integer pipe, not HBM, bounds this kernel)
      uint64_t z = s0 + static_cast<uint64_t>(base[c] + roww + 1) * kGolden;
#pragma unroll
      for (int t = 0; t < 8; ++t, z += kGolden) {
        const float y = __fmul_rn(xs[t], iv);
        int code;
        if (!stochastic) {
          code = __float2int_rn(y);
        } else {
          const float fl = floorf(y);
          const float frac = __fsub_rn(y, fl);
          const float u = unit_f(fmix64(z));
          code = static_cast<int>(fl) + (u < frac ? 1 : 0);
        }
        code = max(-L, min(L, code));
        bits |= (static_cast<uint64_t>(static_cast<uint32_t>(code)) & mask) << (t * qbits);
      }
    }
    uint8_t* dst = payload + st.code_dst + lg * qbits;
    if (qbits == 4) {
      *reinterpret_cast<uint32_t*>(dst) = static_cast<uint32_t>(bits);
    } else if (qbits == 8) {
      *reinterpret_cast<uint2*>(dst) = make_uint2(static_cast<uint32_t>(bits), static_cast<uint32_t>(bits >> 32));
    } else {
      for (int i = 0; i < qbits; ++i) dst[i] = static_cast<uint8_t>(bits >> (8 * i));
    }
    return;
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int64_t idx = lg * 8 + t;
    if (idx >= total) break;
    ++valid;
    const int64_t col = colw, row = roww;
    if (++roww == clen) {
      roww = 0;
      ++colw;
    }
    const int64_t c = st.chunk0 + col;
    int code = 0;
    if (cmax[c] != 0.f) {
      const float y = __fmul_rn(src[col * st.ld + row], inv[c]);
      if (!stochastic) {
        code = __float2int_rn(y);
      } else {
        const float fl = floorf(y);
        const float frac = __fsub_rn(y, fl);
        const float u = unit_f(draw_at(s0, static_cast<uint64_t>(base[c] + row + 1)));
        code = static_cast<int>(fl) + (u < frac ? 1 : 0);
      }
      code = max(-L, min(L, code));
    }
    bits |= (static_cast<uint64_t>(static_cast<uint32_t>(code)) & mask) << (t * qbits);
  }
  uint8_t* dst = payload + st.code_dst + lg * qbits;
  const int nbytes = valid == 8 ? qbits : (valid * qbits + 7) / 8;
  if (nbytes == 4 && qbits == 4) {
    *reinterpret_cast<uint32_t*>(dst) = static_cast<uint32_t>(bits);
  } else if (nbytes == 8) {
    *reinterpret_cast<uint2*>(dst) = make_uint2(static_cast<uint32_t>(bits), static_cast<uint32_t>(bits >> 32));
  } else {
    for (int i = 0; i < nbytes; ++i) dst[i] = static_cast<uint8_t>(bits >> (8 * i));
  }
}

void quantize_all(dlx_ctx* ctx, const Plan& P, const float* pbuf, const float* qbuf,
                  const float* slab, int rounding, uint64_t s0, int cold,
                  const int64_t* d_cold_base_used, uint8_t* payload, uint64_t* d_draws,
                  int* d_mismatch, int64_t* d_cold_base_actual, cudaStream_t s,
                  const uint64_t* s0p) {
  HostProf hp_("quantize_all");
  const int nc = static_cast<int>(P.chunks.size());
  if (nc == 0) {
    DLX_CUDA(cudaMemsetAsync(d_draws, 0, 8, s));
    return;
  }
  auto* cmax = static_cast<float*>(ctx->scratch("q_cmax", sizeof(float) * nc));
  auto* inv = static_cast<float*>(ctx->scratch("q_inv", sizeof(float) * nc));
  auto* base = static_cast<int64_t*>(ctx->scratch("q_base", sizeof(int64_t) * nc));
  k_chunk_max<<<nc, 256, 0, s>>>(P.d_chunks, pbuf, qbuf, slab, cmax);
  DLX_LAUNCHED();
  const int stochastic = rounding == 0 ? 1 : 0;
  k_chunk_scan<<<1, 1024, 0, s>>>(P.d_chunks, nc, cmax, (1 << (P.qbits - 1)) - 1, stochastic,
                                  cold, d_cold_base_used, base, inv,
                                  payload, d_draws, d_mismatch, d_cold_base_actual);
  DLX_LAUNCHED();
  const int64_t ng = P.ngroups;
  k_quant_pack<<<static_cast<unsigned>(ceil_div(ng, 256)), 256, 0, s>>>(
      P.d_streams, static_cast<int>(P.streams.size()), ng, base, inv, cmax, pbuf, qbuf, slab,
      P.qbits, stochastic, s0, s0p, payload);
  DLX_LAUNCHED();
}

// ------------------------------------------------------------------ dequantise factors
// phat / qhat: per 2-D slot k, column-major (ld = lda / ldb) with D*r columns; column
// w*r + j holds worker w's dequantised column j: float(code) * scale (one rounding).
__device__ __forceinline__ int sext(uint64_t bits, int t, int qbits) {
  const int u = static_cast<int>((bits >> (t * qbits)) & ((1ull << qbits) - 1ull));
  return (u & (1 << (qbits - 1))) ? u - (1 << qbits) : u;
}

__device__ __forceinline__ uint64_t load_group(const uint8_t* src, int qbits) {
  uint64_t bits = 0;
  for (int i = 0; i < qbits; ++i) bits |= static_cast<uint64_t>(src[i]) << (8 * i);
  return bits;
}

__global__ void __launch_bounds__(256) k_dequant(const DevStream* __restrict__ streams,
                                                 int nstreams, int64_t ngroups,
                                                 const DevT2* __restrict__ T,
                                                 const uint8_t* __restrict__ gathered,
                                                 int64_t pay_bytes, int qbits, int D,
                                                 float* __restrict__ phat,
                                                 float* __restrict__ qhat) {
  const int w = blockIdx.y;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  __shared__ int s_first;  // the block's first stream (see k_quant_pack)
  if (threadIdx.x == 0) {
    const int64_t g0 = blockIdx.x * (int64_t)blockDim.x;
    int lo = 0, hi = nstreams - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (streams[mid].group0 <= g0) lo = mid; else hi = mid - 1;
    }
    s_first = lo;
  }
  __syncthreads();
  if (g >= ngroups) return;
  int lo = s_first;
  while (lo + 1 < nstreams && streams[lo + 1].group0 <= g) ++lo;
  const DevStream st = streams[lo];
  if (st.t2 < 0) return;  // 1-D tensors are reconstructed in place by the 1-D kernels
  const DevT2 t = T[st.t2];
  const uint8_t* pay = gathered + w * pay_bytes;
  const int64_t lg = g - st.group0;
  const int64_t total = st.col_len * st.ncols;
  const uint64_t bits = load_group(pay + st.code_dst + lg * qbits, qbits);
  const int64_t sc_off = st.buf == 0 ? t.seg_ps : t.seg_qs;
  float* dst = (st.buf == 0 ? phat + D * t.poff : qhat + D * t.qoff);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t idx = lg * 8 + i;
    if (idx >= total) break;
    const int64_t col = idx / st.col_len, row = idx - col * st.col_len;
    const float scale = *reinterpret_cast<const float*>(pay + sc_off + 4 * col);
    dst[(w * t.r + col) * st.ld + row] = __fmul_rn(static_cast<float>(sext(bits, i, qbits)), scale);
  }
}

void dequant_factors(const Plan& P, int D, const uint8_t* gathered, int64_t pay_bytes,
                     float* phat, float* qhat, int64_t, cudaStream_t s) {
  if (P.t2.empty()) return;
  const int64_t ng = P.ngroups;
  k_dequant<<<dim3(static_cast<unsigned>(ceil_div(ng, 256)), D), 256, 0, s>>>(
      P.d_streams, static_cast<int>(P.streams.size()), ng, P.d_t2, gathered, pay_bytes, P.qbits,
      D, phat, qhat);
  DLX_LAUNCHED();
}

}  // namespace dlx
