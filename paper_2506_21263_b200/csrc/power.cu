// power.cu — synthetic inputs, cold-start init, and the power-iteration GEMMs
// (lowrank_approx compress.cpp:56-78):  Y = delta Q  (K1)   and   Z = delta^T P  (K2).
//
// delta is a x b row-major fp32 (slab); P (a x r) and Q (b x r) are column-major with
// padded column strides. Both sweeps are HBM-bound for r <~ 80 (2r flops per 4 B of
// delta); each delta element is read exactly once per sweep. Accumulation is fp32 with a
// fixed per-thread order (deterministic; the reference accumulates in fp64, tolerance).
#include <cstdlib>

#include "dlx_internal.cuh"

namespace dlx {

// --------------------------------------------------------------- synthetic gaussian fill
struct TensorSpan {
  int64_t off, n;
};

__global__ void k_fill_gaussian(const TensorSpan* spans, float* out, const float* base,
                                float scale, uint64_t seed, uint64_t tag, uint64_t worker) {
  const int t = blockIdx.y;
  const TensorSpan sp = spans[t];
  // RngStream(seed, stream_key({tag, worker, t})) (rng.hpp:13-16, 63-66)
  uint64_t h = 0x100000001b3ull;
  h = mix64(h ^ mix64(tag));
  h = mix64(h ^ mix64(worker));
  h = mix64(h ^ mix64(static_cast<uint64_t>(t)));
  const uint64_t s0 = stream_init(seed, h);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < sp.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    // element i consumes draws 12i+1 .. 12i+12 (Tensor::gaussian, rng.hpp:52-56)
    double s = 0.0;
#pragma unroll
    for (int k = 1; k <= 12; ++k) s = __dadd_rn(s, unit_d(draw_at(s0, 12ull * i + k)));
    const float g = (float)__dadd_rn(s, -6.0);
    const float v = __fmul_rn(scale, g);
    out[sp.off + i] = base ? __fadd_rn(base[sp.off + i], v) : v;
  }
}

void launch_fill_gaussian(const dlx_layout& L, float* out, const float* base, float scale,
                          uint64_t seed, uint64_t tag, uint64_t worker, cudaStream_t s) {
  if (L.nt == 0) return;
  std::vector<TensorSpan> spans(L.nt);
  int64_t maxn = 1;
  for (int i = 0; i < L.nt; ++i) {
    spans[i] = {L.offsets[i], L.numel(i)};
    maxn = std::max(maxn, spans[i].n);
  }
  auto* d = static_cast<TensorSpan*>(L.ctx->scratch("fill_spans", sizeof(TensorSpan) * L.nt));
  DLX_CUDA(cudaMemcpyAsync(d, spans.data(), sizeof(TensorSpan) * L.nt, cudaMemcpyHostToDevice, s));
  const int gx = static_cast<int>(std::min<int64_t>(ceil_div(maxn, 256), 1024));
  k_fill_gaussian<<<dim3(gx, L.nt), 256, 0, s>>>(d, out, base, scale, seed, tag, worker);
  DLX_LAUNCHED();
  // the spans upload is pageable; keep it alive until the copy has been consumed
  DLX_CUDA(cudaStreamSynchronize(s));
}

// --------------------------------------------------------------- cold start (compress.cpp:64-69)
// Q0 = uniform(-1, 1)^{b x r} row-major from the shared stream at the tensor's draw base,
// stored column-major. Value = lo + (hi - lo) * u with separate roundings (rng.hpp:39).
// One block per 256 runs of one tensor: blk0[k] = first block of tensor k (prefix over the
// tensors' run counts), found by binary search (a max-work x tensors grid launched 74752
// mostly empty blocks for OPT-1.3B; same time — the 64-bit integer hash is the cost)
__global__ void __launch_bounds__(256) k_cold_init(const DevT2* T, int nt2,
                                                   const int* __restrict__ blk0, float* q,
                                                   const int64_t* bases, uint64_t s0,
                                                   const uint64_t* s0p) {
  if (s0p) s0 = *s0p;
  int lo = 0, hi = nt2 - 1;  // last k with blk0[k] <= blockIdx.x
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (blk0[mid] <= static_cast<int>(blockIdx.x)) lo = mid; else hi = mid - 1;
  }
  const int k = lo;
  const DevT2 t = T[k];
  const uint64_t base = static_cast<uint64_t>(bases[k]);
  // walk the column-major destination in runs of 8 rows (coalesced stores); element (i, j)
  // is row-major draw i * r + j of the tensor's init (Tensor::uniform, tensor.cpp:43-47), so
  // down a run the draw counter steps by r * gamma (one 64-bit multiply per run, not per
  // element: the integer pipe bounds this kernel)
  const uint32_t runs = static_cast<uint32_t>((t.b + 7) / 8);
  const int64_t total = static_cast<int64_t>(runs) * t.r;
  const uint64_t step = static_cast<uint64_t>(t.r) * kGolden;
  const int64_t e = static_cast<int64_t>(blockIdx.x - blk0[k]) * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const uint32_t j = static_cast<uint32_t>(e) / runs;
  const uint32_t i0 = 8 * (static_cast<uint32_t>(e) - j * runs);
  uint64_t z = s0 + (base + static_cast<uint64_t>(i0) * t.r + j + 1) * kGolden;
  float* dst = q + t.qoff + static_cast<int64_t>(j) * t.ldb + i0;
#pragma unroll
  for (int u8 = 0; u8 < 8; ++u8, z += step) {
    if (i0 + u8 >= t.b) break;
    const float u = unit_f(fmix64(z));
    dst[u8] = __fadd_rn(-1.0f, __fmul_rn(2.0f, u));
  }
}

void launch_cold_init(const Plan& P, float* q, const int64_t* d_bases, uint64_t s0,
                      cudaStream_t s, const uint64_t* s0p) {
  if (P.t2.empty()) return;
  struct ColdBlocks : PlanExt {
    int* d = nullptr;
    int total = 0;
  };
  bool fresh = false;
  ColdBlocks& cb = plan_ext<ColdBlocks>(P, "cold_init_blocks", &fresh);
  if (fresh) {
    std::vector<int> blk0;
    int acc = 0;
    for (const DevT2& t : P.t2) {
      blk0.push_back(acc);
      acc += static_cast<int>(ceil_div(ceil_div(t.b, 8) * t.r, 256));
    }
    cb.d = plan_upload(P, blk0);
    cb.total = acc;
  }
  if (cb.total == 0) return;
  k_cold_init<<<cb.total, 256, 0, s>>>(P.d_t2, (int)P.t2.size(), cb.d, q, d_bases, s0, s0p);
  DLX_LAUNCHED();
}

// --------------------------------------------------------------- K1: Y = delta * Q
constexpr int kBK = 32;

template <int BM, int BN>
__global__ void __launch_bounds__(256) k1_gemm(const DevT2* __restrict__ T,
                                               const int4* __restrict__ tiles,
                                               const float* __restrict__ slab,
                                               const float* __restrict__ qbuf,
                                               float* __restrict__ ybuf) {
  constexpr int TX = BN / 4, TY = 256 / TX, TM = BM / TY;
  static_assert(TM == 4, "4x4 register tile");
  __shared__ __align__(16) float As[kBK][BM + 4];
  __shared__ __align__(16) float Bs[kBK][BN + 4];
  const int4 tile = tiles[blockIdx.x];
  const DevT2 t = T[tile.x];
  const int64_t m0 = tile.y;
  const int n0 = tile.z;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const float* A = slab + t.off;
  const float* Q = qbuf + t.qoff;
  const bool vec = (t.b % 4) == 0;
  float acc[TM][4];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int64_t k0 = 0; k0 < t.b; k0 += kBK) {
    // delta tile BM x 32 -> As[k][m]
#pragma unroll
    for (int l = 0; l < BM * 8 / 256; ++l) {
      const int e = tid + 256 * l, row = e / 8, c4 = (e % 8) * 4;
      const int64_t gm = m0 + row, gk = k0 + c4;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (gm < t.a) {
        const float* src = A + gm * t.b + gk;
        if (vec && gk + 3 < t.b) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(src));
          v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = (gk + q < t.b) ? __ldg(src + q) : 0.f;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) As[c4 + q][row] = v[q];
    }
    // Q tile 32 x BN -> Bs[k][n]
#pragma unroll
    for (int l = 0; l < BN * 8 / 256; ++l) {
      const int e = tid + 256 * l, col = e / 8, c4 = (e % 8) * 4;
      const int gn = n0 + col;
      const int64_t gk = k0 + c4;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (gn < t.r) {
        const float* src = Q + gn * t.ldb + gk;
        if (gk + 3 < t.b) {
          const float4 x = *reinterpret_cast<const float4*>(src);
          v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = (gk + q < t.b) ? src[q] : 0.f;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) Bs[c4 + q][col] = v[q];
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < kBK; ++kk) {
      const float4 a4 = *reinterpret_cast<const float4*>(&As[kk][ty * TM]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float av[4] = {a4.x, a4.y, a4.z, a4.w}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* Y = ybuf + t.poff;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int gn = n0 + tx * 4 + j;
    if (gn >= t.r) continue;
    const int64_t gm = m0 + ty * TM;
    float* dst = Y + gn * t.lda + gm;
    if (gm + 3 < t.a) {
      *reinterpret_cast<float4*>(dst) = make_float4(acc[0][j], acc[1][j], acc[2][j], acc[3][j]);
    } else {
#pragma unroll
      for (int i = 0; i < TM; ++i)
        if (gm + i < t.a) dst[i] = acc[i][j];
    }
  }
}

bool& option_tensor_cores() {
  static bool on = [] {
    const char* e = getenv("DLX_TENSOR_CORES");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool use_tc(const Plan& P) { return option_tensor_cores() && tc_supported(P); }

void launch_k1(const Plan& P, const float* slab, const float* q, float* y, cudaStream_t s) {
  HostProf hp_("launch_k1");
  const bool tc = use_tc(P);
  if (tc) launch_k1_tc(P, slab, q, y, s);
  const std::vector<int4>& tiles = tc ? P.k1_rest : P.k1_tiles;
  const int4* d_tiles = tc ? P.d_k1_rest : P.d_k1_tiles;
  if (tiles.empty()) return;
  const int n = static_cast<int>(tiles.size());
  if (P.rmax <= 32)
    k1_gemm<128, 32><<<n, 256, 0, s>>>(P.d_t2, d_tiles, slab, q, y);
  else
    k1_gemm<64, 64><<<n, 256, 0, s>>>(P.d_t2, d_tiles, slab, q, y);
  DLX_LAUNCHED();
}

// --------------------------------------------------------------- K2: Z = delta^T * P
// Tile: 64 columns of delta (rows of Z) x BC factor columns, over one 2048-row k split.
template <int BC>
__global__ void __launch_bounds__(256) k2_gemm(const DevT2* __restrict__ T,
                                               const int4* __restrict__ tiles,
                                               const int* __restrict__ splits,
                                               const int64_t* __restrict__ part_off,
                                               const float* __restrict__ slab,
                                               const float* __restrict__ pbuf,
                                               float* __restrict__ zbuf,
                                               float* __restrict__ part) {
  constexpr int TX = BC / 4, TY = 256 / TX, TM = 64 / TY;
  constexpr int64_t KC = 2048;
  __shared__ __align__(16) float As[kBK][64 + 4];
  __shared__ __align__(16) float Bs[kBK][BC + 4];
  const int4 tile = tiles[blockIdx.x];
  const DevT2 t = T[tile.x];
  const int64_t j0 = tile.y;
  const int c0 = tile.z, sp = tile.w;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const float* A = slab + t.off;
  const float* Pf = pbuf + t.poff;
  const bool vec = (t.b % 4) == 0;
  const int64_t i_begin = sp * KC, i_end = min(t.a, i_begin + KC);
  float acc[TM][4];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int64_t i0 = i_begin; i0 < i_end; i0 += kBK) {
    // delta rows i0..i0+31, cols j0..j0+63 -> As[k][j]
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      const int e = tid + 256 * l, kk = e / 16, c4 = (e % 16) * 4;
      const int64_t gi = i0 + kk, gj = j0 + c4;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (gi < i_end) {
        const float* src = A + gi * t.b + gj;
        if (vec && gj + 3 < t.b) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(src));
          v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = (gj + q < t.b) ? __ldg(src + q) : 0.f;
        }
      }
      *reinterpret_cast<float4*>(&As[kk][c4]) = make_float4(v[0], v[1], v[2], v[3]);
    }
    // P rows i0..i0+31, cols c0..c0+BC-1 -> Bs[k][c]
#pragma unroll
    for (int l = 0; l < BC * 8 / 256; ++l) {
      const int e = tid + 256 * l, col = e / 8, c4 = (e % 8) * 4;
      const int gc = c0 + col;
      const int64_t gi = i0 + c4;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (gc < t.r) {
        const float* src = Pf + gc * t.lda + gi;
        if (gi + 3 < i_end) {
          const float4 x = *reinterpret_cast<const float4*>(src);
          v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = (gi + q < i_end) ? src[q] : 0.f;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) Bs[c4 + q][col] = v[q];
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < kBK; ++kk) {
      float av[TM];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[kk][ty * TM + i];
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  const int ns = splits[tile.x];
  float* Z = ns > 1 ? part + part_off[tile.x] + sp * (t.ldb * t.r) : zbuf + t.qoff;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int gc = c0 + tx * 4 + j;
    if (gc >= t.r) continue;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int64_t gj = j0 + ty * TM + i;
      if (gj < t.b) Z[gc * t.ldb + gj] = acc[i][j];
    }
  }
}

// Deterministic split-K reduction: Z = sum_s part[s] in split order.
__global__ void k2_reduce(const DevT2* __restrict__ T, const int* __restrict__ slots,
                          const int* __restrict__ splits, const int64_t* __restrict__ part_off,
                          const float* __restrict__ part, float* __restrict__ zbuf) {
  const int k = slots[blockIdx.y];
  const DevT2 t = T[k];
  const int ns = splits[k];
  const int64_t total = t.ldb * t.r;
  const float* src = part + part_off[k];
  // 4 consecutive rows per thread (ldb is a multiple of 32, so a 4-row group never straddles
  // a column): one 32-bit division per group instead of a 64-bit modulo per element, 16-B
  // loads, and the splits summed in split order (deterministic) from loads issued together
  const int ldb = static_cast<int>(t.ldb), b = static_cast<int>(t.b);
  const int n4 = static_cast<int>(total / 4);
  for (int e4 = blockIdx.x * blockDim.x + threadIdx.x; e4 < n4; e4 += gridDim.x * blockDim.x) {
    const int e = 4 * e4;
    const int row = e - (e / ldb) * ldb;
    if (row >= b) continue;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int q = 0;
    for (; q + 4 <= ns; q += 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = *reinterpret_cast<const float4*>(src + (q + u) * total + e);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x += v[u].x;
        acc.y += v[u].y;
        acc.z += v[u].z;
        acc.w += v[u].w;
      }
    }
    for (; q < ns; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(src + q * total + e);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    float* dst = zbuf + t.qoff + e;
    if (row + 4 <= b) {
      *reinterpret_cast<float4*>(dst) = acc;
    } else {  // the column's last rows: only those below b
      const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
      for (int i = 0; i < b - row; ++i) dst[i] = a4[i];
    }
  }
}

void launch_k2(const Plan& P, const float* slab, const float* p, float* z, float* part,
               cudaStream_t s) {
  HostProf hp_("launch_k2");
  if (P.k2_tiles.empty()) return;
  const bool tc = use_tc(P);
  if (tc) launch_k2_tc(P, slab, p, z, part, s);
  const std::vector<int4>& tiles = tc ? P.k2_rest : P.k2_tiles;
  const int4* d_tiles = tc ? P.d_k2_rest : P.d_k2_tiles;
  const int n = static_cast<int>(tiles.size());
  if (n > 0) {
    if (P.rmax <= 32)
      k2_gemm<32><<<n, 256, 0, s>>>(P.d_t2, d_tiles, P.d_k2_splits, P.d_k2_part_off, slab, p, z,
                                    part);
    else
      k2_gemm<64><<<n, 256, 0, s>>>(P.d_t2, d_tiles, P.d_k2_splits, P.d_k2_part_off, slab, p, z,
                                    part);
    DLX_LAUNCHED();
  }
  // split slots (static per plan): cache the list in a device arena keyed by the plan
  std::vector<int> slots;
  int64_t mx = 1;
  for (size_t k = 0; k < P.t2.size(); ++k)
    if (P.k2_splits[k] > 1) {
      slots.push_back(static_cast<int>(k));
      mx = std::max(mx, P.t2[k].ldb * P.t2[k].r);
    }
  if (slots.empty()) return;
  struct Slots : PlanExt {
    int* d = nullptr;
  };
  bool fresh = false;
  Slots& sl = plan_ext<Slots>(P, "k2_reduce", &fresh);
  if (fresh) sl.d = plan_upload(P, slots);
  int* d = sl.d;
  const int gx = static_cast<int>(std::min<int64_t>(ceil_div(mx, 256), 1024));
  k2_reduce<<<dim3(gx, slots.size()), 256, 0, s>>>(P.d_t2, d, P.d_k2_splits, P.d_k2_part_off,
                                                  part, z);
  DLX_LAUNCHED();
}

}  // namespace dlx
