// outer.cu — the fused outer update (K5): reconstruction of the averaged pseudo-gradient
// from the all-gathered factors + error feedback + delta staging + Nesterov, in one pass
// over the outer state, plus the reference-API dense helpers (decompress / allreduce_avg /
// stage_deltas / nesterov_outer_step).
//
// Reference semantics (bit-exact op order, -ffp-contract=off):
//   allreduce_avg        collective.cpp:17-46   Delta = float(sum_w double(dec_w) * (1/D))
//   error feedback       engine.cpp:254-257     e = delta_pending - Delta
//   stage_deltas         engine.cpp:266-276     delta = (anchor - local) + e   (pre-update anchor)
//   nesterov_outer_step  optim.cpp:56-78        v = beta v + Delta; anchor -= gamma (Delta + beta v)
// HBM traffic per element of a 2-D tensor: read pending, anchor, local, v; write pending,
// anchor, v = 28 B; Delta itself never touches HBM.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include <map>

#include "dlx_internal.cuh"
#include "ptx.cuh"
#include "epilogue.cuh"

namespace dlx {

__device__ __forceinline__ void stats_add(dlx_round_stats* st, double num, double den,
                                          double dn, double en, double nf, double* red) {
  // warp reduce then one atomic per warp (stats are diagnostics, not state)
  double v[5] = {num, den, dn, en, nf};
#pragma unroll
  for (int k = 0; k < 5; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  if ((threadIdx.x & 31) == 0 && st) {
    if (v[0] != 0.0) atomicAdd(&st->err_num, v[0]);
    if (v[1] != 0.0) atomicAdd(&st->err_den, v[1]);
    if (v[2] != 0.0) atomicAdd(&st->delta_norm_sq, v[2]);
    if (v[3] != 0.0) atomicAdd(&st->err_norm_sq, v[3]);
    if (v[4] != 0.0) atomicAdd(&st->nonfinite, v[4]);
  }
  (void)red;
}

// ------------------------------------------------------------------ K5, 2-D tensors
// Tile 16 rows x 128 cols of delta; 256 threads, each 2 rows x 4 consecutive cols.
// Delta_tile = (1/D) * Phat[rows, :] Qhat[cols, :]^T with K = D*r (fp32 accumulate).
// The four streamed operands of the tile are loaded (evict-first) before the small
// factor GEMM so their HBM latency overlaps it: 256 B in flight per thread.
__device__ __forceinline__ void load4(const float* p, bool full, int nv, float (&v)[4]) {
  if (full) {
    const float4 x = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = j < nv ? p[j] : 0.f;
  }
}

__device__ __forceinline__ void store4(float* p, bool full, int nv, const float (&v)[4]) {
  if (full) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < nv) p[j] = v[j];
  }
}

template <bool SELF>
__global__ void __launch_bounds__(256, 3) k5_outer(const DevT2* __restrict__ T,
                                                   const int4* __restrict__ tiles,
                                                   const float* __restrict__ phat,
                                                   const float* __restrict__ qhat, int D,
                                                   int self_index, int mode,
                                                   float* __restrict__ pending,
                                                   float* __restrict__ anchor,
                                                   const float* __restrict__ local,
                                                   float* __restrict__ velocity, float gamma,
                                                   float beta, int classical,
                                                   dlx_round_stats* stats) {
  // tile: 16 rows x 128 cols; thread (ty, tx) owns rows 2ty, 2ty+1 and cols 4tx..4tx+3
  __shared__ __align__(16) float Ps[32][20];
  __shared__ __align__(16) float Qs[32][132];
  const int4 tile = tiles[blockIdx.x];
  const DevT2 t = T[tile.x];
  const int64_t m0 = tile.y, n0 = tile.z;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int K = D * t.r;
  const float* Ph = phat + D * t.poff;
  const float* Qh = qhat + D * t.qoff;
  const int s_lo = SELF ? self_index * t.r : K, s_hi = s_lo + t.r;
  const bool vec = (t.b % 4) == 0;
  const bool ovl = mode == DLX_MODE_OVERLAPPED;
  const int64_t col = n0 + tx * 4;
  const int nv = col < t.b ? (int)(t.b - col < 4 ? t.b - col : 4) : 0;

  // 1. streamed operands of this thread's 2 rows (issued before the factor GEMM)
  float pd[2][4], an[2][4], lo[2][4], ve[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int64_t row = m0 + ty * 2 + i;
    const bool live = row < t.a && nv > 0;
    const int n = live ? nv : 0;
    const bool full = live && vec && nv == 4;
    const int64_t base = t.off + (live ? row * t.b + col : 0);
    load4(pending + base, full, n, pd[i]);
    load4(anchor + base, full, n, an[i]);
    if (ovl) {
      load4(local + base, full, n, lo[i]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) lo[i][j] = 0.f;
    }
    load4(velocity + base, full, n, ve[i]);
  }

  // 2. factor GEMM: acc = Phat[rows, :] Qhat[cols, :]^T
  float acc[2][4], sacc[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = sacc[i][j] = 0.f;
  for (int k0 = 0; k0 < K; k0 += 32) {
    if (tid < 128) {  // Phat 32(k) x 16(rows)
      const int kk = tid / 4, c4 = (tid % 4) * 4;
      const int k = k0 + kk;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k < K) v = *reinterpret_cast<const float4*>(Ph + (int64_t)k * t.lda + m0 + c4);
      *reinterpret_cast<float4*>(&Ps[kk][c4]) = v;
    }
#pragma unroll
    for (int l = 0; l < 4; ++l) {  // Qhat 32(k) x 128(cols)
      const int e = tid + 256 * l, kk = e / 32, c4 = (e % 32) * 4;
      const int k = k0 + kk;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k < K && n0 + c4 < t.ldb) v = *reinterpret_cast<const float4*>(Qh + (int64_t)k * t.ldb + n0 + c4);
      *reinterpret_cast<float4*>(&Qs[kk][c4]) = v;
    }
    __syncthreads();
    const int kmax = min(32, K - k0);
    for (int kk = 0; kk < kmax; ++kk) {
      const float2 a2 = *reinterpret_cast<const float2*>(&Ps[kk][ty * 2]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Qs[kk][tx * 4]);
      const float av[2] = {a2.x, a2.y}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      // own-payload terms (measure_error), accumulated separately so Delta's summation order
      // never depends on self_index (bitwise-identical Delta on every rank); at D = 1 the
      // own payload is the whole sum and sacc is taken from acc after the loop
      const int k = k0 + kk;
      if (SELF && D > 1 && k >= s_lo && k < s_hi) {  // CTA-uniform branch
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) sacc[i][j] = fmaf(av[i], bv[j], sacc[i][j]);
      }
    }
    __syncthreads();
  }

  if (SELF && D == 1) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) sacc[i][j] = acc[i][j];
  }

  // 3. fused epilogue
  const float invD = __fdiv_rn(1.0f, (float)D);
  double num = 0.0, den = 0.0, dn = 0.0, en = 0.0, nf = 0.0;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int64_t row = m0 + ty * 2 + i;
    if (row >= t.a || nv == 0) continue;
    const int64_t base = t.off + row * t.b + col;
    float op[4], oa[4], ov[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float delta = __fmul_rn(acc[i][j], invD);
      const EpiOut o = epilogue(delta, pd[i][j], an[i][j], lo[i][j], ve[i][j], mode, gamma, beta,
                                classical);
      op[j] = o.pend;
      oa[j] = o.anchor;
      ov[j] = o.v;
      if (j < nv) {
        if (SELF) {
          const double df = (double)sacc[i][j] - (double)pd[i][j];
          num += df * df;
          den += (double)pd[i][j] * (double)pd[i][j];
        }
        en += (double)o.e * (double)o.e;
        if (ovl) dn += (double)o.pend * (double)o.pend;
        if (!isfinite(o.anchor)) nf += 1.0;
      }
    }
    const bool full = vec && nv == 4;
    store4(pending + base, full, nv, op);
    store4(anchor + base, full, nv, oa);
    store4(velocity + base, full, nv, ov);
  }
  stats_add(stats, num, den, dn, en, nf, nullptr);
}

// ------------------------------------------------------------------ K5s: persistent, streamed
// One CTA per SM loops over 16 x 128 tiles (ordered column-block-major so the Qhat tile is
// reused across consecutive tiles). Warp 8 streams the tile's four operand boxes
// (pending, anchor, velocity, local; 16 rows x 512 B each) into a 4-stage shared-memory ring
// with one TMA tensor copy per operand (mbarrier complete_tx); warps 0-7 compute
// the factor GEMM for the tile while the copies land, then run the fused epilogue from
// shared memory and store the three outputs (evict-first). Up to 4 x 32 KB of operand
// traffic is in flight per SM.
constexpr int kK5Stages = 5;
constexpr int kK5StreamBytes = 16 * 128 * 4;               // one operand box: 16 rows x 128
constexpr int kK5StageBytes = 4 * kK5StreamBytes + 32 * 16 * 4;  // 4 operands + Phat tile

struct K5Maps {
  // pending, anchor, velocity, local: dims {b, a}, box {128, 16};
  // [4] = this tensor's dequantised left factors Phat: dims {lda, D*r}, box {16, 32}
  CUtensorMap m[5];
};

// Contiguous tile chunk of this CTA (tiles are column-block-major, so consecutive tiles share
// the Qhat block and it is loaded once per block).
__device__ __forceinline__ void k5_chunk(int ntiles, int& t0, int& t1) {
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  t0 = blockIdx.x * per;
  t1 = min(ntiles, t0 + per);
}

template <bool SELF>
__global__ void __launch_bounds__(288, 1) k5s_outer(const DevT2* __restrict__ T,
                                                    const K5Maps* __restrict__ maps,
                                                    const int4* __restrict__ tiles, int ntiles,
                                                    const float* __restrict__ phat,
                                                    const float* __restrict__ qhat, int D,
                                                    int self_index, int mode, int ps_tma,
                                                    float* __restrict__ pending,
                                                    float* __restrict__ anchor,
                                                    const float* __restrict__ local,
                                                    float* __restrict__ velocity, float gamma,
                                                    float beta, int classical,
                                                    dlx_round_stats* stats) {
  extern __shared__ __align__(128) uint8_t k5smem[];
  float* ring = reinterpret_cast<float*>(k5smem);  // [stage]{[stream][16][128], Ps[32][16]}
  float* Qs = reinterpret_cast<float*>(k5smem + kK5Stages * kK5StageBytes);  // [32][132]
  float* Pg = Qs + 32 * 132;                                                // [32][20]
  uint64_t* full = reinterpret_cast<uint64_t*>(Pg + 32 * 20);
  uint64_t* empty = full + kK5Stages;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const bool ovl = mode == DLX_MODE_OVERLAPPED;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kK5Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);  // one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int t_begin, t_end;
  k5_chunk(ntiles, t_begin, t_end);

  if (warp == 8) {
    // ------------------------------------------------------------ producer (TMA)
    if (lane == 0) {
      uint32_t it = 0;
      for (int ti = t_begin; ti < t_end; ++ti, ++it) {
        const int4 tl = tiles[ti];
        const int s = it % kK5Stages;
        mbar_wait(&empty[s], ((it / kK5Stages) & 1) ^ 1);
        const int nstreams = ovl ? 4 : 3;
        mbar_expect_tx(&full[s], kK5StreamBytes * nstreams + (ps_tma ? 32 * 16 * 4 : 0));
        float* st = ring + s * (kK5StageBytes / 4);
        const K5Maps* mp = maps + tl.x;
        for (int q = 0; q < nstreams; ++q)
          tma_load_2d(st + q * 16 * 128, &mp->m[q], &full[s], tl.z, tl.y);
        if (ps_tma) tma_load_2d(st + 4 * 16 * 128, &mp->m[4], &full[s], tl.y, 0);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers (8 warps)
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  double num = 0.0, den = 0.0, dn = 0.0, en = 0.0, nf = 0.0;
  const float invD = __fdiv_rn(1.0f, (float)D);
  int cached_slot = -1, cached_n0 = -1;
  uint32_t it = 0;
  for (int ti = t_begin; ti < t_end; ++ti, ++it) {
    const int4 tl = tiles[ti];
    const DevT2 t = T[tl.x];
    const int64_t m0 = tl.y, n0 = tl.z;
    const int K = D * t.r;
    const float* Ph = phat + D * t.poff;
    const float* Qh = qhat + D * t.qoff;
    const int s_lo = SELF ? self_index * t.r : K, s_hi = s_lo + t.r;
    const int s = it % kK5Stages;
    const float* st = ring + s * (kK5StageBytes / 4);
    float acc[2][4], sacc[2][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = sacc[i][j] = 0.f;
    const bool one_chunk = K <= 32;
    const bool reuse_q = one_chunk && tl.x == cached_slot && n0 == cached_n0;
    for (int k0 = 0; k0 < K; k0 += 32) {
      const float* Ps;
      int pstride;
      if (!(reuse_q && ps_tma)) {
        named_bar(1, 256);  // previous users of Pg / Qs are done
        if (!ps_tma && tid < 128) {
          const int kk = tid / 4, c4 = (tid % 4) * 4;
          const int k = k0 + kk;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (k < K) v = *reinterpret_cast<const float4*>(Ph + (int64_t)k * t.lda + m0 + c4);
          *reinterpret_cast<float4*>(&Pg[kk * 20 + c4]) = v;
        }
        if (!reuse_q) {
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            const int e = tid + 256 * l, kk = e / 32, c4 = (e % 32) * 4;
            const int k = k0 + kk;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (k < K && n0 + c4 < t.ldb)
              v = *reinterpret_cast<const float4*>(Qh + (int64_t)k * t.ldb + n0 + c4);
            *reinterpret_cast<float4*>(&Qs[kk * 132 + c4]) = v;
          }
        }
        named_bar(1, 256);
      }
      if (ps_tma) {
        if (k0 == 0) mbar_wait(&full[s], (it / kK5Stages) & 1);
        Ps = st + 4 * 16 * 128;  // [k][16] from the TMA box
        pstride = 16;
      } else {
        Ps = Pg;
        pstride = 20;
      }
      const int kmax = min(32, K - k0);
      for (int kk = 0; kk < kmax; ++kk) {
        const float2 a2 = *reinterpret_cast<const float2*>(&Ps[kk * pstride + ty * 2]);
        const float4 b4 = *reinterpret_cast<const float4*>(&Qs[kk * 132 + tx * 4]);
        const float av[2] = {a2.x, a2.y}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        // own-payload terms (measure_error), accumulated separately so Delta's summation order
        // never depends on self_index (bitwise-identical Delta on every rank); at D = 1 the
        // own payload is the whole sum and sacc is taken from acc after the loop
        const int k = k0 + kk;
        if (SELF && D > 1 && k >= s_lo && k < s_hi) {  // CTA-uniform branch
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) sacc[i][j] = fmaf(av[i], bv[j], sacc[i][j]);
        }
      }
    }
    cached_slot = tl.x;
    cached_n0 = static_cast<int>(n0);
    if (SELF && D == 1) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) sacc[i][j] = acc[i][j];
    }

    // epilogue from the landed stage
    if (!ps_tma) mbar_wait(&full[s], (it / kK5Stages) & 1);
    const int64_t col = n0 + tx * 4;
    const int nv = col < t.b ? (int)(t.b - col < 4 ? t.b - col : 4) : 0;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int r = ty * 2 + i;
      const int64_t row = m0 + r;
      float pd[4] = {0.f, 0.f, 0.f, 0.f}, an[4] = {0.f, 0.f, 0.f, 0.f},
            ve[4] = {0.f, 0.f, 0.f, 0.f}, lo[4] = {0.f, 0.f, 0.f, 0.f};
      const bool live = row < t.a && nv > 0;
      if (live) {
        const float4 a = *reinterpret_cast<const float4*>(st + (0 * 16 + r) * 128 + tx * 4);
        const float4 b = *reinterpret_cast<const float4*>(st + (1 * 16 + r) * 128 + tx * 4);
        const float4 c = *reinterpret_cast<const float4*>(st + (2 * 16 + r) * 128 + tx * 4);
        pd[0] = a.x; pd[1] = a.y; pd[2] = a.z; pd[3] = a.w;
        an[0] = b.x; an[1] = b.y; an[2] = b.z; an[3] = b.w;
        ve[0] = c.x; ve[1] = c.y; ve[2] = c.z; ve[3] = c.w;
        if (ovl) {
          const float4 d = *reinterpret_cast<const float4*>(st + (3 * 16 + r) * 128 + tx * 4);
          lo[0] = d.x; lo[1] = d.y; lo[2] = d.z; lo[3] = d.w;
        }
      }
      float op[4], oa[4], ov[4];
      float fnum = 0.f, fden = 0.f, fen = 0.f, fdn = 0.f;  // per-row partials (fp32), folded
      int bad = 0;                                         // into fp64 once per row
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float delta = __fmul_rn(acc[i][j], invD);
        const EpiOut o = epilogue(delta, pd[j], an[j], lo[j], ve[j], mode, gamma, beta, classical);
        op[j] = o.pend;
        oa[j] = o.anchor;
        ov[j] = o.v;
        if (live && j < nv) {
          if (SELF) {
            const float df = sacc[i][j] - pd[j];
            fnum = fmaf(df, df, fnum);
            fden = fmaf(pd[j], pd[j], fden);
          }
          fen = fmaf(o.e, o.e, fen);
          if (ovl) fdn = fmaf(o.pend, o.pend, fdn);
          bad |= !isfinite(o.anchor);
        }
      }
      num += fnum;
      den += fden;
      en += fen;
      dn += fdn;
      nf += bad;
      if (live) {
        const int64_t base = t.off + row * t.b + col;
        const bool full4 = nv == 4;
        store4(pending + base, full4, nv, op);
        store4(anchor + base, full4, nv, oa);
        store4(velocity + base, full4, nv, ov);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  stats_add(stats, num, den, dn, en, nf, nullptr);
}

static PFN_cuTensorMapEncodeTiled_v12000 k5_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    DLX_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) raise(DLX_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

using K5MapCache = MapTableCache<K5Maps, 6>;

static const K5Maps* k5_maps(const Plan& P, int D, const float* pending, const float* anchor,
                             const float* velocity, const float* local, const float* phat,
                             cudaStream_t s) {
  K5MapCache& c = plan_ext<K5MapCache>(P, "k5_maps");
  const void* key[6] = {pending, anchor, velocity, local, phat, reinterpret_cast<const void*>(static_cast<intptr_t>(D))};
  return c.get(key, P.t2.size(), s, [&](K5Maps* h) {
  for (size_t k = 0; k < P.t2.size(); ++k) {
    const DevT2& t = P.t2[k];
    if (t.b % 4 != 0) continue;
    for (int q = 0; q < 4; ++q) {
      if (!key[q]) continue;
      const cuuint64_t dims[2] = {static_cast<cuuint64_t>(t.b), static_cast<cuuint64_t>(t.a)};
      const cuuint64_t strides[1] = {static_cast<cuuint64_t>(t.b) * 4};
      const cuuint32_t box[2] = {128, 16};
      const cuuint32_t estr[2] = {1, 1};
      CUresult r = k5_encode_fn()(&h[k].m[q], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                  const_cast<float*>(static_cast<const float*>(key[q])) + t.off,
                                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) raise(DLX_ERR_CUDA, "cuTensorMapEncodeTiled (K5) failed");
    }
    if (D * t.r <= 32) {  // Phat tile map (box 16 rows x 32 factor columns)
      const cuuint64_t dims[2] = {static_cast<cuuint64_t>(t.lda), static_cast<cuuint64_t>(D * t.r)};
      const cuuint64_t strides[1] = {static_cast<cuuint64_t>(t.lda) * 4};
      const cuuint32_t box[2] = {16, 32};
      const cuuint32_t estr[2] = {1, 1};
      CUresult r = k5_encode_fn()(&h[k].m[4], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                  const_cast<float*>(phat) + D * t.poff, dims, strides, box, estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) raise(DLX_ERR_CUDA, "cuTensorMapEncodeTiled (K5 Phat) failed");
    }
  }
  });
}

static size_t k5s_smem() {
  return kK5Stages * kK5StageBytes + (32 * 132 + 32 * 20) * 4 + 2 * kK5Stages * 8 + 64;
}

bool o5_eligible(const Plan& P, int D, int self_index);
void launch_outer_2d_tc(dlx_ctx* ctx, const Plan& P, int D, const uint8_t* gathered,
                        int self_index, int mode, float* pending, float* anchor,
                        const float* local, float* velocity, float gamma, float beta,
                        int classical, dlx_round_stats* stats, const SlotRange& R,
                        cudaStream_t s);

SlotRange slot_range(const Plan& P, int t_begin, int t_end) {
  SlotRange R;
  auto lo2 = [&](int t) {
    int k = 0;
    while (k < static_cast<int>(P.t2.size()) && P.t2[k].idx < t) ++k;
    return k;
  };
  auto lo1 = [&](int t) {
    int k = 0;
    while (k < static_cast<int>(P.t1.size()) && P.t1[k].idx < t) ++k;
    return k;
  };
  R.s0 = lo2(t_begin);
  R.s1 = lo2(t_end);
  R.u0 = lo1(t_begin);
  R.u1 = lo1(t_end);
  return R;
}

// SIMT K5 tiles of a slot range, built on first use of the SIMT outer update (the tcgen05
// path never needs them): (t2 slot, m0, n0, -); the streamed kernel's list is
// column-block-major, the register kernel's (b % 4 != 0) row-block-major.
struct K5RangeTiles : PlanExt {
  std::vector<int4> k5s, k5;
  int4* d_k5s = nullptr;
  int4* d_k5 = nullptr;
};

bool& option_outer_tc() {
  static bool on = [] {
    const char* e = getenv("DLX_OUTER_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

void launch_outer_2d_impl(dlx_ctx* ctx, const Plan& P, int D, const uint8_t* gathered,
                          int self_index, int mode, float* pending, float* anchor,
                          const float* local, float* velocity, float gamma, float beta,
                          int classical, dlx_round_stats* stats, const SlotRange& R,
                          cudaStream_t s);
void launch_outer_2d(dlx_ctx* ctx, const Plan& P, int D, const uint8_t* gathered,
                     int self_index, int mode, float* pending, float* anchor,
                     const float* local, float* velocity, float gamma, float beta,
                     int classical, dlx_round_stats* stats, const SlotRange& R, cudaStream_t s) {
  HostProf hp("outer_update_2d");
  launch_outer_2d_impl(ctx, P, D, gathered, self_index, mode, pending, anchor, local, velocity,
                       gamma, beta, classical, stats, R, s);
}
void launch_outer_2d_impl(dlx_ctx* ctx, const Plan& P, int D, const uint8_t* gathered,
                     int self_index, int mode, float* pending, float* anchor,
                     const float* local, float* velocity, float gamma, float beta,
                     int classical, dlx_round_stats* stats, const SlotRange& R,
                     cudaStream_t s) {
  if (P.t2.empty() || R.s1 <= R.s0) return;
  if (option_outer_tc() && o5_eligible(P, D, self_index)) {
    launch_outer_2d_tc(ctx, P, D, gathered, self_index, mode, pending, anchor, local, velocity,
                       gamma, beta, classical, stats, R, s);
    return;
  }
  bool fresh = false;
  K5RangeTiles& T = plan_ext<K5RangeTiles>(P, "k5_range:" + R.key(), &fresh);
  if (fresh) {
    for (int k = R.s0; k < R.s1; ++k) {
      const DevT2& t = P.t2[k];
      if (t.b % 4 == 0) {
        for (int64_t n0 = 0; n0 < t.b; n0 += 128)
          for (int64_t m0 = 0; m0 < t.a; m0 += 16)
            T.k5s.push_back(make_int4(k, static_cast<int>(m0), static_cast<int>(n0), 0));
      } else {
        for (int64_t m0 = 0; m0 < t.a; m0 += 16)
          for (int64_t n0 = 0; n0 < t.b; n0 += 128)
            T.k5.push_back(make_int4(k, static_cast<int>(m0), static_cast<int>(n0), 0));
      }
    }
    T.d_k5s = plan_upload(P, T.k5s);
    T.d_k5 = plan_upload(P, T.k5);
  }
  const std::vector<int4>* k5s_tiles = &T.k5s;
  const std::vector<int4>* k5_tiles = &T.k5;
  const int4* d_k5s_tiles = T.d_k5s;
  const int4* d_k5_tiles = T.d_k5;
  float* phat = static_cast<float*>(ctx->scratch("phat", sizeof(float) * P.pelems * D));
  float* qhat = static_cast<float*>(ctx->scratch("qhat", sizeof(float) * P.qelems * D));
  dequant_factors(P, D, gathered, P.payload_bytes, phat, qhat, 0, s);
  if (!k5s_tiles->empty()) {
    smem_optin(reinterpret_cast<const void*>(k5s_outer<true>), (int)k5s_smem());
    smem_optin(reinterpret_cast<const void*>(k5s_outer<false>), (int)k5s_smem());
    int sms = 0, dev = 0;
    DLX_CUDA(cudaGetDevice(&dev));
    DLX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int n = static_cast<int>(k5s_tiles->size());
    const int grid = std::min(n, sms);
    const K5Maps* maps = k5_maps(P, D, pending, anchor, velocity,
                                 mode == DLX_MODE_OVERLAPPED ? local : nullptr, phat, s);
    const int ps_tma = D * P.rmax <= 32 ? 1 : 0;
    if (self_index >= 0)
      k5s_outer<true><<<grid, 288, k5s_smem(), s>>>(P.d_t2, maps, d_k5s_tiles, n, phat, qhat, D,
                                                    self_index, mode, ps_tma, pending, anchor, local,
                                                    velocity, gamma, beta, classical, stats);
    else
      k5s_outer<false><<<grid, 288, k5s_smem(), s>>>(P.d_t2, maps, d_k5s_tiles, n, phat, qhat, D,
                                                     self_index, mode, ps_tma, pending, anchor, local,
                                                     velocity, gamma, beta, classical, stats);
    DLX_LAUNCHED();
  }
  if (!k5_tiles->empty()) {
    if (self_index >= 0)
      k5_outer<true><<<k5_tiles->size(), 256, 0, s>>>(P.d_t2, d_k5_tiles, phat, qhat, D,
                                                       self_index, mode, pending, anchor, local,
                                                       velocity, gamma, beta, classical, stats);
    else
      k5_outer<false><<<k5_tiles->size(), 256, 0, s>>>(P.d_t2, d_k5_tiles, phat, qhat, D,
                                                        self_index, mode, pending, anchor, local,
                                                        velocity, gamma, beta, classical, stats);
    DLX_LAUNCHED();
  }
}

// ------------------------------------------------------------------ 1-D tensors
__device__ __forceinline__ int code_at(const uint8_t* seg, int64_t k, int qbits) {
  const int64_t bit = k * qbits;
  const uint32_t w = static_cast<uint32_t>(seg[bit >> 3]) |
                     (static_cast<uint32_t>(seg[(bit >> 3) + 1]) << 8);
  const int u = static_cast<int>((w >> (bit & 7)) & ((1u << qbits) - 1u));
  return (u & (1 << (qbits - 1))) ? u - (1 << qbits) : u;
}

// Delta of a 1-D tensor exactly as allreduce_avg: dequantise (fp32 product), sum in
// double over workers in order, multiply by 1/D in double, round once.
__device__ __forceinline__ float avg_1d(const uint8_t* gathered, int64_t pay_bytes,
                                        const DevT1& t, int64_t k, int D, int qbits) {
  double acc = 0.0;
  for (int w = 0; w < D; ++w) {
    const uint8_t* pay = gathered + w * pay_bytes;
    const float sc = *reinterpret_cast<const float*>(pay + t.seg_s);
    acc = __dadd_rn(acc, (double)__fmul_rn((float)code_at(pay + t.seg_c, k, qbits), sc));
  }
  return (float)__dmul_rn(acc, 1.0 / (double)D);
}

constexpr int kOuter1dElems = 1024;  // elements per k_outer_1d block (4 per thread)

// One block per 1024-element chunk of a 1-D tensor (host-built chunk table), block-reduced
// stats: one atomic per statistic per block.
__global__ void __launch_bounds__(256) k_outer_1d(const DevT1* __restrict__ T,
                                                  const int2* __restrict__ chunks,
                                                  const uint8_t* __restrict__ gathered,
                                                  int64_t pay_bytes, int qbits, int D,
                                                  int self_index, int mode, float* pending,
                                                  float* anchor, const float* local,
                                                  float* velocity, float gamma, float beta,
                                                  int classical, dlx_round_stats* stats) {
  const int2 ch = chunks[blockIdx.x];  // (tensor, first element)
  const DevT1 t = T[ch.x];
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // num, den, delta_norm, err_norm, nonfinite
#pragma unroll
  for (int u = 0; u < kOuter1dElems / 256; ++u) {
    const int64_t k = ch.y + u * 256 + threadIdx.x;
    if (k >= t.n) break;
    const float delta = avg_1d(gathered, pay_bytes, t, k, D, qbits);
    const int64_t i = t.off + k;
    const float pd = pending[i];
    const EpiOut o = epilogue(delta, pd, anchor[i], mode == DLX_MODE_OVERLAPPED ? local[i] : 0.f,
                              velocity[i], mode, gamma, beta, classical);
    if (self_index >= 0) {
      const uint8_t* pay = gathered + self_index * pay_bytes;
      const float rec = __fmul_rn((float)code_at(pay + t.seg_c, k, qbits),
                                  *reinterpret_cast<const float*>(pay + t.seg_s));
      const double df = (double)rec - (double)pd;
      v[0] += df * df;
      v[1] += (double)pd * (double)pd;
    }
    v[3] += (double)o.e * (double)o.e;
    if (mode == DLX_MODE_OVERLAPPED) v[2] += (double)o.pend * (double)o.pend;
    if (!isfinite(o.anchor)) v[4] += 1.0;
    pending[i] = o.pend;
    anchor[i] = o.anchor;
    velocity[i] = o.v;
  }
  __shared__ double red[8][5];
#pragma unroll
  for (int q = 0; q < 5; ++q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  }
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int q = 0; q < 5; ++q) red[threadIdx.x >> 5][q] = v[q];
  __syncthreads();
  if (threadIdx.x == 0 && stats) {
    double sum[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int w = 0; w < 8; ++w)
      for (int q = 0; q < 5; ++q) sum[q] += red[w][q];
    if (sum[0] != 0.0) atomicAdd(&stats->err_num, sum[0]);
    if (sum[1] != 0.0) atomicAdd(&stats->err_den, sum[1]);
    if (sum[2] != 0.0) atomicAdd(&stats->delta_norm_sq, sum[2]);
    if (sum[3] != 0.0) atomicAdd(&stats->err_norm_sq, sum[3]);
    if (sum[4] != 0.0) atomicAdd(&stats->nonfinite, sum[4]);
  }
}

void launch_outer_1d(const Plan& P, int D, const uint8_t* gathered, int self_index, int mode,
                     float* pending, float* anchor, const float* local, float* velocity,
                     float gamma, float beta, int classical, dlx_round_stats* stats,
                     const SlotRange& R, cudaStream_t s) {
  if (P.t1.empty() || R.u1 <= R.u0) return;
  struct Chunks1d : PlanExt {
    int2* d = nullptr;
    int n = 0;
  };
  bool fresh = false;
  Chunks1d& tb = plan_ext<Chunks1d>(P, "outer_1d:" + R.key(), &fresh);
  if (fresh) {
    std::vector<int2> ch;
    for (size_t i = R.u0; i < static_cast<size_t>(R.u1); ++i)
      for (int64_t k = 0; k < P.t1[i].n; k += kOuter1dElems)
        ch.push_back(make_int2(static_cast<int>(i), static_cast<int>(k)));
    tb.d = plan_upload(P, ch);
    tb.n = static_cast<int>(ch.size());
  }
  if (tb.n == 0) return;
  k_outer_1d<<<tb.n, 256, 0, s>>>(P.d_t1, tb.d, gathered, P.payload_bytes, P.qbits, D,
                                       self_index, mode, pending, anchor, local, velocity, gamma,
                                       beta, classical, stats);
  DLX_LAUNCHED();
}

// ------------------------------------------------------------------ no-compress ablation
// dilocox-no-compress (compress_raw compress.cpp:185-199): the payload is the raw fp32 delta,
// allreduce_avg = float(sum over workers ascending of double(x_w) * (1/D)) — reference-exact
// — then the same fused epilogue. Elementwise over the whole slab (padding is zero).
__global__ void __launch_bounds__(256) k_outer_raw(int64_t n, const float* __restrict__ gathered,
                                                   int64_t slab, int D, int self_index, int mode,
                                                   float* pending, float* anchor,
                                                   const float* local, float* velocity,
                                                   float gamma, float beta, int classical,
                                                   dlx_round_stats* stats) {
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const double inv = 1.0 / (double)D;
  const bool ovl = mode == DLX_MODE_OVERLAPPED;
  // float4 lanes (the slab is a multiple of 64 elements, 256-B aligned)
  for (int64_t i4 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i4 < n / 4;
       i4 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = 4 * i4;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int w = 0; w < D; ++w) {
      const float4 g = __ldcs(reinterpret_cast<const float4*>(gathered + w * slab + i));
      acc[0] = __dadd_rn(acc[0], (double)g.x);
      acc[1] = __dadd_rn(acc[1], (double)g.y);
      acc[2] = __dadd_rn(acc[2], (double)g.z);
      acc[3] = __dadd_rn(acc[3], (double)g.w);
    }
    const float4 p4 = *reinterpret_cast<const float4*>(pending + i);
    const float4 a4 = *reinterpret_cast<const float4*>(anchor + i);
    const float4 v4 = *reinterpret_cast<const float4*>(velocity + i);
    const float4 l4 = ovl ? __ldcs(reinterpret_cast<const float4*>(local + i)) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float pd[4] = {p4.x, p4.y, p4.z, p4.w}, an[4] = {a4.x, a4.y, a4.z, a4.w};
    const float ve[4] = {v4.x, v4.y, v4.z, v4.w}, lo[4] = {l4.x, l4.y, l4.z, l4.w};
    float op[4], oa[4], ov[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float delta = (float)__dmul_rn(acc[j], inv);
      const EpiOut o = epilogue(delta, pd[j], an[j], lo[j], ve[j], mode, gamma, beta, classical);
      if (self_index >= 0) {  // measure_error: the raw payload reconstructs exactly
        const double df = (double)gathered[self_index * slab + i + j] - (double)pd[j];
        v[0] += df * df;
        v[1] += (double)pd[j] * (double)pd[j];
      }
      v[3] += (double)o.e * (double)o.e;
      if (ovl) v[2] += (double)o.pend * (double)o.pend;
      if (!isfinite(o.anchor)) v[4] += 1.0;
      op[j] = o.pend;
      oa[j] = o.anchor;
      ov[j] = o.v;
    }
    *reinterpret_cast<float4*>(pending + i) = make_float4(op[0], op[1], op[2], op[3]);
    *reinterpret_cast<float4*>(anchor + i) = make_float4(oa[0], oa[1], oa[2], oa[3]);
    *reinterpret_cast<float4*>(velocity + i) = make_float4(ov[0], ov[1], ov[2], ov[3]);
  }
  stats_add(stats, v[0], v[1], v[2], v[3], v[4], nullptr);
}

void launch_outer_raw(const dlx_layout& L, int D, const float* gathered, int self_index, int mode,
                      float* pending, float* anchor, const float* local, float* velocity,
                      float gamma, float beta, int classical, dlx_round_stats* stats,
                      cudaStream_t s) {
  int dev = 0, sms = 0;
  DLX_CUDA(cudaGetDevice(&dev));
  DLX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (L.slab % 4 != 0) raise(DLX_ERR_VALIDATION, "outer_update_raw: slab not a multiple of 4");
  // algorithmic bytes: D gathered slabs + pending, anchor, velocity, local read; 3 written
  // (at D = 1 the single gathered slab is usually the pending buffer itself: read once)
  const int reads = D + (mode == DLX_MODE_OVERLAPPED ? 4 : 3) - (gathered == pending ? 1 : 0);
  KernelTimer timer("k_outer_raw", 4.0 * L.slab * (reads + 3), s);
  k_outer_raw<<<sms * 8, 256, 0, s>>>(L.slab, gathered, L.slab, D, self_index, mode, pending,
                                      anchor, local, velocity, gamma, beta, classical, stats);
  DLX_LAUNCHED();
}

// ------------------------------------------------------------------ dense reconstruction
// Reference-exact decompress / allreduce_avg (fp64 accumulation over ascending k per
// worker, float per worker, double sum over workers, * 1/D, float): bit-identical output.
__global__ void __launch_bounds__(256) k_recon_2d(const DevT2* __restrict__ T, int nt2,
                                                  const float* __restrict__ phat,
                                                  const float* __restrict__ qhat, int D,
                                                  float* __restrict__ out) {
  const DevT2 t = T[blockIdx.z];
  const int64_t j = blockIdx.x * 32 + (threadIdx.x & 31);
  const int64_t i = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (i >= t.a || j >= t.b) return;
  const float* Ph = phat + D * t.poff;
  const float* Qh = qhat + D * t.qoff;
  double total = 0.0;
  for (int w = 0; w < D; ++w) {
    double acc = 0.0;
    for (int k = 0; k < t.r; ++k) {
      const int c = w * t.r + k;
      acc = fma((double)Ph[(int64_t)c * t.lda + i], (double)Qh[(int64_t)c * t.ldb + j], acc);
    }
    total = __dadd_rn(total, (double)(float)acc);
  }
  out[t.off + i * t.b + j] = (float)__dmul_rn(total, 1.0 / (double)D);
}

__global__ void k_recon_1d(const DevT1* __restrict__ T, const uint8_t* __restrict__ gathered,
                           int64_t pay_bytes, int qbits, int D, float* __restrict__ out) {
  const DevT1 t = T[blockIdx.y];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < t.n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[t.off + k] = avg_1d(gathered, pay_bytes, t, k, D, qbits);
}

void launch_reconstruct_dense(dlx_ctx* ctx, const Plan& P, int D, const uint8_t* gathered,
                              float* out, cudaStream_t s) {
  if (!P.t2.empty()) {
    float* phat = static_cast<float*>(ctx->scratch("phat", sizeof(float) * P.pelems * D));
    float* qhat = static_cast<float*>(ctx->scratch("qhat", sizeof(float) * P.qelems * D));
    dequant_factors(P, D, gathered, P.payload_bytes, phat, qhat, 0, s);
    int64_t ma = 1, mb = 1;
    for (const DevT2& t : P.t2) {
      ma = std::max(ma, t.a);
      mb = std::max(mb, t.b);
    }
    k_recon_2d<<<dim3(ceil_div(mb, 32), ceil_div(ma, 8), P.t2.size()), 256, 0, s>>>(
        P.d_t2, (int)P.t2.size(), phat, qhat, D, out);
    DLX_LAUNCHED();
  }
  if (!P.t1.empty()) {
    int64_t mx = 1;
    for (const DevT1& t : P.t1) mx = std::max(mx, t.n);
    k_recon_1d<<<dim3(std::min<int64_t>(ceil_div(mx, 256), 64), P.t1.size()), 256, 0, s>>>(
        P.d_t1, gathered, P.payload_bytes, P.qbits, D, out);
    DLX_LAUNCHED();
  }
}

// ------------------------------------------------------------------ stage / nesterov
struct Span {
  int64_t off, n;
};

__global__ void __launch_bounds__(256) k_stage(const Span* __restrict__ spans,
                                               const float* __restrict__ anchor,
                                               const float* __restrict__ local, const float* err,
                                               float* pending, double* norm_sq) {
  const Span sp = spans[blockIdx.y];
  double ss = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < sp.n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = sp.off + k;
    const float e = err ? err[i] : 0.0f;
    const float d = __fadd_rn(__fsub_rn(anchor[i], local[i]), e);  // ps_sub then ps_add
    pending[i] = d;
    ss += (double)d * (double)d;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0 && norm_sq && ss != 0.0) atomicAdd(norm_sq, ss);
}

// Device table of the layout's tensor spans (slab offset, element count), built once per
// layout; returns it and the longest span.
static const Span* layout_spans(const dlx_layout& L, int64_t* longest) {
  std::vector<Span> spans(L.nt);
  int64_t mx = 1;
  for (int i = 0; i < L.nt; ++i) {
    spans[i] = {L.offsets[i], L.numel(i)};
    mx = std::max(mx, spans[i].n);
  }
  Span* d = static_cast<Span*>(L.d_spans);
  if (!d) {
    DLX_CUDA(cudaMalloc(&d, sizeof(Span) * L.nt));
    upload_now(d, spans.data(), sizeof(Span) * L.nt);
    const_cast<dlx_layout&>(L).d_spans = d;
  }
  *longest = mx;
  return d;
}

void launch_stage(const dlx_layout& L, const float* anchor, const float* local,
                  const float* err, float* pending, double* norm_sq, cudaStream_t s) {
  if (L.nt == 0) return;
  int64_t mx = 1;
  const Span* d = layout_spans(L, &mx);
  const int gx = static_cast<int>(std::min<int64_t>(ceil_div(mx, 256), 1024));
  k_stage<<<dim3(gx, L.nt), 256, 0, s>>>(d, anchor, local, err, pending, norm_sq);
  DLX_LAUNCHED();
}

// measure_error (compress.cpp:246-262): out[0] += sum (rec - delta)^2, out[1] += sum delta^2
// over the layout's tensor elements, in fp64 (block partial sums; the summation order is not
// the reference's serial one, so the ratio agrees to ~1e-15 relative, not bit for bit).
__global__ void __launch_bounds__(256) k_sqdiff(const Span* __restrict__ spans,
                                                const float* __restrict__ rec,
                                                const float* __restrict__ delta,
                                                double* out) {
  const Span sp = spans[blockIdx.y];
  double num = 0.0, den = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < sp.n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double d = (double)delta[sp.off + k];
    const double diff = (double)rec[sp.off + k] - d;
    num += diff * diff;
    den += d * d;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  __shared__ double sn[8], sd[8];
  if ((threadIdx.x & 31) == 0) {
    sn[threadIdx.x >> 5] = num;
    sd[threadIdx.x >> 5] = den;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < 8; ++w) {
      a += sn[w];
      b += sd[w];
    }
    if (a != 0.0) atomicAdd(out, a);
    if (b != 0.0) atomicAdd(out + 1, b);
  }
}

void launch_sqdiff(const dlx_layout& L, const float* rec, const float* delta, double* out,
                   cudaStream_t s) {
  if (L.nt == 0) return;
  int64_t mx = 1;
  const Span* d = layout_spans(L, &mx);
  const int gx = static_cast<int>(std::min<int64_t>(ceil_div(mx, 256), 512));
  k_sqdiff<<<dim3(gx, L.nt), 256, 0, s>>>(d, rec, delta, out);
  DLX_LAUNCHED();
}

// Worker-order fp64 mean of D slabs (leading dimension ld): allreduce_avg of RawDense
// payloads (collective.cpp:17-46 over compress_raw, compress.cpp:185-199) and the per-step
// gradient mean of the all-reduce baseline (engine.cpp:559-570): double sum in worker order,
// times the double 1/D, rounded to float once — bit-identical to the reference.
__global__ void __launch_bounds__(256) k_mean_slabs(int64_t n, int64_t ld,
                                                    const float* __restrict__ x, int D,
                                                    float* __restrict__ out) {
  const double inv = 1.0 / (double)D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = (double)x[i];
    for (int w = 1; w < D; ++w) acc = __dadd_rn(acc, (double)x[(int64_t)w * ld + i]);
    out[i] = (float)__dmul_rn(acc, inv);
  }
}

void launch_mean_slabs(int64_t n, int64_t ld, const float* x, int D, float* out,
                       cudaStream_t s) {
  if (n <= 0) return;
  const int g = static_cast<int>(std::min<int64_t>(ceil_div(n, 256), 148 * 16));
  k_mean_slabs<<<g, 256, 0, s>>>(n, ld, x, D, out);
  DLX_LAUNCHED();
}

__global__ void __launch_bounds__(256) k_nesterov(int64_t n, float gamma, float beta,
                                                  int classical, float* anchor, float* v,
                                                  const float* __restrict__ delta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const EpiOut o = epilogue(delta[i], 0.f, anchor[i], 0.f, v[i], DLX_MODE_SYNC, gamma, beta,
                              classical);
    anchor[i] = o.anchor;
    v[i] = o.v;
  }
}

void launch_nesterov(int64_t n, float gamma, float beta, int classical, float* anchor,
                     float* v, const float* delta, cudaStream_t s) {
  if (n <= 0) return;
  const int g = static_cast<int>(std::min<int64_t>(ceil_div(n, 256), 148 * 16));
  k_nesterov<<<g, 256, 0, s>>>(n, gamma, beta, classical, anchor, v, delta);
  DLX_LAUNCHED();
}

}  // namespace dlx
