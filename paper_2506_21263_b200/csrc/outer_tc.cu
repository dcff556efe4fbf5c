// outer_tc.cu — K5 on the tensor cores: the fused outer update (reconstruct + error feedback +
// staging + Nesterov, engine.cpp:254-276 / optim.cpp:56-78) with the averaged
// pseudo-gradient tile computed by tcgen05 into TMEM and every streamed operand moved by TMA.
//
// Tile = 128 rows x 32 columns of a 2-D tensor. Delta_tile = A B^T with
//   A[m][k] = float(code_P(w, m, j))                       (k = w r + j; exact in tf32)
//   B[n][k] = float(code_Q(w, n, j)) * s_P(w, j) s_Q(w, j) / D   (split hi + lo)
// i.e. sum_k (c_p s_p)(c_q s_q) / D with the scales folded onto one side so A is exact and
// only B needs the 2-term tf32 split (2 MMAs per k step). Differs from the reference's
// per-factor rounding (dequantize_columns then matmul_nt) at the 1e-7 relative level.
//
// Per CTA (persistent, contiguous balanced chunk of tiles ordered band-major so the A band
// stays in shared memory): warp 0 = TMA producer, warp 1 = MMA issuer, warps 2-9 =
// epilogue (TMEM -> registers, operands from the swizzled stage, outputs written back into
// the stage and TMA-stored). Two stream stages (pending, anchor, velocity, local + B), two
// A-band buffers and two TMEM accumulators keep loads, MMAs and epilogues overlapped.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "dlx_internal.cuh"
#include "ptx.cuh"
#include "epilogue.cuh"

namespace dlx {

constexpr int kO5Threads = 320;     // tf32 path: producer, MMA, 8 epilogue warps
constexpr int kO5ThreadsTA = 384;   // fp16 / TMEM-A path: + B-operand and A-band loader warps
constexpr int kO5MaxBRing = 4;
constexpr int kO5MaxStages = 6;
constexpr int kO5TileN = 16;                          // tile = 128 rows x 16 columns
constexpr uint32_t kO5StreamBox = 128 * kO5TileN * 4;  // 8 KB per streamed operand (SW64)
constexpr uint32_t kO5ABox = 128 * 128;               // 16 KB: 128 rows x 128 B of K (SW128)
constexpr uint32_t kO5BBox = kO5TileN * 128;          // 2 KB: 16 rows x 128 B of K (SW128)

// Operand kinds of the factor GEMM. K = D r <= 32: tf32, A exact, B = hi + lo (2 MMAs per
// k-step of 8). K > 32 (more workers): fp16 (kind::f16), A exact (|code| <= 127), B
// prescaled per tensor by a power of two (k_o5_escale) and split hi + lo (22 significant
// bits, as the tf32 pair; 2 MMAs per k-step of 16) — half the operand bytes per K of tf32,
// and two planes instead of three bf16 ones, so K = 256 (D = 8 at r = 32) keeps 5 stages.
template <bool BF>
struct O5Kind {
  static constexpr int ES = BF ? 2 : 4;    // bytes per operand element
  static constexpr int AK = 128 / ES;      // K elements per 128-B swizzle atom row
  static constexpr int KS = BF ? 16 : 8;   // MMA K per instruction (32 B)
  static constexpr int NBP = 2;            // B planes (hi + lo)
};

// Per-tensor TMA descriptors, split by what they depend on: the four parameter streams
// depend only on the state buffers (shared by every rank's plan of a layout), the operand
// maps on the rank (K) and the staging buffers.
struct O5StreamMaps {
  CUtensorMap s[4];  // pending, anchor, velocity, local: dims {b, a}, box {16, 128}, SW64
};
struct O5OpMaps {
  CUtensorMap a;     // A (codes of P): dims {KA, lda}, box {AK, 128}, SW128
  CUtensorMap b[2];  // B planes: dims {KA, ldb}, box {AK, 16}, SW128
};

// ------------------------------------------------------------------ prep: A and B operands
template <bool BF>
constexpr int prep_rows() { return BF ? 32 : 64; }  // factor rows per k_o5_prep block

// K columns per worker in the A / B operands: with D > 1 every worker's r columns start on
// an MMA K-step boundary (zero-padded to a multiple of kpad), so the worker's own k-steps
// (the measure_error accumulator) never straddle a neighbour's columns, whatever r is.
__host__ __device__ __forceinline__ int o5_rpad(int r, int D, int kpad) {
  return D > 1 ? (r + kpad - 1) / kpad * kpad : r;
}
// operand kind: tf32 (A band in shared memory) while the padded K fits one 32-wide band,
// fp16 with A in TMEM above
inline bool o5_bf(int rmax, int D) { return D * o5_rpad(rmax, D, 8) > 32; }

// fp16 path: per-tensor power-of-two prescale of B = code_Q s_P s_Q / D, chosen so that
// max |B| 2^e lies in [2^14, 2^15): both fp16 planes stay in range and the scaling is exact
// (undone on the fp32 accumulator in the epilogue). pre = 2^e, post = 2^-e per 2-D slot.
__global__ void __launch_bounds__(256) k_o5_escale(const DevT2* __restrict__ T,
                                                   const uint8_t* __restrict__ gathered,
                                                   int64_t pay_bytes, int qbits, int D,
                                                   float* __restrict__ pre,
                                                   float* __restrict__ post) {
  const DevT2& t = T[blockIdx.x];
  __shared__ float red[8];
  float m = 0.f;
  for (int i = threadIdx.x; i < D * t.r; i += 256) {
    const int w = i / t.r, j = i % t.r;
    const uint8_t* pay = gathered + w * pay_bytes;
    const float sp = *reinterpret_cast<const float*>(pay + t.seg_ps + 4 * j);
    const float sq = *reinterpret_cast<const float*>(pay + t.seg_qs + 4 * j);
    m = fmaxf(m, fabsf(sp * sq));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < 8; ++i) m = fmaxf(m, red[i]);
    const float mb = m * static_cast<float>((1 << (qbits - 1)) - 1) / static_cast<float>(D);
    int e = 0;
    if (mb > 0.f && isfinite(mb)) e = min(max(14 - ilogbf(mb), -120), 120);
    pre[blockIdx.x] = ldexpf(1.f, e);
    post[blockIdx.x] = ldexpf(1.f, -e);
  }
}

// Block = 64 consecutive factor rows: codes are decoded column by column (coalesced over
// rows), staged in shared memory, and written row-major [row][KA] with coalesced stores.
// A = code of P (exact); B = code_Q * s_P * s_Q / D split into NBP planes.
template <bool BF>
__global__ void __launch_bounds__(256) k_o5_prep(
    const DevT2* __restrict__ T, const int4* __restrict__ rows, int nrows,
    const int64_t* __restrict__ aoff, const int64_t* __restrict__ boff,
    const uint8_t* __restrict__ gathered, int64_t pay_bytes, int qbits, int D, int KA, int kpad,
    const float* __restrict__ pre, void* __restrict__ A_, void* __restrict__ B0_,
    void* __restrict__ B1_) {
  float* A = static_cast<float*>(A_);
  float* Bp[2] = {static_cast<float*>(B0_), static_cast<float*>(B1_)};
  constexpr int kPrepRows = prep_rows<BF>();
  __shared__ float tile[kPrepRows][BF ? 257 : 65];
  const int64_t g0 = static_cast<int64_t>(blockIdx.x) * kPrepRows;
  const float invD = __fdiv_rn(1.0f, (float)D);
  // phase 1, task = (K column k, 8-row group): the group's 8 codes are one <= 64-bit field of
  // the column-major factor (segments are 32-row aligned, so groups never straddle one)
  const uint32_t* words = reinterpret_cast<const uint32_t*>(gathered);
  const int64_t nwords = D * pay_bytes / 4;
  const uint32_t mask = (1u << qbits) - 1u;
  const int sh = 32 - qbits;
  constexpr int kGroups = kPrepRows / 8;
  __shared__ int64_t dst_off[kPrepRows];  // element offset of each row's [KA] run; side in bit 62
  if (threadIdx.x < kPrepRows) {
    const int64_t g = g0 + threadIdx.x;
    int64_t o = -1;
    if (g < nrows) {
      const int4 rw = rows[g];
      o = (rw.y == 0 ? aoff[rw.x] : boff[rw.x]) + static_cast<int64_t>(rw.z) * KA;
      if (rw.y != 0) o |= int64_t(1) << 62;
    }
    dst_off[threadIdx.x] = o;
  }
  for (int task = threadIdx.x; task < KA * kGroups; task += 256) {
    const int k = task / kGroups, grp = task % kGroups;
    const int64_t g = g0 + 8 * grp;
    float* dst = &tile[8 * grp][k];
    if (g >= nrows) continue;
    const int4 rw = rows[g];  // (slot, side, row, -) of the group's first row
    const DevT2& t = T[rw.x];
    const int side = rw.y, row0 = rw.z;
    const int64_t n = side == 0 ? t.a : t.b;
    const int rp = o5_rpad(t.r, D, kpad);
    const int w = k / rp, j = k % rp;
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (w < D && j < t.r && row0 < n) {
      const uint8_t* pay = gathered + w * pay_bytes;
      const int64_t bit = (w * pay_bytes + (side == 0 ? t.seg_pc : t.seg_qc)) * 8 +
                          ((int64_t)j * n + row0) * qbits;
      const int64_t wi = bit >> 5;
      const int s = static_cast<int>(bit & 31);
      // only the words the 8 codes touch (q = 4 groups are one aligned word)
      const int span = s + 8 * qbits;
      const uint32_t w0 = words[wi];
      const uint32_t w1 = (span > 32 && wi + 1 < nwords) ? words[wi + 1] : 0u;
      const uint32_t w2 = (span > 64 && wi + 2 < nwords) ? words[wi + 2] : 0u;
      const uint64_t lo = static_cast<uint64_t>(w0) | (static_cast<uint64_t>(w1) << 32);
      const uint64_t f = (lo >> s) | (s ? (static_cast<uint64_t>(w2) << (64 - s)) : 0ull);
      float scale = 1.f, ps = 1.f;
      if (side != 0) {
        const float sp = *reinterpret_cast<const float*>(pay + t.seg_ps + 4 * j);
        const float sq = *reinterpret_cast<const float*>(pay + t.seg_qs + 4 * j);
        scale = __fmul_rn(__fmul_rn(sp, sq), invD);
        if (BF) ps = pre[rw.x];  // power of two: exact
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (row0 + i >= n) break;
        const int c = static_cast<int>((static_cast<uint32_t>(f >> (i * qbits)) & mask) << sh) >> sh;
        v[i] = side == 0 ? static_cast<float>(c)
                         : __fmul_rn(__fmul_rn(static_cast<float>(c), scale), ps);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) dst[i * (BF ? 257 : 65)] = v[i];
  }
  __syncthreads();
  if constexpr (BF) {
    // 8 consecutive k of one row per thread -> one 16-B store per plane; the 8 reads of a
    // lane are rotated by (lane / 4) so a warp's reads of one step hit 32 distinct banks
    const int kg_n = KA / 8;
    for (int e = threadIdx.x; e < kPrepRows * kg_n; e += 256) {
      const int rl = e / kg_n, kg = e - rl * kg_n;
      const int64_t dof = dst_off[rl];
      if (dof < 0) break;
      const int rot = (threadIdx.x & 31) >> 2;
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int ii = (i + rot) & 7;
        v[ii] = tile[rl][8 * kg + ii];
      }
      if (!(dof >> 62)) {  // A: codes, exact in fp16
        uint4 pk;
        uint32_t* w = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const __half2 h2 = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
          w[i] = *reinterpret_cast<const uint32_t*>(&h2);
        }
        *reinterpret_cast<uint4*>(reinterpret_cast<__half*>(A_) + dof + 8 * kg) = pk;
      } else {  // B (prescaled): hi = fp16(v), lo = fp16(v - hi) (v - hi exact in fp32)
        const int64_t o = (dof & ((int64_t(1) << 62) - 1)) + 8 * kg;
        uint4 ph, pl;
        uint32_t* wh = reinterpret_cast<uint32_t*>(&ph);
        uint32_t* wl = reinterpret_cast<uint32_t*>(&pl);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const __half2 h2 = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
          const __half2 l2 = __floats2half2_rn(v[2 * i] - __low2float(h2),
                                               v[2 * i + 1] - __high2float(h2));
          wh[i] = *reinterpret_cast<const uint32_t*>(&h2);
          wl[i] = *reinterpret_cast<const uint32_t*>(&l2);
        }
        *reinterpret_cast<uint4*>(reinterpret_cast<__half*>(Bp[0]) + o) = ph;
        *reinterpret_cast<uint4*>(reinterpret_cast<__half*>(Bp[1]) + o) = pl;
      }
    }
  } else {  // tf32: A exact, B = hi + lo; 4 consecutive k per thread -> 16-B stores (row
            // starts are 16-B aligned: KA is a multiple of 32 floats)
    const int kq_n = KA / 4;
    for (int e = threadIdx.x; e < kPrepRows * kq_n; e += 256) {
      const int rl = e / kq_n, k = 4 * (e - rl * kq_n);
      const int64_t dof = dst_off[rl];
      if (dof < 0) break;
      const float4 v = make_float4(tile[rl][k], tile[rl][k + 1], tile[rl][k + 2], tile[rl][k + 3]);
      if (!(dof >> 62)) {
        *reinterpret_cast<float4*>(A + dof + k) = v;
      } else {
        const int64_t o = (dof & ((int64_t(1) << 62) - 1)) + k;
        const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
        *reinterpret_cast<float4*>(Bp[0] + o) = h;
        *reinterpret_cast<float4*>(Bp[1] + o) = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
      }
    }
  }
}

// ------------------------------------------------------------------ the kernel
// 16-column tiles keep 4-5 stages (36 KB each at K = 32) in flight per SM while one is in
// the epilogue, so the HBM stream does not stall behind a stage that is being written back.
// fp16 path: the B tile (16 columns x K x 2 planes: 16 KB at K = 256) moves through its own
// ring, filled by a dedicated warp that follows the stage descriptors; the stream stages then
// carry only the four 8-KB parameter boxes, so more of them fit (the HBM stream runs further
// ahead) and the MMA of a tile no longer waits for that tile's stream data.
template <bool SELF, bool BF>
__global__ void __launch_bounds__(BF ? kO5ThreadsTA : kO5Threads, 1)
    k_o5(const DevT2* __restrict__ T, const O5StreamMaps* __restrict__ smaps,
         const O5OpMaps* __restrict__ omaps,
         const int4* __restrict__ bands, int nbands, int* __restrict__ band_ctr, int D, int KA,
         int nst, int nab, int nbr, int a_mode, int self_index, int mode, float gamma,
         float beta, int classical, const float* __restrict__ post, dlx_round_stats* stats) {
  using KD = O5Kind<BF>;
  extern __shared__ __align__(1024) uint8_t o5smem[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(o5smem) + 1023) & ~uintptr_t(1023));
  const int nkc = KA / KD::AK;                             // 128-B K chunks
  // bf16 path: A moves through a ring of nab 16-KB boxes into TMEM (tcgen05.cp) and the MMAs
  // read it from there, B through its own ring of nbr slots; tf32 path: nab whole A bands
  // stay in shared memory and B rides in the stream stage
  constexpr bool TA = BF;
  const uint32_t bslot_bytes = KD::NBP * nkc * kO5BBox;
  const uint32_t stage_bytes = 4 * kO5StreamBox + (TA ? 0u : bslot_bytes);
  const uint32_t aband_bytes = TA ? kO5ABox : nkc * kO5ABox;
  uint8_t* bring = smem + nst * stage_bytes;
  uint8_t* abuf = bring + (TA ? nbr * bslot_bytes : 0u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(abuf + nab * aband_bytes);
  uint64_t* sfull = bars;                // [nst]
  uint64_t* sempty = sfull + nst;        // [nst]
  uint64_t* afull = sempty + nst;        // [nab <= 4]
  uint64_t* aempty = afull + 4;          // [nab <= 4]
  uint64_t* accfull = aempty + 4;        // [2]
  uint64_t* accempty = accfull + 2;      // [2]
  uint64_t* tinfo = accempty + 2;        // [nst] stage descriptor written (TA)
  uint64_t* bfull = tinfo + kO5MaxStages;     // [nbr] (TA)
  uint64_t* bempty = bfull + kO5MaxBRing;     // [nbr] (TA)
  uint64_t* adone = bempty + kO5MaxBRing;     // [2] MMAs reading a TMEM A slot done (TA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(adone + 2);
  // TA: who issues the A boxes — 0 the stream producer (after a chunk's first tile), 1 the B
  // warp, 2 a dedicated warp (11); bit 2: the MMA warp drains the next chunk's boxes into
  // the other TMEM slot as they land instead of at the chunk's first tile
  const int a_src = a_mode & 3;
  const bool a_early = (a_mode & 4) != 0;
  // per-stage tile descriptor written by the producer before the stage's arrive:
  // (t2 slot or -1 = end, row m0, column n0, A slot | 2 first-of-band | 4 last-of-band)
  int4* sinfo = reinterpret_cast<int4*>(tmem_slot + 4);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const bool ovl = mode == DLX_MODE_OVERLAPPED;
  const int nstreams = ovl ? 4 : 3;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], 1);
      mbar_init(&tinfo[i], 1);
    }
    for (int i = 0; i < nbr; ++i) {
      mbar_init(&bfull[i], 1);
      mbar_init(&bempty[i], 1);
    }
    for (int i = 0; i < nab; ++i) {
      mbar_init(&afull[i], 1);
      mbar_init(&aempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&accfull[i], 1);
      mbar_init(&accempty[i], 256);
      mbar_init(&adone[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  constexpr uint32_t kTmemCols = TA ? 512 : 64;  // acc [0, 64); TMEM A slots from column 128
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // acc c: cols [32c, 32c+16) Delta, [32c+16, 32c+32) self

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    int s = 0, a = -1, ar = 0;
    uint32_t sph = 0, aph[2] = {0, 0}, arph = 0;
    // (L2 eviction hints on these loads / the stores measured 10 % slower: none)
    // Work is claimed dynamically (one atomic per chunk of 128 columns of a row band) in the
    // global band-major order, so concurrently active CTAs stream ADJACENT column chunks of
    // the same rows (DRAM row-buffer locality: a band per CTA measured 5.5 vs 6.6 TB/s on
    // this 4-read / 3-write mix), the factor tiles of the few tensors in flight stay in L2,
    // and CTAs that start late (side-stream work on their SM) simply take fewer chunks.
    for (;;) {
      int band = 0;
      if (lane == 0) band = atomicAdd(band_ctr, 1);
      band = __shfl_sync(0xffffffffu, band, 0);
      if (band >= nbands) break;
      const int4 bd = bands[band];  // (slot, m0, first column, columns)
      const O5StreamMaps* ms = smaps + bd.x;
      const O5OpMaps* mo = omaps + bd.x;
      const int ntile = (bd.w + kO5TileN - 1) / kO5TileN;
      auto push_tile = [&](int n) {  // TA: stream boxes only (B: warp 10)
        mbar_wait(&sempty[s], sph ^ 1);
        if (elect_one()) {
          const int n0 = bd.z + kO5TileN * n;
          sinfo[s] = make_int4(bd.x, bd.y, n0, (a < 0 ? 0 : a) | (n == 0 ? 2 : 0) | (n == ntile - 1 ? 4 : 0));
          mbar_arrive(&tinfo[s]);
          uint8_t* st = smem + s * stage_bytes;
          mbar_expect_tx(&sfull[s], nstreams * kO5StreamBox);
          for (int q = 0; q < nstreams; ++q)
            tma_load_2d(st + q * kO5StreamBox, &ms->s[q], &sfull[s], n0, bd.y);
        }
        __syncwarp();
        if (++s == nst) {
          s = 0;
          sph ^= 1;
        }
      };
      if (TA) {
        // first tile, then the A boxes through the ring (the MMA warp drains them into TMEM
        // when it reaches that tile), then the rest of the chunk. (Moving the A boxes to the
        // B producer warp, or draining them into TMEM ahead of the chunk, measured slower.)
        push_tile(0);
        for (int kc = 0; kc < nkc && a_src == 0; ++kc) {
          mbar_wait(&aempty[ar], arph ^ 1);
          if (elect_one()) {
            mbar_expect_tx(&afull[ar], kO5ABox);
            tma_load_2d(abuf + ar * kO5ABox, &mo->a, &afull[ar], KD::AK * kc, bd.y);
          }
          __syncwarp();
          if (++ar == nab) {
            ar = 0;
            arph ^= 1;
          }
        }
        for (int n = 1; n < ntile; ++n) push_tile(n);
        continue;
      }
      a = nab == 2 ? (a + 1) & 1 : 0;
      mbar_wait(&aempty[a], aph[a] ^ 1);
      aph[a] ^= 1;
      if (elect_one()) {
        mbar_expect_tx(&afull[a], aband_bytes);
        for (int kc = 0; kc < nkc; ++kc)
          tma_load_2d(abuf + a * aband_bytes + kc * kO5ABox, &mo->a, &afull[a], KD::AK * kc, bd.y);
      }
      __syncwarp();
      for (int n = 0; n < ntile; ++n) {
        mbar_wait(&sempty[s], sph ^ 1);
        if (elect_one()) {
          const int n0 = bd.z + kO5TileN * n;
          sinfo[s] = make_int4(bd.x, bd.y, n0, a | (n == 0 ? 2 : 0) | (n == ntile - 1 ? 4 : 0));
          uint8_t* st = smem + s * stage_bytes;
          mbar_expect_tx(&sfull[s], nstreams * kO5StreamBox + KD::NBP * nkc * kO5BBox);
          for (int q = 0; q < nstreams; ++q)
            tma_load_2d(st + q * kO5StreamBox, &ms->s[q], &sfull[s], n0, bd.y);
          uint8_t* bb = st + 4 * kO5StreamBox;
          for (int pl = 0; pl < KD::NBP; ++pl)
            for (int kc = 0; kc < nkc; ++kc)
              tma_load_2d(bb + (pl * nkc + kc) * kO5BBox, &mo->b[pl], &sfull[s], KD::AK * kc, n0);
        }
        __syncwarp();
        if (++s == nst) {
          s = 0;
          sph ^= 1;
        }
      }
    }
    // end marker: one more stage whose descriptor says "done" (no bytes)
    mbar_wait(&sempty[s], sph ^ 1);
    if (elect_one()) {
      sinfo[s] = make_int4(-1, 0, 0, 0);
      if (TA) mbar_arrive(&tinfo[s]);
      mbar_arrive(&sfull[s]);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    const uint32_t idesc = BF ? idesc_f16(kO5TileN) : idesc_tf32(kO5TileN, false, false);
    int s = 0, a = 0, c = 0;
    uint32_t sph = 0, cph = 0, aph[2] = {0, 0};
    int ar = 0, ta = 1, bs = 0;
    uint32_t arph = 0, bph = 0;
    int pend = 0;             // early mode: boxes of the next chunk already in TMEM
    bool nt_ready = false;    // early mode: the other slot's MMAs are done
    bool aused[2] = {false, false};
    uint32_t adph[2] = {0, 0};

    const uint32_t a_tmem0 = tmem + 128u;
    const uint32_t a_slot_cols = static_cast<uint32_t>(KA / 2);  // bf16: 2 per 32-bit column
    for (;;) {
      mbar_wait(TA ? &tinfo[s] : &sfull[s], sph);  // TA: the descriptor, not the stream data
      const int4 tl = sinfo[s];
      if (tl.x < 0) break;
      const DevT2 t = T[tl.x];
      const bool last_in_band = tl.w & 4;
      // copy A box `kc` of the next chunk (128 rows x 128 B) from the ring into TMEM slot `sl`;
      // tcgen05.cp and tcgen05.mma execute in issue order, so later MMAs see it
      auto drain_box = [&](int sl, int kc) {
        tc_fence_after();
        if (elect_one()) {
          const uint64_t d0 = sdesc(su32(abuf + ar * kO5ABox), 16u, 1024u);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tmem_cp_128x256b(a_tmem0 + sl * a_slot_cols + 8u * (4 * kc + kk), d0 + 2u * kk);
          mma_commit(&aempty[ar]);
        }
        __syncwarp();
        if (++ar == nab) {
          ar = 0;
          arph ^= 1;
        }
      };
      if (TA && (tl.w & 2)) {  // new chunk: (the rest of) its A band into the other TMEM slot
        const int nt = ta ^ 1;
        if (a_early && !nt_ready) {
          if (aused[nt]) {
            mbar_wait(&adone[nt], adph[nt]);
            adph[nt] ^= 1;
          }
          nt_ready = true;
        }
        for (; pend < nkc; ++pend) {
          mbar_wait(&afull[ar], arph);
          drain_box(nt, pend);
        }
        ta = nt;
        pend = 0;
        nt_ready = false;
      } else if (!TA && (tl.w & 2)) {
        a = tl.w & 1;
        mbar_wait(&afull[a], aph[a]);
        aph[a] ^= 1;
      }
      if (TA) mbar_wait(&bfull[bs], bph);
      mbar_wait(&accempty[c], cph ^ 1);
      tc_fence_after();
      const uint32_t abase = su32(abuf + a * aband_bytes);
      const uint32_t bbase = TA ? su32(bring + bs * bslot_bytes)
                                : su32(smem + s * stage_bytes + 4 * kO5StreamBox);
      const uint64_t a0 = sdesc(abase, 16u, 1024u);
      uint64_t b0[KD::NBP];
#pragma unroll
      for (int pl = 0; pl < KD::NBP; ++pl) b0[pl] = sdesc(bbase + pl * nkc * kO5BBox, 16u, 1024u);
      const uint32_t dacc = tmem + 32u * c, sacc = dacc + 16u;
      const int rp = o5_rpad(t.r, D, KD::KS);
      const int K = D * rp;
      const int s_lo = self_index * rp, s_hi = s_lo + rp;
      const uint32_t a_t = a_tmem0 + ta * a_slot_cols;
      auto mma = [&](uint32_t d, uint64_t ad, uint64_t bd, uint32_t acc, int kstep) {
        if (TA)
          mma_bf16_ts(d, a_t + 8u * kstep, bd, idesc, acc);
        else if (BF)
          mma_bf16(d, ad, bd, idesc, acc);
        else
          mma_tf32(d, ad, bd, idesc, acc);
      };
      if (elect_one()) {
        for (int kc = 0; kc < nkc; ++kc) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const int k = KD::AK * kc + KD::KS * kk;
            if (k >= K) break;
            const uint64_t ad = a0 + (uint64_t)((kc * kO5ABox + kk * 32) >> 4);
            const uint64_t boff = (uint64_t)((kc * kO5BBox + kk * 32) >> 4);
            const uint32_t first = (kc == 0 && kk == 0) ? 0u : 1u;
#pragma unroll
            for (int pl = 0; pl < KD::NBP; ++pl) mma(dacc, ad, b0[pl] + boff, pl == 0 ? first : 1u, 4 * kc + kk);
            if (SELF && D > 1 && k >= s_lo && k < s_hi) {
              const uint32_t sfirst = k == s_lo ? 0u : 1u;
#pragma unroll
              for (int pl = 0; pl < KD::NBP; ++pl) mma(sacc, ad, b0[pl] + boff, pl == 0 ? sfirst : 1u, 4 * kc + kk);
            }
          }
        }
        mma_commit(&accfull[c]);
        if (TA) mma_commit(&bempty[bs]);
        if (TA && a_early && last_in_band) mma_commit(&adone[ta]);
        if (!TA && last_in_band) mma_commit(&aempty[a]);
      }
      __syncwarp();
      if (TA && a_early) {
        if (last_in_band) aused[ta] = true;
        const int nt = ta ^ 1;
        if (!nt_ready && (!aused[nt] || mbar_test(&adone[nt], adph[nt]))) {
          if (aused[nt]) adph[nt] ^= 1;
          nt_ready = true;
        }
        while (nt_ready && pend < nkc && mbar_test(&afull[ar], arph)) {
          drain_box(nt, pend);
          ++pend;
        }
      }
      if (++s == nst) {
        s = 0;
        sph ^= 1;
      }
      if (TA && ++bs == nbr) {
        bs = 0;
        bph ^= 1;
      }
      c ^= 1;
      if (c == 0) cph ^= 1;
    }
  } else if (TA && warp == 10) {
    // ---------------------------------------------------------------- B producer (TA)
    int s = 0, bs = 0, ar = 0;
    uint32_t sph = 0, bph = 0, arph = 0;
    for (;;) {
      mbar_wait(&tinfo[s], sph);
      const int4 tl = sinfo[s];
      if (tl.x < 0) break;
      const O5OpMaps* mo = omaps + tl.x;
      if (a_src == 1 && (tl.w & 2)) {
        // the whole A band fits the box ring: issue it as soon as the chunk is scheduled
        for (int kc = 0; kc < nkc; ++kc) {
          mbar_wait(&aempty[ar], arph ^ 1);
          if (elect_one()) {
            mbar_expect_tx(&afull[ar], kO5ABox);
            tma_load_2d(abuf + ar * kO5ABox, &mo->a, &afull[ar], KD::AK * kc, tl.y);
          }
          __syncwarp();
          if (++ar == nab) {
            ar = 0;
            arph ^= 1;
          }
        }
      }
      mbar_wait(&bempty[bs], bph ^ 1);
      if (elect_one()) {
        uint8_t* bb = bring + bs * bslot_bytes;
        mbar_expect_tx(&bfull[bs], bslot_bytes);
        for (int pl = 0; pl < KD::NBP; ++pl)
          for (int kc = 0; kc < nkc; ++kc)
            tma_load_2d(bb + (pl * nkc + kc) * kO5BBox, &mo->b[pl], &bfull[bs], KD::AK * kc, tl.z);
      }
      __syncwarp();
      if (++s == nst) {
        s = 0;
        sph ^= 1;
      }
      if (++bs == nbr) {
        bs = 0;
        bph ^= 1;
      }
    }
  } else if (TA && warp == 11) {
    // ---------------------------------------------------------------- A loader (TA, a_src 2)
    int s = 0, ar = 0;
    uint32_t sph = 0, arph = 0;
    for (; a_src == 2;) {
      mbar_wait(&tinfo[s], sph);
      const int4 tl = sinfo[s];
      if (tl.x < 0) break;
      if (tl.w & 2) {
        const O5OpMaps* mo = omaps + tl.x;
        for (int kc = 0; kc < nkc; ++kc) {
          mbar_wait(&aempty[ar], arph ^ 1);
          if (elect_one()) {
            mbar_expect_tx(&afull[ar], kO5ABox);
            tma_load_2d(abuf + ar * kO5ABox, &mo->a, &afull[ar], KD::AK * kc, tl.y);
          }
          __syncwarp();
          if (++ar == nab) {
            ar = 0;
            arph ^= 1;
          }
        }
      }
      if (++s == nst) {
        s = 0;
        sph ^= 1;
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (8 warps)
    const int et = threadIdx.x - 64;  // 0..255
    const int quarter = warp % 4, half = (warp - 2) / 4;
    const int row = quarter * 32 + lane;  // tile row (TMEM lane)
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    double num = 0.0, den = 0.0, dn = 0.0, en = 0.0, nf = 0.0;
    int s = 0, c = 0, prev_s = -1;
    uint32_t sph = 0, cph = 0;
    for (;;) {
      mbar_wait(&sfull[s], sph);
      const int4 tl = sinfo[s];
      if (tl.x < 0) break;
      const DevT2 t = T[tl.x];
      mbar_wait(&accfull[c], cph);
      tc_fence_after();
      float dv[8], sv[8];
      tmem_ld8(tmem + lane_base + 32u * c + 8u * half, dv);
      if (SELF && D > 1) tmem_ld8(tmem + lane_base + 32u * c + 16u + 8u * half, sv);
      tc_fence_before();
      mbar_arrive(&accempty[c]);
      if (BF) {  // undo the B prescale (power of two: exact)
        const float ps = post[tl.x];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          dv[i] = __fmul_rn(dv[i], ps);
          if (SELF && D > 1) sv[i] = __fmul_rn(sv[i], ps);
        }
      }
      uint8_t* st = smem + s * stage_bytes;
      const int64_t grow = tl.y + row;
      const int64_t col0 = tl.z + 8 * half;
      const bool live_row = grow < t.a;
      float fnum = 0.f, fden = 0.f, fen = 0.f, fdn = 0.f;
      int bad = 0;
#pragma unroll
      for (int q2 = 0; q2 < 2; ++q2) {
        const int chunk = 2 * half + q2;  // 16-B chunk of the 64-B row (SW64)
        const uint32_t off = row * 64u + ((chunk ^ ((row >> 1) & 3)) * 16u);
        float4* pp = reinterpret_cast<float4*>(st + 0 * kO5StreamBox + off);
        float4* pa = reinterpret_cast<float4*>(st + 1 * kO5StreamBox + off);
        float4* pv = reinterpret_cast<float4*>(st + 2 * kO5StreamBox + off);
        const float4 x_p = *pp, x_a = *pa, x_v = *pv;
        const float4 x_l = ovl ? *reinterpret_cast<const float4*>(st + 3 * kO5StreamBox + off)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        const float ip[4] = {x_p.x, x_p.y, x_p.z, x_p.w}, ia[4] = {x_a.x, x_a.y, x_a.z, x_a.w};
        const float iv[4] = {x_v.x, x_v.y, x_v.z, x_v.w}, il[4] = {x_l.x, x_l.y, x_l.z, x_l.w};
        float op[4], oa[4], ov[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float delta = dv[4 * q2 + j];
          const EpiOut o = epilogue(delta, ip[j], ia[j], il[j], iv[j], mode, gamma, beta, classical);
          op[j] = o.pend;
          oa[j] = o.anchor;
          ov[j] = o.v;
          const bool live = live_row && (col0 + 4 * q2 + j) < t.b;
          if (live) {
            if (SELF) {
              const float rec = D > 1 ? __fmul_rn(sv[4 * q2 + j], (float)D) : __fmul_rn(delta, (float)D);
              const float df = rec - ip[j];
              fnum = fmaf(df, df, fnum);
              fden = fmaf(ip[j], ip[j], fden);
            }
            fen = fmaf(o.e, o.e, fen);
            if (ovl) fdn = fmaf(o.pend, o.pend, fdn);
            bad |= !isfinite(o.anchor);
          }
        }
        *pp = make_float4(op[0], op[1], op[2], op[3]);
        *pa = make_float4(oa[0], oa[1], oa[2], oa[3]);
        *pv = make_float4(ov[0], ov[1], ov[2], ov[3]);
      }
      num += fnum;
      den += fden;
      en += fen;
      dn += fdn;
      nf += bad;
      fence_async_smem();
      named_bar(1, 256);
      if (et == 0) {
        const O5StreamMaps* ms = smaps + tl.x;
        for (int q = 0; q < 3; ++q) tma_store_2d(&ms->s[q], st + q * kO5StreamBox, tl.z, tl.y);
        bulk_commit();
        // a stage may be refilled once its stores have read it: release the previous tile's
        // stage (its store group is the older one), keeping the store latency off this path
        if (prev_s >= 0) {
          bulk_wait_read1();
          mbar_arrive(&sempty[prev_s]);
        }
        prev_s = s;
      }
      if (++s == nst) {
        s = 0;
        sph ^= 1;
      }
      c ^= 1;
      if (c == 0) cph ^= 1;
    }
    // stats
    double v[5] = {num, den, dn, en, nf};
#pragma unroll
    for (int k = 0; k < 5; ++k)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    if (lane == 0 && stats) {
      if (v[0] != 0.0) atomicAdd(&stats->err_num, v[0]);
      if (v[1] != 0.0) atomicAdd(&stats->err_den, v[1]);
      if (v[2] != 0.0) atomicAdd(&stats->delta_norm_sq, v[2]);
      if (v[3] != 0.0) atomicAdd(&stats->err_norm_sq, v[3]);
      if (v[4] != 0.0) atomicAdd(&stats->nonfinite, v[4]);
    }
    if (et == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 o5_encode() {
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

static void o5_encode_map(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1,
                          uint64_t stride_bytes, uint32_t b0, uint32_t b1,
                          CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B,
                          CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32) {
  const cuuint64_t dims[2] = {d0, d1};
  const cuuint64_t strides[1] = {stride_bytes};
  const cuuint32_t box[2] = {b0, b1};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = o5_encode()(m, dt, 2, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(DLX_ERR_CUDA, "cuTensorMapEncodeTiled (K5 tc) failed");
}

constexpr int kO5MaxK = 256;

struct O5State : PlanExt {
  int D = 0, KA = 0;
  bool bf = false;         // bf16 x 3 operands (K > 32) vs tf32 x 2
  int nab = 2, nst = 0;    // A-band buffers, stream stages
  int nbr = 0;             // B ring slots (bf16 path)
  int a_mode = 0;          // fp16 path: A-box issuer / early drain (see k_o5)
  size_t smem = 0;
  int nrows = 0;
  const int4* d_rows = nullptr;  // layout-owned (O5Tables)
  std::vector<int64_t> aoff, boff;  // per slot: element offsets of A [lda][KA], B [ldb][KA]
  int64_t a_elems = 0, b_elems = 0;
  int64_t params = 0;  // 2-D parameters covered
  int s0 = 0, s1 = 0;  // slot range
  int nbands = 0;
  const int4* d_bands = nullptr;  // (t2 slot, m0, first column, columns), claim order
  int* d_ctr = nullptr;
  int64_t* d_aoff = nullptr;
  int64_t* d_boff = nullptr;
  MapTableCache<O5OpMaps, 3> maps;  // operand descriptors keyed by the staging buffers
};

bool o5_eligible(const Plan& P, int D, int self_index) {
  if (P.t2.empty()) return false;
  const int ks = o5_bf(P.rmax, D) ? 16 : 8;  // MMA K step of the operand kind
  const int K = D * o5_rpad(P.rmax, D, ks);
  if (K > kO5MaxK) return false;  // A band (128 x K) + B stages must fit shared memory
  for (const DevT2& t : P.t2)
    if (t.b % 4 != 0) return false;
  (void)self_index;
  return true;
}

// Rank-independent work lists of one slot range: row bands (128 rows x `chunk` columns, claimed
// in band-major order) and the factor rows k_o5_prep converts. Owned by the layout.
struct O5Tables : PlanExt {
  std::vector<int4> bands, rows;
  int4* d_bands = nullptr;
  int4* d_rows = nullptr;
  int64_t params = 0;
  ~O5Tables() override {
    if (d_bands) cudaFree(d_bands);
    if (d_rows) cudaFree(d_rows);
  }
};

static const O5Tables& o5_tables(const Plan& P, const SlotRange& R, int64_t chunk) {
  bool fresh = false;
  O5Tables& W = layout_ext<O5Tables>(*P.layout, "o5tab:" + R.key() + ":" + std::to_string(chunk),
                                     &fresh);
  if (!fresh) return W;
  HostProf hp("o5_tables (new)");
  for (int k = R.s0; k < R.s1; ++k) {
    const DevT2& t = P.t2[k];
    for (int64_t m0 = 0; m0 < t.a; m0 += 128)
      for (int64_t n0 = 0; n0 < t.b; n0 += chunk)
        W.bands.push_back(make_int4(k, static_cast<int>(m0), static_cast<int>(n0),
                                    static_cast<int>(std::min(chunk, t.b - n0))));
    for (int side = 0; side < 2; ++side) {
      const int64_t ld = side == 0 ? t.lda : t.ldb;
      for (int64_t r = 0; r < ld; ++r) W.rows.push_back(make_int4(k, side, static_cast<int>(r), 0));
    }
    W.params += t.a * t.b;
  }
  for (auto* v : {&W.bands, &W.rows}) {
    int4*& d = v == &W.bands ? W.d_bands : W.d_rows;
    DLX_CUDA(cudaMalloc(&d, sizeof(int4) * std::max<size_t>(v->size(), 1)));
    upload_now(d, v->data(), sizeof(int4) * v->size());
  }
  return W;
}

static O5State& o5_state(const Plan& P, int D, const SlotRange& R) {
  bool fresh = false;
  O5State& S = plan_ext<O5State>(P, "o5:" + std::to_string(D) + ":" + R.key(), &fresh);
  if (!fresh) return S;
  HostProf hp("o5_state (new)");
  S.D = D;
  S.bf = o5_bf(P.rmax, D);
  const int K = D * o5_rpad(P.rmax, D, S.bf ? O5Kind<true>::KS : O5Kind<false>::KS);
  const int ak = S.bf ? O5Kind<true>::AK : O5Kind<false>::AK;
  const int nbp = S.bf ? 3 : 2;
  S.KA = static_cast<int>(round_up(K, ak));
  S.s0 = R.s0;
  S.s1 = R.s1;
  // shared-memory plan: A band buffers (double if 3+ stream stages still fit) + stages
  // tf32: 215 KB measured best; bf16 (stream-only stages): the whole 227 KB
  static const int budget_kb = [] {  // experiments: DLX_O5_SMEM_KB
    const char* e = getenv("DLX_O5_SMEM_KB");
    return e ? atoi(e) : 0;
  }();
  const size_t budget = static_cast<size_t>(budget_kb ? budget_kb : (S.bf ? 227 : 215)) * 1024;
  const int nkc = S.KA / ak;
  // bf16: B moves through its own ring (nbr slots), the stages carry the stream boxes only
  const size_t bslot = static_cast<size_t>(nbp) * nkc * kO5BBox;
  const size_t stage = 4 * kO5StreamBox + (S.bf ? 0 : bslot) + 2 * 8 + 16;
  // tf32: whole A bands in shared memory; bf16: a 2-box ring feeding A into TMEM
  const size_t aband = S.bf ? kO5ABox : static_cast<size_t>(nkc) * kO5ABox;
  constexpr size_t kBars = 1024;  // barriers, TMEM slot, stage descriptors
  auto stages = [&](int nab, int nbr) {
    const size_t fixed = 1024 + nab * aband + nbr * bslot + kBars;
    return budget > fixed ? static_cast<int>(std::min<size_t>(kO5MaxStages, (budget - fixed) / stage)) : 0;
  };
  if (S.bf) {
    // A box ring: the whole band when that costs no stream stage (its loads are then issued
    // ahead by the B warp and never stall the stream producer), else two boxes (one
    // serialises the band loads: D=8 7.7 -> 8.6 ms; four at the cost of two stages: 7.3 ->
    // 8.0 ms); then B slots
    static const int nab_env = [] {  // experiments: DLX_O5_NAB
      const char* e = getenv("DLX_O5_NAB");
      return e ? atoi(e) : 0;
    }();
    S.nab = nab_env ? nab_env : (nkc <= 4 && stages(nkc, 2) >= stages(2, 2) ? std::max(nkc, 2) : 2);
    S.nab = std::min(S.nab, 4);
    static const int amode_env = [] {  // experiments: DLX_O5_AMODE
      const char* e = getenv("DLX_O5_AMODE");
      return e ? atoi(e) : -1;
    }();
    S.a_mode = amode_env >= 0 ? amode_env : (S.nab >= nkc ? 1 : 0);
    S.nbr = stages(S.nab, 3) >= stages(S.nab, 2) ? 3 : 2;
  } else {
    S.nab = stages(2, 0) >= 3 ? 2 : 1;
    S.nbr = 0;
  }
  S.nst = stages(S.nab, S.nbr);
  if (S.nst < 2) raise(DLX_ERR_VALIDATION, "outer update: K too large for the tensor-core path");
  S.smem = 1024 + S.nab * aband + S.nbr * bslot + kBars + S.nst * stage;
  // A / B staging offsets cover every slot (shared buffers); bands and rows only the range.
  // Work unit = a chunk of a row band (128 rows x chunk columns); chunks are claimed in
  // band-major order so concurrently active CTAs read adjacent columns of the same rows.
  static const int chunk_env = [] {  // experiments: DLX_O5_CHUNK (columns per claimed chunk)
    const char* e = getenv("DLX_O5_CHUNK");
    return e ? atoi(e) : 0;
  }();
  // 128-column chunks (DRAM row locality across concurrently active CTAs); K = 256 (four
  // A boxes per band): 192, the A band's TMEM refill amortised over 12 tiles (7.37 -> 7.05
  // ms at D = 8; 256 measured 7.47); single smem A band (tf32): 256
  const int64_t chunk = chunk_env ? chunk_env
                        : S.bf ? (nkc >= 4 ? 192 : 128)
                               : (S.nab == 2 ? 128 : 256);
  // the band / row work lists do not depend on the rank: shared by every plan of the layout
  const O5Tables& W = o5_tables(P, R, chunk);
  S.nbands = static_cast<int>(W.bands.size());
  S.nrows = static_cast<int>(W.rows.size());
  S.d_bands = W.d_bands;
  S.d_rows = W.d_rows;
  S.params = W.params;
  for (size_t k = 0; k < P.t2.size(); ++k) {
    const DevT2& t = P.t2[k];
    S.aoff.push_back(S.a_elems);
    S.boff.push_back(S.b_elems);
    S.a_elems += t.lda * S.KA;
    S.b_elems += t.ldb * S.KA;
  }
  S.d_ctr = static_cast<int*>(P.dev_alloc(sizeof(int)));
  S.d_aoff = plan_upload(P, S.aoff, 1);
  S.d_boff = plan_upload(P, S.boff, 1);
  return S;
}

template <bool SELF, bool BF>
static void launch_o5(const Plan& P, const O5State& S, const O5StreamMaps* smaps,
                      const O5OpMaps* maps, int grid, int nbands,
                      int D, int self_index,
                      int mode, float gamma, float beta, int classical, const float* post,
                      dlx_round_stats* stats, cudaStream_t s) {
  smem_optin(reinterpret_cast<const void*>(k_o5<SELF, BF>), 227 * 1024);
  k_o5<SELF, BF><<<grid, BF ? kO5ThreadsTA : kO5Threads, S.smem, s>>>(
      P.d_t2, smaps, maps, S.d_bands, nbands, S.d_ctr, D, S.KA, S.nst, S.nab, S.nbr, S.a_mode,
      self_index, mode, gamma, beta, classical, post, stats);
}

void launch_outer_2d_tc(dlx_ctx* ctx, const Plan& P, int D, const uint8_t* gathered,
                        int self_index, int mode, float* pending, float* anchor,
                        const float* local, float* velocity, float gamma, float beta,
                        int classical, dlx_round_stats* stats, const SlotRange& R,
                        cudaStream_t s) {
  O5State& S = o5_state(P, D, R);
  if (S.nbands == 0) return;
  const int KA = S.KA;
  const size_t es = S.bf ? 2 : 4;
  void* A = ctx->scratch("o5_A", es * (S.a_elems + 1024));
  void* B[2] = {ctx->scratch("o5_B0", es * (S.b_elems + 1024)),
                ctx->scratch("o5_B1", es * (S.b_elems + 1024))};
  float* pre = nullptr;
  float* post = nullptr;
  if (S.bf) {  // per-tensor B prescale for the fp16 planes
    pre = static_cast<float*>(ctx->scratch("o5_escale", sizeof(float) * 2 * (P.t2.size() + 1)));
    post = pre + P.t2.size() + 1;
    k_o5_escale<<<static_cast<unsigned>(P.t2.size()), 256, 0, s>>>(P.d_t2, gathered, P.payload_bytes,
                                                                   P.qbits, D, pre, post);
    DLX_LAUNCHED();
  }
  if (S.bf)
    k_o5_prep<true><<<static_cast<unsigned>(ceil_div(S.nrows, prep_rows<true>())), 256, 0, s>>>(
        P.d_t2, S.d_rows, S.nrows, S.d_aoff, S.d_boff, gathered,
        P.payload_bytes, P.qbits, D, KA, S.bf ? O5Kind<true>::KS : O5Kind<false>::KS, pre, A,
        B[0], B[1]);
  else
    k_o5_prep<false><<<static_cast<unsigned>(ceil_div(S.nrows, prep_rows<false>())), 256, 0, s>>>(
        P.d_t2, S.d_rows, S.nrows, S.d_aoff, S.d_boff, gathered,
        P.payload_bytes, P.qbits, D, KA, S.bf ? O5Kind<true>::KS : O5Kind<false>::KS, pre, A,
        B[0], B[1]);
  DLX_LAUNCHED();
  // parameter-stream descriptors: per layout (every rank's plan shares them), all tensors
  const float* srcs[4] = {pending, anchor, velocity,
                          mode == DLX_MODE_OVERLAPPED ? local : nullptr};
  const void* skey[4] = {srcs[0], srcs[1], srcs[2], srcs[3]};
  auto& scache = layout_ext<MapTableCache<O5StreamMaps, 4>>(*P.layout, "o5_stream_maps");
  const O5StreamMaps* smaps = scache.get(skey, P.t2.size(), s, [&](O5StreamMaps* h) {
    for (size_t k = 0; k < P.t2.size(); ++k) {
      const DevT2& t = P.t2[k];
      for (int q = 0; q < 4; ++q)
        if (srcs[q])
          o5_encode_map(&h[k].s[q], srcs[q] + t.off, t.b, t.a, t.b * 4, kO5TileN, 128,
                        CU_TENSOR_MAP_SWIZZLE_64B);
    }
  });
  // operand descriptors: per plan state (K), keyed by the staging buffers
  const void* key[3] = {A, B[0], B[1]};
  const O5OpMaps* maps = S.maps.get(key, P.t2.size(), s, [&](O5OpMaps* h) {
    const CUtensorMapDataType dt = S.bf ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const uint32_t ak = S.bf ? O5Kind<true>::AK : O5Kind<false>::AK;
    for (size_t k = S.s0; k < static_cast<size_t>(S.s1); ++k) {
      const DevT2& t = P.t2[k];
      O5OpMaps& m = h[k];
      o5_encode_map(&m.a, static_cast<uint8_t*>(A) + es * S.aoff[k], KA, t.lda, KA * es, ak, 128,
                    CU_TENSOR_MAP_SWIZZLE_128B, dt);
      for (int pl = 0; pl < 2; ++pl)
        o5_encode_map(&m.b[pl], static_cast<uint8_t*>(B[pl]) + es * S.boff[k], KA, t.ldb, KA * es, ak,
                      kO5TileN, CU_TENSOR_MAP_SWIZZLE_128B, dt);
    }
  });
  int dev = 0, sms = 0;
  DLX_CUDA(cudaGetDevice(&dev));
  DLX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int nbands = S.nbands;
  const int grid = std::min(nbands, sms);
  DLX_CUDA(cudaMemsetAsync(S.d_ctr, 0, sizeof(int), s));
  // algorithmic bytes: read pending, anchor, velocity (+ local in overlapped mode), write
  // pending, anchor, velocity — 28 B/param overlapped, 24 B/param sync
  KernelTimer timer("k_o5", (mode == DLX_MODE_OVERLAPPED ? 28.0 : 24.0) * S.params, s);
  if (self_index >= 0) {
    if (S.bf)
      launch_o5<true, true>(P, S, smaps, maps, grid, nbands, D, self_index, mode, gamma, beta, classical, post, stats, s);
    else
      launch_o5<true, false>(P, S, smaps, maps, grid, nbands, D, self_index, mode, gamma, beta, classical, post, stats, s);
  } else {
    if (S.bf)
      launch_o5<false, true>(P, S, smaps, maps, grid, nbands, D, self_index, mode, gamma, beta, classical, post, stats, s);
    else
      launch_o5<false, false>(P, S, smaps, maps, grid, nbands, D, self_index, mode, gamma, beta, classical, post, stats, s);
  }
  DLX_LAUNCHED();
}

}  // namespace dlx
