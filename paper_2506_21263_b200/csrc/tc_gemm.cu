// tc_gemm.cu — tcgen05 / TMEM / TMA power-iteration sweeps (lowrank_approx
// compress.cpp:70-77):  K1  Y = delta Q  (A = delta, K-major)   and
//                       K2  Z = delta^T P (A = delta^T), deterministic split-K.
// For K2 the delta tile arrives row-major (M contiguous); the split warps transpose it into
// the canonical K-major SW128 layout while splitting, so both sweeps feed the tensor core
// K-major operands (MN-major tf32 operands would need the 32B-atom swizzle variant).
//
// Both sweeps stream every element of delta from HBM exactly once; the factor operand
// (Q or P, <= 256 columns) is the MMA N dimension. Precision: 3xTF32 — each fp32 operand
// tile is split in shared memory into hi (tf32-exact, low 13 mantissa bits cleared) and
// lo = x - hi, and the accumulator (fp32, TMEM) receives hi*hi + hi*lo + lo*hi, i.e.
// ~fp32-grade products (the reference accumulates in fp64; tolerance-tested).
//
// Per CTA (persistent, one per SM): warp 0 = TMA producer (one elected lane), warp 1 =
// tcgen05.mma issuer (one lane; also owns the TMEM allocation), warps 2-5 = 128 threads
// that split each landed stage into hi/lo and, at the end of a tile, drain the TMEM
// accumulator (tcgen05.ld) to the column-major factor buffer.
// Pipeline (mbarriers per stage): full (TMA bytes) -> split (128 arrivals) -> empty
// (tcgen05.commit); per tile: tmem_full (commit) -> tmem_empty (128 arrivals).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>

#include "dlx_internal.cuh"
#include "ptx.cuh"

namespace dlx {

// ------------------------------------------------------------------ kernel
struct TcMaps {
  CUtensorMap a;  // delta: K1 box {32, 128} SW128 (K-major); K2 box {32, 32} plain ([k][m])
  CUtensorMap b;  // factor (Q for K1, P for K2): box {32, N} SW128 (K-major)
};

constexpr int kTcThreads = 320;  // producer warp, MMA warp, 8 split/epilogue warps
constexpr uint32_t kAStage = 128 * 32 * 4;  // 16 KB raw delta tile per stage
constexpr uint32_t kTmemCols = 512;  // [0,N) accumulator, then compute slots of A hi/lo (64 cols)

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Ring position (slot, phase) advanced without integer division.
struct Ring {
  int slot = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void next(int n) {
    if (++slot == n) {
      slot = 0;
      phase ^= 1u;
    }
  }
};

// A_MN: false = K1 (A = delta rows: the TMA tile is already K-major SW128, row m = A row);
// true = K2 (A = delta^T: the raw TMA tile is [k][m], column m = A row).
// KB: 32-column k boxes per pipeline stage (a 16 KB stage costs one mbarrier round trip per
// 16 KB and caps the stream near 5.5 TB/s; 32 KB stages reach the HBM roofline).
// Two rings decouple memory latency from the MMA: a deep LOAD ring (lr stages of raw A + B
// in shared memory, filled by TMA) and a shallow COMPUTE ring (cr slots of A hi/lo in TMEM,
// written with tcgen05.st, + B hi/lo in shared memory). The split warps move a landed load
// stage into a compute slot and immediately release the load stage, so up to lr stages of
// HBM traffic stay in flight per SM independently of the MMA pipeline.
template <bool A_MN, int KB>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_tc_sweep(const DevT2* __restrict__ T, const TcMaps* __restrict__ maps,
               const int4* __restrict__ tiles, const int* __restrict__ cta_off, int N,
               int lr, int cr,
               const int* __restrict__ splits, const int64_t* __restrict__ part_off,
               float* __restrict__ out, float* __restrict__ part, int hints) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t kA = KB * kAStage;          // raw A bytes per stage
  constexpr int KS = 32 * KB;                    // k extent of a stage
  const uint32_t b_box = static_cast<uint32_t>(N) * 128;  // one 32-k box of B (N rows x 128 B)
  const uint32_t b_bytes = KB * b_box;
  const uint32_t ls_bytes = kA + b_bytes;        // load stage: raw A + raw B
  uint8_t* cring = smem + lr * ls_bytes;         // compute slots: B hi + B lo
  uint64_t* bars = reinterpret_cast<uint64_t*>(cring + cr * 2 * b_bytes);
  uint64_t* lfull = bars;
  uint64_t* lempty = lfull + lr;
  uint64_t* cfull = lempty + lr;
  uint64_t* cempty = cfull + cr;
  uint64_t* tfull = cempty + cr;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < lr; ++s) {
      mbar_init(&lfull[s], 1);
      mbar_init(&lempty[s], 256);
    }
    for (int s = 0; s < cr; ++s) {
      mbar_init(&cfull[s], 256);
      mbar_init(&cempty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 256);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t a_base = static_cast<uint32_t>((N + 31) / 32 * 32);  // A slots after the accumulator
  constexpr uint32_t kSlotCols = 64u * KB;  // TMEM columns per compute slot (hi + lo per box)
  constexpr int64_t KC = 2048;

  // k-loop extent of a tile
  auto tile_k = [&](const int4& tl, const DevT2& t, int64_t& k0, int64_t& k1) {
    if (!A_MN) {
      k0 = 0;
      k1 = t.b;
    } else {
      k0 = tl.w * KC;
      k1 = min(t.a, k0 + KC);
    }
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    // warp-uniform loop, one elected lane issues (TMA operands must be uniform)
    // delta streams through once; the factor chunks are re-read by every row band
    const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last();
    Ring L;
    for (int ti = cta_off[blockIdx.x]; ti < cta_off[blockIdx.x + 1]; ++ti) {
      const int4 tl = tiles[ti];
      const DevT2 t = T[tl.x];
      const TcMaps* mp = maps + tl.x;
      if (elect_one()) {
        prefetch_map(&mp->a);
        prefetch_map(&mp->b);
      }
      __syncwarp();
      int64_t k0, k1;
      tile_k(tl, t, k0, k1);
      for (int64_t k = k0; k < k1; k += KS, L.next(lr)) {
        const int s = L.slot;
        mbar_wait(&lempty[s], L.phase ^ 1);
        uint8_t* st = smem + s * ls_bytes;
        if (elect_one()) {
          const int nb = static_cast<int>(min(static_cast<int64_t>(KB), (k1 - k + 31) / 32));  // boxes inside the tile
          mbar_expect_tx(&lfull[s], static_cast<uint32_t>(nb) * (kAStage + b_box));
#pragma unroll
          for (int j = 0; j < KB; ++j) {
            if (j < nb) {
              const int kj = static_cast<int>(k) + 32 * j;
              if (!A_MN) {
                if (hints)
                  tma_load_2d_hint(st + j * kAStage, &mp->a, &lfull[s], kj, tl.y, pol_stream);  // {k, m0}
                else
                  tma_load_2d(st + j * kAStage, &mp->a, &lfull[s], kj, tl.y);
              } else {
#pragma unroll
                for (int q = 0; q < 4; ++q)  // raw [k][m] tile: 4 boxes of 32 rows x 32 columns
                  if (hints)
                    tma_load_2d_hint(st + j * kAStage + q * 4096, &mp->a, &lfull[s], tl.y + 32 * q, kj,
                                     pol_stream);
                  else
                    tma_load_2d(st + j * kAStage + q * 4096, &mp->a, &lfull[s], tl.y + 32 * q, kj);
              }
              if (hints)
                tma_load_2d_hint(st + kA + j * b_box, &mp->b, &lfull[s], kj, 0, pol_keep);  // {k, n}
              else
                tma_load_2d(st + kA + j * b_box, &mp->b, &lfull[s], kj, 0);
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    // The whole warp runs the (warp-uniform) loop so descriptors and TMEM addresses live in
    // uniform registers; one elected lane issues each tcgen05.mma / commit.
    const uint32_t idesc = idesc_tf32(N, false, false);
    // the k step adds 32 B = 2 units of the 16-B start-address field
    const uint64_t bdesc_hi0 = sdesc(su32(cring), 16u, 1024u);
    const uint64_t bdesc_lo0 = sdesc(su32(cring) + b_bytes, 16u, 1024u);
    const uint64_t slot_step = (2u * b_bytes) >> 4;  // start-address units per compute slot
    const uint64_t box_step = b_box >> 4;
    uint32_t tphase = 0;
    Ring C;
    for (int ti = cta_off[blockIdx.x]; ti < cta_off[blockIdx.x + 1]; ++ti) {
      const int4 tl = tiles[ti];
      const DevT2 t = T[tl.x];
      int64_t k0, k1;
      tile_k(tl, t, k0, k1);
      mbar_wait(tempty, tphase ^ 1);
      tc_fence_after();
      uint32_t acc = 0;
      for (int64_t k = k0; k < k1; k += KS, C.next(cr)) {
        const int c = C.slot;
        mbar_wait(&cfull[c], C.phase);
        tc_fence_after();
        const int nb = static_cast<int>(min(static_cast<int64_t>(KB), (k1 - k + 31) / 32));
        if (elect_one()) {
#pragma unroll
          for (int j = 0; j < KB; ++j) {
            if (j < nb) {
              const uint32_t a_hi = tmem + a_base + static_cast<uint32_t>(c) * kSlotCols + 64u * j;
              const uint32_t a_lo = a_hi + 32u;
              const uint64_t bh = bdesc_hi0 + slot_step * c + box_step * j;
              const uint64_t bl = bdesc_lo0 + slot_step * c + box_step * j;
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                mma_tf32_ts(tmem, a_hi + kk * 8u, bh + 2u * kk, idesc, (acc | kk | j) ? 1u : 0u);
                mma_tf32_ts(tmem, a_hi + kk * 8u, bl + 2u * kk, idesc, 1u);
                mma_tf32_ts(tmem, a_lo + kk * 8u, bh + 2u * kk, idesc, 1u);
              }
            }
          }
          mma_commit(&cempty[c]);
        }
        __syncwarp();
        acc = 1u;
      }
      if (elect_one()) mma_commit(tfull);
      __syncwarp();
      tphase ^= 1;
    }
  } else {
    // ---------------------------------------------------------------- split + epilogue
    // 8 warps: two per TMEM lane quarter; warp half h handles columns [16h, 16h + 16) of
    // every 32-column box
    const int et = threadIdx.x - 64;      // 0..255
    const int quarter = warp % 4;         // TMEM lane quarter this warp may access
    const int half = (warp - 2) / 4;      // 0 or 1
    const int row = quarter * 32 + lane;  // A / accumulator row of this thread
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const int bvec = static_cast<int>(b_bytes / 16);
    uint32_t tphase = 0;
    Ring L, C;
    for (int ti = cta_off[blockIdx.x]; ti < cta_off[blockIdx.x + 1]; ++ti) {
      const int4 tl = tiles[ti];
      const DevT2 t = T[tl.x];
      int64_t k0, k1;
      tile_k(tl, t, k0, k1);
      for (int64_t k = k0; k < k1; k += KS, L.next(lr), C.next(cr)) {
        const int s = L.slot, c = C.slot;
        mbar_wait(&lfull[s], L.phase);
        const uint8_t* st = smem + s * ls_bytes;
        const int nb = static_cast<int>(min(static_cast<int64_t>(KB), (k1 - k + 31) / 32));
        // 16 values per box of this thread's A row -> hi / lo registers
        float h[KB][16], l[KB][16];
#pragma unroll
        for (int j = 0; j < KB; ++j) {
          if (j < nb) {
            const uint8_t* sj = st + j * kAStage;
            if (!A_MN) {
              const float4* rowp = reinterpret_cast<const float4*>(sj) + row * 8;
#pragma unroll
              for (int qq = 0; qq < 4; ++qq) {
                const int q = half * 4 + qq;
                const float4 x = rowp[q ^ (row & 7)];  // SW128: chunk q stored at q ^ (row % 8)
                float4 hh, ll;
                split4(x, hh, ll);
                h[j][4 * qq + 0] = hh.x; h[j][4 * qq + 1] = hh.y; h[j][4 * qq + 2] = hh.z; h[j][4 * qq + 3] = hh.w;
                l[j][4 * qq + 0] = ll.x; l[j][4 * qq + 1] = ll.y; l[j][4 * qq + 2] = ll.z; l[j][4 * qq + 3] = ll.w;
              }
            } else {
              const float* raw = reinterpret_cast<const float*>(sj);
              const int q = row >> 5, mm = row & 31;
#pragma unroll
              for (int kk = 0; kk < 16; ++kk) {
                const float x = raw[q * 1024 + (half * 16 + kk) * 32 + mm];
                h[j][kk] = tf32_hi(x);
                l[j][kk] = x - h[j][kk];
              }
            }
          }
        }
        // B: raw (load stage) -> hi / lo (compute slot) once the slot is free
        mbar_wait(&cempty[c], C.phase ^ 1);
        tc_fence_after();
        const float4* braw = reinterpret_cast<const float4*>(st + kA);
        float4* bh = reinterpret_cast<float4*>(cring + c * 2 * b_bytes);
        float4* bl = reinterpret_cast<float4*>(cring + c * 2 * b_bytes + b_bytes);
        const int bv = bvec / KB * nb;
        for (int i = et; i < bv; i += 256) {
          float4 hh, ll;
          split4(braw[i], hh, ll);
          bh[i] = hh;
          bl[i] = ll;
        }
        mbar_arrive(&lempty[s]);  // raw stage consumed (A values are in registers)
#pragma unroll
        for (int j = 0; j < KB; ++j) {
          if (j < nb) {
            const uint32_t a_col = a_base + static_cast<uint32_t>(c) * kSlotCols + 64u * j + half * 16u;
            tmem_st16(tmem + lane_base + a_col, h[j]);
            tmem_st16(tmem + lane_base + a_col + 32u, l[j]);
          }
        }
        tmem_st_wait();
        fence_async_smem();
        tc_fence_before();
        mbar_arrive(&cfull[c]);
      }
      // epilogue: TMEM -> column-major factor (or split-K partial); halves alternate 16-col chunks
      mbar_wait(tfull, tphase);
      tc_fence_after();
      const int64_t m = tl.y + row;
      const int64_t mlim = A_MN ? t.b : t.a;
      const int64_t ld = A_MN ? t.ldb : t.lda;
      float* dst;
      if (!A_MN) {
        dst = out + t.poff;
      } else {
        dst = splits[tl.x] > 1 ? part + part_off[tl.x] + tl.w * (t.ldb * t.r) : out + t.qoff;
      }
      for (int cc = half * 16; cc < N; cc += 32) {
        float v[16];
        tmem_ld16(tmem + lane_base + cc, v);
        if (m < mlim) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (cc + j < t.r) dst[(cc + j) * ld + m] = v[j];
        }
      }
      tc_fence_before();
      mbar_arrive(tempty);
      tphase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
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

static void encode(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t stride1_bytes,
                   uint32_t b0, uint32_t b1, bool swizzle = true) {
  const cuuint64_t dims[2] = {d0, d1};
  const cuuint64_t strides[1] = {stride1_bytes};
  const cuuint32_t box[2] = {b0, b1};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(DLX_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

bool tc_eligible(const DevT2& t) { return (t.b % 4) == 0 && t.r >= 1; }

int tc_n(const Plan& P) { return static_cast<int>(std::max<int64_t>(16, round_up(P.rmax, 16))); }

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    DLX_CUDA(cudaGetDevice(&dev));
    DLX_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

struct TcState : PlanExt {
  int64_t swept_params = 0;  // delta elements one sweep reads on the tensor-core path
  std::vector<int4> k1, k2;  // tiles grouped per CTA (balanced, see balance())
  std::vector<int> off1, off2;
  int4* d_k1 = nullptr;
  int4* d_k2 = nullptr;
  int* d_off1 = nullptr;
  int* d_off2 = nullptr;
  MapTableCache<TcMaps, 2> maps[2];  // K1 / K2 descriptor tables keyed by (slab, factors)
};

static TcState& tc_state(const Plan& P) {
  bool fresh = false;
  TcState* s = &plan_ext<TcState>(P, "tc_sweep", &fresh);
  if (fresh) {
    HostProf hp("tc_state (new)");
    constexpr int64_t KC = 2048;
    for (size_t k = 0; k < P.t2.size(); ++k) {
      const DevT2& t = P.t2[k];
      if (!tc_eligible(t)) continue;
      s->swept_params += t.a * t.b;
      for (int64_t m0 = 0; m0 < t.a; m0 += 128) s->k1.push_back(make_int4((int)k, (int)m0, 0, 0));
      const int sp = static_cast<int>(ceil_div(t.a, KC));
      for (int q = 0; q < sp; ++q)
        for (int64_t j0 = 0; j0 < t.b; j0 += 128) s->k2.push_back(make_int4((int)k, (int)j0, 0, q));
    }
    // Longest-processing-time assignment of tiles to persistent CTAs: tile costs differ 4x
    // (K = 8192 vs 2048 columns), so a round-robin split leaves some SMs with 1.5x the work.
    const int G = num_sms();
    auto balance = [&](std::vector<int4>& tl, std::vector<int>& off, bool k2) {
      std::vector<std::pair<int64_t, int>> cost;
      for (size_t i = 0; i < tl.size(); ++i) {
        const DevT2& t = P.t2[tl[i].x];
        const int64_t kl = k2 ? std::min<int64_t>(KC, t.a - int64_t(tl[i].w) * KC) : t.b;
        cost.push_back({ceil_div(kl, 32) + 8, static_cast<int>(i)});  // + epilogue overhead
      }
      std::stable_sort(cost.begin(), cost.end(), [](auto& x, auto& y) { return x.first > y.first; });
      const int g = static_cast<int>(std::min<size_t>(tl.size(), G));
      std::vector<std::vector<int4>> bins(std::max(g, 1));
      std::vector<int64_t> load(std::max(g, 1), 0);
      for (auto& c : cost) {
        const int b = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
        load[b] += c.first;
        bins[b].push_back(tl[c.second]);
      }
      tl.clear();
      off.assign(1, 0);
      for (auto& b : bins) {
        tl.insert(tl.end(), b.begin(), b.end());
        off.push_back(static_cast<int>(tl.size()));
      }
    };
    balance(s->k1, s->off1, false);
    balance(s->k2, s->off2, true);
    s->d_k1 = plan_upload(P, s->k1);
    s->d_k2 = plan_upload(P, s->k2);
    s->d_off1 = plan_upload(P, s->off1);
    s->d_off2 = plan_upload(P, s->off2);
  }
  return *s;
}

// which = 0: K1 maps (delta box {32,128}, Q); which = 1: K2 maps (delta box {32,32}, P)
static const TcMaps* tc_maps(const Plan& P, int which, const float* slab, const float* fac,
                             cudaStream_t s) {
  TcState& S = tc_state(P);
  const void* key[2] = {slab, fac};
  const int N = tc_n(P);
  return S.maps[which].get(key, P.t2.size(), s, [&](TcMaps* host) {
    for (size_t k = 0; k < P.t2.size(); ++k) {
      const DevT2& t = P.t2[k];
      TcMaps& m = host[k];
      if (!tc_eligible(t)) continue;
      const float* A = slab + t.off;
      if (which == 0) {
        encode(&m.a, A, t.b, t.a, t.b * 4, 32, 128);
        encode(&m.b, fac + t.qoff, t.b, t.r, t.ldb * 4, 32, N);
      } else {
        encode(&m.a, A, t.b, t.a, t.b * 4, 32, 32, /*swizzle=*/false);
        encode(&m.b, fac + t.poff, t.a, t.r, t.lda * 4, 32, N);
      }
    }
  });
}

// Boxes per stage: 2 (32 KB of delta per stage) while the rings still fit; 1 for wide N.
static int tc_kb(int N) { return N <= 64 ? 2 : 1; }

// Ring sizes (load stages lr, compute slots cr) that fit ~220 KB of shared memory and the
// 512 TMEM columns (accumulator N + cr slots of 64 * kb columns).
static void tc_rings(int N, int kb, int& lr, int& cr) {
  const int b = N * 128 * kb;
  const int a = 16384 * kb;
  const int a_base = (N + 31) / 32 * 32;
  for (cr = std::min(kb == 1 ? 7 : 3, (512 - a_base) / (64 * kb)); cr >= 2; --cr) {
    lr = (220 * 1024 - cr * 2 * b) / (a + b);
    if (lr >= (kb == 1 ? 4 : 3) || cr == 2) break;
  }
  lr = std::max(2, std::min(lr, 8));
}

static size_t tc_smem(int N, int kb, int lr, int cr) {
  const int b = N * 128 * kb;
  return 1024 + static_cast<size_t>(lr) * (16384 * kb + b) + static_cast<size_t>(cr) * 2 * b +
         8 * (2 * lr + 2 * cr + 2) + 16;
}

template <bool A_MN, int KB>
static void launch_sweep_kb(const Plan& P, const TcMaps* maps, const int4* d_tiles, int grid,
                            const int* d_off, float* out, float* part, cudaStream_t s) {
  const int N = tc_n(P);
  int lr = 0, cr = 0;
  tc_rings(N, KB, lr, cr);
  const size_t sm = tc_smem(N, KB, lr, cr);
  smem_optin(reinterpret_cast<const void*>(k_tc_sweep<A_MN, KB>), 227 * 1024);
  static const int hints = [] {  // experiments: DLX_SWEEP_HINTS=0 drops the L2 cache hints
    const char* e = getenv("DLX_SWEEP_HINTS");
    return e ? atoi(e) : 1;
  }();
  k_tc_sweep<A_MN, KB><<<grid, kTcThreads, sm, s>>>(P.d_t2, maps, d_tiles, d_off, N, lr, cr,
                                                    P.d_k2_splits, P.d_k2_part_off, out, part,
                                                    hints);
}

template <bool A_MN>
static void launch_sweep(const Plan& P, const TcMaps* maps, const std::vector<int4>& tiles,
                         const int4* d_tiles, const std::vector<int>& off, const int* d_off,
                         float* out, float* part, cudaStream_t s) {
  if (tiles.empty()) return;
  const int grid = static_cast<int>(off.size()) - 1;
  // algorithmic bytes: one fp32 read of every swept delta element (factors are L2-resident)
  KernelTimer timer(A_MN ? "k_tc_sweep_k2" : "k_tc_sweep_k1", 4.0 * tc_state(P).swept_params, s);
  if (tc_kb(tc_n(P)) == 2)
    launch_sweep_kb<A_MN, 2>(P, maps, d_tiles, grid, d_off, out, part, s);
  else
    launch_sweep_kb<A_MN, 1>(P, maps, d_tiles, grid, d_off, out, part, s);
  DLX_LAUNCHED();
}

// Tensor-core sweeps for the eligible tensors; returns false if the plan is outside the
// tcgen05 path (then the SIMT kernels handle every tensor).
bool tc_supported(const Plan& P) { return P.rmax >= 1 && P.rmax <= 256; }

void launch_k1_tc(const Plan& P, const float* slab, const float* q, float* y, cudaStream_t s) {
  TcState& S = tc_state(P);
  const TcMaps* maps = tc_maps(P, 0, slab, q, s);
  launch_sweep<false>(P, maps, S.k1, S.d_k1, S.off1, S.d_off1, y, nullptr, s);
}

void launch_k2_tc(const Plan& P, const float* slab, const float* p, float* z, float* part,
                  cudaStream_t s) {
  TcState& S = tc_state(P);
  const TcMaps* maps = tc_maps(P, 1, slab, p, s);
  launch_sweep<true>(P, maps, S.k2, S.d_k2, S.off2, S.d_off2, z, part, s);
}

}  // namespace dlx
