// dlx_internal.cuh — shared device/host definitions of the B200 outer-sync library.
#pragma once
#include <cuda_runtime.h>
#include <algorithm>
#include <cstring>
#include <exception>
#include <stdint.h>

#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "../../include/dlx_b200.h"

namespace dlx {

// ------------------------------------------------------------------ errors / launches
struct Error {
  dlx_status code;
  std::string msg;
};
struct Comm;  // comm.cu: NCCL communicator + exchange stream of a context
void destroy_comm(Comm* c);
// Derived state owned by a Plan (per rank) or by a layout (rank-independent tables), freed
// with its owner (no address-keyed global caches).
struct PlanExt {
  virtual ~PlanExt() = default;
};
[[noreturn]] void raise(dlx_status code, const std::string& msg);
void set_last_error(const std::string& msg);  // dlx_last_error() of the calling thread
// Runs f, mapping a thrown Error to its status code (and the message to dlx_last_error).
template <class F>
dlx_status guard(F&& f) {
  try {
    f();
    return DLX_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return DLX_ERR_VALIDATION;
  }
}
void check_cuda(cudaError_t e, const char* what);
void count_launch(int n = 1);
// Opt kernel `func` into `bytes` of dynamic shared memory on the CURRENT device. The
// attribute is per device, so the opt-in is cached per (device, kernel, bytes): a second
// context on another device in the same process gets its own.
void smem_optin(const void* func, int bytes);
// NVTX range over one C-ABI stage (compress, exchange, outer update, effective rank): free
// unless a tool (nsys / ncu --nvtx) is attached — NVTX v3 is header-only and loads the
// injection library only then.
struct NvtxRange {
  explicit NvtxRange(const char* name);
  ~NvtxRange();
};

// Host-side wall time per scope, reported at exit when DLX_HOST_PROF=1 (where the host
// spends its time between launches: plan / state builds on a rank change, waits).
struct HostProf {
  explicit HostProf(const char* name);
  ~HostProf();
  const char* name;
  double t0;
  bool on;
};
// Host -> device copy of a small table that returns once the bytes have landed, issued on a
// per-device non-blocking stream: unlike cudaMemcpy it does not wait for the work queued on
// the legacy default stream (a plan built while the previous round's outer update still
// runs — a rank change under the adaptive schedule — must not drain the GPU).
void upload_now(void* dst, const void* src, size_t bytes);
#define DLX_CUDA(x) ::dlx::check_cuda((x), #x)
#define DLX_LAUNCHED() do { ::dlx::check_cuda(cudaGetLastError(), "kernel launch"); ::dlx::count_launch(); } while (0)

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int64_t ceil_div(int64_t x, int64_t m) { return (x + m - 1) / m; }

// ------------------------------------------------------------------ splitmix64 (rng.hpp)
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;

__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) { return fmix64(z + kGolden); }
// k-th draw (1-based) of a stream whose state after construction is s0 (rng.hpp:25-31):
// the counter-based form that lets every element address its own draw.
__host__ __device__ __forceinline__ uint64_t draw_at(uint64_t s0, uint64_t k) {
  return fmix64(s0 + k * kGolden);
}
__device__ __forceinline__ float unit_f(uint64_t v) {  // rng.hpp:37
  return __fmul_rn((float)(uint32_t)(v >> 40), 0x1.0p-24f);
}
__device__ __forceinline__ double unit_d(uint64_t v) {  // rng.hpp:34
  return __dmul_rn((double)(v >> 11), 0x1.0p-53);
}
__host__ __device__ __forceinline__ uint64_t stream_init(uint64_t seed, uint64_t sid) {
  // rng.hpp:13-16
  uint64_t s = mix64(seed ^ kGolden);
  return mix64(s ^ mix64(sid + 0xbf58476d1ce4e5b9ull));
}
__host__ __device__ __forceinline__ uint64_t stream_key4(uint64_t a, uint64_t b, uint64_t c,
                                                         uint64_t d) {  // rng.hpp:63-66
  uint64_t h = 0x100000001b3ull;
  h = mix64(h ^ mix64(a));
  h = mix64(h ^ mix64(b));
  h = mix64(h ^ mix64(c));
  return mix64(h ^ mix64(d));
}
inline uint64_t stream_key(std::initializer_list<uint64_t> parts) {  // rng.hpp:63-66
  uint64_t h = 0x100000001b3ull;
  for (uint64_t p : parts) h = mix64(h ^ mix64(p));
  return h;
}

// ------------------------------------------------------------------ plan tables (device)
// One 2-D tensor of the table with its factor / payload geometry for a given rank.
struct DevT2 {
  int64_t a, b;         // rows, cols of delta (row-major, ld = b)
  int64_t off;          // slab element offset
  int64_t lda, ldb;     // padded column strides of the P (a) and Q (b) factor buffers
  int64_t poff, qoff;   // element offsets into the P / Q factor buffers
  int64_t seg_pc, seg_qc, seg_ps, seg_qs;  // payload byte offsets
  int r;                // r_eff = min(rank, a, b)
  int idx;              // table index
};
struct DevT1 {
  int64_t n, off;       // length, slab offset
  int64_t seg_c, seg_s; // payload byte offsets
  int idx, pad;
};
// Quantisation chunk (one factor column or one 1-D tensor), in draw order.
struct DevChunk {
  int64_t src;          // element offset into its buffer
  int64_t len;
  int64_t scale_dst;    // payload byte offset of its fp32 scale
  int64_t extra;        // draws consumed right before this chunk (cold-start init)
  int buf;              // 0 = P factors, 1 = Q factors, 2 = slab
  int tensor;           // 2-D slot for factor chunks, -1 for 1-D tensors
};
// Code stream (one factor, or one 1-D tensor): packed contiguously in the payload.
struct DevStream {
  int64_t src, ld, col_len, ncols;
  int64_t chunk0;       // chunk index of column 0
  int64_t code_dst;     // payload byte offset
  int64_t group0;       // first 8-code group id of this stream (global numbering)
  int buf, t2;          // buffer id; 2-D tensor slot (or -1)
};
// Batched small-matrix entry for orthonormalisation / Gram work.
struct DevMat {
  int64_t off;          // element offset in its buffer (column-major, ld)
  int64_t n, ld;        // rows, column stride
  int r;                // columns
  int slot;             // index into per-entry scratch
};

struct Plan;

}  // namespace dlx

struct dlx_ctx {
  int device = 0;
  cudaStream_t internal = nullptr;
  dlx::Comm* comm = nullptr;  // dlx_comm_init (worker sync); null = single worker
  cudaStream_t capture = nullptr;  // private stream for CUDA-graph captures (cold-start redo)
  // grow-only scratch arenas
  std::map<std::string, std::pair<void*, size_t>> arenas;
  void* scratch(const std::string& name, size_t bytes, bool zero = false);
  ~dlx_ctx();
};

struct dlx_layout {
  dlx_ctx* ctx = nullptr;
  int nt = 0;
  std::vector<int> ndim;
  std::vector<int64_t> dims;     // 2 per tensor
  std::vector<int64_t> offsets;  // slab offsets
  int64_t slab = 0;
  std::map<std::pair<int, int>, std::unique_ptr<dlx::Plan>> plans;
  void* d_spans = nullptr;  // staging-kernel tensor table (device), freed with the layout
  // rank-independent derived tables (work lists that every plan of this layout shares, so a
  // rank change under the adaptive schedule does not rebuild them)
  std::map<std::string, std::unique_ptr<dlx::PlanExt>> ext;
  dlx::Plan& plan(int rank, int qbits);
  ~dlx_layout() {
    if (d_spans) cudaFree(d_spans);
  }
  int64_t numel(int i) const { return ndim[i] == 2 ? dims[2 * i] * dims[2 * i + 1] : dims[2 * i]; }
};

namespace dlx {


// Host + device description of (layout, rank, qbits).
struct Plan {
  const dlx_layout* layout = nullptr;  // the owning layout (layout_ext tables)
  int rank = 0, qbits = 0;
  std::vector<DevT2> t2;
  std::vector<DevT1> t1;
  std::vector<DevChunk> chunks;
  std::vector<DevStream> streams;
  int64_t payload_bytes = 0;
  uint64_t payload_bits = 0;
  int64_t pelems = 0, qelems = 0;  // factor buffer sizes (elements)
  int64_t ngroups = 0;             // 8-code groups over all streams
  int rmax = 0;                    // max r_eff
  // device copies
  DevT2* d_t2 = nullptr;
  DevT1* d_t1 = nullptr;
  DevChunk* d_chunks = nullptr;
  DevStream* d_streams = nullptr;
  // matrices for the batched Gram/ortho over P (side 0) and Q (side 1)
  std::vector<DevMat> mats[2];
  DevMat* d_mats[2] = {nullptr, nullptr};
  // work tiles
  std::vector<int4> k1_tiles;  // (t2 slot, m0, n0, -)
  std::vector<int4> k2_tiles;  // (t2 slot, j0, c0, split)
  std::vector<int> k2_splits;  // per t2 slot
  std::vector<int64_t> k2_part_off;  // per t2 slot: element offset into the partial buffer
  int64_t k2_part_elems = 0;
  int4* d_k1_tiles = nullptr;
  int4* d_k2_tiles = nullptr;
  int64_t* d_k2_part_off = nullptr;
  int* d_k2_splits = nullptr;
  std::vector<int4> k1_rest, k2_rest;  // SIMT tiles of tensors outside the tcgen05 path
  int4* d_k1_rest = nullptr;
  int4* d_k2_rest = nullptr;
  // speculative cold-start draw bases per 2-D slot, [0] stochastic (assumes no all-zero
  // chunk), [1] nearest (exact: quantisation draws nothing)
  std::vector<int64_t> cold_base_spec[2];
  int64_t* d_cold_base_spec[2] = {nullptr, nullptr};
  // derived state + device buffers owned by the plan
  std::map<std::string, std::unique_ptr<PlanExt>> ext;
  std::vector<void*> owned;
  void* dev_alloc(size_t bytes) const;  // cudaMalloc, freed in ~Plan
  ~Plan();
};

// Typed layout-level ext slot (see dlx_layout::ext).
template <class T>
T& layout_ext(const dlx_layout& L, const std::string& key, bool* fresh = nullptr) {
  auto& e = const_cast<dlx_layout&>(L).ext[key];
  if (fresh) *fresh = !e;
  if (!e) e.reset(new T());
  return *static_cast<T*>(e.get());
}

// Typed ext slot: created empty (default-constructed) on first use; *fresh tells the caller.
template <class T>
T& plan_ext(const Plan& P, const std::string& key, bool* fresh = nullptr) {
  auto& e = const_cast<Plan&>(P).ext[key];
  if (fresh) *fresh = !e;
  if (!e) e.reset(new T());
  return *static_cast<T*>(e.get());
}

// Device copies of per-tensor TMA descriptor tables, keyed by the buffer addresses they were
// encoded for. A caller that alternates buffers (ping-pong local / anchor slabs) hits the
// cache instead of re-encoding. A new entry is encoded on the host and uploaded with
// upload_now (a private non-blocking stream: no wait for the compute streams, no pinned
// allocation — cudaMallocHost measured multi-ms stalls with several processes per node);
// only evicting an entry (more than kEntries distinct keys) waits for the device, since
// in-flight kernels may still read the evicted table.
template <class T, int NK>
struct MapTableCache : PlanExt {
  static constexpr int kEntries = 4;
  struct Entry {
    const void* key[NK];
    T* dev = nullptr;
    uint64_t used = 0;
  };
  std::vector<Entry> entries;
  uint64_t tick = 0;
  ~MapTableCache() override {
    for (Entry& e : entries)
      if (e.dev) cudaFree(e.dev);
  }
  // Returns the device table for `key`; `encode(T* host)` fills a new table of n entries.
  template <class F>
  const T* get(const void* const* key, size_t n, cudaStream_t s, F&& encode) {
    ++tick;
    for (Entry& e : entries)
      if (std::equal(key, key + NK, e.key)) {
        e.used = tick;
        return e.dev;
      }
    if (static_cast<int>(entries.size()) >= kEntries) {
      auto victim = std::min_element(entries.begin(), entries.end(),
                                     [](const Entry& x, const Entry& y) { return x.used < y.used; });
      DLX_CUDA(cudaDeviceSynchronize());
      cudaFree(victim->dev);
      entries.erase(victim);
    }
    HostProf hp("map_table (new)");
    Entry e{};
    std::copy(key, key + NK, e.key);
    const size_t bytes = sizeof(T) * std::max<size_t>(n, 1);
    std::vector<T> host(std::max<size_t>(n, 1));
    std::memset(static_cast<void*>(host.data()), 0, bytes);
    encode(host.data());
    DLX_CUDA(cudaMalloc(&e.dev, bytes));
    upload_now(e.dev, host.data(), bytes);
    (void)s;
    e.used = tick;
    entries.push_back(e);
    return entries.back().dev;
  }
};

// Upload a host vector into a plan-owned device buffer (at least min_elems elements).
template <class T>
T* plan_upload(const Plan& P, const std::vector<T>& v, size_t min_elems = 0) {
  const size_t n = std::max(v.size(), min_elems);
  if (n == 0) return nullptr;
  T* d = static_cast<T*>(P.dev_alloc(sizeof(T) * n));
  if (!v.empty()) upload_now(d, v.data(), sizeof(T) * v.size());
  return d;
}

// Kernel launchers (csrc/*.cu)
void launch_fill_gaussian(const dlx_layout& L, float* out, const float* base, float scale,
                          uint64_t seed, uint64_t tag, uint64_t worker, cudaStream_t s);
// s0p (nullable): read the stream state from device memory instead of s0 (graph replays)
void launch_cold_init(const Plan& P, float* q, const int64_t* d_cold_base, uint64_t s0,
                      cudaStream_t s, const uint64_t* s0p = nullptr);
void launch_k1(const Plan& P, const float* slab, const float* q, float* y, cudaStream_t s);
bool tc_supported(const Plan& P);
bool tc_eligible(const DevT2& t);
void launch_k1_tc(const Plan& P, const float* slab, const float* q, float* y, cudaStream_t s);
void launch_k2_tc(const Plan& P, const float* slab, const float* p, float* z, float* part,
                  cudaStream_t s);
bool& option_tensor_cores();
bool& option_outer_tc();
int& option_effrank_big_from();
bool& option_cholblk();

// Optional CUDA-event timing of the dominant kernels (dlx_set_option("kernel_events", 1)):
// events recorded on the launching stream around one launch, with the launch's algorithmic
// HBM bytes; read back (and cleared) by dlx_kernel_time. Off by default (no events).
struct KernelTimer {
  KernelTimer(const char* name, double bytes, cudaStream_t s);
  ~KernelTimer();
  int slot = -1;
  cudaStream_t stream = nullptr;
};
void launch_k2(const Plan& P, const float* slab, const float* p, float* z, float* part,
               cudaStream_t s);
void orthonormalize_batched(dlx_ctx* ctx, const Plan& P, int side, float* buf, float* tmp,
                            cudaStream_t s);
void quantize_all(dlx_ctx* ctx, const Plan& P, const float* pbuf, const float* qbuf,
                  const float* slab, int rounding, uint64_t s0, int cold,
                  const int64_t* d_cold_base_used, uint8_t* payload, uint64_t* d_draws,
                  int* d_mismatch, int64_t* d_cold_base_actual, cudaStream_t s,
                  const uint64_t* s0p = nullptr);
void dequant_factors(const Plan& P, int D, const uint8_t* gathered, int64_t pay_bytes,
                     float* phat, float* qhat, int64_t lda_tot, cudaStream_t s);
// Slot ranges of one outer-update call: 2-D slots [s0, s1), 1-D slots [u0, u1) (the tensors
// of a layout index range; the whole layout by default).
struct SlotRange {
  int s0 = 0, s1 = 0, u0 = 0, u1 = 0;
  bool full(const Plan& P) const {
    return s0 == 0 && s1 == static_cast<int>(P.t2.size()) && u0 == 0 &&
           u1 == static_cast<int>(P.t1.size());
  }
  std::string key() const {
    return std::to_string(s0) + ":" + std::to_string(s1) + ":" + std::to_string(u0) + ":" +
           std::to_string(u1);
  }
};
SlotRange slot_range(const Plan& P, int t_begin, int t_end);

void launch_outer_2d(dlx_ctx* ctx, const Plan& P, int D, const uint8_t* gathered,
                     int self_index, int mode, float* pending, float* anchor,
                     const float* local, float* velocity, float gamma, float beta,
                     int classical, dlx_round_stats* stats, const SlotRange& R, cudaStream_t s);
void launch_outer_1d(const Plan& P, int D, const uint8_t* gathered, int self_index, int mode,
                     float* pending, float* anchor, const float* local, float* velocity,
                     float gamma, float beta, int classical, dlx_round_stats* stats,
                     const SlotRange& R, cudaStream_t s);
void launch_reconstruct_dense(dlx_ctx* ctx, const Plan& P, int D, const uint8_t* gathered,
                              float* out, cudaStream_t s);
void launch_outer_raw(const dlx_layout& L, int D, const float* gathered, int self_index, int mode,
                      float* pending, float* anchor, const float* local, float* velocity,
                      float gamma, float beta, int classical, dlx_round_stats* stats,
                      cudaStream_t s);
void launch_adamw(int64_t n, float lr, float beta1, float beta2, float eps, float wd,
                  int64_t warmup_steps, int64_t step, float* p, const float* g, float* m,
                  float* v, int* nonfinite, cudaStream_t s);
void launch_stage(const dlx_layout& L, const float* anchor, const float* local,
                  const float* err, float* pending, double* norm_sq, cudaStream_t s);
void launch_sqdiff(const dlx_layout& L, const float* rec, const float* delta, double* out,
                   cudaStream_t s);
void launch_mean_slabs(int64_t n, int64_t ld, const float* x, int D, float* out, cudaStream_t s);
void launch_nesterov(int64_t n, float gamma, float beta, int classical, float* anchor,
                     float* v, const float* delta, cudaStream_t s);
void effective_rank_factors(dlx_ctx* ctx, const Plan& P, int D, const uint8_t* gathered,
                            double tau, int* d_per, double* d_energy, int shard, int nshards,
                            cudaStream_t s);

}  // namespace dlx
