// api.cu — C-ABI entry points (include/dlx_b200.h): validation, plans, orchestration.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <set>
#include <tuple>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "dlx_internal.cuh"

namespace dlx {

static thread_local std::string g_last_error;
static thread_local uint64_t g_launches = 0;

[[noreturn]] void raise(dlx_status code, const std::string& msg) { throw Error{code, msg}; }

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(DLX_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void count_launch(int n) { g_launches += static_cast<uint64_t>(n); }

NvtxRange::NvtxRange(const char* name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }

namespace {
struct ProfEntry {
  int64_t calls = 0;
  double total = 0.0, max = 0.0;
};
std::mutex g_prof_mu;
std::map<std::string, ProfEntry>* g_prof = nullptr;
double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}
bool prof_on() {
  static const bool on = [] {
    const char* e = getenv("DLX_HOST_PROF");
    if (!(e && e[0] == '1')) return false;
    g_prof = new std::map<std::string, ProfEntry>();
    atexit([] {
      for (auto& kv : *g_prof)
        fprintf(stderr, "[dlx host] %-28s calls %6lld total %9.2f ms max %8.3f ms\n",
                kv.first.c_str(), static_cast<long long>(kv.second.calls), kv.second.total,
                kv.second.max);
    });
    return true;
  }();
  return on;
}
}  // namespace

HostProf::HostProf(const char* n) : name(n), t0(0.0), on(prof_on()) {
  if (on) t0 = now_ms();
}
HostProf::~HostProf() {
  if (!on) return;
  const double dt = now_ms() - t0;
  std::lock_guard<std::mutex> lock(g_prof_mu);
  ProfEntry& e = (*g_prof)[name];
  ++e.calls;
  e.total += dt;
  e.max = std::max(e.max, dt);
}

void upload_now(void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  static std::mutex mu;
  static std::map<int, cudaStream_t> streams;
  int dev = 0;
  DLX_CUDA(cudaGetDevice(&dev));
  cudaStream_t s = nullptr;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = streams.find(dev);
    if (it == streams.end()) {
      DLX_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      streams[dev] = s;
    } else {
      s = it->second;
    }
  }
  DLX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
  DLX_CUDA(cudaStreamSynchronize(s));
}

void smem_optin(const void* func, int bytes) {
  static std::mutex mu;
  static std::set<std::tuple<int, const void*, int>> done;
  int dev = 0;
  DLX_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({dev, func, bytes})) return;
  DLX_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert({dev, func, bytes});
}

namespace {
struct TimedLaunch {
  std::string name;
  double bytes;
  cudaEvent_t a, b;
};
bool g_kernel_events = false;
std::vector<TimedLaunch> g_timed;  // recorded launches (events owned, destroyed on read)
}  // namespace

KernelTimer::KernelTimer(const char* name, double bytes, cudaStream_t s) : stream(s) {
  if (!g_kernel_events) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) return;
  TimedLaunch t{name, bytes, nullptr, nullptr};
  DLX_CUDA(cudaEventCreate(&t.a));
  DLX_CUDA(cudaEventCreate(&t.b));
  DLX_CUDA(cudaEventRecord(t.a, s));
  slot = static_cast<int>(g_timed.size());
  g_timed.push_back(t);
}

KernelTimer::~KernelTimer() {
  if (slot >= 0) cudaEventRecord(g_timed[slot].b, stream);
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

template <class T>
static T* upload(const std::vector<T>& v) {
  if (v.empty()) return nullptr;
  T* d = nullptr;
  DLX_CUDA(cudaMalloc(&d, sizeof(T) * v.size()));
  upload_now(d, v.data(), sizeof(T) * v.size());
  return d;
}

void* Plan::dev_alloc(size_t bytes) const {
  void* p = nullptr;
  DLX_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
  const_cast<Plan*>(this)->owned.push_back(p);
  return p;
}

Plan::~Plan() {
  for (void* p : owned) cudaFree(p);
  void* ptrs[] = {d_t2, d_t1, d_chunks, d_streams, d_mats[0], d_mats[1], d_k1_tiles,
                  d_k2_tiles, d_k2_part_off, d_k2_splits, d_cold_base_spec[0],
                  d_cold_base_spec[1], d_k1_rest, d_k2_rest};
  for (void* p : ptrs)
    if (p) cudaFree(p);
}

static void validate_quant(int rank, int qbits) {
  if (qbits < 2 || qbits > 8) raise(DLX_ERR_VALIDATION, "quantization bits must be in [2, 8]");
  if (rank < 1) raise(DLX_ERR_VALIDATION, "compress: rank must be >= 1");
}

static std::unique_ptr<Plan> build_plan(const dlx_layout& L, int rank, int qbits) {
  HostProf hp("build_plan");
  auto P = std::make_unique<Plan>();
  P->layout = &L;
  P->rank = rank;
  P->qbits = qbits;
  int64_t cur = 0, poff = 0, qoff = 0;
  auto codes_bytes = [&](int64_t n) { return ceil_div(n * qbits, 8); };
  for (int i = 0; i < L.nt; ++i) {
    if (L.ndim[i] == 2) {
      DevT2 t{};
      t.a = L.dims[2 * i];
      t.b = L.dims[2 * i + 1];
      t.off = L.offsets[i];
      t.r = static_cast<int>(std::min<int64_t>(rank, std::min(t.a, t.b)));
      t.idx = i;
      t.lda = round_up(t.a, 32);
      t.ldb = round_up(t.b, 32);
      t.poff = poff;
      t.qoff = qoff;
      poff += t.lda * t.r;
      qoff += t.ldb * t.r;
      t.seg_pc = cur;
      cur = round_up(cur + codes_bytes(t.a * t.r), 16);
      t.seg_qc = cur;
      cur = round_up(cur + codes_bytes(t.b * t.r), 16);
      t.seg_ps = cur;
      cur += 4 * t.r;
      t.seg_qs = cur;
      cur = round_up(cur + 4 * t.r, 16);
      P->rmax = std::max(P->rmax, t.r);
      P->t2.push_back(t);
      P->payload_bits += static_cast<uint64_t>(t.a + t.b) * t.r * qbits + 64ull * t.r;
    } else {
      DevT1 t{};
      t.n = L.dims[2 * i];
      t.off = L.offsets[i];
      t.idx = i;
      t.seg_c = cur;
      cur = round_up(cur + codes_bytes(t.n), 16);
      t.seg_s = cur;
      cur = round_up(cur + 4, 16);
      P->t1.push_back(t);
      P->payload_bits += static_cast<uint64_t>(t.n) * qbits + 32ull;
    }
  }
  P->payload_bytes = cur;
  P->pelems = std::max<int64_t>(poff, 32);
  P->qelems = std::max<int64_t>(qoff, 32);

  // chunks + streams in reference draw order (compress.cpp:153-180)
  int s2 = 0, s1 = 0;
  int64_t group = 0;
  for (int i = 0; i < L.nt; ++i) {
    if (L.ndim[i] == 2) {
      const DevT2& t = P->t2[s2];
      for (int side = 0; side < 2; ++side) {
        const int64_t len = side == 0 ? t.a : t.b;
        const int64_t ld = side == 0 ? t.lda : t.ldb;
        const int64_t base = side == 0 ? t.poff : t.qoff;
        DevStream st{};
        st.src = base;
        st.ld = ld;
        st.col_len = len;
        st.ncols = t.r;
        st.chunk0 = static_cast<int64_t>(P->chunks.size());
        st.code_dst = side == 0 ? t.seg_pc : t.seg_qc;
        st.group0 = group;
        st.buf = side;
        st.t2 = s2;
        group += ceil_div(len * t.r, 8);
        P->streams.push_back(st);
        for (int j = 0; j < t.r; ++j) {
          DevChunk c{};
          c.src = base + j * ld;
          c.len = len;
          c.scale_dst = (side == 0 ? t.seg_ps : t.seg_qs) + 4 * j;
          c.extra = (side == 0 && j == 0) ? t.b * t.r : 0;  // cold init precedes P (compress.cpp:64-69)
          c.buf = side;
          c.tensor = s2;  // 2-D slot
          P->chunks.push_back(c);
        }
      }
      ++s2;
    } else {
      const DevT1& t = P->t1[s1];
      DevStream st{};
      st.src = t.off;
      st.ld = t.n;
      st.col_len = t.n;
      st.ncols = 1;
      st.chunk0 = static_cast<int64_t>(P->chunks.size());
      st.code_dst = t.seg_c;
      st.group0 = group;
      st.buf = 2;
      st.t2 = -1;
      group += ceil_div(t.n, 8);
      P->streams.push_back(st);
      DevChunk c{};
      c.src = t.off;
      c.len = t.n;
      c.scale_dst = t.seg_s;
      c.extra = 0;
      c.buf = 2;
      c.tensor = -1;
      P->chunks.push_back(c);
      ++s1;
    }
  }
  P->ngroups = group;

  // speculative cold-start bases
  for (int mode = 0; mode < 2; ++mode) {
    int64_t O = 0;
    int k2 = 0;
    for (int i = 0; i < L.nt; ++i) {
      if (L.ndim[i] == 2) {
        const DevT2& t = P->t2[k2++];
        P->cold_base_spec[mode].push_back(O);
        O += t.b * t.r;
        if (mode == 0) O += (t.a + t.b) * t.r;
      } else if (mode == 0) {
        O += L.dims[2 * i];
      }
    }
  }

  // batched ortho entries
  for (size_t k = 0; k < P->t2.size(); ++k) {
    const DevT2& t = P->t2[k];
    P->mats[0].push_back(DevMat{t.poff, t.a, t.lda, t.r, static_cast<int>(k)});
    P->mats[1].push_back(DevMat{t.qoff, t.b, t.ldb, t.r, static_cast<int>(k)});
  }

  // K1 tiles: Y = delta Q, rows of delta in BM blocks, factor columns in BN blocks
  const int bm1 = P->rmax <= 32 ? 128 : 64, bn1 = P->rmax <= 32 ? 32 : 64;
  // K2 tiles: Z = delta^T P, columns of delta in 64-blocks, k split in 2048-row chunks
  const int bc2 = P->rmax <= 32 ? 32 : 64;
  const int64_t kc = 2048;
  int64_t part = 0;
  for (size_t k = 0; k < P->t2.size(); ++k) {
    const DevT2& t = P->t2[k];
    const bool tc = tc_eligible(t);
    for (int64_t m0 = 0; m0 < t.a; m0 += bm1)
      for (int n0 = 0; n0 < t.r; n0 += bn1) {
        P->k1_tiles.push_back(make_int4(static_cast<int>(k), static_cast<int>(m0), n0, 0));
        if (!tc) P->k1_rest.push_back(P->k1_tiles.back());
      }
    const int splits = static_cast<int>(ceil_div(t.a, kc));
    P->k2_splits.push_back(splits);
    P->k2_part_off.push_back(part);
    if (splits > 1) part += static_cast<int64_t>(splits) * t.ldb * t.r;
    for (int s = 0; s < splits; ++s)
      for (int64_t j0 = 0; j0 < t.b; j0 += 64)
        for (int c0 = 0; c0 < t.r; c0 += bc2) {
          P->k2_tiles.push_back(make_int4(static_cast<int>(k), static_cast<int>(j0), c0, s));
          if (!tc) P->k2_rest.push_back(P->k2_tiles.back());
        }
  }
  P->k2_part_elems = std::max<int64_t>(part, 32);

  P->d_t2 = upload(P->t2);
  P->d_t1 = upload(P->t1);
  P->d_chunks = upload(P->chunks);
  P->d_streams = upload(P->streams);
  P->d_mats[0] = upload(P->mats[0]);
  P->d_mats[1] = upload(P->mats[1]);
  P->d_k1_tiles = upload(P->k1_tiles);
  P->d_k2_tiles = upload(P->k2_tiles);
  P->d_k2_part_off = upload(P->k2_part_off);
  P->d_k2_splits = upload(P->k2_splits);
  P->d_k1_rest = upload(P->k1_rest);
  P->d_k2_rest = upload(P->k2_rest);
  P->d_cold_base_spec[0] = upload(P->cold_base_spec[0]);
  P->d_cold_base_spec[1] = upload(P->cold_base_spec[1]);
  return P;
}

}  // namespace dlx

using namespace dlx;

void* dlx_ctx::scratch(const std::string& name, size_t bytes, bool zero) {
  auto it = arenas.find(name);
  if (it != arenas.end() && it->second.second >= bytes) {
    if (zero) DLX_CUDA(cudaMemsetAsync(it->second.first, 0, bytes, internal));
    return it->second.first;
  }
  if (it != arenas.end()) {
    DLX_CUDA(cudaDeviceSynchronize());
    cudaFree(it->second.first);
    arenas.erase(it);
  }
  void* p = nullptr;
  bytes = std::max<size_t>(bytes, 256);
  DLX_CUDA(cudaMalloc(&p, bytes));
  DLX_CUDA(cudaMemset(p, 0, bytes));
  arenas[name] = {p, bytes};
  return p;
}

dlx_ctx::~dlx_ctx() {
  if (comm) dlx::destroy_comm(comm);
  if (capture) cudaStreamDestroy(capture);
  for (auto& kv : arenas) cudaFree(kv.second.first);
  if (internal) cudaStreamDestroy(internal);
}

Plan& dlx_layout::plan(int rank, int qbits) {
  auto key = std::make_pair(rank, qbits);
  auto it = plans.find(key);
  if (it == plans.end()) it = plans.emplace(key, build_plan(*this, rank, qbits)).first;
  return *it->second;
}

static cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static void set_device(dlx_ctx* ctx) {
  if (!ctx) raise(DLX_ERR_VALIDATION, "null context");
  DLX_CUDA(cudaSetDevice(ctx->device));
}

extern "C" {

const char* dlx_version(void) { return "dlx_b200 0.1 (sm_100a)"; }
const char* dlx_last_error(void) { return g_last_error.c_str(); }
dlx_status dlx_set_option(const char* key, int value) {
  return guard([&] {
    const std::string k = key ? key : "";
    if (k == "tensor_cores") {
      option_tensor_cores() = value != 0;
    } else if (k == "outer_tensor_cores") {
      option_outer_tc() = value != 0;
    } else if (k == "effrank_big_from") {
      option_effrank_big_from() = value;
    } else if (k == "cholqr_blocked") {
      option_cholblk() = value != 0;
    } else if (k == "kernel_events") {
      g_kernel_events = value != 0;
    } else {
      raise(DLX_ERR_VALIDATION, "unknown option: " + k);
    }
  });
}

dlx_status dlx_debug_sweep(dlx_ctx* ctx, const dlx_layout* layout, int rank, int which,
                           const float* d_slab, const float* d_in, float* d_out, int use_tc,
                           void* stream) {
  return guard([&] {
    set_device(ctx);
    Plan& P = const_cast<dlx_layout*>(layout)->plan(rank, 8);
    const bool saved = option_tensor_cores();
    option_tensor_cores() = use_tc != 0;
    cudaStream_t s = as_stream(stream);
    if (which == 0) {
      launch_k1(P, d_slab, d_in, d_out, s);
    } else {
      float* part = static_cast<float*>(ctx->scratch("k2part", sizeof(float) * P.k2_part_elems));
      launch_k2(P, d_slab, d_in, d_out, part, s);
    }
    option_tensor_cores() = saved;
  });
}

dlx_status dlx_kernel_time(const char* name, double* ms_total, double* bytes_total,
                           int64_t* launches) {
  return guard([&] {
    const std::string n = name ? name : "";
    double ms = 0.0, bytes = 0.0;
    int64_t cnt = 0;
    std::vector<TimedLaunch> keep;
    for (TimedLaunch& t : g_timed) {
      if (t.name != n) {
        keep.push_back(t);
        continue;
      }
      DLX_CUDA(cudaEventSynchronize(t.b));
      float x = 0.f;
      DLX_CUDA(cudaEventElapsedTime(&x, t.a, t.b));
      ms += x;
      bytes += t.bytes;
      ++cnt;
      cudaEventDestroy(t.a);
      cudaEventDestroy(t.b);
    }
    g_timed.swap(keep);
    if (ms_total) *ms_total = ms;
    if (bytes_total) *bytes_total = bytes;
    if (launches) *launches = cnt;
  });
}

uint64_t dlx_take_launch_count(void) {
  const uint64_t n = g_launches;
  g_launches = 0;
  return n;
}

dlx_status dlx_ctx_create(int device, dlx_ctx** out) {
  return guard([&] {
    int n = 0;
    DLX_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) raise(DLX_ERR_VALIDATION, "bad device index");
    DLX_CUDA(cudaSetDevice(device));
    auto* c = new dlx_ctx();
    c->device = device;
    DLX_CUDA(cudaStreamCreateWithFlags(&c->internal, cudaStreamNonBlocking));
    *out = c;
  });
}

dlx_status dlx_ctx_create_dist(int device, int rank, int world, const void* unique_id,
                               dlx_ctx** out) {
  dlx_ctx* c = nullptr;
  dlx_status st = dlx_ctx_create(device, &c);
  if (st != DLX_OK) return st;
  st = dlx_comm_init(c, rank, world, unique_id);
  if (st != DLX_OK) {
    const std::string msg = g_last_error;
    dlx_ctx_destroy(c);
    g_last_error = msg;
    return st;
  }
  *out = c;
  return DLX_OK;
}

dlx_status dlx_ctx_destroy(dlx_ctx* ctx) {
  return guard([&] {
    if (ctx) {
      cudaSetDevice(ctx->device);
      cudaDeviceSynchronize();
      delete ctx;
    }
  });
}

dlx_status dlx_layout_create(dlx_ctx* ctx, int nt, const int* ndim, const int64_t* dims,
                             dlx_layout** out) {
  return guard([&] {
    set_device(ctx);
    if (nt < 0) raise(DLX_ERR_VALIDATION, "negative tensor count");
    auto* L = new dlx_layout();
    L->ctx = ctx;
    L->nt = nt;
    int64_t off = 0;
    for (int i = 0; i < nt; ++i) {
      if (ndim[i] != 1 && ndim[i] != 2) {
        delete L;
        raise(DLX_ERR_SHAPE, "compress: only 1-D and 2-D tensors are supported");
      }
      const int64_t d0 = dims[2 * i], d1 = ndim[i] == 2 ? dims[2 * i + 1] : 1;
      if (d0 <= 0 || d1 <= 0) {
        delete L;
        raise(DLX_ERR_SHAPE, "tensor dimensions must be positive");
      }
      L->ndim.push_back(ndim[i]);
      L->dims.push_back(d0);
      L->dims.push_back(d1);
      L->offsets.push_back(off);
      off = round_up(off + d0 * d1, 64);
    }
    L->slab = std::max<int64_t>(off, 64);
    *out = L;
  });
}

dlx_status dlx_layout_destroy(dlx_layout* layout) {
  return guard([&] { delete layout; });
}

int64_t dlx_layout_slab_elems(const dlx_layout* L) { return L ? L->slab : -1; }

dlx_status dlx_layout_offsets(const dlx_layout* L, int64_t* offsets) {
  return guard([&] { std::memcpy(offsets, L->offsets.data(), sizeof(int64_t) * L->nt); });
}

int64_t dlx_factor_offsets(const dlx_layout* L, int rank, int side, int64_t* offsets) {
  int64_t total = -1;
  const dlx_status st = guard([&] {
    validate_quant(rank, 2);
    Plan& P = const_cast<dlx_layout*>(L)->plan(rank, 8);
    size_t k = 0;
    for (int i = 0; i < L->nt; ++i) {
      if (offsets) offsets[i] = L->ndim[i] == 2 ? (side == 0 ? P.t2[k].poff : P.t2[k].qoff) : -1;
      if (L->ndim[i] == 2) ++k;
    }
    total = side == 0 ? P.pelems : P.qelems;
  });
  return st == DLX_OK ? total : -static_cast<int64_t>(st);
}

int64_t dlx_payload_bytes(const dlx_layout* L, int rank, int qbits) {
  int64_t n = -1;
  const dlx_status st = guard([&] {
    validate_quant(rank, qbits);
    n = const_cast<dlx_layout*>(L)->plan(rank, qbits).payload_bytes;
  });
  return st == DLX_OK ? n : -static_cast<int64_t>(st);
}

dlx_status dlx_payload_segments(const dlx_layout* L, int rank, int qbits, int64_t* seg) {
  return guard([&] {
    validate_quant(rank, qbits);
    Plan& P = const_cast<dlx_layout*>(L)->plan(rank, qbits);
    size_t k2 = 0, k1 = 0;
    for (int i = 0; i < L->nt; ++i) {
      if (L->ndim[i] == 2) {
        const DevT2& t = P.t2[k2++];
        seg[4 * i] = t.seg_pc;
        seg[4 * i + 1] = t.seg_qc;
        seg[4 * i + 2] = t.seg_ps;
        seg[4 * i + 3] = t.seg_qs;
      } else {
        const DevT1& t = P.t1[k1++];
        seg[4 * i] = t.seg_c;
        seg[4 * i + 1] = -1;
        seg[4 * i + 2] = t.seg_s;
        seg[4 * i + 3] = -1;
      }
    }
  });
}

uint64_t dlx_payload_bits(const dlx_layout* L, int rank, int qbits) {
  uint64_t b = 0;
  guard([&] {
    validate_quant(rank, qbits);
    b = const_cast<dlx_layout*>(L)->plan(rank, qbits).payload_bits;
  });
  return b;
}

dlx_status dlx_fill_gaussian(dlx_ctx* ctx, const dlx_layout* L, float* d_out,
                             const float* d_base, float scale, uint64_t seed, uint64_t tag,
                             uint64_t worker, void* stream) {
  return guard([&] {
    set_device(ctx);
    launch_fill_gaussian(*L, d_out, d_base, scale, seed, tag, worker, as_stream(stream));
  });
}

// ---- device-side verification of the speculative cold-start draw bases
// A cold start (no usable warm Q, compress.cpp:161-164) draws each 2-D tensor's b*r initial
// values right before its quantisation draws, so its offset depends on how many draws every
// earlier chunk consumed — and all-zero chunks consume none (compress.cpp:28-30), which is
// only known after the power iteration. The first pass speculates "no all-zero chunk"; the
// quantiser's scan records the actual bases and a mismatch flag. A CUDA graph with a WHILE
// node re-runs the compress body from the actual bases until they agree, entirely on the
// device: no host synchronisation, so the round stays asynchronous across a rank change.
// Non-convergence (more redo passes than 2-D tensors) sets *draws = UINT64_MAX.
__global__ void k_cold_cond_init(cudaGraphConditionalHandle h, const int* mismatch, int* attempts) {
  *attempts = 0;
  cudaGraphSetConditional(h, *mismatch ? 1u : 0u);
}
__global__ void k_cold_cond(cudaGraphConditionalHandle h, const int* mismatch, int* attempts,
                            int max_attempts, uint64_t* draws) {
  unsigned again = *mismatch ? 1u : 0u;
  if (again && ++*attempts > max_attempts) {
    *draws = ~0ull;
    again = 0u;
  }
  cudaGraphSetConditional(h, again);
}
__global__ void k_set_u64(uint64_t* p, uint64_t v) { *p = v; }

namespace {
struct CompressBufs {
  const float* delta;
  float *pbuf, *ptmp, *qbuf, *qtmp, *part;
  uint8_t* payload;
  uint64_t* draws;
  int* mismatch;
  int64_t *base_actual, *base_try;
  uint64_t* s0dev;
  int* attempts;
};

// the compress body from the cold init on: cold-start Q0 at `bases`, power iteration,
// quantise (writes mismatch / base_actual when cold)
void compress_body(dlx_ctx* ctx, const Plan& P, const CompressBufs& B, int rounding, int iters,
                   uint64_t s0, const uint64_t* s0p, bool cold, const int64_t* bases,
                   cudaStream_t s) {
  if (cold && !P.t2.empty()) {
    launch_cold_init(P, B.qbuf, bases, s0, s, s0p);
    orthonormalize_batched(ctx, P, 1, B.qbuf, B.qtmp, s);
  }
  for (int it = 0; it < iters; ++it) {
    launch_k1(P, B.delta, B.qbuf, B.pbuf, s);
    orthonormalize_batched(ctx, P, 0, B.pbuf, B.ptmp, s);
    launch_k2(P, B.delta, B.pbuf, B.qbuf, B.part, s);
    orthonormalize_batched(ctx, P, 1, B.qbuf, B.qtmp, s);
  }
  launch_k1(P, B.delta, B.qbuf, B.pbuf, s);
  DLX_CUDA(cudaMemsetAsync(B.mismatch, 0, sizeof(int), s));
  quantize_all(ctx, P, B.pbuf, B.qbuf, B.delta, rounding, s0, cold ? 1 : 0, bases, B.payload,
               B.draws, B.mismatch, B.base_actual, s, s0p);
}

struct ColdRedo : PlanExt {
  struct Entry {
    std::vector<const void*> key;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
  };
  std::vector<Entry> entries;
  ~ColdRedo() override {
    for (Entry& e : entries) {
      if (e.exec) cudaGraphExecDestroy(e.exec);
      if (e.graph) cudaGraphDestroy(e.graph);
    }
  }
};

cudaGraphExec_t cold_redo_graph(dlx_ctx* ctx, const Plan& P, const CompressBufs& B, int iters) {
  ColdRedo& R = plan_ext<ColdRedo>(P, "cold_redo");
  const std::vector<const void*> key = {B.delta, B.pbuf, B.ptmp, B.qbuf, B.qtmp, B.part,
                                        B.payload, B.draws, B.mismatch, B.base_actual,
                                        B.base_try, B.s0dev, B.attempts,
                                        reinterpret_cast<const void*>(static_cast<intptr_t>(iters))};
  for (auto& e : R.entries)
    if (e.key == key) return e.exec;
  HostProf hp("cold_redo_graph (new)");
  if (R.entries.size() >= 4) {  // bounded: evict the oldest (wait for in-flight replays)
    DLX_CUDA(cudaDeviceSynchronize());
    cudaGraphExecDestroy(R.entries.front().exec);
    cudaGraphDestroy(R.entries.front().graph);
    R.entries.erase(R.entries.begin());
  }
  if (!ctx->capture) DLX_CUDA(cudaStreamCreateWithFlags(&ctx->capture, cudaStreamNonBlocking));
  cudaStream_t cs = ctx->capture;
  ColdRedo::Entry e;
  e.key = key;
  DLX_CUDA(cudaGraphCreate(&e.graph, 0));
  cudaGraphConditionalHandle h;
  DLX_CUDA(cudaGraphConditionalHandleCreate(&h, e.graph, 0, cudaGraphCondAssignDefault));
  const uint64_t saved = dlx_take_launch_count();  // captured launches are not launches
  // head: condition = first pass's mismatch
  DLX_CUDA(cudaStreamBeginCaptureToGraph(cs, e.graph, nullptr, nullptr, 0,
                                         cudaStreamCaptureModeRelaxed));
  k_cold_cond_init<<<1, 1, 0, cs>>>(h, B.mismatch, B.attempts);
  DLX_CUDA(cudaGetLastError());
  cudaGraph_t g2 = nullptr;
  DLX_CUDA(cudaStreamEndCapture(cs, &g2));
  size_t n = 0;
  DLX_CUDA(cudaGraphGetNodes(e.graph, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  DLX_CUDA(cudaGraphGetNodes(e.graph, nodes.data(), &n));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t wnode;
  DLX_CUDA(cudaGraphAddNode(&wnode, e.graph, nodes.data(), n, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  // body: redo from the observed bases, then re-evaluate
  DLX_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                         cudaStreamCaptureModeRelaxed));
  DLX_CUDA(cudaMemcpyAsync(B.base_try, B.base_actual, sizeof(int64_t) * P.t2.size(),
                           cudaMemcpyDeviceToDevice, cs));
  compress_body(ctx, P, B, 0, iters, 0, B.s0dev, true, B.base_try, cs);
  k_cold_cond<<<1, 1, 0, cs>>>(h, B.mismatch, B.attempts, static_cast<int>(P.t2.size()) + 2,
                               B.draws);
  DLX_CUDA(cudaGetLastError());
  cudaGraph_t b2 = nullptr;
  DLX_CUDA(cudaStreamEndCapture(cs, &b2));
  DLX_CUDA(cudaGraphInstantiate(&e.exec, e.graph, 0));
  dlx_take_launch_count();
  count_launch(static_cast<int>(saved));
  R.entries.push_back(e);
  return R.entries.back().exec;
}
}  // namespace

static void run_compress(dlx_ctx* ctx, dlx_layout* L, const float* d_delta, int rank, int qbits,
                         int rounding, int iters, uint64_t s0, const float* d_warm_q,
                         int warm_rank, uint8_t* d_payload, float* d_q_out, uint64_t* d_draws,
                         cudaStream_t s) {
  HostProf hp("compress");
  NvtxRange nv("dlx_compress");
  validate_quant(rank, qbits);
  if (iters < 1) raise(DLX_ERR_VALIDATION, "lowrank_approx: iters must be >= 1");
  if (rounding != 0 && rounding != 1) raise(DLX_ERR_VALIDATION, "unknown rounding mode");
  if (!d_delta || !d_payload) raise(DLX_ERR_VALIDATION, "null buffer");
  Plan& P = L->plan(rank, qbits);
  CompressBufs B{};
  B.delta = d_delta;
  B.pbuf = static_cast<float*>(ctx->scratch("pbuf", sizeof(float) * P.pelems));
  B.ptmp = static_cast<float*>(ctx->scratch("ptmp", sizeof(float) * P.pelems));
  B.qtmp = static_cast<float*>(ctx->scratch("qtmp", sizeof(float) * P.qelems));
  B.qbuf = d_q_out ? d_q_out : static_cast<float*>(ctx->scratch("qbuf", sizeof(float) * P.qelems));
  B.part = static_cast<float*>(ctx->scratch("k2part", sizeof(float) * P.k2_part_elems));
  B.payload = d_payload;
  // the draw count lands in a context buffer (a stable address for the redo graph) and is
  // copied out to the caller's at the end
  B.draws = static_cast<uint64_t*>(ctx->scratch("draws", 8));
  B.mismatch = static_cast<int*>(ctx->scratch("mismatch", sizeof(int)));
  const size_t nb = std::max<size_t>(P.t2.size(), 1);
  B.base_actual = static_cast<int64_t*>(ctx->scratch("cold_actual", 8 * nb));
  B.base_try = static_cast<int64_t*>(ctx->scratch("cold_try", 8 * nb));
  B.s0dev = static_cast<uint64_t*>(ctx->scratch("cold_s0", 8));
  B.attempts = static_cast<int*>(ctx->scratch("cold_attempts", sizeof(int)));
  const bool cold = !(d_warm_q && warm_rank == rank);
  if (!cold && d_warm_q != B.qbuf)
    DLX_CUDA(cudaMemcpyAsync(B.qbuf, d_warm_q, sizeof(float) * P.qelems, cudaMemcpyDeviceToDevice, s));
  compress_body(ctx, P, B, rounding, iters, s0, nullptr, cold,
                P.d_cold_base_spec[rounding == 0 ? 0 : 1], s);
  // Nearest rounding draws nothing while quantising, so its cold bases are exact; the
  // stochastic bases are verified (and the body redone) on the device
  if (cold && rounding == 0 && !P.t2.empty()) {
    cudaGraphExec_t g = cold_redo_graph(ctx, P, B, iters);
    k_set_u64<<<1, 1, 0, s>>>(B.s0dev, s0);
    DLX_LAUNCHED();
    DLX_CUDA(cudaGraphLaunch(g, s));
    count_launch(2);
  }
  if (d_draws) DLX_CUDA(cudaMemcpyAsync(d_draws, B.draws, 8, cudaMemcpyDeviceToDevice, s));
}

dlx_status dlx_compress(dlx_ctx* ctx, const dlx_layout* layout, const float* d_delta, int rank,
                        int qbits, int rounding, int power_iters, uint64_t rng_state,
                        const float* d_warm_q, int warm_rank, uint8_t* d_payload,
                        float* d_q_out, uint64_t* d_draws, void* stream) {
  return guard([&] {
    set_device(ctx);
    run_compress(ctx, const_cast<dlx_layout*>(layout), d_delta, rank, qbits, rounding,
                 power_iters, rng_state, d_warm_q, warm_rank, d_payload, d_q_out, d_draws,
                 as_stream(stream));
  });
}

dlx_status dlx_quantize_factors(dlx_ctx* ctx, const dlx_layout* layout, const float* d_p,
                                const float* d_q, const float* d_delta, int rank, int qbits,
                                int rounding, uint64_t rng_state, int cold,
                                uint8_t* d_payload, uint64_t* d_draws, void* stream) {
  return guard([&] {
    set_device(ctx);
    validate_quant(rank, qbits);
    Plan& P = const_cast<dlx_layout*>(layout)->plan(rank, qbits);
    uint64_t* draws = d_draws ? d_draws : static_cast<uint64_t*>(ctx->scratch("draws", 8));
    int* mismatch = static_cast<int*>(ctx->scratch("mismatch", sizeof(int)));
    int64_t* base_actual = static_cast<int64_t*>(
        ctx->scratch("cold_actual", 8 * std::max<size_t>(P.t2.size(), 1)));
    quantize_all(ctx, P, d_p, d_q, d_delta, rounding, rng_state, cold, nullptr, d_payload,
                 draws, mismatch, base_actual, as_stream(stream));
  });
}

dlx_status dlx_decompress(dlx_ctx* ctx, const dlx_layout* layout, int rank, int qbits,
                          const uint8_t* d_payload, float* d_out, void* stream) {
  return guard([&] {
    set_device(ctx);
    validate_quant(rank, qbits);
    Plan& P = const_cast<dlx_layout*>(layout)->plan(rank, qbits);
    launch_reconstruct_dense(ctx, P, 1, d_payload, d_out, as_stream(stream));
  });
}

dlx_status dlx_allreduce_avg(dlx_ctx* ctx, const dlx_layout* layout, int rank, int qbits,
                             int D, const uint8_t* d_gathered, float* d_out, void* stream) {
  return guard([&] {
    set_device(ctx);
    validate_quant(rank, qbits);
    if (D < 1) raise(DLX_ERR_VALIDATION, "allreduce_avg: no payloads");
    Plan& P = const_cast<dlx_layout*>(layout)->plan(rank, qbits);
    launch_reconstruct_dense(ctx, P, D, d_gathered, d_out, as_stream(stream));
  });
}

dlx_status dlx_outer_update_range(dlx_ctx* ctx, const dlx_layout* layout, int rank, int qbits,
                                  int D, const uint8_t* d_gathered, int self_index, int mode,
                                  float* d_pending, float* d_anchor, const float* d_local,
                                  float* d_velocity, float gamma, float beta, int classical,
                                  dlx_round_stats* d_stats, int t_begin, int t_end,
                                  void* stream) {
  return guard([&] {
    set_device(ctx);
    validate_quant(rank, qbits);
    if (D < 1) raise(DLX_ERR_VALIDATION, "allreduce_avg: no payloads");
    if (mode != DLX_MODE_OVERLAPPED && mode != DLX_MODE_SYNC)
      raise(DLX_ERR_VALIDATION, "unknown outer-update mode");
    if (self_index >= D) raise(DLX_ERR_VALIDATION, "self_index out of range");
    if (mode == DLX_MODE_OVERLAPPED && !d_local)
      raise(DLX_ERR_VALIDATION, "overlapped mode needs the local parameters");
    Plan& P = const_cast<dlx_layout*>(layout)->plan(rank, qbits);
    cudaStream_t s = as_stream(stream);
    if (t_begin < 0 || t_end > layout->nt || t_begin > t_end)
      raise(DLX_ERR_VALIDATION, "outer_update: tensor range out of bounds");
    const SlotRange R = slot_range(P, t_begin, t_end);
    NvtxRange nv("dlx_outer_update");
    if (d_stats && t_begin == 0) DLX_CUDA(cudaMemsetAsync(d_stats, 0, sizeof(dlx_round_stats), s));
    launch_outer_2d(ctx, P, D, d_gathered, self_index, mode, d_pending, d_anchor, d_local,
                    d_velocity, gamma, beta, classical, d_stats, R, s);
    launch_outer_1d(P, D, d_gathered, self_index, mode, d_pending, d_anchor, d_local,
                    d_velocity, gamma, beta, classical, d_stats, R, s);
  });
}

dlx_status dlx_adamw_step(dlx_ctx* ctx, int64_t n, float lr, float beta1, float beta2, float eps,
                          float weight_decay, int64_t warmup_steps, int64_t* step, float* d_p,
                          const float* d_g, float* d_m, float* d_v, int* d_nonfinite,
                          void* stream) {
  return guard([&] {
    set_device(ctx);
    if (n < 0 || !step) raise(DLX_ERR_VALIDATION, "adamw_step: bad arguments");
    *step += 1;  // optim.cpp:20
    if (n == 0) return;
    launch_adamw(n, lr, beta1, beta2, eps, weight_decay, warmup_steps, *step, d_p, d_g, d_m, d_v,
                 d_nonfinite, as_stream(stream));
  });
}

dlx_status dlx_outer_update_raw(dlx_ctx* ctx, const dlx_layout* layout, int D,
                                const float* d_gathered, int self_index, int mode,
                                float* d_pending, float* d_anchor, const float* d_local,
                                float* d_velocity, float gamma, float beta, int classical,
                                dlx_round_stats* d_stats, void* stream) {
  return guard([&] {
    set_device(ctx);
    if (D < 1) raise(DLX_ERR_VALIDATION, "allreduce_avg: no payloads");
    if (mode != DLX_MODE_OVERLAPPED && mode != DLX_MODE_SYNC)
      raise(DLX_ERR_VALIDATION, "unknown outer-update mode");
    if (self_index >= D) raise(DLX_ERR_VALIDATION, "self_index out of range");
    if (mode == DLX_MODE_OVERLAPPED && !d_local)
      raise(DLX_ERR_VALIDATION, "overlapped mode needs the local parameters");
    cudaStream_t s = as_stream(stream);
    if (d_stats) DLX_CUDA(cudaMemsetAsync(d_stats, 0, sizeof(dlx_round_stats), s));
    launch_outer_raw(*layout, D, d_gathered, self_index, mode, d_pending, d_anchor, d_local,
                     d_velocity, gamma, beta, classical, d_stats, s);
  });
}

dlx_status dlx_outer_update(dlx_ctx* ctx, const dlx_layout* layout, int rank, int qbits, int D,
                            const uint8_t* d_gathered, int self_index, int mode,
                            float* d_pending, float* d_anchor, const float* d_local,
                            float* d_velocity, float gamma, float beta, int classical,
                            dlx_round_stats* d_stats, void* stream) {
  return dlx_outer_update_range(ctx, layout, rank, qbits, D, d_gathered, self_index, mode,
                                d_pending, d_anchor, d_local, d_velocity, gamma, beta, classical,
                                d_stats, 0, layout ? layout->nt : 0, stream);
}

dlx_status dlx_stage_deltas(dlx_ctx* ctx, const dlx_layout* layout, const float* d_anchor,
                            const float* d_local, const float* d_err, float* d_pending,
                            double* d_norm_sq, void* stream) {
  return guard([&] {
    set_device(ctx);
    cudaStream_t s = as_stream(stream);
    if (d_norm_sq) DLX_CUDA(cudaMemsetAsync(d_norm_sq, 0, sizeof(double), s));
    launch_stage(*layout, d_anchor, d_local, d_err, d_pending, d_norm_sq, s);
  });
}

dlx_status dlx_measure_error(dlx_ctx* ctx, const dlx_layout* layout, int rank, int qbits,
                             const uint8_t* d_payload, const float* d_delta, double* d_out,
                             void* stream) {
  return guard([&] {
    set_device(ctx);
    validate_quant(rank, qbits);
    if (!d_payload || !d_delta || !d_out) raise(DLX_ERR_VALIDATION, "null buffer");
    Plan& P = const_cast<dlx_layout*>(layout)->plan(rank, qbits);
    cudaStream_t s = as_stream(stream);
    float* rec = static_cast<float*>(ctx->scratch("measure_rec", sizeof(float) * layout->slab));
    launch_reconstruct_dense(ctx, P, 1, d_payload, rec, s);
    DLX_CUDA(cudaMemsetAsync(d_out, 0, 2 * sizeof(double), s));
    launch_sqdiff(*layout, rec, d_delta, d_out, s);
  });
}

dlx_status dlx_sqdiff_slabs(dlx_ctx* ctx, const dlx_layout* layout, const float* d_rec,
                            const float* d_delta, double* d_out, void* stream) {
  return guard([&] {
    set_device(ctx);
    if (!d_rec || !d_delta || !d_out) raise(DLX_ERR_VALIDATION, "null buffer");
    cudaStream_t s = as_stream(stream);
    DLX_CUDA(cudaMemsetAsync(d_out, 0, 2 * sizeof(double), s));
    launch_sqdiff(*layout, d_rec, d_delta, d_out, s);
  });
}

dlx_status dlx_mean_slabs(dlx_ctx* ctx, int64_t n, int64_t ld, int D, const float* d_in,
                          float* d_out, void* stream) {
  return guard([&] {
    set_device(ctx);
    if (D < 1) raise(DLX_ERR_VALIDATION, "allreduce_avg: no payloads");
    if (n < 0 || ld < n) raise(DLX_ERR_VALIDATION, "mean_slabs: bad sizes");
    launch_mean_slabs(n, ld, d_in, D, d_out, as_stream(stream));
  });
}

dlx_status dlx_nesterov(dlx_ctx* ctx, int64_t n, float gamma, float beta, int classical,
                        float* d_anchor, float* d_velocity, const float* d_delta, void* stream) {
  return guard([&] {
    set_device(ctx);
    launch_nesterov(n, gamma, beta, classical, d_anchor, d_velocity, d_delta, as_stream(stream));
  });
}

dlx_status dlx_effective_rank_shard(dlx_ctx* ctx, const dlx_layout* layout, int rank,
                                    int qbits, int D, const uint8_t* d_gathered, double tau,
                                    int shard, int nshards, int* d_per_tensor, double* d_energy,
                                    void* stream) {
  return guard([&] {
    set_device(ctx);
    validate_quant(rank, qbits);
    if (!(tau > 0.0) || !(tau < 1.0)) raise(DLX_ERR_VALIDATION, "effective_rank: need 0 < tau < 1");
    if (D < 1) raise(DLX_ERR_VALIDATION, "effective_rank: no payloads");
    Plan& P = const_cast<dlx_layout*>(layout)->plan(rank, qbits);
    NvtxRange nv("dlx_effective_rank");
    effective_rank_factors(ctx, P, D, d_gathered, tau, d_per_tensor, d_energy, shard, nshards,
                           as_stream(stream));
  });
}

dlx_status dlx_effective_rank(dlx_ctx* ctx, const dlx_layout* layout, int rank, int qbits,
                              int D, const uint8_t* d_gathered, double tau, int* d_per_tensor,
                              double* d_energy, void* stream) {
  return dlx_effective_rank_shard(ctx, layout, rank, qbits, D, d_gathered, tau, 0, 1,
                                  d_per_tensor, d_energy, stream);
}

dlx_status dlx_effective_rank_reduce(const dlx_layout* layout, const int* per_tensor,
                                     const double* energy, int r_max, int* aggregate,
                                     int* all_zero) {
  return guard([&] {
    // compress.cpp:333-343
    if (r_max < 1) raise(DLX_ERR_VALIDATION, "effective_rank: need r_max >= 1");
    double weighted = 0.0, total = 0.0;
    int64_t weight = 0;
    int k = 0;
    for (int i = 0; i < layout->nt; ++i) {
      if (layout->ndim[i] != 2) continue;
      const int64_t sz = layout->numel(i);
      weighted += static_cast<double>(sz) * static_cast<double>(per_tensor[k]);
      weight += sz;
      total += energy[k];
      ++k;
    }
    *all_zero = 0;
    if (weight == 0 || total == 0.0) {
      *aggregate = 1;
      *all_zero = total == 0.0 ? 1 : 0;
      return;
    }
    const int agg = static_cast<int>(std::ceil(weighted / static_cast<double>(weight)));
    *aggregate = std::min(std::max(agg, 1), r_max);
  });
}

dlx_status dlx_adapt_compression(const int* window, int len, int r1, int H1, int c, int h_min,
                                 int* r_out, int* h_out) {
  return guard([&] {
    // engine.cpp:294-308
    if (r1 < 1 || H1 < 1 || c < 1) raise(DLX_ERR_VALIDATION, "adapt_compression: bad parameters");
    if (h_min < 1) raise(DLX_ERR_VALIDATION, "adapt_compression: H_min must be >= 1");
    if (len < c) {
      *r_out = r1;
      *h_out = H1;
      return;
    }
    double sum = 0.0;
    for (int i = len - c; i < len; ++i) sum += static_cast<double>(window[i]);
    int r = static_cast<int>(std::ceil(sum / static_cast<double>(c)));
    r = std::min(std::max(r, 1), r1);
    const double alpha = static_cast<double>(r1 - r) / static_cast<double>(r1);
    int h = static_cast<int>(std::llround(static_cast<double>(H1) * alpha));
    h = std::min(std::max(h, h_min), H1);
    *r_out = r;
    *h_out = h;
  });
}

double dlx_omega_bound(int r, int d, int q) {
  // compress.cpp:240-244
  if (r < 1 || r > d || q < 0) {
    g_last_error = "omega_bound: need 1 <= r <= d and q >= 0";
    return -1.0;
  }
  return 1.0 - (static_cast<double>(r) / static_cast<double>(d)) * std::pow(2.0, -q);
}

// ------------------------------------------------------------------------- wire format
static void put_le(std::vector<uint8_t>& o, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) o.push_back(static_cast<uint8_t>(v >> (8 * i)));
}

int64_t dlx_serialize(const dlx_layout* L, int rank, int qbits, const char* const* names,
                      const uint8_t* pay, uint8_t* out, int64_t cap) {
  int64_t size = -1;
  const dlx_status st = guard([&] {
    validate_quant(rank, qbits);
    Plan& P = const_cast<dlx_layout*>(L)->plan(rank, qbits);
    std::vector<uint8_t> o;
    put_le(o, 0x43584c44u, 4);  // "DLXC" (compress.cpp:397)
    put_le(o, 1u, 4);
    put_le(o, static_cast<uint32_t>(rank), 4);
    put_le(o, static_cast<uint32_t>(qbits), 4);
    put_le(o, static_cast<uint32_t>(L->nt), 4);
    size_t k2 = 0, k1 = 0;
    for (int i = 0; i < L->nt; ++i) {
      const std::string nm = names ? names[i] : ("t" + std::to_string(i));
      if (nm.size() > 0xffff) raise(DLX_ERR_FORMAT, "string too long for wire format");
      put_le(o, nm.size(), 2);
      o.insert(o.end(), nm.begin(), nm.end());
      const bool two = L->ndim[i] == 2;
      o.push_back(two ? 0 : 1);
      o.push_back(static_cast<uint8_t>(L->ndim[i]));
      for (int d = 0; d < L->ndim[i]; ++d) put_le(o, static_cast<uint64_t>(L->dims[2 * i + d]), 8);
      if (two) {
        const DevT2& t = P.t2[k2++];
        put_le(o, static_cast<uint32_t>(t.r), 4);
        put_le(o, static_cast<uint32_t>(qbits), 4);
        const int64_t pc = ceil_div(t.a * t.r * qbits, 8), qc = ceil_div(t.b * t.r * qbits, 8);
        o.insert(o.end(), pay + t.seg_pc, pay + t.seg_pc + pc);
        o.insert(o.end(), pay + t.seg_qc, pay + t.seg_qc + qc);
        o.insert(o.end(), pay + t.seg_ps, pay + t.seg_ps + 4 * t.r);
        o.insert(o.end(), pay + t.seg_qs, pay + t.seg_qs + 4 * t.r);
      } else {
        const DevT1& t = P.t1[k1++];
        put_le(o, 0u, 4);
        put_le(o, static_cast<uint32_t>(qbits), 4);
        o.insert(o.end(), pay + t.seg_c, pay + t.seg_c + ceil_div(t.n * qbits, 8));
        o.insert(o.end(), pay + t.seg_s, pay + t.seg_s + 4);
      }
    }
    size = static_cast<int64_t>(o.size());
    if (out && cap >= size) std::memcpy(out, o.data(), o.size());
  });
  return st == DLX_OK ? size : -static_cast<int64_t>(st);
}

dlx_status dlx_parse(const dlx_layout* L, int rank, int qbits, const uint8_t* bytes,
                     int64_t size, uint8_t* pay) {
  return guard([&] {
    // parse_compressed (compress.cpp:428-482), checked against this layout
    validate_quant(rank, qbits);
    Plan& P = const_cast<dlx_layout*>(L)->plan(rank, qbits);
    int64_t pos = 0;
    auto need = [&](int64_t n) -> const uint8_t* {
      if (pos + n > size) raise(DLX_ERR_FORMAT, "truncated payload");
      const uint8_t* p = bytes + pos;
      pos += n;
      return p;
    };
    auto rd = [&](int n) {
      const uint8_t* p = need(n);
      uint64_t v = 0;
      for (int i = 0; i < n; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
      return v;
    };
    if (rd(4) != 0x43584c44u) raise(DLX_ERR_FORMAT, "bad compressed payload magic");
    if (rd(4) != 1u) raise(DLX_ERR_FORMAT, "unsupported compressed payload version");
    rd(4);
    if (static_cast<int>(rd(4)) != qbits) raise(DLX_ERR_FORMAT, "payload qbits disagree");
    if (static_cast<int>(rd(4)) != L->nt) raise(DLX_ERR_FORMAT, "payload tensor count disagrees");
    std::memset(pay, 0, static_cast<size_t>(P.payload_bytes));
    size_t k2 = 0, k1 = 0;
    for (int i = 0; i < L->nt; ++i) {
      need(static_cast<int64_t>(rd(2)));
      const int kind = static_cast<int>(rd(1));
      const int nd = static_cast<int>(rd(1));
      if (nd != L->ndim[i]) raise(DLX_ERR_FORMAT, "payload ndim disagrees");
      for (int d = 0; d < nd; ++d)
        if (static_cast<int64_t>(rd(8)) != L->dims[2 * i + d]) raise(DLX_ERR_FORMAT, "payload shape disagrees");
      const int r = static_cast<int>(rd(4));
      if (static_cast<int>(rd(4)) != qbits) raise(DLX_ERR_FORMAT, "bad qbits in payload");
      if (nd == 2) {
        const DevT2& t = P.t2[k2++];
        if (kind != 0 || r != t.r) raise(DLX_ERR_FORMAT, "bad rank in payload");
        const int64_t pc = ceil_div(t.a * t.r * qbits, 8), qc = ceil_div(t.b * t.r * qbits, 8);
        std::memcpy(pay + t.seg_pc, need(pc), pc);
        std::memcpy(pay + t.seg_qc, need(qc), qc);
        std::memcpy(pay + t.seg_ps, need(4 * t.r), 4 * t.r);
        std::memcpy(pay + t.seg_qs, need(4 * t.r), 4 * t.r);
      } else {
        const DevT1& t = P.t1[k1++];
        if (kind != 1) raise(DLX_ERR_FORMAT, "unknown payload kind");
        const int64_t nc = ceil_div(t.n * qbits, 8);
        std::memcpy(pay + t.seg_c, need(nc), nc);
        std::memcpy(pay + t.seg_s, need(4), 4);
      }
    }
    if (pos != size) raise(DLX_ERR_FORMAT, "trailing bytes in compressed payload");
  });
}

}  // extern "C"
