// dilocox_b200.cpp — the reference's hot-path C++ API, same signatures, backed by the B200
// C-ABI (include/dlx_b200.h, paper_2506_21263_b200/libdlx_b200.so).
//
// Drop-in at link time: cpp/Makefile compiles the reference's own proj/core sources (where
// they lie under /root/reference, unmodified), WEAKENS in their objects exactly the symbols
// this translation unit defines, and links this TU in. The reference engine —
// run_round_overlapped / run_round_sync / run_experiment (engine.cpp:423-509, 595-610),
// collective_average (engine.cpp:215-263) — then runs unchanged with its hot path on the GPU:
//
//   compress            compress.hpp:94-95   -> dlx_compress (power iteration + quantise)
//   decompress          compress.hpp:100     -> dlx_parse + dlx_decompress
//   measure_error       compress.hpp:106     -> dlx_measure_error / dlx_sqdiff_slabs
//   effective_rank      compress.hpp:130     -> dlx_effective_rank (factor space)
//   allreduce_avg       collective.hpp:23    -> dlx_allreduce_avg / dlx_mean_slabs
//   nesterov_outer_step optim.hpp:48         -> dlx_nesterov
//
// Host-resident ParamSets cross to the device on every call (this is the value-semantics
// API of the reference); the device-resident production path is the C-ABI itself
// (dlx_compress -> dlx_exchange -> dlx_outer_update), see cpp/worker_main.cpp.
//
// Semantics kept: the RngStream& argument advances by exactly the draws consumed; payloads
// are the reference's CompressedDelta (built by the reference's own parse_compressed from the
// device payload's DLXC bytes); exceptions are the reference's types with the reference's
// messages where the check is the reference's. Differences (documented in INTEGRATION.md):
//   * a WarmStart that covers only some 2-D tensors throws ValidationError (the reference
//     mixes warm and cold tensors; its engine never produces such a WarmStart);
//   * effective_rank works in factor space, so its input must be the result of the last
//     allreduce_avg of compressed payloads (which is how collective_average calls it);
//     anything else throws ValidationError rather than running a CPU SVD.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "dilocox/collective.hpp"
#include "dilocox/compress.hpp"
#include "dilocox/errors.hpp"
#include "dilocox/optim.hpp"
#include "dilocox/params.hpp"
#include "dilocox/rng.hpp"
#include "dlx_b200.h"

static_assert(sizeof(dilocox::RngStream) == sizeof(uint64_t), "RngStream is one splitmix state");

namespace dilocox {
namespace {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;

[[noreturn]] void rethrow(dlx_status s) {
  const std::string m = dlx_last_error();
  switch (s) {
    case DLX_ERR_VALIDATION: throw ValidationError(m);
    case DLX_ERR_SHAPE: throw ShapeError(m);
    case DLX_ERR_FORMAT: throw FormatError(m);
    case DLX_ERR_NUMERIC: throw NumericError(m);
    case DLX_ERR_IO: throw IoError(m);
    default: throw Error(m);
  }
}
void ok(dlx_status s) {
  if (s != DLX_OK) rethrow(s);
}
void cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(std::string("CUDA (") + what + "): " + cudaGetErrorString(e));
}

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  void* get(size_t bytes) {
    if (bytes > n) {
      if (p) cudaFree(p);
      p = nullptr;
      cu(cudaMalloc(&p, std::max<size_t>(bytes, 256)), "cudaMalloc");
      n = std::max<size_t>(bytes, 256);
    }
    return p;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct Layout {
  dlx_layout* h = nullptr;
  std::vector<int64_t> offsets;
  int64_t slab = 0;
  std::vector<std::string> names;
  std::vector<const char*> cnames;
  std::vector<std::vector<int64_t>> shapes;
};

struct Runtime {
  dlx_ctx* ctx = nullptr;
  int device = 0;
  std::map<std::string, std::unique_ptr<Layout>> layouts;
  DevBuf a, b, c, pay, q, gathered, scratch8;
  // factor form of the last allreduce_avg result over compressed payloads
  struct {
    bool valid = false;
    uint64_t fp = 0;
    Layout* L = nullptr;
    int rank = 0, qbits = 0, D = 0;
    DevBuf gathered;
  } last;
};

std::mutex g_mu;  // the reference calls compress from parallel_over threads (engine.cpp:223-234)

Runtime& rt() {
  static Runtime* r = [] {
    auto* x = new Runtime();
    const char* e = std::getenv("DLX_DEVICE");
    x->device = e ? std::atoi(e) : 0;
    ok(dlx_ctx_create(x->device, &x->ctx));
    return x;
  }();
  cu(cudaSetDevice(r->device), "cudaSetDevice");
  return *r;
}

std::string signature(const ParamSet& ps) {
  std::string k;
  for (int i = 0; i < ps.count(); ++i) {
    k += ps.name(i);
    k += ':';
    for (int64_t d : ps.tensor(i).shape()) k += std::to_string(d) + 'x';
    k += ';';
  }
  return k;
}

Layout& layout_of(Runtime& R, const ParamSet& ps) {
  const std::string key = signature(ps);
  auto it = R.layouts.find(key);
  if (it != R.layouts.end()) return *it->second;
  auto L = std::make_unique<Layout>();
  std::vector<int> nd;
  std::vector<int64_t> dims;
  for (int i = 0; i < ps.count(); ++i) {
    const Tensor& t = ps.tensor(i);
    nd.push_back(t.ndim());
    dims.push_back(t.ndim() >= 1 ? t.dim(0) : 0);
    dims.push_back(t.ndim() == 2 ? t.dim(1) : 1);
    L->names.push_back(ps.name(i));
    L->shapes.push_back(t.shape());
  }
  ok(dlx_layout_create(R.ctx, ps.count(), nd.data(), dims.data(), &L->h));
  L->offsets.resize(static_cast<size_t>(ps.count()));
  if (ps.count()) ok(dlx_layout_offsets(L->h, L->offsets.data()));
  L->slab = dlx_layout_slab_elems(L->h);
  for (const std::string& n : L->names) L->cnames.push_back(n.c_str());
  Layout& ref = *L;
  R.layouts.emplace(key, std::move(L));
  return ref;
}

// ParamSet <-> device slab (tensor i at offsets[i]; the alignment padding is zeroed)
float* upload(const Layout& L, const ParamSet& ps, DevBuf& buf) {
  auto* d = static_cast<float*>(buf.get(sizeof(float) * L.slab));
  cu(cudaMemset(d, 0, sizeof(float) * L.slab), "cudaMemset");
  for (int i = 0; i < ps.count(); ++i) {
    const Tensor& t = ps.tensor(i);
    cu(cudaMemcpy(d + L.offsets[i], t.data(), sizeof(float) * t.size(), cudaMemcpyHostToDevice),
       "H2D");
  }
  return d;
}
ParamSet download(const Layout& L, const float* d) {
  ParamSet out;
  for (size_t i = 0; i < L.names.size(); ++i) {
    Tensor t(L.shapes[i]);
    cu(cudaMemcpy(t.data(), d + L.offsets[i], sizeof(float) * t.size(), cudaMemcpyDeviceToHost),
       "D2H");
    out.add(L.names[i], std::move(t));
  }
  return out;
}

uint64_t fingerprint(const ParamSet& ps) {  // FNV-1a over names, shapes and value bits
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* p, size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  };
  for (int i = 0; i < ps.count(); ++i) {
    mix(ps.name(i).data(), ps.name(i).size());
    for (int64_t d : ps.tensor(i).shape()) mix(&d, sizeof(d));
    mix(ps.tensor(i).data(), sizeof(float) * ps.tensor(i).size());
  }
  return h;
}

bool all_raw(const CompressedDelta& cd) {
  for (const TensorPayload& t : cd.tensors)
    if (t.kind != PayloadKind::RawDense) return false;
  return !cd.tensors.empty();
}
bool any_raw(const CompressedDelta& cd) {
  for (const TensorPayload& t : cd.tensors)
    if (t.kind == PayloadKind::RawDense) return true;
  return false;
}

// CompressedDelta -> the empty ParamSet of its layout (names + shapes), for layout_of
ParamSet skeleton(const CompressedDelta& cd) {
  ParamSet ps;
  for (const TensorPayload& t : cd.tensors) ps.add(t.name, Tensor(t.shape));
  return ps;
}

// CompressedDelta (quantised kinds) -> device payload bytes via its DLXC wire form
void to_device_payload(Runtime& R, const Layout& L, const CompressedDelta& cd, uint8_t* d_pay) {
  const std::vector<uint8_t> wire = serialize(cd);
  const int64_t pb = dlx_payload_bytes(L.h, cd.rank, cd.qbits);
  if (pb < 0) rethrow(static_cast<dlx_status>(-pb));
  std::vector<uint8_t> host(static_cast<size_t>(pb));
  ok(dlx_parse(L.h, cd.rank, cd.qbits, wire.data(), static_cast<int64_t>(wire.size()), host.data()));
  cu(cudaMemcpy(d_pay, host.data(), host.size(), cudaMemcpyHostToDevice), "H2D payload");
  (void)R;
}

}  // namespace

// ------------------------------------------------------------------ compress.hpp:94-95
CompressResult compress(const ParamSet& delta, int rank, const QuantSpec& spec,
                        const WarmStart* warm, int power_iters, RngStream& rng) {
  spec.validate();
  if (rank < 1) throw ValidationError("compress: rank must be >= 1");
  bool has2d = false;
  for (int i = 0; i < delta.count(); ++i) {
    if (delta.tensor(i).ndim() != 1 && delta.tensor(i).ndim() != 2)
      throw ShapeError("compress: only 1-D and 2-D tensors are supported");
    has2d |= delta.tensor(i).ndim() == 2;
  }
  if (has2d && power_iters < 1) throw ValidationError("lowrank_approx: iters must be >= 1");
  std::lock_guard<std::mutex> lock(g_mu);
  Runtime& R = rt();
  Layout& L = layout_of(R, delta);
  const int q = spec.qbits;
  float* d_delta = upload(L, delta, R.a);
  const int64_t pb = dlx_payload_bytes(L.h, rank, q);
  if (pb < 0) rethrow(static_cast<dlx_status>(-pb));
  std::vector<int64_t> qoff(L.names.size());
  const int64_t qel = dlx_factor_offsets(L.h, rank, 1, qoff.data());
  if (qel < 0) rethrow(static_cast<dlx_status>(-qel));
  auto* d_pay = static_cast<uint8_t*>(R.pay.get(static_cast<size_t>(pb)));
  auto* d_q = static_cast<float*>(R.q.get(sizeof(float) * qel));
  auto* d_draws = static_cast<uint64_t*>(R.scratch8.get(8));
  // warm start: the reference uses warm->q_factors[name] when warm->rank == rank and the
  // factor is b x r_eff (compress.cpp:160-164, 64-66); the device path is all-or-nothing
  int n2 = 0, nwarm = 0;
  for (int i = 0; i < delta.count(); ++i) {
    const Tensor& t = delta.tensor(i);
    if (t.ndim() != 2) continue;
    ++n2;
    if (warm && warm->rank == rank) {
      auto it = warm->q_factors.find(delta.name(i));
      const int64_t r_eff = std::min<int64_t>(rank, std::min(t.rows(), t.cols()));
      if (it != warm->q_factors.end() && it->second.ndim() == 2 &&
          it->second.rows() == t.cols() && it->second.cols() == r_eff)
        ++nwarm;
    }
  }
  const bool use_warm = n2 > 0 && nwarm == n2;
  if (nwarm > 0 && nwarm < n2)
    throw ValidationError("compress (B200): a warm start covering only some tensors is not supported");
  if (use_warm) {  // column-major, column stride round_up(b, 32) (dlx_factor_offsets)
    std::vector<float> host(static_cast<size_t>(qel), 0.0f);
    for (int i = 0; i < delta.count(); ++i) {
      const Tensor& t = delta.tensor(i);
      if (t.ndim() != 2) continue;
      const Tensor& wq = warm->q_factors.at(delta.name(i));
      const int64_t b = wq.rows(), r = wq.cols(), ld = (b + 31) / 32 * 32;
      for (int64_t j = 0; j < r; ++j)
        for (int64_t k = 0; k < b; ++k) host[qoff[i] + j * ld + k] = wq.at(k, j);
    }
    cu(cudaMemcpy(d_q, host.data(), sizeof(float) * qel, cudaMemcpyHostToDevice), "H2D warm");
  }
  uint64_t s0;
  std::memcpy(&s0, static_cast<const void*>(&rng), sizeof(s0));
  ok(dlx_compress(R.ctx, L.h, d_delta, rank, q,
                  spec.rounding == Rounding::Stochastic ? DLX_ROUND_STOCHASTIC : DLX_ROUND_NEAREST,
                  std::max(power_iters, 1), s0, use_warm ? d_q : nullptr, use_warm ? rank : 0,
                  d_pay, d_q, d_draws, nullptr));
  uint64_t draws = 0;
  cu(cudaMemcpy(&draws, d_draws, 8, cudaMemcpyDeviceToHost), "D2H draws");
  const uint64_t s1 = s0 + draws * kGolden;  // the caller's stream advances by the draws used
  std::memcpy(static_cast<void*>(&rng), &s1, sizeof(s1));
  std::vector<uint8_t> host(static_cast<size_t>(pb));
  cu(cudaMemcpy(host.data(), d_pay, host.size(), cudaMemcpyDeviceToHost), "D2H payload");
  const int64_t wn = dlx_serialize(L.h, rank, q, L.cnames.data(), host.data(), nullptr, 0);
  if (wn < 0) rethrow(static_cast<dlx_status>(-wn));
  std::vector<uint8_t> wire(static_cast<size_t>(wn));
  dlx_serialize(L.h, rank, q, L.cnames.data(), host.data(), wire.data(), wn);
  CompressResult out;
  out.delta = parse_compressed(wire);  // the reference's own parser
  out.delta.rank = rank;
  out.delta.qbits = q;
  std::vector<float> qh(static_cast<size_t>(qel));
  cu(cudaMemcpy(qh.data(), d_q, sizeof(float) * qel, cudaMemcpyDeviceToHost), "D2H Q");
  for (int i = 0; i < delta.count(); ++i) {
    const Tensor& t = delta.tensor(i);
    if (t.ndim() != 2) continue;
    const int64_t b = t.cols(), r = std::min<int64_t>(rank, std::min(t.rows(), t.cols()));
    const int64_t ld = (b + 31) / 32 * 32;
    Tensor qt({b, r});
    for (int64_t k = 0; k < b; ++k)
      for (int64_t j = 0; j < r; ++j) qt.at(k, j) = qh[qoff[i] + j * ld + k];
    out.q_factors.emplace(delta.name(i), std::move(qt));
  }
  return out;
}

// ------------------------------------------------------------------ compress.hpp:100
ParamSet decompress(const CompressedDelta& cd) {
  if (all_raw(cd)) {  // RawDense is a passthrough copy (compress.cpp:227-233): no arithmetic
    ParamSet out;
    for (const TensorPayload& pay : cd.tensors) {
      Tensor t(pay.shape);
      if (static_cast<int64_t>(pay.raw.size()) != t.size())
        throw FormatError("raw payload count mismatch");
      std::copy(pay.raw.begin(), pay.raw.end(), t.values().begin());
      out.add(pay.name, std::move(t));
    }
    return out;
  }
  if (any_raw(cd)) throw ValidationError("decompress (B200): mixed raw / quantised payload");
  std::lock_guard<std::mutex> lock(g_mu);
  Runtime& R = rt();
  Layout& L = layout_of(R, skeleton(cd));
  const int64_t pb = dlx_payload_bytes(L.h, cd.rank, cd.qbits);
  if (pb < 0) rethrow(static_cast<dlx_status>(-pb));
  auto* d_pay = static_cast<uint8_t*>(R.pay.get(static_cast<size_t>(pb)));
  to_device_payload(R, L, cd, d_pay);
  auto* d_out = static_cast<float*>(R.b.get(sizeof(float) * L.slab));
  ok(dlx_decompress(R.ctx, L.h, cd.rank, cd.qbits, d_pay, d_out, nullptr));
  return download(L, d_out);
}

// ------------------------------------------------------------------ compress.hpp:106
double measure_error(const ParamSet& delta, const CompressedDelta& cd) {
  const ParamSet skel = skeleton(cd);
  if (!skel.same_layout(delta)) throw ShapeError("measure_error: layouts disagree");
  std::lock_guard<std::mutex> lock(g_mu);
  Runtime& R = rt();
  Layout& L = layout_of(R, delta);
  float* d_delta = upload(L, delta, R.a);
  auto* d_out = static_cast<double*>(R.scratch8.get(16));
  if (all_raw(cd)) {
    ParamSet rec;
    for (const TensorPayload& pay : cd.tensors) {
      Tensor t(pay.shape);
      std::copy(pay.raw.begin(), pay.raw.end(), t.values().begin());
      rec.add(pay.name, std::move(t));
    }
    float* d_rec = upload(L, rec, R.b);
    ok(dlx_sqdiff_slabs(R.ctx, L.h, d_rec, d_delta, d_out, nullptr));
  } else {
    if (any_raw(cd)) throw ValidationError("measure_error (B200): mixed raw / quantised payload");
    const int64_t pb = dlx_payload_bytes(L.h, cd.rank, cd.qbits);
    if (pb < 0) rethrow(static_cast<dlx_status>(-pb));
    auto* d_pay = static_cast<uint8_t*>(R.pay.get(static_cast<size_t>(pb)));
    to_device_payload(R, L, cd, d_pay);
    ok(dlx_measure_error(R.ctx, L.h, cd.rank, cd.qbits, d_pay, d_delta, d_out, nullptr));
  }
  double h[2];
  cu(cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost), "D2H error");
  return h[1] == 0.0 ? 0.0 : h[0] / h[1];
}

// ------------------------------------------------------------------ collective.hpp:23
ParamSet allreduce_avg(const std::vector<CompressedDelta>& payloads) {
  if (payloads.empty()) throw ValidationError("allreduce_avg: no payloads");
  for (size_t i = 1; i < payloads.size(); ++i)
    if (!payloads[0].same_metadata(payloads[i]))
      throw ValidationError("allreduce_avg: payload metadata disagrees across workers");
  const int D = static_cast<int>(payloads.size());
  const CompressedDelta& first = payloads[0];
  std::lock_guard<std::mutex> lock(g_mu);
  Runtime& R = rt();
  Layout& L = layout_of(R, skeleton(first));
  auto* d_out = static_cast<float*>(R.b.get(sizeof(float) * L.slab));
  if (all_raw(first)) {  // compress_raw payloads (dilocox-no-compress): exact fp64 mean
    auto* g = static_cast<float*>(R.gathered.get(sizeof(float) * L.slab * D));
    cu(cudaMemset(g, 0, sizeof(float) * L.slab * D), "cudaMemset");
    for (int w = 0; w < D; ++w)
      for (size_t i = 0; i < payloads[w].tensors.size(); ++i) {
        const std::vector<float>& raw = payloads[w].tensors[i].raw;
        cu(cudaMemcpy(g + static_cast<int64_t>(w) * L.slab + L.offsets[i], raw.data(),
                      sizeof(float) * raw.size(), cudaMemcpyHostToDevice), "H2D raw");
      }
    ok(dlx_mean_slabs(R.ctx, L.slab, L.slab, D, g, d_out, nullptr));
    R.last.valid = false;
    return download(L, d_out);
  }
  if (any_raw(first)) throw ValidationError("allreduce_avg (B200): mixed raw / quantised payload");
  const int64_t pb = dlx_payload_bytes(L.h, first.rank, first.qbits);
  if (pb < 0) rethrow(static_cast<dlx_status>(-pb));
  auto* g = static_cast<uint8_t*>(R.last.gathered.get(static_cast<size_t>(pb) * D));
  for (int w = 0; w < D; ++w) to_device_payload(R, L, payloads[w], g + static_cast<int64_t>(w) * pb);
  ok(dlx_allreduce_avg(R.ctx, L.h, first.rank, first.qbits, D, g, d_out, nullptr));
  ParamSet out = download(L, d_out);
  R.last.valid = true;
  R.last.fp = fingerprint(out);
  R.last.L = &L;
  R.last.rank = first.rank;
  R.last.qbits = first.qbits;
  R.last.D = D;
  return out;
}

// ------------------------------------------------------------------ compress.hpp:130
EffectiveRank effective_rank(const ParamSet& delta, double tau, int r_max) {
  if (!(tau > 0.0) || !(tau < 1.0)) throw ValidationError("effective_rank: need 0 < tau < 1");
  if (r_max < 1) throw ValidationError("effective_rank: need r_max >= 1");
  int n2 = 0;
  for (int i = 0; i < delta.count(); ++i) n2 += delta.tensor(i).ndim() == 2;
  EffectiveRank out;
  if (n2 == 0) {  // compress.cpp:333-339: no 2-D tensor -> aggregate 1, flagged all-zero
    out.aggregate = 1;
    out.all_zero = true;
    return out;
  }
  std::lock_guard<std::mutex> lock(g_mu);
  Runtime& R = rt();
  if (!R.last.valid || R.last.fp != fingerprint(delta))
    throw ValidationError(
        "effective_rank (B200): the input must be the last allreduce_avg result of compressed "
        "payloads (the device measures it in factor space)");
  Layout& L = *R.last.L;
  auto* d_per = static_cast<int*>(R.c.get(sizeof(int) * n2 + sizeof(double) * n2 + 64));
  auto* d_en = reinterpret_cast<double*>(reinterpret_cast<char*>(d_per) +
                                         (sizeof(int) * n2 + 15) / 16 * 16);
  ok(dlx_effective_rank(R.ctx, L.h, R.last.rank, R.last.qbits, R.last.D,
                        static_cast<const uint8_t*>(R.last.gathered.p), tau, d_per, d_en,
                        nullptr));
  std::vector<int> per(static_cast<size_t>(n2));
  std::vector<double> en(static_cast<size_t>(n2));
  cu(cudaMemcpy(per.data(), d_per, sizeof(int) * n2, cudaMemcpyDeviceToHost), "D2H rank");
  cu(cudaMemcpy(en.data(), d_en, sizeof(double) * n2, cudaMemcpyDeviceToHost), "D2H energy");
  int agg = 1, allz = 0;
  ok(dlx_effective_rank_reduce(L.h, per.data(), en.data(), r_max, &agg, &allz));
  out.aggregate = agg;
  out.all_zero = allz != 0;
  int k = 0;
  for (int i = 0; i < delta.count(); ++i)
    if (delta.tensor(i).ndim() == 2) out.per_tensor.emplace_back(delta.name(i), per[k++]);
  return out;
}

// ------------------------------------------------------------------ optim.hpp:48
void nesterov_outer_step(NesterovState& state, ParamSet& anchor, const ParamSet& delta) {
  if (!anchor.same_layout(delta) || !anchor.same_layout(state.velocity))
    throw ShapeError("nesterov_outer_step: layouts disagree");
  std::lock_guard<std::mutex> lock(g_mu);
  Runtime& R = rt();
  Layout& L = layout_of(R, anchor);
  float* dA = upload(L, anchor, R.a);
  float* dV = upload(L, state.velocity, R.b);
  float* dD = upload(L, delta, R.c);
  // the padding between tensors is zero in all three slabs and stays zero
  ok(dlx_nesterov(R.ctx, L.slab, state.hyper.lr, state.hyper.momentum,
                  state.hyper.classical ? 1 : 0, dA, dV, dD, nullptr));
  cu(cudaDeviceSynchronize(), "sync");
  ParamSet a = download(L, dA), v = download(L, dV);
  for (int i = 0; i < anchor.count(); ++i) {
    anchor.tensor(i).values() = std::move(a.tensor(i).values());
    state.velocity.tensor(i).values() = std::move(v.tensor(i).values());
  }
}

}  // namespace dilocox
