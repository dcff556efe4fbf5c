// ref_shim.cpp — C shim over the REFERENCE implementation (TEST INFRASTRUCTURE ONLY).
//
// Compiled by oracle/Makefile against the reference's own proj/core sources where they
// lie under /root/reference (nothing copied into this repo); output goes only to
// oracle/_ref/libdlxref.so. It exports the dlx_oracle.h interface so tests can run the
// same checks against the real reference and against the plain-C restatement
// (oracle/dlx_oracle.c), and bench.py can time the reference's CPU path.
#include <cstring>
#include <exception>
#include <functional>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "dilocox/collective.hpp"
#include "dilocox/data.hpp"
#include "dilocox/model.hpp"
#include "dilocox/compress.hpp"
#include "dilocox/engine.hpp"
#include "dilocox/optim.hpp"
#include "dilocox/params.hpp"
#include "dilocox/rng.hpp"
#include "dilocox/tensor.hpp"
#include "dlx_oracle.h"
#include "test_support.hpp"  // proj/tests: reference_overlapped_run (the reference's own oracle)

using namespace dilocox;

static_assert(sizeof(RngStream) == sizeof(uint64_t), "RngStream must be a bare splitmix state");

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 1;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return 2;
  } catch (const FormatError& e) {
    g_err = e.what();
    return 3;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 4;
  } catch (const IoError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

RngStream rng_from(uint64_t state) {
  RngStream r(0, 0);
  std::memcpy(static_cast<void*>(&r), &state, sizeof(state));
  return r;
}
uint64_t state_of(const RngStream& r) {
  uint64_t s;
  std::memcpy(&s, static_cast<const void*>(&r), sizeof(s));
  return s;
}

std::string tname(int i) { return "t" + std::to_string(i); }

int64_t numel(const int* ndim, const int64_t* dims, int i) {
  return ndim[i] == 2 ? dims[2 * i] * dims[2 * i + 1] : dims[2 * i];
}

std::vector<int64_t> shape_of(const int* ndim, const int64_t* dims, int i) {
  if (ndim[i] == 2) return {dims[2 * i], dims[2 * i + 1]};
  return {dims[2 * i]};
}

ParamSet make_ps(int nt, const int* ndim, const int64_t* dims, const float* data) {
  ParamSet ps;
  int64_t off = 0;
  for (int i = 0; i < nt; ++i) {
    Tensor t(shape_of(ndim, dims, i));
    const int64_t n = t.size();
    if (data) std::memcpy(t.data(), data + off, sizeof(float) * static_cast<size_t>(n));
    off += n;
    ps.add(tname(i), std::move(t));
  }
  return ps;
}

void unmake_ps(const ParamSet& ps, float* out) {
  int64_t off = 0;
  for (int i = 0; i < ps.count(); ++i) {
    const Tensor& t = ps.tensor(i);
    std::memcpy(out + off, t.data(), sizeof(float) * static_cast<size_t>(t.size()));
    off += t.size();
  }
}

int r_eff_of(const int* ndim, const int64_t* dims, int i, int rank) {
  if (ndim[i] != 2) return 0;
  const int64_t m = std::min(dims[2 * i], dims[2 * i + 1]);
  return static_cast<int>(std::min<int64_t>(rank, m));
}

WarmStart make_warm(int nt, const int* ndim, const int64_t* dims, int warm_rank,
                    const float* warm_q) {
  WarmStart w;
  w.rank = warm_rank;
  if (warm_rank <= 0 || warm_q == nullptr) return w;
  int64_t off = 0;
  for (int i = 0; i < nt; ++i) {
    if (ndim[i] != 2) continue;
    const int64_t b = dims[2 * i + 1];
    const int r = r_eff_of(ndim, dims, i, warm_rank);
    Tensor q({b, static_cast<int64_t>(r)});
    std::memcpy(q.data(), warm_q + off, sizeof(float) * static_cast<size_t>(b * r));
    off += b * r;
    w.q_factors.emplace(tname(i), std::move(q));
  }
  return w;
}

// Payload (unpacked) <-> CompressedDelta.
void unpack_cd(const CompressedDelta& cd, int8_t* codes, float* scales, int* ranks) {
  int64_t co = 0, so = 0;
  for (size_t i = 0; i < cd.tensors.size(); ++i) {
    const TensorPayload& t = cd.tensors[i];
    if (t.kind == PayloadKind::LowRankQuant) {
      if (ranks) ranks[i] = t.rank;
      if (codes) {
        std::memcpy(codes + co, t.p_codes.data(), t.p_codes.size());
        std::memcpy(codes + co + t.p_codes.size(), t.q_codes.data(), t.q_codes.size());
      }
      co += static_cast<int64_t>(t.p_codes.size() + t.q_codes.size());
      if (scales) {
        std::memcpy(scales + so, t.p_scales.data(), sizeof(float) * t.p_scales.size());
        std::memcpy(scales + so + t.rank, t.q_scales.data(), sizeof(float) * t.q_scales.size());
      }
      so += 2 * t.rank;
    } else {
      if (ranks) ranks[i] = 0;
      if (codes) std::memcpy(codes + co, t.dense.codes.data(), t.dense.codes.size());
      co += static_cast<int64_t>(t.dense.codes.size());
      if (scales) scales[so] = t.dense.scale;
      so += 1;
    }
  }
}

CompressedDelta pack_cd(int nt, const int* ndim, const int64_t* dims, const int* ranks,
                        int qbits, const int8_t* codes, const float* scales) {
  CompressedDelta cd;
  cd.qbits = qbits;
  int rank = 0;
  int64_t co = 0, so = 0;
  for (int i = 0; i < nt; ++i) {
    TensorPayload t;
    t.name = tname(i);
    t.shape = shape_of(ndim, dims, i);
    t.qbits = qbits;
    if (ndim[i] == 2) {
      const int64_t a = dims[2 * i], b = dims[2 * i + 1];
      const int r = ranks[i];
      rank = std::max(rank, r);
      t.kind = PayloadKind::LowRankQuant;
      t.rank = r;
      t.p_codes.assign(codes + co, codes + co + a * r);
      t.q_codes.assign(codes + co + a * r, codes + co + a * r + b * r);
      co += (a + b) * r;
      t.p_scales.assign(scales + so, scales + so + r);
      t.q_scales.assign(scales + so + r, scales + so + 2 * r);
      so += 2 * r;
    } else {
      const int64_t n = dims[2 * i];
      t.kind = PayloadKind::DenseQuant;
      t.dense.codes.assign(codes + co, codes + co + n);
      t.dense.scale = scales[so];
      co += n;
      so += 1;
    }
    cd.tensors.push_back(std::move(t));
  }
  cd.rank = rank;
  cd.payload_bits = payload_bits_formula(cd);
  return cd;
}

QuantSpec spec_of(int qbits, int rounding) {
  QuantSpec s;
  s.qbits = qbits;
  s.rounding = rounding == 0 ? Rounding::Stochastic : Rounding::Nearest;
  return s;
}

void parallel_for(int n, int threads, const std::function<void(int)>& fn) {
  if (threads <= 1 || n <= 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  const int workers = std::min(threads, n);
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(static_cast<size_t>(workers));
  for (int w = 0; w < workers; ++w)
    pool.emplace_back([&, w] {
      try {
        for (int i = w; i < n; i += workers) fn(i);
      } catch (...) {
        errs[static_cast<size_t>(w)] = std::current_exception();
      }
    });
  for (auto& t : pool) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
const char* orc_backend(void) { return "reference"; }

uint64_t orc_stream_key(const uint64_t* parts, int n) {
  // stream_key takes an initializer_list; fold identically (rng.hpp:63-66).
  uint64_t h = 0x100000001b3ull;
  for (int i = 0; i < n; ++i) h = RngStream::mix(h ^ RngStream::mix(parts[i]));
  return h;
}
uint64_t orc_stream_init(uint64_t seed, uint64_t stream_id) {
  return state_of(RngStream(seed, stream_id));
}
uint64_t orc_next_u64(uint64_t* state) {
  RngStream r = rng_from(*state);
  const uint64_t v = r.next_u64();
  *state = state_of(r);
  return v;
}
void orc_gaussian(uint64_t* state, int64_t n, float* out) {
  RngStream r = rng_from(*state);
  Tensor t = Tensor::gaussian({n}, r);
  std::memcpy(out, t.data(), sizeof(float) * static_cast<size_t>(n));
  *state = state_of(r);
}
void orc_uniform(uint64_t* state, int64_t n, float lo, float hi, float* out) {
  RngStream r = rng_from(*state);
  Tensor t = Tensor::uniform({n}, lo, hi, r);
  std::memcpy(out, t.data(), sizeof(float) * static_cast<size_t>(n));
  *state = state_of(r);
}

int orc_matmul(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c) {
  return guarded([&] {
    Tensor ta({m, k}), tb({k, n});
    std::memcpy(ta.data(), a, sizeof(float) * static_cast<size_t>(m * k));
    std::memcpy(tb.data(), b, sizeof(float) * static_cast<size_t>(k * n));
    Tensor tc = matmul(ta, tb);
    std::memcpy(c, tc.data(), sizeof(float) * static_cast<size_t>(m * n));
  });
}
int orc_matmul_tn(int64_t k, int64_t m, int64_t n, const float* a, const float* b, float* c) {
  return guarded([&] {
    Tensor ta({k, m}), tb({k, n});
    std::memcpy(ta.data(), a, sizeof(float) * static_cast<size_t>(k * m));
    std::memcpy(tb.data(), b, sizeof(float) * static_cast<size_t>(k * n));
    Tensor tc = matmul_tn(ta, tb);
    std::memcpy(c, tc.data(), sizeof(float) * static_cast<size_t>(m * n));
  });
}
int orc_matmul_nt(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c) {
  return guarded([&] {
    Tensor ta({m, k}), tb({n, k});
    std::memcpy(ta.data(), a, sizeof(float) * static_cast<size_t>(m * k));
    std::memcpy(tb.data(), b, sizeof(float) * static_cast<size_t>(n * k));
    Tensor tc = matmul_nt(ta, tb);
    std::memcpy(c, tc.data(), sizeof(float) * static_cast<size_t>(m * n));
  });
}
int orc_orthonormalize(int64_t n, int64_t r, const float* in, float* out, int* replaced) {
  return guarded([&] {
    Tensor t({n, r});
    std::memcpy(t.data(), in, sizeof(float) * static_cast<size_t>(n * r));
    OrthoResult o = orthonormalize(t);
    std::memcpy(out, o.q.data(), sizeof(float) * static_cast<size_t>(n * r));
    if (replaced) *replaced = o.replaced_columns;
  });
}
int orc_singular_values(int64_t a, int64_t b, const float* m, double* sv_out) {
  return guarded([&] {
    Tensor t({a, b});
    std::memcpy(t.data(), m, sizeof(float) * static_cast<size_t>(a * b));
    std::vector<double> sv = singular_values(t);
    std::memcpy(sv_out, sv.data(), sizeof(double) * sv.size());
  });
}

int orc_lowrank_approx(int64_t a, int64_t b, const float* m, int r, const float* warm_q,
                       int iters, uint64_t* state, float* p_out, float* q_out) {
  return guarded([&] {
    Tensor t({a, b});
    std::memcpy(t.data(), m, sizeof(float) * static_cast<size_t>(a * b));
    Tensor wq;
    const Tensor* wp = nullptr;
    if (warm_q) {
      wq = Tensor({b, static_cast<int64_t>(r)});
      std::memcpy(wq.data(), warm_q, sizeof(float) * static_cast<size_t>(b * r));
      wp = &wq;
    }
    RngStream rng = rng_from(*state);
    LowRankResult lr = lowrank_approx(t, r, wp, iters, rng);
    *state = state_of(rng);
    std::memcpy(p_out, lr.p.data(), sizeof(float) * static_cast<size_t>(a * r));
    std::memcpy(q_out, lr.q.data(), sizeof(float) * static_cast<size_t>(b * r));
  });
}

int orc_quantize(const float* x, int64_t n, int qbits, int rounding, uint64_t* state,
                 int8_t* codes, float* scale) {
  return guarded([&] {
    RngStream rng = rng_from(*state);
    QuantChunk c = quantize(x, n, spec_of(qbits, rounding), rng);
    *state = state_of(rng);
    std::memcpy(codes, c.codes.data(), c.codes.size());
    *scale = c.scale;
  });
}

int64_t orc_codes_count(int nt, const int* ndim, const int64_t* dims, const int* ranks) {
  int64_t c = 0;
  for (int i = 0; i < nt; ++i)
    c += ndim[i] == 2 ? (dims[2 * i] + dims[2 * i + 1]) * ranks[i] : dims[2 * i];
  return c;
}
int64_t orc_scales_count(int nt, const int* ndim, const int64_t* dims, const int* ranks) {
  (void)dims;
  int64_t c = 0;
  for (int i = 0; i < nt; ++i) c += ndim[i] == 2 ? 2 * ranks[i] : 1;
  return c;
}
int64_t orc_qfactor_count(int nt, const int* ndim, const int64_t* dims, const int* ranks) {
  int64_t c = 0;
  for (int i = 0; i < nt; ++i)
    if (ndim[i] == 2) c += dims[2 * i + 1] * ranks[i];
  return c;
}

int orc_compress(int nt, const int* ndim, const int64_t* dims, const float* data, int rank,
                 int qbits, int rounding, int iters, int warm_rank, const float* warm_q,
                 uint64_t* state, int8_t* codes, float* scales, float* q_out, int* ranks,
                 uint64_t* payload_bits) {
  return guarded([&] {
    ParamSet ps = make_ps(nt, ndim, dims, data);
    WarmStart warm = make_warm(nt, ndim, dims, warm_rank, warm_q);
    RngStream rng = rng_from(*state);
    CompressResult res =
        compress(ps, rank, spec_of(qbits, rounding), warm_rank > 0 ? &warm : nullptr, iters, rng);
    *state = state_of(rng);
    unpack_cd(res.delta, codes, scales, ranks);
    if (q_out) {
      int64_t off = 0;
      for (int i = 0; i < nt; ++i) {
        if (ndim[i] != 2) continue;
        const Tensor& q = res.q_factors.at(tname(i));
        std::memcpy(q_out + off, q.data(), sizeof(float) * static_cast<size_t>(q.size()));
        off += q.size();
      }
    }
    if (payload_bits) *payload_bits = res.delta.payload_bits;
  });
}

int orc_decompress(int nt, const int* ndim, const int64_t* dims, const int* ranks,
                   const int8_t* codes, const float* scales, float* out) {
  return guarded([&] {
    CompressedDelta cd = pack_cd(nt, ndim, dims, ranks, 8, codes, scales);
    unmake_ps(decompress(cd), out);
  });
}

int orc_allreduce_avg(int D, int nt, const int* ndim, const int64_t* dims, const int* ranks,
                      const int8_t* const* codes, const float* const* scales, float* out) {
  return guarded([&] {
    std::vector<CompressedDelta> ps;
    for (int w = 0; w < D; ++w) ps.push_back(pack_cd(nt, ndim, dims, ranks, 8, codes[w], scales[w]));
    unmake_ps(allreduce_avg(ps), out);
  });
}

int orc_measure_error(int nt, const int* ndim, const int64_t* dims, const float* delta,
                      const int* ranks, const int8_t* codes, const float* scales, double* err) {
  return guarded([&] {
    ParamSet ps = make_ps(nt, ndim, dims, delta);
    *err = measure_error(ps, pack_cd(nt, ndim, dims, ranks, 8, codes, scales));
  });
}

int orc_adamw_step(int64_t n, float lr, float beta1, float beta2, float eps, float weight_decay,
                   int64_t warmup_steps, int64_t* step, float* p, const float* g, float* m,
                   float* v) {
  return guarded([&] {
    ParamSet ps, gs;
    Tensor tp({n}), tg({n});
    std::memcpy(tp.data(), p, sizeof(float) * static_cast<size_t>(n));
    std::memcpy(tg.data(), g, sizeof(float) * static_cast<size_t>(n));
    ps.add("x", std::move(tp));
    gs.add("x", std::move(tg));
    AdamWHyper h;
    h.lr = lr;
    h.beta1 = beta1;
    h.beta2 = beta2;
    h.eps = eps;
    h.weight_decay = weight_decay;
    h.warmup_steps = warmup_steps;
    AdamWState st = make_adamw_state(ps, h);
    st.step = *step;
    std::memcpy(st.m.tensor(0).data(), m, sizeof(float) * static_cast<size_t>(n));
    std::memcpy(st.v.tensor(0).data(), v, sizeof(float) * static_cast<size_t>(n));
    adamw_step(st, ps, gs);
    *step = st.step;
    std::memcpy(p, ps.tensor(0).data(), sizeof(float) * static_cast<size_t>(n));
    std::memcpy(m, st.m.tensor(0).data(), sizeof(float) * static_cast<size_t>(n));
    std::memcpy(v, st.v.tensor(0).data(), sizeof(float) * static_cast<size_t>(n));
  });
}

int orc_nesterov(int64_t n, float gamma, float beta, int classical, float* anchor, float* v,
                 const float* delta) {
  return guarded([&] {
    ParamSet a, d;
    Tensor ta({n}), td({n});
    std::memcpy(ta.data(), anchor, sizeof(float) * static_cast<size_t>(n));
    std::memcpy(td.data(), delta, sizeof(float) * static_cast<size_t>(n));
    a.add("x", std::move(ta));
    d.add("x", std::move(td));
    NesterovHyper h;
    h.lr = gamma;
    h.momentum = beta;
    h.classical = classical != 0;
    NesterovState st = make_nesterov_state(a, h);
    std::memcpy(st.velocity.tensor(0).data(), v, sizeof(float) * static_cast<size_t>(n));
    nesterov_outer_step(st, a, d);
    std::memcpy(anchor, a.tensor(0).data(), sizeof(float) * static_cast<size_t>(n));
    std::memcpy(v, st.velocity.tensor(0).data(), sizeof(float) * static_cast<size_t>(n));
  });
}

int orc_effective_rank(int nt, const int* ndim, const int64_t* dims, const float* data,
                       double tau, int r_max, int* per_tensor, int* aggregate, int* all_zero) {
  return guarded([&] {
    ParamSet ps = make_ps(nt, ndim, dims, data);
    EffectiveRank er = effective_rank(ps, tau, r_max);
    if (per_tensor)
      for (size_t i = 0; i < er.per_tensor.size(); ++i) per_tensor[i] = er.per_tensor[i].second;
    *aggregate = er.aggregate;
    *all_zero = er.all_zero ? 1 : 0;
  });
}

int orc_adapt_compression(const int* window, int len, int r1, int H1, int c, int h_min,
                          int* r_out, int* h_out) {
  return guarded([&] {
    std::vector<int> w(window, window + len);
    auto [r, h] = adapt_compression(w, r1, H1, c, h_min);
    *r_out = r;
    *h_out = h;
  });
}

double orc_omega_bound(int r, int d, int q) {
  double out = -1.0;
  if (guarded([&] { out = omega_bound(r, d, q); }) != 0) return -1.0;
  return out;
}

uint64_t orc_payload_bits(int nt, const int* ndim, const int64_t* dims, const int* ranks,
                          int qbits) {
  CompressedDelta cd;
  for (int i = 0; i < nt; ++i) {
    TensorPayload t;
    t.shape = shape_of(ndim, dims, i);
    t.qbits = qbits;
    t.kind = ndim[i] == 2 ? PayloadKind::LowRankQuant : PayloadKind::DenseQuant;
    t.rank = ranks[i];
    cd.tensors.push_back(std::move(t));
  }
  return payload_bits_formula(cd);
}

int64_t orc_serialize(int nt, const int* ndim, const int64_t* dims, const int* ranks, int rank,
                      int qbits, const int8_t* codes, const float* scales, uint8_t* out,
                      int64_t cap) {
  int64_t size = -1;
  const int rc = guarded([&] {
    CompressedDelta cd = pack_cd(nt, ndim, dims, ranks, qbits, codes, scales);
    cd.rank = rank;
    std::vector<uint8_t> bytes = serialize(cd);
    size = static_cast<int64_t>(bytes.size());
    if (out && cap >= size) std::memcpy(out, bytes.data(), bytes.size());
  });
  return rc == 0 ? size : -rc;
}

int orc_outer_round(int D, int nt, const int* ndim, const int64_t* dims, uint64_t seed,
                    int64_t round_index, int rank, int qbits, int rounding, int iters,
                    int adaptive, double tau, int r1, float gamma, float beta, int classical,
                    int threads, float* anchor, float* velocity, float* pending,
                    const float* local, int* warm_rank, float* warm_q, int* r_prime,
                    double* comp_error, uint64_t* payload_bits, double* err_norm0,
                    double* max_delta_norm) {
  return guarded([&] {
    int64_t n = 0;
    for (int i = 0; i < nt; ++i) n += numel(ndim, dims, i);
    ParamSet anc = make_ps(nt, ndim, dims, anchor);
    NesterovHyper h;
    h.lr = gamma;
    h.momentum = beta;
    h.classical = classical != 0;
    NesterovState outer = make_nesterov_state(anc, h);
    outer.velocity = make_ps(nt, ndim, dims, velocity);
    WarmStart warm = make_warm(nt, ndim, dims, *warm_rank, warm_q);
    std::vector<ParamSet> pend, loc;
    for (int w = 0; w < D; ++w) {
      pend.push_back(make_ps(nt, ndim, dims, pending + w * n));
      loc.push_back(make_ps(nt, ndim, dims, local + w * n));
    }
    const QuantSpec spec = spec_of(qbits, rounding);
    // collective_average (engine.cpp:215-263)
    std::vector<CompressedDelta> payloads(static_cast<size_t>(D));
    std::vector<std::map<std::string, Tensor>> factors(static_cast<size_t>(D));
    parallel_for(D, threads, [&](int w) {
      RngStream rng(seed, stream_key({0xc09c, static_cast<uint64_t>(round_index)}));
      CompressResult res = compress(pend[static_cast<size_t>(w)], rank, spec,
                                    &warm, iters, rng);
      payloads[static_cast<size_t>(w)] = std::move(res.delta);
      factors[static_cast<size_t>(w)] = std::move(res.q_factors);
    });
    ParamSet avg = allreduce_avg(payloads);
    *comp_error = measure_error(pend[0], payloads[0]);
    *payload_bits = payloads[0].payload_bits;
    std::vector<ParamSet> err;
    for (int w = 0; w < D; ++w) err.push_back(ps_sub(pend[static_cast<size_t>(w)], avg));
    *r_prime = 0;
    if (adaptive) *r_prime = effective_rank(avg, tau, r1).aggregate;
    // stage_deltas (engine.cpp:266-276) against the pre-update anchor
    double maxn = 0.0;
    for (int w = 0; w < D; ++w) {
      ParamSet d = ps_sub(anc, loc[static_cast<size_t>(w)]);
      ps_add(d, err[static_cast<size_t>(w)]);
      maxn = std::max(maxn, ps_l2_norm(d));
      unmake_ps(d, pending + w * n);
    }
    *max_delta_norm = maxn;
    *err_norm0 = ps_l2_norm(err[0]);
    // nesterov_outer_step + warm refresh (engine.cpp:494-501)
    nesterov_outer_step(outer, anc, avg);
    unmake_ps(anc, anchor);
    unmake_ps(outer.velocity, velocity);
    *warm_rank = rank;
    int64_t off = 0;
    for (int i = 0; i < nt; ++i) {
      if (ndim[i] != 2) continue;
      const Tensor& q = factors[0].at(tname(i));
      std::memcpy(warm_q + off, q.data(), sizeof(float) * static_cast<size_t>(q.size()));
      off += q.size();
    }
  });
}

// The reference's full overlapped training run (test_support.hpp:114-218) on the mlp /
// synthetic-regression workload (mode dilocox, M = 1): returns the initial model, the final
// anchor, the per-round mean last-step losses and the train split it trained on.
int orc_ref_mlp_overlapped_run(const int* widths, int nw, int tanh_act, int64_t samples,
                               int teacher_hidden, uint64_t seed, int D, int H1,
                               int64_t total_steps, int batch, int rank1, int qbits,
                               int rounding, int power_iters, int adaptive,
                               double eval_fraction, float* anchor0, float* anchor_out,
                               double* losses, int* nrounds, float* train_x, float* train_y,
                               int64_t* ntrain) {
  return guarded([&] {
    EngineConfig cfg;
    cfg.mode = Mode::Dilocox;
    cfg.D = D;
    cfg.M = 1;
    cfg.total_inner_steps = total_steps;
    cfg.batch = batch;
    cfg.seed = seed;
    cfg.model = mlp_spec(std::vector<int>(widths, widths + nw),
                         tanh_act ? Activation::Tanh : Activation::Relu);
    cfg.schedule.H1 = H1;
    cfg.schedule.adaptive = adaptive != 0;
    cfg.compression.rank1 = rank1;
    cfg.compression.quant.qbits = qbits;
    cfg.compression.quant.rounding = rounding ? Rounding::Nearest : Rounding::Stochastic;
    cfg.compression.power_iters = power_iters;
    Dataset full = make_synthetic_regression(samples, widths[0], widths[nw - 1], teacher_hidden,
                                             seed);
    ParamSet a0 = build_model(cfg.model, cfg.seed);
    int64_t off = 0;
    for (int i = 0; i < a0.count(); ++i) {
      const Tensor& t = a0.tensor(i);
      std::memcpy(anchor0 + off, t.data(), sizeof(float) * static_cast<size_t>(t.size()));
      off += t.size();
    }
    auto split = split_train_eval(full, eval_fraction);
    const Dataset& train = split.first;
    *ntrain = train.features.rows();
    std::memcpy(train_x, train.features.data(), sizeof(float) * static_cast<size_t>(train.features.size()));
    std::memcpy(train_y, train.targets.data(), sizeof(float) * static_cast<size_t>(train.targets.size()));
    testsup::ReferenceResult res = testsup::reference_overlapped_run(cfg, full, eval_fraction);
    off = 0;
    for (int i = 0; i < res.anchor.count(); ++i) {
      const Tensor& t = res.anchor.tensor(i);
      std::memcpy(anchor_out + off, t.data(), sizeof(float) * static_cast<size_t>(t.size()));
      off += t.size();
    }
    *nrounds = static_cast<int>(res.train_losses.size());
    for (size_t i = 0; i < res.train_losses.size(); ++i) losses[i] = res.train_losses[i];
  });
}

}  // extern "C"
