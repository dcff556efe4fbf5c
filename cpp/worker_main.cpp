// worker_main.cpp — one DiLoCoX worker process per GPU driving the device-resident outer
// sync through the C-ABI alone (no PyTorch): the multi-GPU production path a C++ host
// (the reference's engine, one process per worker) runs.
//
//   dlx_comm_unique_id (rank 0) -> file -> dlx_ctx_create_dist (NCCL communicator)
//   per round (run_round_overlapped order, engine.cpp:458-509):
//     dlx_compress(pending, warm Q)           compress.cpp:146-183, shared stream engine.cpp:226
//     dlx_exchange(payload -> gathered, Q0)   collective_average's exchange, engine.cpp:215-263
//     dlx_effective_rank(gathered)            r' (engine.cpp:258-261), read before the update
//     dlx_outer_update(overlapped)            e, staging, Nesterov (engine.cpp:254-276, 494-501)
//     dlx_adapt_compression(window)           next round's rank (engine.cpp:476-487)
//
// usage: worker_main rank world device uid_file out_prefix [rounds r1 q adaptive]
// The parameter table is the SURVEY C1 mini-OPT layout; inputs come from the device
// generator bit-identical to the reference's Tensor::gaussian (dlx_fill_gaussian): anchor
// 0.02 N(0,1) (seed 7), local_w = anchor - 1e-3 N(0,1) (seed 1, worker w).
// Writes out_prefix.bin (the final anchor, fp32, ParamSet order) and out_prefix.txt (one line
// per round: round r_t r_prime comp_error).
#include <cuda_runtime.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "dlx_b200.h"

namespace {

void ok(dlx_status s, const char* what) {
  if (s != DLX_OK) {
    std::fprintf(stderr, "%s failed (%d): %s\n", what, static_cast<int>(s), dlx_last_error());
    std::exit(3);
  }
}
void cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    std::fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
    std::exit(4);
  }
}

// splitmix64 stream construction (rng.hpp:13-16, 63-66): the host only builds the state
constexpr uint64_t kG = 0x9e3779b97f4a7c15ull;
uint64_t fmix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
uint64_t mix(uint64_t z) { return fmix(z + kG); }
uint64_t stream_key2(uint64_t a, uint64_t b) {
  uint64_t h = 0x100000001b3ull;
  h = mix(h ^ mix(a));
  return mix(h ^ mix(b));
}
uint64_t stream_init(uint64_t seed, uint64_t sid) {
  const uint64_t s = mix(seed ^ kG);
  return mix(s ^ mix(sid + 0xbf58476d1ce4e5b9ull));
}

struct Shape {
  int nd;
  int64_t a, b;
};

std::vector<Shape> mini_opt() {  // h=512, ffn=2048, L=2, vocab 8192, pos 514
  const int64_t h = 512, f = 2048;
  std::vector<Shape> t = {{2, 8192, h}, {2, 514, h}};
  for (int l = 0; l < 2; ++l) {
    for (int p = 0; p < 4; ++p) {
      t.push_back({2, h, h});
      t.push_back({1, h, 1});
    }
    t.push_back({1, h, 1});
    t.push_back({1, h, 1});
    t.push_back({2, h, f});
    t.push_back({1, f, 1});
    t.push_back({2, f, h});
    t.push_back({1, h, 1});
    t.push_back({1, h, 1});
    t.push_back({1, h, 1});
  }
  t.push_back({1, h, 1});
  t.push_back({1, h, 1});
  return t;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 6) {
    std::fprintf(stderr, "usage: %s rank world device uid_file out_prefix [rounds r1 q adaptive]\n",
                 argv[0]);
    return 2;
  }
  const int rank = std::atoi(argv[1]), world = std::atoi(argv[2]), device = std::atoi(argv[3]);
  const std::string uid_file = argv[4], out = argv[5];
  const int rounds = argc > 6 ? std::atoi(argv[6]) : 4;
  const int r1 = argc > 7 ? std::atoi(argv[7]) : 8;
  const int q = argc > 8 ? std::atoi(argv[8]) : 4;
  const bool adaptive = argc > 9 ? std::atoi(argv[9]) != 0 : false;
  const float gamma = 0.7f, beta = 0.9f;
  const double tau = 0.5;
  const int window_c = 5, H1 = 125, h_min = (H1 + 9) / 10;

  // ---- bootstrap: rank 0 publishes the NCCL unique id through a file
  unsigned char uid[DLX_UNIQUE_ID_BYTES];
  if (rank == 0) {
    ok(dlx_comm_unique_id(uid), "dlx_comm_unique_id");
    const std::string tmp = uid_file + ".tmp";
    std::ofstream(tmp, std::ios::binary).write(reinterpret_cast<char*>(uid), sizeof(uid));
    std::rename(tmp.c_str(), uid_file.c_str());
  } else {
    for (int i = 0;; ++i) {
      std::ifstream f(uid_file, std::ios::binary);
      if (f && f.read(reinterpret_cast<char*>(uid), sizeof(uid))) break;
      if (i > 6000) {
        std::fprintf(stderr, "no unique id at %s\n", uid_file.c_str());
        return 5;
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(10));
    }
  }
  dlx_ctx* ctx = nullptr;
  ok(dlx_ctx_create_dist(device, rank, world, uid, &ctx), "dlx_ctx_create_dist");
  cu(cudaSetDevice(device), "cudaSetDevice");
  cudaStream_t s;
  cu(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");

  // ---- layout + device state (RoundState's outer fields, engine.hpp:114-132)
  const std::vector<Shape> shapes = mini_opt();
  std::vector<int> nd;
  std::vector<int64_t> dims;
  int n2 = 0;
  for (const Shape& x : shapes) {
    nd.push_back(x.nd);
    dims.push_back(x.a);
    dims.push_back(x.b);
    n2 += x.nd == 2;
  }
  dlx_layout* L = nullptr;
  ok(dlx_layout_create(ctx, static_cast<int>(shapes.size()), nd.data(), dims.data(), &L),
     "dlx_layout_create");
  const int64_t slab = dlx_layout_slab_elems(L);
  const int64_t pb = dlx_payload_bytes(L, r1, q);
  const int64_t qel = dlx_factor_offsets(L, r1, 1, nullptr);
  float *anchor, *velocity, *pending, *local, *warm_q;
  uint8_t *payload, *gathered;
  dlx_round_stats* stats;
  int* per;
  double* energy;
  uint64_t* draws;
  cu(cudaMalloc(&anchor, 4 * slab), "malloc");
  cu(cudaMalloc(&velocity, 4 * slab), "malloc");
  cu(cudaMalloc(&pending, 4 * slab), "malloc");
  cu(cudaMalloc(&local, 4 * slab), "malloc");
  cu(cudaMalloc(&warm_q, 4 * qel), "malloc");
  cu(cudaMalloc(&payload, pb), "malloc");
  cu(cudaMalloc(&gathered, pb * world), "malloc");
  cu(cudaMalloc(&stats, sizeof(dlx_round_stats)), "malloc");
  cu(cudaMalloc(&per, sizeof(int) * n2), "malloc");
  cu(cudaMalloc(&energy, sizeof(double) * n2), "malloc");
  cu(cudaMalloc(&draws, 8), "malloc");
  // zeroed on the worker stream (a legacy-stream memset would race the non-blocking stream)
  for (float* p : {anchor, velocity, pending, local})
    cu(cudaMemsetAsync(p, 0, 4 * slab, s), "memset");
  ok(dlx_fill_gaussian(ctx, L, anchor, nullptr, 0.02f, 7, 0xA7C4, 0, s), "fill anchor");
  ok(dlx_fill_gaussian(ctx, L, local, anchor, -1e-3f, 1, 0xDA7A, rank, s), "fill local");

  std::vector<int> window;
  int r_t = r1, warm_rank = 0;
  std::FILE* log = std::fopen((out + ".txt").c_str(), "w");
  for (int round = 1; round <= rounds; ++round) {
    if (round == 1) {  // no exchange in round 1: stage delta only (engine.cpp:473)
      ok(dlx_stage_deltas(ctx, L, anchor, local, nullptr, pending, nullptr, s), "stage");
      std::fprintf(log, "%d %d 0 0\n", round, r_t);
      continue;
    }
    const uint64_t st = stream_init(1, stream_key2(0xC09C, static_cast<uint64_t>(round)));
    const int64_t pbr = dlx_payload_bytes(L, r_t, q);
    const int64_t qelr = dlx_factor_offsets(L, r_t, 1, nullptr);
    ok(dlx_exchange_wait_warm(ctx, s), "wait warm");
    ok(dlx_compress(ctx, L, pending, r_t, q, DLX_ROUND_STOCHASTIC, 2, st,
                    warm_rank == r_t ? warm_q : nullptr, warm_rank, payload, warm_q, draws, s),
       "dlx_compress");
    ok(dlx_exchange(ctx, payload, pbr, gathered, warm_q, qelr, 0, s), "dlx_exchange");
    int rp = 0;
    if (adaptive)  // r' of every averaged round (engine.cpp:258-261), before the update
      ok(dlx_effective_rank(ctx, L, r_t, q, world, gathered, tau, per, energy, s), "effrank");
    ok(dlx_outer_update(ctx, L, r_t, q, world, gathered, rank, DLX_MODE_OVERLAPPED, pending,
                        anchor, local, velocity, gamma, beta, 0, stats, s),
       "dlx_outer_update");
    std::vector<int> h_per(static_cast<size_t>(n2));
    std::vector<double> h_en(static_cast<size_t>(n2));
    cu(cudaMemcpyAsync(h_per.data(), per, sizeof(int) * n2, cudaMemcpyDeviceToHost, s), "d2h");
    cu(cudaMemcpyAsync(h_en.data(), energy, sizeof(double) * n2, cudaMemcpyDeviceToHost, s), "d2h");
    dlx_round_stats hs;
    cu(cudaMemcpyAsync(&hs, stats, sizeof(hs), cudaMemcpyDeviceToHost, s), "d2h");
    cu(cudaStreamSynchronize(s), "sync");
    ok(dlx_comm_check(ctx), "dlx_comm_check");
    if (adaptive) {
      int allz = 0;
      ok(dlx_effective_rank_reduce(L, h_per.data(), h_en.data(), r1, &rp, &allz), "reduce");
      window.push_back(rp);  // push_rank_window (engine.cpp:278-284)
      if (static_cast<int>(window.size()) > window_c) window.erase(window.begin());
    }
    warm_rank = r_t;
    int r_next = r_t, h_next = H1;
    ok(dlx_adapt_compression(window.data(), static_cast<int>(window.size()), r1, H1, window_c,
                             h_min, &r_next, &h_next), "adapt");
    const double ce = hs.err_den > 0 ? hs.err_num / hs.err_den : 0.0;
    std::fprintf(log, "%d %d %d %.17g\n", round, r_t, rp, ce);
    if (adaptive) r_t = r_next;
  }
  std::fclose(log);
  std::vector<float> h(static_cast<size_t>(slab));
  cu(cudaMemcpy(h.data(), anchor, 4 * slab, cudaMemcpyDeviceToHost), "d2h anchor");
  std::vector<int64_t> off(shapes.size());
  ok(dlx_layout_offsets(L, off.data()), "offsets");
  std::ofstream bin(out + ".bin", std::ios::binary);
  for (size_t i = 0; i < shapes.size(); ++i) {
    const int64_t n = shapes[i].nd == 2 ? shapes[i].a * shapes[i].b : shapes[i].a;
    bin.write(reinterpret_cast<const char*>(h.data() + off[i]), static_cast<std::streamsize>(4 * n));
  }
  dlx_layout_destroy(L);
  dlx_ctx_destroy(ctx);
  return 0;
}
