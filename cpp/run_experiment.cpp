// run_experiment.cpp — drives the reference's own public engine API, run_experiment
// (engine.hpp:159-160, engine.cpp:595-610), on the mlp / synthetic-regression workload.
//
// Built twice by cpp/Makefile from this one source:
//   cpp/_build/dropin_run   linked against libdilocox_core_b200.so: the reference's proj/core
//                           with the hot path (compress / allreduce_avg / measure_error /
//                           effective_rank / nesterov_outer_step) on the B200 (dilocox_b200.cpp)
//   oracle/_ref/ref_run     linked against the unmodified reference objects (test oracle)
// so tests/test_gpu_dropin.py can compare the two runs round by round.
//
// usage: run [key=value ...] out_prefix
//   mode=dilocox|dilocox-no-overlap|dilocox-no-compress|diloco-sync|allreduce-per-step
//   D, widths=16,64,64,8, act=tanh|relu, samples, teacher, seed, H1, steps, batch, r1, q,
//   rounding=stochastic|nearest, iters, adaptive=0|1, window, tau, threads
// writes out_prefix.jsonl (one line per RoundRecord), out_prefix.bin (final params, fp32,
// ParamSet order) and out_prefix.init.bin (the initial model, build_model(model, seed)).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "dilocox/data.hpp"
#include "dilocox/engine.hpp"
#include "dilocox/model.hpp"

using namespace dilocox;

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s [key=value ...] out_prefix\n", argv[0]);
    return 2;
  }
  std::map<std::string, std::string> kv = {
      {"mode", "dilocox"}, {"D", "1"}, {"widths", "16,64,64,8"}, {"act", "tanh"},
      {"samples", "2000"}, {"teacher", "32"}, {"seed", "5"}, {"H1", "5"}, {"steps", "40"},
      {"batch", "8"}, {"r1", "8"}, {"q", "4"}, {"rounding", "stochastic"}, {"iters", "2"},
      {"adaptive", "1"}, {"window", "5"}, {"tau", "0.5"}, {"threads", "1"}};
  for (int i = 1; i + 1 < argc; ++i) {
    std::string a = argv[i];
    const size_t eq = a.find('=');
    if (eq == std::string::npos) {
      std::fprintf(stderr, "bad argument %s\n", a.c_str());
      return 2;
    }
    kv[a.substr(0, eq)] = a.substr(eq + 1);
  }
  const std::string out = argv[argc - 1];
  try {
    EngineConfig cfg;
    cfg.mode = mode_from_string(kv["mode"]);
    cfg.D = std::stoi(kv["D"]);
    cfg.M = 1;
    cfg.total_inner_steps = std::stoll(kv["steps"]);
    cfg.batch = std::stoi(kv["batch"]);
    cfg.seed = std::stoull(kv["seed"]);
    cfg.threads = std::stoi(kv["threads"]);
    std::vector<int> widths;
    std::stringstream ws(kv["widths"]);
    for (std::string x; std::getline(ws, x, ',');) widths.push_back(std::stoi(x));
    cfg.model = mlp_spec(widths, kv["act"] == "relu" ? Activation::Relu : Activation::Tanh);
    cfg.schedule.H1 = std::stoi(kv["H1"]);
    cfg.schedule.adaptive = kv["adaptive"] == "1";
    cfg.schedule.window_c = std::stoi(kv["window"]);
    cfg.schedule.tau = std::stod(kv["tau"]);
    cfg.compression.rank1 = std::stoi(kv["r1"]);
    cfg.compression.quant.qbits = std::stoi(kv["q"]);
    cfg.compression.quant.rounding = rounding_from_string(kv["rounding"]);
    cfg.compression.power_iters = std::stoi(kv["iters"]);
    Dataset full = make_synthetic_regression(std::stoll(kv["samples"]), widths.front(),
                                             widths.back(), std::stoi(kv["teacher"]), cfg.seed);
    {  // the initial model (init_round_state builds it the same way, engine.cpp:316-347)
      const ParamSet a0 = build_model(cfg.model, cfg.seed);
      std::ofstream bin(out + ".init.bin", std::ios::binary);
      for (int i = 0; i < a0.count(); ++i)
        bin.write(reinterpret_cast<const char*>(a0.tensor(i).data()),
                  static_cast<std::streamsize>(sizeof(float) * a0.tensor(i).size()));
    }
    ExperimentResult res = run_experiment(cfg, full, 0.05);
    std::ofstream js(out + ".jsonl");
    for (const RoundRecord& r : res.log.rounds) js << jsonl_line(r) << "\n";
    std::ofstream bin(out + ".bin", std::ios::binary);
    for (int i = 0; i < res.final_params.count(); ++i) {
      const Tensor& t = res.final_params.tensor(i);
      bin.write(reinterpret_cast<const char*>(t.data()),
                static_cast<std::streamsize>(sizeof(float) * t.size()));
    }
  } catch (const ValidationError& e) {
    std::fprintf(stderr, "ValidationError: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 4;
  }
  return 0;
}
