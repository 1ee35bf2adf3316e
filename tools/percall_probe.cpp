// percall_probe — where the wall time of one reference-style drop-in call
// goes (the `ratprog search --size N` pattern, one tuple per process):
// process start -> CUDA context -> plan (kernel selection, uploads) ->
// search -> teardown.  Prints one JSON line (milliseconds).
//   percall_probe MODELS.json PROFILE [generic|specialized|fastcm]
#include <chrono>
#include <cstdio>
#include <string>

#include <cuda_runtime.h>

#include "ratprog_b200/ratprog.hpp"

using namespace ratprog;
using clk = std::chrono::steady_clock;

static double ms(clk::time_point a, clk::time_point b) {
  return std::chrono::duration<double, std::milli>(b - a).count();
}

int main(int argc, char** argv) {
  const auto t0 = clk::now();
  if (argc < 3) return 1;
  const std::string mode = argc > 3 ? argv[3] : "generic";
  cudaFree(nullptr);  // context creation
  const auto t1 = clk::now();
  auto models = pipe::read_models(argv[1]);
  perf::DeviceProfile hw = perf::load_profile(argv[2]);
  perf::MetricSpec spec = pipe::to_metric_spec(models);
  auto space = data::enumerate_configs();
  pipe::SearchOptions opts;
  opts.metrics = &spec;
  if (mode == "specialized") opts.kernel = pipe::Kernel::Specialized;
  if (mode == "fastcm") opts.arith = pipe::Arith::FastCM;
  const auto t2 = clk::now();
  pipe::SearchResult r = pipe::search_optimal(pipe::generate_rp(models, hw), {1024}, hw, space, opts);
  const auto t3 = clk::now();
  pipe::SearchResult r2 = pipe::search_optimal(pipe::generate_rp(models, hw), {2048}, hw, space, opts);
  const auto t4 = clk::now();
  int64_t compiles = 0, hits = 0;
  rpg_jit_stats(&compiles, &hits);
  printf("{\"mode\": \"%s\", \"context_ms\": %.3f, \"parse_ms\": %.3f, \"first_search_ms\": %.3f, "
         "\"second_search_ms\": %.3f, \"nvrtc_compiles\": %lld, \"disk_hits\": %lld, \"best\": \"%lldx%lld\", "
         "\"ties\": %zu}\n",
         mode.c_str(), ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), (long long)compiles,
         (long long)hits, r.best().config.bx, r.best().config.by, r2.ties);
  return 0;
}
