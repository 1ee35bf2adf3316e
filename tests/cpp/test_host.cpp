// C++ drop-in API tests (include/ratprog_b200/ratprog.hpp).
//   test_host cpu   — host logic only (no device calls)
//   test_host gpu   — search through librpgpu.so, checked against oracle O1
//                     (oracle/build/libo1.so, linked as test infrastructure)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <string>
#include <vector>

#include "../../oracle/o1.h"
#include "ratprog_b200/ratprog.hpp"

using namespace ratprog;

static int g_fail = 0;
#define CHECK(c)                                                                  \
  do {                                                                            \
    if (!(c)) {                                                                   \
      ++g_fail;                                                                   \
      std::cerr << __FILE__ << ":" << __LINE__ << ": CHECK failed: " #c "\n";    \
    }                                                                             \
  } while (0)

template <class E, class F>
static bool throws_with(F f, const std::string& frag) {
  try {
    f();
  } catch (const E& e) {
    return std::string(e.what()).find(frag) != std::string::npos;
  } catch (...) {
    return false;
  }
  return false;
}

static std::string root;

static void cpu_tests() {
  perf::DeviceProfile hw = perf::load_profile(root + "/data/sample_device.profile");
  CHECK(hw.W_max == 48 && hw.num_SM == 16 && hw.freq_GHz == 1.3);
  CHECK(throws_with<perf::ProfileError>([] { perf::parse_profile("R_max 1\n"); }, "expected 'key = value'"));
  CHECK(throws_with<perf::ProfileError>([] { perf::parse_profile("bogus = 1\n"); }, "unknown key"));
  CHECK(throws_with<perf::ProfileError>([] { perf::parse_profile("R_max = 1\n"); }, "missing key"));
  CHECK(poly::monomial_basis({1, 1}) == (std::vector<std::vector<int>>{{0, 0}, {0, 1}, {1, 0}, {1, 1}}));
  CHECK(poly::monomial_basis({2, 1, 1}).size() == 12);
  CHECK(data::enumerate_configs().size() == 51);
  CHECK(data::enumerate_configs(64, 64, 3).size() == 28);
  CHECK(data::integer_configs().size() == 7262);
  auto models = pipe::read_models(root + "/data/polybench/gemm.models.json");
  CHECK(models.variables == (std::vector<std::string>{"D1", "bx", "by"}));
  CHECK(models.models.size() == 5);
  CHECK(models.models.at(perf::kMetricComp).fn.num.coeffs.size() == 27);
  perf::MetricSpec spec = pipe::to_metric_spec(models);
  CHECK(spec.constants.at(perf::kMetricRegs) == 24.0);
  {
    // AltArr interop: graded-lex polynomial -> AltArr -> graded-lex, zeros dropped.
    const poly::Polynomial& p = models.models.at(perf::kMetricComp).fn.num;
    std::vector<double> c;
    std::vector<uint8_t> e;
    for (size_t k = 0; k < p.coeffs.size(); ++k)
      if (p.coeffs[k] != 0.0) {
        c.push_back(p.coeffs[k]);
        for (int x : p.basis[k]) e.push_back((uint8_t)x);
      }
    rpg_poly rp{(int32_t)c.size(), 0, c.data(), e.data()};
    std::vector<rpg_aa_elem> el(c.size());
    rpg_altarr aa{0, (int32_t)el.size(), 3, 0, el.data()};
    CHECK(rpg_aa_from_poly(&rp, 3, &aa, nullptr, 0) == RPG_OK && aa.size == (int)c.size());
    for (int i = 1; i < aa.size; ++i) CHECK(el[i].degs < el[i - 1].degs);
    poly::Polynomial back = poly::from_altarr(aa, p.variables);
    CHECK(back.coeffs == c);
    for (size_t k = 0; k < back.basis.size(); ++k)
      for (int v = 0; v < 3; ++v) CHECK(back.basis[k][v] == e[k * 3 + v]);
    std::swap(el[0], el[1]);
    CHECK(throws_with<std::invalid_argument>([&] { poly::from_altarr(aa, p.variables); }, "decreasing degree order"));
  }
  CHECK(throws_with<pipe::PipelineError>([] { pipe::parse_models("{ not json"); }, "not valid JSON"));
  CHECK(throws_with<pipe::PipelineError>([] { pipe::parse_models("{\"schema\":\"other-v9\"}"); }, "ratprog-models-v1"));
  auto missing = models;
  missing.models.erase(perf::kMetricSynch);
  CHECK(throws_with<perf::ModelError>([&] { pipe::to_metric_spec(missing); }, perf::kMetricSynch));
}

static rpg_profile prof(const perf::DeviceProfile& hw) { return pipe::detail::to_rpg(hw); }

static void gpu_tests() {
  perf::DeviceProfile hw = perf::load_profile(root + "/data/b200.profile");
  for (const char* k : {"2dconv", "gemm", "atax1"}) {
    auto models = pipe::read_models(root + "/data/polybench/" + k + ".models.json");
    perf::MetricSpec spec = pipe::to_metric_spec(models);
    auto space = data::integer_configs();
    std::vector<std::vector<long long>> tuples;
    for (long long n = 64; n <= 65536; n += 4093) tuples.push_back({n});
    for (pipe::Arith ar : {pipe::Arith::Exact, pipe::Arith::Fast}) {
      pipe::SearchOptions opts;
      opts.arith = ar;
      auto got = pipe::search_optimal_batch(spec, tuples, hw, space, opts);
      // oracle
      pipe::detail::PackedModel pk(spec);
      rpg_profile p = prof(hw);
      rpg_options o = pipe::detail::to_rpg(opts);
      std::vector<rpg_config> cfg;
      for (auto& c : space) cfg.push_back({c.bx, c.by, c.bz});
      std::vector<int64_t> flat;
      for (auto& t : tuples) flat.push_back(t[0]);
      std::vector<rpg_winner> want(tuples.size());
      o1_search_batch(&pk.model, &p, &o, cfg.data(), (int64_t)cfg.size(), flat.data(),
                      (int64_t)tuples.size(), 1, 8, want.data());
      for (size_t i = 0; i < tuples.size(); ++i) {
        CHECK(got[i].cfg_index == want[i].cfg_idx);
        CHECK(got[i].estimated_cycles == want[i].ec);
        CHECK(got[i].ties == (size_t)want[i].ties);
        CHECK(got[i].feasible == (size_t)want[i].n_feasible);
      }
    }
  }
  // Reference-shaped call sequence of do_search (ratprog_cli.cpp:277-332).
  perf::DeviceProfile sample = perf::load_profile(root + "/data/sample_device.profile");
  auto models = pipe::read_models(root + "/data/polybench/2dconv.models.json");
  perf::MetricSpec spec = pipe::to_metric_spec(models);
  ir::RationalProgram rp = pipe::generate_rp(models, sample);
  pipe::SearchOptions opts;
  opts.metrics = &spec;
  auto space = data::enumerate_configs();
  for (long long n : {1024LL, 2048LL}) {
    pipe::SearchResult r = pipe::search_optimal(rp, {n}, sample, space, opts);
    CHECK(r.evaluated == space.size());
    CHECK(r.ranking.size() + r.infeasible == space.size());
    for (size_t i = 1; i < r.ranking.size(); ++i)
      CHECK(r.ranking[i - 1].estimated_cycles <= r.ranking[i].estimated_cycles * (1 + 1e-12) ||
            i < r.ties);
    pipe::detail::PackedModel pk(spec);
    rpg_profile p = prof(sample);
    rpg_options o = pipe::detail::to_rpg(opts);
    std::vector<rpg_config> cfg;
    for (auto& c : space) cfg.push_back({c.bx, c.by, c.bz});
    int64_t d = n;
    rpg_winner w;
    std::vector<int32_t> order(space.size());
    o1_search_one(&pk.model, &p, &o, cfg.data(), (int64_t)cfg.size(), &d, 1, &w, order.data());
    CHECK((size_t)w.n_feasible == r.ranking.size());
    for (int i = 0; i < w.n_feasible; ++i) CHECK(r.ranking[i].config == space[order[i]]);
    CHECK(r.ties == (size_t)w.ties);
    const std::string csv = pipe::format_search_csv(r);
    CHECK(csv.rfind("bx,by,bz,Ec,occupancy,case\n", 0) == 0);
  }
  CHECK(throws_with<std::invalid_argument>([&] { pipe::search_optimal(spec, {64}, sample, {}, opts); },
                                           "configuration space is empty"));
  perf::MetricSpec s2 = spec;
  s2.variables = {"D2", "bx", "by"};
  for (auto& kv : s2.models) kv.second.num.variables = kv.second.den.variables = s2.variables;
  CHECK(throws_with<pipe::PipelineError>([&] { pipe::search_optimal(s2, {64}, sample, space); }, "D2"));
}

int main(int argc, char** argv) {
  root = argc > 2 ? argv[2] : ".";
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  if (mode == "cpu") cpu_tests();
  else gpu_tests();
  if (g_fail) {
    std::cerr << g_fail << " check(s) failed\n";
    return 1;
  }
  std::cout << "test_host " << mode << ": ok\n";
  return 0;
}
