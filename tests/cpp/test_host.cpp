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

  // Direct model on the GPU: the reference's known answers
  // (test_perfmodel.cpp:228-290, 373-377).
  perf::DeviceProfile sh = perf::load_profile(root + "/data/sample_device.profile");
  CHECK(perf::active_blocks(sh, 20, 0, 256) == 6);
  CHECK(perf::active_warps(sh, 6, 256) == 48);
  CHECK(perf::occupancy(sh, 20, 0, 256) == 1.0);
  CHECK(perf::active_blocks(sh, 64, 0, 256) == 4);
  CHECK(perf::active_blocks(sh, 0, 5000, 256) == 2);
  CHECK(perf::active_blocks(sh, 20, 0, 2048) == 0);
  CHECK(perf::active_blocks(sh, 300, 0, 1024) == 0);
  perf::DeviceProfile oh;
  oh.R_max = 100000; oh.Z_max = 100000; oh.T_max = 1024; oh.B_max = 4; oh.W_max = 48; oh.num_SM = 1;
  oh.freq_GHz = 1; oh.mem_latency_cycles = 300; oh.departure_del_coal_cycles = 150;
  oh.departure_del_uncoal_cycles = 50; oh.mem_bandwidth_GBps = 2; oh.issue_cycles = 4;
  oh.load_bytes_per_warp = 100; oh.uncoal_per_mw = 5;
  perf::KernelMetrics km;
  km.comp_insts_per_thread = 18; km.uncoal_mem_insts_per_thread = 1; km.coal_mem_insts_per_thread = 1;
  km.mem_insts_per_thread = 2; km.synch_insts_per_block = 0; km.total_blocks = 4;
  auto br = perf::mwpcwp_cycles(oh, km, perf::LaunchConfig{32, 1, 1});
  CHECK(br.b_active == 4 && br.n_active_warps == 4);
  CHECK(br.case_tag == perf::CaseTag::CwpBound && br.total_cycles == 1640.0);
  perf::KernelMetrics bad = km;
  bad.mem_insts_per_thread = 3;
  CHECK(throws_with<perf::ModelError>([&] { perf::mwpcwp_cycles(oh, bad, perf::LaunchConfig{32, 1, 1}); },
                                      "metrics inconsistent"));
  perf::DeviceProfile oh1 = oh;
  oh1.B_max = 1;
  CHECK(throws_with<perf::ZeroOccupancy>([&] { perf::mwpcwp_cycles(oh1, km, perf::LaunchConfig{8, 1, 1}); },
                                         "no resident"));

  // The fit on the GPU: an exact rational ground truth is recovered
  // (test_polyfit.cpp:142-228 criterion: coefficients up to scale, < 1e-8).
  poly::PointValueSet pv;
  for (int d = 64; d <= 4096; d += 64)
    for (int bx : {1, 2, 4, 8, 16, 32})
      for (int by : {1, 2, 4, 8}) {
        pv.points.push_back({(double)d, (double)bx, (double)by});
        pv.values.push_back((3.0 * d + 20.0 * bx) / (1.0 + 0.5 * by));
      }
  poly::DegreeBounds fb{{1, 1, 0}, {0, 0, 1}};
  auto fitted = poly::fit_rational(pv, {"D1", "bx", "by"}, fb);
  const auto& fn = fitted.first;
  double worst = 0;
  for (size_t i = 0; i < pv.points.size(); i += 7) {
    double p = 0, q = 0;
    for (size_t k = 0; k < fn.num.coeffs.size(); ++k) {
      double m = 1;
      for (int v = 0; v < 3; ++v) m *= std::pow(pv.points[i][v], fn.num.basis[k][v]);
      p += fn.num.coeffs[k] * m;
    }
    for (size_t k = 0; k < fn.den.coeffs.size(); ++k) {
      double m = 1;
      for (int v = 0; v < 3; ++v) m *= std::pow(pv.points[i][v], fn.den.basis[k][v]);
      q += fn.den.coeffs[k] * m;
    }
    worst = std::max(worst, std::fabs(p / q - pv.values[i]) / std::max(1.0, std::fabs(pv.values[i])));
  }
  CHECK(worst < 1e-8);
  CHECK(fitted.second.numerical_rank >= 4);
  // fit_all_metrics over a SampleSet (pipeline.hpp:145-184).
  data::SampleSet set;
  set.metric_names = {"comp_insts_per_thread"};
  for (size_t i = 0; i < pv.points.size(); ++i) {
    data::Sample smp;
    smp.data_params = {(long long)pv.points[i][0]};
    smp.config = perf::LaunchConfig{(long long)pv.points[i][1], (long long)pv.points[i][2], 1};
    smp.metric_values["comp_insts_per_thread"] = pv.values[i];
    set.samples.push_back(smp);
  }
  auto ms = pipe::fit_all_metrics(set, {{"comp_insts_per_thread", fb}}, {{"regs_per_thread", 20.0}});
  CHECK(ms.variables == (std::vector<std::string>{"D1", "bx", "by"}));
  CHECK(ms.models.count("comp_insts_per_thread") == 1 && ms.failures.empty());
  CHECK(throws_with<pipe::PipelineError>(
      [&] { pipe::fit_all_metrics(set, {}, {{"comp_insts_per_thread", 1.0}}); }, "both a sample column"));
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
