// C++ drop-in API tests (include/ratprog_b200/ratprog.hpp).
//   test_host cpu   — host logic only (no device calls)
//   test_host gpu   — search through librpgpu.so, checked against oracle O1
//                     (oracle/build/libo1.so, linked as test infrastructure)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
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
  {
    std::ifstream f(root + "/data/sample_device.profile");
    std::stringstream ss;
    ss << f.rdbuf();
    const std::string base = ss.str();
    auto with = [&](const std::string& from, const std::string& to) {
      std::string t = base;
      t.replace(t.find(from), from.size(), to);
      return t;
    };
    CHECK(throws_with<perf::ProfileError>([&] { perf::parse_profile(base + "W_max = 48\n"); }, "duplicate key 'W_max'"));
    CHECK(throws_with<perf::ProfileError>([&] { perf::parse_profile(with("W_max = 48", "W_max = -4")); }, "'W_max' must be positive"));
    CHECK(throws_with<perf::ProfileError>([&] { perf::parse_profile(with("W_max = 48", "W_max = 4.5")); }, "'W_max' must be an integer"));
    CHECK(throws_with<perf::ProfileError>([&] { perf::parse_profile(with("W_max = 48", "W_max = 4x")); }, "bad numeric value '4x'"));
    CHECK(throws_with<perf::ProfileError>([&] { perf::parse_profile(with("T_max = 1024", "T_max = 2048")); }, "T_max exceeds 1024"));
    CHECK(perf::parse_profile(with("W_max = 48", "W_max = 0x30   # hex")).W_max == 48);
  }
  CHECK(data::enumerate_configs(1024, 32, 1).size() == 6);
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

// Bare-program text and literal lowering (ir_text.hpp, rational.hpp:109-148):
// correctly rounded doubles (Python float(Fraction) gives the expected bits).
static void ir_tests() {
  const std::pair<const char*, double> lits[] = {
      {"1/3", 0x1.5555555555555p-2},
      {"-7/2", -0x1.cp+1},
      {"123456789012345678901234567890123456789/1000000000000000000000000000000000000000",
       0x1.f9add3746f65fp-4},
      {"9007199254740993", 0x1p+53},
      {"9007199254740995/1", 0x1.0000000000002p+53},
      {"1/10", 0x1.999999999999ap-4},
      {"333333333333333333333333333333333333333333/999999999999999999999999999999999999999999999",
       0x1.5d867c3ece2a5p-12},
      {"2.5", 0x1.4p+1},
      {"-0.125", -0x1p-3},
      {"12345678901234567890123456789", 0x1.3f20d99235f65p+93},
      {"0/5", 0.0}};
  for (const auto& [text, want] : lits) CHECK(to_double(parse_rational(text)) == want);
  CHECK(throws_with<std::invalid_argument>([] { parse_rational("3/0"); }, "zero denominator"));
  CHECK(throws_with<std::invalid_argument>([] { parse_rational("3x"); }, "trailing characters"));
  const char* text =
      "# comment\n"
      "inputs: D1 bx by issue_cycles\n"
      "output: y\n"
      "0: mul t D1 bx   # trailing comment\n"
      "1: cmp_lt c t 4096\n"
      "2: branch_if c -> 3 5\n"
      "3: floor_div y t 7/2\n"
      "4: jump -> 6\n"
      "5: neg y 1\n"
      "6: halt_return y\n";
  ir::RationalProgram p = ir::parse(text);
  CHECK(p.inputs.size() == 4 && p.output == "y" && p.body.size() == 7);
  CHECK(p.body[2].op == ir::Opcode::BranchIf && p.body[2].jump_targets == (std::vector<size_t>{3, 5}));
  CHECK(p.body[3].operands[1].lit == Rational(7, 2));
  CHECK(throws_with<ir::ParseError>([] { ir::parse("inputs: a\noutput: y\n0: frob y a\n"); },
                                    "line 3, column 4: unknown opcode 'frob'"));
  CHECK(throws_with<ir::ParseError>([] { ir::parse("inputs: a\noutput: y\n1: neg y a\n"); },
                                    "out of order; expected 0"));
  CHECK(throws_with<ir::ParseError>([] { ir::parse("inputs: a\noutput: y\n0: add y a 1.5\n"); },
                                    "decimal literals"));
  CHECK(throws_with<ir::ParseError>([] { ir::parse("inputs: a\noutput: y\n"); }, "empty program body"));
  // make_binding_plan's errors (pipeline.hpp:482-516) surface before any GPU
  // work: an unknown input, a data parameter the tuple does not have.
  perf::DeviceProfile hw = perf::parse_profile(
      "R_max = 65536\nZ_max = 12288\nT_max = 1024\nB_max = 8\nW_max = 48\nnum_SM = 16\n"
      "freq_GHz = 1.3\nmem_latency_cycles = 436\ndeparture_del_coal_cycles = 4\n"
      "departure_del_uncoal_cycles = 40\nmem_bandwidth_GBps = 144\nissue_cycles = 4\n"
      "load_bytes_per_warp = 128\nuncoal_per_mw = 32\n");
  const auto space = data::enumerate_configs();
  ir::RationalProgram q7 = ir::parse("inputs: Q7 bx\noutput: y\n0: mul y Q7 bx\n1: halt_return y\n");
  CHECK(throws_with<pipe::PipelineError>([&] { pipe::search_optimal(q7, {64}, hw, space); },
                                         "program input 'Q7' is neither a block dimension"));
  ir::RationalProgram d2 = ir::parse("inputs: D2 bx\noutput: y\n0: mul y D2 bx\n1: halt_return y\n");
  CHECK(throws_with<pipe::PipelineError>([&] { pipe::search_optimal(d2, {64}, hw, space); },
                                         "program input 'D2' has no value: 1 data parameter(s) were given"));
  CHECK(throws_with<std::invalid_argument>([&] { pipe::search_optimal(d2, {64, 3}, hw, {}); },
                                           "configuration space is empty"));
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
  // Several devices behind one call (device 0 listed three times here):
  // winners identical to one device, on both axes (8 and 2 tuples).
  {
    auto models = pipe::read_models(root + "/data/polybench/gemm.models.json");
    perf::MetricSpec spec = pipe::to_metric_spec(models);
    auto space = data::integer_configs();
    for (size_t nt : {8u, 2u}) {
      std::vector<std::vector<long long>> tuples;
      for (size_t i = 0; i < nt; ++i) tuples.push_back({(long long)(100 + 977 * i)});
      pipe::SearchOptions one;
      pipe::SearchOptions three;
      three.devices = {0, 0, 0};
      auto a = pipe::search_optimal_batch(spec, tuples, hw, space, one);
      auto b = pipe::search_optimal_batch(spec, tuples, hw, space, three);
      for (size_t i = 0; i < nt; ++i) {
        CHECK(a[i].cfg_index == b[i].cfg_index && a[i].estimated_cycles == b[i].estimated_cycles);
        CHECK(a[i].ties == b[i].ties && a[i].feasible == b[i].feasible && a[i].case_tag == b[i].case_tag);
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

  // Program from generate_rp without opts.metrics: Ec from the program,
  // occupancy from opts regs/shared, tag "-" (pipeline.hpp:648-650).
  {
    pipe::SearchOptions o2;
    o2.regs_per_thread = 64;
    pipe::SearchResult r = pipe::search_optimal(rp, {2048}, sample, space, o2);
    pipe::SearchResult full = pipe::search_optimal(rp, {2048}, sample, space, opts);
    CHECK(r.evaluated == full.evaluated && r.infeasible == full.infeasible);
    for (const auto& row : r.ranking) {
      CHECK(row.case_tag == "-");
      CHECK(row.occupancy == perf::occupancy(sample, 64, 0, row.config.threads()));
    }
    std::vector<double> a, b;
    for (const auto& row : r.ranking) a.push_back(row.estimated_cycles);
    for (const auto& row : full.ranking) b.push_back(row.estimated_cycles);
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    CHECK(a == b);
  }

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
  // Full MwpCwpBreakdown KATs (test_perfmodel.cpp:253-396).
  auto mk = [](double comp, double unc, double coal, double synch, double blocks) {
    perf::KernelMetrics k;
    k.comp_insts_per_thread = comp; k.uncoal_mem_insts_per_thread = unc;
    k.coal_mem_insts_per_thread = coal; k.mem_insts_per_thread = unc + coal;
    k.synch_insts_per_block = synch; k.total_blocks = blocks;
    return k;
  };
  const perf::LaunchConfig c32{32, 1, 1};
  perf::KernelMetrics km = mk(18, 1, 1, 0, 4);
  auto br = perf::mwpcwp_cycles(oh, km, c32);  // cwp-bound oracle
  CHECK(br.b_active == 4 && br.n_active_warps == 4);
  CHECK(br.mem_cycles == 800.0 && br.comp_cycles == 80.0);
  CHECK(br.mwp == 2.0 && br.cwp == 4.0 && br.rep == 1.0);
  CHECK(br.case_tag == perf::CaseTag::CwpBound);
  CHECK(br.cycles_pre_synch == 1640.0 && br.synch_cost == 0.0 && br.total_cycles == 1640.0);
  {  // both-saturated oracle
    perf::DeviceProfile h = oh;
    h.B_max = 2; h.departure_del_coal_cycles = 50;
    auto r = perf::mwpcwp_cycles(h, mk(23, 0, 2, 3, 2), c32);
    CHECK(r.b_active == 2 && r.n_active_warps == 2);
    CHECK(r.mem_cycles == 600.0 && r.comp_cycles == 100.0 && r.mwp == 2.0 && r.cwp == 2.0);
    CHECK(r.case_tag == perf::CaseTag::BothSaturated);
    CHECK(r.cycles_pre_synch == 750.0 && r.synch_cost == 300.0 && r.total_cycles == 1050.0);
  }
  {  // mwp-bound oracle
    perf::DeviceProfile h = oh;
    h.B_max = 8; h.num_SM = 2; h.departure_del_coal_cycles = 75; h.mem_bandwidth_GBps = 4;
    auto r = perf::mwpcwp_cycles(h, mk(98, 0, 2, 0, 16), c32);
    CHECK(r.b_active == 8 && r.n_active_warps == 8);
    CHECK(r.mem_cycles == 600.0 && r.comp_cycles == 400.0 && r.mwp == 4.0 && r.cwp == 2.5);
    CHECK(r.rep == 1.0 && r.case_tag == perf::CaseTag::MwpBound && r.total_cycles == 3500.0);
    // raw latency, not the weighted one (test_perfmodel.cpp:313-332)
    h.departure_del_coal_cycles = 30; h.departure_del_uncoal_cycles = 30;
    auto r2 = perf::mwpcwp_cycles(h, mk(98, 1, 1, 0, 16), c32);
    CHECK(r2.mwp == 4.0 && r2.case_tag == perf::CaseTag::MwpBound && r2.total_cycles == 3500.0);
  }
  {  // compute-only (test_perfmodel.cpp:334-353)
    auto r = perf::mwpcwp_cycles(oh, mk(50, 0, 0, 2, 4), c32);
    CHECK(r.b_active == 4 && r.n_active_warps == 4 && r.mem_cycles == 0.0 && r.comp_cycles == 200.0);
    CHECK(r.mwp == 4.0 && r.case_tag == perf::CaseTag::CwpBound);
    CHECK(r.cycles_pre_synch == 200.0 && r.synch_cost == 150.0 * 3 * 2 * 4);
    CHECK(r.total_cycles == 200.0 + 3600.0);
    CHECK(perf::mwpcwp_cycles(oh, mk(50, 0, 0, 0, 4), c32).total_cycles == 200.0);
  }
  {  // repetition count (test_perfmodel.cpp:385-396)
    auto real = perf::mwpcwp_cycles(oh, mk(50, 0, 0, 0, 5), c32, perf::RepMode::Real);
    CHECK(real.rep == 1.25 && real.total_cycles == 250.0);
    auto ceil = perf::mwpcwp_cycles(oh, mk(50, 0, 0, 0, 5), c32, perf::RepMode::Ceil);
    CHECK(ceil.rep == 2.0 && ceil.total_cycles == 400.0);
  }
  // rejections (test_perfmodel.cpp:355-383)
  perf::KernelMetrics bad = mk(10, 1, 1, 0, 4);
  bad.mem_insts_per_thread = 3;
  CHECK(throws_with<perf::ModelError>([&] { perf::mwpcwp_cycles(oh, bad, c32); },
                                      "metrics inconsistent"));
  perf::KernelMetrics neg = mk(10, 1, 1, 0, 4);
  neg.comp_insts_per_thread = -1;
  CHECK(throws_with<perf::ModelError>([&] { perf::mwpcwp_cycles(oh, neg, c32); }, "non-negative"));
  CHECK(throws_with<perf::ZeroOccupancy>(
      [&] { perf::mwpcwp_cycles(oh, mk(10, 1, 1, 0, 4), perf::LaunchConfig{64, 32, 1}); },
      "no resident block"));
  perf::DeviceProfile oh1 = oh;
  oh1.B_max = 1;
  CHECK(throws_with<perf::ZeroOccupancy>([&] { perf::mwpcwp_cycles(oh1, km, perf::LaunchConfig{8, 1, 1}); },
                                         "no resident warp"));
  perf::KernelMetrics heavy = mk(10, 1, 1, 0, 4);
  heavy.regs_per_thread = 1e9;
  CHECK(throws_with<perf::ZeroOccupancy>([&] { perf::mwpcwp_cycles(oh, heavy, c32); }, "no resident"));

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
  if (mode == "cpu") {
    cpu_tests();
    ir_tests();
  }
  else gpu_tests();
  if (g_fail) {
    std::cerr << g_fail << " check(s) failed\n";
    return 1;
  }
  std::cout << "test_host " << mode << ": ok\n";
  return 0;
}
