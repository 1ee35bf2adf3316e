// ratprog_b200/ratprog.hpp — C++17 drop-in for the reference `ratprog` hot
// path, running on the B200 evaluator behind include/rpg.h (librpgpu.so).
//
// Same namespaces, type names, function names, argument meanings and
// exception types/messages as the reference headers for the search path
// (citations relative to /root/reference/proj/include/ratprog):
//   perf::DeviceProfile / parse_profile / load_profile   perfmodel.hpp:50-208
//   perf::LaunchConfig, RepMode, CaseTag, MetricSpec,
//   check_metric_spec                                     perfmodel.hpp:79-84, 271-282, 401-456
//   poly::DegreeBounds / monomial_basis / Polynomial /
//   RationalFunction                                      polyfit.hpp:41-84
//   data::enumerate_configs                               datakit.hpp:79-94
//   pipe::MetricModelSet / parse_models / read_models /
//   to_metric_spec / generate_rp                          pipeline.hpp:58-68, 188-255, 1020-1089
//   pipe::SearchOptions / SearchRow / SearchResult /
//   search_optimal                                        pipeline.hpp:438-680
//   pipe::format_search_{csv,text,jsonl}                  pipeline.hpp:897-934
//   poly::PointValueSet / fit_rational                    polyfit.hpp:133-135, 337-427
//   data::Sample / SampleSet, pipe::sample_variables /
//   default_bounds / metric_points / fit_all_metrics      datakit.hpp:40-75, pipeline.hpp:72-184
//   perf::KernelMetrics / MwpCwpBreakdown /
//   active_blocks / active_warps / occupancy /
//   mwpcwp_cycles                                          perfmodel.hpp:68-77, 239-395
//   poly::from_altarr / ratfunc_from_altarr (KLARAPTOR AltArr_t interop)
// A caller of the reference's `--models` search path (ratprog_cli.cpp:
// 277-332) compiles against this header unchanged: `generate_rp` returns an
// ir::RationalProgram that carries the metric spec, and `search_optimal`
// evaluates it on the GPU.  New: `search_optimal_batch` sweeps many data
// tuples per launch.  Every number is computed by librpgpu.so; there is no
// CPU evaluator here.
#pragma once

#include <algorithm>
#include <array>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <fstream>
#include <map>
#include <memory>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <cctype>
#include <vector>

#include "rpg.h"

namespace ratprog {

// ---------------------------------------------------------------------------
namespace poly {

struct DimensionMismatch : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DenominatorNearZero : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct DegreeBounds {
  std::vector<int> num, den;
};

// Graded-lex exponent tuples (polyfit.hpp:50-73): every tuple e with
// 0 <= e_i <= bounds_i, grouped by total degree (ascending), each group in
// lexicographic order.  Built with a mixed-radix counter (lex order) whose
// tuples are appended to their degree's bucket.
inline std::vector<std::vector<int>> monomial_basis(const std::vector<int>& bounds) {
  for (int b : bounds)
    if (b < 0) throw std::invalid_argument("negative degree bound");
  const size_t nv = bounds.size();
  const int max_deg = std::accumulate(bounds.begin(), bounds.end(), 0);
  std::vector<std::vector<std::vector<int>>> by_degree(max_deg + 1);
  std::vector<int> e(nv, 0);
  for (;;) {
    by_degree[std::accumulate(e.begin(), e.end(), 0)].push_back(e);
    size_t i = nv;  // increment the last digit, carrying leftwards
    while (i > 0 && e[i - 1] == bounds[i - 1]) e[--i] = 0;
    if (i == 0) break;
    ++e[i - 1];
  }
  std::vector<std::vector<int>> out;
  for (auto& bucket : by_degree)
    for (auto& t : bucket) out.push_back(std::move(t));
  return out;
}

struct Polynomial {
  std::vector<std::string> variables;
  std::vector<std::vector<int>> basis;
  std::vector<double> coeffs;
};

struct RationalFunction {
  Polynomial num, den;
};

struct FitReport {
  double residual_norm = 0.0;
  int numerical_rank = 0;
  std::vector<double> singular_values;
  bool truncated = false;
};

// Paper-artifact interop (KLARAPTOR per-metric AltArr_t polynomials,
// PAPER.md:39-56; rpg_aa_* in rpg.h): an AltArr-form polynomial -> the
// reference's Polynomial with terms in graded-lex basis order (the
// evaluator's summation order).  Throws std::invalid_argument on a
// non-canonical AltArr.
inline Polynomial from_altarr(const rpg_altarr& a, const std::vector<std::string>& variables) {
  if ((int)variables.size() != a.nvar)
    throw std::invalid_argument("from_altarr: variable count does not match nvar");
  const int cap = std::max(a.size, 1);
  std::vector<double> c(cap);
  std::vector<uint8_t> e((size_t)cap * std::max(a.nvar, 1));
  int32_t n = 0;
  char err[512] = {0};
  if (rpg_aa_to_poly(&a, c.data(), e.data(), cap, &n, err, sizeof err) != RPG_OK)
    throw std::invalid_argument(err);
  Polynomial p;
  p.variables = variables;
  for (int k = 0; k < n; ++k) {
    p.basis.emplace_back(e.begin() + (size_t)k * a.nvar, e.begin() + (size_t)(k + 1) * a.nvar);
    p.coeffs.push_back(c[k]);
  }
  return p;
}

inline RationalFunction ratfunc_from_altarr(const rpg_altarr& num, const rpg_altarr& den,
                                            const std::vector<std::string>& variables) {
  return RationalFunction{from_altarr(num, variables), from_altarr(den, variables)};
}

// ---- the fit (polyfit.hpp:133-135, 337-427) on the GPU (rpg_fit_rational)
struct DegenerateFit : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SvdFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline constexpr double kDefaultRankTol = 1e-10;

struct PointValueSet {
  std::vector<std::vector<double>> points;
  std::vector<double> values;
};

// poly::fit_rational: homogeneous least-squares rational fit over the
// graded-lex bases of `bounds`, including the positivity safeguard.  Every
// FLOP runs in the K3 kernels; this only packs arguments.
inline std::pair<RationalFunction, FitReport> fit_rational(const PointValueSet& pv,
                                                           const std::vector<std::string>& variables,
                                                           const DegreeBounds& bounds,
                                                           double rank_tol = kDefaultRankTol,
                                                           int device = 0) {
  const size_t nv = variables.size();
  if (bounds.num.size() != nv || bounds.den.size() != nv)
    throw DimensionMismatch("fit_rational: degree bounds do not match the variables");
  if (pv.points.size() != pv.values.size())
    throw DimensionMismatch("fit_rational: points/values size mismatch");
  std::vector<double> X;
  X.reserve(pv.points.size() * nv);
  for (const auto& x : pv.points) {
    if (x.size() != nv) throw DimensionMismatch("fit_rational: point dimension mismatch");
    X.insert(X.end(), x.begin(), x.end());
  }
  const auto nb = monomial_basis(bounds.num), db = monomial_basis(bounds.den);
  const size_t n = nb.size() + db.size();
  std::vector<double> coef(n), sigma(std::max<size_t>(1, std::min(pv.values.size(), n)));
  int32_t rank = 0, truncated = 0, safeguard = 0;
  double residual = 0.0;
  char err[512] = {0};
  const int rc = rpg_fit_rational(X.data(), pv.values.data(), (int64_t)pv.values.size(),
                                  (int32_t)nv, bounds.num.data(), bounds.den.data(), rank_tol,
                                  device, coef.data(), sigma.data(), &rank, &truncated, &residual,
                                  &safeguard, err, sizeof err);
  if (rc == RPG_E_FIT) {
    if (std::string(err).find("svd") == 0) throw SvdFailure(err);
    throw DegenerateFit(err);
  }
  if (rc == RPG_E_INVALID) throw std::invalid_argument(err);
  if (rc != RPG_OK) throw std::runtime_error(std::string("librpgpu: ") + err);
  RationalFunction f;
  f.num = Polynomial{variables, nb, std::vector<double>(coef.begin(), coef.begin() + nb.size())};
  f.den = Polynomial{variables, db, std::vector<double>(coef.begin() + nb.size(), coef.end())};
  FitReport rep;
  rep.residual_norm = residual;
  rep.numerical_rank = rank;
  rep.singular_values.assign(sigma.begin(), sigma.begin() + std::min(pv.values.size(), n));
  rep.truncated = truncated != 0;
  return {std::move(f), std::move(rep)};
}

}  // namespace poly

// ---------------------------------------------------------------------------
namespace perf {

struct ProfileError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ModelError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct DeviceProfile {
  long long R_max = 0, Z_max = 0, T_max = 0, B_max = 0, W_max = 0, num_SM = 0;
  double freq_GHz = 0, mem_latency_cycles = 0, departure_del_coal_cycles = 0,
         departure_del_uncoal_cycles = 0, mem_bandwidth_GBps = 0, issue_cycles = 0;
  long long load_bytes_per_warp = 0, uncoal_per_mw = 0;
};

struct ZeroOccupancy : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// perf::KernelMetrics (perfmodel.hpp:68-77).
struct KernelMetrics {
  double regs_per_thread = 0;
  double shared_words_per_block = 0;
  double comp_insts_per_thread = 0;
  double mem_insts_per_thread = 0;
  double uncoal_mem_insts_per_thread = 0;
  double coal_mem_insts_per_thread = 0;
  double synch_insts_per_block = 0;
  double total_blocks = 0;
};

struct LaunchConfig {
  long long bx = 1, by = 1, bz = 1;
  long long threads() const { return bx * by * bz; }
  bool operator==(const LaunchConfig& o) const { return bx == o.bx && by == o.by && bz == o.bz; }
  bool operator<(const LaunchConfig& o) const {
    if (bx != o.bx) return bx < o.bx;
    if (by != o.by) return by < o.by;
    return bz < o.bz;
  }
};

enum class RepMode { Real, Ceil };
enum class CaseTag { BothSaturated, CwpBound, MwpBound };

inline const char* case_name(CaseTag t) {
  switch (t) {
    case CaseTag::BothSaturated: return "both_saturated";
    case CaseTag::CwpBound: return "cwp_bound";
    case CaseTag::MwpBound: return "mwp_bound";
  }
  return "?";
}

// perf::MwpCwpBreakdown (perfmodel.hpp:284-296): every field is filled by
// the GPU direct model (rpg_mwpcwp_breakdown_batch).
struct MwpCwpBreakdown {
  long long b_active = 0;
  long long n_active_warps = 0;
  double mem_cycles = 0;
  double comp_cycles = 0;
  double mwp = 0;
  double cwp = 0;
  double rep = 0;
  CaseTag case_tag = CaseTag::CwpBound;
  double cycles_pre_synch = 0;
  double synch_cost = 0;
  double total_cycles = 0;
};

namespace detail {
inline rpg_profile profile_to_rpg(const DeviceProfile& hw) {
  rpg_profile p;
  p.R_max = hw.R_max; p.Z_max = hw.Z_max; p.T_max = hw.T_max; p.B_max = hw.B_max;
  p.W_max = hw.W_max; p.num_SM = hw.num_SM; p.freq_GHz = hw.freq_GHz;
  p.mem_latency_cycles = hw.mem_latency_cycles;
  p.departure_del_coal_cycles = hw.departure_del_coal_cycles;
  p.departure_del_uncoal_cycles = hw.departure_del_uncoal_cycles;
  p.mem_bandwidth_GBps = hw.mem_bandwidth_GBps; p.issue_cycles = hw.issue_cycles;
  p.load_bytes_per_warp = hw.load_bytes_per_warp; p.uncoal_per_mw = hw.uncoal_per_mw;
  return p;
}

// One row through rpg_mwpcwp_cycles_batch (the GPU direct model).
inline void direct_row(const DeviceProfile& hw, const KernelMetrics& m, const LaunchConfig& c,
                       RepMode mode, double* total, int32_t* b, int32_t* w, uint8_t* tag,
                       int32_t* status) {
  const double mv[RPG_N_METRICS] = {m.regs_per_thread, m.shared_words_per_block,
                                    m.comp_insts_per_thread, m.uncoal_mem_insts_per_thread,
                                    m.coal_mem_insts_per_thread, m.synch_insts_per_block,
                                    m.total_blocks};
  const rpg_profile p = profile_to_rpg(hw);
  const rpg_config cfg{c.bx, c.by, c.bz};
  char err[512] = {0};
  const int rc = rpg_mwpcwp_cycles_batch(&p, mv, &cfg, 1,
                                         mode == RepMode::Ceil ? RPG_REP_CEIL : RPG_REP_REAL, 0,
                                         total, b, w, tag, status, err, sizeof err);
  if (rc == RPG_E_PROFILE) throw ProfileError(err);
  if (rc == RPG_E_INVALID) throw std::invalid_argument(err);
  if (rc != RPG_OK) throw std::runtime_error(std::string("librpgpu: ") + err);
}
}  // namespace detail

// perf::active_blocks / active_warps / occupancy (perfmodel.hpp:239-266),
// evaluated by the GPU direct-model kernel.
inline long long active_blocks(const DeviceProfile& hw, double R, double Z, long long T) {
  KernelMetrics m;
  m.regs_per_thread = R;
  m.shared_words_per_block = Z;
  int32_t b = 0, w = 0, st = 0;
  uint8_t tag = 0;
  double tot = 0;
  detail::direct_row(hw, m, LaunchConfig{T, 1, 1}, RepMode::Real, &tot, &b, &w, &tag, &st);
  return b;
}

inline long long active_warps(const DeviceProfile& hw, long long b_active, long long T) {
  if (b_active <= 0) return 0;
  const long long w = b_active * T / 32;  // floor, perfmodel.hpp:258
  return w < hw.W_max ? w : hw.W_max;
}

inline double occupancy(const DeviceProfile& hw, double R, double Z, long long T) {
  if (hw.W_max <= 0) return 0.0;
  return static_cast<double>(active_warps(hw, active_blocks(hw, R, Z, T), T)) /
         static_cast<double>(hw.W_max);
}

// perf::mwpcwp_cycles (perfmodel.hpp:298-395) on the GPU, the full
// breakdown.  Same exceptions in the same order: ModelError for inconsistent
// or negative metrics, ZeroOccupancy when no block or no warp is resident.
inline MwpCwpBreakdown mwpcwp_cycles(const DeviceProfile& hw, const KernelMetrics& m,
                                     const LaunchConfig& config, RepMode mode = RepMode::Real) {
  const double km[8] = {m.regs_per_thread, m.shared_words_per_block, m.comp_insts_per_thread,
                        m.mem_insts_per_thread, m.uncoal_mem_insts_per_thread,
                        m.coal_mem_insts_per_thread, m.synch_insts_per_block, m.total_blocks};
  const rpg_profile p = detail::profile_to_rpg(hw);
  const rpg_config cfg{config.bx, config.by, config.bz};
  rpg_breakdown o{};
  char err[512] = {0};
  const int rc = rpg_mwpcwp_breakdown_batch(
      &p, km, &cfg, 1, mode == RepMode::Ceil ? RPG_REP_CEIL : RPG_REP_REAL, 0, &o, err, sizeof err);
  if (rc == RPG_E_PROFILE) throw ProfileError(err);
  if (rc == RPG_E_INVALID) throw std::invalid_argument(err);
  if (rc != RPG_OK) throw std::runtime_error(std::string("librpgpu: ") + err);
  switch (o.status) {
    case 3: throw ModelError("metrics inconsistent: uncoal + coal must equal mem_insts");
    case 2: throw ModelError("metrics must be non-negative");
    case 1: throw ZeroOccupancy("configuration cannot launch (no resident block)");
    case 4: throw ZeroOccupancy("configuration yields no resident warp");
    default: break;
  }
  MwpCwpBreakdown r;
  r.b_active = o.b_active;
  r.n_active_warps = o.n_active_warps;
  r.mem_cycles = o.mem_cycles;
  r.comp_cycles = o.comp_cycles;
  r.mwp = o.mwp;
  r.cwp = o.cwp;
  r.rep = o.rep;
  r.case_tag = o.case_tag == RPG_CASE_BOTH_SATURATED ? CaseTag::BothSaturated
               : o.case_tag == RPG_CASE_MWP_BOUND   ? CaseTag::MwpBound
                                                    : CaseTag::CwpBound;
  r.cycles_pre_synch = o.cycles_pre_synch;
  r.synch_cost = o.synch_cost;
  r.total_cycles = o.total_cycles;
  return r;
}

namespace detail {
// DeviceProfile's fields in the profile-file key order (perfmodel.hpp:91-108):
// name, and a pointer to the count (integer) or rate member.
struct ProfileField {
  const char* name;
  long long DeviceProfile::*count;
  double DeviceProfile::*rate;
};
inline const std::vector<ProfileField>& profile_fields() {
  static const std::vector<ProfileField> f = {
      {"R_max", &DeviceProfile::R_max, nullptr},
      {"Z_max", &DeviceProfile::Z_max, nullptr},
      {"T_max", &DeviceProfile::T_max, nullptr},
      {"B_max", &DeviceProfile::B_max, nullptr},
      {"W_max", &DeviceProfile::W_max, nullptr},
      {"num_SM", &DeviceProfile::num_SM, nullptr},
      {"freq_GHz", nullptr, &DeviceProfile::freq_GHz},
      {"mem_latency_cycles", nullptr, &DeviceProfile::mem_latency_cycles},
      {"departure_del_coal_cycles", nullptr, &DeviceProfile::departure_del_coal_cycles},
      {"departure_del_uncoal_cycles", nullptr, &DeviceProfile::departure_del_uncoal_cycles},
      {"mem_bandwidth_GBps", nullptr, &DeviceProfile::mem_bandwidth_GBps},
      {"issue_cycles", nullptr, &DeviceProfile::issue_cycles},
      {"load_bytes_per_warp", &DeviceProfile::load_bytes_per_warp, nullptr},
      {"uncoal_per_mw", &DeviceProfile::uncoal_per_mw, nullptr}};
  return f;
}
inline const std::vector<std::string>& profile_keys() {
  static const std::vector<std::string> keys = [] {
    std::vector<std::string> k;
    for (const ProfileField& f : profile_fields()) k.push_back(f.name);
    return k;
  }();
  return keys;
}
// The text between the first and last character that is not a blank.
inline std::string trim(const std::string& s) {
  size_t b = 0, e = s.size();
  auto blank = [](char c) { return c == ' ' || c == '\t' || c == '\r'; };
  while (b < e && blank(s[b])) ++b;
  while (e > b && blank(s[e - 1])) --e;
  return s.substr(b, e - b);
}
}  // namespace detail

// perf::parse_profile (perfmodel.hpp:111-180): "key = value" lines, '#'
// comments, blank lines; every key exactly once; values parsed by std::stod
// with full consumption, positive; count fields integral; T_max <= 1024.
// Same checks, order and messages as the reference.
inline DeviceProfile parse_profile(const std::string& text) {
  const auto& fields = detail::profile_fields();
  std::vector<double> value(fields.size(), 0.0);
  std::vector<bool> given(fields.size(), false);
  size_t line_no = 0, pos = 0;
  auto fail = [&](const std::string& what) -> void {
    throw ProfileError("profile line " + std::to_string(line_no) + ": " + what);
  };
  while (pos <= text.size()) {
    size_t nl = text.find('\n', pos);
    if (nl == std::string::npos) nl = text.size();
    std::string line = text.substr(pos, nl - pos);
    pos = nl + 1;
    ++line_no;
    line = detail::trim(line.substr(0, line.find('#')));
    if (!line.empty()) {
      const size_t eq = line.find('=');
      if (eq == std::string::npos) fail("expected 'key = value'");
      const std::string key = detail::trim(line.substr(0, eq));
      const std::string val = detail::trim(line.substr(eq + 1));
      size_t k = 0;
      while (k < fields.size() && key != fields[k].name) ++k;
      if (k == fields.size()) fail("unknown key '" + key + "'");
      if (given[k]) fail("duplicate key '" + key + "'");
      double v = 0.0;
      bool ok = !val.empty();
      if (ok) {
        try {
          size_t used = 0;
          v = std::stod(val, &used);
          ok = used == val.size();
        } catch (const std::exception&) {
          ok = false;
        }
      }
      if (!ok) fail("bad numeric value '" + val + "'");
      if (!(v > 0)) fail("'" + key + "' must be positive");
      value[k] = v;
      given[k] = true;
    }
    if (nl == text.size()) break;
  }
  for (size_t k = 0; k < fields.size(); ++k)
    if (!given[k]) throw ProfileError(std::string("profile is missing key '") + fields[k].name + "'");
  DeviceProfile hw;
  for (size_t k = 0; k < fields.size(); ++k) {
    if (fields[k].count) {
      if (value[k] != std::floor(value[k]))
        throw ProfileError(std::string("profile key '") + fields[k].name + "' must be an integer");
      hw.*(fields[k].count) = static_cast<long long>(value[k]);
    } else {
      hw.*(fields[k].rate) = value[k];
    }
  }
  if (hw.T_max > 1024) throw ProfileError("T_max exceeds 1024, the architectural block limit");
  return hw;
}

inline DeviceProfile load_profile(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ProfileError("cannot open device profile '" + path + "'");
  std::ostringstream buf;
  buf << in.rdbuf();
  try {
    return parse_profile(buf.str());
  } catch (const ProfileError& e) {
    throw ProfileError(path + ": " + e.what());
  }
}

inline constexpr const char* kMetricComp = "comp_insts_per_thread";
inline constexpr const char* kMetricUncoal = "uncoal_mem_insts_per_thread";
inline constexpr const char* kMetricCoal = "coal_mem_insts_per_thread";
inline constexpr const char* kMetricSynch = "synch_insts_per_block";
inline constexpr const char* kMetricTotalBlocks = "total_blocks";
inline constexpr const char* kMetricRegs = "regs_per_thread";
inline constexpr const char* kMetricShared = "shared_words_per_block";

inline const std::vector<std::string>& required_metric_names() {
  static const std::vector<std::string> names = {kMetricComp, kMetricUncoal, kMetricCoal,
                                                 kMetricSynch, kMetricTotalBlocks};
  return names;
}

struct MetricSpec {
  std::vector<std::string> variables;
  std::map<std::string, poly::RationalFunction> models;
  std::map<std::string, double> constants;
  bool covers(const std::string& name) const {
    return models.count(name) || constants.count(name);
  }
};

// perf::check_metric_spec (perfmodel.hpp:428-456): the five required
// metrics and regs/shared each need a model or a constant; variables are
// D<k> data parameters or bx/by/bz (never a profile field name), bx and by
// both present; every model uses the shared variable order.
inline void check_metric_spec(const MetricSpec& spec) {
  std::vector<std::string> need = required_metric_names();
  need.push_back(kMetricRegs);
  need.push_back(kMetricShared);
  for (const std::string& name : need)
    if (!spec.covers(name)) throw ModelError("metric '" + name + "' has neither a model nor a constant");
  const auto& hw_keys = detail::profile_keys();
  int blocks_seen = 0;  // bit 0: bx, bit 1: by
  for (const std::string& v : spec.variables) {
    if (std::count(hw_keys.begin(), hw_keys.end(), v))
      throw ModelError("variable '" + v + "' collides with a hardware field");
    if (v == "bx") blocks_seen |= 1;
    else if (v == "by") blocks_seen |= 2;
    else if (v != "bz" && !(v.size() >= 2 && v[0] == 'D' &&
                            std::all_of(v.begin() + 1, v.end(), [](char c) { return c >= '0' && c <= '9'; })))
      throw ModelError("variable '" + v + "' is not a data parameter (D1..Dd) or block dimension");
  }
  if (blocks_seen != 3) throw ModelError("metric variables must include bx and by");
  for (const auto& entry : spec.models)
    if (entry.second.num.variables != spec.variables)
      throw ModelError("model '" + entry.first + "' disagrees with the shared variable order");
}

struct EmitOptions {
  RepMode rep_mode = RepMode::Real;
  int scale_pow10 = 40;
};

}  // namespace perf

// ---------------------------------------------------------------------------
namespace data {

// data::Sample / SampleSet (datakit.hpp:40-75): the fit's input rows.
struct Provenance {
  enum class Kind { Measured, Synthetic };
  Kind kind = Kind::Measured;
  std::uint64_t seed = 0;
  double noise_rel = 0;
};

struct Sample {
  std::vector<long long> data_params;
  perf::LaunchConfig config;
  std::map<std::string, double> metric_values;
};

struct SampleSet {
  std::vector<std::string> metric_names;
  std::vector<Sample> samples;
  Provenance provenance;
  std::size_t dims() const { return samples.empty() ? 0 : samples.front().data_params.size(); }
};

// data::enumerate_configs (datakit.hpp:79-94): power-of-two block shapes
// 2^i x 2^j x 2^k (j = 0 unless dims >= 2, k = 0 unless dims == 3, each
// dimension <= 1024) with min_threads <= threads <= max_threads, in lex
// order of (bx, by, bz).
inline std::vector<perf::LaunchConfig> enumerate_configs(long long max_threads = 1024,
                                                         long long min_threads = 32,
                                                         int dims = 2) {
  if (min_threads < 1 || min_threads > max_threads || max_threads > 1024)
    throw std::invalid_argument("enumerate_configs: need 1 <= min_threads <= max_threads <= 1024");
  if (dims < 1 || dims > 3) throw std::invalid_argument("enumerate_configs: dims must be 1, 2 or 3");
  const int ey = dims >= 2 ? 10 : 0, ez = dims == 3 ? 10 : 0;
  std::vector<perf::LaunchConfig> out;
  for (int i = 0; i <= 10; ++i)
    for (int j = 0; j <= ey; ++j)
      for (int k = 0; k <= ez; ++k) {
        const perf::LaunchConfig c{1LL << i, 1LL << j, 1LL << k};
        if (c.threads() >= min_threads && c.threads() <= max_threads) out.push_back(c);
      }
  return out;
}

// Every integer block shape with min <= bx*by[*bz] <= max (the dense grids
// of the benchmark sweeps; lex order).
inline std::vector<perf::LaunchConfig> integer_configs(long long max_threads = 1024, int dims = 2,
                                                       long long min_threads = 1) {
  std::vector<perf::LaunchConfig> out;
  for (long long bx = 1; bx <= max_threads; ++bx)
    for (long long by = 1; by <= (dims >= 2 ? max_threads / bx : 1); ++by)
      for (long long bz = 1; bz <= (dims >= 3 ? max_threads / (bx * by) : 1); ++bz)
        if (bx * by * bz >= min_threads) out.push_back({bx, by, bz});
  return out;
}

}  // namespace data

// ---------------------------------------------------------------------------
// Minimal JSON reader for the models / kernel-spec files.
namespace json {

struct Value {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  bool b = false;
  double num = 0;
  std::string str;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;
  const Value* find(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}
  Value parse() {
    Value v = value();
    ws();
    if (i_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  size_t i_ = 0;
  [[noreturn]] void fail(const char* why) {
    throw ParseError(std::string(why) + " at offset " + std::to_string(i_));
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\t' || s_[i_] == '\r')) ++i_;
  }
  Value value() {
    ws();
    if (i_ >= s_.size()) fail("unexpected end");
    const char c = s_[i_];
    Value v;
    if (c == '{') {
      v.kind = Value::Object;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == '}') { ++i_; return v; }
      while (true) {
        ws();
        if (i_ >= s_.size() || s_[i_] != '"') fail("expected key");
        std::string k = string();
        ws();
        if (i_ >= s_.size() || s_[i_] != ':') fail("expected ':'");
        ++i_;
        v.obj.emplace_back(std::move(k), value());
        ws();
        if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
        if (i_ < s_.size() && s_[i_] == '}') { ++i_; break; }
        fail("expected ',' or '}'");
      }
    } else if (c == '[') {
      v.kind = Value::Array;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == ']') { ++i_; return v; }
      while (true) {
        v.arr.push_back(value());
        ws();
        if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
        if (i_ < s_.size() && s_[i_] == ']') { ++i_; break; }
        fail("expected ',' or ']'");
      }
    } else if (c == '"') {
      v.kind = Value::String;
      v.str = string();
    } else if (s_.compare(i_, 4, "true") == 0) {
      v.kind = Value::Bool; v.b = true; i_ += 4;
    } else if (s_.compare(i_, 5, "false") == 0) {
      v.kind = Value::Bool; i_ += 5;
    } else if (s_.compare(i_, 4, "null") == 0) {
      i_ += 4;
    } else {
      v.kind = Value::Number;
      const char* b = s_.c_str() + i_;
      char* e = nullptr;
      v.num = std::strtod(b, &e);
      if (e == b) fail("bad value");
      i_ += static_cast<size_t>(e - b);
    }
    return v;
  }
  std::string string() {
    ++i_;  // opening quote
    std::string out;
    while (i_ < s_.size() && s_[i_] != '"') {
      if (s_[i_] == '\\') {
        ++i_;
        if (i_ >= s_.size()) fail("bad escape");
        const char e = s_[i_];
        out += e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e;
      } else {
        out += s_[i_];
      }
      ++i_;
    }
    if (i_ >= s_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
};

inline Value parse(const std::string& text) { return Parser(text).parse(); }

}  // namespace json

// ---------------------------------------------------------------------------
namespace pipe {

struct PipelineError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NoFeasibleConfig : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct MetricModel {
  poly::RationalFunction fn;
  poly::FitReport report;
};

struct MetricModelSet {
  std::vector<std::string> variables;
  std::map<std::string, MetricModel> models;
  std::map<std::string, double> constants;
  std::map<std::string, std::string> failures;
};

struct AllMetricsFailed : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// pipe::sample_variables / default_bounds / metric_points (pipeline.hpp:72-133).
// The model variables of a sample set (pipeline.hpp:72-86): D1..Dd, bx, by,
// and bz when some sample uses a third block dimension.
inline std::vector<std::string> sample_variables(const data::SampleSet& set) {
  const bool uses_bz = std::any_of(set.samples.begin(), set.samples.end(),
                                   [](const data::Sample& s) { return s.config.bz != 1; });
  std::vector<std::string> vars(set.dims());
  for (std::size_t i = 0; i < vars.size(); ++i) vars[i] = "D" + std::to_string(i + 1);
  vars.insert(vars.end(), {"bx", "by"});
  if (uses_bz) vars.emplace_back("bz");
  return vars;
}

// pipe::default_bounds (pipeline.hpp:88-93): numerator 2, denominator 1 per
// variable.
inline poly::DegreeBounds default_bounds(std::size_t n_variables) {
  return poly::DegreeBounds{std::vector<int>(n_variables, 2), std::vector<int>(n_variables, 1)};
}

namespace detail {
// Column-major-by-sample coordinates (m x nv, row per sample) of a sample
// set in `variables` order (pipeline.hpp:97-113 coordinate rules).
inline std::vector<double> sample_matrix(const data::SampleSet& set,
                                         const std::vector<std::string>& variables) {
  const size_t nv = variables.size();
  // per variable: -1 bx, -2 by, -3 bz, k >= 0 data parameter k
  std::vector<long> src(nv);
  for (size_t j = 0; j < nv; ++j) {
    const std::string& v = variables[j];
    if (v == "bx") src[j] = -1;
    else if (v == "by") src[j] = -2;
    else if (v == "bz") src[j] = -3;
    else if (v.size() >= 2 && v[0] == 'D') src[j] = (long)std::stoul(v.substr(1)) - 1;
    else throw PipelineError("variable '" + v + "' is not a data parameter or block dimension");
  }
  std::vector<double> X(set.samples.size() * nv);
  for (size_t r = 0; r < set.samples.size(); ++r) {
    const data::Sample& s = set.samples[r];
    for (size_t j = 0; j < nv; ++j) {
      const long k = src[j];
      double x;
      if (k == -1) x = (double)s.config.bx;
      else if (k == -2) x = (double)s.config.by;
      else if (k == -3) x = (double)s.config.bz;
      else if (k >= 0 && (size_t)k < s.data_params.size()) x = (double)s.data_params[k];
      else throw PipelineError("variable '" + variables[j] + "' exceeds the sample's data-parameter count");
      X[r * nv + j] = x;
    }
  }
  return X;
}

inline std::vector<double> metric_column(const data::SampleSet& set, const std::string& metric) {
  std::vector<double> y(set.samples.size());
  for (size_t r = 0; r < y.size(); ++r) {
    auto it = set.samples[r].metric_values.find(metric);
    if (it == set.samples[r].metric_values.end())
      throw PipelineError("sample set has no metric column '" + metric + "'");
    y[r] = it->second;
  }
  return y;
}
}  // namespace detail

// pipe::metric_points (pipeline.hpp:115-133): one metric column as
// (point, value) pairs.
inline poly::PointValueSet metric_points(const data::SampleSet& set, const std::string& metric,
                                         const std::vector<std::string>& variables) {
  const std::vector<double> y = detail::metric_column(set, metric);
  const std::vector<double> X = detail::sample_matrix(set, variables);
  poly::PointValueSet out;
  out.values = y;
  out.points.resize(y.size());
  for (size_t r = 0; r < y.size(); ++r)
    out.points[r].assign(X.begin() + r * variables.size(), X.begin() + (r + 1) * variables.size());
  return out;
}

struct FitOptions {
  double rank_tol = poly::kDefaultRankTol;
  int device = 0;
};

// pipe::fit_all_metrics (pipeline.hpp:145-184) the B200 way: the sample
// coordinates are laid out once (m x nv) and every metric column is fitted
// concurrently on the GPU (rpg_fit_rational_multi: one upload of X, one
// stream per metric).  The reference's argument checks run first, in its
// metric order and with its messages; numerical failures (DegenerateFit /
// SvdFailure) are recorded per metric, a full wipeout raises
// AllMetricsFailed.  Each metric's model is what poly::fit_rational returns
// for it alone.
inline MetricModelSet fit_all_metrics(const data::SampleSet& samples,
                                      const std::map<std::string, poly::DegreeBounds>& bounds,
                                      const std::map<std::string, double>& constants,
                                      const FitOptions& opts = {}) {
  if (samples.samples.empty()) throw std::invalid_argument("fit_all_metrics: sample set is empty");
  MetricModelSet out;
  out.variables = sample_variables(samples);
  out.constants = constants;
  const size_t nv = out.variables.size(), m = samples.samples.size(), k = samples.metric_names.size();
  std::vector<poly::DegreeBounds> b(k);
  std::vector<std::vector<double>> ys(k);
  for (size_t i = 0; i < k; ++i) {
    const std::string& metric = samples.metric_names[i];
    if (constants.count(metric))
      throw PipelineError("metric '" + metric + "' is both a sample column and a declared constant");
    auto it = bounds.find(metric);
    b[i] = it != bounds.end() ? it->second : default_bounds(nv);
    if (b[i].num.size() != nv || b[i].den.size() != nv)
      throw PipelineError("degree bounds for metric '" + metric + "' must have " +
                          std::to_string(nv) + " entries per side");
    ys[i] = detail::metric_column(samples, metric);
  }
  const std::vector<double> X = detail::sample_matrix(samples, out.variables);
  struct Out {
    std::vector<double> coef, sigma;
    int32_t rank = 0, truncated = 0, safeguard = 0;
    double residual = 0.0;
  };
  std::vector<Out> res(k);
  std::vector<rpg_fit_job> jobs(k);
  for (size_t i = 0; i < k; ++i) {
    const size_t n = poly::monomial_basis(b[i].num).size() + poly::monomial_basis(b[i].den).size();
    res[i].coef.assign(n, 0.0);
    res[i].sigma.assign(std::max<size_t>(1, std::min(m, n)), 0.0);
    rpg_fit_job& J = jobs[i];
    J = rpg_fit_job{};
    J.y = ys[i].data();
    J.num_bounds = b[i].num.data();
    J.den_bounds = b[i].den.data();
    J.coef_out = res[i].coef.data();
    J.sigma_out = res[i].sigma.data();
    J.rank_out = &res[i].rank;
    J.truncated_out = &res[i].truncated;
    J.residual_out = &res[i].residual;
    J.safeguard_out = &res[i].safeguard;
  }
  char err[512] = {0};
  const int rc = rpg_fit_rational_multi(X.data(), (int64_t)m, (int32_t)nv, jobs.data(), (int32_t)k,
                                        opts.rank_tol, opts.device, err, sizeof err);
  if (rc == RPG_E_INVALID) throw std::invalid_argument(err);
  if (rc != RPG_OK) throw std::runtime_error(std::string("librpgpu: ") + err);
  for (size_t i = 0; i < k; ++i) {
    const std::string& metric = samples.metric_names[i];
    if (jobs[i].status == RPG_E_FIT) {
      out.failures[metric] = jobs[i].message;
      continue;
    }
    if (jobs[i].status == RPG_E_INVALID) throw std::invalid_argument(jobs[i].message);
    if (jobs[i].status != RPG_OK) throw std::runtime_error(std::string("librpgpu: ") + jobs[i].message);
    const auto nb = poly::monomial_basis(b[i].num), db = poly::monomial_basis(b[i].den);
    MetricModel mm;
    mm.fn.num = poly::Polynomial{out.variables, nb,
                                 std::vector<double>(res[i].coef.begin(), res[i].coef.begin() + nb.size())};
    mm.fn.den = poly::Polynomial{out.variables, db,
                                 std::vector<double>(res[i].coef.begin() + nb.size(), res[i].coef.end())};
    const size_t n_sig = std::min(m, nb.size() + db.size());
    mm.report.residual_norm = res[i].residual;
    mm.report.numerical_rank = res[i].rank;
    mm.report.singular_values.assign(res[i].sigma.begin(), res[i].sigma.begin() + n_sig);
    mm.report.truncated = res[i].truncated != 0;
    out.models[metric] = std::move(mm);
  }
  if (out.models.empty()) {
    std::string msg = "no metric could be fitted:";
    for (const auto& f : out.failures) msg += " [" + f.first + ": " + f.second + "]";
    throw AllMetricsFailed(msg);
  }
  return out;
}

namespace detail {

inline std::vector<int> int_array(const json::Value& v, const std::string& what) {
  if (v.kind != json::Value::Array) throw PipelineError(what + " must be an array");
  std::vector<int> out;
  for (const auto& x : v.arr) out.push_back(static_cast<int>(x.num));
  return out;
}

inline std::vector<double> num_array(const json::Value& v, const std::string& what) {
  if (v.kind != json::Value::Array) throw PipelineError(what + " must be an array");
  std::vector<double> out;
  for (const auto& x : v.arr) out.push_back(x.num);
  return out;
}

// datakit.hpp:491-517 (ratfunc_from_json): same messages.
inline poly::RationalFunction ratfunc_from_json(const json::Value& j,
                                                const std::vector<std::string>& variables,
                                                const std::string& metric) {
  for (const char* key : {"num_bounds", "num_coeffs", "den_bounds", "den_coeffs"})
    if (!j.find(key))
      throw PipelineError("metric '" + metric + "' is missing '" + key + "'");
  poly::RationalFunction f;
  auto read_poly = [&](const char* bkey, const char* ckey, poly::Polynomial& p) {
    const std::vector<int> bounds = int_array(*j.find(bkey), bkey);
    if (bounds.size() != variables.size())
      throw PipelineError("metric '" + metric + "': '" + bkey + "' must have one entry per variable");
    p.variables = variables;
    p.basis = poly::monomial_basis(bounds);
    p.coeffs = num_array(*j.find(ckey), ckey);
    if (p.coeffs.size() != p.basis.size())
      throw PipelineError("metric '" + metric + "': '" + std::string(ckey) + "' must have " +
                          std::to_string(p.basis.size()) + " entries for these bounds");
  };
  read_poly("num_bounds", "num_coeffs", f.num);
  read_poly("den_bounds", "den_coeffs", f.den);
  return f;
}

}  // namespace detail

// pipe::parse_models (pipeline.hpp:1020-1069).
inline MetricModelSet parse_models(const std::string& text) {
  json::Value j;
  try {
    j = json::parse(text);
  } catch (const json::ParseError& e) {
    throw PipelineError(std::string("models file is not valid JSON: ") + e.what());
  }
  const json::Value* schema = j.find("schema");
  if (!schema || schema->str != "ratprog-models-v1")
    throw PipelineError("models file schema must be 'ratprog-models-v1'");
  MetricModelSet m;
  const json::Value* vars = j.find("variables");
  if (!vars) throw PipelineError("models file is malformed: missing 'variables'");
  for (const auto& v : vars->arr) m.variables.push_back(v.str);
  if (m.variables.empty()) throw PipelineError("models file declares no variables");
  if (const json::Value* c = j.find("constants"))
    for (const auto& kv : c->obj) m.constants[kv.first] = kv.second.num;
  const json::Value* metrics = j.find("metrics");
  if (!metrics || metrics->kind != json::Value::Object)
    throw PipelineError("models file is missing the 'metrics' object");
  for (const auto& [name, body] : metrics->obj) {
    MetricModel model;
    model.fn = detail::ratfunc_from_json(body, m.variables, name);
    if (const json::Value* rep = body.find("report")) {
      if (const json::Value* r = rep->find("residual_norm")) model.report.residual_norm = r->num;
      if (const json::Value* r = rep->find("numerical_rank"))
        model.report.numerical_rank = static_cast<int>(r->num);
      if (const json::Value* r = rep->find("truncated")) model.report.truncated = r->b;
    }
    m.models[name] = std::move(model);
  }
  if (const json::Value* f = j.find("failures"))
    for (const auto& kv : f->obj) m.failures[kv.first] = kv.second.str;
  return m;
}

inline MetricModelSet read_models(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw PipelineError("cannot open '" + path + "' for reading");
  std::ostringstream buf;
  buf << in.rdbuf();
  try {
    return parse_models(buf.str());
  } catch (const PipelineError& e) {
    throw PipelineError(path + ": " + e.what());
  }
}

// pipe::to_metric_spec (pipeline.hpp:188-195).
inline perf::MetricSpec to_metric_spec(const MetricModelSet& m) {
  perf::MetricSpec spec;
  spec.variables = m.variables;
  for (const auto& [name, model] : m.models) spec.models[name] = model.fn;
  spec.constants = m.constants;
  perf::check_metric_spec(spec);
  return spec;
}

}  // namespace pipe

// ---------------------------------------------------------------------------
// Rational literals of bare programs.  The reference's Rational is Boost's
// cpp_rational (rational.hpp:17-19); on the B200 path a literal only ever
// enters the evaluator as the nearest double (the reference's C lowering
// prints to_double of each literal, pipeline.hpp:276-433), so the shim keeps
// the exact value as sign + decimal digit strings (any length) and converts
// with correct rounding.  No arithmetic is offered on it.
struct DivisionByZero : std::runtime_error {
  DivisionByZero() : std::runtime_error("division by zero") {}
  explicit DivisionByZero(const std::string& what) : std::runtime_error(what) {}
};

struct Rational {
  bool negative = false;
  std::string num = "0", den = "1";  // decimal digits, no leading zeros
  Rational() = default;
  Rational(long long v) : negative(v < 0), num(std::to_string(v < 0 ? -(unsigned long long)v : (unsigned long long)v)) {}
  Rational(long long n, long long d) {
    if (d == 0) throw DivisionByZero("make_rational: zero denominator");
    negative = (n < 0) != (d < 0) && n != 0;
    unsigned long long un = n < 0 ? -(unsigned long long)n : (unsigned long long)n;
    unsigned long long ud = d < 0 ? -(unsigned long long)d : (unsigned long long)d;
    const unsigned long long g = std::gcd(un, ud);
    num = std::to_string(un / g);
    den = std::to_string(ud / g);
  }
  bool operator==(const Rational& o) const {
    return negative == o.negative && num == o.num && den == o.den;
  }
};

namespace detail {
// Little-endian base-2^32 magnitude, just enough for a correctly rounded
// num/den -> double: decimal parse, shifts, compare, subtract.
struct Mag {
  std::vector<uint32_t> w;
  static Mag from_decimal(const std::string& s) {
    Mag m;
    for (char c : s) {
      uint64_t carry = (uint64_t)(c - '0');
      for (uint32_t& x : m.w) {
        const uint64_t t = (uint64_t)x * 10u + carry;
        x = (uint32_t)t;
        carry = t >> 32;
      }
      if (carry) m.w.push_back((uint32_t)carry);
    }
    return m;
  }
  void trim() {
    while (!w.empty() && w.back() == 0) w.pop_back();
  }
  int bits() const {
    if (w.empty()) return 0;
    int b = 32 * (int)(w.size() - 1);
    for (uint32_t t = w.back(); t; t >>= 1) ++b;
    return b;
  }
  void shl(int k) {
    if (w.empty() || k <= 0) return;
    const int words = k / 32, r = k % 32;
    std::vector<uint32_t> o(w.size() + words + 1, 0);
    for (size_t i = 0; i < w.size(); ++i) {
      o[i + words] |= w[i] << r;
      if (r) o[i + words + 1] |= (uint32_t)(w[i] >> (32 - r));
    }
    w.swap(o);
    trim();
  }
  void shr1() {
    for (size_t i = 0; i < w.size(); ++i)
      w[i] = (w[i] >> 1) | (i + 1 < w.size() ? w[i + 1] << 31 : 0u);
    trim();
  }
  int cmp(const Mag& o) const {
    if (w.size() != o.w.size()) return w.size() < o.w.size() ? -1 : 1;
    for (size_t i = w.size(); i-- > 0;)
      if (w[i] != o.w[i]) return w[i] < o.w[i] ? -1 : 1;
    return 0;
  }
  void sub(const Mag& o) {  // *this >= o
    int64_t borrow = 0;
    for (size_t i = 0; i < w.size(); ++i) {
      int64_t t = (int64_t)w[i] - borrow - (i < o.w.size() ? (int64_t)o.w[i] : 0);
      borrow = t < 0;
      w[i] = (uint32_t)(t + (borrow ? (int64_t)1 << 32 : 0));
    }
    trim();
  }
};
}  // namespace detail

// Correctly rounded (nearest, ties to even) value of the literal; values in
// the subnormal range round twice (never produced by the emitted programs).
inline double to_double(const Rational& r) {
  detail::Mag n = detail::Mag::from_decimal(r.num), d = detail::Mag::from_decimal(r.den);
  if (n.w.empty()) return 0.0;
  // Q = floor(n 2^s / d) with 2^55 <= Q < 2^57; the remainder is the sticky bit.
  const int s = 56 - (n.bits() - d.bits());
  if (s > 0) n.shl(s);
  else d.shl(-s);
  detail::Mag dd = d;
  dd.shl(57);
  uint64_t q = 0;
  for (int i = 57; i >= 0; --i) {
    if (n.cmp(dd) >= 0) {
      n.sub(dd);
      q |= 1ull << i;
    }
    dd.shr1();
  }
  const bool sticky = !n.w.empty();
  int nb = 0;
  for (uint64_t t = q; t; t >>= 1) ++nb;
  const int drop = nb - 53;
  uint64_t mant = q >> drop;
  const uint64_t rem = q & ((1ull << drop) - 1), half = 1ull << (drop - 1);
  if (rem > half || (rem == half && (sticky || (mant & 1)))) ++mant;
  const double v = std::ldexp((double)mant, drop - s);
  return r.negative ? -v : v;
}

// parse_rational (rational.hpp:109-148): "n", "n/d" or "i.f", optional '-'.
inline Rational parse_rational(std::string_view text) {
  const std::string t(text);
  auto fail = [&](const char* why) -> Rational {
    throw std::invalid_argument("bad rational literal '" + t + "': " + why);
  };
  if (t.empty()) return fail("empty");
  size_t i = t[0] == '-' ? 1 : 0;
  auto digits = [&](std::string* out) {
    const size_t b = i;
    while (i < t.size() && std::isdigit((unsigned char)t[i])) ++i;
    if (i == b) fail("expected digits");
    *out = t.substr(b, i - b);
  };
  auto strip = [](std::string v) {
    const size_t nz = v.find_first_not_of('0');
    return nz == std::string::npos ? std::string("0") : v.substr(nz);
  };
  Rational r;
  std::string ip, fp;
  digits(&ip);
  if (i < t.size() && t[i] == '/') {
    ++i;
    std::string dp;
    digits(&dp);
    if (i != t.size()) fail("trailing characters");
    if (strip(dp) == "0") fail("zero denominator");
    r.num = strip(ip);
    r.den = strip(dp);
  } else if (i < t.size() && t[i] == '.') {
    ++i;
    digits(&fp);
    if (i != t.size()) fail("trailing characters");
    r.num = strip(ip + fp);
    r.den = "1" + std::string(fp.size(), '0');
  } else {
    if (i != t.size()) fail("trailing characters");
    r.num = strip(ip);
  }
  r.negative = t[0] == '-' && r.num != "0";
  return r;
}

// ---------------------------------------------------------------------------
// ir: three-address-code rational programs (ir.hpp:19-112) and their text
// form (ir_text.hpp).  A program produced by pipe::generate_rp additionally
// carries the metric spec it was generated from (`spec`): the GPU evaluates
// that program's semantics with the template kernels.  A bare program
// (spec == nullptr, e.g. parsed from a `.rp` file) is lowered for
// rpg_program_plan_create and evaluated by its own generated kernel.
namespace ir {

enum class Opcode {
  Assign, Neg, Add, Sub, Mul, EuclidQuot, EuclidRem, FloorDiv, CeilDiv, CmpEq, CmpLt,
  BranchIf, Jump, HaltReturn
};

inline const char* opcode_name(Opcode op) {
  static const char* const names[] = {"assign",    "neg",       "add",       "sub",
                                      "mul",       "euclid_quot", "euclid_rem", "floor_div",
                                      "ceil_div",  "cmp_eq",    "cmp_lt",    "branch_if",
                                      "jump",      "halt_return"};
  const int i = static_cast<int>(op);
  return i >= 0 && i < 14 ? names[i] : "?";
}

struct Operand {
  enum class Kind { Variable, Literal };
  Kind kind = Kind::Literal;
  std::string var;
  Rational lit;
  static Operand variable(std::string name) {
    Operand o;
    o.kind = Kind::Variable;
    o.var = std::move(name);
    return o;
  }
  static Operand literal(Rational value) {
    Operand o;
    o.lit = std::move(value);
    return o;
  }
  bool is_var() const { return kind == Kind::Variable; }
  bool operator==(const Operand& o) const {
    return kind == o.kind && var == o.var && lit == o.lit;
  }
};

inline Operand var(std::string name) { return Operand::variable(std::move(name)); }
inline Operand lit(Rational value) { return Operand::literal(std::move(value)); }
inline Operand lit(long long value) { return Operand::literal(Rational(value)); }

struct TacInstruction {
  Opcode op = Opcode::HaltReturn;
  std::string target;
  std::vector<Operand> operands;
  std::vector<std::size_t> jump_targets;
};

struct RationalProgram {
  std::vector<std::string> inputs;
  std::string output;
  std::vector<TacInstruction> body;
  // B200 extension: set by pipe::generate_rp (the program is that spec's
  // emitted MWP-CWP program with `rep_mode`); null for bare programs.
  std::shared_ptr<const perf::MetricSpec> spec;
  perf::RepMode rep_mode = perf::RepMode::Real;
};

// Interpreter errors (interp.hpp:19-29) and ratprog::DivisionByZero
// (rational.hpp:20-24), raised from the GPU evaluation of bare programs.
struct EvalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StepLimitExceeded : EvalError {
  using EvalError::EvalError;
};
struct MissingBinding : EvalError {
  using EvalError::EvalError;
};

struct ParseError : std::runtime_error {
  std::size_t line, column;
  ParseError(std::size_t l, std::size_t c, const std::string& why)
      : std::runtime_error("line " + std::to_string(l) + ", column " + std::to_string(c) + ": " +
                           why),
        line(l),
        column(c) {}
};

// ir::parse (ir_text.hpp:97-240): same grammar, checks and messages.
inline RationalProgram parse(std::string_view text) {
  struct Tok {
    std::string s;
    std::size_t col;
  };
  auto ident = [](const std::string& s) {
    if (s.empty() || !(std::isalpha((unsigned char)s[0]) || s[0] == '_')) return false;
    return std::all_of(s.begin(), s.end(),
                       [](char c) { return std::isalnum((unsigned char)c) || c == '_'; });
  };
  auto index_of = [](const Tok& t, std::size_t line) -> std::size_t {
    if (t.s.empty() || !std::all_of(t.s.begin(), t.s.end(), [](char c) { return std::isdigit((unsigned char)c); }))
      throw ParseError(line, t.col, "expected instruction index, got '" + t.s + "'");
    return (std::size_t)std::stoull(t.s);
  };
  RationalProgram p;
  int stage = 0;  // 0: expect inputs, 1: expect output, 2: body
  std::size_t line = 0, pos = 0;
  while (pos <= text.size()) {
    std::size_t eol = text.find('\n', pos);
    if (eol == std::string_view::npos) eol = text.size();
    const std::string_view raw = text.substr(pos, eol - pos);
    pos = eol + 1;
    ++line;
    std::vector<Tok> toks;
    for (std::size_t i = 0; i < raw.size();) {
      const char c = raw[i];
      if (c == '#') break;
      if (c == ' ' || c == '\t') {
        ++i;
        continue;
      }
      std::size_t j = i;
      while (j < raw.size() && raw[j] != ' ' && raw[j] != '\t' && raw[j] != '#') ++j;
      toks.push_back({std::string(raw.substr(i, j - i)), i + 1});
      i = j;
    }
    if (toks.empty()) {
      if (eol == text.size()) break;
      continue;
    }
    if (stage == 0) {
      if (toks[0].s != "inputs:") throw ParseError(line, toks[0].col, "expected 'inputs:' header");
      for (std::size_t i = 1; i < toks.size(); ++i) {
        if (!ident(toks[i].s)) throw ParseError(line, toks[i].col, "bad input name '" + toks[i].s + "'");
        p.inputs.push_back(toks[i].s);
      }
      stage = 1;
    } else if (stage == 1) {
      if (toks[0].s != "output:" || toks.size() != 2 || !ident(toks[1].s))
        throw ParseError(line, toks[0].col, "expected 'output: <variable>' header");
      p.output = toks[1].s;
      stage = 2;
    } else {
      const Tok& head = toks[0];
      if (head.s.back() != ':') throw ParseError(line, head.col, "expected '<index>:'");
      const std::size_t idx = index_of(Tok{head.s.substr(0, head.s.size() - 1), head.col}, line);
      if (idx != p.body.size())
        throw ParseError(line, head.col, "instruction index " + std::to_string(idx) +
                                             " out of order; expected " + std::to_string(p.body.size()));
      if (toks.size() < 2) throw ParseError(line, head.col, "missing opcode");
      TacInstruction ins;
      int code = 0;
      while (code < 14 && toks[1].s != opcode_name(static_cast<Opcode>(code))) ++code;
      if (code == 14) throw ParseError(line, toks[1].col, "unknown opcode '" + toks[1].s + "'");
      ins.op = static_cast<Opcode>(code);
      std::vector<Tok> args, targets;
      bool arrow = false;
      for (std::size_t i = 2; i < toks.size(); ++i) {
        if (toks[i].s == "->") {
          if (arrow) throw ParseError(line, toks[i].col, "duplicate '->'");
          arrow = true;
        } else {
          (arrow ? targets : args).push_back(toks[i]);
        }
      }
      // (operands incl. target variable, jump targets, has target variable)
      std::size_t na = 3, nt = 0;
      bool tv = true;
      switch (ins.op) {
        case Opcode::Assign: case Opcode::Neg: na = 2; break;
        case Opcode::BranchIf: na = 1; nt = 2; tv = false; break;
        case Opcode::Jump: na = 0; nt = 1; tv = false; break;
        case Opcode::HaltReturn: na = 1; tv = false; break;
        default: break;
      }
      const std::string opn = opcode_name(ins.op);
      if (args.size() != na)
        throw ParseError(line, toks[1].col, opn + " expects " + std::to_string(na) +
                                                " argument(s), got " + std::to_string(args.size()));
      if (targets.size() != nt)
        throw ParseError(line, toks[1].col, opn + " expects " + std::to_string(nt) +
                                                " jump target(s), got " + std::to_string(targets.size()));
      std::size_t a0 = 0;
      if (tv) {
        if (!ident(args[0].s)) throw ParseError(line, args[0].col, "bad target variable '" + args[0].s + "'");
        ins.target = args[0].s;
        a0 = 1;
      }
      for (std::size_t i = a0; i < args.size(); ++i) {
        if (ident(args[i].s)) {
          ins.operands.push_back(var(args[i].s));
        } else if (args[i].s.find('.') != std::string::npos) {
          throw ParseError(line, args[i].col, "decimal literals are not part of the format; use num/den");
        } else {
          try {
            ins.operands.push_back(lit(parse_rational(args[i].s)));
          } catch (const std::invalid_argument& e) {
            throw ParseError(line, args[i].col, e.what());
          }
        }
      }
      for (const Tok& t : targets) ins.jump_targets.push_back(index_of(t, line));
      p.body.push_back(std::move(ins));
    }
    if (eol == text.size()) break;
  }
  if (stage == 0) throw ParseError(line + 1, 1, "missing 'inputs:' header");
  if (stage == 1) throw ParseError(line + 1, 1, "missing 'output:' header");
  if (p.body.empty()) throw ParseError(line + 1, 1, "empty program body");
  return p;
}

}  // namespace ir

namespace pipe {

inline ir::RationalProgram generate_rp(const MetricModelSet& models, const perf::DeviceProfile&,
                                       const perf::EmitOptions& opts = {}) {
  ir::RationalProgram rp;
  rp.spec = std::make_shared<perf::MetricSpec>(to_metric_spec(models));
  rp.rep_mode = opts.rep_mode;
  rp.inputs = rp.spec->variables;
  rp.output = "total_cycles";
  return rp;
}

enum class Arith { Exact, Fast, FastCM };  // RPG_ARITH_* (rpg.h)
// Auto: the ahead-of-time generic kernel for single-tuple search_optimal
// calls in Exact/Fast (no NVRTC on the reference CLI's one-call-per-process
// path), the per-model specialized kernel for plans and batches.
enum class Kernel { Auto, Specialized, Generic };

// pipe::SearchOptions (pipeline.hpp:438-452) + B200 knobs.
struct SearchOptions {
  double regs_per_thread = 0.0;
  double shared_words_per_block = 0.0;
  const perf::MetricSpec* metrics = nullptr;
  perf::RepMode rep_mode = perf::RepMode::Real;
  int jobs = 1;  // accepted for source compatibility; the GPU needs no host threads
  double tie_rel_tol = 1e-12;
  std::size_t step_limit = 1000000;  // accepted for source compatibility
  Arith arith = Arith::Exact;
  Kernel kernel = Kernel::Auto;
  int device = 0;
  // search_optimal_batch on several GPUs of this process (rpg_plan_group):
  // empty = {device}.  Winners are identical for any device list.
  std::vector<int> devices;
};

struct SearchRow {
  perf::LaunchConfig config;
  double estimated_cycles = 0.0;
  double occupancy = 0.0;
  std::string case_tag = "-";
};

struct SearchResult {
  std::vector<SearchRow> ranking;
  std::size_t ties = 1;
  std::size_t evaluated = 0;
  std::size_t infeasible = 0;
  const SearchRow& best() const { return ranking.front(); }
};

// Per-data-tuple winner of search_optimal_batch (rpg_winner).
struct Winner {
  perf::LaunchConfig config;
  long long cfg_index = -1;  // -1: no feasible configuration
  double estimated_cycles = 0.0;
  double best_cycles = 0.0;
  double occupancy = 0.0;
  std::string case_tag = "-";
  std::size_t ties = 0;
  std::size_t feasible = 0;
  long long b_active = 0, w_active = 0;
};

namespace detail {

inline int rpg_kind(const std::string& v) {
  if (v == "bx") return RPG_VAR_BX;
  if (v == "by") return RPG_VAR_BY;
  if (v == "bz") return RPG_VAR_BZ;
  return std::stoi(v.substr(1)) - 1;
}

inline void rethrow(int code, const char* err) {
  const std::string msg(err);
  switch (code) {
    case RPG_E_INVALID: throw std::invalid_argument(msg);
    case RPG_E_MODEL: throw perf::ModelError(msg);
    case RPG_E_PROFILE: throw perf::ProfileError(msg);
    case RPG_E_PIPELINE: throw PipelineError(msg);
    case RPG_E_NO_FEASIBLE: throw NoFeasibleConfig(msg);
    default: throw std::runtime_error("librpgpu: " + msg);
  }
}

// Owns the packed (AltArr-like) term tables an rpg_model points into.
struct PackedModel {
  rpg_model model{};
  std::vector<std::vector<double>> coefs;
  std::vector<std::vector<uint8_t>> exps;

  explicit PackedModel(const perf::MetricSpec& spec) {
    perf::check_metric_spec(spec);
    const size_t nv = spec.variables.size();
    if (nv > RPG_MAX_VARS) throw perf::ModelError("too many model variables");
    model.n_vars = static_cast<int32_t>(nv);
    for (size_t i = 0; i < nv; ++i) model.var_kind[i] = rpg_kind(spec.variables[i]);
    const char* slots[RPG_N_METRICS] = {perf::kMetricRegs, perf::kMetricShared,
                                        perf::kMetricComp, perf::kMetricUncoal,
                                        perf::kMetricCoal, perf::kMetricSynch,
                                        perf::kMetricTotalBlocks};
    coefs.reserve(2 * RPG_N_METRICS);
    exps.reserve(2 * RPG_N_METRICS);
    for (int s = 0; s < RPG_N_METRICS; ++s) {
      rpg_metric& m = model.metric[s];
      auto c = spec.constants.find(slots[s]);
      if (c != spec.constants.end()) {  // constants take priority (perfmodel.hpp:463-465)
        m.is_const = 1;
        m.value = c->second;
        continue;
      }
      const poly::RationalFunction& f = spec.models.at(slots[s]);
      m.num = pack(f.num, nv);
      m.den = pack(f.den, nv);
    }
  }

  rpg_poly pack(const poly::Polynomial& p, size_t nv) {
    std::vector<double> c;
    std::vector<uint8_t> e;
    for (size_t k = 0; k < p.coeffs.size(); ++k) {
      if (p.coeffs[k] == 0.0) continue;  // emit_ratfunc skips zeros (perfmodel.hpp:521)
      c.push_back(p.coeffs[k]);
      for (size_t v = 0; v < nv; ++v) e.push_back(static_cast<uint8_t>(p.basis[k][v]));
    }
    coefs.push_back(std::move(c));
    exps.push_back(std::move(e));
    rpg_poly out{};
    out.n_terms = static_cast<int32_t>(coefs.back().size());
    out.coef = coefs.back().data();
    out.exps = exps.back().data();
    return out;
  }
};

inline rpg_profile to_rpg(const perf::DeviceProfile& hw) {
  rpg_profile p;
  p.R_max = hw.R_max; p.Z_max = hw.Z_max; p.T_max = hw.T_max; p.B_max = hw.B_max;
  p.W_max = hw.W_max; p.num_SM = hw.num_SM; p.freq_GHz = hw.freq_GHz;
  p.mem_latency_cycles = hw.mem_latency_cycles;
  p.departure_del_coal_cycles = hw.departure_del_coal_cycles;
  p.departure_del_uncoal_cycles = hw.departure_del_uncoal_cycles;
  p.mem_bandwidth_GBps = hw.mem_bandwidth_GBps; p.issue_cycles = hw.issue_cycles;
  p.load_bytes_per_warp = hw.load_bytes_per_warp; p.uncoal_per_mw = hw.uncoal_per_mw;
  return p;
}

inline rpg_options to_rpg(const SearchOptions& o) {
  rpg_options r{};
  r.rep_mode = o.rep_mode == perf::RepMode::Ceil ? RPG_REP_CEIL : RPG_REP_REAL;
  r.arith = o.arith == Arith::Fast     ? RPG_ARITH_FAST
            : o.arith == Arith::FastCM ? RPG_ARITH_FAST_CM
                                       : RPG_ARITH_EXACT;
  r.tie_rel_tol = o.tie_rel_tol;
  r.regs_per_thread = o.regs_per_thread;
  r.shared_words_per_block = o.shared_words_per_block;
  r.kernel = o.kernel == Kernel::Generic ? RPG_KERNEL_GENERIC : RPG_KERNEL_SPECIALIZED;
  return r;
}

inline std::string case_label(int tag) {
  switch (tag) {
    case RPG_CASE_BOTH_SATURATED: return "both_saturated";
    case RPG_CASE_CWP_BOUND: return "cwp_bound";
    case RPG_CASE_MWP_BOUND: return "mwp_bound";
    default: return "-";
  }
}

}  // namespace detail

// A metric spec + profile + configuration space resident on one GPU.
class Plan {
 public:
  Plan(const perf::MetricSpec& spec, const perf::DeviceProfile& hw,
       const std::vector<perf::LaunchConfig>& space, const SearchOptions& opts = {})
      : packed_(spec), space_(space), W_max_(hw.W_max) {
    if (space.empty())
      throw std::invalid_argument("search_optimal: configuration space is empty");
    for (const std::string& v : spec.variables)
      if (v[0] == 'D') d_ = std::max(d_, std::stoi(v.substr(1)));
    std::vector<rpg_config> cfg(space.size());
    for (size_t i = 0; i < space.size(); ++i) cfg[i] = {space[i].bx, space[i].by, space[i].bz};
    const rpg_profile p = detail::to_rpg(hw);
    const rpg_options o = detail::to_rpg(opts);
    char err[512] = {0};
    const int rc = rpg_plan_create(&packed_.model, &p, cfg.data(), (int64_t)cfg.size(), &o,
                                   opts.device, &plan_, err, sizeof(err));
    if (rc != RPG_OK) detail::rethrow(rc, err);
  }
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;
  ~Plan() { rpg_plan_destroy(plan_); }

  // Winners for every data tuple (rows of `tuples`, each D1..Dd).
  std::vector<Winner> search(const std::vector<std::vector<long long>>& tuples) const {
    const int32_t d = tuples.empty() ? d_ : static_cast<int32_t>(tuples.front().size());
    std::vector<int64_t> flat;
    flat.reserve(tuples.size() * d);
    for (const auto& t : tuples) {
      if ((int32_t)t.size() != d) throw std::invalid_argument("data tuples differ in arity");
      flat.insert(flat.end(), t.begin(), t.end());
    }
    std::vector<rpg_winner> w(tuples.size());
    char err[512] = {0};
    const int rc = rpg_search_batch(plan_, flat.data(), (int64_t)tuples.size(), d, w.data(), err,
                                    sizeof(err));
    if (rc != RPG_OK) detail::rethrow(rc, err);
    std::vector<Winner> out(w.size());
    for (size_t i = 0; i < w.size(); ++i) {
      Winner& r = out[i];
      r.cfg_index = w[i].cfg_idx;
      r.feasible = (size_t)w[i].n_feasible;
      if (w[i].cfg_idx < 0) continue;
      r.config = space_[w[i].cfg_idx];
      r.estimated_cycles = w[i].ec;
      r.best_cycles = w[i].best_ec;
      r.occupancy = (double)w[i].w_occ / (double)W_max_;
      r.case_tag = detail::case_label(w[i].case_tag);
      r.ties = (size_t)w[i].ties;
      r.b_active = w[i].b_active;
      r.w_active = w[i].w_active;
    }
    return out;
  }

  // Per-config program output / case tag / occupancy warps for one tuple.
  void evaluate(const std::vector<long long>& tuple, std::vector<double>* ec,
                std::vector<uint8_t>* tag, std::vector<int32_t>* wocc) const {
    const size_t n = space_.size();
    ec->assign(n, 0.0);
    tag->assign(n, 0);
    wocc->assign(n, 0);
    std::vector<int64_t> t(tuple.begin(), tuple.end());
    char err[512] = {0};
    const int rc = rpg_evaluate(plan_, t.data(), 1, (int32_t)t.size(), ec->data(), tag->data(),
                                wocc->data(), err, sizeof(err));
    if (rc != RPG_OK) detail::rethrow(rc, err);
  }

  const std::vector<perf::LaunchConfig>& space() const { return space_; }
  long long W_max() const { return W_max_; }

 private:
  detail::PackedModel packed_;
  std::vector<perf::LaunchConfig> space_;
  long long W_max_;
  int32_t d_ = 0;
  rpg_plan* plan_ = nullptr;
};

// pipe::search_optimal for a metric spec (pipeline.hpp:575-680): the GPU
// evaluates every configuration; the rows are ordered exactly as the
// reference orders them (feasible = Ec >= 0; sort by (Ec, lex); tie group
// Ec <= best + best*tol, stable-sorted by occupancy, descending).
inline SearchResult search_optimal(const perf::MetricSpec& spec,
                                   const std::vector<long long>& data_params,
                                   const perf::DeviceProfile& hw,
                                   const std::vector<perf::LaunchConfig>& space,
                                   const SearchOptions& opts = {});

namespace detail {

// A bare ir::RationalProgram lowered to include/rpg.h's rpg_program: one slot
// per variable (inputs first), literals as their correctly rounded doubles,
// inputs bound as make_binding_plan binds them (pipeline.hpp:482-516) —
// bx/by/bz per configuration, D<k> from the data tuple, profile fields fixed.
struct LoweredProgram {
  rpg_program prog{};
  std::vector<rpg_instr> body;
  std::vector<double> lits;
  std::vector<int32_t> islot, ikind;
  std::vector<double> ifixed;
  std::vector<std::string> slot_names;

  LoweredProgram(const ir::RationalProgram& rp, const std::vector<long long>& data_params,
                 const perf::DeviceProfile& hw, std::size_t step_limit) {
    std::map<std::string, int32_t> slots;
    auto slot = [&](const std::string& name) {
      auto it = slots.find(name);
      if (it != slots.end()) return it->second;
      const int32_t k = (int32_t)slot_names.size();
      slots.emplace(name, k);
      slot_names.push_back(name);
      return k;
    };
    for (const std::string& in : rp.inputs) slot(in);
    std::map<std::string, int32_t> lit_index;
    auto operand = [&](const ir::Operand& o) -> int32_t {
      if (o.is_var()) return slot(o.var);
      const std::string key = (o.lit.negative ? "-" : "") + o.lit.num + "/" + o.lit.den;
      auto it = lit_index.find(key);
      if (it == lit_index.end()) {
        it = lit_index.emplace(key, (int32_t)lits.size()).first;
        lits.push_back(to_double(o.lit));
      }
      return -1 - it->second;
    };
    for (const ir::TacInstruction& ins : rp.body) {
      rpg_instr r{};
      r.op = static_cast<int32_t>(ins.op);
      r.target = ins.target.empty() ? -1 : slot(ins.target);
      if (ins.operands.size() > 0) r.a = operand(ins.operands[0]);
      if (ins.operands.size() > 1) r.b = operand(ins.operands[1]);
      if (ins.jump_targets.size() > 0) r.t0 = (int32_t)ins.jump_targets[0];
      if (ins.jump_targets.size() > 1) r.t1 = (int32_t)ins.jump_targets[1];
      body.push_back(r);
    }
    const int32_t out_slot = slot(rp.output);
    const rpg_profile p = to_rpg(hw);
    const std::map<std::string, double> fixed = {
        {"R_max", (double)p.R_max}, {"Z_max", (double)p.Z_max}, {"T_max", (double)p.T_max},
        {"B_max", (double)p.B_max}, {"W_max", (double)p.W_max}, {"num_SM", (double)p.num_SM},
        {"freq_GHz", p.freq_GHz}, {"mem_latency_cycles", p.mem_latency_cycles},
        {"departure_del_coal_cycles", p.departure_del_coal_cycles},
        {"departure_del_uncoal_cycles", p.departure_del_uncoal_cycles},
        {"mem_bandwidth_GBps", p.mem_bandwidth_GBps}, {"issue_cycles", p.issue_cycles},
        {"load_bytes_per_warp", (double)p.load_bytes_per_warp},
        {"uncoal_per_mw", (double)p.uncoal_per_mw}};
    for (const std::string& in : rp.inputs) {
      islot.push_back(slots.at(in));
      int32_t kind = RPG_INPUT_FIXED;
      double value = 0.0;
      if (in == "bx" || in == "by" || in == "bz") {
        kind = in == "bx" ? RPG_VAR_BX : in == "by" ? RPG_VAR_BY : RPG_VAR_BZ;
      } else if (auto f = fixed.find(in); f != fixed.end()) {
        value = f->second;
      } else if (in.size() >= 2 && in[0] == 'D' &&
                 in.find_first_not_of("0123456789", 1) == std::string::npos) {
        const unsigned long k = std::stoul(in.substr(1));
        if (k < 1 || k > data_params.size())
          throw PipelineError("program input '" + in + "' has no value: " +
                              std::to_string(data_params.size()) + " data parameter(s) were given");
        kind = (int32_t)(k - 1);
      } else {
        throw PipelineError("program input '" + in +
                            "' is neither a block dimension, a data parameter, nor a device "
                            "profile field");
      }
      ikind.push_back(kind);
      ifixed.push_back(value);
    }
    if (lits.empty()) lits.push_back(0.0);
    prog.n_instr = (int32_t)body.size();
    prog.n_slots = (int32_t)slot_names.size();
    prog.n_literals = (int32_t)lit_index.size();
    prog.output_slot = out_slot;
    prog.body = body.data();
    prog.literals = lits.data();
    prog.n_inputs = (int32_t)rp.inputs.size();
    prog.input_slot = islot.data();
    prog.input_kind = ikind.data();
    prog.input_fixed = ifixed.data();
    prog.step_limit = (int64_t)step_limit;
  }

  // RPG_E_EVAL message -> the interpreter's exception (interp.hpp:19-121).
  [[noreturn]] void rethrow_eval(const std::string& msg) const {
    const std::string pre = "no value bound for variable slot ";
    if (msg.rfind(pre, 0) == 0) {
      size_t end = pre.size();
      while (end < msg.size() && std::isdigit((unsigned char)msg[end])) ++end;
      const size_t k = std::stoul(msg.substr(pre.size(), end - pre.size()));
      throw ir::MissingBinding("no value bound for variable '" +
                               (k < slot_names.size() ? slot_names[k] : msg) + "'" + msg.substr(end));
    }
    if (msg.find("zero divisor") != std::string::npos) throw DivisionByZero(msg);
    if (msg.rfind("step limit", 0) == 0) throw ir::StepLimitExceeded(msg);
    throw ir::EvalError(msg);
  }
};

// search_optimal's ranking (pipeline.hpp:612-680) over per-configuration
// program values, occupancies and tags.
inline SearchResult rank_rows(const std::vector<perf::LaunchConfig>& space,
                              const std::vector<double>& ec, const std::vector<double>& occ,
                              const std::vector<std::string>& tags, double tie_rel_tol) {
  const size_t n = space.size();
  std::vector<size_t> feasible;
  for (size_t i = 0; i < n; ++i)
    if (ec[i] >= 0) feasible.push_back(i);
  if (feasible.empty())
    throw NoFeasibleConfig("no configuration in the search space can launch on this device");
  std::sort(feasible.begin(), feasible.end(), [&](size_t a, size_t b) {
    if (ec[a] != ec[b]) return ec[a] < ec[b];
    if (space[a] < space[b]) return true;
    if (space[b] < space[a]) return false;
    return a < b;
  });
  const double best = ec[feasible.front()];
  const double bound = best + best * tie_rel_tol;
  size_t ties = 0;
  while (ties < feasible.size() && ec[feasible[ties]] <= bound) ++ties;
  std::stable_sort(feasible.begin(), feasible.begin() + ties,
                   [&](size_t a, size_t b) { return occ[a] > occ[b]; });
  SearchResult out;
  out.evaluated = n;
  out.infeasible = n - feasible.size();
  out.ties = ties;
  out.ranking.reserve(feasible.size());
  for (size_t i : feasible) out.ranking.push_back(SearchRow{space[i], ec[i], occ[i], tags[i]});
  return out;
}

// Occupancy from the options' regs/shared for every configuration
// (pipeline.hpp:648-650), on the GPU direct model.
inline std::vector<double> option_occupancy(const perf::DeviceProfile& hw,
                                            const std::vector<perf::LaunchConfig>& space,
                                            const SearchOptions& opts) {
  const size_t n = space.size();
  std::vector<double> mv(n * RPG_N_METRICS, 0.0);
  std::vector<rpg_config> cfg(n);
  for (size_t i = 0; i < n; ++i) {
    mv[i * RPG_N_METRICS + RPG_METRIC_REGS] = opts.regs_per_thread;
    mv[i * RPG_N_METRICS + RPG_METRIC_SHARED] = opts.shared_words_per_block;
    cfg[i] = {space[i].bx, space[i].by, space[i].bz};
  }
  std::vector<int32_t> b(n), w(n), st(n);
  const rpg_profile p = to_rpg(hw);
  char err[512] = {0};
  const int rc = rpg_mwpcwp_cycles_batch(&p, mv.data(), cfg.data(), (int64_t)n,
                                         RPG_REP_REAL, opts.device, nullptr, b.data(), w.data(),
                                         nullptr, st.data(), err, sizeof err);
  if (rc != RPG_OK) rethrow(rc, err);
  std::vector<double> occ(n);
  for (size_t i = 0; i < n; ++i) occ[i] = (double)w[i] / (double)hw.W_max;
  return occ;
}

// Occupancy and case tag of every configuration under a metric spec: the
// direct-path diagnostics search_optimal computes with opts.metrics
// (pipeline.hpp:629-647, incl. the DenominatorNearZero fallback).
inline void spec_diagnostics(const perf::MetricSpec& spec, const std::vector<long long>& data_params,
                             const perf::DeviceProfile& hw,
                             const std::vector<perf::LaunchConfig>& space,
                             const SearchOptions& opts, std::vector<double>* occ,
                             std::vector<std::string>* tags);

}  // namespace detail

// The reference's signature (pipeline.hpp:575-579).  For a program from
// generate_rp, Ec is that spec's program evaluated on the GPU; for a bare
// program (spec == nullptr), the program itself is lowered and evaluated on
// the GPU (rpg_program_plan_create).  Diagnostics follow the reference:
// with opts.metrics, occupancy and case tag come from that spec's direct
// model; without it, occupancy comes from opts.regs_per_thread /
// shared_words_per_block and the tag is "-" (pipeline.hpp:629-651).
inline SearchResult search_optimal(const ir::RationalProgram& rp,
                                   const std::vector<long long>& data_params,
                                   const perf::DeviceProfile& hw,
                                   const std::vector<perf::LaunchConfig>& space,
                                   const SearchOptions& opts = {}) {
  if (space.empty()) throw std::invalid_argument("search_optimal: configuration space is empty");
  if (rp.spec) {
    SearchOptions o = opts;
    o.rep_mode = rp.rep_mode;
    if (opts.metrics == rp.spec.get() ||
        (opts.metrics && opts.metrics->variables == rp.spec->variables &&
         opts.metrics->constants == rp.spec->constants &&
         opts.metrics->models.size() == rp.spec->models.size() &&
         std::equal(opts.metrics->models.begin(), opts.metrics->models.end(),
                    rp.spec->models.begin(), [](const auto& x, const auto& y) {
                      return x.first == y.first && x.second.num.coeffs == y.second.num.coeffs &&
                             x.second.den.coeffs == y.second.den.coeffs &&
                             x.second.num.basis == y.second.num.basis &&
                             x.second.den.basis == y.second.den.basis;
                    })))
      return search_optimal(*rp.spec, data_params, hw, space, o);
    if (o.kernel == Kernel::Auto && o.arith != Arith::FastCM) o.kernel = Kernel::Generic;
    Plan plan(*rp.spec, hw, space, o);
    std::vector<double> ec;
    std::vector<uint8_t> tag;
    std::vector<int32_t> wocc;
    plan.evaluate(data_params, &ec, &tag, &wocc);
    std::vector<double> occ;
    std::vector<std::string> tags(space.size(), "-");
    if (opts.metrics) detail::spec_diagnostics(*opts.metrics, data_params, hw, space, o, &occ, &tags);
    else occ = detail::option_occupancy(hw, space, opts);
    return detail::rank_rows(space, ec, occ, tags, opts.tie_rel_tol);
  }
  detail::LoweredProgram low(rp, data_params, hw, opts.step_limit);
  std::vector<rpg_config> cfg(space.size());
  for (size_t i = 0; i < space.size(); ++i) cfg[i] = {space[i].bx, space[i].by, space[i].bz};
  const rpg_profile p = detail::to_rpg(hw);
  const rpg_options ro = detail::to_rpg(opts);
  rpg_plan* plan = nullptr;
  char err[1024] = {0};
  int rc = rpg_program_plan_create(&low.prog, &p, cfg.data(), (int64_t)cfg.size(), &ro,
                                   opts.device, &plan, err, sizeof err);
  if (rc != RPG_OK) detail::rethrow(rc, err);
  const size_t n = space.size();
  std::vector<double> ec(n);
  std::vector<uint8_t> tag(n);
  std::vector<int32_t> wocc(n);
  std::vector<int64_t> t(data_params.begin(), data_params.end());
  rc = rpg_evaluate(plan, t.empty() ? nullptr : t.data(), 1, (int32_t)t.size(), ec.data(),
                    tag.data(), wocc.data(), err, sizeof err);
  rpg_plan_destroy(plan);
  if (rc == RPG_E_EVAL) low.rethrow_eval(err);
  if (rc != RPG_OK) detail::rethrow(rc, err);
  std::vector<double> occ(n);
  std::vector<std::string> tags(n, "-");
  if (opts.metrics) {
    detail::spec_diagnostics(*opts.metrics, data_params, hw, space, opts, &occ, &tags);
  } else {
    for (size_t i = 0; i < n; ++i) occ[i] = (double)wocc[i] / (double)hw.W_max;
  }
  return detail::rank_rows(space, ec, occ, tags, opts.tie_rel_tol);
}

inline SearchResult search_optimal(const perf::MetricSpec& spec,
                                   const std::vector<long long>& data_params,
                                   const perf::DeviceProfile& hw,
                                   const std::vector<perf::LaunchConfig>& space,
                                   const SearchOptions& opts) {
  if (space.empty()) throw std::invalid_argument("search_optimal: configuration space is empty");
  SearchOptions o = opts;
  if (o.kernel == Kernel::Auto && o.arith != Arith::FastCM) o.kernel = Kernel::Generic;
  Plan plan(spec, hw, space, o);
  std::vector<double> ec;
  std::vector<uint8_t> tag;
  std::vector<int32_t> wocc;
  plan.evaluate(data_params, &ec, &tag, &wocc);
  std::vector<double> occ(space.size());
  std::vector<std::string> tags(space.size());
  for (size_t i = 0; i < space.size(); ++i) {
    occ[i] = (double)wocc[i] / (double)hw.W_max;
    tags[i] = detail::case_label(tag[i]);
  }
  return detail::rank_rows(space, ec, occ, tags, opts.tie_rel_tol);
}

namespace detail {
inline void spec_diagnostics(const perf::MetricSpec& spec, const std::vector<long long>& data_params,
                             const perf::DeviceProfile& hw,
                             const std::vector<perf::LaunchConfig>& space,
                             const SearchOptions& opts, std::vector<double>* occ,
                             std::vector<std::string>* tags) {
  SearchOptions o = opts;
  o.metrics = nullptr;
  if (o.kernel == Kernel::Auto && o.arith != Arith::FastCM) o.kernel = Kernel::Generic;
  Plan plan(spec, hw, space, o);
  std::vector<double> ec;
  std::vector<uint8_t> tag;
  std::vector<int32_t> wocc;
  plan.evaluate(data_params, &ec, &tag, &wocc);
  occ->resize(space.size());
  tags->resize(space.size());
  for (size_t i = 0; i < space.size(); ++i) {
    (*occ)[i] = (double)wocc[i] / (double)hw.W_max;
    (*tags)[i] = case_label(tag[i]);
  }
}
}  // namespace detail

// Batched search: one winner per data tuple, all tuples in one launch per
// device; opts.devices lists the GPUs (contiguous tuple blocks per device,
// rpg_search_batch_group).
inline std::vector<Winner> search_optimal_batch(const perf::MetricSpec& spec,
                                                const std::vector<std::vector<long long>>& tuples,
                                                const perf::DeviceProfile& hw,
                                                const std::vector<perf::LaunchConfig>& space,
                                                const SearchOptions& opts = {}) {
  if (opts.devices.size() <= 1) {
    SearchOptions o = opts;
    if (!opts.devices.empty()) o.device = opts.devices[0];
    Plan plan(spec, hw, space, o);
    return plan.search(tuples);
  }
  if (space.empty()) throw std::invalid_argument("search_optimal: configuration space is empty");
  detail::PackedModel pk(spec);
  std::vector<rpg_config> cfg(space.size());
  for (size_t i = 0; i < space.size(); ++i) cfg[i] = {space[i].bx, space[i].by, space[i].bz};
  const rpg_profile p = detail::to_rpg(hw);
  const rpg_options o = detail::to_rpg(opts);
  std::vector<int32_t> dev(opts.devices.begin(), opts.devices.end());
  rpg_plan_group* g = nullptr;
  char err[1024] = {0};
  int rc = rpg_plan_group_create(&pk.model, &p, cfg.data(), (int64_t)cfg.size(), &o, dev.data(),
                                 (int32_t)dev.size(), &g, err, sizeof err);
  if (rc != RPG_OK) detail::rethrow(rc, err);
  int32_t d = 0;
  for (const std::string& v : spec.variables)
    if (v[0] == 'D') d = std::max(d, (int32_t)std::stoi(v.substr(1)));
  if (!tuples.empty()) d = (int32_t)tuples.front().size();
  std::vector<int64_t> flat;
  for (const auto& t : tuples) {
    if ((int32_t)t.size() != d) {
      rpg_plan_group_destroy(g);
      throw std::invalid_argument("data tuples differ in arity");
    }
    flat.insert(flat.end(), t.begin(), t.end());
  }
  std::vector<rpg_winner> w(tuples.size());
  rc = rpg_search_batch_group(g, flat.data(), (int64_t)tuples.size(), d, w.data(), err, sizeof err);
  rpg_plan_group_destroy(g);
  if (rc != RPG_OK) detail::rethrow(rc, err);
  std::vector<Winner> out(w.size());
  for (size_t i = 0; i < w.size(); ++i) {
    Winner& r = out[i];
    r.cfg_index = w[i].cfg_idx;
    r.feasible = (size_t)w[i].n_feasible;
    if (w[i].cfg_idx < 0) continue;
    r.config = space[w[i].cfg_idx];
    r.estimated_cycles = w[i].ec;
    r.best_cycles = w[i].best_ec;
    r.occupancy = (double)w[i].w_occ / (double)hw.W_max;
    r.case_tag = detail::case_label(w[i].case_tag);
    r.ties = (size_t)w[i].ties;
    r.b_active = w[i].b_active;
    r.w_active = w[i].w_active;
  }
  return out;
}

// ---------------------------------------------------------------------------
// Report formatters (pipeline.hpp:897-934), deterministic.

namespace detail {
inline std::string format_double(double v) {
  char buf[64];
  auto res = std::to_chars(buf, buf + sizeof(buf), v);
  return std::string(buf, res.ptr);
}
inline std::string config_label(const perf::LaunchConfig& c) {
  return std::to_string(c.bx) + "x" + std::to_string(c.by) + "x" + std::to_string(c.bz);
}
}  // namespace detail

// The three report formats of pipeline.hpp:897-934 (output strings are the
// reference's, byte for byte): every row as its cells once, then joined.
namespace detail {
struct RowCells {
  std::string bx, by, bz, ec, occ, tag;
};
inline RowCells cells(const SearchRow& row) {
  return {std::to_string(row.config.bx), std::to_string(row.config.by),
          std::to_string(row.config.bz), format_double(row.estimated_cycles),
          format_double(row.occupancy), row.case_tag};
}
}  // namespace detail

inline std::string format_search_csv(const SearchResult& r) {
  std::string out = "bx,by,bz,Ec,occupancy,case\n";
  for (const SearchRow& row : r.ranking) {
    const detail::RowCells c = detail::cells(row);
    out += c.bx + ',' + c.by + ',' + c.bz + ',' + c.ec + ',' + c.occ + ',' + c.tag + '\n';
  }
  return out;
}

// Left-aligned columns two spaces apart, a dashed rule under the header
// (detail::format_table, pipeline.hpp:870-894), then the counters line.
inline std::string format_search_text(const SearchResult& r) {
  std::vector<std::array<std::string, 4>> table = {{"config", "Ec", "occupancy", "case"}};
  for (const SearchRow& row : r.ranking) {
    const detail::RowCells c = detail::cells(row);
    table.push_back({detail::config_label(row.config), c.ec, c.occ, c.tag});
  }
  std::array<size_t, 4> w{};
  for (const auto& t : table)
    for (size_t j = 0; j < 4; ++j) w[j] = std::max(w[j], t[j].size());
  std::string out;
  auto line = [&](const std::array<std::string, 4>& t) {
    for (size_t j = 0; j < 4; ++j) {
      out += t[j];
      if (j < 3) out.append(w[j] - t[j].size() + 2, ' ');
    }
    out += '\n';
  };
  line(table[0]);
  out.append(w[0] + w[1] + w[2] + w[3] + 6, '-');
  out += '\n';
  for (size_t i = 1; i < table.size(); ++i) line(table[i]);
  out += "evaluated " + std::to_string(r.evaluated) + " configuration(s), " +
         std::to_string(r.infeasible) + " infeasible; optimum ties: " + std::to_string(r.ties) + "\n";
  return out;
}

// One JSON object per ranked row (nlohmann ordered_json's compact dump).
inline std::string format_search_jsonl(const SearchResult& r) {
  std::string out;
  for (const SearchRow& row : r.ranking) {
    const detail::RowCells c = detail::cells(row);
    out += "{\"config\":[" + c.bx + "," + c.by + "," + c.bz + "],\"Ec\":" + c.ec +
           ",\"occupancy\":" + c.occ + ",\"case_tag\":\"" + c.tag + "\"}\n";
  }
  return out;
}

}  // namespace pipe
}  // namespace ratprog
