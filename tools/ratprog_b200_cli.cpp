// ratprog-b200 — the reference CLI's hot-path subcommand (`search`,
// ratprog_cli.cpp:277-332) on the B200 evaluator, plus `sweep`, the batched
// form (one winner per data size over a whole N range in one launch).
//
//   ratprog-b200 search (--models M | --rp PROGRAM) --profile P --size N [--size N2 ...]
//       [--format text|csv|json] [-o FILE] [--dump-jsonl FILE]
//       [--rep-mode real|ceil] [--regs-per-thread R] [--shared-words Z]
//       [--max-threads T] [--min-threads T] [--dims 1|2|3] [--jobs J]
//       [--arith exact|fast|fastcm] [--kernel auto|specialized|generic]
//   ratprog-b200 sweep --models M --profile P --from LO --to HI
//       [--space pow2|dense] [--dims 2|3] [-o FILE] [--arith ...]
//
// Exit codes as the reference: 0 ok, 1 usage error, 2 runtime error.
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "ratprog_b200/ratprog.hpp"

using namespace ratprog;

namespace {

int usage_error(const std::string& message) {
  std::cerr << "usage error: " << message << "\n";
  return 1;
}

void write_output(const std::string& path, const std::string& content) {
  if (path == "-") {
    std::cout << content;
    return;
  }
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open '" + path + "' for writing");
  out << content;
  out.flush();
  if (!out) throw std::runtime_error("failed writing '" + path + "'");
}

struct Args {
  std::string cmd, models, rp, profile, output = "-", dump_jsonl, format = "text",
                               rep_mode = "real", arith = "exact", kernel = "auto",
                               space = "pow2";
  std::vector<long long> sizes;
  long long lo = 0, hi = -1, max_threads = 1024, min_threads = 32;
  int dims = 2, jobs = 1;
  double regs = 0.0, shared = 0.0;
};

pipe::SearchOptions options(const Args& a) {
  pipe::SearchOptions o;
  o.jobs = a.jobs;
  if (a.rep_mode == "ceil") o.rep_mode = perf::RepMode::Ceil;
  else if (a.rep_mode != "real") throw std::runtime_error("--rep-mode must be 'real' or 'ceil'");
  o.regs_per_thread = a.regs;
  o.shared_words_per_block = a.shared;
  o.arith = a.arith == "fast"     ? pipe::Arith::Fast
            : a.arith == "fastcm" ? pipe::Arith::FastCM
                                  : pipe::Arith::Exact;
  if (a.kernel != "auto" && a.kernel != "generic" && a.kernel != "specialized")
    throw std::runtime_error("--kernel must be 'auto', 'specialized' or 'generic'");
  o.kernel = a.kernel == "generic"       ? pipe::Kernel::Generic
             : a.kernel == "specialized" ? pipe::Kernel::Specialized
                                         : pipe::Kernel::Auto;
  return o;
}

int do_search(const Args& a) {
  if (a.profile.empty()) return usage_error("--profile is required (or set RATPROG_PROFILE)");
  if (a.models.empty() == a.rp.empty())
    return usage_error("exactly one of --models or --rp must be given");
  if (a.sizes.empty()) return usage_error("--size is required");
  if (a.format != "text" && a.format != "csv" && a.format != "json")
    return usage_error("--format must be text, csv, or json");
  perf::DeviceProfile hw = perf::load_profile(a.profile);
  auto space = data::enumerate_configs(a.max_threads, a.min_threads, a.dims);
  pipe::SearchOptions opts = options(a);
  ir::RationalProgram rp;
  perf::MetricSpec spec;
  if (!a.models.empty()) {
    pipe::MetricModelSet models = pipe::read_models(a.models);
    spec = pipe::to_metric_spec(models);
    perf::EmitOptions emit;
    emit.rep_mode = opts.rep_mode;
    rp = pipe::generate_rp(models, hw, emit);
    opts.metrics = &spec;
  } else {
    // bare program (`--rp`, ratprog_cli.cpp:104-110, 305-307), lowered and
    // evaluated on the GPU
    std::ifstream in(a.rp, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open '" + a.rp + "'");
    std::stringstream text;
    text << in.rdbuf();
    try {
      rp = ir::parse(text.str());
    } catch (const ir::ParseError& e) {
      throw std::runtime_error(a.rp + ": " + e.what());
    }
  }
  pipe::SearchResult found = pipe::search_optimal(rp, a.sizes, hw, space, opts);
  std::string report = a.format == "csv"    ? pipe::format_search_csv(found)
                       : a.format == "json" ? pipe::format_search_jsonl(found)
                                            : pipe::format_search_text(found);
  write_output(a.output, report);
  if (!a.dump_jsonl.empty()) write_output(a.dump_jsonl, pipe::format_search_jsonl(found));
  const pipe::SearchRow& best = found.best();
  std::cerr << "chosen " << best.config.bx << "x" << best.config.by << "x" << best.config.bz
            << "  Ec=" << pipe::detail::format_double(best.estimated_cycles)
            << "  occupancy=" << pipe::detail::format_double(best.occupancy)
            << "  ties=" << found.ties << "\n";
  return 0;
}

int do_sweep(const Args& a) {
  if (a.profile.empty()) return usage_error("--profile is required (or set RATPROG_PROFILE)");
  if (a.models.empty()) return usage_error("--models is required");
  if (a.hi < a.lo || a.lo < 1) return usage_error("--from/--to must give 1 <= LO <= HI");
  perf::DeviceProfile hw = perf::load_profile(a.profile);
  auto space = a.space == "dense" ? data::integer_configs(a.max_threads, a.dims)
                                  : data::enumerate_configs(a.max_threads, a.min_threads, a.dims);
  perf::MetricSpec spec = pipe::to_metric_spec(pipe::read_models(a.models));
  std::vector<std::vector<long long>> tuples;
  for (long long n = a.lo; n <= a.hi; ++n) tuples.push_back({n});
  pipe::Plan plan(spec, hw, space, options(a));
  std::vector<pipe::Winner> w = plan.search(tuples);
  std::string out = "D1,bx,by,bz,Ec,occupancy,case,ties,feasible\n";
  for (size_t i = 0; i < w.size(); ++i) {
    out += std::to_string(tuples[i][0]) + ",";
    if (w[i].cfg_index < 0) {
      out += ",,,,,,0,0\n";
      continue;
    }
    out += std::to_string(w[i].config.bx) + "," + std::to_string(w[i].config.by) + "," +
           std::to_string(w[i].config.bz) + "," + pipe::detail::format_double(w[i].estimated_cycles) +
           "," + pipe::detail::format_double(w[i].occupancy) + "," + w[i].case_tag + "," +
           std::to_string(w[i].ties) + "," + std::to_string(w[i].feasible) + "\n";
  }
  write_output(a.output, out);
  std::cerr << "swept " << w.size() << " data size(s) x " << space.size() << " configuration(s)\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  Args a;
  if (const char* p = std::getenv("RATPROG_PROFILE")) a.profile = p;
  if (argc < 2) return usage_error("no subcommand given (search | sweep)");
  a.cmd = argv[1];
  try {
    for (int i = 2; i < argc; ++i) {
      const std::string k = argv[i];
      auto val = [&]() -> std::string {
        if (i + 1 >= argc) throw std::invalid_argument(k + " needs a value");
        return argv[++i];
      };
      if (k == "--models") a.models = val();
      else if (k == "--rp") a.rp = val();
      else if (k == "--profile") a.profile = val();
      else if (k == "--size") a.sizes.push_back(std::stoll(val()));
      else if (k == "-o" || k == "--output") a.output = val();
      else if (k == "--dump-jsonl") a.dump_jsonl = val();
      else if (k == "--format") a.format = val();
      else if (k == "--rep-mode") a.rep_mode = val();
      else if (k == "--regs-per-thread") a.regs = std::stod(val());
      else if (k == "--shared-words") a.shared = std::stod(val());
      else if (k == "--max-threads") a.max_threads = std::stoll(val());
      else if (k == "--min-threads") a.min_threads = std::stoll(val());
      else if (k == "--dims") a.dims = std::stoi(val());
      else if (k == "--jobs") a.jobs = std::stoi(val());
      else if (k == "--arith") a.arith = val();
      else if (k == "--kernel") a.kernel = val();
      else if (k == "--from") a.lo = std::stoll(val());
      else if (k == "--to") a.hi = std::stoll(val());
      else if (k == "--space") a.space = val();
      else return usage_error("unknown option " + k);
    }
  } catch (const std::exception& e) {
    return usage_error(e.what());
  }
  try {
    if (a.cmd == "search") return do_search(a);
    if (a.cmd == "sweep") return do_sweep(a);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
  return usage_error("unknown subcommand '" + a.cmd + "'");
}
