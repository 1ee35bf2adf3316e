// rpg_multi.cu — several GPUs behind one drop-in call (include/rpg.h
// rpg_plan_group_*): the reference parallelises search_optimal inside the
// call with std::threads over static slices (pipeline.hpp:595-614); here the
// slices are GPUs of one process.
//
//   tuple axis (n_tuples >= n_devices): device g searches the contiguous
//     block [n g / G, n (g+1) / G) of the data tuples (the reference's
//     partition, pipeline.hpp:602) with its own plan; every winner record
//     is computed by one device exactly as a single-device call computes it,
//     so the output is byte-identical for any device count;
//   configuration axis (n_tuples < n_devices, SURVEY.md 8(e) fallback):
//     device g owns the contiguous slice [S g / G, S (g+1) / G) of the
//     configuration space.  Phase 1 evaluates every (tuple, config) point of
//     the slice (rpg_evaluate; the same point evaluator and bits as the
//     search); the host takes the global minimum Ec per tuple and the tie
//     group Ec <= best + best tol (pipeline.hpp:660-665).  Phase 2 ranks
//     each device's members of the group on that device
//     (rpg_search_batch_subsets: all of them are inside the device's own tie
//     bound, since its local best >= the global best), and the host merges
//     the per-device winners with the reference's key — higher occupancy,
//     then lower Ec, then lex (bx, by, bz) (pipeline.hpp:654-669) — and sums
//     the tie and feasible counts.  Byte-identical to the single-device
//     record.  FAST_CM plans have no subset search: with fewer tuples than
//     devices they run on the first device alone.
// Devices may repeat in the list (several plans on one GPU): the host logic
// is then exercised on a one-GPU machine.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "rpg.h"

namespace {

int merr(char* err, size_t errlen, int code, const char* fmt, ...) {
  if (err && errlen) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, errlen, fmt, ap);
    va_end(ap);
  }
  return code;
}

}  // namespace

struct rpg_plan_group {
  rpg_model model{};
  bool is_model = true;
  rpg_profile hw{};
  rpg_options opts{};
  std::vector<rpg_config> space;
  std::vector<int32_t> lex;           // global lex rank of every configuration
  std::vector<int32_t> devices;
  std::vector<rpg_plan*> full;        // full-space plan per device (tuple axis)
  std::vector<rpg_plan*> slice;       // slice plans (configuration axis), lazy
  std::vector<int64_t> slice_lo;      // G + 1 slice bounds
  // Owned copies of the model's term arrays (the slice plans are built
  // lazily, after the caller's buffers may be gone).
  std::vector<std::vector<double>> coefs;
  std::vector<std::vector<uint8_t>> exps;
  std::mutex mu;
};

namespace {

// Runs f(g) for every device on its own host thread; returns the first
// (lowest-device-index) error.
template <class F>
int for_devices(int G, char* err, size_t errlen, F f) {
  std::vector<int> rc(G, RPG_OK);
  std::vector<std::string> msg(G);
  std::vector<std::thread> th;
  for (int g = 0; g < G; ++g)
    th.emplace_back([&, g] {
      char e[1024] = {0};
      rc[g] = f(g, e, sizeof e);
      msg[g] = e;
    });
  for (auto& t : th) t.join();
  for (int g = 0; g < G; ++g)
    if (rc[g] != RPG_OK) return merr(err, errlen, rc[g], "%s", msg[g].c_str());
  return RPG_OK;
}

int ensure_slices(rpg_plan_group* pg, char* err, size_t errlen) {
  if (!pg->slice.empty()) return RPG_OK;
  const int G = (int)pg->devices.size();
  const int64_t S = (int64_t)pg->space.size();
  pg->slice_lo.resize(G + 1);
  for (int g = 0; g <= G; ++g) pg->slice_lo[g] = S * g / G;
  std::vector<rpg_plan*> plans(G, nullptr);
  int rc = for_devices(G, err, errlen, [&](int g, char* e, size_t el) -> int {
    const int64_t lo = pg->slice_lo[g], hi = pg->slice_lo[g + 1];
    if (hi <= lo) return RPG_OK;
    return rpg_plan_create(&pg->model, &pg->hw, pg->space.data() + lo, hi - lo, &pg->opts,
                           pg->devices[g], &plans[g], e, el);
  });
  if (rc != RPG_OK) {
    for (rpg_plan* p : plans)
      if (p) rpg_plan_destroy(p);
    return rc;
  }
  pg->slice = plans;
  return RPG_OK;
}

int search_config_axis(rpg_plan_group* pg, const int64_t* data, int64_t n, int32_t d,
                       rpg_winner* out, char* err, size_t errlen) {
  int rc = ensure_slices(pg, err, errlen);
  if (rc != RPG_OK) return rc;
  const int G = (int)pg->devices.size();
  const double tol = pg->opts.tie_rel_tol;
  // Phase 1: every point of every slice.
  std::vector<std::vector<double>> ec(G);
  rc = for_devices(G, err, errlen, [&](int g, char* e, size_t el) -> int {
    const int64_t w = pg->slice_lo[g + 1] - pg->slice_lo[g];
    if (w <= 0) return RPG_OK;
    ec[g].resize((size_t)(n * w));
    return rpg_evaluate(pg->slice[g], data, n, d, ec[g].data(), nullptr, nullptr, e, el);
  });
  if (rc != RPG_OK) return rc;
  // Host: global best, feasible count and the tie-group members per device.
  std::vector<double> best(n, INFINITY);
  std::vector<int32_t> nfeas(n, 0);
  std::vector<char> empty(n, 0);
  for (int g = 0; g < G; ++g) {
    const int64_t w = pg->slice_lo[g + 1] - pg->slice_lo[g];
    for (int64_t t = 0; t < n; ++t)
      for (int64_t c = 0; c < w; ++c) {
        const double v = ec[g][t * w + c];
        if (v >= 0.0) {
          ++nfeas[t];
          if (v < best[t]) best[t] = v;
        }
      }
  }
  std::vector<std::vector<int64_t>> off(G, std::vector<int64_t>(n + 1, 0));
  std::vector<std::vector<int32_t>> list(G);
  for (int64_t t = 0; t < n; ++t) {
    const double bound = best[t] + best[t] * tol;  // pipeline.hpp:661 (TieRule)
    empty[t] = !(bound == bound);
    for (int g = 0; g < G; ++g) {
      const int64_t w = pg->slice_lo[g + 1] - pg->slice_lo[g];
      for (int64_t c = 0; c < w && nfeas[t] > 0; ++c) {
        const double v = ec[g][t * w + c];
        if (v >= 0.0 && (empty[t] ? v == best[t] : v <= bound)) list[g].push_back((int32_t)c);
      }
      off[g][t + 1] = (int64_t)list[g].size();
    }
  }
  // Phase 2: rank each device's members on that device.
  std::vector<std::vector<rpg_winner>> part(G, std::vector<rpg_winner>(n));
  rc = for_devices(G, err, errlen, [&](int g, char* e, size_t el) -> int {
    if (list[g].empty()) {
      for (auto& r : part[g]) r.cfg_idx = -1;
      return RPG_OK;
    }
    return rpg_search_batch_subsets(pg->slice[g], data, n, d, off[g].data(), list[g].data(),
                                    part[g].data(), e, el);
  });
  if (rc != RPG_OK) return rc;
  // Merge with the device kernels' key (rpg_kernels.cuh key_better).
  for (int64_t t = 0; t < n; ++t) {
    rpg_winner r{};
    if (nfeas[t] == 0) {
      r.cfg_idx = -1;
      r.case_tag = RPG_CASE_UNKNOWN;
      out[t] = r;
      continue;
    }
    int wg = -1;
    int64_t wi = -1;
    int32_t ties = 0;
    for (int g = 0; g < G; ++g) {
      const rpg_winner& c = part[g][t];
      if (c.cfg_idx < 0) continue;
      ties += (int32_t)(off[g][t + 1] - off[g][t]);
      const int64_t gi = pg->slice_lo[g] + c.cfg_idx;
      if (wg < 0) {
        wg = g;
        wi = gi;
        continue;
      }
      const rpg_winner& b = part[wg][t];
      const int ow_c = empty[t] ? 0 : c.w_occ, ow_b = empty[t] ? 0 : b.w_occ;
      bool better;
      if (ow_c != ow_b) better = ow_c > ow_b;
      else if (c.ec != b.ec) better = c.ec < b.ec;
      else if (pg->lex[gi] != pg->lex[wi]) better = pg->lex[gi] < pg->lex[wi];
      else better = gi < wi;
      if (better) {
        wg = g;
        wi = gi;
      }
    }
    r = part[wg][t];
    r.cfg_idx = (int32_t)wi;
    r.best_ec = best[t];
    r.ties = empty[t] ? 0 : ties;
    r.n_feasible = nfeas[t];
    r.reserved = 0;
    out[t] = r;
  }
  return RPG_OK;
}

}  // namespace

extern "C" {

int rpg_plan_group_create(const rpg_model* model, const rpg_profile* hw, const rpg_config* space,
                          int64_t n_space, const rpg_options* opts, const int32_t* devices,
                          int32_t n_devices, rpg_plan_group** out, char* err, size_t errlen) {
  if (!model || !hw || !opts || !out || (n_space > 0 && !space) || !devices)
    return merr(err, errlen, RPG_E_INVALID, "rpg_plan_group_create: null argument");
  if (n_devices < 1) return merr(err, errlen, RPG_E_INVALID, "rpg_plan_group_create: no device");
  *out = nullptr;
  rpg_plan_group* pg = new rpg_plan_group();
  pg->model = *model;
  if (model->n_vars < 1 || model->n_vars > RPG_MAX_VARS) {
    delete pg;
    return merr(err, errlen, RPG_E_MODEL, "model: n_vars must be in [1, %d]", RPG_MAX_VARS);
  }
  for (int s = 0; s < RPG_N_METRICS; ++s) {
    rpg_metric& mt = pg->model.metric[s];
    if (mt.is_const) continue;
    for (rpg_poly* p : {&mt.num, &mt.den}) {
      const size_t nt = (size_t)std::max(p->n_terms, 0);
      pg->coefs.emplace_back(p->coef ? p->coef : nullptr, p->coef ? p->coef + nt : nullptr);
      pg->exps.emplace_back(p->exps ? p->exps : nullptr,
                            p->exps ? p->exps + nt * (size_t)model->n_vars : nullptr);
      p->coef = pg->coefs.back().data();
      p->exps = pg->exps.back().data();
    }
  }
  pg->hw = *hw;
  pg->opts = *opts;
  pg->space.assign(space, space + std::max<int64_t>(n_space, 0));
  pg->devices.assign(devices, devices + n_devices);
  std::vector<int32_t> order(pg->space.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    const rpg_config &x = pg->space[a], &y = pg->space[b];
    if (x.bx != y.bx) return x.bx < y.bx;
    if (x.by != y.by) return x.by < y.by;
    return x.bz < y.bz;
  });
  pg->lex.resize(order.size());
  for (size_t r = 0; r < order.size(); ++r) pg->lex[order[r]] = (int32_t)r;
  pg->full.assign(n_devices, nullptr);
  // The first plan validates the arguments (and compiles the specialized
  // module once: the others hit the module cache).
  int rc = rpg_plan_create(model, hw, space, n_space, opts, devices[0], &pg->full[0], err, errlen);
  if (rc == RPG_OK && n_devices > 1)
    rc = for_devices(n_devices - 1, err, errlen, [&](int g, char* e, size_t el) -> int {
      return rpg_plan_create(model, hw, space, n_space, opts, devices[g + 1], &pg->full[g + 1], e,
                             el);
    });
  if (rc != RPG_OK) {
    rpg_plan_group_destroy(pg);
    return rc;
  }
  *out = pg;
  return RPG_OK;
}

int rpg_plan_group_destroy(rpg_plan_group* pg) {
  if (!pg) return RPG_OK;
  for (rpg_plan* p : pg->full)
    if (p) rpg_plan_destroy(p);
  for (rpg_plan* p : pg->slice)
    if (p) rpg_plan_destroy(p);
  delete pg;
  return RPG_OK;
}

int rpg_search_batch_group(rpg_plan_group* pg, const int64_t* data, int64_t n_tuples, int32_t d,
                           rpg_winner* out, char* err, size_t errlen) {
  if (!pg || (n_tuples > 0 && (!out || (d > 0 && !data))))
    return merr(err, errlen, RPG_E_INVALID, "rpg_search_batch_group: null argument");
  if (n_tuples <= 0) return RPG_OK;
  std::lock_guard<std::mutex> lock(pg->mu);
  const int G = (int)pg->devices.size();
  if (G == 1 || (n_tuples < G && pg->opts.arith == RPG_ARITH_FAST_CM))
    return rpg_search_batch(pg->full[0], data, n_tuples, d, out, err, errlen);
  if (n_tuples < G) return search_config_axis(pg, data, n_tuples, d, out, err, errlen);
  return for_devices(G, err, errlen, [&](int g, char* e, size_t el) -> int {
    const int64_t lo = n_tuples * g / G, hi = n_tuples * (g + 1) / G;
    if (hi <= lo) return RPG_OK;
    return rpg_search_batch(pg->full[g], data + lo * d, hi - lo, d, out + lo, e, el);
  });
}

int32_t rpg_plan_group_size(const rpg_plan_group* pg) { return pg ? (int32_t)pg->devices.size() : 0; }

}  // extern "C"
