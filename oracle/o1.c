/*
 * o1.c — ORACLE O1: CPU restatement of the reference's FP64 evaluation path.
 * TEST INFRASTRUCTURE ONLY: linked by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs; never by the product.
 * See o1.h for the function-by-function reference map.
 *
 * Build (oracle/Makefile): cc -O2 -ffp-contract=off -fPIC -shared -pthread.
 */
#include "o1.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Polynomials — polyfit.hpp:96-130.                                         */

/* detail::eval_monomial (polyfit.hpp:96-105): per variable p = x*x*...*x
 * starting from 1.0, then m *= p, in variable order. */
double o1_eval_monomial(const uint8_t* exps, const double* x, int32_t n_vars) {
  double m = 1.0;
  for (int32_t i = 0; i < n_vars; ++i) {
    double p = 1.0;
    for (int e = 0; e < exps[i]; ++e) p *= x[i];
    m *= p;
  }
  return m;
}

/* eval_poly (polyfit.hpp:109-119): acc += c_k * m_k in basis order. */
double o1_eval_poly(const rpg_poly* p, int32_t n_vars, const double* x) {
  double acc = 0.0;
  for (int32_t k = 0; k < p->n_terms; ++k)
    acc += p->coef[k] * o1_eval_monomial(p->exps + (size_t)k * n_vars, x, n_vars);
  return acc;
}

/* eval_ratfunc (polyfit.hpp:121-130): DenominatorNearZero when
 * |q| < 1e-12 * max(1, |p|). */
int o1_eval_ratfunc(const rpg_poly* num, const rpg_poly* den, int32_t n_vars,
                    const double* x, double* out) {
  double pnum = o1_eval_poly(num, n_vars, x);
  double pden = o1_eval_poly(den, n_vars, x);
  double mag = fabs(pnum);
  if (fabs(pden) < 1e-12 * (mag > 1.0 ? mag : 1.0)) return O1_DEN_NEAR_ZERO;
  *out = pnum / pden;
  return O1_OK;
}

/* ------------------------------------------------------------------------ */
/* FAST twin of the polynomial evaluation (GPU RPG_ARITH_FAST).              */
/*                                                                          */
/* For a polynomial over variables with kinds var_kind[], the terms are     */
/* grouped by their block-dimension exponent pattern.  Per pattern the data */
/* part is collapsed in basis order with fma: C = fma(c_k, mD_k, C), where  */
/* mD_k is the eval_monomial product over the data variables only.  The     */
/* block part is then a nested Horner over the block variables in model    */
/* order (first block variable outermost), every step an fma.               */

#define O1_MAXDEG 8

static double fast_poly(const rpg_model* model, const rpg_poly* p,
                        const double* x) {
  const int32_t nv = model->n_vars;
  int cfg_vars[3];
  int ncfg = 0;
  for (int v = 0; v < nv; ++v)
    if (model->var_kind[v] < 0) cfg_vars[ncfg++] = v;
  int maxd[3] = {0, 0, 0};
  for (int32_t k = 0; k < p->n_terms; ++k)
    for (int j = 0; j < ncfg; ++j) {
      int e = p->exps[(size_t)k * nv + cfg_vars[j]];
      if (e > maxd[j]) maxd[j] = e;
    }
  /* C[a][b][c] with strides over (maxd+1). */
  int s0 = maxd[0] + 1, s1 = ncfg > 1 ? maxd[1] + 1 : 1,
      s2 = ncfg > 2 ? maxd[2] + 1 : 1;
  double C[(O1_MAXDEG + 1) * (O1_MAXDEG + 1) * (O1_MAXDEG + 1)];
  for (int i = 0; i < s0 * s1 * s2; ++i) C[i] = 0.0;
  for (int32_t k = 0; k < p->n_terms; ++k) {
    const uint8_t* ex = p->exps + (size_t)k * nv;
    double mD = 1.0;
    for (int v = 0; v < nv; ++v) {
      if (model->var_kind[v] < 0) continue;
      double pw = 1.0;
      for (int e = 0; e < ex[v]; ++e) pw *= x[v];
      mD *= pw;
    }
    int a = ex[cfg_vars[0]];
    int b = ncfg > 1 ? ex[cfg_vars[1]] : 0;
    int c = ncfg > 2 ? ex[cfg_vars[2]] : 0;
    double* slot = &C[(a * s1 + b) * s2 + c];
    *slot = fma(p->coef[k], mD, *slot);
  }
  double xv0 = x[cfg_vars[0]];
  double xv1 = ncfg > 1 ? x[cfg_vars[1]] : 0.0;
  double xv2 = ncfg > 2 ? x[cfg_vars[2]] : 0.0;
  double outer = 0.0;
  for (int a = s0 - 1; a >= 0; --a) {
    double mid = 0.0;
    for (int b = s1 - 1; b >= 0; --b) {
      double inner = C[(a * s1 + b) * s2 + (s2 - 1)];
      for (int c = s2 - 2; c >= 0; --c)
        inner = fma(inner, xv2, C[(a * s1 + b) * s2 + c]);
      mid = (b == s1 - 1) ? inner : fma(mid, xv1, inner);
    }
    outer = (a == s0 - 1) ? mid : fma(outer, xv0, mid);
  }
  return outer;
}

/* FAST_CM twin (GPU RPG_ARITH_FAST_CM): the same two steps with the roles  */
/* swapped.  Per data-exponent pattern the block-dimension part is          */
/* collapsed in basis order with fma: C = fma(c_k, mB_k, C), mB_k the       */
/* eval_monomial product over the block variables only (the GPU does this   */
/* once per configuration when the plan is built); the data part is then a */
/* nested Horner over the data variables in model order, every step an fma */
/* (at most three data variables).                                          */
static double fast_cm_poly(const rpg_model* model, const rpg_poly* p,
                           const double* x) {
  const int32_t nv = model->n_vars;
  int dv[3];
  int nd = 0;
  for (int v = 0; v < nv; ++v)
    if (model->var_kind[v] >= 0 && nd < 3) dv[nd++] = v;
  int maxd[3] = {0, 0, 0};
  for (int32_t k = 0; k < p->n_terms; ++k)
    for (int j = 0; j < nd; ++j) {
      int e = p->exps[(size_t)k * nv + dv[j]];
      if (e > maxd[j]) maxd[j] = e;
    }
  int s0 = nd > 0 ? maxd[0] + 1 : 1, s1 = nd > 1 ? maxd[1] + 1 : 1,
      s2 = nd > 2 ? maxd[2] + 1 : 1;
  double C[(O1_MAXDEG + 1) * (O1_MAXDEG + 1) * (O1_MAXDEG + 1)];
  for (int i = 0; i < s0 * s1 * s2; ++i) C[i] = 0.0;
  for (int32_t k = 0; k < p->n_terms; ++k) {
    const uint8_t* ex = p->exps + (size_t)k * nv;
    double mB = 1.0;
    for (int v = 0; v < nv; ++v) {
      if (model->var_kind[v] >= 0) continue;
      double pw = 1.0;
      for (int e = 0; e < ex[v]; ++e) pw *= x[v];
      mB *= pw;
    }
    int a = nd > 0 ? ex[dv[0]] : 0;
    int b = nd > 1 ? ex[dv[1]] : 0;
    int c = nd > 2 ? ex[dv[2]] : 0;
    double* slot = &C[(a * s1 + b) * s2 + c];
    *slot = fma(p->coef[k], mB, *slot);
  }
  double xv0 = nd > 0 ? x[dv[0]] : 0.0;
  double xv1 = nd > 1 ? x[dv[1]] : 0.0;
  double xv2 = nd > 2 ? x[dv[2]] : 0.0;
  double outer = 0.0;
  for (int a = s0 - 1; a >= 0; --a) {
    double mid = 0.0;
    for (int b = s1 - 1; b >= 0; --b) {
      double inner = C[(a * s1 + b) * s2 + (s2 - 1)];
      for (int c = s2 - 2; c >= 0; --c)
        inner = fma(inner, xv2, C[(a * s1 + b) * s2 + c]);
      mid = (b == s1 - 1) ? inner : fma(mid, xv1, inner);
    }
    outer = (a == s0 - 1) ? mid : fma(outer, xv0, mid);
  }
  return outer;
}

/* ------------------------------------------------------------------------ */
/* Occupancy — perfmodel.hpp:239-266 (direct path).                          */

/* `floor(...)` results are compared against b in the double domain: equal to
 * the reference's static_cast<long long>(floor(..)) wherever that cast is
 * defined, and well-defined for huge quotients. */
int64_t o1_active_blocks(const rpg_profile* hw, double R, double Z, int64_t T) {
  if (T < 1 || T > hw->T_max) return 0;
  int64_t warps_per_block = (T + 31) / 32;
  int64_t b = hw->B_max;
  int64_t lw = hw->W_max / warps_per_block;
  if (lw < b) b = lw;
  if (R > 0) {
    double lim = floor((double)hw->R_max / (R * (double)T));
    if (lim < (double)b) b = (int64_t)lim;
  }
  if (Z > 0) {
    double lim = floor((double)hw->Z_max / Z);
    if (lim < (double)b) b = (int64_t)lim;
  }
  return b < 1 ? 0 : b;
}

int64_t o1_active_warps(const rpg_profile* hw, int64_t b_active, int64_t T) {
  if (b_active <= 0) return 0;
  int64_t w = b_active * T / 32;
  return w < hw->W_max ? w : hw->W_max;
}

double o1_occupancy(const rpg_profile* hw, double R, double Z, int64_t T) {
  int64_t b = o1_active_blocks(hw, R, Z, T);
  return (double)o1_active_warps(hw, b, T) / (double)hw->W_max;
}

/* ------------------------------------------------------------------------ */
/* MWP-CWP — perfmodel.hpp:298-395 (direct path).                            */

static double dmin(double a, double b) { return b < a ? b : a; } /* std::min */

/* The with-memory / compute-only core shared by the direct path and the
 * program path; b and n are the resident blocks / warps. */
static void mwpcwp_core(const rpg_profile* hw, const o1_metrics* m, int64_t b,
                        int64_t W, int32_t rep_mode, int program_cwp,
                        o1_breakdown* out) {
  const double mem = m->mem_insts_per_thread;
  const double n = (double)W;
  out->b_active = b;
  out->n_active_warps = W;
  const double mem_l_coal = hw->mem_latency_cycles;
  const double mem_l_uncoal =
      hw->mem_latency_cycles +
      ((double)hw->uncoal_per_mw - 1.0) * hw->departure_del_uncoal_cycles;
  out->comp_cycles = hw->issue_cycles * (m->comp_insts_per_thread + mem);
  double rep_den = (double)b * (double)hw->num_SM;
  out->rep = m->total_blocks / rep_den;
  if (rep_mode == RPG_REP_CEIL) out->rep = ceil(out->rep);

  if (mem == 0.0) {
    out->mem_cycles = 0.0;
    out->mwp = n;
    out->cwp = out->comp_cycles > 0.0 ? 1.0 : n;
    out->case_tag = RPG_CASE_CWP_BOUND;
    out->cycles_pre_synch = out->comp_cycles * out->rep;
    out->synch_cost = hw->departure_del_coal_cycles * (out->mwp - 1.0) *
                      m->synch_insts_per_block * (double)b * out->rep;
    out->total_cycles = out->cycles_pre_synch + out->synch_cost;
    return;
  }
  const double r_uncoal = m->uncoal_mem_insts_per_thread / mem;
  const double weighted_mem_l =
      r_uncoal * mem_l_uncoal + (1.0 - r_uncoal) * mem_l_coal;
  const double departure_delay =
      r_uncoal * hw->departure_del_uncoal_cycles * (double)hw->uncoal_per_mw +
      (1.0 - r_uncoal) * hw->departure_del_coal_cycles;
  out->mem_cycles = m->uncoal_mem_insts_per_thread * mem_l_uncoal +
                    m->coal_mem_insts_per_thread * mem_l_coal;
  const double mwp_no_bw = weighted_mem_l / departure_delay;
  const double bw_per_warp =
      hw->freq_GHz * (double)hw->load_bytes_per_warp / hw->mem_latency_cycles;
  const double mwp_peak_bw =
      hw->mem_bandwidth_GBps / (bw_per_warp * (double)hw->num_SM);
  out->mwp = dmin(dmin(mwp_no_bw, mwp_peak_bw), n);
  double cwp_full;
  if (program_cwp) {
    /* Program: cwp = warps when comp_cycles == 0, else min(cwp_full, warps)
     * (perfmodel.hpp:762-773) — also for negative comp_cycles. */
    cwp_full = out->comp_cycles == 0.0
                   ? INFINITY
                   : (out->mem_cycles + out->comp_cycles) / out->comp_cycles;
  } else {
    cwp_full = out->comp_cycles > 0.0
                   ? (out->mem_cycles + out->comp_cycles) / out->comp_cycles
                   : INFINITY;
  }
  out->cwp = dmin(cwp_full, n);
  const double comp_per_mem = out->comp_cycles / mem;
  if (out->mwp == n && out->cwp == n) {
    out->case_tag = RPG_CASE_BOTH_SATURATED;
    out->cycles_pre_synch =
        (out->mem_cycles + out->comp_cycles + comp_per_mem * (out->mwp - 1.0)) *
        out->rep;
  } else if (out->cwp >= out->mwp || out->comp_cycles > out->mem_cycles) {
    out->case_tag = RPG_CASE_CWP_BOUND;
    out->cycles_pre_synch =
        (out->mem_cycles * n / out->mwp + comp_per_mem * (out->mwp - 1.0)) *
        out->rep;
  } else {
    out->case_tag = RPG_CASE_MWP_BOUND;
    out->cycles_pre_synch =
        (hw->mem_latency_cycles + out->comp_cycles * n) * out->rep;
  }
  out->synch_cost = departure_delay * (out->mwp - 1.0) *
                    m->synch_insts_per_block * (double)b * out->rep;
  out->total_cycles = out->cycles_pre_synch + out->synch_cost;
}

static int metrics_negative(const o1_metrics* m) {
  return m->comp_insts_per_thread < 0 || m->mem_insts_per_thread < 0 ||
         m->uncoal_mem_insts_per_thread < 0 ||
         m->coal_mem_insts_per_thread < 0 || m->synch_insts_per_block < 0 ||
         m->total_blocks < 0;
}

int o1_mwpcwp_cycles(const rpg_profile* hw, const o1_metrics* m,
                     const rpg_config* c, int32_t rep_mode, o1_breakdown* out) {
  const double mem = m->mem_insts_per_thread;
  double sum = m->uncoal_mem_insts_per_thread + m->coal_mem_insts_per_thread;
  if (fabs(sum - mem) > 1e-9 * (mem > 1.0 ? mem : 1.0)) return O1_MODEL_ERROR;
  if (metrics_negative(m)) return O1_MODEL_ERROR;
  const int64_t T = c->bx * c->by * c->bz;
  int64_t b = o1_active_blocks(hw, m->regs_per_thread,
                               m->shared_words_per_block, T);
  if (b == 0) return O1_ZERO_OCCUPANCY;
  int64_t W = o1_active_warps(hw, b, T);
  if (W == 0) return O1_ZERO_OCCUPANCY;
  mwpcwp_core(hw, m, b, W, rep_mode, 0, out);
  return O1_OK;
}

/* ------------------------------------------------------------------------ */
/* Metrics — perfmodel.hpp:460-478.                                          */

static int metric_value(const rpg_model* model, int slot, const double* x,
                        int fast, double* v, int* near_zero, int* den_zero) {
  const rpg_metric* mt = &model->metric[slot];
  if (mt->is_const) {
    *v = mt->value;
    return 0;
  }
  double p, q;
  if (fast == RPG_ARITH_FAST_CM) {
    p = fast_cm_poly(model, &mt->num, x);
    q = fast_cm_poly(model, &mt->den, x);
  } else if (fast) {
    p = fast_poly(model, &mt->num, x);
    q = fast_poly(model, &mt->den, x);
  } else {
    p = o1_eval_poly(&mt->num, model->n_vars, x);
    q = o1_eval_poly(&mt->den, model->n_vars, x);
  }
  double mag = fabs(p);
  if (fabs(q) < 1e-12 * (mag > 1.0 ? mag : 1.0)) *near_zero = 1;
  if (q == 0.0) {
    *den_zero = 1;
    return 1;
  }
  *v = p / q;
  return 0;
}

/* Evaluates the seven metric sources in evaluate_metrics order.  Returns
 * nonzero when a denominator is exactly zero (program: infeasible).  Sets
 * *near_zero when the direct path would throw DenominatorNearZero. */
static int eval_all_metrics(const rpg_model* model, const double* x, int fast,
                            o1_metrics* m, int* near_zero) {
  int den_zero = 0;
  *near_zero = 0;
  double v[RPG_N_METRICS];
  for (int s = 0; s < RPG_N_METRICS; ++s) {
    v[s] = 0.0;
    metric_value(model, s, x, fast, &v[s], near_zero, &den_zero);
  }
  m->regs_per_thread = v[RPG_METRIC_REGS];
  m->shared_words_per_block = v[RPG_METRIC_SHARED];
  m->comp_insts_per_thread = v[RPG_METRIC_COMP];
  m->uncoal_mem_insts_per_thread = v[RPG_METRIC_UNCOAL];
  m->coal_mem_insts_per_thread = v[RPG_METRIC_COAL];
  m->mem_insts_per_thread =
      m->uncoal_mem_insts_per_thread + m->coal_mem_insts_per_thread;
  m->synch_insts_per_block = v[RPG_METRIC_SYNCH];
  m->total_blocks = v[RPG_METRIC_TOTAL_BLOCKS];
  return den_zero;
}

int o1_evaluate_metrics(const rpg_model* model, const double* x,
                        o1_metrics* out) {
  int nz = 0;
  int dz = eval_all_metrics(model, x, 0, out, &nz);
  return (dz || nz) ? O1_DEN_NEAR_ZERO : O1_OK;
}

/* ------------------------------------------------------------------------ */
/* One search point: program semantics for Ec/feasibility, direct-path       */
/* semantics for the occupancy tie-break and the case tag.                   */

static void point_coords(const rpg_model* model, const int64_t* data,
                         const rpg_config* c, double* x) {
  for (int v = 0; v < model->n_vars; ++v) {
    int k = model->var_kind[v];
    if (k == RPG_VAR_BX) x[v] = (double)c->bx;
    else if (k == RPG_VAR_BY) x[v] = (double)c->by;
    else if (k == RPG_VAR_BZ) x[v] = (double)c->bz;
    else x[v] = (double)data[k];
  }
}

static int model_has_bz(const rpg_model* model) {
  for (int v = 0; v < model->n_vars; ++v)
    if (model->var_kind[v] == RPG_VAR_BZ) return 1;
  return 0;
}

/* Program occupancy (emit_occupancy_core, perfmodel.hpp:545-614): limits
 * apply when R / Z are nonzero (not just positive). */
static int64_t program_blocks(const rpg_profile* hw, double R, double Z,
                              int64_t T) {
  if (T > hw->T_max || T < 1) return 0;
  int64_t wpb = (T + 31) / 32;
  int64_t b = hw->B_max;
  int64_t lw = hw->W_max / wpb;
  if (lw < b) b = lw;
  if (R != 0.0) {
    double lim = floor((double)hw->R_max / (R * (double)T));
    if (lim < (double)b) b = (int64_t)lim;
  }
  if (Z != 0.0) {
    double lim = floor((double)hw->Z_max / Z);
    if (lim < (double)b) b = (int64_t)lim;
  }
  return b < 1 ? 0 : b;
}

static int eval_point_impl(const rpg_model* model, const rpg_profile* hw,
                           const rpg_options* opts, const int64_t* data,
                           const rpg_config* c, int fast, o1_point* out) {
  double x[RPG_MAX_VARS];
  point_coords(model, data, c, x);
  out->ec = -1.0;
  out->feasible = 0;
  out->b_active = 0;
  out->w_active = 0;
  out->w_occ = 0;
  out->tag = RPG_CASE_UNKNOWN;

  int64_t T = c->bx * c->by;
  if (model_has_bz(model)) T *= c->bz;
  const int64_t T_dir = c->bx * c->by * c->bz;

  o1_metrics m;
  int near_zero = 0;
  int den_zero = eval_all_metrics(model, x, fast, &m, &near_zero);

  /* Direct-path occupancy for the tie-break (pipeline.hpp:629-651). */
  {
    double R = near_zero ? opts->regs_per_thread : m.regs_per_thread;
    double Z = near_zero ? opts->shared_words_per_block : m.shared_words_per_block;
    int64_t b = o1_active_blocks(hw, R, Z, T_dir);
    out->w_occ = (int32_t)o1_active_warps(hw, b, T_dir);
  }
  if (den_zero) return 0;

  int64_t b = program_blocks(hw, m.regs_per_thread, m.shared_words_per_block, T);
  if (b < 1) return 0;
  int64_t W = (b * T) / 32;
  if (W > hw->W_max) W = hw->W_max;
  if (W < 1) return 0;
  out->b_active = (int32_t)b;
  out->w_active = (int32_t)W;

  o1_breakdown br;
  mwpcwp_core(hw, &m, b, W, opts->rep_mode, 1, &br);
  out->ec = br.total_cycles;
  out->feasible = br.total_cycles >= 0.0;

  /* Direct-path case tag (pipeline.hpp:635-647). */
  if (!near_zero && !metrics_negative(&m)) {
    int64_t bd = o1_active_blocks(hw, m.regs_per_thread,
                                  m.shared_words_per_block, T_dir);
    int64_t Wd = o1_active_warps(hw, bd, T_dir);
    if (bd > 0 && Wd > 0) {
      if (bd == b && Wd == W) {
        out->tag = br.case_tag;
      } else {
        o1_breakdown bd_br;
        mwpcwp_core(hw, &m, bd, Wd, opts->rep_mode, 0, &bd_br);
        out->tag = bd_br.case_tag;
      }
    }
  }
  return 0;
}

int o1_eval_point(const rpg_model* model, const rpg_profile* hw,
                  const rpg_options* opts, const int64_t* data, int32_t d,
                  const rpg_config* c, o1_point* out) {
  (void)d;
  return eval_point_impl(model, hw, opts, data, c, opts->arith,
                         out);
}

/* ------------------------------------------------------------------------ */
/* Ranking — pipeline.hpp:616-679.                                           */

typedef struct {
  const rpg_config* space;
  const double* ec;
} sort_ctx;

static int lex_cmp(const rpg_config* a, const rpg_config* b) {
  if (a->bx != b->bx) return a->bx < b->bx ? -1 : 1;
  if (a->by != b->by) return a->by < b->by ? -1 : 1;
  if (a->bz != b->bz) return a->bz < b->bz ? -1 : 1;
  return 0;
}

static void sort_by_ec_lex(int32_t* idx, int64_t n, const double* ec,
                           const rpg_config* space) {
  /* insertion-merge sort (stable) keyed on (Ec, lex, index) */
  if (n < 2) return;
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  for (int64_t width = 1; width < n; width *= 2) {
    for (int64_t lo = 0; lo < n; lo += 2 * width) {
      int64_t mid = lo + width < n ? lo + width : n;
      int64_t hi = lo + 2 * width < n ? lo + 2 * width : n;
      int64_t i = lo, j = mid, k = lo;
      while (i < mid && j < hi) {
        int32_t a = idx[i], b = idx[j];
        int take_b;
        if (ec[a] != ec[b]) take_b = ec[b] < ec[a];
        else {
          int lc = lex_cmp(&space[b], &space[a]);
          take_b = lc < 0 || (lc == 0 && b < a);
        }
        tmp[k++] = take_b ? idx[j++] : idx[i++];
      }
      while (i < mid) tmp[k++] = idx[i++];
      while (j < hi) tmp[k++] = idx[j++];
    }
    memcpy(idx, tmp, sizeof(int32_t) * (size_t)n);
  }
  free(tmp);
}

static void stable_sort_by_occ_desc(int32_t* idx, int64_t n,
                                    const int32_t* w_occ) {
  for (int64_t i = 1; i < n; ++i) {
    int32_t v = idx[i];
    int64_t j = i - 1;
    while (j >= 0 && w_occ[idx[j]] < w_occ[v]) {
      idx[j + 1] = idx[j];
      --j;
    }
    idx[j + 1] = v;
  }
}

static int search_one_impl(const rpg_model* model, const rpg_profile* hw,
                           const rpg_options* opts, const rpg_config* space,
                           int64_t n_space, const int64_t* data,
                           rpg_winner* out, int32_t* order, double* ec,
                           int32_t* w_occ, int32_t* idx, o1_point* pts) {
  int fast = opts->arith;  /* RPG_ARITH_*: selects the polynomial order */
  int64_t nf = 0;
  for (int64_t i = 0; i < n_space; ++i) {
    eval_point_impl(model, hw, opts, data, &space[i], fast, &pts[i]);
    ec[i] = pts[i].ec;
    w_occ[i] = pts[i].w_occ;
    if (pts[i].feasible) idx[nf++] = (int32_t)i;
  }
  memset(out, 0, sizeof(*out));
  out->cfg_idx = -1;
  out->case_tag = RPG_CASE_UNKNOWN;
  out->n_feasible = (int32_t)nf;
  if (nf == 0) return 0;
  sort_by_ec_lex(idx, nf, ec, space);
  double best = ec[idx[0]];
  double bound = best + best * opts->tie_rel_tol;
  int64_t ties = 0;
  while (ties < nf && ec[idx[ties]] <= bound) ++ties;
  stable_sort_by_occ_desc(idx, ties, w_occ);
  int32_t w = idx[0];
  out->ec = ec[w];
  out->best_ec = best;
  out->cfg_idx = w;
  out->ties = (int32_t)ties;
  out->b_active = pts[w].b_active;
  out->w_active = pts[w].w_active;
  out->w_occ = pts[w].w_occ;
  out->case_tag = pts[w].tag;
  if (order) memcpy(order, idx, sizeof(int32_t) * (size_t)nf);
  return 0;
}

int o1_search_one(const rpg_model* model, const rpg_profile* hw,
                  const rpg_options* opts, const rpg_config* space,
                  int64_t n_space, const int64_t* data, int32_t d,
                  rpg_winner* out, int32_t* order) {
  (void)d;
  double* ec = (double*)malloc(sizeof(double) * (size_t)n_space);
  int32_t* w_occ = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_space);
  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_space);
  o1_point* pts = (o1_point*)malloc(sizeof(o1_point) * (size_t)n_space);
  int rc = search_one_impl(model, hw, opts, space, n_space, data, out, order,
                           ec, w_occ, idx, pts);
  free(ec);
  free(w_occ);
  free(idx);
  free(pts);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Threaded batch drivers: static slices over tuples, as the reference       */
/* slices configs over std::thread workers (pipeline.hpp:595-614).           */

typedef struct {
  const rpg_model* model;
  const rpg_profile* hw;
  const rpg_options* opts;
  const rpg_config* space;
  int64_t n_space;
  const int64_t* data;
  int32_t d;
  int64_t lo, hi;
  rpg_winner* out;
  double* ec;
  uint8_t* tag;
  int32_t* w_occ;
} batch_job;

static void* search_worker(void* arg) {
  batch_job* j = (batch_job*)arg;
  size_t n = (size_t)j->n_space;
  double* ec = (double*)malloc(sizeof(double) * n);
  int32_t* w_occ = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * n);
  o1_point* pts = (o1_point*)malloc(sizeof(o1_point) * n);
  for (int64_t t = j->lo; t < j->hi; ++t)
    search_one_impl(j->model, j->hw, j->opts, j->space, j->n_space,
                    j->data + (size_t)t * j->d, &j->out[t], NULL, ec, w_occ,
                    idx, pts);
  free(ec);
  free(w_occ);
  free(idx);
  free(pts);
  return NULL;
}

static void* evaluate_worker(void* arg) {
  batch_job* j = (batch_job*)arg;
  int fast = j->opts->arith;
  for (int64_t t = j->lo; t < j->hi; ++t)
    for (int64_t c = 0; c < j->n_space; ++c) {
      o1_point p;
      eval_point_impl(j->model, j->hw, j->opts, j->data + (size_t)t * j->d,
                      &j->space[c], fast, &p);
      size_t at = (size_t)t * (size_t)j->n_space + (size_t)c;
      if (j->ec) j->ec[at] = p.ec;
      if (j->tag) j->tag[at] = (uint8_t)p.tag;
      if (j->w_occ) j->w_occ[at] = p.w_occ;
    }
  return NULL;
}

static int run_batch(batch_job* proto, int64_t n_tuples, int32_t n_threads,
                     void* (*fn)(void*)) {
  if (n_threads < 1) n_threads = 1;
  if (n_threads > n_tuples) n_threads = (int32_t)(n_tuples > 0 ? n_tuples : 1);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  batch_job* jobs = (batch_job*)malloc(sizeof(batch_job) * (size_t)n_threads);
  for (int32_t w = 0; w < n_threads; ++w) {
    jobs[w] = *proto;
    jobs[w].lo = n_tuples * w / n_threads;
    jobs[w].hi = n_tuples * (w + 1) / n_threads;
    pthread_create(&th[w], NULL, fn, &jobs[w]);
  }
  for (int32_t w = 0; w < n_threads; ++w) pthread_join(th[w], NULL);
  free(th);
  free(jobs);
  return 0;
}

int o1_search_batch(const rpg_model* model, const rpg_profile* hw,
                    const rpg_options* opts, const rpg_config* space,
                    int64_t n_space, const int64_t* data, int64_t n_tuples,
                    int32_t d, int32_t n_threads, rpg_winner* out) {
  batch_job proto = {model, hw, opts, space, n_space, data, d, 0, 0,
                     out, NULL, NULL, NULL};
  return run_batch(&proto, n_tuples, n_threads, search_worker);
}

int o1_evaluate_batch(const rpg_model* model, const rpg_profile* hw,
                      const rpg_options* opts, const rpg_config* space,
                      int64_t n_space, const int64_t* data, int64_t n_tuples,
                      int32_t d, int32_t n_threads, double* ec, uint8_t* tag,
                      int32_t* w_occ) {
  batch_job proto = {model, hw, opts, space, n_space, data, d, 0, 0,
                     NULL, ec, tag, w_occ};
  return run_batch(&proto, n_tuples, n_threads, evaluate_worker);
}
