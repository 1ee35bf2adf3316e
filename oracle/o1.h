/*
 * o1.h — ORACLE O1 (test infrastructure only; never linked into the product).
 *
 * A line-by-line FP64 restatement of the reference's direct evaluation path
 * (ratprog, /root/reference/proj/include/ratprog):
 *   eval_monomial / eval_poly / eval_ratfunc   polyfit.hpp:96-130
 *   active_blocks / active_warps / occupancy   perfmodel.hpp:239-266
 *   mwpcwp_cycles                              perfmodel.hpp:298-395
 *   evaluate_metrics                           perfmodel.hpp:460-478
 *   search_optimal ranking + tie rules         pipeline.hpp:575-680
 * with the *program* feasibility rules of emit_mwpcwp_rp
 * (perfmodel.hpp:533-536, 545-614, 648-834): sentinel -1 for T outside
 * [1, T_max], blocks < 1, warps < 1 or an exactly-zero metric denominator,
 * and feasibility = program output >= 0 (pipeline.hpp:591).
 *
 * Compiled with -O2 -ffp-contract=off so every mul/add rounds separately, as
 * the reference's x86-64 SSE2 build does.  The O1_FAST twin restates the
 * GPU's RPG_ARITH_FAST operation order with std fma() so that mode can be
 * checked bit-for-bit as well.
 *
 * Parity anchors: the reference's own known-answer tests (KATs) are ported in
 * tests/test_oracle_kat.py; the exact-rational semantics of the shipped
 * search (ir::evaluate over the emitted program) are restated separately in
 * oracle/o2_exact.py for spot checks.
 */
#ifndef O1_H_
#define O1_H_

#include <stdint.h>

#include "../include/rpg.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { O1_OK = 0, O1_ZERO_OCCUPANCY = 1, O1_MODEL_ERROR = 2, O1_DEN_NEAR_ZERO = 3 };

/* perf::KernelMetrics (perfmodel.hpp:68-77). */
typedef struct {
  double regs_per_thread, shared_words_per_block, comp_insts_per_thread,
      mem_insts_per_thread, uncoal_mem_insts_per_thread,
      coal_mem_insts_per_thread, synch_insts_per_block, total_blocks;
} o1_metrics;

/* perf::MwpCwpBreakdown (perfmodel.hpp:284-296). */
typedef struct {
  int64_t b_active, n_active_warps;
  double mem_cycles, comp_cycles, mwp, cwp, rep;
  int32_t case_tag;
  double cycles_pre_synch, synch_cost, total_cycles;
} o1_breakdown;

/* One (tuple, config) point under the search semantics. */
typedef struct {
  double ec;        /* program output; -1 sentinel when guarded */
  int32_t feasible; /* ec >= 0 and not guarded */
  int32_t b_active; /* program-path blocks (0 when guarded) */
  int32_t w_active; /* program-path warps (0 when guarded) */
  int32_t w_occ;    /* direct-path occupancy warps (pipeline.hpp:629-651) */
  int32_t tag;      /* RPG_CASE_* from the direct path */
  int32_t reserved;
} o1_point;

double o1_eval_monomial(const uint8_t* exps, const double* x, int32_t n_vars);
double o1_eval_poly(const rpg_poly* p, int32_t n_vars, const double* x);
int o1_eval_ratfunc(const rpg_poly* num, const rpg_poly* den, int32_t n_vars,
                    const double* x, double* out);

int64_t o1_active_blocks(const rpg_profile* hw, double R, double Z, int64_t T);
int64_t o1_active_warps(const rpg_profile* hw, int64_t b_active, int64_t T);
double o1_occupancy(const rpg_profile* hw, double R, double Z, int64_t T);
int o1_mwpcwp_cycles(const rpg_profile* hw, const o1_metrics* m,
                     const rpg_config* c, int32_t rep_mode, o1_breakdown* out);
int o1_evaluate_metrics(const rpg_model* model, const double* x,
                        o1_metrics* out);

int o1_eval_point(const rpg_model* model, const rpg_profile* hw,
                  const rpg_options* opts, const int64_t* data, int32_t d,
                  const rpg_config* c, o1_point* out);

/* search_optimal for one data tuple.  order (nullable, n_space entries):
 * ranking of the feasible configs (indices), best first; returns the
 * winner record (cfg_idx -1 when nothing is feasible). */
int o1_search_one(const rpg_model* model, const rpg_profile* hw,
                  const rpg_options* opts, const rpg_config* space,
                  int64_t n_space, const int64_t* data, int32_t d,
                  rpg_winner* out, int32_t* order);

int o1_search_batch(const rpg_model* model, const rpg_profile* hw,
                    const rpg_options* opts, const rpg_config* space,
                    int64_t n_space, const int64_t* data, int64_t n_tuples,
                    int32_t d, int32_t n_threads, rpg_winner* out);

int o1_evaluate_batch(const rpg_model* model, const rpg_profile* hw,
                      const rpg_options* opts, const rpg_config* space,
                      int64_t n_space, const int64_t* data, int64_t n_tuples,
                      int32_t d, int32_t n_threads, double* ec, uint8_t* tag,
                      int32_t* w_occ);

#ifdef __cplusplus
}
#endif

#endif /* O1_H_ */
