/*
 * rpg.h — C ABI of the B200 rational-program evaluator (librpgpu.so).
 *
 * The reference (`ratprog`, arXiv 1906.00142 / KLARAPTOR restatement) has no
 * FFI: its hot path is a header-only C++ API.  This header is the thin,
 * plain-pointer boundary that sits under the C++ drop-in
 * (`ratprog::pipe::search_optimal` & co.) and that any
 * ctypes / cgo / JNI binding would use.  No torch or CUDA types appear here;
 * every buffer passed to a non-`_device` entry point is caller-owned HOST
 * memory, copied in and out, and no pointer is retained after the call
 * returns (the reference returns by value).
 *
 * Entry points and the reference interface each one replaces:
 *
 *   rpg_plan_create        — the one-time setup done by
 *                            pipe::generate_rp + make_binding_plan
 *                            (pipeline.hpp:233-255, 482-516) and
 *                            perf::check_metric_spec (perfmodel.hpp:428-456):
 *                            validates the metric spec / profile / space and
 *                            uploads them to the device once.
 *   rpg_search_batch       — pipe::search_optimal (pipeline.hpp:575-680),
 *                            batched over data tuples: per tuple, the winning
 *                            configuration under the reference's ranking
 *                            (min Ec, tie group Ec <= best*(1+tol), max
 *                            occupancy, then Ec, then lex (bx,by,bz)).
 *   rpg_evaluate           — the per-config values search_optimal computes
 *                            before ranking: the program output
 *                            (ir::evaluate of emit_mwpcwp_rp,
 *                            perfmodel.hpp:648-834; -1 sentinel when the
 *                            program branches to `infeasible`), the occupancy
 *                            used for tie-breaking and the case tag
 *                            (pipeline.hpp:623-652).
 *   rpg_search             — one-shot create + search_batch + destroy.
 *   rpg_fit_rational       — poly::fit_rational (polyfit.hpp:337-427).
 *
 * Error convention: 0 on success, a negative RPG_E_* code otherwise, with a
 * NUL-terminated message written to `err` (may be NULL).  Messages reuse the
 * reference's wording so the C++ shim can rethrow the same exception types.
 */
#ifndef RPG_H_
#define RPG_H_

#ifndef __CUDACC_RTC__
#include <stddef.h>
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define RPG_ABI_VERSION 1

#define RPG_MAX_VARS 8
#define RPG_N_METRICS 7

/* Metric slots, in the order evaluate_metrics reads them
 * (perfmodel.hpp:468-476). */
enum {
  RPG_METRIC_REGS = 0,         /* regs_per_thread */
  RPG_METRIC_SHARED = 1,       /* shared_words_per_block */
  RPG_METRIC_COMP = 2,         /* comp_insts_per_thread */
  RPG_METRIC_UNCOAL = 3,       /* uncoal_mem_insts_per_thread */
  RPG_METRIC_COAL = 4,         /* coal_mem_insts_per_thread */
  RPG_METRIC_SYNCH = 5,        /* synch_insts_per_block */
  RPG_METRIC_TOTAL_BLOCKS = 6  /* total_blocks */
};

/* Variable kinds (model variable order is data-driven, perfmodel.hpp:416-420):
 * k >= 0 is data parameter D(k+1); negative codes are block dimensions. */
enum { RPG_VAR_BX = -1, RPG_VAR_BY = -2, RPG_VAR_BZ = -3 };

/* perf::CaseTag (perfmodel.hpp:273) plus "-" for rows whose direct-path
 * diagnostics threw (pipeline.hpp:637-647). */
enum {
  RPG_CASE_BOTH_SATURATED = 0,
  RPG_CASE_CWP_BOUND = 1,
  RPG_CASE_MWP_BOUND = 2,
  RPG_CASE_UNKNOWN = 3
};

/* perf::RepMode (perfmodel.hpp:271). */
enum { RPG_REP_REAL = 0, RPG_REP_CEIL = 1 };

/* Arithmetic mode of the evaluator.
 *   RPG_ARITH_EXACT: IEEE mul/add in the reference's basis order, no FMA
 *                    contraction — bit-identical to oracle O1.
 *   RPG_ARITH_FAST:  per-data-tuple collapse of the data-parameter part of
 *                    every polynomial and DFMA Horner evaluation of the
 *                    block-dimension part (bit-identical to O1's FAST twin).
 *   RPG_ARITH_FAST_CM: the dual order — per-configuration collapse of the
 *                    block-dimension part (fma in basis order, once per
 *                    plan) and DFMA Horner in the data parameter per point
 *                    (bit-identical to O1's FAST_CM twin).  Searches only
 *                    (rpg_search_batch / _device); models with one data
 *                    parameter whose regs/shared metrics are constants. */
enum { RPG_ARITH_EXACT = 0, RPG_ARITH_FAST = 1, RPG_ARITH_FAST_CM = 2 };

enum {
  RPG_OK = 0,
  RPG_E_INVALID = -1,      /* std::invalid_argument */
  RPG_E_MODEL = -2,        /* perf::ModelError */
  RPG_E_PROFILE = -3,      /* perf::ProfileError */
  RPG_E_CUDA = -4,         /* device / driver failure */
  RPG_E_NO_FEASIBLE = -5,  /* pipe::NoFeasibleConfig (single-tuple calls) */
  RPG_E_PIPELINE = -6,     /* pipe::PipelineError */
  RPG_E_FIT = -7,          /* poly::DegenerateFit / SvdFailure */
  RPG_E_EVAL = -8,         /* ir::EvalError / DivisionByZero (bare programs) */
  RPG_E_CSV = -9           /* data::CsvError */
};

/* perf::DeviceProfile, same fields and order (perfmodel.hpp:50-65). */
typedef struct {
  int64_t R_max, Z_max, T_max, B_max, W_max, num_SM;
  double freq_GHz, mem_latency_cycles, departure_del_coal_cycles,
      departure_del_uncoal_cycles, mem_bandwidth_GBps, issue_cycles;
  int64_t load_bytes_per_warp, uncoal_per_mw;
} rpg_profile;

/* One polynomial in sparse "AltArr-like" form: term k is
 * coef[k] * prod_v x_v^exps[k*n_vars+v], terms in graded-lex basis order
 * (polyfit.hpp:50-73).  The order fixes the FP summation order. */
typedef struct {
  int32_t n_terms;
  int32_t reserved;
  const double* coef;
  const uint8_t* exps;
} rpg_poly;

/* One metric source: a constant or a fitted p/q (perfmodel.hpp:416-426). */
typedef struct {
  int32_t is_const;
  int32_t reserved;
  double value;
  rpg_poly num, den;
} rpg_metric;

/* perf::MetricSpec: variables (D1..Dd, bx, by[, bz] in any order) and the
 * seven metric sources indexed by RPG_METRIC_*. */
typedef struct {
  int32_t n_vars;
  int32_t var_kind[RPG_MAX_VARS];
  rpg_metric metric[RPG_N_METRICS];
} rpg_model;

/* perf::LaunchConfig (perfmodel.hpp:79-84). */
typedef struct {
  int64_t bx, by, bz;
} rpg_config;

/* Which device implementation evaluates the points (both are sm_100a CUDA;
 * both are bit-identical to oracle O1):
 *   RPG_KERNEL_SPECIALIZED: a kernel generated for this model at plan time
 *                           (NVRTC, sm_100a): straight-line polynomial code,
 *                           coefficients as immediates (default);
 *   RPG_KERNEL_GENERIC:     the ahead-of-time table-driven kernel. */
enum { RPG_KERNEL_SPECIALIZED = 0, RPG_KERNEL_GENERIC = 1 };

/* pipe::SearchOptions subset (pipeline.hpp:438-452). */
typedef struct {
  int32_t rep_mode;       /* RPG_REP_* */
  int32_t arith;          /* RPG_ARITH_* */
  double tie_rel_tol;     /* default 1e-12 */
  double regs_per_thread; /* occupancy context on DenominatorNearZero */
  double shared_words_per_block;
  int32_t kernel;         /* RPG_KERNEL_* */
  int32_t reserved;
} rpg_options;

/* Per-tuple search result (the head of pipe::SearchResult::ranking plus its
 * counters).  cfg_idx = -1 when no configuration is feasible. */
typedef struct {
  double ec;          /* estimated cycles of the winner */
  double best_ec;     /* minimum Ec over the tuple (tie-group anchor) */
  int32_t cfg_idx;    /* index into the plan's configuration space */
  int32_t ties;       /* size of the leading tie group */
  int32_t n_feasible; /* evaluated - infeasible */
  int32_t b_active;   /* resident blocks per SM of the winner */
  int32_t w_active;   /* resident warps per SM of the winner */
  int32_t w_occ;      /* warps behind the winner's occupancy (w_occ/W_max) */
  int32_t case_tag;   /* RPG_CASE_* of the winner */
  int32_t reserved;
} rpg_winner;

typedef struct rpg_plan rpg_plan;

const char* rpg_version(void);
int rpg_device_count(void);

int rpg_plan_create(const rpg_model* model, const rpg_profile* hw,
                    const rpg_config* space, int64_t n_space,
                    const rpg_options* opts, int32_t device, rpg_plan** out,
                    char* err, size_t errlen);
int rpg_plan_destroy(rpg_plan* plan);

/* data: n_tuples x d int64 data-parameter values (D1..Dd), host memory.
 * out: n_tuples winners, host memory. */
int rpg_search_batch(rpg_plan* plan, const int64_t* data, int64_t n_tuples,
                     int32_t d, rpg_winner* out, char* err, size_t errlen);

/* Same, with device-resident inputs/outputs on the given cudaStream_t
 * (passed as void*).  Asynchronous: returns after enqueueing. */
int rpg_search_batch_device(rpg_plan* plan, const int64_t* d_data,
                            int64_t n_tuples, int32_t d, rpg_winner* d_out,
                            void* stream, char* err, size_t errlen);

/* Full per-point table, tuple-major (index t*n_space + c).  ec: program
 * output (-1 sentinel for launch/denominator infeasibility; negative values
 * are infeasible for the search too).  tag: RPG_CASE_*.  w_occ: occupancy
 * warps.  Any output pointer may be NULL.  Host memory. */
int rpg_evaluate(rpg_plan* plan, const int64_t* data, int64_t n_tuples,
                 int32_t d, double* ec, uint8_t* tag, int32_t* w_occ,
                 char* err, size_t errlen);

int rpg_evaluate_device(rpg_plan* plan, const int64_t* d_data,
                        int64_t n_tuples, int32_t d, double* d_ec,
                        uint8_t* d_tag, int32_t* d_w_occ, void* stream,
                        char* err, size_t errlen);

/* The CUDA source of the specialized kernels a plan compiles for this model
 * (the B200 counterpart of pipe::emit_c_source, pipeline.hpp:276-433).
 * Writes up to buflen bytes (NUL-terminated; buf may be NULL) and returns the
 * full source length, or a negative RPG_E_* code.  With compile != 0 the
 * source is also compiled for sm_100a with NVRTC (no GPU needed) and
 * *cubin_bytes (nullable) receives the cubin size. */
int64_t rpg_emit_cuda_source(const rpg_model* model, const rpg_profile* hw,
                             const rpg_options* opts, int32_t compile, char* buf,
                             size_t buflen, int64_t* cubin_bytes, char* err,
                             size_t errlen);

/* poly::fit_rational (polyfit.hpp:337-427) on the GPU: the homogeneous
 * least-squares rational fit of y over the points X (m x n_vars, row-major,
 * host memory) with graded-lex numerator/denominator bases of the given
 * per-variable degree bounds, including the reference's positivity safeguard.
 * Outputs (host, caller-allocated): coef_out[n] (numerator coefficients then
 * denominator coefficients, unit 2-norm, first |den| > 1e-10 positive),
 * sigma_out[min(m, n)] (singular values of the equilibrated sample matrix,
 * non-increasing), rank / truncated / residual as FitReport, safeguard_out =
 * whether the safeguard ran.  Any output pointer may be NULL.
 * Errors: RPG_E_INVALID (no samples, bad bounds, n > 64), RPG_E_FIT
 * (DegenerateFit / SvdFailure messages of the reference). */
int rpg_fit_rational(const double* X, const double* y, int64_t m, int32_t n_vars,
                     const int32_t* num_bounds, const int32_t* den_bounds,
                     double rank_tol, int32_t device, double* coef_out,
                     double* sigma_out, int32_t* rank_out, int32_t* truncated_out,
                     double* residual_out, int32_t* safeguard_out, char* err,
                     size_t errlen);

/* rpg_fit_rational with the safeguard's intermediate results (parity
 * diagnostics: the stages of polyfit.hpp:364-414 compared one by one with a
 * CPU restatement).  stage_coef[0] = the unconstrained candidate (smallest
 * right singular vector .* column scale), [1] = the first positive-
 * denominator minimizer result, [2..] = each accepted reweighted round, all
 * raw coordinates before make_ratfunc_from_coeffs' normalisation;
 * round_qmin[r] = min_k q(x_k) of the vector entering reweighted round r
 * (the guard polyfit.hpp:398); stop_reason says why the rounds ended. */
#define RPG_FIT_TRACE_STAGES 5
#define RPG_FIT_MAX_COLS 64
enum {
  RPG_FIT_STOP_NO_SAFEGUARD = -1, /* trigger not met: stage 0 is the result */
  RPG_FIT_STOP_ROUNDS = 0,        /* all reweighted rounds ran */
  RPG_FIT_STOP_QMIN = 1,          /* qprev.minCoeff() > 0 failed */
  RPG_FIT_STOP_EMPTY = 2,         /* a reweighted minimizer returned empty */
  RPG_FIT_STOP_FIRST_EMPTY = 3    /* the first minimizer returned empty */
};
typedef struct {
  int32_t n_stages, stop_reason;
  double stage_coef[RPG_FIT_TRACE_STAGES][RPG_FIT_MAX_COLS];
  double round_qmin[RPG_FIT_TRACE_STAGES];
} rpg_fit_trace;

int rpg_fit_rational_traced(const double* X, const double* y, int64_t m, int32_t n_vars,
                            const int32_t* num_bounds, const int32_t* den_bounds, double rank_tol,
                            int32_t device, double* coef_out, double* sigma_out,
                            int32_t* rank_out, int32_t* truncated_out, double* residual_out,
                            int32_t* safeguard_out, rpg_fit_trace* trace, char* err,
                            size_t errlen);

/* Several fits over one sample set (pipe::fit_all_metrics' loop over the
 * metric columns, pipeline.hpp:145-184): X (m x n_vars, host) is uploaded
 * once and the jobs run concurrently (one host thread and CUDA stream each).
 * Per job: y (m values, host), bounds, the outputs of rpg_fit_rational
 * (nullable) and an optional trace; status / message receive that fit's own
 * return code and error text (RPG_E_FIT for DegenerateFit / SvdFailure).
 * The call itself fails only on bad arguments or a failed upload. */
typedef struct {
  const double* y;
  const int32_t* num_bounds;
  const int32_t* den_bounds;
  double* coef_out;
  double* sigma_out;
  int32_t* rank_out;
  int32_t* truncated_out;
  double* residual_out;
  int32_t* safeguard_out;
  rpg_fit_trace* trace;
  int32_t status;
  char message[252];
} rpg_fit_job;

int rpg_fit_rational_multi(const double* X, int64_t m, int32_t n_vars, rpg_fit_job* jobs,
                           int32_t n_jobs, double rank_tol, int32_t device, char* err,
                           size_t errlen);

/* A bare rational program (ir::RationalProgram, ir.hpp:19-112) lowered for
 * the GPU: variables are slots, literals are doubles (to_double of each
 * rational, as the reference's C lowering prints them, pipeline.hpp:276-433).
 * op: ir::Opcode order (assign, neg, add, sub, mul, euclid_quot, euclid_rem,
 * floor_div, ceil_div, cmp_eq, cmp_lt, branch_if, jump, halt_return).
 * Operands a/b: slot index >= 0, or literal -1-k.  t0/t1: jump targets. */
typedef struct {
  int32_t op, target, a, b, t0, t1;
} rpg_instr;

#define RPG_INPUT_FIXED (-100)

typedef struct {
  int32_t n_instr, n_slots, n_literals, output_slot;
  const rpg_instr* body;
  const double* literals;
  int32_t n_inputs;
  int32_t reserved;
  const int32_t* input_slot;  /* slot of each declared input */
  const int32_t* input_kind;  /* RPG_VAR_BX/BY/BZ, data index >= 0, RPG_INPUT_FIXED */
  const double* input_fixed;  /* value of RPG_INPUT_FIXED inputs (profile fields) */
  int64_t step_limit;         /* interp.hpp:31 (1e6) */
} rpg_program;

/* pipe::search_optimal for a bare program (no metric spec; the `--rp`
 * path, ratprog_cli.cpp:305-307): Ec = the program's value (evaluated with
 * the reference C lowering's double semantics on the GPU), feasible iff >= 0,
 * occupancy from opts->regs_per_thread / shared_words_per_block
 * (pipeline.hpp:648-650), case tag "-".  The returned plan works with
 * rpg_search_batch / rpg_evaluate and their _device variants; evaluation
 * errors (zero divisor, step limit, control falling off the end, reading an
 * unassigned variable — the exact interpreter's throws, interp.hpp:44-121)
 * fail the host-buffer calls with RPG_E_EVAL (see rpg_plan_poll_error for
 * the _device calls).  Inputs bind as make_binding_plan does
 * (pipeline.hpp:482-516): bx/by/bz per configuration, D<k> from the data
 * tuple, device-profile fields fixed (input_fixed). */
int rpg_program_plan_create(const rpg_program* prog, const rpg_profile* hw,
                            const rpg_config* space, int64_t n_space,
                            const rpg_options* opts, int32_t device,
                            rpg_plan** out, char* err, size_t errlen);

/* The CUDA source of the kernels rpg_program_plan_create compiles for a
 * bare program (the counterpart of pipe::emit_c_source, pipeline.hpp:
 * 276-433); same buffer / compile / return conventions as
 * rpg_emit_cuda_source. */
int64_t rpg_emit_program_cuda_source(const rpg_program* prog, const rpg_profile* hw,
                                     const rpg_options* opts, int32_t compile, char* buf,
                                     size_t buflen, int64_t* cubin_bytes, char* err,
                                     size_t errlen);

/* Errors of _device calls on a bare-program plan: synchronizes `stream`
 * (may be NULL), then returns and clears the first evaluation error recorded
 * since the last check (RPG_E_EVAL with the interpreter's message and the
 * failing tuple/configuration), or RPG_OK.  No-op for metric-spec plans. */
int rpg_plan_poll_error(rpg_plan* plan, void* stream, char* err, size_t errlen);

/* FAST_CM range certificate (diagnostics).  counts[64 m + k] = number of the
 * plan's configurations for which, for every N in [2^k, 2^(k+1)] (k = 0..63),
 * pass 1's point is proven to stay on the division fast paths (m = 0: the
 * search kernel skips the per-point range checks there) and, for m = 1, 2, 3,
 * also to fall in MWP-CWP case cwp_bound, mwp_bound, both_saturated (the
 * kernel then evaluates only that case).  Results are identical either way.
 * All zero when the plan has no certificate (not FAST_CM, or RPG_CM_CERT=0). */
int rpg_plan_cert_counts(rpg_plan* plan, int64_t counts[256], char* err, size_t errlen);

/* search_optimal over a per-tuple subset of the plan's configuration space
 * (sanity_report searches each data tuple over its own sampled
 * configurations, pipeline.hpp:816-824): tuple t searches the space indices
 * list[offsets[t] .. offsets[t+1]) (distinct, any order; offsets[0] = 0).
 * Ranking, ties and counts are those of search_optimal over that subset. */
int rpg_search_batch_subsets(rpg_plan* plan, const int64_t* data, int64_t n_tuples,
                             int32_t d, const int64_t* offsets, const int32_t* list,
                             rpg_winner* out, char* err, size_t errlen);
int rpg_search_batch_subsets_device(rpg_plan* plan, const int64_t* d_data,
                                    int64_t n_tuples, int32_t d, const int64_t* d_offsets,
                                    const int32_t* d_list, rpg_winner* d_out, void* stream,
                                    char* err, size_t errlen);

/* perf::mwpcwp_cycles (perfmodel.hpp:298-395) over n rows of given metric
 * values (n x RPG_N_METRICS, RPG_METRIC_* order; mem = uncoal + coal as
 * metrics_from_sample forms it, pipeline.hpp:733-752) and configurations:
 * the direct model, IEEE arithmetic in the reference's order.  Per row:
 * total cycles, resident blocks / warps, case tag, and status 0 = ok,
 * 1 = ZeroOccupancy, 2 = ModelError (negative metric), 3 = ModelError
 * (inconsistent mem).  Output pointers other than status_out may be NULL. */
int rpg_mwpcwp_cycles_batch(const rpg_profile* hw, const double* metrics,
                            const rpg_config* configs, int64_t n, int32_t rep_mode,
                            int32_t device, double* total_out, int32_t* b_out,
                            int32_t* w_out, uint8_t* tag_out, int32_t* status_out,
                            char* err, size_t errlen);

/* perf::MwpCwpBreakdown (perfmodel.hpp:284-296), every field, plus the
 * outcome of the call: status 0 = ok, 1 = ZeroOccupancy "configuration
 * cannot launch (no resident block)", 2 = ModelError "metrics must be
 * non-negative", 3 = ModelError "metrics inconsistent: uncoal + coal must
 * equal mem_insts", 4 = ZeroOccupancy "configuration yields no resident
 * warp" (the reference's checks in its order, perfmodel.hpp:302-320). */
typedef struct {
  int64_t b_active, n_active_warps;
  double mem_cycles, comp_cycles, mwp, cwp, rep;
  int32_t case_tag; /* RPG_CASE_* */
  int32_t status;
  double cycles_pre_synch, synch_cost, total_cycles;
} rpg_breakdown;

/* perf::mwpcwp_cycles (perfmodel.hpp:298-395) over n rows of
 * perf::KernelMetrics in its field order (perfmodel.hpp:68-77: regs, shared,
 * comp, mem, uncoal, coal, synch, total_blocks — 8 doubles per row; mem is
 * read as given) and configurations, on the GPU.  out[n] host memory.
 * Small calls reuse a per-device stream and staging buffers (no allocation
 * per call). */
int rpg_mwpcwp_breakdown_batch(const rpg_profile* hw, const double* kernel_metrics,
                               const rpg_config* configs, int64_t n, int32_t rep_mode,
                               int32_t device, rpg_breakdown* out, char* err, size_t errlen);

/* poly::eval_ratfunc (polyfit.hpp:96-130) at m points X (m x n_vars): out =
 * p/q, status 1 where DenominatorNearZero (|q| < 1e-12 max(1, |p|)). */
int rpg_eval_ratfunc_batch(const rpg_poly* num, const rpg_poly* den, int32_t n_vars,
                           const double* X, int64_t m, int32_t device, double* out,
                           int32_t* status_out, char* err, size_t errlen);

/* n draws of rng::uniform_real(lo, hi) (rng.hpp:14-21) from
 * std::mt19937_64(seed), in order (host). */
int rpg_uniform_stream(uint64_t seed, int64_t n, double lo, double hi, double* out);

/* ---------------------------------------------------------------------------
 * Paper-artifact interop: KLARAPTOR ships each fitted
 * metric as numerator / denominator polynomials in the BPAS library's
 * sparse AltArr_t encoding (the reference itself drops it,
 * SPEC.md:14).  rpg_altarr mirrors AltArr_t's shape — size, alloc, nvar,
 * unpacked flag, then (coefficient, packed degrees) elements in decreasing
 * packed-degree order — with binary64 coefficients (the fitted values the
 * pipeline carries) instead of GMP rationals.  Degrees pack variable 0 into
 * the most significant field: field width w = 64 / nvar bits, variable v at
 * bits [64 - (v+1) w, 64 - v w) — so descending packed order is descending
 * lex order with variable 0 most significant.  nvar <= RPG_MAX_VARS. */
typedef struct {
  double coef;
  uint64_t degs;
} rpg_aa_elem;

typedef struct {
  int32_t size, alloc, nvar, unpacked;
  rpg_aa_elem* elems;
} rpg_altarr;

uint64_t rpg_aa_pack_degs(const uint8_t* exps, int32_t nvar);
void rpg_aa_unpack_degs(uint64_t degs, int32_t nvar, uint8_t* exps);

/* rpg_poly (graded-lex basis order) -> AltArr: exact-zero coefficients
 * dropped (as emit_ratfunc does, perfmodel.hpp:521), elements sorted by
 * decreasing packed degrees.  out->elems must hold out->alloc elements;
 * out->size receives the term count.  RPG_E_INVALID on capacity or nvar. */
int rpg_aa_from_poly(const rpg_poly* p, int32_t nvar, rpg_altarr* out, char* err,
                     size_t errlen);

/* AltArr -> rpg_poly arrays: terms reordered into the reference's graded-lex
 * basis order (polyfit.hpp:50-73: ascending total degree, then lex with
 * variable 0 most significant), which fixes the evaluator's summation order
 * (so a model imported from AltArr evaluates bit-identically to the same
 * model read from ratprog-models-v1 JSON).  Zero coefficients are dropped.
 * coef[cap], exps[cap * nvar] caller-allocated; *n_terms receives the count.
 * RPG_E_INVALID on capacity, nvar, an unsorted or duplicated monomial (not a
 * canonical AltArr), or a non-finite coefficient. */
int rpg_aa_to_poly(const rpg_altarr* a, double* coef, uint8_t* exps, int32_t cap,
                   int32_t* n_terms, char* err, size_t errlen);

/* C header text of one metric in the paper's per-metric-header form
 * (PAPER.md:27-56): static rpg_aa_elem / rpg_altarr definitions
 * `<name>_num` and `<name>_den` (coefficients as exact hex-float literals).
 * Same buffer / return conventions as rpg_emit_cuda_source. */
int64_t rpg_emit_altarr_header(const rpg_poly* num, const rpg_poly* den, int32_t nvar,
                               const char* const* var_names, const char* name, char* buf,
                               size_t buflen, char* err, size_t errlen);

/* ---------------------------------------------------------------------------
 * Several GPUs behind one call (the reference parallelises search_optimal
 * inside the call over std::threads, pipeline.hpp:595-614).  A plan group
 * holds one plan per listed device (a device may be listed more than once).
 * rpg_search_batch_group shards the data tuples into contiguous blocks, one
 * per device (pipeline.hpp:602's partition); with fewer tuples than devices
 * it splits the configuration space instead and reduces in two phases
 * (global best Ec -> tie group -> per-device ranking of the members -> key
 * merge), except for RPG_ARITH_FAST_CM plans, which then use the first
 * device.  The winners are byte-identical to rpg_search_batch on one plan
 * for any device list.  The group copies every input it needs. */
typedef struct rpg_plan_group rpg_plan_group;
int rpg_plan_group_create(const rpg_model* model, const rpg_profile* hw, const rpg_config* space,
                          int64_t n_space, const rpg_options* opts, const int32_t* devices,
                          int32_t n_devices, rpg_plan_group** out, char* err, size_t errlen);
int rpg_plan_group_destroy(rpg_plan_group* group);
int32_t rpg_plan_group_size(const rpg_plan_group* group);
int rpg_search_batch_group(rpg_plan_group* group, const int64_t* data, int64_t n_tuples,
                           int32_t d, rpg_winner* out, char* err, size_t errlen);

/* ---------------------------------------------------------------------------
 * Profiled samples at scale: data::parse_samples /
 * format_samples (datakit.hpp:272-415) — the same CSV schema, provenance
 * comment, checks, error precedence and CsvError messages (RPG_E_CSV) —
 * columnar and multi-threaded (n_threads <= 0: all hardware threads).
 * A parsed set holds n rows: data (n x d int64), configs (n x 3 int64),
 * values (n x n_metrics float64, header order).  provenance_kind: 0 =
 * measured, 1 = synthetic (seed, noise_rel). */
typedef struct rpg_samples rpg_samples;
int rpg_samples_parse(const char* text, size_t len, int32_t n_threads, rpg_samples** out,
                      char* err, size_t errlen);
int rpg_samples_info(const rpg_samples* s, int64_t* n_rows, int32_t* d, int32_t* n_metrics,
                     int32_t* provenance_kind, uint64_t* seed, double* noise_rel);
const char* rpg_samples_metric_name(const rpg_samples* s, int32_t k);
int rpg_samples_copy(const rpg_samples* s, int64_t* data, int64_t* configs, double* values);
void rpg_samples_free(rpg_samples* s);
/* The CSV text (std::to_chars shortest round-trip reals).  Writes up to
 * buflen bytes (NUL-terminated; buf may be NULL) and returns the full text
 * length, or RPG_E_CSV ("cannot format an empty sample set", "metric 'x'
 * has a non-finite value"). */
int64_t rpg_samples_format(const int64_t* data, const int64_t* configs, const double* values,
                           int64_t n, int32_t d, const char* const* metric_names,
                           int32_t n_metrics, int32_t provenance_kind, uint64_t seed,
                           double noise_rel, int32_t n_threads, char* buf, size_t buflen,
                           char* err, size_t errlen);

/* Specialized-kernel module statistics of this process: NVRTC compilations
 * and modules loaded from the persistent cubin cache (directory
 * $RPG_CACHE_DIR, else $XDG_CACHE_HOME/rpgpu, else $HOME/.cache/rpgpu;
 * RPG_CACHE_DIR=off disables it).  Either pointer may be NULL. */
void rpg_jit_stats(int64_t* compiles, int64_t* disk_hits);

/* One-shot convenience for FFI callers. */
int rpg_search(const rpg_model* model, const rpg_profile* hw,
               const rpg_config* space, int64_t n_space,
               const rpg_options* opts, const int64_t* data,
               int64_t n_tuples, int32_t d, int32_t device, rpg_winner* out,
               char* err, size_t errlen);

#ifdef __cplusplus
}
#endif

#endif /* RPG_H_ */
