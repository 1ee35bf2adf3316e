// rpg_search.cu — sm_100a evaluator kernels and the C ABI of librpgpu.so.
//
// K1+K2 fused ("search"): one CTA per data tuple (persistent over tuples).
//   prologue  per-tuple data-parameter monomial prefixes mD[k] for every
//             polynomial term (EXACT) or the per-tuple collapsed
//             coefficients of every block-dimension pattern (FAST), in SMEM;
//   pass 1    every thread evaluates its strided share of the configuration
//             space (one thread per (tuple, config) point): metrics ->
//             occupancy -> MWP-CWP Ec (rpg_device.cuh); Ec and the tie-break
//             occupancy are kept in SMEM (or a per-CTA global scratch slice
//             for spaces too large for SMEM); block-min of Ec;
//   pass 2    the tie group Ec <= best + best*tol is scanned and reduced
//             with the reference's key (max occupancy, min Ec, lex (bx,by,bz),
//             pipeline.hpp:654-669) plus a tie count; one thread recomputes
//             the winner's diagnostics and writes a 48-byte rpg_winner.
// K1 ("evaluate"): same prologue and per-point model, writing the full
// Ec / case-tag / occupancy table (the Ec-dump mode, HBM-store bound).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "rpg_device.cuh"

using namespace rpg;

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxData = 64;  // data parameters D1..D64

// ---------------------------------------------------------------------------
// Shared-memory layout (dynamic), identical for both kernels.
struct SmemLayout {
  size_t coef, exps, mD, slots, xd, red, ec, wocc, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline SmemLayout smem_layout(int n_terms, int n_slots,
                                                  int n_space, bool ec_in_smem) {
  SmemLayout L;
  size_t o = 0;
  L.coef = o;  o = align16(o + sizeof(double) * (size_t)n_terms);
  L.exps = o;  o = align16(o + sizeof(uint64_t) * (size_t)n_terms);
  L.mD = o;    o = align16(o + sizeof(double) * (size_t)n_terms);
  L.slots = o; o = align16(o + sizeof(double) * (size_t)n_slots);
  L.xd = o;    o = align16(o + sizeof(double) * kMaxData);
  L.red = o;   o = align16(o + 32 * kWarps);
  if (ec_in_smem) {
    L.ec = o;   o = align16(o + sizeof(double) * (size_t)n_space);
    L.wocc = o; o = align16(o + sizeof(uint16_t) * (size_t)n_space);
  } else {
    L.ec = L.wocc = 0;
  }
  L.total = o;
  return L;
}

// ---------------------------------------------------------------------------
// Polynomial evaluation.

struct TupleCtx {
  const double* coef;   // smem
  const uint64_t* exps; // smem
  const double* mD;     // smem, per tuple
  const double* slots;  // smem, per tuple (FAST)
  const double* xd;     // smem, data-parameter values of the tuple
};

__device__ __forceinline__ double var_value(const Params& P, int v,
                                            const TupleCtx& T, double bx,
                                            double by, double bz) {
  int k = P.var_kind[v];
  return k == RPG_VAR_BX ? bx : k == RPG_VAR_BY ? by : k == RPG_VAR_BZ ? bz : T.xd[k];
}

// eval_poly in basis order with the data-parameter prefix hoisted per tuple:
// m_k = ((mD_k * p_{n_prefix}) * p_{n_prefix+1}) ..., acc = acc + c_k * m_k —
// the same rounding sequence as polyfit.hpp:96-119.
__device__ __forceinline__ double poly_exact(const Params& P, const PolyDesc& pd,
                                             const TupleCtx& T, double bx,
                                             double by, double bz) {
  double acc = 0.0;
  for (int k = pd.term_off; k < pd.term_off + pd.n_terms; ++k) {
    double m = T.mD[k];
    const uint64_t ex = T.exps[k];
    for (int v = P.n_prefix; v < P.n_vars; ++v) {
      int e = (int)((ex >> (8 * v)) & 0xff);
      if (e) m = __dmul_rn(m, ipow(var_value(P, v, T, bx, by, bz), e));
    }
    acc = __dadd_rn(acc, __dmul_rn(T.coef[k], m));
  }
  return acc;
}

// FAST: nested DFMA Horner over the collapsed per-pattern coefficients
// (restated in oracle/o1.c fast_poly).
__device__ __forceinline__ double poly_fast(const Params& P, const PolyDesc& pd,
                                            const TupleCtx& T, double x0,
                                            double x1, double x2) {
  const double* C = T.slots + pd.slot_off;
  const int s0 = pd.s0, s1 = pd.s1, s2 = pd.s2;
  double outer = 0.0;
  for (int a = s0 - 1; a >= 0; --a) {
    double mid = 0.0;
    for (int b = s1 - 1; b >= 0; --b) {
      const double* row = C + (a * s1 + b) * s2;
      double inner = row[s2 - 1];
      for (int c = s2 - 2; c >= 0; --c) inner = fma(inner, x2, row[c]);
      mid = (b == s1 - 1) ? inner : fma(mid, x1, inner);
    }
    outer = (a == s0 - 1) ? mid : fma(outer, x0, mid);
  }
  return outer;
}

template <bool FAST>
__device__ __forceinline__ PointOut eval_point(const Params& P, const TupleCtx& T,
                                               int64_t ibx, int64_t iby,
                                               int64_t ibz, bool want_tag) {
  const double bx = (double)ibx, by = (double)iby, bz = (double)ibz;
  double x0 = 0, x1 = 0, x2 = 0;
  if (FAST) {
    x0 = var_value(P, P.cfg_var[0], T, bx, by, bz);
    x1 = var_value(P, P.cfg_var[1], T, bx, by, bz);
    x2 = P.n_cfg_vars > 2 ? var_value(P, P.cfg_var[2], T, bx, by, bz) : 0.0;
  }
  double v[RPG_N_METRICS];
  bool den_zero = false, near_zero = false;
#pragma unroll
  for (int s = 0; s < RPG_N_METRICS; ++s) {
    const MetricDesc& md = P.metric[s];
    if (md.is_const) {
      v[s] = md.value;
      continue;
    }
    double p, q;
    if (FAST) {
      p = poly_fast(P, md.num, T, x0, x1, x2);
      q = md.den_is_one ? 1.0 : poly_fast(P, md.den, T, x0, x1, x2);
    } else {
      p = poly_exact(P, md.num, T, bx, by, bz);
      q = md.den_is_one ? 1.0 : poly_exact(P, md.den, T, bx, by, bz);
    }
    const double mag = fabs(p);
    if (fabs(q) < __dmul_rn(1e-12, mag > 1.0 ? mag : 1.0)) near_zero = true;
    if (q == 0.0) {
      den_zero = true;
      v[s] = 0.0;
    } else {
      v[s] = md.den_is_one ? p : __ddiv_rn(p, q);
    }
  }
  Metrics m;
  m.regs = v[RPG_METRIC_REGS];
  m.shared = v[RPG_METRIC_SHARED];
  m.comp = v[RPG_METRIC_COMP];
  m.uncoal = v[RPG_METRIC_UNCOAL];
  m.coal = v[RPG_METRIC_COAL];
  m.mem = __dadd_rn(m.uncoal, m.coal);
  m.synch = v[RPG_METRIC_SYNCH];
  m.tb = v[RPG_METRIC_TOTAL_BLOCKS];
  return finish_point(P, m, den_zero, near_zero, ibx, iby, ibz, want_tag);
}

// ---------------------------------------------------------------------------
// Per-CTA staging and per-tuple prologue.

__device__ __forceinline__ void stage_terms(const Params& P, double* coef,
                                            uint64_t* exps) {
  for (int k = threadIdx.x; k < P.n_terms; k += blockDim.x) {
    coef[k] = P.coef[k];
    exps[k] = P.exps[k];
  }
}

template <bool FAST>
__device__ __forceinline__ void tuple_prologue(const Params& P, const int64_t* data,
                                               int64_t t, TupleCtx& T, double* mD,
                                               double* slots, double* xd) {
  if (threadIdx.x < P.d && threadIdx.x < kMaxData)
    xd[threadIdx.x] = (double)data[t * P.d + threadIdx.x];
  __syncthreads();
  // mD_k: EXACT — product over the leading data variables (the shared prefix
  // of eval_monomial); FAST — product over every data variable.
  const int vend = FAST ? P.n_vars : P.n_prefix;
  for (int k = threadIdx.x; k < P.n_terms; k += blockDim.x) {
    const uint64_t ex = T.exps[k];
    double m = 1.0;
    for (int v = 0; v < vend; ++v) {
      int kind = P.var_kind[v];
      if (kind < 0) continue;
      int e = (int)((ex >> (8 * v)) & 0xff);
      double p = ipow(xd[kind], e);
      m = __dmul_rn(m, p);
    }
    mD[k] = m;
  }
  if (FAST) {
    __syncthreads();
    for (int s = threadIdx.x; s < P.n_slots; s += blockDim.x) {
      double c = 0.0;
      for (int j = P.slot_begin[s]; j < P.slot_begin[s + 1]; ++j) {
        int k = P.slot_terms[j];
        c = fma(T.coef[k], mD[k], c);
      }
      slots[s] = c;
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Block reductions.

__device__ __forceinline__ double block_min(double v, unsigned char* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  double* s = reinterpret_cast<double*>(red);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) s[w] = v;
  __syncthreads();
  double r = s[0];
  for (int i = 1; i < kWarps; ++i) r = fmin(r, s[i]);
  return r;
}

__device__ __forceinline__ int block_sum(int v, unsigned char* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int* s = reinterpret_cast<int*>(red);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) s[w] = v;
  __syncthreads();
  int r = 0;
  for (int i = 0; i < kWarps; ++i) r += s[i];
  return r;
}

struct Key {
  double ec;
  int32_t wocc, lex, idx;
};

// pipeline.hpp:654-669: within the tie group, higher occupancy first; the
// stable sort keeps (Ec, lex) order among equal occupancy.
__device__ __forceinline__ bool key_better(const Key& a, const Key& b) {
  if (a.wocc != b.wocc) return a.wocc > b.wocc;
  if (a.ec != b.ec) return a.ec < b.ec;
  if (a.lex != b.lex) return a.lex < b.lex;
  return a.idx < b.idx;
}

__device__ __forceinline__ Key block_best(Key k, unsigned char* red) {
  for (int o = 16; o > 0; o >>= 1) {
    Key other;
    other.ec = __shfl_xor_sync(0xffffffffu, k.ec, o);
    other.wocc = __shfl_xor_sync(0xffffffffu, k.wocc, o);
    other.lex = __shfl_xor_sync(0xffffffffu, k.lex, o);
    other.idx = __shfl_xor_sync(0xffffffffu, k.idx, o);
    if (key_better(other, k)) k = other;
  }
  Key* s = reinterpret_cast<Key*>(red);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) s[w] = k;
  __syncthreads();
  Key r = s[0];
  for (int i = 1; i < kWarps; ++i)
    if (key_better(s[i], r)) r = s[i];
  return r;
}

// ---------------------------------------------------------------------------
// Kernels.

template <bool FAST, bool EC_SMEM>
__global__ void __launch_bounds__(kThreads)
search_kernel(const Params P, const int64_t* __restrict__ data, int64_t n_tuples,
              rpg_winner* __restrict__ out, double* __restrict__ g_ec,
              uint16_t* __restrict__ g_wocc) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemLayout L = smem_layout(P.n_terms, P.n_slots, P.n_space, EC_SMEM);
  double* coef = reinterpret_cast<double*>(smem + L.coef);
  uint64_t* exps = reinterpret_cast<uint64_t*>(smem + L.exps);
  double* mD = reinterpret_cast<double*>(smem + L.mD);
  double* slots = reinterpret_cast<double*>(smem + L.slots);
  double* xd = reinterpret_cast<double*>(smem + L.xd);
  unsigned char* red = smem + L.red;
  double* ec_s = EC_SMEM ? reinterpret_cast<double*>(smem + L.ec)
                         : g_ec + (size_t)blockIdx.x * P.n_space;
  uint16_t* wocc_s = EC_SMEM ? reinterpret_cast<uint16_t*>(smem + L.wocc)
                             : g_wocc + (size_t)blockIdx.x * P.n_space;

  stage_terms(P, coef, exps);
  __syncthreads();
  TupleCtx T{coef, exps, mD, slots, xd};
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  const double pinf = __longlong_as_double(0x7ff0000000000000LL);

  for (int64_t t = blockIdx.x; t < n_tuples; t += gridDim.x) {
    tuple_prologue<FAST>(P, data, t, T, mD, slots, xd);

    // Pass 1: evaluate every config of this tuple.
    double lmin = pinf;
    int lfeas = 0;
    for (int c = threadIdx.x; c < P.n_space; c += kThreads) {
      const int4 cf = P.cfg[c];
      PointOut o = eval_point<FAST>(P, T, cf.x, cf.y, cf.z, false);
      ec_s[c] = o.feasible ? o.ec : qnan;
      wocc_s[c] = (uint16_t)o.w_occ;
      if (o.feasible) {
        ++lfeas;
        lmin = o.ec < lmin ? o.ec : lmin;
      }
    }
    const int nfeas = block_sum(lfeas, red);
    const double best = block_min(lmin, red);

    rpg_winner* w = out + t;
    if (nfeas == 0) {
      if (threadIdx.x == 0) {
        rpg_winner r;
        r.ec = 0.0;
        r.best_ec = 0.0;
        r.ties = 0;
        r.n_feasible = 0;
        r.b_active = r.w_active = r.w_occ = 0;
        r.reserved = 0;
        r.cfg_idx = -1;
        r.case_tag = RPG_CASE_UNKNOWN;
        *w = r;
      }
      __syncthreads();
      continue;
    }
    // Pass 2: the tie group and its winner (pipeline.hpp:660-669).
    const double bound = __dadd_rn(best, __dmul_rn(best, P.tie_rel_tol));
    Key k;
    k.ec = pinf;
    k.wocc = -1;
    k.lex = 0x7fffffff;
    k.idx = 0x7fffffff;
    int lties = 0;
    for (int c = threadIdx.x; c < P.n_space; c += kThreads) {
      const double v = ec_s[c];
      if (v <= bound) {
        ++lties;
        Key cand{v, (int32_t)wocc_s[c], P.cfg[c].w, c};
        if (key_better(cand, k)) k = cand;
      }
    }
    const int ties = block_sum(lties, red);
    const Key win = block_best(k, red);
    if (threadIdx.x == 0) {
      const int4 cf = P.cfg[win.idx];
      PointOut o = eval_point<FAST>(P, T, cf.x, cf.y, cf.z, true);
      rpg_winner r;
      r.ec = win.ec;
      r.best_ec = best;
      r.cfg_idx = win.idx;
      r.ties = ties;
      r.n_feasible = nfeas;
      r.b_active = o.b;
      r.w_active = o.w;
      r.w_occ = o.w_occ;
      r.case_tag = o.tag;
      r.reserved = 0;
      *w = r;
    }
    __syncthreads();
  }
}

template <bool FAST>
__global__ void __launch_bounds__(kThreads)
evaluate_kernel(const Params P, const int64_t* __restrict__ data, int64_t n_tuples,
                double* __restrict__ ec_out, uint8_t* __restrict__ tag_out,
                int32_t* __restrict__ wocc_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemLayout L = smem_layout(P.n_terms, P.n_slots, P.n_space, false);
  double* coef = reinterpret_cast<double*>(smem + L.coef);
  uint64_t* exps = reinterpret_cast<uint64_t*>(smem + L.exps);
  double* mD = reinterpret_cast<double*>(smem + L.mD);
  double* slots = reinterpret_cast<double*>(smem + L.slots);
  double* xd = reinterpret_cast<double*>(smem + L.xd);
  stage_terms(P, coef, exps);
  __syncthreads();
  TupleCtx T{coef, exps, mD, slots, xd};
  const bool want_tag = tag_out != nullptr;
  for (int64_t t = blockIdx.x; t < n_tuples; t += gridDim.x) {
    tuple_prologue<FAST>(P, data, t, T, mD, slots, xd);
    const size_t base = (size_t)t * P.n_space;
    for (int c = threadIdx.x; c < P.n_space; c += kThreads) {
      const int4 cf = P.cfg[c];
      PointOut o = eval_point<FAST>(P, T, cf.x, cf.y, cf.z, want_tag);
      if (ec_out) ec_out[base + c] = o.ec;
      if (tag_out) tag_out[base + c] = (uint8_t)o.tag;
      if (wocc_out) wocc_out[base + c] = o.w_occ;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Host side.

int set_err(char* err, size_t errlen, int code, const char* fmt, ...) {
  if (err && errlen) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, errlen, fmt, ap);
    va_end(ap);
  }
  return code;
}

#define CUDA_TRY(expr)                                                         \
  do {                                                                         \
    cudaError_t e_ = (expr);                                                   \
    if (e_ != cudaSuccess)                                                     \
      return set_err(err, errlen, RPG_E_CUDA, "%s: %s", #expr,                 \
                     cudaGetErrorString(e_));                                  \
  } while (0)

}  // namespace

struct rpg_plan {
  int device = 0;
  Params P{};
  int max_data_index = -1;  // highest D index the model reads (0-based)
  bool ec_smem = true;
  size_t smem_search = 0, smem_eval = 0;
  int grid_search = 0, grid_eval = 0;
  int sm_count = 0;
  // device buffers
  double* d_coef = nullptr;
  uint64_t* d_exps = nullptr;
  int32_t* d_slot_begin = nullptr;
  int32_t* d_slot_terms = nullptr;
  int4* d_cfg = nullptr;
  double* d_scratch_ec = nullptr;
  uint16_t* d_scratch_wocc = nullptr;
  // host-API staging
  std::mutex mu;
  cudaStream_t stream = nullptr;
  int64_t* d_data = nullptr;
  size_t d_data_cap = 0;
  void* d_out = nullptr;
  size_t d_out_cap = 0;
};

namespace {

int validate_profile(const rpg_profile* hw, char* err, size_t errlen) {
  const int64_t counts[] = {hw->R_max, hw->Z_max, hw->T_max, hw->B_max, hw->W_max,
                            hw->num_SM, hw->load_bytes_per_warp, hw->uncoal_per_mw};
  const char* cnames[] = {"R_max", "Z_max", "T_max", "B_max", "W_max",
                          "num_SM", "load_bytes_per_warp", "uncoal_per_mw"};
  for (int i = 0; i < 8; ++i)
    if (!(counts[i] > 0))
      return set_err(err, errlen, RPG_E_PROFILE, "profile: '%s' must be positive", cnames[i]);
  const double reals[] = {hw->freq_GHz, hw->mem_latency_cycles, hw->departure_del_coal_cycles,
                          hw->departure_del_uncoal_cycles, hw->mem_bandwidth_GBps,
                          hw->issue_cycles};
  const char* rnames[] = {"freq_GHz", "mem_latency_cycles", "departure_del_coal_cycles",
                          "departure_del_uncoal_cycles", "mem_bandwidth_GBps",
                          "issue_cycles"};
  for (int i = 0; i < 6; ++i)
    if (!(reals[i] > 0) || !std::isfinite(reals[i]))
      return set_err(err, errlen, RPG_E_PROFILE, "profile: '%s' must be positive", rnames[i]);
  if (hw->T_max > 1024)
    return set_err(err, errlen, RPG_E_PROFILE,
                   "T_max exceeds 1024, the architectural block limit");
  if (hw->W_max > 65535)
    return set_err(err, errlen, RPG_E_PROFILE, "profile: W_max above 65535 is not supported");
  return RPG_OK;
}

const char* metric_name(int s) {
  static const char* names[] = {"regs_per_thread", "shared_words_per_block",
                                "comp_insts_per_thread", "uncoal_mem_insts_per_thread",
                                "coal_mem_insts_per_thread", "synch_insts_per_block",
                                "total_blocks"};
  return names[s];
}

}  // namespace

extern "C" {

const char* rpg_version(void) { return "librpgpu 0.1.0 (sm_100a; ABI 1)"; }

int rpg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int rpg_plan_destroy(rpg_plan* plan) {
  if (!plan) return RPG_OK;
  cudaSetDevice(plan->device);
  if (plan->stream) cudaStreamSynchronize(plan->stream);
  cudaFree(plan->d_coef);
  cudaFree(plan->d_exps);
  cudaFree(plan->d_slot_begin);
  cudaFree(plan->d_slot_terms);
  cudaFree(plan->d_cfg);
  cudaFree(plan->d_scratch_ec);
  cudaFree(plan->d_scratch_wocc);
  cudaFree(plan->d_data);
  cudaFree(plan->d_out);
  if (plan->stream) cudaStreamDestroy(plan->stream);
  delete plan;
  return RPG_OK;
}

int rpg_plan_create(const rpg_model* model, const rpg_profile* hw,
                    const rpg_config* space, int64_t n_space,
                    const rpg_options* opts, int32_t device, rpg_plan** out,
                    char* err, size_t errlen) {
  if (!model || !hw || !opts || !out)
    return set_err(err, errlen, RPG_E_INVALID, "rpg_plan_create: null argument");
  *out = nullptr;
  if (n_space <= 0 || !space)
    return set_err(err, errlen, RPG_E_INVALID,
                   "search_optimal: configuration space is empty");
  if (n_space > (int64_t)0x7ffffff0)
    return set_err(err, errlen, RPG_E_INVALID, "configuration space too large");
  int rc = validate_profile(hw, err, errlen);
  if (rc) return rc;
  if (opts->rep_mode != RPG_REP_REAL && opts->rep_mode != RPG_REP_CEIL)
    return set_err(err, errlen, RPG_E_INVALID, "rep_mode must be real or ceil");
  if (opts->arith != RPG_ARITH_EXACT && opts->arith != RPG_ARITH_FAST)
    return set_err(err, errlen, RPG_E_INVALID, "arith must be exact or fast");
  const int nv = model->n_vars;
  if (nv < 1 || nv > RPG_MAX_VARS)
    return set_err(err, errlen, RPG_E_MODEL, "model must have 1..%d variables", RPG_MAX_VARS);

  Params P{};
  P.hw = *hw;
  P.rep_mode = opts->rep_mode;
  P.arith = opts->arith;
  P.tie_rel_tol = opts->tie_rel_tol;
  P.fb_regs = opts->regs_per_thread;
  P.fb_shared = opts->shared_words_per_block;
  P.n_vars = nv;
  bool has_bx = false, has_by = false, in_prefix = true;
  int max_d = -1;
  P.n_prefix = 0;
  P.n_cfg_vars = 0;
  for (int v = 0; v < nv; ++v) {
    int k = model->var_kind[v];
    P.var_kind[v] = k;
    if (k >= 0) {
      if (k >= 64)
        return set_err(err, errlen, RPG_E_MODEL, "data parameter D%d out of range", k + 1);
      max_d = std::max(max_d, k);
      if (in_prefix) ++P.n_prefix;
    } else {
      in_prefix = false;
      if (k == RPG_VAR_BX) has_bx = true;
      else if (k == RPG_VAR_BY) has_by = true;
      else if (k == RPG_VAR_BZ) P.has_bz = 1;
      else return set_err(err, errlen, RPG_E_MODEL, "bad variable kind %d", k);
      if (P.n_cfg_vars >= 3)
        return set_err(err, errlen, RPG_E_MODEL, "duplicate block dimension variable");
      P.cfg_var[P.n_cfg_vars++] = v;
    }
  }
  if (!has_bx || !has_by)
    return set_err(err, errlen, RPG_E_MODEL, "metric variables must include bx and by");

  // Terms, metric descriptors and (FAST) collapsed pattern slots.
  std::vector<double> coef;
  std::vector<uint64_t> exps;
  std::vector<int32_t> slot_begin{0}, slot_terms;
  auto add_poly = [&](const rpg_poly& p, PolyDesc& pd, int slot, const char* side) -> int {
    if (p.n_terms < 0 || (p.n_terms > 0 && (!p.coef || !p.exps)))
      return set_err(err, errlen, RPG_E_MODEL, "metric '%s' %s polynomial is malformed",
                     metric_name(slot), side);
    pd.term_off = (int32_t)coef.size();
    pd.n_terms = p.n_terms;
    int maxd[3] = {0, 0, 0};
    for (int k = 0; k < p.n_terms; ++k) {
      if (!std::isfinite(p.coef[k]))
        return set_err(err, errlen, RPG_E_MODEL, "metric '%s' has a non-finite coefficient",
                       metric_name(slot));
      uint64_t packed = 0;
      for (int v = 0; v < nv; ++v)
        packed |= (uint64_t)p.exps[(size_t)k * nv + v] << (8 * v);
      coef.push_back(p.coef[k]);
      exps.push_back(packed);
      for (int j = 0; j < P.n_cfg_vars; ++j)
        maxd[j] = std::max<int>(maxd[j], p.exps[(size_t)k * nv + P.cfg_var[j]]);
    }
    pd.s0 = maxd[0] + 1;
    pd.s1 = P.n_cfg_vars > 1 ? maxd[1] + 1 : 1;
    pd.s2 = P.n_cfg_vars > 2 ? maxd[2] + 1 : 1;
    pd.slot_off = (int32_t)slot_begin.size() - 1;
    const int n = pd.s0 * pd.s1 * pd.s2;
    if (pd.slot_off + n > kMaxCollapsed)
      return set_err(err, errlen, RPG_E_MODEL, "model too large for the FAST collapse");
    for (int s = 0; s < n; ++s) {
      const int a = s / (pd.s1 * pd.s2), b = (s / pd.s2) % pd.s1, c = s % pd.s2;
      for (int k = 0; k < p.n_terms; ++k) {
        const uint8_t* e = p.exps + (size_t)k * nv;
        const int ea = e[P.cfg_var[0]];
        const int eb = P.n_cfg_vars > 1 ? e[P.cfg_var[1]] : 0;
        const int ec = P.n_cfg_vars > 2 ? e[P.cfg_var[2]] : 0;
        if (ea == a && eb == b && ec == c) slot_terms.push_back(pd.term_off + k);
      }
      slot_begin.push_back((int32_t)slot_terms.size());
    }
    return RPG_OK;
  };
  for (int s = 0; s < RPG_N_METRICS; ++s) {
    const rpg_metric& m = model->metric[s];
    MetricDesc& md = P.metric[s];
    md.is_const = m.is_const ? 1 : 0;
    md.value = m.value;
    if (md.is_const) {
      if (!std::isfinite(m.value))
        return set_err(err, errlen, RPG_E_MODEL, "metric '%s' constant is not finite",
                       metric_name(s));
      continue;
    }
    if ((rc = add_poly(m.num, md.num, s, "numerator"))) return rc;
    if ((rc = add_poly(m.den, md.den, s, "denominator"))) return rc;
    bool one = m.den.n_terms == 1 && m.den.coef[0] == 1.0;
    for (int v = 0; one && v < nv; ++v) one = m.den.exps[v] == 0;
    md.den_is_one = one ? 1 : 0;
  }
  P.n_terms = (int32_t)coef.size();
  P.n_slots = (int32_t)slot_begin.size() - 1;

  // Configuration table: int4 {bx, by, bz, lex rank}.
  std::vector<int4> cfg((size_t)n_space);
  std::vector<int32_t> order((size_t)n_space);
  std::iota(order.begin(), order.end(), 0);
  for (int64_t i = 0; i < n_space; ++i) {
    const rpg_config& c = space[i];
    if (c.bx < INT32_MIN || c.bx > INT32_MAX || c.by < INT32_MIN || c.by > INT32_MAX ||
        c.bz < INT32_MIN || c.bz > INT32_MAX)
      return set_err(err, errlen, RPG_E_INVALID, "block dimension out of int32 range");
  }
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    const rpg_config &x = space[a], &y = space[b];
    if (x.bx != y.bx) return x.bx < y.bx;
    if (x.by != y.by) return x.by < y.by;
    return x.bz < y.bz;
  });
  for (int64_t r = 0; r < n_space; ++r) {
    const int32_t i = order[r];
    cfg[i] = make_int4((int)space[i].bx, (int)space[i].by, (int)space[i].bz, (int)r);
  }

  rpg_plan* plan = new rpg_plan();
  plan->device = device;
  plan->max_data_index = max_d;
  auto fail = [&](int code) {
    rpg_plan_destroy(plan);
    return code;
  };
  cudaError_t ce = cudaSetDevice(device);
  if (ce != cudaSuccess)
    return fail(set_err(err, errlen, RPG_E_CUDA, "cudaSetDevice(%d): %s", device,
                        cudaGetErrorString(ce)));
#define PLAN_CUDA(expr)                                                          \
  do {                                                                           \
    cudaError_t e_ = (expr);                                                     \
    if (e_ != cudaSuccess)                                                       \
      return fail(set_err(err, errlen, RPG_E_CUDA, "%s: %s", #expr,              \
                          cudaGetErrorString(e_)));                              \
  } while (0)
  PLAN_CUDA(cudaStreamCreateWithFlags(&plan->stream, cudaStreamNonBlocking));
  PLAN_CUDA(cudaDeviceGetAttribute(&plan->sm_count, cudaDevAttrMultiProcessorCount, device));
  const size_t nt = std::max<size_t>(coef.size(), 1);
  PLAN_CUDA(cudaMalloc(&plan->d_coef, sizeof(double) * nt));
  PLAN_CUDA(cudaMalloc(&plan->d_exps, sizeof(uint64_t) * nt));
  PLAN_CUDA(cudaMalloc(&plan->d_slot_begin, sizeof(int32_t) * slot_begin.size()));
  PLAN_CUDA(cudaMalloc(&plan->d_slot_terms, sizeof(int32_t) * std::max<size_t>(slot_terms.size(), 1)));
  PLAN_CUDA(cudaMalloc(&plan->d_cfg, sizeof(int4) * cfg.size()));
  if (!coef.empty()) {
    PLAN_CUDA(cudaMemcpy(plan->d_coef, coef.data(), sizeof(double) * coef.size(), cudaMemcpyHostToDevice));
    PLAN_CUDA(cudaMemcpy(plan->d_exps, exps.data(), sizeof(uint64_t) * exps.size(), cudaMemcpyHostToDevice));
  }
  PLAN_CUDA(cudaMemcpy(plan->d_slot_begin, slot_begin.data(), sizeof(int32_t) * slot_begin.size(), cudaMemcpyHostToDevice));
  if (!slot_terms.empty())
    PLAN_CUDA(cudaMemcpy(plan->d_slot_terms, slot_terms.data(), sizeof(int32_t) * slot_terms.size(), cudaMemcpyHostToDevice));
  PLAN_CUDA(cudaMemcpy(plan->d_cfg, cfg.data(), sizeof(int4) * cfg.size(), cudaMemcpyHostToDevice));
  P.coef = plan->d_coef;
  P.exps = plan->d_exps;
  P.slot_begin = plan->d_slot_begin;
  P.slot_terms = plan->d_slot_terms;
  P.cfg = plan->d_cfg;
  P.n_space = (int32_t)n_space;
  P.d = 0;

  // Launch geometry: Ec in SMEM when at least two CTAs still fit per SM.
  int smem_optin = 0;
  PLAN_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  const SmemLayout with_ec = smem_layout(P.n_terms, P.n_slots, P.n_space, true);
  const SmemLayout no_ec = smem_layout(P.n_terms, P.n_slots, P.n_space, false);
  if (no_ec.total > (size_t)smem_optin)
    return fail(set_err(err, errlen, RPG_E_MODEL, "model too large for shared memory"));
  plan->ec_smem = with_ec.total <= 100 * 1024;
  plan->smem_search = plan->ec_smem ? with_ec.total : no_ec.total;
  plan->smem_eval = no_ec.total;

  auto setup = [&](const void* fn, size_t smem, int* grid) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem);
    if (e != cudaSuccess) return e;
    *grid = std::max(1, per_sm) * plan->sm_count;
    return cudaSuccess;
  };
  const bool fast = P.arith == RPG_ARITH_FAST;
  const void* sk = fast ? (plan->ec_smem ? (const void*)search_kernel<true, true> : (const void*)search_kernel<true, false>)
                        : (plan->ec_smem ? (const void*)search_kernel<false, true> : (const void*)search_kernel<false, false>);
  const void* ek = fast ? (const void*)evaluate_kernel<true> : (const void*)evaluate_kernel<false>;
  PLAN_CUDA(setup(sk, plan->smem_search, &plan->grid_search));
  PLAN_CUDA(setup(ek, plan->smem_eval, &plan->grid_eval));
  if (!plan->ec_smem) {
    PLAN_CUDA(cudaMalloc(&plan->d_scratch_ec, sizeof(double) * (size_t)plan->grid_search * n_space));
    PLAN_CUDA(cudaMalloc(&plan->d_scratch_wocc, sizeof(uint16_t) * (size_t)plan->grid_search * n_space));
  }
  plan->P = P;
#undef PLAN_CUDA
  *out = plan;
  return RPG_OK;
}

}  // extern "C"

namespace {

int check_arity(const rpg_plan* plan, int32_t d, char* err, size_t errlen) {
  if (d < 0 || d > 64)
    return set_err(err, errlen, RPG_E_INVALID, "data arity %d out of range", d);
  if (plan->max_data_index >= d)
    return set_err(err, errlen, RPG_E_PIPELINE,
                   "program input 'D%d' has no value: %d data parameter(s) were given",
                   plan->max_data_index + 1, d);
  return RPG_OK;
}

int launch_search(rpg_plan* plan, const int64_t* d_data, int64_t n, int32_t d,
                  rpg_winner* d_out, cudaStream_t s, char* err, size_t errlen) {
  if (n <= 0) return RPG_OK;
  Params P = plan->P;
  P.d = d;
  const int grid = (int)std::min<int64_t>(n, plan->grid_search);
  const bool fast = P.arith == RPG_ARITH_FAST;
  if (fast) {
    if (plan->ec_smem)
      search_kernel<true, true><<<grid, kThreads, plan->smem_search, s>>>(P, d_data, n, d_out, nullptr, nullptr);
    else
      search_kernel<true, false><<<grid, kThreads, plan->smem_search, s>>>(P, d_data, n, d_out, plan->d_scratch_ec, plan->d_scratch_wocc);
  } else {
    if (plan->ec_smem)
      search_kernel<false, true><<<grid, kThreads, plan->smem_search, s>>>(P, d_data, n, d_out, nullptr, nullptr);
    else
      search_kernel<false, false><<<grid, kThreads, plan->smem_search, s>>>(P, d_data, n, d_out, plan->d_scratch_ec, plan->d_scratch_wocc);
  }
  CUDA_TRY(cudaGetLastError());
  return RPG_OK;
}

int launch_evaluate(rpg_plan* plan, const int64_t* d_data, int64_t n, int32_t d,
                    double* ec, uint8_t* tag, int32_t* wocc, cudaStream_t s,
                    char* err, size_t errlen) {
  if (n <= 0) return RPG_OK;
  Params P = plan->P;
  P.d = d;
  const int grid = (int)std::min<int64_t>(n, plan->grid_eval);
  if (P.arith == RPG_ARITH_FAST)
    evaluate_kernel<true><<<grid, kThreads, plan->smem_eval, s>>>(P, d_data, n, ec, tag, wocc);
  else
    evaluate_kernel<false><<<grid, kThreads, plan->smem_eval, s>>>(P, d_data, n, ec, tag, wocc);
  CUDA_TRY(cudaGetLastError());
  return RPG_OK;
}

template <typename T>
cudaError_t ensure(T** p, size_t* cap, size_t bytes) {
  if (*cap >= bytes) return cudaSuccess;
  cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), bytes);
  if (e == cudaSuccess) *cap = bytes;
  return e;
}

}  // namespace

extern "C" {

int rpg_search_batch_device(rpg_plan* plan, const int64_t* d_data, int64_t n_tuples,
                            int32_t d, rpg_winner* d_out, void* stream, char* err,
                            size_t errlen) {
  if (!plan) return set_err(err, errlen, RPG_E_INVALID, "null plan");
  int rc = check_arity(plan, d, err, errlen);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(plan->device));
  return launch_search(plan, d_data, n_tuples, d, d_out, (cudaStream_t)stream, err, errlen);
}

int rpg_search_batch(rpg_plan* plan, const int64_t* data, int64_t n_tuples, int32_t d,
                     rpg_winner* out, char* err, size_t errlen) {
  if (!plan) return set_err(err, errlen, RPG_E_INVALID, "null plan");
  int rc = check_arity(plan, d, err, errlen);
  if (rc) return rc;
  if (n_tuples <= 0) return RPG_OK;
  std::lock_guard<std::mutex> lock(plan->mu);
  CUDA_TRY(cudaSetDevice(plan->device));
  const size_t in_bytes = sizeof(int64_t) * (size_t)n_tuples * (size_t)std::max(d, 1);
  const size_t out_bytes = sizeof(rpg_winner) * (size_t)n_tuples;
  CUDA_TRY(ensure(&plan->d_data, &plan->d_data_cap, in_bytes));
  CUDA_TRY(ensure(reinterpret_cast<char**>(&plan->d_out), &plan->d_out_cap, out_bytes));
  if (d > 0)
    CUDA_TRY(cudaMemcpyAsync(plan->d_data, data, sizeof(int64_t) * (size_t)n_tuples * d,
                             cudaMemcpyHostToDevice, plan->stream));
  rc = launch_search(plan, plan->d_data, n_tuples, d, (rpg_winner*)plan->d_out, plan->stream,
                     err, errlen);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(out, plan->d_out, out_bytes, cudaMemcpyDeviceToHost, plan->stream));
  CUDA_TRY(cudaStreamSynchronize(plan->stream));
  return RPG_OK;
}

int rpg_evaluate_device(rpg_plan* plan, const int64_t* d_data, int64_t n_tuples, int32_t d,
                        double* d_ec, uint8_t* d_tag, int32_t* d_wocc, void* stream,
                        char* err, size_t errlen) {
  if (!plan) return set_err(err, errlen, RPG_E_INVALID, "null plan");
  int rc = check_arity(plan, d, err, errlen);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(plan->device));
  return launch_evaluate(plan, d_data, n_tuples, d, d_ec, d_tag, d_wocc,
                         (cudaStream_t)stream, err, errlen);
}

int rpg_evaluate(rpg_plan* plan, const int64_t* data, int64_t n_tuples, int32_t d,
                 double* ec, uint8_t* tag, int32_t* wocc, char* err, size_t errlen) {
  if (!plan) return set_err(err, errlen, RPG_E_INVALID, "null plan");
  int rc = check_arity(plan, d, err, errlen);
  if (rc) return rc;
  if (n_tuples <= 0) return RPG_OK;
  std::lock_guard<std::mutex> lock(plan->mu);
  CUDA_TRY(cudaSetDevice(plan->device));
  const size_t npts = (size_t)n_tuples * (size_t)plan->P.n_space;
  const size_t in_bytes = sizeof(int64_t) * (size_t)n_tuples * (size_t)std::max(d, 1);
  const size_t out_bytes = npts * (sizeof(double) + 1 + sizeof(int32_t)) + 64;
  CUDA_TRY(ensure(&plan->d_data, &plan->d_data_cap, in_bytes));
  CUDA_TRY(ensure(reinterpret_cast<char**>(&plan->d_out), &plan->d_out_cap, out_bytes));
  double* d_ec = reinterpret_cast<double*>(plan->d_out);
  int32_t* d_wocc = reinterpret_cast<int32_t*>(d_ec + npts);
  uint8_t* d_tag = reinterpret_cast<uint8_t*>(d_wocc + npts);
  if (d > 0)
    CUDA_TRY(cudaMemcpyAsync(plan->d_data, data, sizeof(int64_t) * (size_t)n_tuples * d,
                             cudaMemcpyHostToDevice, plan->stream));
  rc = launch_evaluate(plan, plan->d_data, n_tuples, d, ec ? d_ec : nullptr,
                       tag ? d_tag : nullptr, wocc ? d_wocc : nullptr, plan->stream, err,
                       errlen);
  if (rc) return rc;
  if (ec) CUDA_TRY(cudaMemcpyAsync(ec, d_ec, npts * sizeof(double), cudaMemcpyDeviceToHost, plan->stream));
  if (wocc) CUDA_TRY(cudaMemcpyAsync(wocc, d_wocc, npts * sizeof(int32_t), cudaMemcpyDeviceToHost, plan->stream));
  if (tag) CUDA_TRY(cudaMemcpyAsync(tag, d_tag, npts, cudaMemcpyDeviceToHost, plan->stream));
  CUDA_TRY(cudaStreamSynchronize(plan->stream));
  return RPG_OK;
}

int rpg_search(const rpg_model* model, const rpg_profile* hw, const rpg_config* space,
               int64_t n_space, const rpg_options* opts, const int64_t* data,
               int64_t n_tuples, int32_t d, int32_t device, rpg_winner* out, char* err,
               size_t errlen) {
  rpg_plan* plan = nullptr;
  int rc = rpg_plan_create(model, hw, space, n_space, opts, device, &plan, err, errlen);
  if (rc) return rc;
  rc = rpg_search_batch(plan, data, n_tuples, d, out, err, errlen);
  rpg_plan_destroy(plan);
  return rc;
}

}  // extern "C"
