// rpg_search.cu — plan management and the C ABI of librpgpu.so (include/rpg.h).
//
// A plan holds one rational program (metric spec), device profile and
// configuration space resident on one GPU: the polynomial term tables, the
// configuration table {bx, by, bz, lex rank}, the per-config occupancy table
// (when regs/shared are constants) and the kernels that evaluate it — the
// per-model specialized kernels (rpg_jit.cu, default) or the ahead-of-time
// generic kernels below.  Kernel bodies: rpg_kernels.cuh; point model:
// rpg_device.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "rpg_jit.h"
#include "rpg_kernels.cuh"

using namespace rpg;

namespace {

// ---------------------------------------------------------------------------
// Ahead-of-time generic kernels.

template <bool FAST>
__global__ void __launch_bounds__(kThreads)
generic_search(const __grid_constant__ Params P, const int64_t* __restrict__ data, int64_t n,
               rpg_winner* __restrict__ out) {
  search_body<FAST, GenericEval<FAST>>(P, data, n, out);
}

template <bool FAST>
__global__ void __launch_bounds__(kThreads)
generic_evaluate(const __grid_constant__ Params P, const int64_t* __restrict__ data, int64_t n,
                 double* __restrict__ ec, uint8_t* __restrict__ tag,
                 int32_t* __restrict__ wocc) {
  evaluate_body<FAST, GenericEval<FAST>>(P, data, n, ec, tag, wocc);
}

__global__ void occ_table_kernel(const __grid_constant__ Params P, int4* __restrict__ occ,
                                 double* __restrict__ rcp, int4* __restrict__ lean,
                                 double2* __restrict__ rep_tab) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < P.n_space) {
    const int4 cf = P.cfg[c];
    const int4 e = occ_entry(P, cf);
    occ[c] = e;
    const int b = e.x & 0xffff;
    // RN(1 / (b * num_SM)): the repetition denominator's reciprocal (RcpDiv).
    rcp[c] = b ? __ddiv_rn(1.0, (double)__int_as_float(e.w)) : 0.0;
    if (lean) {
      const int W = (int)((unsigned)e.x >> 16), bd = e.y & 0xffff, Wd = (int)((unsigned)e.y >> 16);
      lean[c] = make_int4(cf.x | (cf.y << 16), cf.z | (b << 16), (int)((unsigned)W | ((unsigned)Wd << 16)),
                          (bd == b && Wd == W) ? 1 : 0);
    }
  }
  if (rep_tab && c <= P.hw.B_max) {
    const double d = (double)c * (double)P.hw.num_SM;
    rep_tab[c] = make_double2(d, c ? __ddiv_rn(1.0, d) : 0.0);
  }
}

// One warp per (configuration, half): lane k of half h certifies binade
// 32 h + k (N in [2^(32h+k), 2^(32h+k+1)]) of configuration c.  Layout:
// cert[4c + m % 4] = mask of the binades where scan mode m (kScanFree,
// kScanCwp, kScanMwp, kScanBoth) is proven.
__global__ void __launch_bounds__(256) cm_cert_kernel(const __grid_constant__ Params P,
                                                      unsigned long long* __restrict__ cert) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int c = warp >> 1, half = warp & 1;
  if (c >= P.n_space) return;
  const int k = 32 * half + lane;
  const int4 rec = P.lean[c];
  const int b = (int)((unsigned)rec.y >> 16), W = rec.z & 0xffff;
  // The binade is proven piecewise: kCertPieces sub-boxes (exact bounds: the
  // width is a power of two) keep the enclosures' dependency overestimate
  // small; a mode holds on the binade iff it holds on every piece.
  constexpr int kCertPieces = 16;
  unsigned modes = 0u;
  if (k < 62) {
    const double* row = P.cm + (size_t)c * P.n_cm;
    const double lo = ldexp(1.0, k), step = ldexp(1.0, k - 4);
    modes = ~0u;
    for (int s = 0; s < kCertPieces && modes != 0u; ++s)
      modes &= cm_certify(P, row, b, W, lo + s * step, lo + (s + 1) * step);
  }
  unsigned* out = reinterpret_cast<unsigned*>(cert + 4 * (size_t)c);
  for (int m = kScanFree; m <= kScanBoth; ++m) {
    const unsigned bits = __ballot_sync(0xffffffffu, (modes >> m) & 1u);
    if (lane == 0) out[2 * (m % 4) + half] = bits;
  }
}

// RPG_ARITH_FAST_CM table: per configuration and metric polynomial, the
// coefficient of each power of D1, C_j = fma(c_k, mB_k, C_j) over the terms
// in basis order, mB_k = the product over the block variables in model
// order of x^e built by repeated multiplication (O1 fast_cm_poly).
__global__ void cm_table_kernel(const __grid_constant__ Params P, double* __restrict__ cm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)P.n_space * (2 * RPG_N_METRICS)) return;
  const int c = (int)(i / (2 * RPG_N_METRICS));
  const int s = (int)(i % (2 * RPG_N_METRICS)) >> 1, side = (int)(i & 1);
  double* row = cm + (size_t)c * P.n_cm;
  if (s == 0 && side == 0) {  // padding slots
    const int last = P.cm_deg[RPG_N_METRICS - 1][1];
    for (int j = P.cm_off[RPG_N_METRICS - 1][1] + (last >= 0 ? last + 1 : 0); j < P.n_cm; ++j)
      row[j] = 0.0;
  }
  const int deg = P.cm_deg[s][side];
  if (deg < 0) return;
  const PolyDesc pd = side ? P.metric[s].den : P.metric[s].num;
  const int4 cf = P.cfg[c];
  double C[16];
  for (int j = 0; j <= deg; ++j) C[j] = 0.0;
  for (int k = pd.term_off; k < pd.term_off + pd.n_terms; ++k) {
    const uint64_t ex = P.exps[k];
    double m = 1.0;
    int jd = 0;
    for (int v = 0; v < P.n_vars; ++v) {
      const int kind = P.var_kind[v];
      const int e = (int)((ex >> (8 * v)) & 0xff);
      if (kind >= 0) {
        jd = e;
        continue;
      }
      const double x = kind == RPG_VAR_BX ? (double)cf.x : kind == RPG_VAR_BY ? (double)cf.y
                                                                               : (double)cf.z;
      m = __dmul_rn(m, ipow(x, e));
    }
    C[jd] = fma(P.coef[k], m, C[jd]);
  }
  for (int j = 0; j <= deg; ++j) row[P.cm_off[s][side] + j] = C[j];
}

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

const char* metric_name(int s) {
  static const char* names[] = {"regs_per_thread", "shared_words_per_block",
                                "comp_insts_per_thread", "uncoal_mem_insts_per_thread",
                                "coal_mem_insts_per_thread", "synch_insts_per_block",
                                "total_blocks"};
  return names[s];
}

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
  if (hw->W_max > 16383 || hw->B_max > 4095 || hw->num_SM > 4095)
    return set_err(err, errlen, RPG_E_PROFILE,
                   "profile: W_max above 16383, B_max or num_SM above 4095 is not supported");
  return RPG_OK;
}

}  // namespace

struct rpg_plan {
  int device = 0;
  Params P{};
  bool fast = false;
  bool specialized = true;
  int max_data_index = -1;
  size_t smem = 0;
  int grid_search = 0, grid_eval = 0;
  int threads = kThreads;  // blockDim of the search / evaluate kernels
  int sm_count = 0;
  rpg_jit::Module jit;
  double* d_coef = nullptr;
  uint64_t* d_exps = nullptr;
  int32_t* d_slot_begin = nullptr;
  int32_t* d_slot_terms = nullptr;
  int4* d_cfg = nullptr;
  int4* d_occ = nullptr;
  double* d_occ_rcp = nullptr;
  int4* d_lean = nullptr;
  double2* d_rep_tab = nullptr;
  double* d_cm = nullptr;      // RPG_ARITH_FAST_CM per-configuration table
  unsigned long long* d_cert = nullptr;  // FAST_CM range certificate (cm_cert_kernel)
  int tuples_per_cta = 1;      // FAST_CM: 32 tuples (one per lane) per CTA
  // bare-program plans: first evaluation error (Params::err_flag)
  bool is_program = false;
  long long step_limit = 0;
  unsigned long long* d_err = nullptr;
  // host-API staging
  std::mutex mu;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // host-API D2H of finished chunks
  std::vector<cudaEvent_t> chunk_done;
  int64_t* d_data = nullptr;
  size_t d_data_cap = 0;
  void* d_out = nullptr;
  size_t d_out_cap = 0;
};

namespace {

// Hardware-only sub-expressions, evaluated once in the reference's operation
// order (perfmodel.hpp:324-327, 362-367).  This translation unit's host code
// is compiled with -ffp-contract=off.
void hoist_hardware(Params& P) {
  const rpg_profile& hw = P.hw;
  P.mlu = hw.mem_latency_cycles +
          ((double)hw.uncoal_per_mw - 1.0) * hw.departure_del_uncoal_cycles;
  P.bw_per_warp = hw.freq_GHz * (double)hw.load_bytes_per_warp / hw.mem_latency_cycles;
  P.mwp_peak = hw.mem_bandwidth_GBps / (P.bw_per_warp * (double)hw.num_SM);
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

const void* search_fn(const rpg_plan* plan) {
  if (plan->specialized) return reinterpret_cast<const void*>(plan->jit.search);
  return plan->fast ? reinterpret_cast<const void*>(generic_search<true>)
                    : reinterpret_cast<const void*>(generic_search<false>);
}

const void* evaluate_fn(const rpg_plan* plan) {
  if (plan->specialized) return reinterpret_cast<const void*>(plan->jit.evaluate);
  return plan->fast ? reinterpret_cast<const void*>(generic_evaluate<true>)
                    : reinterpret_cast<const void*>(generic_evaluate<false>);
}

}  // namespace

namespace {

struct ModelTables {
  std::vector<double> coef;
  std::vector<uint64_t> exps;
  std::vector<int32_t> slot_begin{0}, slot_terms;
  int max_d = -1;
};

// Validates the model against check_metric_spec's rules (perfmodel.hpp:
// 428-456) and lays out the term tables, metric descriptors and FAST
// collapse slots.
int prepare_model(const rpg_model* model, const rpg_profile* hw, const rpg_options* opts,
                  Params& P, ModelTables& tab, char* err, size_t errlen) {
  int rc = validate_profile(hw, err, errlen);
  if (rc) return rc;
  if (opts->rep_mode != RPG_REP_REAL && opts->rep_mode != RPG_REP_CEIL)
    return set_err(err, errlen, RPG_E_INVALID, "rep_mode must be real or ceil");
  if (opts->arith != RPG_ARITH_EXACT && opts->arith != RPG_ARITH_FAST &&
      opts->arith != RPG_ARITH_FAST_CM)
    return set_err(err, errlen, RPG_E_INVALID, "arith must be exact, fast or fast_cm");
  if (opts->kernel != RPG_KERNEL_SPECIALIZED && opts->kernel != RPG_KERNEL_GENERIC)
    return set_err(err, errlen, RPG_E_INVALID, "kernel must be specialized or generic");
  if (!std::isfinite(opts->tie_rel_tol) || opts->tie_rel_tol < 0.0)
    return set_err(err, errlen, RPG_E_INVALID, "tie_rel_tol must be finite and non-negative");
  P = Params{};
  P.hw = *hw;
  hoist_hardware(P);
  P.rep_mode = opts->rep_mode;
  P.arith = opts->arith;
  P.tie_rel_tol = opts->tie_rel_tol;
  P.fb_regs = opts->regs_per_thread;
  P.fb_shared = opts->shared_words_per_block;
  std::vector<double>& coef = tab.coef;
  std::vector<uint64_t>& exps = tab.exps;
  std::vector<int32_t>& slot_begin = tab.slot_begin;
  std::vector<int32_t>& slot_terms = tab.slot_terms;
  int& max_d = tab.max_d;
  const int nv = model->n_vars;
  if (nv < 1 || nv > RPG_MAX_VARS)
    return set_err(err, errlen, RPG_E_MODEL, "model must have 1..%d variables", RPG_MAX_VARS);

  P.n_vars = nv;
  bool has_bx = false, has_by = false, in_prefix = true;
  for (int v = 0; v < nv; ++v) {
    const int k = model->var_kind[v];
    P.var_kind[v] = k;
    if (k >= 0) {
      if (k >= kMaxData)
        return set_err(err, errlen, RPG_E_MODEL, "data parameter D%d out of range", k + 1);
      max_d = std::max(max_d, k);
      if (in_prefix) ++P.n_prefix;
    } else {
      in_prefix = false;
      if (k == RPG_VAR_BX) {
        if (has_bx) return set_err(err, errlen, RPG_E_MODEL, "duplicate variable bx");
        has_bx = true;
      } else if (k == RPG_VAR_BY) {
        if (has_by) return set_err(err, errlen, RPG_E_MODEL, "duplicate variable by");
        has_by = true;
      } else if (k == RPG_VAR_BZ) {
        if (P.has_bz) return set_err(err, errlen, RPG_E_MODEL, "duplicate variable bz");
        P.has_bz = 1;
      } else {
        return set_err(err, errlen, RPG_E_MODEL, "bad variable kind %d", k);
      }
      P.cfg_var[P.n_cfg_vars++] = v;
    }
  }
  if (!has_bx || !has_by)
    return set_err(err, errlen, RPG_E_MODEL, "metric variables must include bx and by");

  // Term tables, metric descriptors, FAST collapse slots.
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
      for (int v = 0; v < nv; ++v) packed |= (uint64_t)p.exps[(size_t)k * nv + v] << (8 * v);
      coef.push_back(p.coef[k]);
      exps.push_back(packed);
      for (int j = 0; j < P.n_cfg_vars; ++j)
        maxd[j] = std::max<int>(maxd[j], p.exps[(size_t)k * nv + P.cfg_var[j]]);
    }
    pd.s0 = maxd[0] + 1;
    pd.s1 = P.n_cfg_vars > 1 ? maxd[1] + 1 : 1;
    pd.s2 = P.n_cfg_vars > 2 ? maxd[2] + 1 : 1;
    // Even slot offsets: the specialized kernels read slot pairs (LDS.128).
    if ((slot_begin.size() - 1) % 2) slot_begin.push_back((int32_t)slot_terms.size());
    pd.slot_off = (int32_t)slot_begin.size() - 1;
    const int n = pd.s0 * pd.s1 * pd.s2;
    if (pd.slot_off + n > 8192)
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
  if ((slot_begin.size() - 1) % 2) slot_begin.push_back((int32_t)slot_terms.size());
  P.n_terms = (int32_t)coef.size();
  P.n_slots = (int32_t)slot_begin.size() - 1;
  P.occ_const = P.metric[RPG_METRIC_REGS].is_const && P.metric[RPG_METRIC_SHARED].is_const;

  if (P.arith == RPG_ARITH_FAST_CM) {
    // Configuration-major collapse: one data parameter (D1), one slot per
    // power of D1 up to the polynomial's degree in it (O1's fast_cm_poly).
    if (opts->kernel != RPG_KERNEL_SPECIALIZED)
      return set_err(err, errlen, RPG_E_INVALID, "arith fast_cm needs the specialized kernel");
    if (max_d > 0)
      return set_err(err, errlen, RPG_E_INVALID,
                     "arith fast_cm supports models with one data parameter (D1)");
    if (!P.occ_const)
      return set_err(err, errlen, RPG_E_INVALID,
                     "arith fast_cm needs constant register and shared-memory metrics");
    int off = 0;
    for (int s = 0; s < RPG_N_METRICS; ++s) {
      const MetricDesc& md = P.metric[s];
      for (int side = 0; side < 2; ++side) {
        P.cm_off[s][side] = off;
        P.cm_deg[s][side] = -1;
        if (md.is_const || (side == 1 && md.den_is_one)) continue;
        const PolyDesc& pd = side ? md.den : md.num;
        int deg = 0;
        for (int k = pd.term_off; k < pd.term_off + pd.n_terms; ++k)
          for (int v = 0; v < nv; ++v)
            if (P.var_kind[v] == 0) deg = std::max(deg, (int)((exps[k] >> (8 * v)) & 0xff));
        if (deg > 15)
          return set_err(err, errlen, RPG_E_MODEL, "arith fast_cm: degree in D1 above 15");
        P.cm_deg[s][side] = deg;
        off += deg + 1;
      }
    }
    P.n_cm = std::max(2, (off + 1) & ~1);  // even: rows are read as double2 pairs
    P.cm_lanes = std::min(rpg_jit::cm_tuples(), rpg_jit::cm_threads());
    P.cm_j = rpg_jit::cm_j();
    P.cm_scan = rpg_jit::cm_scan();
    if (!P.cm_scan && P.cm_j > 2) P.cm_j = 2;
  }
  return RPG_OK;
}

// The compact per-config record path of the specialized search kernels
// applies when occupancy is per-config (constant regs/shared) and the
// per-b repetition table is small; the block dimensions must also fit 16-bit
// fields (checked against the space in build_plan).
bool lean_eligible(const Params& P) {
  return P.occ_const && P.hw.B_max <= 1024 && P.hw.W_max <= 0xffff;
}

int check_space(const rpg_config* space, int64_t n_space, char* err, size_t errlen) {
  if (n_space <= 0 || !space)
    return set_err(err, errlen, RPG_E_INVALID, "search_optimal: configuration space is empty");
  if (n_space > (int64_t)0x7ffffff0)
    return set_err(err, errlen, RPG_E_INVALID, "configuration space too large");
  for (int64_t i = 0; i < n_space; ++i) {
    const rpg_config& c = space[i];
    if (c.bx < INT32_MIN || c.bx > INT32_MAX || c.by < INT32_MIN || c.by > INT32_MAX ||
        c.bz < INT32_MIN || c.bz > INT32_MAX)
      return set_err(err, errlen, RPG_E_INVALID, "block dimension out of int32 range");
  }
  return RPG_OK;
}

// Shared tail of plan creation: configuration table {bx, by, bz, lex rank},
// term tables, occupancy table, kernels (`jit` loads the specialized module)
// and launch geometry.
template <class Jit>
int build_plan(Params& P, const ModelTables& tab, const rpg_config* space, int64_t n_space,
               int32_t device, bool fast, bool specialized, bool is_program, const Jit& jit,
               rpg_plan** out, char* err, size_t errlen) {
  const std::vector<double>& coef = tab.coef;
  const std::vector<uint64_t>& exps = tab.exps;
  const std::vector<int32_t>& slot_begin = tab.slot_begin;
  const std::vector<int32_t>& slot_terms = tab.slot_terms;

  std::vector<int4> cfg((size_t)n_space);
  std::vector<int32_t> order((size_t)n_space);
  std::iota(order.begin(), order.end(), 0);
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
  plan->max_data_index = tab.max_d;
  plan->fast = fast;
  plan->specialized = specialized;
  plan->is_program = is_program;
  auto fail = [&](int code) {
    rpg_plan_destroy(plan);
    return code;
  };
#define PLAN_CUDA(expr)                                                          \
  do {                                                                           \
    cudaError_t e_ = (expr);                                                     \
    if (e_ != cudaSuccess)                                                       \
      return fail(set_err(err, errlen, RPG_E_CUDA, "%s: %s", #expr,              \
                          cudaGetErrorString(e_)));                              \
  } while (0)
  PLAN_CUDA(cudaSetDevice(device));
  PLAN_CUDA(cudaStreamCreateWithFlags(&plan->stream, cudaStreamNonBlocking));
  PLAN_CUDA(cudaStreamCreateWithFlags(&plan->copy_stream, cudaStreamNonBlocking));
  PLAN_CUDA(cudaDeviceGetAttribute(&plan->sm_count, cudaDevAttrMultiProcessorCount, device));
  const size_t nt = std::max<size_t>(coef.size(), 1);
  PLAN_CUDA(cudaMalloc(&plan->d_coef, sizeof(double) * nt));
  PLAN_CUDA(cudaMalloc(&plan->d_exps, sizeof(uint64_t) * nt));
  PLAN_CUDA(cudaMalloc(&plan->d_slot_begin, sizeof(int32_t) * slot_begin.size()));
  PLAN_CUDA(cudaMalloc(&plan->d_slot_terms, sizeof(int32_t) * std::max<size_t>(slot_terms.size(), 1)));
  PLAN_CUDA(cudaMalloc(&plan->d_cfg, sizeof(int4) * cfg.size()));
  PLAN_CUDA(cudaMalloc(&plan->d_occ, sizeof(int4) * cfg.size()));
  PLAN_CUDA(cudaMalloc(&plan->d_occ_rcp, sizeof(double) * cfg.size()));
  // Compact records of the specialized search pass: block dimensions and
  // occupancy must fit 16-bit fields, and the per-b repetition table SMEM.
  P.lean_ok = 0;
  if (specialized && !is_program && lean_eligible(P)) {
    bool fits = true;
    for (const int4& c : cfg) fits = fits && c.x >= 0 && c.x <= 0xffff && c.y >= 0 && c.y <= 0x7fff &&
                                     c.z >= 0 && c.z <= 0xffff;
    P.lean_ok = fits ? 1 : 0;
  }
  if (P.lean_ok) {
    PLAN_CUDA(cudaMalloc(&plan->d_lean, sizeof(int4) * cfg.size()));
    PLAN_CUDA(cudaMalloc(&plan->d_rep_tab, sizeof(double2) * (size_t)(P.hw.B_max + 1)));
  }
  PLAN_CUDA(cudaMalloc(&plan->d_err, sizeof(unsigned long long)));
  PLAN_CUDA(cudaMemset(plan->d_err, 0xff, sizeof(unsigned long long)));
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
  P.occ = plan->d_occ;
  P.occ_rcp = plan->d_occ_rcp;
  P.lean = plan->d_lean;
  P.rep_tab = plan->d_rep_tab;
  P.err_flag = plan->d_err;
  P.d = 0;
  if (P.arith == RPG_ARITH_FAST_CM) {
    if (!P.lean_ok)
      return fail(set_err(err, errlen, RPG_E_INVALID,
                          "arith fast_cm: block dimensions or occupancy limits out of range"));
    PLAN_CUDA(cudaMalloc(&plan->d_cm, sizeof(double) * (size_t)P.n_cm * (size_t)n_space));
    P.cm = plan->d_cm;
    const int64_t nthr = n_space * 2 * RPG_N_METRICS;
    cm_table_kernel<<<(int)((nthr + 255) / 256), 256, 0, plan->stream>>>(P, plan->d_cm);
    PLAN_CUDA(cudaGetLastError());
    plan->tuples_per_cta = P.cm_lanes * P.cm_j;
  }
  if (P.occ_const) {
    const int64_t nthr = std::max<int64_t>(n_space, P.lean_ok ? P.hw.B_max + 1 : 0);
    occ_table_kernel<<<(int)((nthr + 255) / 256), 256, 0, plan->stream>>>(
        P, plan->d_occ, plan->d_occ_rcp, plan->d_lean, plan->d_rep_tab);
    PLAN_CUDA(cudaGetLastError());
    if (P.arith == RPG_ARITH_FAST_CM && P.cm_scan && P.lean && rpg_jit::cm_cert()) {
      // the pass-1 range certificate: 64 binades of N per configuration
      PLAN_CUDA(cudaMalloc(&plan->d_cert, 4 * sizeof(unsigned long long) * (size_t)n_space));
      cm_cert_kernel<<<(int)((n_space * 64 + 255) / 256), 256, 0, plan->stream>>>(P, plan->d_cert);
      PLAN_CUDA(cudaGetLastError());
      P.cert = plan->d_cert;
    }
    PLAN_CUDA(cudaStreamSynchronize(plan->stream));
  }

  plan->smem = P.arith == RPG_ARITH_FAST_CM
                   ? std::max(cm_smem_bytes(P, rpg_jit::cm_threads() * P.cm_j), cm_eval_smem_bytes(P))
                   : smem_layout(smem_terms(P), P.n_slots, rep_entries(P)).total;
  int smem_optin = 0;
  PLAN_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  if (plan->smem > (size_t)smem_optin)
    return fail(set_err(err, errlen, RPG_E_MODEL, "model too large for shared memory"));
  if (plan->specialized) {
    std::string jerr;
    // Resident CTAs per SM the specialized kernels are register-budgeted for
    // (launch bounds); RPG_JIT_MIN_BLOCKS overrides it for tuning sweeps.
    const int threads = P.arith == RPG_ARITH_FAST_CM
                            ? rpg_jit::cm_threads()
                            : rpg_jit::jit_threads(!is_program && P.arith == RPG_ARITH_EXACT);
    const int min_blocks = P.arith == RPG_ARITH_FAST_CM ? rpg_jit::cm_min_blocks(threads, P.cm_j)
                                                      : rpg_jit::default_min_blocks(threads);
    if (jit(min_blocks, threads, &plan->jit, &jerr) != 0)
      return fail(set_err(err, errlen, RPG_E_CUDA, "%s", jerr.c_str()));
    plan->threads = threads;
  }
  auto setup = [&](const void* fn, int* grid) -> cudaError_t {
    // Only ever raise a function's dynamic-SMEM limit (under a lock):
    // plans of other models share the ahead-of-time kernels and may be
    // created concurrently (rpg_plan_group_create) — lowering the limit
    // under another plan's launch would fail it.
    cudaError_t e;
    {
      static std::mutex mu;
      static std::map<std::pair<const void*, int>, size_t> cur;
      std::lock_guard<std::mutex> lk(mu);
      size_t& c = cur[{fn, device}];
      e = plan->smem <= c ? cudaSuccess
                          : cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)plan->smem);
      if (e == cudaSuccess && plan->smem > c) c = plan->smem;
    }
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, plan->threads, plan->smem);
    if (e != cudaSuccess) return e;
    *grid = std::max(1, per_sm) * plan->sm_count;
    return cudaSuccess;
  };
  PLAN_CUDA(setup(search_fn(plan), &plan->grid_search));
  if (plan->specialized && plan->jit.search_alt) {
    int g = 0;
    PLAN_CUDA(setup(reinterpret_cast<const void*>(plan->jit.search_alt), &g));
  }
  PLAN_CUDA(setup(evaluate_fn(plan), &plan->grid_eval));
  plan->P = P;
#undef PLAN_CUDA
  *out = plan;
  return RPG_OK;
}

// Validates a bare program (include/rpg.h rpg_program) and builds its Params:
// no metric tables; the occupancy context of every row is opts regs/shared
// (pipeline.hpp:648-650), served by the constant-metric occupancy table.
int prepare_program(const rpg_program* prog, const rpg_profile* hw, const rpg_options* opts,
                    Params& P, ModelTables& tab, char* err, size_t errlen) {
  int rc = validate_profile(hw, err, errlen);
  if (rc) return rc;
  if (opts->rep_mode != RPG_REP_REAL && opts->rep_mode != RPG_REP_CEIL)
    return set_err(err, errlen, RPG_E_INVALID, "rep_mode must be real or ceil");
  if (prog->step_limit < 1)
    return set_err(err, errlen, RPG_E_INVALID, "step_limit must be >= 1");
  if (prog->n_instr < 1 || !prog->body)
    return set_err(err, errlen, RPG_E_INVALID, "empty program body");
  if (prog->n_slots < 1 || prog->n_slots > (1 << 20) || prog->n_literals < 0 ||
      (prog->n_literals > 0 && !prog->literals) || prog->n_inputs < 0 ||
      (prog->n_inputs > 0 && (!prog->input_slot || !prog->input_kind || !prog->input_fixed)))
    return set_err(err, errlen, RPG_E_INVALID, "malformed rpg_program");
  if (prog->output_slot < 0 || prog->output_slot >= prog->n_slots)
    return set_err(err, errlen, RPG_E_INVALID, "malformed rpg_program: output slot");
  for (int i = 0; i < prog->n_inputs; ++i) {
    const int s = prog->input_slot[i], k = prog->input_kind[i];
    if (s < 0 || s >= prog->n_slots)
      return set_err(err, errlen, RPG_E_INVALID, "malformed rpg_program: input slot");
    if (k >= kMaxData)
      return set_err(err, errlen, RPG_E_PIPELINE, "program input 'D%d' out of range", k + 1);
    if (k != RPG_VAR_BX && k != RPG_VAR_BY && k != RPG_VAR_BZ && k != RPG_INPUT_FIXED && k < 0)
      return set_err(err, errlen, RPG_E_INVALID, "malformed rpg_program: input kind %d", k);
    if (k == RPG_INPUT_FIXED && !std::isfinite(prog->input_fixed[i]))
      return set_err(err, errlen, RPG_E_INVALID, "malformed rpg_program: input value");
    if (k >= 0) tab.max_d = std::max(tab.max_d, k);
  }
  for (int i = 0; i < prog->n_instr; ++i) {
    const rpg_instr& in = prog->body[i];
    if (in.op < 0 || in.op > 13)
      return set_err(err, errlen, RPG_E_INVALID, "malformed rpg_program: opcode at %d", i);
    const int nops = (in.op == 0 || in.op == 1 || in.op == 11 || in.op == 13) ? 1
                     : in.op == 12                                          ? 0
                                                                            : 2;
    const int ops[2] = {in.a, in.b};
    for (int k = 0; k < nops; ++k)
      if (ops[k] >= prog->n_slots || (ops[k] < 0 && -1 - ops[k] >= prog->n_literals))
        return set_err(err, errlen, RPG_E_INVALID, "malformed rpg_program: operand at %d", i);
    if (in.op <= 10 && (in.target < 0 || in.target >= prog->n_slots))
      return set_err(err, errlen, RPG_E_INVALID, "malformed rpg_program: target at %d", i);
  }
  for (int i = 0; i < prog->n_literals; ++i)
    if (!std::isfinite(prog->literals[i]))
      return set_err(err, errlen, RPG_E_INVALID, "program literal %d is not finite as a double", i);

  if (!std::isfinite(opts->tie_rel_tol) || opts->tie_rel_tol < 0.0)
    return set_err(err, errlen, RPG_E_INVALID, "tie_rel_tol must be finite and non-negative");
  P = Params{};
  P.hw = *hw;
  hoist_hardware(P);
  P.rep_mode = opts->rep_mode;
  P.arith = RPG_ARITH_EXACT;
  P.tie_rel_tol = opts->tie_rel_tol;
  P.fb_regs = opts->regs_per_thread;
  P.fb_shared = opts->shared_words_per_block;
  P.n_vars = 0;
  for (int i = 0; i < prog->n_inputs; ++i)
    if (prog->input_kind[i] == RPG_VAR_BZ) P.has_bz = 1;
  for (int s = 0; s < RPG_N_METRICS; ++s) P.metric[s].is_const = 1;
  P.metric[RPG_METRIC_REGS].value = opts->regs_per_thread;
  P.metric[RPG_METRIC_SHARED].value = opts->shared_words_per_block;
  P.occ_const = 1;
  return RPG_OK;
}

// Reads and clears a program plan's error word (plan->mu held, stream idle).
int take_program_error(rpg_plan* plan, char* err, size_t errlen) {
  unsigned long long key = ~0ull;
  CUDA_TRY(cudaMemcpy(&key, plan->d_err, sizeof(key), cudaMemcpyDeviceToHost));
  if (key == ~0ull) return RPG_OK;
  CUDA_TRY(cudaMemset(plan->d_err, 0xff, sizeof(key)));
  const unsigned long long point = key >> 24;
  const long long t = (long long)(point / (unsigned long long)plan->P.n_space);
  const int c = (int)(point % (unsigned long long)plan->P.n_space);
  const int kind = (int)(key & 15), detail = (int)((key >> 4) & 0xfffff);
  char what[160];
  switch (kind) {
    case kProgErrFloorDiv: snprintf(what, sizeof(what), "floor_div: zero divisor"); break;
    case kProgErrCeilDiv: snprintf(what, sizeof(what), "ceil_div: zero divisor"); break;
    case kProgErrEuclidQuot: snprintf(what, sizeof(what), "euclid_quot: zero divisor"); break;
    case kProgErrEuclidRem: snprintf(what, sizeof(what), "euclid_rem: zero divisor"); break;
    case kProgErrStepLimit:
      snprintf(what, sizeof(what),
               "step limit of %lld instructions exceeded (possible non-termination)",
               (long long)plan->step_limit);
      break;
    case kProgErrFellOff: snprintf(what, sizeof(what), "control fell off the end of the program"); break;
    case kProgErrMissing:
      snprintf(what, sizeof(what), "no value bound for variable slot %d", detail);
      break;
    default: snprintf(what, sizeof(what), "program evaluation failed (code %d)", kind); break;
  }
  return set_err(err, errlen, RPG_E_EVAL, "%s [tuple %lld, configuration %d]", what, t, c);
}

}  // namespace

extern "C" {

const char* rpg_version(void) { return "librpgpu 0.2.0 (sm_100a; ABI 1)"; }

void rpg_jit_stats(int64_t* compiles, int64_t* disk_hits) {
  if (compiles) *compiles = rpg_jit::jit_compiles();
  if (disk_hits) *disk_hits = rpg_jit::jit_disk_hits();
}

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
  cudaFree(plan->d_occ);
  cudaFree(plan->d_occ_rcp);
  cudaFree(plan->d_lean);
  cudaFree(plan->d_cert);
  cudaFree(plan->d_rep_tab);
  cudaFree(plan->d_err);
  cudaFree(plan->d_data);
  cudaFree(plan->d_out);
  if (plan->stream) cudaStreamDestroy(plan->stream);
  if (plan->copy_stream) cudaStreamDestroy(plan->copy_stream);
  for (cudaEvent_t e : plan->chunk_done) cudaEventDestroy(e);
  if (plan->d_cm) cudaFree(plan->d_cm);
  delete plan;  // specialized modules stay cached for the process
  return RPG_OK;
}

int rpg_plan_create(const rpg_model* model, const rpg_profile* hw, const rpg_config* space,
                    int64_t n_space, const rpg_options* opts, int32_t device,
                    rpg_plan** out, char* err, size_t errlen) {
  if (!model || !hw || !opts || !out)
    return set_err(err, errlen, RPG_E_INVALID, "rpg_plan_create: null argument");
  *out = nullptr;
  Params P;
  ModelTables tab;
  int rc = check_space(space, n_space, err, errlen);
  if (rc) return rc;
  rc = prepare_model(model, hw, opts, P, tab, err, errlen);
  if (rc) return rc;
  const bool fast = P.arith == RPG_ARITH_FAST;
  return build_plan(P, tab, space, n_space, device, fast,
                    opts->kernel == RPG_KERNEL_SPECIALIZED, false,
                    [&](int min_blocks, int threads, rpg_jit::Module* m, std::string* jerr) {
                      return rpg_jit::get_module(P, tab.coef, tab.exps, fast, device,
                                                 min_blocks, threads, m, jerr);
                    },
                    out, err, errlen);
}

int rpg_program_plan_create(const rpg_program* prog, const rpg_profile* hw,
                            const rpg_config* space, int64_t n_space, const rpg_options* opts,
                            int32_t device, rpg_plan** out, char* err, size_t errlen) {
  if (!prog || !hw || !opts || !out)
    return set_err(err, errlen, RPG_E_INVALID, "rpg_program_plan_create: null argument");
  *out = nullptr;
  int rc = check_space(space, n_space, err, errlen);
  if (rc) return rc;
  Params P;
  ModelTables tab;
  if ((rc = prepare_program(prog, hw, opts, P, tab, err, errlen))) return rc;
  const rpg_program prog_copy = *prog;
  rc = build_plan(P, tab, space, n_space, device, false, true, true,
                  [&](int min_blocks, int threads, rpg_jit::Module* m, std::string* jerr) {
                    return rpg_jit::get_module_src(
                        rpg_jit::generate_program_source(prog_copy, P), device, min_blocks,
                        threads, m, jerr);
                  },
                  out, err, errlen);
  if (rc == RPG_OK) (*out)->step_limit = prog->step_limit;
  return rc;
}

int rpg_plan_poll_error(rpg_plan* plan, void* stream, char* err, size_t errlen) {
  if (!plan) return set_err(err, errlen, RPG_E_INVALID, "null plan");
  if (!plan->is_program) return RPG_OK;
  std::lock_guard<std::mutex> lock(plan->mu);
  CUDA_TRY(cudaSetDevice(plan->device));
  if (stream) CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return take_program_error(plan, err, errlen);
}

int rpg_plan_cert_counts(rpg_plan* plan, int64_t counts[256], char* err, size_t errlen) {
  if (!plan || !counts) return set_err(err, errlen, RPG_E_INVALID, "null plan or counts");
  for (int k = 0; k < 256; ++k) counts[k] = 0;
  if (!plan->d_cert) return RPG_OK;
  std::lock_guard<std::mutex> lock(plan->mu);
  CUDA_TRY(cudaSetDevice(plan->device));
  std::vector<unsigned long long> h(4 * (size_t)plan->P.n_space);
  CUDA_TRY(cudaMemcpy(h.data(), plan->d_cert, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
  static const int slot[4] = {kScanFree % 4, kScanCwp % 4, kScanMwp % 4, kScanBoth % 4};
  for (size_t c = 0; c < (size_t)plan->P.n_space; ++c)
    for (int m = 0; m < 4; ++m)
      for (int k = 0; k < 64; ++k) counts[64 * m + k] += (h[4 * c + slot[m]] >> k) & 1ull;
  return RPG_OK;
}

}  // extern "C"

namespace {

int check_arity(const rpg_plan* plan, int32_t d, char* err, size_t errlen) {
  if (d < 0 || d > kMaxData)
    return set_err(err, errlen, RPG_E_INVALID, "data arity %d out of range", d);
  if (plan->max_data_index >= d)
    return set_err(err, errlen, RPG_E_PIPELINE,
                   "program input 'D%d' has no value: %d data parameter(s) were given",
                   plan->max_data_index + 1, d);
  return RPG_OK;
}

// FAST_CM plans serve whole-space searches and evaluations (no subsets).
int check_not_cm(const rpg_plan* plan, const char* what, char* err, size_t errlen) {
  if (plan->P.arith == RPG_ARITH_FAST_CM)
    return set_err(err, errlen, RPG_E_INVALID, "%s: not available with arith fast_cm (whole-space searches and evaluations only)",
                   what);
  return RPG_OK;
}

int launch_search(rpg_plan* plan, const int64_t* d_data, int64_t n, int32_t d,
                  rpg_winner* d_out, cudaStream_t s, char* err, size_t errlen,
                  const int64_t* d_sub_off = nullptr, const int32_t* d_sub_list = nullptr) {
  if (n <= 0) return RPG_OK;
  Params P = plan->P;
  P.d = d;
  P.sub_off = d_sub_off;
  P.sub_list = d_sub_list;
  auto launch = [&](const void* fn, const int64_t* dd, int64_t cnt, rpg_winner* o,
                    int64_t per_unit) -> cudaError_t {
    const int64_t units = (cnt + per_unit - 1) / per_unit;
    const int grid = (int)std::min<int64_t>(units, plan->grid_search);
    void* args[] = {&P, &dd, &cnt, &o};
    return cudaLaunchKernel(fn, dim3(grid), dim3(plan->threads), args, plan->smem, s);
  };
  if (plan->specialized && plan->jit.search_alt) {
    // J = 3 (96-tuple groups) and the J = 2 alternate (64): the whole batch
    // with either, or the J = 3 full waves followed by the rest with J = 2,
    // whichever takes the fewest J = 3 wave-times — a J = 2 wave takes
    // (64 / 96) x 1.117 of one (rate(J=3) / rate(J=2) = 1.117 per full wave,
    // profiles/r02s3_j_sweep.txt).  The 1-GPU C2 step runs 4 J = 3 waves +
    // one J = 2 wave instead of 4.6 J = 3 waves; strong-scaled shards of it
    // on 2-8 GPUs run J = 2.
    const int64_t t3 = plan->tuples_per_cta, t2 = t3 / 3 * 2, g = plan->grid_search;
    const double w2 = (double)t2 / (double)t3 * 1.117;
    const int64_t full3 = n / (t3 * g) * (t3 * g), rest = n - full3;
    const double c_all3 = (double)((n + t3 * g - 1) / (t3 * g));
    const double c_all2 = w2 * (double)((n + t2 * g - 1) / (t2 * g));
    const double c_split = (double)(full3 / (t3 * g)) + w2 * (double)((rest + t2 * g - 1) / (t2 * g));
    const void* alt = reinterpret_cast<const void*>(plan->jit.search_alt);
    if (c_split < c_all3 && c_split <= c_all2 && full3 > 0 && rest > 0) {
      CUDA_TRY(launch(search_fn(plan), d_data, full3, d_out, t3));
      CUDA_TRY(launch(alt, d_data + full3 * d, rest, d_out + full3, t2));
    } else if (c_all2 < c_all3) {
      CUDA_TRY(launch(alt, d_data, n, d_out, t2));
    } else {
      CUDA_TRY(launch(search_fn(plan), d_data, n, d_out, t3));
    }
    return RPG_OK;
  }
  CUDA_TRY(launch(search_fn(plan), d_data, n, d_out, plan->tuples_per_cta));
  return RPG_OK;
}

int launch_evaluate(rpg_plan* plan, const int64_t* d_data, int64_t n, int32_t d, double* ec,
                    uint8_t* tag, int32_t* wocc, cudaStream_t s, char* err, size_t errlen) {
  if (n <= 0) return RPG_OK;
  Params P = plan->P;
  P.d = d;
  int64_t units = n;
  if (P.arith == RPG_ARITH_FAST_CM)  // evaluate_body_cm tiles: 32 configs x (warps x 4) tuples
    units = (P.n_space + 31) / 32 *
            ((n + (plan->threads / 32) * kCmEvalTuplesPerWarp - 1) / ((plan->threads / 32) * kCmEvalTuplesPerWarp));
  const int grid = (int)std::min<int64_t>(units, plan->grid_eval);
  void* args[] = {&P, &d_data, &n, &ec, &tag, &wocc};
  CUDA_TRY(cudaLaunchKernel(evaluate_fn(plan), dim3(grid), dim3(plan->threads), args, plan->smem, s));
  return RPG_OK;
}

}  // namespace

extern "C" {

int rpg_search_batch_device(rpg_plan* plan, const int64_t* d_data, int64_t n_tuples, int32_t d,
                            rpg_winner* d_out, void* stream, char* err, size_t errlen) {
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
  if (plan->is_program)
    CUDA_TRY(cudaMemsetAsync(plan->d_err, 0xff, sizeof(unsigned long long), plan->stream));
  // Large batches run as chunks of whole persistent-grid waves so the D2H of
  // a finished chunk overlaps the kernels of the next ones (no extra tail:
  // every chunk but the last is an exact multiple of the resident grid).
  const int64_t chunk = 4LL * std::max(1, plan->grid_search) * plan->tuples_per_cta;
  const int64_t n_chunks = plan->is_program ? 1 : std::max<int64_t>(1, std::min<int64_t>(8, n_tuples / chunk));
  if (n_chunks <= 1) {
    rc = launch_search(plan, plan->d_data, n_tuples, d, (rpg_winner*)plan->d_out, plan->stream,
                       err, errlen);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(out, plan->d_out, out_bytes, cudaMemcpyDeviceToHost, plan->stream));
    CUDA_TRY(cudaStreamSynchronize(plan->stream));
    return plan->is_program ? take_program_error(plan, err, errlen) : RPG_OK;
  }
  // Chunks of `chunk` tuples, the remainder folded into the second-to-last
  // chunk, and a last chunk of one wave so the only exposed copy is small.
  const int64_t wave = (int64_t)std::max(1, plan->grid_search) * plan->tuples_per_cta;
  int64_t lo[10], cnt[10];
  int64_t nc = 0;
  for (int64_t at = 0; at < n_tuples;) {
    const int64_t left = n_tuples - at;
    int64_t take = left <= wave ? left : (left < chunk + 2 * wave ? left - wave : chunk);
    if (nc == 8) take = left;
    lo[nc] = at;
    cnt[nc] = take;
    ++nc;
    at += take;
  }
  while ((int64_t)plan->chunk_done.size() < nc) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    plan->chunk_done.push_back(e);
  }
  rpg_winner* d_out = (rpg_winner*)plan->d_out;
  for (int64_t i = 0; i < nc; ++i) {
    rc = launch_search(plan, plan->d_data + lo[i] * d, cnt[i], d, d_out + lo[i], plan->stream, err,
                       errlen);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(plan->chunk_done[i], plan->stream));
  }
  for (int64_t i = 0; i < nc; ++i) {
    CUDA_TRY(cudaStreamWaitEvent(plan->copy_stream, plan->chunk_done[i], 0));
    CUDA_TRY(cudaMemcpyAsync(out + lo[i], d_out + lo[i], sizeof(rpg_winner) * (size_t)cnt[i],
                             cudaMemcpyDeviceToHost, plan->copy_stream));
  }
  CUDA_TRY(cudaStreamSynchronize(plan->copy_stream));
  CUDA_TRY(cudaStreamSynchronize(plan->stream));
  return RPG_OK;
}

int rpg_evaluate_device(rpg_plan* plan, const int64_t* d_data, int64_t n_tuples, int32_t d,
                        double* d_ec, uint8_t* d_tag, int32_t* d_wocc, void* stream, char* err,
                        size_t errlen) {
  if (!plan) return set_err(err, errlen, RPG_E_INVALID, "null plan");
  int rc = check_arity(plan, d, err, errlen);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(plan->device));
  return launch_evaluate(plan, d_data, n_tuples, d, d_ec, d_tag, d_wocc, (cudaStream_t)stream,
                         err, errlen);
}

int rpg_evaluate(rpg_plan* plan, const int64_t* data, int64_t n_tuples, int32_t d, double* ec,
                 uint8_t* tag, int32_t* wocc, char* err, size_t errlen) {
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
  if (plan->is_program)
    CUDA_TRY(cudaMemsetAsync(plan->d_err, 0xff, sizeof(unsigned long long), plan->stream));
  rc = launch_evaluate(plan, plan->d_data, n_tuples, d, ec ? d_ec : nullptr,
                       tag ? d_tag : nullptr, wocc ? d_wocc : nullptr, plan->stream, err, errlen);
  if (rc) return rc;
  if (ec) CUDA_TRY(cudaMemcpyAsync(ec, d_ec, npts * sizeof(double), cudaMemcpyDeviceToHost, plan->stream));
  if (wocc) CUDA_TRY(cudaMemcpyAsync(wocc, d_wocc, npts * sizeof(int32_t), cudaMemcpyDeviceToHost, plan->stream));
  if (tag) CUDA_TRY(cudaMemcpyAsync(tag, d_tag, npts, cudaMemcpyDeviceToHost, plan->stream));
  CUDA_TRY(cudaStreamSynchronize(plan->stream));
  return plan->is_program ? take_program_error(plan, err, errlen) : RPG_OK;
}

// Host-side check of a CSR subset description (offsets[0] = 0,
// non-decreasing, entries in range and distinct per tuple).
static int check_subsets(const rpg_plan* plan, int64_t n_tuples, const int64_t* off,
                         const int32_t* list, char* err, size_t errlen) {
  if (!off || (off[n_tuples] > 0 && !list))
    return set_err(err, errlen, RPG_E_INVALID, "subsets: null offsets or list");
  if (off[0] != 0) return set_err(err, errlen, RPG_E_INVALID, "subsets: offsets[0] must be 0");
  std::vector<int64_t> seen((size_t)plan->P.n_space, -1);
  for (int64_t t = 0; t < n_tuples; ++t) {
    if (off[t + 1] < off[t])
      return set_err(err, errlen, RPG_E_INVALID, "subsets: offsets must be non-decreasing");
    if (off[t + 1] - off[t] > plan->P.n_space)
      return set_err(err, errlen, RPG_E_INVALID, "subsets: tuple %lld lists more configurations "
                     "than the space holds", (long long)t);
    for (int64_t k = off[t]; k < off[t + 1]; ++k) {
      const int32_t c = list[k];
      if (c < 0 || c >= plan->P.n_space)
        return set_err(err, errlen, RPG_E_INVALID, "subsets: configuration index %d out of range", c);
      if (seen[(size_t)c] == t)
        return set_err(err, errlen, RPG_E_INVALID, "subsets: configuration %d listed twice for "
                       "tuple %lld", c, (long long)t);
      seen[(size_t)c] = t;
    }
  }
  return RPG_OK;
}

int rpg_search_batch_subsets_device(rpg_plan* plan, const int64_t* d_data, int64_t n_tuples,
                                    int32_t d, const int64_t* d_offsets, const int32_t* d_list,
                                    rpg_winner* d_out, void* stream, char* err, size_t errlen) {
  if (!plan) return set_err(err, errlen, RPG_E_INVALID, "null plan");
  int rc = check_arity(plan, d, err, errlen);
  if (rc) return rc;
  if ((rc = check_not_cm(plan, "rpg_search_batch_subsets_device", err, errlen))) return rc;
  CUDA_TRY(cudaSetDevice(plan->device));
  return launch_search(plan, d_data, n_tuples, d, d_out, (cudaStream_t)stream, err, errlen,
                       d_offsets, d_list);
}

int rpg_search_batch_subsets(rpg_plan* plan, const int64_t* data, int64_t n_tuples, int32_t d,
                             const int64_t* offsets, const int32_t* list, rpg_winner* out,
                             char* err, size_t errlen) {
  if (!plan) return set_err(err, errlen, RPG_E_INVALID, "null plan");
  int rc = check_arity(plan, d, err, errlen);
  if (rc) return rc;
  if ((rc = check_not_cm(plan, "rpg_search_batch_subsets", err, errlen))) return rc;
  if (n_tuples <= 0) return RPG_OK;
  if ((rc = check_subsets(plan, n_tuples, offsets, list, err, errlen))) return rc;
  std::lock_guard<std::mutex> lock(plan->mu);
  CUDA_TRY(cudaSetDevice(plan->device));
  const int64_t n_list = offsets[n_tuples];
  const size_t in_bytes = sizeof(int64_t) * (size_t)n_tuples * (size_t)std::max(d, 1);
  const size_t out_bytes = sizeof(rpg_winner) * (size_t)n_tuples;
  const size_t off_bytes = sizeof(int64_t) * (size_t)(n_tuples + 1);
  const size_t list_bytes = sizeof(int32_t) * (size_t)std::max<int64_t>(n_list, 1);
  CUDA_TRY(ensure(&plan->d_data, &plan->d_data_cap, in_bytes));
  CUDA_TRY(ensure(reinterpret_cast<char**>(&plan->d_out), &plan->d_out_cap,
                  out_bytes + off_bytes + list_bytes + 16));
  char* base = reinterpret_cast<char*>(plan->d_out);
  int64_t* d_off = reinterpret_cast<int64_t*>(base + ((out_bytes + 7) & ~(size_t)7));
  int32_t* d_list = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(d_off) + off_bytes);
  if (d > 0)
    CUDA_TRY(cudaMemcpyAsync(plan->d_data, data, sizeof(int64_t) * (size_t)n_tuples * d,
                             cudaMemcpyHostToDevice, plan->stream));
  CUDA_TRY(cudaMemcpyAsync(d_off, offsets, off_bytes, cudaMemcpyHostToDevice, plan->stream));
  if (n_list > 0)
    CUDA_TRY(cudaMemcpyAsync(d_list, list, sizeof(int32_t) * (size_t)n_list,
                             cudaMemcpyHostToDevice, plan->stream));
  if (plan->is_program)
    CUDA_TRY(cudaMemsetAsync(plan->d_err, 0xff, sizeof(unsigned long long), plan->stream));
  rc = launch_search(plan, plan->d_data, n_tuples, d, (rpg_winner*)plan->d_out, plan->stream,
                     err, errlen, d_off, d_list);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(out, plan->d_out, out_bytes, cudaMemcpyDeviceToHost, plan->stream));
  CUDA_TRY(cudaStreamSynchronize(plan->stream));
  return plan->is_program ? take_program_error(plan, err, errlen) : RPG_OK;
}

int rpg_search(const rpg_model* model, const rpg_profile* hw, const rpg_config* space,
               int64_t n_space, const rpg_options* opts, const int64_t* data, int64_t n_tuples,
               int32_t d, int32_t device, rpg_winner* out, char* err, size_t errlen) {
  rpg_plan* plan = nullptr;
  int rc = rpg_plan_create(model, hw, space, n_space, opts, device, &plan, err, errlen);
  if (rc) return rc;
  rc = rpg_search_batch(plan, data, n_tuples, d, out, err, errlen);
  rpg_plan_destroy(plan);
  return rc;
}

}  // extern "C"

extern "C" int64_t rpg_emit_cuda_source(const rpg_model* model, const rpg_profile* hw,
                                        const rpg_options* opts, int32_t compile, char* buf,
                                        size_t buflen, int64_t* cubin_bytes, char* err,
                                        size_t errlen) {
  if (!model || !hw || !opts)
    return set_err(err, errlen, RPG_E_INVALID, "rpg_emit_cuda_source: null argument");
  Params P;
  ModelTables tab;
  int rc = prepare_model(model, hw, opts, P, tab, err, errlen);
  if (rc) return rc;
  P.lean_ok = opts->kernel == RPG_KERNEL_SPECIALIZED && lean_eligible(P);  // as for a plan whose space fits
  const std::string src =
      rpg_jit::generate_source(P, tab.coef, tab.exps, opts->arith == RPG_ARITH_FAST,
                               getenv("RPG_JIT_ILP") && atoi(getenv("RPG_JIT_ILP")) == 2);
  if (buf && buflen) {
    const size_t n = std::min(buflen - 1, src.size());
    memcpy(buf, src.data(), n);
    buf[n] = '\0';
  }
  if (compile) {
    std::vector<char> cubin;
    std::string log;
    const bool cm = opts->arith == RPG_ARITH_FAST_CM;
    const int threads = cm ? rpg_jit::cm_threads() : rpg_jit::jit_threads(opts->arith == RPG_ARITH_EXACT);
    const int mb = cm ? rpg_jit::cm_min_blocks(threads, P.cm_j) : rpg_jit::default_min_blocks(threads);
    if (rpg_jit::compile(src, mb, threads, &cubin, &log) != 0)
      return set_err(err, errlen, RPG_E_CUDA, "NVRTC: %s", log.substr(0, 1500).c_str());
    if (cubin_bytes) *cubin_bytes = (int64_t)cubin.size();
  }
  return (int64_t)src.size();
}

extern "C" int64_t rpg_emit_program_cuda_source(const rpg_program* prog, const rpg_profile* hw,
                                                const rpg_options* opts, int32_t compile,
                                                char* buf, size_t buflen, int64_t* cubin_bytes,
                                                char* err, size_t errlen) {
  if (!prog || !hw || !opts)
    return set_err(err, errlen, RPG_E_INVALID, "rpg_emit_program_cuda_source: null argument");
  Params P;
  ModelTables tab;
  int rc = prepare_program(prog, hw, opts, P, tab, err, errlen);
  if (rc) return rc;
  const std::string src = rpg_jit::generate_program_source(*prog, P);
  if (buf && buflen) {
    const size_t n = std::min(buflen - 1, src.size());
    memcpy(buf, src.data(), n);
    buf[n] = '\0';
  }
  if (compile) {
    std::vector<char> cubin;
    std::string log;
    const int threads = rpg_jit::jit_threads(false);
    if (rpg_jit::compile(src, rpg_jit::default_min_blocks(threads), threads, &cubin, &log) != 0)
      return set_err(err, errlen, RPG_E_CUDA, "NVRTC: %s", log.substr(0, 1500).c_str());
    if (cubin_bytes) *cubin_bytes = (int64_t)cubin.size();
  }
  return (int64_t)src.size();
}

// ---------------------------------------------------------------------------
// perf::mwpcwp_cycles over a batch of (metrics, configuration) rows — the
// "collected" side of sanity_report (pipeline.hpp:797-814) and any caller of
// the direct model.  IEEE arithmetic in the reference's operation order.
namespace {

__global__ void direct_cycles_kernel(const Params P, const double* __restrict__ metrics,
                                     const rpg_config* __restrict__ cfgs, int64_t n,
                                     double* __restrict__ total, int32_t* __restrict__ b_out,
                                     int32_t* __restrict__ w_out, uint8_t* __restrict__ tag_out,
                                     int32_t* __restrict__ status) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* mv = metrics + i * RPG_N_METRICS;
    Metrics m;
    m.regs = mv[RPG_METRIC_REGS];
    m.shared = mv[RPG_METRIC_SHARED];
    m.comp = mv[RPG_METRIC_COMP];
    m.uncoal = mv[RPG_METRIC_UNCOAL];
    m.coal = mv[RPG_METRIC_COAL];
    m.mem = __dadd_rn(m.uncoal, m.coal);  // metrics_from_sample (pipeline.hpp:746-747)
    m.synch = mv[RPG_METRIC_SYNCH];
    m.tb = mv[RPG_METRIC_TOTAL_BLOCKS];
    int st = 0, tag = RPG_CASE_UNKNOWN;
    int64_t b = 0, W = 0;
    double ec = 0.0;
    // perfmodel.hpp:302-310
    const double chk = __dadd_rn(__dadd_rn(m.uncoal, m.coal), -m.mem);
    if (fabs(chk) > __dmul_rn(1e-9, m.mem > 1.0 ? m.mem : 1.0)) st = 3;
    else if (metrics_negative(m)) st = 2;
    if (!st) {
      const rpg_config c = cfgs[i];
      const int64_t T = c.bx * c.by * c.bz;
      b = active_blocks(P.hw, m.regs, m.shared, T, false);
      W = b ? active_warps(P.hw, b, T) : 0;
      if (b == 0 || W == 0) {
        st = 1;
      } else {
        bool ok = true;
        ec = mwpcwp_core<IeeeDiv>(P, m, b, W, false, &tag, ok);
      }
    }
    if (total) total[i] = ec;
    if (b_out) b_out[i] = (int32_t)b;
    if (w_out) w_out[i] = (int32_t)W;
    if (tag_out) tag_out[i] = (uint8_t)tag;
    if (status) status[i] = st;
  }
}

// perf::mwpcwp_cycles with the full breakdown; rows in KernelMetrics field
// order (perfmodel.hpp:68-77).  Checks in the reference's order
// (perfmodel.hpp:302-320).
__global__ void breakdown_kernel(const Params P, const double* __restrict__ km,
                                 const rpg_config* __restrict__ cfgs, int64_t n,
                                 rpg_breakdown* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* mv = km + i * 8;
    Metrics m;
    m.regs = mv[0];
    m.shared = mv[1];
    m.comp = mv[2];
    m.mem = mv[3];
    m.uncoal = mv[4];
    m.coal = mv[5];
    m.synch = mv[6];
    m.tb = mv[7];
    rpg_breakdown o;
    o.b_active = o.n_active_warps = 0;
    o.mem_cycles = o.comp_cycles = o.mwp = o.cwp = o.rep = 0.0;
    o.cycles_pre_synch = o.synch_cost = o.total_cycles = 0.0;
    o.case_tag = RPG_CASE_CWP_BOUND;
    o.status = 0;
    const double chk = __dadd_rn(__dadd_rn(m.uncoal, m.coal), -m.mem);
    if (fabs(chk) > __dmul_rn(1e-9, m.mem > 1.0 ? m.mem : 1.0)) {
      o.status = 3;
    } else if (metrics_negative(m)) {
      o.status = 2;
    } else {
      const rpg_config c = cfgs[i];
      const int64_t T = c.bx * c.by * c.bz;
      const int64_t b = active_blocks(P.hw, m.regs, m.shared, T, false);
      const int64_t W = b ? active_warps(P.hw, b, T) : 0;
      o.b_active = b;
      o.n_active_warps = W;
      if (b == 0) o.status = 1;
      else if (W == 0) o.status = 4;
      else mwpcwp_breakdown(P, m, b, W, o);
    }
    out[i] = o;
  }
}

// poly::eval_ratfunc (polyfit.hpp:96-130) over m points: basis-order
// products and sums, DenominatorNearZero flagged (status 1).
__global__ void ratfunc_kernel(const double* __restrict__ num_c, const uint8_t* __restrict__ num_e,
                               int32_t n_num, const double* __restrict__ den_c,
                               const uint8_t* __restrict__ den_e, int32_t n_den, int32_t nv,
                               const double* __restrict__ X, int64_t m,
                               double* __restrict__ out, int32_t* __restrict__ status) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* x = X + i * nv;
    auto poly = [&](const double* c, const uint8_t* e, int nt) {
      double acc = 0.0;
      for (int k = 0; k < nt; ++k) {
        double mono = 1.0;
        for (int v = 0; v < nv; ++v) {  // eval_monomial: per-variable power, then product
          double pw = 1.0;
          for (int j = 0; j < e[k * nv + v]; ++j) pw = __dmul_rn(pw, x[v]);
          mono = __dmul_rn(mono, pw);
        }
        acc = __dadd_rn(acc, __dmul_rn(c[k], mono));
      }
      return acc;
    };
    const double p = poly(num_c, num_e, n_num);
    const double q = poly(den_c, den_e, n_den);
    const double mag = fabs(p);
    if (fabs(q) < __dmul_rn(1e-12, mag > 1.0 ? mag : 1.0)) {
      out[i] = 0.0;
      status[i] = 1;
    } else {
      out[i] = __ddiv_rn(p, q);
      status[i] = 0;
    }
  }
}

// Per-device context of the direct-model entry points: one stream and one
// growing device buffer, reused across calls (a scalar perf::active_blocks
// through the C++ shim is one H2D, one launch and one D2H — no stream
// creation or allocation per call).  Calls on one device serialize on the
// context's mutex.
struct DirectCtx {
  std::mutex mu;
  cudaStream_t s = nullptr;
  char* buf = nullptr;
  size_t cap = 0;
  int sms = 148;
};

DirectCtx* direct_ctx(int device, cudaError_t* e) {
  static std::mutex g;
  static std::vector<DirectCtx*> ctx;
  std::lock_guard<std::mutex> lk(g);
  if (device < 0) {
    *e = cudaErrorInvalidDevice;
    return nullptr;
  }
  if ((int)ctx.size() <= device) ctx.resize(device + 1, nullptr);
  if (!ctx[device]) {
    *e = cudaSetDevice(device);
    if (*e != cudaSuccess) return nullptr;
    DirectCtx* c = new DirectCtx;
    *e = cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking);
    if (*e != cudaSuccess) {
      delete c;
      return nullptr;
    }
    cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
    ctx[device] = c;
  }
  *e = cudaSuccess;
  return ctx[device];
}

}  // namespace

extern "C" int rpg_mwpcwp_breakdown_batch(const rpg_profile* hw, const double* kernel_metrics,
                                          const rpg_config* configs, int64_t n, int32_t rep_mode,
                                          int32_t device, rpg_breakdown* out, char* err,
                                          size_t errlen) {
  if (!hw || (n > 0 && (!kernel_metrics || !configs || !out)))
    return set_err(err, errlen, RPG_E_INVALID, "rpg_mwpcwp_breakdown_batch: null argument");
  int rc = validate_profile(hw, err, errlen);
  if (rc) return rc;
  if (rep_mode != RPG_REP_REAL && rep_mode != RPG_REP_CEIL)
    return set_err(err, errlen, RPG_E_INVALID, "rep_mode must be real or ceil");
  if (n <= 0) return RPG_OK;
  Params P{};
  P.hw = *hw;
  hoist_hardware(P);
  P.rep_mode = rep_mode;
  cudaError_t e;
  DirectCtx* c = direct_ctx(device, &e);
  if (!c) return set_err(err, errlen, RPG_E_CUDA, "rpg_mwpcwp_breakdown_batch: %s", cudaGetErrorString(e));
  std::lock_guard<std::mutex> lk(c->mu);
  CUDA_TRY(cudaSetDevice(device));
  const size_t in_m = sizeof(double) * 8 * (size_t)n;
  const size_t in_c = sizeof(rpg_config) * (size_t)n;
  const size_t o_b = sizeof(rpg_breakdown) * (size_t)n;
  CUDA_TRY(ensure(&c->buf, &c->cap, in_m + in_c + o_b));
  double* d_m = reinterpret_cast<double*>(c->buf);
  rpg_config* d_c = reinterpret_cast<rpg_config*>(c->buf + in_m);
  rpg_breakdown* d_o = reinterpret_cast<rpg_breakdown*>(c->buf + in_m + in_c);
  CUDA_TRY(cudaMemcpyAsync(d_m, kernel_metrics, in_m, cudaMemcpyHostToDevice, c->s));
  CUDA_TRY(cudaMemcpyAsync(d_c, configs, in_c, cudaMemcpyHostToDevice, c->s));
  const int grid = (int)std::min<int64_t>((n + 127) / 128, (int64_t)c->sms * 8);
  breakdown_kernel<<<grid, 128, 0, c->s>>>(P, d_m, d_c, n, d_o);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(out, d_o, o_b, cudaMemcpyDeviceToHost, c->s));
  CUDA_TRY(cudaStreamSynchronize(c->s));
  return RPG_OK;
}

extern "C" int rpg_mwpcwp_cycles_batch(const rpg_profile* hw, const double* metrics,
                                       const rpg_config* configs, int64_t n, int32_t rep_mode,
                                       int32_t device, double* total_out, int32_t* b_out,
                                       int32_t* w_out, uint8_t* tag_out, int32_t* status_out,
                                       char* err, size_t errlen) {
  if (!hw || (n > 0 && (!metrics || !configs || !status_out)))
    return set_err(err, errlen, RPG_E_INVALID, "rpg_mwpcwp_cycles_batch: null argument");
  int rc = validate_profile(hw, err, errlen);
  if (rc) return rc;
  if (rep_mode != RPG_REP_REAL && rep_mode != RPG_REP_CEIL)
    return set_err(err, errlen, RPG_E_INVALID, "rep_mode must be real or ceil");
  if (n <= 0) return RPG_OK;
  Params P{};
  P.hw = *hw;
  hoist_hardware(P);
  P.rep_mode = rep_mode;
  cudaError_t e;
  DirectCtx* c = direct_ctx(device, &e);
  if (!c) return set_err(err, errlen, RPG_E_CUDA, "rpg_mwpcwp_cycles_batch: %s", cudaGetErrorString(e));
  std::lock_guard<std::mutex> lk(c->mu);
  CUDA_TRY(cudaSetDevice(device));
  const size_t in_m = sizeof(double) * RPG_N_METRICS * (size_t)n;
  const size_t in_c = sizeof(rpg_config) * (size_t)n;
  const size_t o_t = sizeof(double) * (size_t)n, o_i = sizeof(int32_t) * (size_t)n;
  CUDA_TRY(ensure(&c->buf, &c->cap, in_m + in_c + o_t + 3 * o_i + (size_t)n + 64));
  char* buf = c->buf;
  double* d_m = reinterpret_cast<double*>(buf);
  rpg_config* d_c = reinterpret_cast<rpg_config*>(buf + in_m);
  double* d_t = reinterpret_cast<double*>(buf + in_m + in_c);
  int32_t* d_b = reinterpret_cast<int32_t*>(buf + in_m + in_c + o_t);
  int32_t* d_w = d_b + n;
  int32_t* d_s = d_w + n;
  uint8_t* d_g = reinterpret_cast<uint8_t*>(d_s + n);
  CUDA_TRY(cudaMemcpyAsync(d_m, metrics, in_m, cudaMemcpyHostToDevice, c->s));
  CUDA_TRY(cudaMemcpyAsync(d_c, configs, in_c, cudaMemcpyHostToDevice, c->s));
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)c->sms * 8);
  direct_cycles_kernel<<<grid, 256, 0, c->s>>>(P, d_m, d_c, n, d_t, d_b, d_w, d_g, d_s);
  CUDA_TRY(cudaGetLastError());
  if (total_out) CUDA_TRY(cudaMemcpyAsync(total_out, d_t, o_t, cudaMemcpyDeviceToHost, c->s));
  if (b_out) CUDA_TRY(cudaMemcpyAsync(b_out, d_b, o_i, cudaMemcpyDeviceToHost, c->s));
  if (w_out) CUDA_TRY(cudaMemcpyAsync(w_out, d_w, o_i, cudaMemcpyDeviceToHost, c->s));
  if (tag_out) CUDA_TRY(cudaMemcpyAsync(tag_out, d_g, (size_t)n, cudaMemcpyDeviceToHost, c->s));
  CUDA_TRY(cudaMemcpyAsync(status_out, d_s, o_i, cudaMemcpyDeviceToHost, c->s));
  CUDA_TRY(cudaStreamSynchronize(c->s));
  return RPG_OK;
}

extern "C" int rpg_eval_ratfunc_batch(const rpg_poly* num, const rpg_poly* den, int32_t n_vars,
                                      const double* X, int64_t m, int32_t device, double* out,
                                      int32_t* status_out, char* err, size_t errlen) {
  if (!num || !den || (m > 0 && (!X || !out || !status_out)))
    return set_err(err, errlen, RPG_E_INVALID, "rpg_eval_ratfunc_batch: null argument");
  if (n_vars < 1 || n_vars > RPG_MAX_VARS || num->n_terms < 0 || den->n_terms < 0)
    return set_err(err, errlen, RPG_E_INVALID, "rpg_eval_ratfunc_batch: bad shape");
  if (m <= 0) return RPG_OK;
  CUDA_TRY(cudaSetDevice(device));
  cudaStream_t s;
  CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const size_t tn = (size_t)std::max(num->n_terms, 1), td = (size_t)std::max(den->n_terms, 1);
  const size_t bx = sizeof(double) * (size_t)m * n_vars;
  const size_t total = bx + sizeof(double) * (size_t)m + sizeof(int32_t) * (size_t)m +
                       sizeof(double) * (tn + td) + (tn + td) * n_vars + 64;
  char* buf = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&buf), total, s);
  if (e == cudaSuccess) {
    double* d_x = reinterpret_cast<double*>(buf);
    double* d_o = reinterpret_cast<double*>(buf + bx);
    double* d_nc = d_o + m;
    double* d_dc = d_nc + tn;
    int32_t* d_s = reinterpret_cast<int32_t*>(d_dc + td);
    uint8_t* d_ne = reinterpret_cast<uint8_t*>(d_s + m);
    uint8_t* d_de = d_ne + tn * n_vars;
    cudaMemcpyAsync(d_x, X, bx, cudaMemcpyHostToDevice, s);
    if (num->n_terms) {
      cudaMemcpyAsync(d_nc, num->coef, sizeof(double) * num->n_terms, cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(d_ne, num->exps, (size_t)num->n_terms * n_vars, cudaMemcpyHostToDevice, s);
    }
    if (den->n_terms) {
      cudaMemcpyAsync(d_dc, den->coef, sizeof(double) * den->n_terms, cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(d_de, den->exps, (size_t)den->n_terms * n_vars, cudaMemcpyHostToDevice, s);
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int grid = (int)std::min<int64_t>((m + 255) / 256, (int64_t)sms * 8);
    ratfunc_kernel<<<grid, 256, 0, s>>>(d_nc, d_ne, num->n_terms, d_dc, d_de, den->n_terms,
                                        n_vars, d_x, m, d_o, d_s);
    e = cudaGetLastError();
    if (e == cudaSuccess) {
      cudaMemcpyAsync(out, d_o, sizeof(double) * (size_t)m, cudaMemcpyDeviceToHost, s);
      cudaMemcpyAsync(status_out, d_s, sizeof(int32_t) * (size_t)m, cudaMemcpyDeviceToHost, s);
      e = cudaStreamSynchronize(s);
    }
    cudaFreeAsync(buf, s);
  }
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (e != cudaSuccess)
    return set_err(err, errlen, RPG_E_CUDA, "rpg_eval_ratfunc_batch: %s", cudaGetErrorString(e));
  return RPG_OK;
}

// rng::uniform_real draws (rng.hpp:14-21) from std::mt19937_64(seed): the
// noise stream of data::synthesize (datakit.hpp:199-203), which is
// sequential by construction (one draw per kept point and metric).
#include <random>
extern "C" int rpg_uniform_stream(uint64_t seed, int64_t n, double lo, double hi, double* out) {
  if (n < 0 || (n > 0 && !out)) return RPG_E_INVALID;
  std::mt19937_64 g(seed);
  const double span = hi - lo;
  for (int64_t i = 0; i < n; ++i) {
    const double c = static_cast<double>(g() >> 11) * 0x1.0p-53;
    const double t = span * c;  // -ffp-contract=off: no fused multiply-add
    out[i] = lo + t;
  }
  return RPG_OK;
}
