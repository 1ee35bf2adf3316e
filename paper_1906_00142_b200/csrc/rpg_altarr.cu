// rpg_altarr.cu — host-side interop with the paper's per-metric polynomial
// encoding (BPAS AltArr_t).  See rpg.h
// for the layout.  No device code: conversion happens once, before
// rpg_plan_create packs the model for the GPU.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "rpg.h"

namespace {

int aa_err(char* err, size_t errlen, int code, const char* fmt, ...) {
  if (err && errlen) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, errlen, fmt, ap);
    va_end(ap);
  }
  return code;
}

int field_width(int nvar) { return 64 / nvar; }

// Graded-lex comparison of exponent tuples (polyfit.hpp:50-73): ascending
// total degree, ties lexicographic with variable 0 most significant.
bool grlex_less(const uint8_t* a, const uint8_t* b, int nvar) {
  int sa = 0, sb = 0;
  for (int v = 0; v < nvar; ++v) {
    sa += a[v];
    sb += b[v];
  }
  if (sa != sb) return sa < sb;
  for (int v = 0; v < nvar; ++v)
    if (a[v] != b[v]) return a[v] < b[v];
  return false;
}

std::string hexd(double v) {
  char b[64];
  snprintf(b, sizeof b, "%a", v);
  return b;
}

}  // namespace

extern "C" uint64_t rpg_aa_pack_degs(const uint8_t* exps, int32_t nvar) {
  if (nvar < 1 || nvar > RPG_MAX_VARS) return 0;
  const int w = field_width(nvar);
  uint64_t d = 0;
  for (int v = 0; v < nvar; ++v) d |= (uint64_t)exps[v] << (64 - (v + 1) * w);
  return d;
}

extern "C" void rpg_aa_unpack_degs(uint64_t degs, int32_t nvar, uint8_t* exps) {
  if (nvar < 1 || nvar > RPG_MAX_VARS) return;
  const int w = field_width(nvar);
  const uint64_t mask = w >= 64 ? ~0ull : ((1ull << w) - 1);
  for (int v = 0; v < nvar; ++v) exps[v] = (uint8_t)((degs >> (64 - (v + 1) * w)) & mask);
}

extern "C" int rpg_aa_from_poly(const rpg_poly* p, int32_t nvar, rpg_altarr* out, char* err,
                                size_t errlen) {
  if (!p || !out || (p->n_terms > 0 && (!p->coef || !p->exps)))
    return aa_err(err, errlen, RPG_E_INVALID, "rpg_aa_from_poly: null argument");
  if (nvar < 1 || nvar > RPG_MAX_VARS)
    return aa_err(err, errlen, RPG_E_INVALID, "rpg_aa_from_poly: nvar must be in [1, %d]", RPG_MAX_VARS);
  std::vector<rpg_aa_elem> el;
  for (int k = 0; k < p->n_terms; ++k) {
    if (p->coef[k] == 0.0) continue;
    el.push_back({p->coef[k], rpg_aa_pack_degs(p->exps + (size_t)k * nvar, nvar)});
  }
  std::stable_sort(el.begin(), el.end(),
                   [](const rpg_aa_elem& a, const rpg_aa_elem& b) { return a.degs > b.degs; });
  for (size_t i = 1; i < el.size(); ++i)
    if (el[i].degs == el[i - 1].degs)
      return aa_err(err, errlen, RPG_E_INVALID, "rpg_aa_from_poly: duplicated monomial");
  if ((int64_t)el.size() > out->alloc || (!out->elems && !el.empty()))
    return aa_err(err, errlen, RPG_E_INVALID,
                  "rpg_aa_from_poly: %zu terms exceed the AltArr allocation (%d)", el.size(), out->alloc);
  if (!el.empty()) memcpy(out->elems, el.data(), el.size() * sizeof(rpg_aa_elem));
  out->size = (int32_t)el.size();
  out->nvar = nvar;
  out->unpacked = 0;
  return RPG_OK;
}

extern "C" int rpg_aa_to_poly(const rpg_altarr* a, double* coef, uint8_t* exps, int32_t cap,
                              int32_t* n_terms, char* err, size_t errlen) {
  if (!a || (a->size > 0 && !a->elems))
    return aa_err(err, errlen, RPG_E_INVALID, "rpg_aa_to_poly: null argument");
  const int nvar = a->nvar;
  if (nvar < 1 || nvar > RPG_MAX_VARS)
    return aa_err(err, errlen, RPG_E_INVALID, "rpg_aa_to_poly: nvar must be in [1, %d]", RPG_MAX_VARS);
  if (a->unpacked)
    return aa_err(err, errlen, RPG_E_INVALID, "rpg_aa_to_poly: unpacked AltArr is not supported");
  if (a->size < 0)
    return aa_err(err, errlen, RPG_E_INVALID, "rpg_aa_to_poly: negative size");
  struct Term {
    double c;
    uint8_t e[RPG_MAX_VARS];
  };
  std::vector<Term> t;
  for (int i = 0; i < a->size; ++i) {
    const rpg_aa_elem& el = a->elems[i];
    if (i > 0 && !(el.degs < a->elems[i - 1].degs))
      return aa_err(err, errlen, RPG_E_INVALID,
                    "rpg_aa_to_poly: element %d is not in strictly decreasing degree order", i);
    if (!std::isfinite(el.coef))
      return aa_err(err, errlen, RPG_E_INVALID, "rpg_aa_to_poly: element %d has a non-finite coefficient", i);
    if (el.coef == 0.0) continue;
    Term x{};
    x.c = el.coef;
    rpg_aa_unpack_degs(el.degs, nvar, x.e);
    if (rpg_aa_pack_degs(x.e, nvar) != el.degs)
      return aa_err(err, errlen, RPG_E_INVALID,
                    "rpg_aa_to_poly: element %d has an exponent wider than 8 bits", i);
    t.push_back(x);
  }
  std::stable_sort(t.begin(), t.end(),
                   [nvar](const Term& x, const Term& y) { return grlex_less(x.e, y.e, nvar); });
  if ((int64_t)t.size() > cap)
    return aa_err(err, errlen, RPG_E_INVALID, "rpg_aa_to_poly: %zu terms exceed capacity %d", t.size(), cap);
  for (size_t k = 0; k < t.size(); ++k) {
    coef[k] = t[k].c;
    memcpy(exps + k * nvar, t[k].e, nvar);
  }
  if (n_terms) *n_terms = (int32_t)t.size();
  return RPG_OK;
}

extern "C" int64_t rpg_emit_altarr_header(const rpg_poly* num, const rpg_poly* den, int32_t nvar,
                                          const char* const* var_names, const char* name,
                                          char* buf, size_t buflen, char* err, size_t errlen) {
  if (!num || !den || !name)
    return aa_err(err, errlen, RPG_E_INVALID, "rpg_emit_altarr_header: null argument");
  std::ostringstream o;
  o << "/* " << name << " = " << name << "_num / " << name << "_den over (";
  for (int v = 0; v < nvar; ++v) o << (v ? ", " : "") << (var_names ? var_names[v] : "x");
  o << ")\n * generated by librpgpu rpg_emit_altarr_header: AltArr-form rational\n"
       " * function (packed degrees, variable 0 most significant, "
    << 64 / std::max(nvar, 1) << " bits per variable). */\n";
  o << "#include \"rpg.h\"\n";
  const rpg_poly* polys[2] = {num, den};
  const char* part[2] = {"num", "den"};
  for (int j = 0; j < 2; ++j) {
    std::vector<rpg_aa_elem> el(std::max(polys[j]->n_terms, 1));
    rpg_altarr aa{0, (int32_t)el.size(), nvar, 0, el.data()};
    const int rc = rpg_aa_from_poly(polys[j], nvar, &aa, err, errlen);
    if (rc != RPG_OK) return rc;
    o << "static rpg_aa_elem " << name << "_" << part[j] << "_elems[" << std::max(aa.size, 1)
      << "] = {\n";
    for (int i = 0; i < aa.size; ++i) {
      char d[32];
      snprintf(d, sizeof d, "0x%016llxull", (unsigned long long)el[i].degs);
      o << "  {" << hexd(el[i].coef) << ", " << d << "},\n";
    }
    if (aa.size == 0) o << "  {0.0, 0ull}\n";
    o << "};\n";
    o << "static rpg_altarr " << name << "_" << part[j] << " = {" << aa.size << ", "
      << std::max(aa.size, 1) << ", " << nvar << ", 0, " << name << "_" << part[j] << "_elems};\n";
  }
  const std::string s = o.str();
  if (buf && buflen) {
    const size_t n = std::min(buflen - 1, s.size());
    memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return (int64_t)s.size();
}
