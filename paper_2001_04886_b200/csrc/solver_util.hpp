// solver_util.hpp -- host-side helpers shared by the solver orchestrators: descriptor
// builders that split oversized update / inner-product sets into chained launches while
// preserving the reference's per-element accumulation order, and report bookkeeping.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "skc_internal.hpp"

namespace skc {

inline size_t pad_n(int64_t n) { return (size_t)((n + 31) / 32 * 32); }

// sstep.hpp:62-67
inline void validate_block_size(const SStepCfg& cfg, Report& rep) {
  require(cfg.s >= 1 && cfg.s <= 8, "s-step: s must be in 1..8");
  if (cfg.s > 5)
    rep.notes.push_back("s=" + std::to_string(cfg.s) + " exceeds the stability guideline of 5; expect basis collapse");
}

// GramSolver's breakdown text (small_dense.hpp:52-53, 62-64)
inline std::string gram_message(int singular1, double ratio) {
  if (singular1) return "sym_solve: singular 1x1 Gram system";
  return "sym_solve: numerically singular Gram system (pivot ratio " + fmt_double(ratio) + ")";
}

inline void add(skc_op_counter& c, uint64_t dots, uint64_t mv, uint64_t upd) {
  c.dotprods += dots;
  c.matvecs += mv;
  c.vec_updates += upd;
}

// Fused update y_o = base_o [* scale] + sum_j c_{j,o} in_j (j in insertion order) with
// optional inner products of the results. Inputs beyond LC_MAXIN continue in further
// launches that update the outputs in place, which keeps every element's accumulation
// order identical to a single pass.
struct LinBuilder {
  struct Term {
    const double* v;
    uint16_t mask;
    int16_t cbase;
  };
  std::vector<Term> terms;
  std::vector<double*> out;
  std::vector<const double*> base;
  std::vector<int16_t> bscale;
  std::vector<const double*> xin;
  std::vector<std::pair<int, int>> dots;

  int add_out(double* o, const double* b, int scale_idx = -1) {
    out.push_back(o);
    base.push_back(b);
    bscale.push_back((int16_t)scale_idx);
    return (int)out.size() - 1;
  }
  void add_term(const double* v, uint16_t mask, int cbase) { terms.push_back({v, mask, (int16_t)cbase}); }
  int add_extra(const double* v) {
    xin.push_back(v);
    return (int)(out.size() + xin.size() - 1);  // value id (valid once all outputs are added)
  }
  void add_dot(int a, int b) { dots.push_back({a, b}); }

  void launch(Ctx& c, const Geo& g, const double* coef, int ncoef, double* partials, int dot0, const int* halt,
              const int* cond, const char* name) const {
    require(out.size() <= (size_t)LC_MAXOUT && xin.size() <= (size_t)LC_MAXX && dots.size() <= (size_t)LC_MAXD,
            "lincomb: too many outputs/dots");
    size_t t0 = 0;
    bool first = true;
    do {
      const size_t t1 = std::min(terms.size(), t0 + (size_t)LC_MAXIN);
      const bool last = t1 == terms.size();
      LinDesc d;
      std::memset(&d, 0, sizeof d);
      d.nin = (int)(t1 - t0);
      for (size_t t = t0; t < t1; ++t) {
        d.in[t - t0] = terms[t].v;
        d.mask[t - t0] = terms[t].mask;
        d.cbase[t - t0] = terms[t].cbase;
      }
      d.nout = (int)out.size();
      for (size_t q = 0; q < out.size(); ++q) {
        d.out[q] = out[q];
        d.base[q] = first ? base[q] : out[q];
        d.bscale[q] = first ? bscale[q] : (int16_t)-1;
      }
      if (last) {
        d.nx = (int)xin.size();
        for (size_t x = 0; x < xin.size(); ++x) d.xin[x] = xin[x];
        d.nd = (int)dots.size();
        for (size_t k = 0; k < dots.size(); ++k) {
          d.da[k] = (uint8_t)dots[k].first;
          d.db[k] = (uint8_t)dots[k].second;
        }
      }
      d.coef = coef;
      d.ncoef = ncoef;
      d.partials = partials;
      d.dot0 = dot0;
      d.G = g.G;
      d.n = g.n;
      d.range = g.range;
    d.cpg = g.cpg;
    d.gsize = g.gsize;
      d.cpg = g.cpg;
      d.gsize = g.gsize;
      d.halt = halt;
      d.cond = cond;
      launch_lincomb(c, d, name);
      t0 = t1;
      first = false;
    } while (t0 < terms.size());
  }
};

// Inner products L_l . R_r at dot index dot0 + l*nr + r, split over launches of GR_MAXL rows.
// Left rows per launch: every distinct operand of a launch is staged per point tile, so many
// operands force small tiles (kilobyte-sized bulk copies, thousands of concurrent DRAM streams;
// measured 1.8 TB/s with 72 operands vs 6+ TB/s with ~20).  Wide Grams are therefore split into
// launches of at most ~kGramOperands operands; each re-reads the right operands (few) once more.
inline size_t gram_chunk(size_t nr) {
  // measured on C4 (s = 8): Scalar1 products (nr = 1) best at ~24 operands, the cross
  // products (nr = s = 8) at ~32
  static const int target = [] {
    const char* e = std::getenv("SKC_GRAM_U");
    return e ? std::atoi(e) : 0;
  }();
  const int t = target > 0 ? target : nr <= 2 ? 24 : 32;
  const int c = std::max(8, t - (int)nr);
  return (size_t)std::min(c, GR_MAXL);
}

inline void launch_gram_list(Ctx& c, const Geo& g, const std::vector<const double*>& L,
                             const std::vector<const double*>& R, double* partials, int dot0, const int* halt,
                             const int* cond, const char* name = "gram") {
  require(!R.empty() && R.size() <= (size_t)GR_MAXR, "gram: right operand count out of range");
  const size_t chunk = gram_chunk(R.size());
  for (size_t l0 = 0; l0 < L.size(); l0 += chunk) {
    const size_t l1 = std::min(L.size(), l0 + chunk);
    GramDesc d;
    std::memset(&d, 0, sizeof d);
    d.nl = (int)(l1 - l0);
    d.nr = (int)R.size();
    for (size_t l = l0; l < l1; ++l) d.L[l - l0] = L[l];
    for (size_t r = 0; r < R.size(); ++r) d.R[r] = R[r];
    d.partials = partials;
    d.dot0 = dot0 + (int)(l0 * R.size());
    d.G = g.G;
    d.n = g.n;
    d.range = g.range;
    d.cpg = g.cpg;
    d.gsize = g.gsize;
    d.halt = halt;
    d.cond = cond;
    launch_gram(c, d, name);
  }
}

// Gram products with an explicit output map per right operand: L[l] . R[r] -> dot
// col[r].base + l*col[r].stride for l < col[r].lmax (one pass over L and R).
struct GramCol {
  int base, stride, lmax;
};
inline void launch_gram_map(Ctx& c, const Geo& g, const std::vector<const double*>& L,
                            const std::vector<const double*>& R, const std::vector<GramCol>& cols, double* partials,
                            const int* halt, const int* cond, const char* name) {
  require(!R.empty() && R.size() <= (size_t)GR_MAXR && cols.size() == R.size(), "gram: right operand count out of range");
  const size_t chunk = gram_chunk(R.size());
  for (size_t l0 = 0; l0 < L.size(); l0 += chunk) {
    const size_t l1 = std::min(L.size(), l0 + chunk);
    GramDesc d;
    std::memset(&d, 0, sizeof d);
    d.nl = (int)(l1 - l0);
    d.nr = (int)R.size();
    for (size_t l = l0; l < l1; ++l) d.L[l - l0] = L[l];
    d.mapped = 1;
    for (size_t r = 0; r < R.size(); ++r) {
      d.R[r] = R[r];
      d.rbase[r] = cols[r].base + (int)l0 * cols[r].stride;
      d.rstride[r] = cols[r].stride;
      d.lmax[r] = std::max(0, cols[r].lmax - (int)l0);
    }
    d.partials = partials;
    d.G = g.G;
    d.n = g.n;
    d.range = g.range;
    d.cpg = g.cpg;
    d.gsize = g.gsize;
    d.halt = halt;
    d.cond = cond;
    launch_gram(c, d, name);
  }
}

// x == 0 test on the device (initial_residual's is_zero, kernels.hpp:70-74)
bool device_is_zero(Ctx& c, const double* x, int64_t n);

}  // namespace skc
