// skrylov_b200/accounting.hpp -- op-count predictions and the audit of a SolveReport's counter
// deltas (drop-in for skrylov/accounting.hpp:54-191 over skrylov::b200::SolveReport).
//
//     #include "skrylov/accounting.hpp"   ->  #include "skrylov_b200/accounting.hpp"
//
// Header-only host code: the GPU solvers record op_history / steady_iteration exactly as the
// reference does, so the same predictions and slacks apply.  Counter differences wrap like the
// reference's std::size_t arithmetic; termination inner products are never audited.
#ifndef SKRYLOV_B200_ACCOUNTING_HPP
#define SKRYLOV_B200_ACCOUNTING_HPP

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "sstep.hpp"

namespace skrylov::b200 {

enum class AuditMode { exact, bounded, off };

inline OpCounter counter_delta(const OpCounter& a, const OpCounter& b) {  // report.hpp:43-51
  OpCounter d{};
  d.dotprods = a.dotprods - b.dotprods;
  d.matvecs = a.matvecs - b.matvecs;
  d.vec_updates = a.vec_updates - b.vec_updates;
  d.stored_vectors = a.stored_vectors;  // a peak, not a delta
  d.termination_dots = a.termination_dots - b.termination_dots;
  return d;
}

// accounting.hpp:54-70: iteration j of (s-)Orthomin(k)
inline OpCounter predicted_omin(std::uint64_t j, std::uint64_t k, std::uint64_t s) {
  const std::uint64_t s2 = s * s, tri = s * (s + 1) / 2;
  OpCounter c{};
  const bool classic = s == 1 && j >= k;
  c.dotprods = classic ? k + 2 : std::min((j + 1) * s2 + tri, k * s2 + tri);
  c.vec_updates = classic ? 2 * k + 2 : std::min(2 * (j + 1) * s2 + s, 2 * k * s2 + tri);
  c.matvecs = s;
  c.stored_vectors = 2 * k * s + s + 1;
  return c;
}

struct PredictedGmresCosts {  // accounting.hpp:72-75
  OpCounter gmres{};   // one cycle of GMRES(s m)
  OpCounter sgmres{};  // one cycle of s-GMRES(m)
};

inline PredictedGmresCosts predicted_gmres(std::uint64_t m, std::uint64_t s) {  // accounting.hpp:77-92
  PredictedGmresCosts p;
  const std::uint64_t ms = m * s;
  p.gmres.dotprods = ms + ms * (ms + 1) / 2;
  p.gmres.matvecs = ms + 1;
  p.gmres.vec_updates = (ms * ms + ms) / 2 + 2 * ms;
  p.gmres.stored_vectors = ms + 1;
  p.sgmres.dotprods = m * (m - 1) * s * s / 2 + s * (s + 1) / 2 + s;
  p.sgmres.matvecs = s * (m + 1);
  p.sgmres.vec_updates = m * (m + 1) * s * s;
  p.sgmres.stored_vectors = s * (m + 1) * m / 2 + m;
  return p;
}

inline OpCounter somin_audit_slack(std::uint64_t s) {  // accounting.hpp:97-102
  OpCounter c{};
  c.dotprods = s;
  c.vec_updates = 2 * s;
  return c;
}

inline OpCounter gmres_audit_slack() {  // accounting.hpp:106-111
  OpCounter c{};
  c.vec_updates = 2;
  return c;
}

inline OpCounter sgmres_audit_slack(std::uint64_t m, std::uint64_t s) {  // accounting.hpp:116-132
  const std::uint64_t tri = s * (s + 1) / 2;
  const std::uint64_t mine = s * m * (m + 1) / 2 + m + m * tri +
                             (2 * s * (s - 1) + s * s) * (m - 1) * m / 2 + (m - 1) * s;
  const std::uint64_t table = m * (m - 1) * s * s / 2 + tri + s;
  OpCounter c{};
  c.dotprods = mine > table ? mine - table : 0;
  c.vec_updates = 2;
  return c;
}

struct AuditReport {  // accounting.hpp:134-140
  bool ok = true;
  bool matvecs_exact = true;
  bool dotprods_exact = true;
  bool updates_exact = true;
  std::vector<std::string> diffs;
};

// accounting.hpp:149-191
inline AuditReport audit(const SolveReport& rep, const OpCounter& predicted, AuditMode mode,
                         const OpCounter& slack = OpCounter{}) {
  AuditReport out;
  if (mode == AuditMode::off || rep.op_history.size() < 2) return out;
  auto check = [&](std::size_t iv, const char* name, std::uint64_t got, std::uint64_t want, bool bad,
                   const char* rel) {
    if (!bad) return;
    out.ok = false;
    out.diffs.push_back("interval " + std::to_string(iv) + ": " + name + " " + std::to_string(got) + " " +
                        rel + " " + std::to_string(want));
  };
  for (std::size_t t = 1; t < rep.op_history.size(); ++t) {
    const OpCounter d = counter_delta(rep.op_history[t], rep.op_history[t - 1]);
    const std::size_t iv = t - 1;
    const bool steady = iv >= rep.steady_iteration;
    out.matvecs_exact &= d.matvecs == predicted.matvecs;
    if (steady) {
      out.dotprods_exact &= d.dotprods == predicted.dotprods;
      out.updates_exact &= d.vec_updates == predicted.vec_updates;
    }
    if (mode == AuditMode::exact) {
      const char* rel = steady ? "!=" : ">";
      check(iv, "dotprods", d.dotprods, predicted.dotprods,
            steady ? d.dotprods != predicted.dotprods : d.dotprods > predicted.dotprods, rel);
      check(iv, "vec_updates", d.vec_updates, predicted.vec_updates,
            steady ? d.vec_updates != predicted.vec_updates : d.vec_updates > predicted.vec_updates, rel);
    } else {
      const std::uint64_t wd = predicted.dotprods + slack.dotprods;
      const std::uint64_t wu = predicted.vec_updates + slack.vec_updates;
      check(iv, "dotprods", d.dotprods, wd, d.dotprods > wd, ">");
      check(iv, "vec_updates", d.vec_updates, wu, d.vec_updates > wu, ">");
    }
    check(iv, "matvecs", d.matvecs, predicted.matvecs, d.matvecs != predicted.matvecs, "!=");
  }
  return out;
}

}  // namespace skrylov::b200

#endif  // SKRYLOV_B200_ACCOUNTING_HPP
