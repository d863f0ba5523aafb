// Drives include/skrylov_b200/accounting.hpp from a line protocol on stdin (tests/test_accounting.py):
//   P kind a b c                       -> the prediction / slack (5 counters)
//   A n steady mode p[5] slack[5] h[n][5] -> ok matvecs_exact dotprods_exact updates_exact ndiffs, then the diffs
#include <cstdint>
#include <iostream>
#include <string>

#include "skrylov_b200/accounting.hpp"

using namespace skrylov::b200;

static OpCounter read_counter(std::istream& in) {
  OpCounter c{};
  in >> c.dotprods >> c.matvecs >> c.vec_updates >> c.stored_vectors >> c.termination_dots;
  return c;
}

static void print(const OpCounter& c) {
  std::cout << c.dotprods << ' ' << c.matvecs << ' ' << c.vec_updates << ' ' << c.stored_vectors << ' '
            << c.termination_dots << '\n';
}

int main() {
  std::string tag;
  while (std::cin >> tag) {
    if (tag == "P") {
      int kind;
      std::uint64_t a, b, c;
      std::cin >> kind >> a >> b >> c;
      switch (kind) {
        case 0: print(predicted_omin(a, b, c)); break;
        case 1: print(predicted_gmres(a, b).gmres); break;
        case 2: print(predicted_gmres(a, b).sgmres); break;
        case 3: print(somin_audit_slack(a)); break;
        case 4: print(gmres_audit_slack()); break;
        default: print(sgmres_audit_slack(a, b)); break;
      }
    } else {
      std::size_t n, steady;
      int mode;
      std::cin >> n >> steady >> mode;
      const OpCounter p = read_counter(std::cin), sl = read_counter(std::cin);
      SolveReport rep;
      rep.steady_iteration = steady;
      for (std::size_t i = 0; i < n; ++i) rep.op_history.push_back(read_counter(std::cin));
      const AuditMode m = mode == 0 ? AuditMode::exact : mode == 1 ? AuditMode::bounded : AuditMode::off;
      const AuditReport v = audit(rep, p, m, sl);
      std::cout << v.ok << ' ' << v.matvecs_exact << ' ' << v.dotprods_exact << ' ' << v.updates_exact << ' '
                << v.diffs.size() << '\n';
      for (const auto& d : v.diffs) std::cout << d << '\n';
    }
  }
  return 0;
}
