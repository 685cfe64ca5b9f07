// sim_main.cpp — drives the REFERENCE simulator's run() (proj/src/simulator.cpp)
// on a config + trace and prints its summary JSON (report.cpp summary_json)
// followed by its samples CSV (report.cpp samples_csv).
//
// Built twice by examples/Makefile from the unmodified reference sources:
//   _build/sim_ref    simulator.cpp as shipped (analytic layer_forward_time)
//   _build/sim_b200   simulator.cpp with ONE line changed at :194 —
//                     layer_forward_time(...) -> b200::layer_forward_time(...)
//                     (include/moeless/b200_layer.hpp, force-included), linked
//                     against libmoe_b200.so: every MoE-layer forward of run()
//                     runs on the B200.
//
//   sim_{ref,b200} CONFIG TRACE [MAX_REQUESTS]
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>
#include <vector>

#include "moeless/config.hpp"
#include "moeless/report.hpp"
#include "moeless/simulator.hpp"
#include "moeless/workload.hpp"

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s CONFIG TRACE [MAX_REQUESTS]\n", argv[0]);
    return 2;
  }
  try {
    const moeless::SimConfig cfg = moeless::load_config(argv[1]);
    std::vector<moeless::Request> trace = moeless::parse_trace(argv[2]);
    if (argc > 3) {
      const size_t n = static_cast<size_t>(std::atol(argv[3]));
      if (n < trace.size()) trace.resize(n);
    }
    const moeless::MetricsReport rep = moeless::run(cfg, trace);
    std::fputs(moeless::summary_json(rep).c_str(), stdout);
    std::fputs("---\n", stdout);
    std::fputs(moeless::samples_csv(rep).c_str(), stdout);
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
