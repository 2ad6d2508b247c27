// The reference's exception types cross the boundary unchanged.
//
// Compiled WITH the reference's headers on the include path (oracle/Makefile
// builds it into oracle/_ref/ where /root/reference exists; the GPU tests run
// the prebuilt binary), so include/appo_b200.hpp throws ::appo::ContractError /
// ConfigError / NumericError (common.hpp:20-40).  main() catches them in the
// order the reference CLI does (tools/appo_cli.cpp:151-163) and returns the
// CLI's exit codes (runner.hpp:28-33): a device-detected non-finite value must
// exit 3 (numeric halt), an invalid V-trace config 2, everything else 4.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <type_traits>
#include <vector>

#include "appo_b200.hpp"

static_assert(APPO_B200_REFERENCE_ERRORS == 1, "reference common.hpp must be on the include path");
static_assert(std::is_same_v<appo_b200::NumericError, appo::NumericError>);
static_assert(std::is_same_v<appo_b200::ConfigError, appo::ConfigError>);
static_assert(std::is_same_v<appo_b200::ContractError, appo::ContractError>);

namespace {

void scenario(const std::string& what) {
  using namespace appo_b200;
  Context ctx(0, 1);
  std::vector<double> r{1.0, 1.0}, v{0.0, 0.0}, tl{-0.5, -0.7}, bl{-0.5, -0.7};
  std::vector<uint8_t> d{0, 0};
  VTraceConfig cfg{1.0, 1.0, 0.99};
  if (what == "ok") {
    ctx.vtrace(r, v, 0.0, tl, bl, d, cfg);
  } else if (what == "config") {  // rho_bar < c_bar (offpolicy.hpp:23-27)
    ctx.vtrace(r, v, 0.0, tl, bl, d, VTraceConfig{0.5, 1.0, 0.99});
  } else if (what == "numeric-vtrace") {  // non-finite reward, found on the device
    r[1] = NAN;
    ctx.vtrace(r, v, 0.0, tl, bl, d, cfg);
  } else if (what == "numeric-adam") {  // optimizer_step: non-finite gradient
    PolicyParams p;
    p.theta.assign(64, 0.5);
    std::vector<double> g(64, 0.1);
    g[17] = INFINITY;
    ctx.optimizer_step(p, g, AdamConfig{});
  } else if (what == "contract") {  // shape mismatch (APPO_CHECK)
    std::vector<double> r3{1.0, 1.0, 1.0};
    try {
      ctx.vtrace(r3, v, 0.0, tl, bl, d, cfg);
    } catch (const appo::ContractError&) {
      std::printf("caught appo::ContractError\n");
      throw;
    }
  } else {
    throw appo::ConfigError("unknown scenario " + what);
  }
}

}  // namespace

int main(int argc, char** argv) {
  const std::string what = argc > 1 ? argv[1] : "ok";
  try {
    scenario(what);
  } catch (const appo::ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 2;
  } catch (const appo::NumericError& e) {
    std::fprintf(stderr, "numeric halt: %s\n", e.what());
    return 3;
  } catch (const std::bad_alloc&) {
    std::fprintf(stderr, "resource exhaustion\n");
    return 4;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 4;
  }
  return 0;
}
