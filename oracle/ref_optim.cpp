// Test-infrastructure driver: runs the UNMODIFIED reference update rule
// ppsim::detail::apply_update (optim.hpp:234-268) on seeded vectors and prints the
// iterates as JSON, to pin the oracle's restatement and the GPU optimizer kernel.
#include <cstdio>
#include <random>
#include <vector>

#include "ppsim/optim.hpp"

using namespace ppsim;

int main() {
  std::mt19937_64 rng(2605);
  std::normal_distribution<double> nd(0.0, 1.0);
  const int p = 257, steps = 5;
  struct Case { const char* name; OptimizerSpec spec; };
  OptimizerSpec adam = OptimizerSpec::adam_type(0.01, 0.9, 0.999, 1e-3);
  OptimizerSpec adam_clamped = OptimizerSpec::adam_type(0.1, 0.9, 0.9, 0.25);
  adam_clamped.clamp_min = 0.25;
  adam_clamped.clamp_max = 3.0;
  const Case cases[] = {{"sgd", OptimizerSpec::sgd(0.1)},
                        {"momentum", OptimizerSpec::momentum(0.05, 0.9)},
                        {"adamtype", adam},
                        {"adamtype_clamped", adam_clamped}};
  std::printf("[");
  bool first_case = true;
  for (const auto& c : cases) {
    std::vector<double> theta(p);
    for (double& x : theta) x = nd(rng);
    std::vector<std::vector<double>> grads(steps, std::vector<double>(p));
    for (auto& g : grads)
      for (double& x : g) x = nd(rng) * 0.5;
    detail::OptState st;
    st.init(p);
    double pmin = 1e300, pmax = 0;
    std::printf("%s{\"name\":\"%s\",\"eta\":%.17g,\"beta1\":%.17g,\"beta2\":%.17g,\"epsilon\":%.17g,"
                "\"clamp_min\":%.17g,\"clamp_max\":%.17g,\"theta0\":[",
                first_case ? "" : ",", c.name, c.spec.eta, c.spec.beta1, c.spec.beta2, c.spec.epsilon,
                c.spec.clamp_min, c.spec.clamp_max);
    first_case = false;
    for (int k = 0; k < p; ++k) std::printf("%s%.17g", k ? "," : "", theta[static_cast<size_t>(k)]);
    std::printf("],\"grads\":[");
    for (int s = 0; s < steps; ++s) {
      std::printf("%s[", s ? "," : "");
      for (int k = 0; k < p; ++k) std::printf("%s%.17g", k ? "," : "", grads[static_cast<size_t>(s)][static_cast<size_t>(k)]);
      std::printf("]");
    }
    std::printf("],\"iterates\":[");
    for (int s = 0; s < steps; ++s) {
      detail::apply_update(c.spec, st, theta, grads[static_cast<size_t>(s)], pmin, pmax);
      std::printf("%s[", s ? "," : "");
      for (int k = 0; k < p; ++k) std::printf("%s%.17g", k ? "," : "", theta[static_cast<size_t>(k)]);
      std::printf("]");
    }
    std::printf("]}");
  }
  std::printf("]\n");
  return 0;
}
