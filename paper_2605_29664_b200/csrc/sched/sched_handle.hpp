// Internal: the object behind an `amdp_schedule*` handle.
#pragma once

#include <string>
#include <vector>

#include "amdp_sched.h"
#include "ppsim/ppsim.hpp"

namespace amdp {

struct SchedHandle {
  ppsim::ClusterSpec cl;
  ppsim::PolicyConfig cfg;
  ppsim::TaskGraph g;
  ppsim::Timeline tl;
  std::vector<int> order;  // dispatch order of g under cl
  bool has_graph = false;
  bool has_timeline = false;
};

ppsim::Rat from_c(const amdp_rat& r);
ppsim::ClusterSpec cluster_from_c(const amdp_cluster_spec* c);
ppsim::PolicyConfig policy_from_c(const amdp_policy_config* p);
std::string report_json(const ppsim::Timeline& tl, const ppsim::ClusterSpec& cl,
                        const ppsim::PolicyConfig& cfg, int warmup);

}  // namespace amdp
