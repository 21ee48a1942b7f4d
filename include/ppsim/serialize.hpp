// Drop-in path of the reference's ppsim/serialize.hpp (serialize.hpp:18-165): the
// deterministic JSON emitters of timelines and analysis reports, as nlohmann::ordered_json
// values with the reference's key order and number formatting, plus timeline_csv
// (ppsim/ppsim.hpp).  Like the reference, this header needs nlohmann/json on the include
// path (e.g. -I<site-packages>/include/cudnn_frontend/thirdparty); nothing in libamdp.so
// depends on it (the library's own JSON text comes from timeline_json_text()).
//
// Not provided: the delayed-optimizer report emitters (verdict_json, trace_csv,
// scaling_json, bound_json, lipschitz_json; serialize.hpp:167-235) — their analytic harness
// (optim.hpp:23-152, 270-556) is outside the AMDP training path.
#pragma once

#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include <nlohmann/json.hpp>

#include "ppsim/ppsim.hpp"

namespace ppsim {

using ordered_json = nlohmann::ordered_json;

// An integral Rat is a JSON integer; any other is the string "num/den".
inline ordered_json rat_json(const Rat& r) {
  return r.den() == 1 ? ordered_json(r.num()) : ordered_json(r.str());
}

inline std::string format_double(double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.12g", v);
  return buf;
}

inline ordered_json timeline_json(const Timeline& t) {
  ordered_json devices = ordered_json::array();
  for (const auto& events : t.per_device) {
    ordered_json row = ordered_json::array();
    for (const TaskEvent& e : events)
      row.push_back(ordered_json{{"kind", kind_name(e.kind)}, {"stage", e.stage}, {"minibatch", e.minibatch},
                                 {"pipeline", e.pipeline}, {"window", e.window}, {"preloaded", e.preloaded},
                                 {"start", rat_json(e.start)}, {"duration", rat_json(e.duration)}});
    devices.push_back(std::move(row));
  }
  return ordered_json{{"policy", policy_name(t.policy)}, {"depth", t.depth}, {"devices", t.devices},
                      {"threshold", t.threshold}, {"makespan", rat_json(t.makespan)},
                      {"per_device", std::move(devices)}};
}

inline ordered_json mismatch_json(const MismatchReport& r) {
  ordered_json entries = ordered_json::array(), stages = ordered_json::array(), missing = ordered_json::array();
  for (const auto& kv : r.entries)
    entries.push_back(ordered_json{{"stage", kv.first.first}, {"minibatch", kv.first.second},
                                   {"updates_between", kv.second}});
  for (const auto& kv : r.max_per_stage) stages.push_back(ordered_json{{"stage", kv.first}, {"max", kv.second}});
  for (const auto& sm : r.missing) missing.push_back(ordered_json{{"stage", sm.first}, {"minibatch", sm.second}});
  return ordered_json{{"entries", std::move(entries)}, {"max_per_stage", std::move(stages)},
                      {"max_overall", r.max_overall()}, {"missing_backward", std::move(missing)}};
}

inline ordered_json window_json(const WindowReport& r) {
  ordered_json windows = ordered_json::array();
  for (const WindowEntry& w : r.windows)
    windows.push_back(ordered_json{{"window", w.window}, {"window_size", w.window_size},
                                   {"update_count", w.update_count}, {"mismatched_minibatches", w.mismatched}});
  return ordered_json{{"windows", std::move(windows)}};
}

inline ordered_json memory_json(const MemoryReport& r) {
  ordered_json devices = ordered_json::array();
  for (const DeviceMemory& d : r.per_device)
    devices.push_back(ordered_json{{"weight", rat_json(d.weight)}, {"activation_peak", rat_json(d.activation_peak)},
                                   {"gradient", rat_json(d.gradient)},
                                   {"optimizer_state", rat_json(d.optimizer_state)}});
  const Table1View& c = r.table1;
  return ordered_json{{"per_device", std::move(devices)},
                      {"closed_form", ordered_json{{"bubble", c.bubble ? rat_json(*c.bubble) : ordered_json(nullptr)},
                                                   {"weight_min", rat_json(c.weight_min)},
                                                   {"weight_max", rat_json(c.weight_max)},
                                                   {"activation_peak", rat_json(c.activation_peak)}}}};
}

}  // namespace ppsim
