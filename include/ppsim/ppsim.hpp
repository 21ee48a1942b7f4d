// ppsim-compatible C++ API of the AMDP-B200 engine (namespace ppsim).
//
// Drop-in for the reference's header-only library (/root/reference/proj/include/ppsim):
// same type names, fields, function names, argument meaning and exception behaviour
// (invalid_argument for bad configuration/usage, runtime_error for cycles/deadlock,
// overflow_error/domain_error from Rat).  The implementation is this repository's own
// (paper_2605_29664_b200/csrc/sched/*.cpp): e.g. `simulate` dispatches from per-device
// ordered ready sets in O(N log N) instead of the reference's O(N * |ready|) scan, with
// the identical dispatch rule, so its timelines are byte-identical (tests/test_sched_*).
//
// What the reference cannot do and this library adds: `ppsim::execute` (amdp/engine.hpp)
// runs a TaskGraph on B200s and returns the same `Timeline` type with measured times, so
// every analysis below applies unchanged to a real run.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "ppsim/rat.hpp"

#define PPSIM_API __attribute__((visibility("default")))

namespace ppsim {

// types.hpp:15 — event kinds; the enum order is the dispatch tie-break rank (types.hpp:18)
enum class Kind : std::uint8_t { Forward, Backward, Reduce, Broadcast, Update };
inline int kind_rank(Kind k) { return static_cast<int>(k); }
PPSIM_API const char* kind_name(Kind k);

// types.hpp:31-38
enum class Policy : std::uint8_t { AMDP, DAPPLE, GPipe, Interleaved1F1B, Chimera, PipeDreamAsync };
PPSIM_API const char* policy_name(Policy p);
PPSIM_API std::optional<Policy> policy_from_name(const std::string& s);

// types.hpp:60-109 — the declared cost model a schedule is built and ordered under
struct ClusterSpec {
  int depth = 0;
  int devices = 0;
  std::vector<Rat> fwd_cost;
  std::vector<Rat> bwd_cost;
  Rat update_cost = Rat(0);
  Rat comm_cost = Rat(0);
  std::vector<std::vector<int>> nodes;
  std::optional<Rat> inter_node_cost;

  PPSIM_API static ClusterSpec uniform(int depth, int devices, Rat fwd, Rat bwd,
                                       Rat update = Rat(0), Rat comm = Rat(0));
  PPSIM_API int node_of(int device) const;
  PPSIM_API Rat gap(int from_device, int to_device) const;
  PPSIM_API Rat mean_fwd() const;
  PPSIM_API Rat mean_bwd() const;
};

// types.hpp:111-119 — the partition/policy configuration
struct PolicyConfig {
  Policy policy = Policy::DAPPLE;
  int injection_limit = 1;
  int num_pipelines = 1;
  int accumulation_threshold = 1;
  int num_minibatches = 1;
  bool zero_enabled = false;
  bool injection_override = false;
};

// builder.hpp:17-26
struct Task {
  Kind kind = Kind::Forward;
  int stage = 0;
  int minibatch = 0;  // Reduce/Broadcast/Update: window index
  int pipeline = 0;
  int device = 0;
  Rat duration;
  int window = 0;
  bool preloaded = false;
};

// builder.hpp:28-37
struct TaskGraph {
  Policy policy = Policy::DAPPLE;
  int depth = 0;
  int devices = 0;
  int threshold = 1;
  std::vector<Task> tasks;
  std::vector<std::pair<int, int>> deps;  // (pred, succ)
  std::vector<std::vector<int>> lanes;    // strict per-replica orders (non-AMDP policies)

  // builder.hpp:38-76: per-device merge of lanes by dispatch key
  PPSIM_API std::vector<std::vector<int>> fifo_hint() const;
};

// types.hpp:121-133
struct TaskEvent {
  Kind kind = Kind::Forward;
  int stage = 0;
  int minibatch = 0;
  int pipeline = 0;
  int device = 0;
  Rat start;
  Rat duration;
  bool preloaded = false;
  int window = 0;
  Rat finish() const { return start + duration; }
};

// types.hpp:135-150
struct Timeline {
  Policy policy = Policy::DAPPLE;
  int depth = 0;
  int devices = 0;
  int threshold = 1;
  std::vector<std::vector<TaskEvent>> per_device;
  Rat makespan;
  int window_of(const TaskEvent& e) const { return e.window; }
  PPSIM_API std::vector<TaskEvent> flat() const;
};

// types.hpp:152-207 — reports
struct MismatchReport {
  std::map<std::pair<int, int>, int> entries;
  std::map<int, int> max_per_stage;
  std::vector<std::pair<int, int>> missing;
  PPSIM_API int max_overall() const;
};
struct MemoryModel {
  Rat weight_per_stage{1};
  Rat activation_per_stage_per_minibatch{1};
  Rat optimizer_state_multiplier{2};
  Rat gradient_multiplier{1};
};
struct WindowEntry {
  int window = 0;
  std::vector<int> mismatched;
  int window_size = 0;
  int update_count = 0;
};
struct WindowReport {
  std::vector<WindowEntry> windows;
};
struct DeviceMemory {
  Rat weight;
  Rat activation_peak;
  Rat gradient;
  Rat optimizer_state;
};
struct Table1View {
  std::optional<Rat> bubble;
  Rat weight_min;
  Rat weight_max;
  Rat activation_peak;
};
struct MemoryReport {
  std::vector<DeviceMemory> per_device;
  Table1View table1;
};
struct CommVolume {
  Rat reduce;
  Rat broadcast;
  Rat allreduce;
};
// types.hpp:204-207 — outcome of a property check
struct Verdict {
  bool pass = false;
  std::string detail;
};

// ---- validate.hpp
PPSIM_API std::vector<std::string> validate_cluster(const ClusterSpec& c);
PPSIM_API std::vector<std::string> validate_policy(const PolicyConfig& p, const ClusterSpec& c);
PPSIM_API std::vector<std::string> validate_causality(const Timeline& t, const ClusterSpec& c);
PPSIM_API std::vector<std::string> validate_non_overlap(const Timeline& t);

// ---- builder.hpp
PPSIM_API int map_stage_to_device(int pipeline, int stage, int depth);
PPSIM_API int default_num_pipelines(int depth);
PPSIM_API Rat active_ratio(int injection_limit, int depth);
PPSIM_API int preload_count(const Rat& bwd, const Rat& fwd);
PPSIM_API TaskGraph build(const PolicyConfig& cfg, const ClusterSpec& cl);

// ---- engine.hpp
PPSIM_API Timeline simulate(const TaskGraph& g, const ClusterSpec& cl);
// Same as simulate, also returning the global dispatch order (task ids).  The dispatch
// order is a topological order of g; the GPU executor replays it.
PPSIM_API Timeline simulate_with_order(const TaskGraph& g, const ClusterSpec& cl,
                                       std::vector<int>* order);
PPSIM_API Rat bubble_ratio(const Timeline& tl, int warmup_windows = 0);

// ---- analysis.hpp
PPSIM_API MismatchReport mismatch_report(const Timeline& t);
PPSIM_API WindowReport window_mismatch(const Timeline& t, int depth);
PPSIM_API MemoryReport memory_report(const Timeline& t, const PolicyConfig& policy,
                                     const MemoryModel& mem);
PPSIM_API CommVolume reduce_broadcast_cost(int replicas, const Rat& bytes);
// analysis.hpp:96-121: PipeDreamAsync steady staleness = min(n, depth - stage) - 1 per stage
PPSIM_API Verdict verify_steady_mismatch(int depth, int injection_limit);
// analysis.hpp:161-221: AMDP's one-step bound under random costs, comm gaps, node
// partitions, device relabelings and ring reflections (deterministic in `seed`)
PPSIM_API Verdict verify_topology_invariance(int depth, int trials, std::uint64_t seed);

// ---- serialize.hpp (the trace wire format; the nlohmann::ordered_json emitters of the
// reference — timeline_json, mismatch_json, window_json, memory_json, rat_json — are in
// ppsim/serialize.hpp, which needs nlohmann/json on the include path like the reference's)
PPSIM_API std::string timeline_csv(const Timeline& t);
// timeline_json(t).dump() of the reference, as text (no nlohmann dependency)
PPSIM_API std::string timeline_json_text(const Timeline& t);
// Version trace: timeline_csv with start/duration dropped and a `version` column
// (parameter updates of the stage visible to the task) appended.  Byte-comparable
// between the reference's simulated order and a measured GPU run.
PPSIM_API std::string version_trace_csv(const Timeline& t);

}  // namespace ppsim
