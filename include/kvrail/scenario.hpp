// kvrail-b200 — end-to-end serving scenario: the per-step Driver that calls
// the hot path (pager verbs -> one commit per session -> stage/reduce ->
// fixed-shape step).
//
// Drop-in for the reference's kvrail/scenario.hpp (scenario.hpp:31-117). The
// Driver is a twin of scenario.cpp:124-683: with the same config and events it
// makes the same pager/transport calls in the same order, so steps.csv,
// report.json and the per-step parity trace are byte-identical to the
// reference's. With `b200.device >= 0` the fixed-shape "kernel" is real: a
// captured CUDA graph per step on the B200 (kvrail/device_step.hpp).
#pragma once

#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "kvrail/far_view.hpp"
#include "kvrail/metrics.hpp"
#include "kvrail/pager.hpp"
#include "kvrail/placement.hpp"
#include "kvrail/sim_engine.hpp"
#include "kvrail/transport.hpp"
#include "kvrail/workload.hpp"

namespace kvrail {

/// B200 extension of the scenario (JSON key "b200"; ignored by the reference).
struct B200Config {
    int device = -1;          // CUDA device; < 0 = host-only twin driver (run_scenario: the
                              // KVRAIL_B200_DEVICE environment variable, when set)
    uint32_t kv_heads = 0;    // 0: 1 head of kv_head_dim
    uint32_t head_dim = 0;    // 0: kv_head_dim / kv_heads
    uint32_t q_heads = 0;     // 0: kv_heads (MHA); GQA group = q_heads / kv_heads
    std::string payload = "bytes"; // "bytes": reference fill_token_payload; "lanes": float
                                   // lane pattern rounded to dtype (finite for attention);
                                   // "wide": the same bytes as lanes of [-16, 16) (peaked softmax)
    std::string query = "exact";   // decode queries: "exact" in the KV type | "f32" (24-bit)
    std::string transfer = "reference"; // transfer groups: "reference" (exact byte abutment,
                                        // bit-exact with the reference) | "page_runs" (B200
                                        // policy: physically consecutive pages merge across
                                        // page-end slack, TransportConfig::run_page_bytes)
    std::string dtype = "auto";    // fp16 | bf16 | fp32 | auto (elem_bytes 4 -> fp32, 2 -> fp16)
    bool trace = false;            // record the per-step parity trace
    bool attention = true;         // run the window attention kernel each step
    std::string attention_kernel = "auto"; // auto | cuda_core | tcgen05 (GQA groups, head_dim 128)
    uint32_t ring_rows = 0;        // window ring rows per (slot, layer); 0 = auto
    uint64_t max_tokens = 0;       // per-slot token capacity of the device page table; 0 = auto
    uint32_t graph = 1;            // replay the step as a captured CUDA graph
    bool check = false;            // compare the device K-scan with host reduce() every step
    uint64_t prefill_budget = 0;   // cold prompt rows written per step (deferred queue); 0 = all
    std::string utility = "synthetic"; // placement observations: "synthetic" (the reference's,
                                       // scenario.cpp:526-529) | "attention" (K-mass, measured)
    int32_t utility_layer = -1;    // K-mass probe layer; < 0 = the last layer
    uint32_t utility_every = 1;    // K-mass runs on steps with step % utility_every == 0
    uint32_t shard_rank = 0;       // requests shard by sequence across GPUs:
    uint32_t shard_world = 1;      //   this rank keeps request_id % world == rank
};

/// Keep this rank's share of an event stream (request_id % world == rank).
std::vector<TraceEvent> shard_events(const std::vector<TraceEvent> &events, uint32_t rank,
                                     uint32_t world);

struct ScenarioConfig {
    std::string label = "run";
    PagerConfig pager;
    PlacementConfig placement;
    TransportConfig transport;
    FarViewConfig far_view;
    CostModel cost;
    std::optional<WorkloadSpec> workload;
    std::optional<std::string> trace_path;
    double replay_window_seconds = 0.0;
    bool pager_enabled = true;
    FragRegime regime = FragRegime::contiguous;
    uint64_t steps = 2000;
    Step warmup_steps = 100;
    uint64_t seed = 1;
    double step_ms = 20.0;
    uint32_t span_blocks = 9;
    uint32_t staged_refresh_period = 32;
    uint32_t demand_refresh_period = 16;
    uint32_t demand_gather_tokens = 46;
    double share_probability = 0.3;
    uint32_t shared_prefix_tokens = 64;
    uint32_t static_slot_tokens = 2816;
    uint32_t arena_headroom_pages = 1024;
    std::optional<uint32_t> arena_pages_override;
    Step eos_burst_step = 0;
    double eos_burst_fraction = 0.5;
    B200Config b200;

    void validate() const;
    uint32_t compiled_width() const {
        return far_view.enabled ? far_view.near_window + far_view.cap : far_view.near_window;
    }
};

struct RunResult {
    ScenarioConfig config;
    RunReport report;
    std::vector<StepRecord> records;
    WorkloadAudit workload_audit;
    WorkCounters pager_counters;
};

RunResult run_scenario(const ScenarioConfig &cfg);
std::vector<TraceEvent> resolve_events(const ScenarioConfig &cfg);
RunResult run_scenario_on(const ScenarioConfig &cfg, const std::vector<TraceEvent> &events);

std::string report_to_json(const RunResult &result);
std::string report_to_text(const RunResult &result);
std::string steps_to_csv(const std::vector<StepRecord> &records);
/// The reference steps.csv columns followed by the B200 measurements of each step
/// (device time, inter-token latency, per-phase device time, bytes moved), so a
/// simulated run and a measured run compare column for column.
std::string measured_steps_csv(const std::vector<StepRecord> &records);
/// Measured counterpart of report.json over the post-warm-up steps: decode tok/s on
/// device time, device step and inter-token latency percentiles (nearest rank,
/// metrics.cpp:23-33) beside the modeled ones, attention and gather bandwidth.
std::string measured_report_json(const std::vector<StepRecord> &records, uint64_t warmup_steps);
std::string delta_to_text(const DeltaReport &d);
void write_file(const std::string &path, const std::string &content);

ScenarioConfig config_from_json_file(const std::string &path);
ScenarioConfig config_from_json_text(const std::string &text);
std::string config_to_json(const ScenarioConfig &cfg);
ScenarioConfig default_audit_config();

class DeviceStep;

/// Steppable twin of the reference Driver (scenario.cpp:124-683).
class ScenarioDriver {
public:
    ScenarioDriver(const ScenarioConfig &cfg, std::vector<TraceEvent> events);
    ~ScenarioDriver();
    ScenarioDriver(const ScenarioDriver &) = delete;
    ScenarioDriver &operator=(const ScenarioDriver &) = delete;

    /// Run Driver::step for the next step index and return its record.
    StepRecord step();
    bool done() const;
    uint64_t steps_done() const;
    const ScenarioConfig &config() const;
    const std::vector<StepRecord> &records() const;
    /// Record of an executed step, completed with its device measurements
    /// (waits for the device if that step is still in flight).
    const StepRecord &record(uint64_t step);
    const std::vector<TraceEvent> &events() const;
    /// Parity trace text; empty unless b200.trace.
    const std::string &trace() const;
    RunResult result() const;
    Pager *pager() const;
    DeviceStep *device() const;
    struct LiveInfo {
        uint32_t slot;
        SessionId session;
        uint64_t written;
    };
    std::vector<LiveInfo> live() const;
    /// b200.check results: steps checked, mismatching steps, first mismatch.
    void device_check(uint64_t &checked, uint64_t &mismatches, std::string &first) const;
    /// b200.trace on a device: staged tokens whose trace hash was read from K-gather's
    /// destination (window ring / far rows), near rows behind the live window (read from
    /// the arena: not part of the window), and rows missing from the window otherwise.
    void staged_rows(uint64_t &delivered, uint64_t &behind, uint64_t &missing) const;
    /// Join the per-step counts all-reduce over NCCL (kvr_comm_init) before the first
    /// step; records then carry job-wide counts and the single-commit audit is job-wide.
    void comm_init(const uint8_t id[128], int rank, int world);
    /// Test hook (kvr_dev_fault): corrupt K-gather on every later step.
    void fault(int what, uint64_t arg);

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

} // namespace kvrail
