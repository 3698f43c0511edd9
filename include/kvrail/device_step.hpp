// kvrail-b200 — the B200 side of one decode step, as seen from host C++.
//
// Replaces the reference's fixed-shape device stub SimEngine::execute_step
// (sim_engine.cpp:33-72) with real work on an sm_100a GPU. Everything the
// host decided during a step (allocations, copy-on-write, token writes,
// committed view deltas, staging needs, far-view selections) is sealed into
// ONE committed step descriptor in pinned host memory, published with one
// cudaMemcpyAsync and consumed by a captured CUDA graph:
//
//   K-apply   zero recycled slots, copy-on-write pages          (arena)
//   K-write   generate the step's token payloads into the arena and
//             the per-slot window ring                          (arena, ring)
//   K-far     far-view chunk summaries into summary slots       (arena)
//   K-map     apply committed view edits to the device page table
//   K-prime   fill window rows not covered by this step's writes
//   K-scan    stage+reduce on device: descriptors and train boundaries
//   K-gather  move each train's pages into the fixed-shape window
//   K-attn    fixed-shape window attention for every slot
//
// The host never waits for a step before building the next one; it reads the
// step's small record (counters, device time) one step later.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <span>
#include <vector>

#include "kvrail/payload_store.hpp"
#include "kvrail/transport.hpp"
#include "kvr_cuda.h"
#include "kvrail_c.h"

namespace kvrail {

struct DeviceStepStats {
    uint64_t step = 0;
    double device_ms = 0.0;     // CUDA-event time of the step's device work
    double gather_ms = 0.0;     // K-gather alone
    double attn_ms = 0.0;       // K-attn alone
    double phase_ms[8] = {};    // kvr_step_stats::phase_ms
    uint32_t trains = 0;        // computed by K-scan
    uint32_t descriptors = 0;
    uint64_t train_bytes = 0;   // sum of train bytes (gather read side)
    uint64_t writeback_tokens = 0;
    uint64_t attn_bytes = 0;    // KV bytes the attention read
    uint64_t h2d_bytes = 0;     // committed descriptor bytes published this step
    uint32_t scan_status = 0;   // 0 ok; else capacity overflow flags
    uint64_t end_ns = 0;        // device %globaltimer at the end of the step
    int64_t global_counts[KVR_COUNTS] = {}; // KVR_COUNT_* summed over the communicator
};

class DeviceStep {
public:
    explicit DeviceStep(const kvr_geometry &geometry);
    ~DeviceStep();
    DeviceStep(const DeviceStep &) = delete;
    DeviceStep &operator=(const DeviceStep &) = delete;

    const kvr_geometry &geometry() const;
    kvr_dev *handle() const;
    /// Payload store over the device arena (give it to the Pager).
    std::shared_ptr<PayloadStore> store();

    /// Mirror session `sid`'s committed view into device slot `slot`.
    void bind(SessionId sid, uint32_t slot);
    void unbind(SessionId sid);

    // ---- per-step inputs (cleared by launch) ----
    void slot_state(uint32_t slot, SessionId sid, uint64_t written, bool live);
    void need(uint32_t slot, SessionId sid, TrainKind kind, std::span<const StagedSpan> spans,
              std::span<const uint64_t> first_tokens);
    /// Window rows [tok_begin, tok_end) of `slot` copied from the arena (an aliased
    /// prefix): `rows` holds each token's source row as a global slot (block *
    /// tokens_per_page + slot, KVR_NO_SLOT: unmapped) in the committed view. `src`: the
    /// session owning those rows (the alias source) — its pending rows are written
    /// before K-prime reads them.
    static constexpr SessionId kNoPrimeSource = 0xffffffffu;
    void prime(uint32_t slot, uint64_t tok_begin, uint64_t tok_end, SessionId src, std::span<const uint32_t> rows);
    void far_selection(uint32_t slot, std::span<const uint64_t> chunk_ids);

    /// This GPU's per-step counts (KVR_COUNT_*), carried in the next launched descriptor
    /// and all-reduced inside its graph when a communicator is set.
    void counts(const int64_t c[KVR_COUNTS]);
    /// Join the per-step counts all-reduce (kvr_comm_init) before the first launch.
    void comm_init(const uint8_t id[128], int rank, int world);
    /// Seal the step descriptor, publish it and launch the step (async).
    void launch(uint64_t step, double now, const TransportConfig &tc);
    /// Stats of `step` (blocks until that step has finished on the device).
    DeviceStepStats collect(uint64_t step);
    /// Wait for all launched work.
    void sync();
    /// Whether `step` is the last step launched from its ring slot.
    bool launched(uint64_t step) const;
    /// Attention-utility observations K-mass measured in `step` (geometry.utility):
    /// (block, softmax mass of the probe layer, mean over q-heads) per run of window
    /// rows, for the slots whose session `keep` accepts. Waits for the step.
    std::vector<std::pair<BlockId, double>> utility(uint64_t step,
                                                    const std::function<bool(SessionId)> &keep);
    /// The same, per device slot (empty for slots that were not live).
    std::vector<std::vector<kvr_mass_run>> utility_runs(uint64_t step);
    /// Flush byte ops queued outside a step (Pager API use without a Driver).
    void flush();
    /// Write at most `tokens` cold prompt rows per step (0 = all of them, the
    /// default). Rows behind the window wait in a queue; a row is forced out
    /// before a gather, far summary, page copy or host read touches it, and
    /// dropped when its page is recycled.
    void set_prefill_budget(uint64_t tokens);
    uint64_t deferred_tokens() const; // queued now
    uint64_t dropped_tokens() const;  // never written: their page was recycled before any read

    // ---- parity / inspection (synchronous) ----
    void read_arena(uint64_t offset, uint64_t bytes, void *out);
    void read_ring_token(uint32_t slot, uint64_t token, void *out); // token image (tb bytes)
    void read_page_table(uint32_t slot, uint64_t tok_begin, uint64_t count, uint32_t *out);
    void read_attention(uint32_t slot, float *out); // [L][Hq][hd]
    void read_query(uint32_t slot, float *out);     // [L][Hq][hd]
    void read_far_row(uint32_t slot, uint64_t chunk, void *out); // token image of a far row
    /// Far chunks the last launched step showed to the attention of `slot`.
    std::vector<uint64_t> far_selection_of(uint32_t slot) const;
    /// Last K-scan result: trains (desc_begin/count index `descs`).
    void read_scan(std::vector<kvr_train> &trains, std::vector<kvr_descriptor> &descs);
    /// K-gather's destination bytes of the last step's staged tokens [tok_begin, +count)
    /// in train order, token-major (kvr_dev_read_staged); in_window[i] = 0 for a token
    /// with a row the window does not hold (read from the arena instead).
    void read_staged(uint64_t tok_begin, uint64_t count, void *out, uint8_t *in_window);
    /// Test hook (kvr_dev_fault): KVR_FAULT_DROP_SPAN / KVR_FAULT_SHIFT_ROWS in K-gather.
    void fault(int what, uint64_t arg);

    struct Impl; // public so the arena-backed PayloadStore can reach it

private:
    std::unique_ptr<Impl> impl_;
};

} // namespace kvrail
