// kvrail-b200 — where a Pager keeps page payload bytes.
//
// The reference Pager owns lazily materialised host pages (pager.hpp:200,
// pager.cpp:247-254). Here the metadata (allocator, refcounts, views) stays on
// the host — block ids must be bit-exact with the reference allocator — while
// the bytes live behind this interface: HostPayloadStore for CPU use and the
// device arena (kvrail/device_step.hpp) on a B200. The Pager reports every
// byte-level event (fresh page, COW copy, token write, commit of a view) here.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <span>
#include <vector>

#include "kvrail/types.hpp"

namespace kvrail {

/// One committed mapping change, resolved: tokens [tok_begin, tok_end) map
/// to `block` starting at slot `slot_begin`, or are unmapped when block ==
/// kInvalidBlock. Emitted after a frame commit so a device mirror of the
/// committed view can be updated without re-deriving the edit journal.
struct ViewEdit {
    uint64_t tok_begin = 0;
    uint64_t tok_end = 0;
    BlockId block = kInvalidBlock;
    uint32_t slot_begin = 0;
};

/// A token write whose payload is produced where the bytes live (the device
/// payload generator) instead of being copied from a host buffer.
struct GeneratedWrite {
    SessionId session = 0;
    uint64_t token = 0;     // logical token of the first slot
    BlockId block = kInvalidBlock;
    uint32_t slot = 0;
    uint32_t count = 0;     // consecutive slots in `block`
    uint32_t source = 0;    // 0 = synthetic token payload, 1 = far-view summary job
    uint64_t aux = 0;       // source-specific (summary: chunk begin token)
    /// summary jobs: the chunk's rows as global slots (block * tokens_per_page + slot)
    /// in the committed view the summary reads (resolved by the caller)
    std::span<const uint32_t> src_slots;
};

class PayloadStore {
public:
    virtual ~PayloadStore() = default;
    /// Pages handed out by the allocator read as zeros (pager.cpp:181-184).
    virtual void on_alloc(BlockId head, uint32_t count) = 0;
    /// Copy-on-write: whole-page copy (pager.cpp:622-629).
    virtual void copy_page(BlockId src, BlockId dst) = 0;
    /// Host payload for `count` consecutive slots of one block.
    virtual void write(BlockId block, uint32_t slot, uint32_t count, const std::byte *bytes) = 0;
    /// Payload generated in place (device stores only).
    virtual void write_generated(const GeneratedWrite &w);
    virtual void read(BlockId block, uint32_t slot, uint32_t count, std::byte *out) = 0;
    /// Committed-view delta of one session (after frame_commit).
    virtual void on_commit(SessionId, bool eos, std::span<const ViewEdit>) {}
};

/// Lazily materialised host pages; unmaterialised pages read as zeros.
class HostPayloadStore final : public PayloadStore {
public:
    HostPayloadStore(uint32_t pages, uint64_t page_bytes, uint64_t token_bytes);
    void on_alloc(BlockId head, uint32_t count) override;
    void copy_page(BlockId src, BlockId dst) override;
    void write(BlockId block, uint32_t slot, uint32_t count, const std::byte *bytes) override;
    void read(BlockId block, uint32_t slot, uint32_t count, std::byte *out) override;

private:
    uint64_t page_bytes_, token_bytes_;
    std::vector<std::unique_ptr<std::byte[]>> pages_;
};

} // namespace kvrail
