// kvrail-b200 — bounded far-history summaries and the attention oracle.
//
// Drop-in for the reference's kvrail/far_view.hpp (far_view.hpp:27-75). A
// token image is 2*L*d_kv float lanes, per layer [K_l | V_l]. On the B200 the
// summaries are produced by the K-far kernel and consumed by the window
// attention kernel; these host functions define the results (summaries
// bit-exact, attention within 1e-3 relative).
#pragma once

#include <cstdint>
#include <functional>
#include <span>
#include <vector>

#include "kvrail/types.hpp"

namespace kvrail {

struct FarViewConfig {
    bool enabled = false;
    uint32_t near_window = 512;  // W*
    uint32_t cap = 64;           // far representatives
    uint32_t chunk_tokens = 128; // sv_chunk
    void validate() const;
};

/// Elementwise mean of `count` token images (double accumulation).
std::vector<float> summarize_chunk(std::span<const float> tokens, uint32_t lanes, uint64_t count);

struct ViewSlot {
    bool padded = true;
    uint64_t origin = 0; // near: token index; far: chunk id
    std::vector<float> image;
};

struct SummarizedView {
    uint32_t visible_width = 0; // W* + cap
    uint32_t lanes = 0;
    uint32_t near_count = 0;
    uint32_t far_count = 0;
    std::vector<ViewSlot> slots; // [far chunks ascending..., near tokens oldest first...]
};

using TokenReader = std::function<void(uint64_t token, float *out)>;

SummarizedView build_view(const TokenReader &read, uint64_t history_tokens,
                          const std::vector<double> &chunk_scores, uint32_t lanes,
                          const FarViewConfig &cfg);

std::vector<float> attend(const SummarizedView &view, std::span<const float> query,
                          uint32_t layer, uint32_t kv_head_dim);

std::vector<uint64_t> select_chunks(const std::vector<double> &chunk_scores, uint32_t cap);

} // namespace kvrail
