// Test infrastructure (oracle) — NOT product code.
//
// Declarations shared by the reference build's scenario.cpp translation unit
// (via ref_hook.hpp, force-included) and ref_shim.cpp. They let the shim
// observe the UNMODIFIED reference Driver (scenario.cpp:124-683) from the
// outside: the Pager it constructs (scenario.cpp:226) and every stage()/
// reduce() call it makes (scenario.cpp:662-664). Nothing in the reference's
// behaviour changes: the hooks forward to the real functions.
#pragma once

#include <cstdint>
#include <vector>

#include "kvrail/pager.hpp"
#include "kvrail/transport.hpp"

namespace kvrail {

class HookedPager : public Pager {
public:
    explicit HookedPager(PagerConfig cfg);
};

std::vector<Descriptor> kvr_hook_stage(const std::vector<StageNeed> &needs, uint64_t page_bytes,
                                       uint64_t token_bytes, double now);
std::vector<DmaTrain> kvr_hook_reduce(std::vector<Descriptor> descriptors,
                                      const TransportConfig &cfg, double now);

} // namespace kvrail
