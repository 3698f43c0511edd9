// Test infrastructure (oracle) — force-included (-include) into the reference
// scenario.cpp only. Pulls in every header that TU needs first (so include
// guards keep them untouched), then renames three tokens so the Driver's
// calls land in the forwarding hooks of ref_shim.cpp.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>
#include <fstream>
#include <functional>
#include <memory>
#include <numeric>
#include <set>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include <json.hpp>

#include "kvrail/far_view.hpp"
#include "kvrail/metrics.hpp"
#include "kvrail/placement.hpp"
#include "kvrail/sim_engine.hpp"
#include "kvrail/workload.hpp"
#include "ref_hook_decl.hpp"

#define Pager HookedPager
#define stage kvr_hook_stage
#define reduce kvr_hook_reduce
