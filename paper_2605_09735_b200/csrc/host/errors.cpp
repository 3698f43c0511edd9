// kvrail-b200 error names (contract: types.cpp:20-46 of the reference).
#include "kvrail/types.hpp"

namespace kvrail {

const char *errc_name(Errc c) {
    static const char *const names[] = {
        "OutOfPages",      "PrefixOutOfRange", "AliasOverlap",  "UnmappedRange",
        "FutureDelta",     "UnknownSession",   "SessionClosed", "EmptyChunk",
        "DimensionMismatch", "ShapeViolation", "MultiCommit",   "UnmappedBlock",
        "ParseError",      "NonMonotoneTime",  "EmptyStream",   "UnknownRegime",
        "InfeasibleSpec",  "WorkloadAuditFailed", "EmptyRun",   "WorkloadMismatch",
        "BadConfig",       "IoError",
    };
    const auto i = static_cast<unsigned>(c);
    return i < sizeof(names) / sizeof(names[0]) ? names[i] : "UnknownError";
}

} // namespace kvrail
