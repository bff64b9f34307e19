// diag.h -- tuning / diagnostic environment knobs, compiled in only with
// -DLCMA_DIAG (tools/ builds for experiments).  The product build reads no
// environment: every setting that changes what a plan runs is fixed at plan
// time from lcma_plan_desc.
#pragma once
#include <cstdlib>

namespace lcma {
inline const char* diag_env(const char* name) {
#ifdef LCMA_DIAG
    return std::getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}
}  // namespace lcma
