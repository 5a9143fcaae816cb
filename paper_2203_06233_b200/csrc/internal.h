// internal.h -- host-side declarations shared by the translation units of libstap.so
// (not part of the C ABI).
#pragma once
#include <stddef.h>
#include <stdint.h>

#include "../../include/stap.h"

namespace stapk {

// Output geometry of a plan (include/stap.h: out [batch][dop_count][S][R] complex64).
struct PlanOutGeom {
  int32_t batch, dop_count, S, R, device;
  size_t out_bytes;
};
bool plan_out_geom(const stap_plan* plan, PlanOutGeom* g);

}  // namespace stapk
