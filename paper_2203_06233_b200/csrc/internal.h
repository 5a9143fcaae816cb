// internal.h -- host-side declarations shared by the translation units of libstap.so
// (not part of the C ABI).
#pragma once
#include <stddef.h>
#include <stdint.h>

#include <cuda_runtime.h>

#include "../../include/stap.h"

namespace stapk {

// Output geometry of a plan (include/stap.h: out [batch][dop_count][S][R] complex64).
struct PlanOutGeom {
  int32_t batch, dop_count, S, R, device;
  size_t out_bytes;
};
bool plan_out_geom(const stap_plan* plan, PlanOutGeom* g);

// The chol.cuh solver kernels live in their own translation unit (solve.cu) so that they
// compile in parallel with the rest; `sel` is a CholSel from chol_select (chol.cuh).
struct CholSel;
cudaError_t solve_chol_set_attr(const CholSel& sel);
void solve_chol_launch(const CholSel& sel, int grid, cudaStream_t st, int N, int S, long long units,
                       const float2* cov, const float2* steer, float2* w, float* g, int32_t* info);

}  // namespace stapk
