// solve.cu -- the chol.cuh solver kernels (K2 for N >= 13) in a translation unit of their own:
// every CholCfg instantiation of STAPK_CHOL_CFGS compiles here, in parallel with stap_abi.cu.
#include "chol.cuh"
#include "internal.h"

namespace stapk {

cudaError_t solve_chol_set_attr(const CholSel& sel) { return chol_set_attr(sel); }

void solve_chol_launch(const CholSel& sel, int grid, cudaStream_t st, int N, int S, long long units,
                       const float2* cov, const float2* steer, float2* w, float* g, int32_t* info) {
  chol_launch(sel, grid, st, N, S, units, cov, steer, w, g, info);
}

}  // namespace stapk
