// Shared helpers for the mdp_b200 CUDA sources (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/mdp_b200.h"

namespace mdp {

void set_error(const char* fmt, ...);
void note_launch();

// every kernel launch is followed by check_launch, which also counts it
// (mdp_launch_count: the bench reports how many of our kernels ran)
inline int check_launch(const char* what) {
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return MDP_ECUDA;
  }
  return MDP_OK;
}

#define MDP_REQUIRE(cond, ...)       \
  do {                               \
    if (!(cond)) {                   \
      ::mdp::set_error(__VA_ARGS__); \
      return MDP_EINVAL;             \
    }                                \
  } while (0)

#define MDP_LAUNCH_CHECK(what)                    \
  do {                                            \
    int _rc = ::mdp::check_launch(what);          \
    if (_rc) return _rc;                          \
  } while (0)

__device__ __forceinline__ int sys_of(const int32_t* sel, int i) { return sel ? sel[i] : i; }

// Programmatic dependent launch (opt-in, MDP_PDL=1): kernels are launched
// with programmatic stream serialisation (also inside captured CUDA graphs),
// so the next grid is scheduled while this one drains.  Each kernel enters
// with MDP_PDL_ENTER(): wait until the preceding grid has completed and its
// memory is visible, then allow the following grid to launch (both are
// no-ops for a normal launch).  Nothing touches global memory before the
// wait, so the ordering is the plain stream order.
#define MDP_PDL_ENTER()                                             \
  do {                                                              \
    asm volatile("griddepcontrol.wait;" ::: "memory");              \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
  } while (0)

bool pdl_enabled();  // MDP_PDL=0 disables the attribute (A/B timing)

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<Args&&>(args)...);
}

// Launch as a programmatic dependent of the previous kernel in the stream regardless of MDP_PDL: the
// kernel itself decides how much of its prologue (loads of launch-invariant data only) runs before its
// griddepcontrol.wait.
template <typename... KArgs, typename... Args>
inline void launch_k_dependent(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                               Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<Args&&>(args)...);
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

int sm_count();

// Deterministic block reduction of a double (blockDim.x multiple of 32, <= 1024).
__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    int nw = blockDim.x >> 5;
    t = lane < nw ? sh[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;  // valid in thread 0
}

}  // namespace mdp
