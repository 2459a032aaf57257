// Geometric multigrid baseline preconditioner (krylov.py:302-387) on the
// device: Galerkin levels P^T A P are host-built CSR matrices (the reference's
// own construction), the V-cycle runs on these kernels.  Every row is summed
// by one thread in CSR index order, so results are deterministic and follow
// scipy's csr_matvec order.  Off the north-star hot path: the comparator the
// paper's tables set the neural preconditioner against.
#include "common.cuh"

namespace mdp {

__device__ __forceinline__ double csr_row(const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                          const double* __restrict__ val, const double* __restrict__ x, int i) {
  double s = 0.0;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) s += val[k] * x[col[k]];
  return s;
}

// xo = x + (omega (r - A x)) / d  (x == NULL: xo = (omega r) / d), krylov.py:296-298
__global__ void csr_jacobi_kernel(int n, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                  const double* __restrict__ val, const double* __restrict__ d,
                                  const double* __restrict__ r, const double* __restrict__ x,
                                  double* __restrict__ xo, double omega) {
  MDP_PDL_ENTER();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (x)
      xo[i] = x[i] + (omega * (r[i] - csr_row(ptr, col, val, x, i))) / d[i];
    else
      xo[i] = (omega * r[i]) / d[i];
  }
}

// res = r - A x
__global__ void csr_residual_kernel(int n, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                    const double* __restrict__ val, const double* __restrict__ r,
                                    const double* __restrict__ x, double* __restrict__ res) {
  MDP_PDL_ENTER();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    res[i] = r[i] - csr_row(ptr, col, val, x, i);
}

// y = A x, or y = y + A x
__global__ void csr_spmv_kernel(int n, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
                                int accumulate) {
  MDP_PDL_ENTER();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double s = csr_row(ptr, col, val, x, i);
    y[i] = accumulate ? y[i] + s : s;
  }
}

// coarsest level: y = M x with M the host-inverted (tiny) coarse matrix, one warp per row
__global__ void dense_matvec_kernel(int n, const double* __restrict__ M, const double* __restrict__ x,
                                    double* __restrict__ y) {
  MDP_PDL_ENTER();
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += gridDim.x * (blockDim.x >> 5)) {
    double s = 0.0;
    for (int k = lane; k < n; k += 32) s += M[(int64_t)i * n + k] * x[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[i] = s;
  }
}

static dim3 rows_grid(int n) {
  int b = ceil_div(n, 256);
  const int cap = 8 * sm_count();
  return dim3(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace mdp

using namespace mdp;

extern "C" int mdp_csr_jacobi(int32_t n, const int32_t* ptr, const int32_t* col, const double* val, const double* d,
                              const double* r, const double* x, double* xo, double omega, void* stream) {
  MDP_REQUIRE(n >= 0 && ptr && col && val && d && r && xo, "csr jacobi: null argument");
  if (n == 0) return MDP_OK;
  ::mdp::launch_k(csr_jacobi_kernel, rows_grid(n), 256, 0, (cudaStream_t)stream, n, ptr, col, val, d, r, x, xo,
                  omega);
  MDP_LAUNCH_CHECK("csr_jacobi_kernel");
  return MDP_OK;
}

extern "C" int mdp_csr_residual(int32_t n, const int32_t* ptr, const int32_t* col, const double* val,
                                const double* r, const double* x, double* res, void* stream) {
  MDP_REQUIRE(n >= 0 && ptr && col && val && r && x && res, "csr residual: null argument");
  if (n == 0) return MDP_OK;
  ::mdp::launch_k(csr_residual_kernel, rows_grid(n), 256, 0, (cudaStream_t)stream, n, ptr, col, val, r, x, res);
  MDP_LAUNCH_CHECK("csr_residual_kernel");
  return MDP_OK;
}

extern "C" int mdp_csr_spmv(int32_t n, const int32_t* ptr, const int32_t* col, const double* val, const double* x,
                            double* y, int32_t accumulate, void* stream) {
  MDP_REQUIRE(n >= 0 && ptr && col && val && x && y, "csr spmv: null argument");
  if (n == 0) return MDP_OK;
  ::mdp::launch_k(csr_spmv_kernel, rows_grid(n), 256, 0, (cudaStream_t)stream, n, ptr, col, val, x, y,
                  (int)accumulate);
  MDP_LAUNCH_CHECK("csr_spmv_kernel");
  return MDP_OK;
}

extern "C" int mdp_dense_matvec(int32_t n, const double* M, const double* x, double* y, void* stream) {
  MDP_REQUIRE(n >= 0 && M && x && y, "dense matvec: null argument");
  if (n == 0) return MDP_OK;
  ::mdp::launch_k(dense_matvec_kernel, dim3(ceil_div(n, 8)), 256, 0, (cudaStream_t)stream, n, M, x, y);
  MDP_LAUNCH_CHECK("dense_matvec_kernel");
  return MDP_OK;
}
