// FGMRES vector kernels (krylov.py:88-182) and the 1D ILU(0) sweeps
// (krylov.py:219-233), float64.
//
// Reductions are two-stage and deterministic: a fixed element partition
// (a function of n and the SM count only, never of the batch) writes
// per-block partials, and one CTA per system sums them in a fixed order,
// so a system's results do not depend on which other systems share the
// launch (batched == serial, bitwise).
#include "common.cuh"

namespace mdp {

enum OrthMode { DOT = 0, UPD_DOT = 1, UPD_NORM = 2, NORM = 3 };

inline int red_blocks(int64_t n) {
  int nb = ceil_div(n, 1024);
  int cap = 2 * sm_count();
  return nb < 1 ? 1 : (nb > cap ? cap : nb);
}

// One pass over V[0..nv) and w for a block's chunk of elements.
//   DOT:      acc_k = sum V_k w
//   UPD_DOT:  w <- w - sum c_k V_k ; acc_k = sum V_k w
//   UPD_NORM: w <- w - sum c_k V_k ; acc_0 = sum w^2
//   NORM:     acc_0 = sum w^2
template <int NV, int MODE>
__global__ void __launch_bounds__(128) orth_pass_kernel(const int32_t* sel, const double* __restrict__ V,
                                                         int64_t ldv_sys, int64_t ldv_vec,
                                                         const int32_t* __restrict__ nvs, double* w,
                                                         int64_t ldw, int64_t n,
                                                         const double* __restrict__ coef, int cstride,
                                                         double* __restrict__ partial, int pstride) {
  __shared__ double sh[32];
  __shared__ double csh[NV > 0 ? NV : 1];
  const int i = blockIdx.y;
  const int s = sys_of(sel, i);
  const int nv = nvs ? nvs[i] : 0;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = blockIdx.x * chunk, e1 = min(n, e0 + chunk);
  const double* Vs = V ? V + s * ldv_sys : nullptr;
  double* ws = w + s * ldw;
  if (MODE == UPD_DOT || MODE == UPD_NORM) {
    for (int k = threadIdx.x; k < NV; k += blockDim.x) csh[k] = k < nv ? coef[i * cstride + k] : 0.0;
    __syncthreads();
  }
  constexpr int NACC = (MODE == DOT || MODE == UPD_DOT) ? (NV > 0 ? NV : 1) : 1;
  double acc[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    double we = ws[e];
    if (MODE == UPD_DOT || MODE == UPD_NORM) {
#pragma unroll
      for (int k = 0; k < NV; ++k)
        if (k < nv) we -= csh[k] * __ldg(Vs + k * ldv_vec + e);
      ws[e] = we;
    }
    if (MODE == DOT || MODE == UPD_DOT) {
#pragma unroll
      for (int k = 0; k < NACC; ++k)
        if (k < nv) acc[k] += __ldg(Vs + k * ldv_vec + e) * we;
    } else {
      acc[0] += we * we;
    }
  }
  double* out = partial + ((int64_t)i * gridDim.x + blockIdx.x) * pstride;
#pragma unroll
  for (int k = 0; k < NACC; ++k) {
    if (NACC > 1 && k >= nv) break;
    double t = block_sum(acc[k], sh);
    if (threadIdx.x == 0) out[k] = t;
  }
}

// out[i][k] = sum_b partial[i][b][k] in block order; one CTA per system.
__global__ void reduce_partials_kernel(const double* __restrict__ partial, int nblk, int pstride,
                                       int nk, double* __restrict__ out, int ostride) {
  const int i = blockIdx.x;
  for (int k = threadIdx.x; k < nk; k += blockDim.x) {
    double t = 0.0;
    const double* p = partial + (int64_t)i * nblk * pstride + k;
    for (int b = 0; b < nblk; ++b) t += p[(int64_t)b * pstride];
    out[i * ostride + k] = t;
  }
}

// hcol[i][k] = h1 + h2 (k < nv), hcol[i][kmax+1] = ||w||
__global__ void arnoldi_finalize_kernel(const int32_t* __restrict__ nvs, const double* h1,
                                        const double* h2, const double* nrm2, int kmax,
                                        double* hcol) {
  const int i = blockIdx.x;
  const int nv = nvs[i];
  for (int k = threadIdx.x; k <= kmax; k += blockDim.x)
    hcol[i * (kmax + 2) + k] = k < nv ? h1[i * (kmax + 1) + k] + h2[i * (kmax + 1) + k] : 0.0;
  if (threadIdx.x == 0) hcol[i * (kmax + 2) + kmax + 1] = sqrt(nrm2[i]);
}

// V[s][nv] = w / hn  (and vcur), exact division like krylov.py:165
__global__ void arnoldi_next_kernel(const int32_t* sel, double* V, int64_t ldv_sys, int64_t ldv_vec,
                                    const int32_t* __restrict__ nvs, int kmax,
                                    const double* __restrict__ w, int64_t ldw, int64_t n,
                                    const double* __restrict__ hcol, double* vcur, int64_t ldc) {
  const int i = blockIdx.y;
  const int s = sys_of(sel, i);
  const int nv = nvs[i];
  const double hn = hcol[i * (kmax + 2) + kmax + 1];
  double* dst = nv <= kmax ? V + s * ldv_sys + nv * ldv_vec : nullptr;
  const double* ws = w + s * ldw;
  double* vc = vcur ? vcur + s * ldc : nullptr;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double v = ws[e] / hn;
    if (dst) dst[e] = v;
    if (vc) vc[e] = v;
  }
}

template <int MODE>
static void launch_orth(int nv_max, dim3 grid, cudaStream_t st, const int32_t* sel, const double* V,
                        int64_t ldv_sys, int64_t ldv_vec, const int32_t* nvs, double* w, int64_t ldw,
                        int64_t n, const double* coef, int cstride, double* partial, int pstride) {
#define MDP_ORTH(NVT)                                                                            \
  orth_pass_kernel<NVT, MODE><<<grid, 128, 0, st>>>(sel, V, ldv_sys, ldv_vec, nvs, w, ldw, n, \
                                                    coef, cstride, partial, pstride)
  if (MODE == NORM) {
    MDP_ORTH(0);
  } else if (nv_max <= 4) {
    MDP_ORTH(4);
  } else if (nv_max <= 8) {
    MDP_ORTH(8);
  } else if (nv_max <= 16) {
    MDP_ORTH(16);
  } else if (nv_max <= 32) {
    MDP_ORTH(32);
  } else {
    MDP_ORTH(64);
  }
#undef MDP_ORTH
}

// ---------------------------------------------------------------------------

__global__ void scale_kernel(const int32_t* sel, const double* __restrict__ x, int64_t ldx,
                             const double* __restrict__ num, const double* __restrict__ den,
                             double* __restrict__ y, int64_t ldy, int64_t n) {
  const int i = blockIdx.y;
  const int s = sys_of(sel, i);
  const double* xs = x + s * ldx;
  double* ys = y + s * ldy;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    ys[e] = den ? xs[e] / den[i] : xs[e] * num[i];
  }
}

__global__ void basis_update_kernel(const int32_t* sel, double* x, int64_t ldx,
                                    const double* __restrict__ Z, int64_t ldz_sys, int64_t ldz_vec,
                                    const int32_t* __restrict__ cnt, const double* __restrict__ y,
                                    int ystride, int64_t n) {
  const int i = blockIdx.y;
  const int s = sys_of(sel, i);
  const int c = cnt[i];
  if (c <= 0) return;
  double* xs = x + s * ldx;
  const double* Zs = Z + s * ldz_sys;
  const double* ys = y + i * ystride;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int k = 0; k < c; ++k) t += __ldg(Zs + k * ldz_vec + e) * ys[k];
    xs[e] += t;
  }
}

// r = b - y, partial sum of squares
__global__ void __launch_bounds__(128) residual_kernel(const int32_t* sel, const double* __restrict__ b,
                                                        const double* __restrict__ y, double* r,
                                                        int64_t ld, int64_t n, double* partial) {
  __shared__ double sh[32];
  const int i = blockIdx.y;
  const int s = sys_of(sel, i);
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = blockIdx.x * chunk, e1 = min(n, e0 + chunk);
  double acc = 0.0;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    double v = b[s * ld + e] - y[s * ld + e];
    r[s * ld + e] = v;
    acc += v * v;
  }
  double t = block_sum(acc, sh);
  if (threadIdx.x == 0) partial[(int64_t)i * gridDim.x + blockIdx.x] = t;
}

__global__ void sqrt_kernel(double* v, int m) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) v[i] = sqrt(v[i]);
}

__global__ void axpby_kernel(const int32_t* sel, double a, const double* __restrict__ x, double b,
                             double* y, int64_t ld, int64_t n) {
  const int s = sys_of(sel, blockIdx.y);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double yv = b == 0.0 ? 0.0 : b * y[s * ld + e];
    y[s * ld + e] = a * x[s * ld + e] + yv;
  }
}

__global__ void copy_vec_kernel(const int32_t* sel, const double* __restrict__ src, int64_t lds,
                                double* __restrict__ dst, int64_t ldd, const int32_t* __restrict__ slot,
                                int64_t slot_stride, int64_t n) {
  const int i = blockIdx.y;
  const int s = sys_of(sel, i);
  const double* a = src + s * lds;
  double* d = dst + s * ldd + (slot ? (int64_t)slot[i] * slot_stride : 0);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    d[e] = a[e];
}

// ILU(0) sweeps, one CTA per system, level-scheduled.  The per-row
// arithmetic is the reference's sequential sum with explicitly rounded
// operations (no FMA contraction), so results equal krylov.ilu0_apply
// bitwise.
__global__ void __launch_bounds__(256) ilu0_apply_kernel(const mdp_ilu F, const int32_t* sel,
                                                          const double* __restrict__ r,
                                                          double* __restrict__ z, int64_t ld) {
  extern __shared__ double xsh[];
  const int s = sys_of(sel, blockIdx.x);
  const int rs = F.row_start[s], nrow = F.row_start[s + 1] - rs;
  const double* rp = r + s * ld;
  const int* levf = F.lev_f + (int64_t)s * F.lev_stride;  // nlev+1 boundaries
  const int* levb = F.lev_b + (int64_t)s * F.lev_stride;
  const int* pf = F.perm_f + rs;
  const int* pb = F.perm_b + rs;
  for (int L = 0; L < F.nlev_f[s]; ++L) {
    for (int t = levf[L] + threadIdx.x; t < levf[L + 1]; t += blockDim.x) {
      int row = pf[t];
      int g = rs + row;
      double acc = rp[row];
      for (int p = F.ptr[g]; p < F.diag[g]; ++p) acc = __dsub_rn(acc, __dmul_rn(F.val[p], xsh[F.col[p]]));
      xsh[row] = acc;
    }
    __syncthreads();
  }
  for (int L = 0; L < F.nlev_b[s]; ++L) {
    for (int t = levb[L] + threadIdx.x; t < levb[L + 1]; t += blockDim.x) {
      int row = pb[t];
      int g = rs + row;
      double acc = xsh[row];
      for (int p = F.diag[g] + 1; p < F.ptr[g + 1]; ++p)
        acc = __dsub_rn(acc, __dmul_rn(F.val[p], xsh[F.col[p]]));
      xsh[row] = __ddiv_rn(acc, F.val[F.diag[g]]);
    }
    __syncthreads();
  }
  double* zp = z + s * ld;
  for (int t = threadIdx.x; t < nrow; t += blockDim.x) zp[t] = xsh[t];
}

inline dim3 ew_grid(int64_t n, int nsel) {
  int bx = ceil_div(n, 256);
  int cap = 4 * sm_count();
  bx = bx > cap ? cap : bx;
  return dim3(bx < 1 ? 1 : bx, nsel);
}

}  // namespace mdp

using namespace mdp;

extern "C" size_t mdp_arnoldi_work_bytes(int32_t nsel, int32_t kmax, int64_t n) {
  int nb = red_blocks(n);
  size_t partial = (size_t)nsel * nb * 65;
  size_t small = (size_t)nsel * (2 * (kmax + 1) + 1);
  return (partial + small) * sizeof(double) + 256;
}

extern "C" int mdp_arnoldi(int32_t nsel, const int32_t* sel, double* V, int64_t ldv_sys,
                           int64_t ldv_vec, const int32_t* nv, int32_t kmax, double* w, int64_t ldw,
                           int64_t n, double* hcol, double* vcur, int64_t ldc, void* work,
                           void* stream) {
  MDP_REQUIRE(kmax >= 1 && kmax <= 63, "kmax %d outside [1, 63]", kmax);
  MDP_REQUIRE(n > 0, "empty vectors");
  if (nsel == 0) return MDP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = red_blocks(n);
  const int pstride = 65;
  double* partial = (double*)work;
  double* h1 = partial + (size_t)nsel * nb * pstride;
  double* h2 = h1 + (size_t)nsel * (kmax + 1);
  double* nrm2 = h2 + (size_t)nsel * (kmax + 1);
  dim3 grid(nb, nsel);
  const int nvmax = kmax + 1;
  launch_orth<DOT>(nvmax, grid, st, sel, V, ldv_sys, ldv_vec, nv, w, ldw, n, nullptr, 0, partial, pstride);
  MDP_LAUNCH_CHECK("orth_pass DOT");
  reduce_partials_kernel<<<nsel, 64, 0, st>>>(partial, nb, pstride, kmax + 1, h1, kmax + 1);
  MDP_LAUNCH_CHECK("reduce_partials");
  launch_orth<UPD_DOT>(nvmax, grid, st, sel, V, ldv_sys, ldv_vec, nv, w, ldw, n, h1, kmax + 1, partial,
                       pstride);
  MDP_LAUNCH_CHECK("orth_pass UPD_DOT");
  reduce_partials_kernel<<<nsel, 64, 0, st>>>(partial, nb, pstride, kmax + 1, h2, kmax + 1);
  MDP_LAUNCH_CHECK("reduce_partials");
  launch_orth<UPD_NORM>(nvmax, grid, st, sel, V, ldv_sys, ldv_vec, nv, w, ldw, n, h2, kmax + 1, partial,
                        pstride);
  MDP_LAUNCH_CHECK("orth_pass UPD_NORM");
  reduce_partials_kernel<<<nsel, 32, 0, st>>>(partial, nb, pstride, 1, nrm2, 1);
  MDP_LAUNCH_CHECK("reduce_partials");
  arnoldi_finalize_kernel<<<nsel, 64, 0, st>>>(nv, h1, h2, nrm2, kmax, hcol);
  MDP_LAUNCH_CHECK("arnoldi_finalize");
  arnoldi_next_kernel<<<ew_grid(n, nsel), 256, 0, st>>>(sel, V, ldv_sys, ldv_vec, nv, kmax, w, ldw, n,
                                                         hcol, vcur, ldc);
  MDP_LAUNCH_CHECK("mdp_arnoldi");
  return MDP_OK;
}

extern "C" int mdp_norms(int32_t nsel, const int32_t* sel, const double* x, int64_t ldx, int64_t n,
                         double* out, void* work, void* stream) {
  if (nsel == 0) return MDP_OK;
  MDP_REQUIRE(n > 0, "empty vectors");
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = red_blocks(n);
  double* partial = (double*)work;
  orth_pass_kernel<0, NORM><<<dim3(nb, nsel), 128, 0, st>>>(sel, nullptr, 0, 0, nullptr,
                                                            const_cast<double*>(x), ldx, n, nullptr, 0,
                                                            partial, 1);
  MDP_LAUNCH_CHECK("orth_pass NORM");
  reduce_partials_kernel<<<nsel, 32, 0, st>>>(partial, nb, 1, 1, out, 1);
  MDP_LAUNCH_CHECK("reduce_partials");
  sqrt_kernel<<<ceil_div(nsel, 128), 128, 0, st>>>(out, nsel);
  MDP_LAUNCH_CHECK("mdp_norms");
  return MDP_OK;
}

extern "C" int mdp_scale(int32_t nsel, const int32_t* sel, const double* x, int64_t ldx,
                         const double* num, const double* den, double* y, int64_t ldy, int64_t n,
                         void* stream) {
  if (nsel == 0) return MDP_OK;
  MDP_REQUIRE(num || den, "scale needs num or den");
  scale_kernel<<<ew_grid(n, nsel), 256, 0, (cudaStream_t)stream>>>(sel, x, ldx, num, den, y, ldy, n);
  MDP_LAUNCH_CHECK("mdp_scale");
  return MDP_OK;
}

extern "C" int mdp_basis_update(int32_t nsel, const int32_t* sel, double* x, int64_t ldx,
                                const double* Z, int64_t ldz_sys, int64_t ldz_vec, const int32_t* cnt,
                                const double* y, int32_t ystride, int64_t n, void* stream) {
  if (nsel == 0) return MDP_OK;
  basis_update_kernel<<<ew_grid(n, nsel), 256, 0, (cudaStream_t)stream>>>(sel, x, ldx, Z, ldz_sys,
                                                                          ldz_vec, cnt, y, ystride, n);
  MDP_LAUNCH_CHECK("mdp_basis_update");
  return MDP_OK;
}

extern "C" int mdp_residual(int32_t nsel, const int32_t* sel, const double* b, const double* y,
                            double* r, int64_t ld, int64_t n, double* rn, void* work, void* stream) {
  if (nsel == 0) return MDP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = red_blocks(n);
  double* partial = (double*)work;
  residual_kernel<<<dim3(nb, nsel), 128, 0, st>>>(sel, b, y, r, ld, n, partial);
  MDP_LAUNCH_CHECK("residual_kernel");
  reduce_partials_kernel<<<nsel, 32, 0, st>>>(partial, nb, 1, 1, rn, 1);
  MDP_LAUNCH_CHECK("reduce_partials");
  sqrt_kernel<<<ceil_div(nsel, 128), 128, 0, st>>>(rn, nsel);
  MDP_LAUNCH_CHECK("mdp_residual");
  return MDP_OK;
}

extern "C" int mdp_axpby(int32_t nsel, const int32_t* sel, double a, const double* x, double b,
                         double* y, int64_t ld, int64_t n, void* stream) {
  if (nsel == 0) return MDP_OK;
  axpby_kernel<<<ew_grid(n, nsel), 256, 0, (cudaStream_t)stream>>>(sel, a, x, b, y, ld, n);
  MDP_LAUNCH_CHECK("mdp_axpby");
  return MDP_OK;
}

extern "C" int mdp_copy_vec(int32_t nsel, const int32_t* sel, const double* src, int64_t lds,
                            double* dst, int64_t ldd, const int32_t* dst_slot, int64_t slot_stride,
                            int64_t n, void* stream) {
  if (nsel == 0) return MDP_OK;
  copy_vec_kernel<<<ew_grid(n, nsel), 256, 0, (cudaStream_t)stream>>>(sel, src, lds, dst, ldd, dst_slot,
                                                                      slot_stride, n);
  MDP_LAUNCH_CHECK("mdp_copy_vec");
  return MDP_OK;
}

extern "C" int mdp_ilu0_apply(const mdp_ilu* f, int32_t nsel, const int32_t* sel, const double* r,
                              double* z, int64_t ld, void* stream) {
  MDP_REQUIRE(f != nullptr, "null ILU descriptor");
  if (nsel == 0) return MDP_OK;
  // shared memory holds one system's solution; 1D blocks here are <= ~8k rows
  const int smem = 64 * 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ilu0_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  ilu0_apply_kernel<<<nsel, 256, smem, (cudaStream_t)stream>>>(*f, sel, r, z, ld);
  MDP_LAUNCH_CHECK("mdp_ilu0_apply");
  return MDP_OK;
}
