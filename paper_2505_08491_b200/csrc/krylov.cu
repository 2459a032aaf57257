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

enum OrthMode { DOT = 0, UPD_DOT = 1, UPD_NORM = 2, NORM = 3, DOT_SOLVE = 4, UPD_DOT_NORM = 5 };

// orth-pass tuning (tools/arnoldi_ab.py, profiles/): blocks per SM cap, elements per
// thread step (2 = 16-byte loads), independent basis loads per batch
#ifndef ORTH_CAP
#define ORTH_CAP 4
#endif
#ifndef ORTH_VEC
#define ORTH_VEC 2
#endif
#ifndef ORTH_KB
#define ORTH_KB 8
#endif

#ifndef ORTH_ELEMS
#define ORTH_ELEMS 256  // elements per reduction block before the ORTH_CAP x SMs cap (256 vs 512: -2.5% cfg2 solve)
#endif

// Reduction partition: blocks of a power-of-two chunk (>= ORTH_ELEMS elements)
// chosen from the power-of-two band of n, so a longer zero-padded tail (a batch
// whose 1D parts are longer) only adds trailing blocks with zero partials: the
// summation order of a system's real entries does not depend on the batch.
inline int64_t red_chunk(int64_t n) {
  int64_t c = ORTH_ELEMS;
  const int64_t cap = (int64_t)ORTH_CAP * sm_count();
  while ((n + c - 1) / c > cap) c *= 2;
  return c;
}

inline int red_blocks(int64_t n) {
  const int64_t nb = (n + red_chunk(n) - 1) / red_chunk(n);
  return nb < 1 ? 1 : (int)nb;
}

// Deterministic grid reduction without a second launch: every block
// writes its partial row, the last block to finish (atomic ticket per
// system) sums the partials in a fixed order (lane-strided, then a
// shuffle tree) and resets the ticket.  The order depends on n and the SM
// count only, never on the batch.
struct RedOut {
  double* out;      // [nsel][ostride]
  int ostride;
  int nk;           // entries to reduce
  int mode;         // 0 plain, 1 sqrt, 2 arnoldi finalize (out = ||w||^2),
                    // 3 MGS coefficients from the Gram rows, 4 new Gram row + ||w||
  const double* h1; // mode 2: the two projections, [nsel][kmax+1]
  const double* h2;
  double* hcol;     // modes 2-4: [nsel][kmax+2] Hessenberg column + ||w||
  int kmax;
  const int32_t* nvs;
  double* gram;     // modes 3, 4: [nsys][kmax+1][kmax+1], row m = V_m . V_c for c < m
  const int32_t* sel;
};

template <int NL = 0>
__device__ __forceinline__ void finish_reduction(const double* __restrict__ partial, int pstride,
                                                 unsigned int* ticket, const RedOut& R, const double* mine) {
  __shared__ bool last;
  __shared__ double Ls[NL > 0 ? NL * (NL + 1) : 1];  // mode 3: Gram rows, padded row stride
  const int i = blockIdx.y;
  if (threadIdx.x < R.nk) {
    double* dst = const_cast<double*>(partial) + ((int64_t)i * gridDim.x + blockIdx.x) * pstride;
    dst[threadIdx.x] = mine[threadIdx.x];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&ticket[i], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // tpk threads per entry (a power of two <= 32, all in one warp), each
  // summing a fixed block-strided subset with independent loads in flight,
  // then a fixed xor-shuffle tree: the order depends on n and the SM count only
  int tpk = 32;
  while (tpk > 1 && tpk * R.nk > (int)blockDim.x) tpk >>= 1;
  const int k = threadIdx.x / tpk, j = threadIdx.x % tpk;
  const double* base = partial + (int64_t)i * gridDim.x * pstride;
  const int nblk = gridDim.x;
  double t = 0.0;
  if (k < R.nk) {
    int b = j;
    for (; b + 3 * tpk < nblk; b += 4 * tpk) {
      const double p0 = __ldcg(base + (int64_t)b * pstride + k);
      const double p1 = __ldcg(base + (int64_t)(b + tpk) * pstride + k);
      const double p2 = __ldcg(base + (int64_t)(b + 2 * tpk) * pstride + k);
      const double p3 = __ldcg(base + (int64_t)(b + 3 * tpk) * pstride + k);
      t += p0;
      t += p1;
      t += p2;
      t += p3;
    }
    for (; b < nblk; b += tpk) t += __ldcg(base + (int64_t)b * pstride + k);
  }
  for (int o = tpk >> 1; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (k < R.nk && j == 0) R.out[i * R.ostride + k] = R.mode == 1 ? sqrt(t) : t;
  if (R.mode == 2) {  // hcol[k] = h1 + h2 (k < nv), hcol[kmax+1] = ||w||
    __syncthreads();
    const int nv = R.nvs[i];
    for (int k = threadIdx.x; k <= R.kmax; k += blockDim.x)
      R.hcol[i * (R.kmax + 2) + k] = k < nv ? R.h1[i * (R.kmax + 1) + k] + R.h2[i * (R.kmax + 1) + k] : 0.0;
    if (threadIdx.x == 0) R.hcol[i * (R.kmax + 2) + R.kmax + 1] = sqrt(R.out[i * R.ostride]);
  }
  if constexpr (NL > 0) {
    // Modified Gram-Schmidt from ONE pass of dot products (krylov.py:138-140):
    // the sequential projections h_m = V_m . (w - sum_{c<m} h_c V_c) equal
    // h_m = a_m - sum_{c<m} (V_m . V_c) h_c with a = V^T w, i.e. the unit lower
    // triangular system (I + L) h = a over the strictly lower Gram rows L kept
    // from the previous steps of this cycle.  Column-oriented forward
    // substitution in one warp (lane l owns entries l and l + 32), fixed order.
    const int nv = R.nvs[i];
    const int s = sys_of(R.sel, i);
    const double* G = R.gram + (int64_t)s * (R.kmax + 1) * (R.kmax + 1);
    for (int t2 = threadIdx.x; t2 < nv * nv; t2 += blockDim.x) {
      const int m = t2 / nv, c = t2 - m * nv;
      if (c < m) Ls[m * (NL + 1) + c] = __ldcg(G + m * (R.kmax + 1) + c);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int l = threadIdx.x;
      double* a = R.out + i * R.ostride;
      double x0 = l < nv ? a[l] : 0.0, x1 = (NL > 32 && l + 32 < nv) ? a[l + 32] : 0.0;
      for (int c = 0; c < nv; ++c) {
        const double hc = __shfl_sync(0xffffffffu, c < 32 ? x0 : x1, c & 31);
        if (l > c && l < nv) x0 -= Ls[l * (NL + 1) + c] * hc;
        if (NL > 32 && l + 32 > c && l + 32 < nv) x1 -= Ls[(l + 32) * (NL + 1) + c] * hc;
      }
      if (l < nv) a[l] = x0;
      if (NL > 32 && l + 32 < nv) a[l + 32] = x1;
      for (int k = l; k <= R.kmax; k += 32)
        R.hcol[i * (R.kmax + 2) + k] = k < nv ? (k < 32 ? x0 : x1) : 0.0;
    }
  }
  if (R.mode == 4) {  // out[0..nv) = V^T w', out[nv] = ||w'||^2: Gram row of the new vector w'/||w'||
    __syncthreads();
    const int nv = R.nvs[i];
    const int s = sys_of(R.sel, i);
    const double hn = sqrt(R.out[i * R.ostride + nv]);
    double* G = R.gram + (int64_t)s * (R.kmax + 1) * (R.kmax + 1) + (int64_t)nv * (R.kmax + 1);
    if (nv <= R.kmax && hn > 0.0)
      for (int k = threadIdx.x; k < nv; k += blockDim.x) G[k] = R.out[i * R.ostride + k] / hn;
    if (threadIdx.x == 0) R.hcol[i * (R.kmax + 2) + R.kmax + 1] = hn;
  }
  if (threadIdx.x == 0) ticket[i] = 0u;
}

// Sum each of N per-lane values over the warp.  N >= 32: transpose
// reduction (31 shuffles per 32 values), afterwards lane l holds the sum of
// value (g * 32 + l) in v[g * 32]; N < 32: one xor tree per value, every lane
// holds every sum.  Fixed order either way.
template <int N>
__device__ __forceinline__ void warp_sums(double* v) {
  if constexpr (N >= 32) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int g = 0; g < N / 32; ++g) {
      double* u = v + g * 32;
#pragma unroll
      for (int off = 16, cnt = 16; off >= 1; off >>= 1, cnt >>= 1) {
        const bool upper = lane & off;
#pragma unroll
        for (int j = 0; j < cnt; ++j) {
          const double send = upper ? u[j] : u[j + cnt];
          const double keep = upper ? u[j + cnt] : u[j];
          u[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
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
                                                         double* __restrict__ partial, int pstride,
                                                         unsigned int* ticket, RedOut R, int64_t chunk) {
  MDP_PDL_ENTER();
  constexpr bool UPD = MODE == UPD_DOT || MODE == UPD_NORM || MODE == UPD_DOT_NORM;
  constexpr bool DOTS = MODE == DOT || MODE == UPD_DOT || MODE == DOT_SOLVE || MODE == UPD_DOT_NORM;
  constexpr bool BOTH = MODE == UPD_DOT_NORM;  // dots and ||w||^2 in the same pass
  constexpr int NACC = DOTS ? (NV > 0 ? NV : 1) : 1;
  __shared__ double csh[NV > 0 ? NV : 1];
  __shared__ double wsum[4][NACC + 1];
  __shared__ double mine[NACC + 1];
  const int i = blockIdx.y;
  const int s = sys_of(sel, i);
  const int nv = nvs ? nvs[i] : 0;
  // chunk: red_chunk(n), a power of two >= 256 (even: 16-byte aligned pairs)
  const int64_t e0 = blockIdx.x * chunk, e1 = min(n, e0 + chunk);
  const double* Vs = V ? V + s * ldv_sys : nullptr;
  double* ws = w + s * ldw;
  if (UPD) {
    for (int k = threadIdx.x; k < NV; k += blockDim.x) csh[k] = k < nv ? coef[i * cstride + k] : 0.0;
    __syncthreads();
  }
  double acc[NACC];
  double accn = 0.0;
#pragma unroll
  for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
  // Each thread walks element pairs (16-byte loads: longer contiguous runs per
  // basis vector per warp), the basis values of one element batch loaded in
  // groups of KB independent loads ahead of their FMAs.  Per element the
  // operation order is that of a plain k loop.
  constexpr int KB = NV < ORTH_KB ? (NV > 0 ? NV : 1) : ORTH_KB;
  for (int64_t e = e0 + ORTH_VEC * threadIdx.x; e < e1; e += ORTH_VEC * blockDim.x) {
    if (ORTH_VEC == 2 && e + 1 < e1) {
      double2 w2 = *reinterpret_cast<const double2*>(ws + e);
      if (UPD) {
#pragma unroll
        for (int k0 = 0; k0 < NV; k0 += KB) {
          double2 vv[KB];
#pragma unroll
          for (int j = 0; j < KB; ++j)
            vv[j] = k0 + j < nv ? __ldg(reinterpret_cast<const double2*>(Vs + (k0 + j) * ldv_vec + e))
                                : make_double2(0.0, 0.0);
#pragma unroll
          for (int j = 0; j < KB; ++j)
            if (k0 + j < nv) {
              w2.x -= csh[k0 + j] * vv[j].x;
              w2.y -= csh[k0 + j] * vv[j].y;
            }
        }
        *reinterpret_cast<double2*>(ws + e) = w2;
      }
      if (BOTH) {
        accn += w2.x * w2.x;
        accn += w2.y * w2.y;
      }
      if (DOTS) {
#pragma unroll
        for (int k0 = 0; k0 < NACC; k0 += KB) {
          double2 vv[KB];
#pragma unroll
          for (int j = 0; j < KB; ++j)
            vv[j] = k0 + j < nv ? __ldg(reinterpret_cast<const double2*>(Vs + (k0 + j) * ldv_vec + e))
                                : make_double2(0.0, 0.0);
#pragma unroll
          for (int j = 0; j < KB; ++j)
            if (k0 + j < nv) {
              acc[k0 + j] += vv[j].x * w2.x;
              acc[k0 + j] += vv[j].y * w2.y;
            }
        }
      } else {
        acc[0] += w2.x * w2.x;
        acc[0] += w2.y * w2.y;
      }
      continue;
    }
    for (int64_t f = e; f < e + ORTH_VEC && f < e1; ++f) {
      double we = ws[f];
      if (UPD) {
#pragma unroll
        for (int k0 = 0; k0 < NV; k0 += KB) {
          double vv[KB];
#pragma unroll
          for (int j = 0; j < KB; ++j) vv[j] = k0 + j < nv ? __ldg(Vs + (k0 + j) * ldv_vec + f) : 0.0;
#pragma unroll
          for (int j = 0; j < KB; ++j)
            if (k0 + j < nv) we -= csh[k0 + j] * vv[j];
        }
        ws[f] = we;
      }
      if (BOTH) accn += we * we;
      if (DOTS) {
#pragma unroll
        for (int k0 = 0; k0 < NACC; k0 += KB) {
          double vv[KB];
#pragma unroll
          for (int j = 0; j < KB; ++j) vv[j] = k0 + j < nv ? __ldg(Vs + (k0 + j) * ldv_vec + f) : 0.0;
#pragma unroll
          for (int j = 0; j < KB; ++j)
            if (k0 + j < nv) acc[k0 + j] += vv[j] * we;
        }
      } else {
        acc[0] += we * we;
      }
    }
  }
  const int nk = (NACC > 1) ? nv : 1;
  warp_sums<NACC>(acc);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if constexpr (NACC >= 32) {
#pragma unroll
    for (int g = 0; g < NACC / 32; ++g) wsum[wid][g * 32 + lane] = acc[g * 32];
  } else {
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < NACC; ++k) wsum[wid][k] = acc[k];
  }
  if constexpr (BOTH) {  // the norm rides behind the nv dot products (slot nv)
    for (int o = 16; o > 0; o >>= 1) accn += __shfl_xor_sync(0xffffffffu, accn, o);
    if (lane == 0) wsum[wid][NACC] = accn;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nk; k += blockDim.x)
    mine[k] = ((wsum[0][k] + wsum[1][k]) + wsum[2][k]) + wsum[3][k];
  if (BOTH && threadIdx.x == nk)  // the thread that hands slot nk to finish_reduction
    mine[nk] = ((wsum[0][NACC] + wsum[1][NACC]) + wsum[2][NACC]) + wsum[3][NACC];
  RedOut Rl = R;
  Rl.nk = BOTH ? nk + 1 : nk;
  finish_reduction<MODE == DOT_SOLVE ? NV : 0>(partial, pstride, ticket, Rl, mine);
}

// Wide bases (33..64 vectors, restart 50): the plain pass needs one accumulator per
// vector and thread (255 registers at 64, 8 warps per SM).  Here the four warps of
// a block split the BASIS (warp q owns vectors [16 q, 16 q + 16)) and share the
// elements: a tile is 64 elements, one pair per lane.  A warp loads its 16 basis
// values of the tile ONCE and keeps them in registers for both the update and the
// dot products; the update's partial sums meet in shared memory (fixed warp order),
// so V is read once per pass whatever nv is, and warps whose vectors lie beyond nv
// issue no loads.  DOT_SOLVE: a = V^T w.  UPD_DOT_NORM: w' = w - V c, V^T w', ||w'||^2.
template <int MODE>
__global__ void __launch_bounds__(128) orth_wide_kernel(const int32_t* sel, const double* __restrict__ V,
                                                        int64_t ldv_sys, int64_t ldv_vec,
                                                        const int32_t* __restrict__ nvs, double* w, int64_t ldw,
                                                        int64_t n, const double* __restrict__ coef, int cstride,
                                                        double* __restrict__ partial, int pstride,
                                                        unsigned int* ticket, RedOut R, int64_t chunk) {
  MDP_PDL_ENTER();
  constexpr bool UPD = MODE == UPD_DOT_NORM;
  constexpr int GS = 16;
  __shared__ double csh[64];
  __shared__ double2 part[2][4][32];
  __shared__ double mine[65];
  const int i = blockIdx.y;
  const int s = sys_of(sel, i);
  const int nv = nvs[i];
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  const int64_t e0 = blockIdx.x * chunk, e1 = min(n, e0 + chunk);
  const double* Vs = V + s * ldv_sys + (int64_t)(GS * q) * ldv_vec;
  double* ws = w + s * ldw;
  const int mynv = min(GS, max(0, nv - GS * q));  // vectors this warp owns
  if (UPD) {
    for (int k = threadIdx.x; k < 64; k += blockDim.x) csh[k] = k < nv ? coef[i * cstride + k] : 0.0;
    __syncthreads();
  }
  double acc[GS];
  double accn = 0.0;
#pragma unroll
  for (int k = 0; k < GS; ++k) acc[k] = 0.0;
  int buf = 0;
  for (int64_t e = e0 + 2 * lane; e < e1 + 2 * lane; e += 64) {  // uniform trip count (block barriers inside)
    const bool in0 = e < e1, in1 = e + 1 < e1;
    double2 w2 = make_double2(0.0, 0.0);
    if (in1) w2 = *reinterpret_cast<const double2*>(ws + e);
    else if (in0) w2.x = ws[e];
    double2 vv[GS];
#pragma unroll
    for (int k = 0; k < GS; ++k) {
      vv[k] = make_double2(0.0, 0.0);
      if (k < mynv) {
        if (in1) vv[k] = __ldg(reinterpret_cast<const double2*>(Vs + k * ldv_vec + e));
        else if (in0) vv[k].x = __ldg(Vs + k * ldv_vec + e);
      }
    }
    if (UPD) {
      double2 p = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < GS; ++k) {
        p.x = fma(csh[GS * q + k], vv[k].x, p.x);
        p.y = fma(csh[GS * q + k], vv[k].y, p.y);
      }
      part[buf][q][lane] = p;
      __syncthreads();
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        w2.x -= part[buf][g][lane].x;
        w2.y -= part[buf][g][lane].y;
      }
      buf ^= 1;
      if (q == 0) {
        if (in1) *reinterpret_cast<double2*>(ws + e) = w2;
        else if (in0) ws[e] = w2.x;
        accn = fma(w2.x, w2.x, accn);
        accn = fma(w2.y, w2.y, accn);
      }
    }
#pragma unroll
    for (int k = 0; k < GS; ++k) {
      acc[k] = fma(vv[k].x, w2.x, acc[k]);
      acc[k] = fma(vv[k].y, w2.y, acc[k]);
    }
  }
  warp_sums<GS>(acc);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < GS; ++k) mine[GS * q + k] = acc[k];
  __syncthreads();  // mine[0..64) complete before slot nv takes the norm
  if (UPD && q == 0) {
    for (int o = 16; o > 0; o >>= 1) accn += __shfl_xor_sync(0xffffffffu, accn, o);
    if (lane == 0) mine[nv] = accn;
  }
  __syncthreads();
  RedOut Rl = R;
  Rl.nk = UPD ? nv + 1 : nv;
  finish_reduction<MODE == DOT_SOLVE ? 64 : 0>(partial, pstride, ticket, Rl, mine);
}

// V[s][nv] = w / hn  (and vcur), exact division like krylov.py:165
// optional first weighted-Jacobi sweep from zero of the NEXT preconditioner
// apply, fused into the kernel that writes its input v: out = (omega v) / diag
// (jacobi_update_kernel's arithmetic, krylov.py:290-299)
struct JacPre {
  double* out;
  double omega;
  const double* diag;
};

struct GivensArgs {  // optional fused Givens step of the fixed-step inner FGMRES (j = step)
  int j, k;
  double *H, *cs, *sn, *g, *flag;
};
__device__ __forceinline__ void givens_one(int i, int k, int j, const double* __restrict__ hcol, double* H,
                                           double* cs, double* sn, double* g, double* flag);

__global__ void arnoldi_next_kernel(const int32_t* sel, double* V, int64_t ldv_sys, int64_t ldv_vec,
                                    const int32_t* __restrict__ nvs, int kmax,
                                    const double* __restrict__ w, int64_t ldw, int64_t n,
                                    const double* __restrict__ hcol, double* vcur, int64_t ldc,
                                    const GivensArgs GA, const JacPre J) {
  MDP_PDL_ENTER();
  const int i = blockIdx.y;
  if (GA.H && blockIdx.x == 0 && threadIdx.x == 0) givens_one(i, GA.k, GA.j, hcol, GA.H, GA.cs, GA.sn, GA.g, GA.flag);
  const int s = sys_of(sel, i);
  const int nv = nvs[i];
  const double hn = hcol[i * (kmax + 2) + kmax + 1];
  double* dst = nv <= kmax ? V + s * ldv_sys + nv * ldv_vec : nullptr;
  const double* ws = w + s * ldw;
  double* vc = vcur ? vcur + s * ldc : nullptr;
  // four independent loads per thread in flight (one 8-byte load per grid-stride step left the
  // 17 MB vectors at ~2 TB/s: too few bytes in flight for the HBM latency)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e0 < n; e0 += 4 * stride) {
    double wv[4], dg[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t e = e0 + k * stride;
      wv[k] = e < n ? ws[e] : 0.0;
      dg[k] = (J.out && e < n) ? J.diag[s * ldc + e] : 1.0;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t e = e0 + k * stride;
      if (e >= n) break;
      const double v = wv[k] / hn;
      if (dst) dst[e] = v;
      if (vc) vc[e] = v;
      if (J.out) J.out[s * ldc + e] = (J.omega * v) / dg[k];
    }
  }
}

template <int MODE>
static void launch_orth(int nv_max, dim3 grid, cudaStream_t st, const int32_t* sel, const double* V,
                        int64_t ldv_sys, int64_t ldv_vec, const int32_t* nvs, double* w, int64_t ldw,
                        int64_t n, const double* coef, int cstride, double* partial, int pstride,
                        unsigned int* ticket, const RedOut& R) {
#define MDP_ORTH(NVT)                                                                            \
  ::mdp::launch_k(orth_pass_kernel<NVT, MODE>, grid, 128, 0, st, sel, V, ldv_sys, ldv_vec, nvs, w, ldw, n, \
                                                    coef, cstride, partial, pstride, ticket, R, red_chunk(n))
  if (MODE == NORM) {
    MDP_ORTH(0);
  } else if ((MODE == DOT_SOLVE || MODE == UPD_DOT_NORM) && nv_max > 32) {
    ::mdp::launch_k(orth_wide_kernel<(MODE == DOT_SOLVE || MODE == UPD_DOT_NORM) ? MODE : (int)DOT_SOLVE>, grid, 128, 0, st,
                    sel, V, ldv_sys, ldv_vec, nvs, w, ldw, n, coef, cstride, partial, pstride, ticket, R, red_chunk(n));
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
  MDP_PDL_ENTER();
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
  MDP_PDL_ENTER();
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

// r = b - y and ||r|| (fused deterministic reduction)
__global__ void __launch_bounds__(128) residual_kernel(const int32_t* sel, const double* __restrict__ b,
                                                        const double* __restrict__ y, double* r,
                                                        int64_t ld, int64_t n, double* partial,
                                                        unsigned int* ticket, RedOut R, int64_t chunk) {
  MDP_PDL_ENTER();
  __shared__ double sh[32];
  __shared__ double mine[1];
  const int i = blockIdx.y;
  const int s = sys_of(sel, i);
  const int64_t e0 = blockIdx.x * chunk, e1 = min(n, e0 + chunk);
  double acc = 0.0;
  for (int64_t ea = e0 + threadIdx.x; ea < e1; ea += 4 * (int64_t)blockDim.x) {  // 8 loads in flight, same sum order
    double bv[4], yv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t e = ea + k * (int64_t)blockDim.x;
      bv[k] = e < e1 ? b[s * ld + e] : 0.0;
      yv[k] = e < e1 ? y[s * ld + e] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t e = ea + k * (int64_t)blockDim.x;
      if (e >= e1) break;
      const double v = bv[k] - yv[k];
      r[s * ld + e] = v;
      acc += v * v;
    }
  }
  double t = block_sum(acc, sh);
  if (threadIdx.x == 0) mine[0] = t;
  finish_reduction(partial, 1, ticket, R, mine);
}

__global__ void axpby_kernel(const int32_t* sel, double a, const double* __restrict__ x, double b,
                             double* y, int64_t ld, int64_t n) {
  MDP_PDL_ENTER();
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
  MDP_PDL_ENTER();
  const int i = blockIdx.y;
  const int s = sys_of(sel, i);
  const double* a = src + s * lds;
  double* d = dst + s * ldd + (slot ? (int64_t)slot[i] * slot_stride : 0);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e0 < n; e0 += 4 * stride) {
    double v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = e0 + k * stride < n ? a[e0 + k * stride] : 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (e0 + k * stride < n) d[e0 + k * stride] = v[k];
  }
}

// ILU(0) sweeps, one CTA per system, level-scheduled.  The per-row
// arithmetic is the reference's sequential sum with explicitly rounded
// operations (no FMA contraction), so results equal krylov.ilu0_apply
// bitwise.  The system's factor is first staged in shared memory (when it
// fits) so each level costs a barrier plus shared-memory latency only.
// staged: 1 = factor, schedule and x in shared memory; 0 = x in shared memory;
// -1 = everything in global memory, x kept in z (the 3D ILU(0) baseline on C,
// too large for shared memory; L2 reads after each level barrier)
__global__ void __launch_bounds__(1024) ilu0_apply_kernel(const mdp_ilu F, const int32_t* sel,
                                                           const double* __restrict__ r,
                                                           double* __restrict__ z, int64_t ld, int staged) {
  MDP_PDL_ENTER();
  extern __shared__ double xsh_[];
  const bool xglob = staged < 0;
  if (xglob) staged = 0;
  double* xsh = xglob ? z + sys_of(sel, blockIdx.x) * ld : xsh_;
  const int s = sys_of(sel, blockIdx.x);
  const int rs = F.row_start[s], nrow = F.row_start[s + 1] - rs;
  const int p0 = F.ptr[rs], nnz = F.ptr[rs + nrow] - p0;
  const int nlf = F.nlev_f[s], nlb = F.nlev_b[s];
  const double* val = F.val + p0;
  const int* col = F.col + p0;
  const int* levf = F.lev_f + (int64_t)s * F.lev_stride;  // nlev+1 boundaries
  const int* levb = F.lev_b + (int64_t)s * F.lev_stride;
  const int* pf = F.perm_f + rs;
  const int* pb = F.perm_b + rs;
  const double* rp = r + s * ld;
  // staged: the whole factor, the level schedule and r live in shared memory,
  // so each level costs a barrier plus shared-memory latency only
  double* vsh = xsh + nrow;
  int* csh = (int*)(vsh + (staged ? nnz : 0));
  int* psh = csh + (staged ? nnz : 0);
  int* dsh = psh + (staged ? nrow + 1 : 0);
  int* pfs = dsh + (staged ? nrow : 0);
  int* pbs = pfs + (staged ? nrow : 0);
  int* lfs = pbs + (staged ? nrow : 0);
  int* lbs = lfs + (staged ? nlf + 1 : 0);
  if (staged) {
    // eight independent loads per thread in flight before the first shared-memory store: the plain
    // copy loops paid one DRAM / L2 round trip per iteration (~50 of the sweep's 66 us at 2049 rows)
    constexpr int UB = 8;
    const int bd = blockDim.x;
    for (int t0 = threadIdx.x; t0 < nnz; t0 += UB * bd) {
      double v[UB];
      int c[UB];
#pragma unroll
      for (int k = 0; k < UB; ++k) {
        const int t = t0 + k * bd;
        v[k] = t < nnz ? __ldg(val + t) : 0.0;
        c[k] = t < nnz ? __ldg(col + t) : 0;
      }
#pragma unroll
      for (int k = 0; k < UB; ++k) {
        const int t = t0 + k * bd;
        if (t < nnz) {
          vsh[t] = v[k];
          csh[t] = c[k];
        }
      }
    }
    for (int t0 = threadIdx.x; t0 <= nrow; t0 += UB * bd) {
      int a[UB], d[UB], f[UB], g[UB];
#pragma unroll
      for (int k = 0; k < UB; ++k) {
        const int t = t0 + k * bd;
        a[k] = t <= nrow ? __ldg(F.ptr + rs + t) : 0;
        d[k] = t < nrow ? __ldg(F.diag + rs + t) : 0;
        f[k] = t < nrow ? __ldg(pf + t) : 0;
        g[k] = t < nrow ? __ldg(pb + t) : 0;
      }
#pragma unroll
      for (int k = 0; k < UB; ++k) {
        const int t = t0 + k * bd;
        if (t <= nrow) psh[t] = a[k] - p0;
        if (t < nrow) {
          dsh[t] = d[k] - p0;
          pfs[t] = f[k];
          pbs[t] = g[k];
        }
      }
    }
    for (int t = threadIdx.x; t <= nlf; t += blockDim.x) lfs[t] = levf[t];
    for (int t = threadIdx.x; t <= nlb; t += blockDim.x) lbs[t] = levb[t];
    val = vsh;
    col = csh;
    levf = lfs;
    levb = lbs;
    pf = pfs;
    pb = pbs;
  }
  // x = P r (the forward sweep reads x[row] before writing it)
  const int32_t* gp = F.perm ? F.perm + rs : nullptr;
  if (!xglob) {
    for (int t0 = threadIdx.x; t0 < nrow; t0 += 8 * blockDim.x) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int t = t0 + k * blockDim.x;
        v[k] = t < nrow ? rp[gp ? gp[t] : t] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int t = t0 + k * blockDim.x;
        if (t < nrow) xsh[t] = v[k];
      }
    }
  }
  else if (rp != xsh)
    for (int t = threadIdx.x; t < nrow; t += blockDim.x) xsh[t] = rp[t];
  __syncthreads();
  for (int L = 0; L < nlf; ++L) {
    for (int t = levf[L] + threadIdx.x; t < levf[L + 1]; t += blockDim.x) {
      const int row = pf[t];
      const int a = staged ? psh[row] : F.ptr[rs + row] - p0;
      const int d = staged ? dsh[row] : F.diag[rs + row] - p0;
      double acc = xglob ? __ldcg(xsh + row) : xsh[row];
      for (int p = a; p < d; ++p)
        acc = __dsub_rn(acc, __dmul_rn(val[p], xglob ? __ldcg(xsh + col[p]) : xsh[col[p]]));
      if (xglob) __stcg(xsh + row, acc); else xsh[row] = acc;
    }
    __syncthreads();
  }
  for (int L = 0; L < nlb; ++L) {
    for (int t = levb[L] + threadIdx.x; t < levb[L + 1]; t += blockDim.x) {
      const int row = pb[t];
      const int d = staged ? dsh[row] : F.diag[rs + row] - p0;
      const int e = staged ? psh[row + 1] : F.ptr[rs + row + 1] - p0;
      double acc = xglob ? __ldcg(xsh + row) : xsh[row];
      for (int p = d + 1; p < e; ++p)
        acc = __dsub_rn(acc, __dmul_rn(val[p], xglob ? __ldcg(xsh + col[p]) : xsh[col[p]]));
      if (xglob) __stcg(xsh + row, __ddiv_rn(acc, val[d])); else xsh[row] = __ddiv_rn(acc, val[d]);
    }
    __syncthreads();
  }
  if (xglob) return;  // x already is z
  double* zp = z + s * ld;
  for (int t = threadIdx.x; t < nrow; t += blockDim.x) zp[gp ? gp[t] : t] = xsh[t];
}

// ---- device-side Hessenberg work for the fixed-step inner FGMRES ----------
// Same arithmetic as krylov.py:142-172 (explicitly rounded, no FMA); state
// per selection index i: H [(k+1) x k] row-major, cs, sn [k], g [k+1].
// flag: 0 ok, 1 Arnoldi breakdown, 2 lucky breakdown, 4 zero right-hand side
// (any nonzero flag sends the system through the host-driven exact path).
__device__ __forceinline__ void fixed_init_one(int i, int k, const double* __restrict__ beta, double* H, double* cs,
                                               double* sn, double* g, double* flag) {
  for (int t = 0; t < (k + 1) * k; ++t) H[(int64_t)i * (k + 1) * k + t] = 0.0;
  for (int t = 0; t < k; ++t) cs[i * k + t] = sn[i * k + t] = 0.0;
  for (int t = 0; t <= k; ++t) g[i * (k + 1) + t] = 0.0;
  g[i * (k + 1)] = beta[i];
  flag[i] = beta[i] == 0.0 ? 4.0 : 0.0;
}

__global__ void fixed_init_kernel(int nsel, int k, const double* __restrict__ beta, double* H, double* cs,
                                  double* sn, double* g, double* flag) {
  MDP_PDL_ENTER();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nsel) return;
  fixed_init_one(i, k, beta, H, cs, sn, g, flag);
}

// one Givens update of system i's Hessenberg column j (krylov.py:142-157)
__device__ __forceinline__ void givens_one(int i, int k, int j, const double* __restrict__ hcol, double* H,
                                           double* cs, double* sn, double* g, double* flag) {
  if (flag[i] != 0.0) return;
  double* Hi = H + (int64_t)i * (k + 1) * k;
  double* c = cs + i * k;
  double* s = sn + i * k;
  double* gi = g + i * (k + 1);
  const double* hc = hcol + (int64_t)i * (k + 2);
  for (int r = 0; r <= j; ++r) Hi[r * k + j] = hc[r];
  const double hn = hc[k + 1];
  for (int r = 0; r < j; ++r) {
    double a = Hi[r * k + j], b = Hi[(r + 1) * k + j];
    double t = __dadd_rn(__dmul_rn(c[r], a), __dmul_rn(s[r], b));
    Hi[(r + 1) * k + j] = __dadd_rn(__dmul_rn(-s[r], a), __dmul_rn(c[r], b));
    Hi[r * k + j] = t;
  }
  const double denom = hypot(Hi[j * k + j], hn);
  if (denom < 1e-14) {
    flag[i] = 1.0;
    return;
  }
  c[j] = __ddiv_rn(Hi[j * k + j], denom);
  s[j] = __ddiv_rn(hn, denom);
  Hi[j * k + j] = denom;
  gi[j + 1] = __dmul_rn(-s[j], gi[j]);
  gi[j] = __dmul_rn(c[j], gi[j]);
  if (hn < 1e-14) flag[i] = 2.0;
}

__global__ void givens_step_kernel(int nsel, int k, int j, const double* __restrict__ hcol, double* H, double* cs,
                                   double* sn, double* g, double* flag) {
  MDP_PDL_ENTER();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nsel) return;
  givens_one(i, k, j, hcol, H, cs, sn, g, flag);
}

// y = H[:m,:m]^-1 g[:m] by back substitution (krylov.py:168-171); y = 0 for flagged systems
__device__ __forceinline__ void backsub_one(int i, int k, int m, const double* __restrict__ H,
                                            const double* __restrict__ g, const double* __restrict__ flag,
                                            double* yi) {
  const double* Hi = H + (int64_t)i * (k + 1) * k;
  if (flag[i] != 0.0) {
    for (int r = 0; r < k; ++r) yi[r] = 0.0;
    return;
  }
  for (int r = m - 1; r >= 0; --r) {
    double acc = 0.0;
    for (int c = r + 1; c < m; ++c) acc = __dadd_rn(acc, __dmul_rn(Hi[r * k + c], yi[c]));
    yi[r] = __ddiv_rn(__dsub_rn(g[i * (k + 1) + r], acc), Hi[r * k + r]);
  }
}

__global__ void backsub_kernel(int nsel, int k, int m, const double* __restrict__ H, const double* __restrict__ g,
                               const double* __restrict__ flag, double* y) {
  MDP_PDL_ENTER();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nsel) return;
  backsub_one(i, k, m, H, g, flag, y + i * k);
}

// Fused start of the fixed-step inner FGMRES: V0 = b / beta, vcur = V0, and
// (block 0 of each system) the Hessenberg / Givens state init.  Replaces
// mdp_scale + mdp_copy_vec + mdp_fixed_init with the same arithmetic.
struct FixedState {
  int k;
  double *H, *cs, *sn, *g, *flag;
};


__global__ void fixed_start_kernel(const int32_t* sel, const double* __restrict__ b, int64_t ldb,
                                   const double* __restrict__ beta, double* __restrict__ v0, int64_t ldv,
                                   double* __restrict__ vcur, int64_t ldc, int64_t n, const FixedState F,
                                   const JacPre J) {
  MDP_PDL_ENTER();
  const int i = blockIdx.y;
  const int s = sys_of(sel, i);
  if (blockIdx.x == 0 && threadIdx.x == 0) fixed_init_one(i, F.k, beta, F.H, F.cs, F.sn, F.g, F.flag);
  const double* bs = b + s * ldb;
  double* vs = v0 + s * ldv;
  double* cs = vcur + s * ldc;
  const double bi = beta[i];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e0 < n; e0 += 4 * stride) {
    double bv[4], dg[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t e = e0 + k * stride;
      bv[k] = e < n ? bs[e] : 0.0;
      dg[k] = (J.out && e < n) ? J.diag[s * ldc + e] : 1.0;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t e = e0 + k * stride;
      if (e >= n) break;
      const double v = bv[k] / bi;
      vs[e] = v;
      cs[e] = v;
      if (J.out) J.out[s * ldc + e] = (J.omega * v) / dg[k];
    }
  }
}

// Fused end of the fixed-step inner FGMRES: y = H^-1 g (every block solves the
// tiny triangular system itself, same order as backsub_kernel), then
// x = sum_k y_k Z_k written straight into the destination (replaces
// mdp_backsub + mdp_fill + mdp_basis_update + the copy out).
__global__ void fixed_finish_kernel(const int32_t* sel, int m, const double* __restrict__ Z, int64_t ldz_sys,
                                    int64_t ldz_vec, double* __restrict__ x, int64_t ldx, int64_t n,
                                    const FixedState F) {
  MDP_PDL_ENTER();
  __shared__ double ysh[64];
  const int i = blockIdx.y;
  const int s = sys_of(sel, i);
  if (threadIdx.x == 0) backsub_one(i, F.k, m, F.H, F.g, F.flag, ysh);
  __syncthreads();
  const double* Zs = Z + s * ldz_sys;
  double* xs = x + s * ldx;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e0 < n; e0 += 2 * stride) {
    const int64_t e1 = e0 + stride;  // two elements per thread: 2 m loads in flight
    double t0 = 0.0, t1 = 0.0;
    for (int k = 0; k < m; ++k) {
      const double z0 = __ldg(Zs + k * ldz_vec + e0);
      const double z1 = e1 < n ? __ldg(Zs + k * ldz_vec + e1) : 0.0;
      t0 += z0 * ysh[k];
      t1 += z1 * ysh[k];
    }
    xs[e0] = 0.0 + t0;  // as fill(0) followed by basis_update's x += t
    if (e1 < n) xs[e1] = 0.0 + t1;
  }
}

__global__ void copy_slot_kernel(const int32_t* sel, const double* __restrict__ src, int64_t lds,
                                 const int32_t* __restrict__ slot, int64_t slot_stride, double* __restrict__ dst,
                                 int64_t ldd, int64_t n) {
  MDP_PDL_ENTER();
  const int i = blockIdx.y;
  const int s = sys_of(sel, i);
  const double* a = src + s * lds + (int64_t)slot[i] * slot_stride;
  double* d = dst + s * ldd;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    d[e] = a[e];
}

__global__ void fill_kernel(const int32_t* sel, double* y, int64_t ld, int64_t n, double v) {
  MDP_PDL_ENTER();
  const int s = sys_of(sel, blockIdx.y);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    y[s * ld + e] = v;
}

inline dim3 ew_grid(int64_t n, int nsel) {
  int bx = ceil_div(n, 256);
  int cap = 8 * sm_count();  // 2048 resident threads per SM; the hot loops also keep 4 loads per thread in flight
  bx = bx > cap ? cap : bx;
  return dim3(bx < 1 ? 1 : bx, nsel);
}

}  // namespace mdp

using namespace mdp;

// workspace: [tickets: nsel, padded][partials nsel x nb x 65][h1, h2: nsel x (kmax+1)][nrm2: nsel]
// The tickets sit at a fixed offset for every entry point sharing a
// workspace and must start at zero: callers allocate the workspace zeroed
// once; every kernel resets its tickets when it finishes.
struct Work {
  double* partial;
  double* h1;
  double* h2;
  double* nrm2;
  unsigned int* ticket;
};
static Work carve(void* work, int32_t nsel, int32_t kmax, int64_t n) {
  Work W;
  const int nb = red_blocks(n);
  W.ticket = (unsigned int*)work;
  W.partial = (double*)((char*)work + ((size_t)nsel * sizeof(unsigned int) + 255) / 256 * 256);
  W.h1 = W.partial + (size_t)nsel * nb * 65;
  W.h2 = W.h1 + (size_t)nsel * (kmax + 1);
  W.nrm2 = W.h2 + (size_t)nsel * (kmax + 1);
  return W;
}

extern "C" size_t mdp_arnoldi_work_bytes(int32_t nsel, int32_t kmax, int64_t n) {
  int nb = red_blocks(n);
  size_t d = (size_t)nsel * nb * 65 + (size_t)nsel * (2 * (kmax + 1) + 1);
  return d * sizeof(double) + ((size_t)nsel * sizeof(unsigned int) + 255) / 256 * 256 + 256;
}

static int arnoldi_impl(int32_t nsel, const int32_t* sel, double* V, int64_t ldv_sys, int64_t ldv_vec,
                        const int32_t* nv, int32_t kmax, double* w, int64_t ldw, int64_t n, double* hcol,
                        double* vcur, int64_t ldc, double* gram, void* work, void* stream, const GivensArgs& GA,
                        const JacPre& J);

extern "C" int mdp_arnoldi(int32_t nsel, const int32_t* sel, double* V, int64_t ldv_sys,
                           int64_t ldv_vec, const int32_t* nv, int32_t kmax, double* w, int64_t ldw,
                           int64_t n, double* hcol, double* vcur, int64_t ldc, double* gram, void* work,
                           void* stream) {
  return arnoldi_impl(nsel, sel, V, ldv_sys, ldv_vec, nv, kmax, w, ldw, n, hcol, vcur, ldc, gram, work, stream,
                      GivensArgs{0, 0, nullptr, nullptr, nullptr, nullptr, nullptr}, JacPre{nullptr, 0.0, nullptr});
}

extern "C" int mdp_arnoldi_givens(int32_t nsel, const int32_t* sel, double* V, int64_t ldv_sys, int64_t ldv_vec,
                                  const int32_t* nv, int32_t kmax, double* w, int64_t ldw, int64_t n,
                                  double* hcol, double* vcur, int64_t ldc, double* gram, void* work, int32_t j,
                                  double* H, double* cs, double* sn, double* g, double* flag, double* jac_out,
                                  double omega, const double* diag, void* stream) {
  MDP_REQUIRE(H && cs && sn && g && flag && j >= 0 && j < kmax, "fused Givens step needs the fixed-step state");
  MDP_REQUIRE(!jac_out || (vcur && diag), "the fused first Jacobi sweep needs vcur and diag");
  return arnoldi_impl(nsel, sel, V, ldv_sys, ldv_vec, nv, kmax, w, ldw, n, hcol, vcur, ldc, gram, work, stream,
                      GivensArgs{j, kmax, H, cs, sn, g, flag}, JacPre{jac_out, omega, diag});
}

static int arnoldi_impl(int32_t nsel, const int32_t* sel, double* V, int64_t ldv_sys, int64_t ldv_vec,
                        const int32_t* nv, int32_t kmax, double* w, int64_t ldw, int64_t n, double* hcol,
                        double* vcur, int64_t ldc, double* gram, void* work, void* stream, const GivensArgs& GA,
                        const JacPre& J) {
  MDP_REQUIRE(kmax >= 1 && kmax <= 63, "kmax %d outside [1, 63]", kmax);
  MDP_REQUIRE(n > 0, "empty vectors");
  MDP_REQUIRE(((uintptr_t)V | (uintptr_t)w) % 16 == 0 && (ldv_sys | ldv_vec | ldw) % 2 == 0,
              "V and w must be 16-byte aligned with even strides (element pairs are loaded as double2)");
  if (nsel == 0) return MDP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = red_blocks(n);
  const int pstride = 65;
  Work W = carve(work, nsel, kmax, n);
  dim3 grid(nb, nsel);
  const int nvmax = kmax + 1;
  RedOut R{};
  R.out = W.h1;
  R.ostride = kmax + 1;
  R.mode = 0;
  if (gram) {
    // MGS from one pass of dot products (the Gram rows of earlier steps stand in for
    // the sequential projections): V is read twice per step instead of three times
    R.mode = 3;
    R.hcol = hcol;
    R.kmax = kmax;
    R.nvs = nv;
    R.gram = gram;
    R.sel = sel;
    launch_orth<DOT_SOLVE>(nvmax, grid, st, sel, V, ldv_sys, ldv_vec, nv, w, ldw, n, nullptr, 0, W.partial, pstride,
                           W.ticket, R);
    MDP_LAUNCH_CHECK("orth_pass DOT_SOLVE");
    R.out = W.h2;
    R.mode = 4;
    launch_orth<UPD_DOT_NORM>(nvmax, grid, st, sel, V, ldv_sys, ldv_vec, nv, w, ldw, n, W.h1, kmax + 1, W.partial,
                              pstride, W.ticket, R);
    MDP_LAUNCH_CHECK("orth_pass UPD_DOT_NORM");
    ::mdp::launch_k(arnoldi_next_kernel, ew_grid(n, nsel), 256, 0, st, sel, V, ldv_sys, ldv_vec, nv, kmax, w, ldw, n,
                    hcol, vcur, ldc, GA, J);
    MDP_LAUNCH_CHECK("mdp_arnoldi");
    return MDP_OK;
  }
  launch_orth<DOT>(nvmax, grid, st, sel, V, ldv_sys, ldv_vec, nv, w, ldw, n, nullptr, 0, W.partial, pstride,
                   W.ticket, R);
  MDP_LAUNCH_CHECK("orth_pass DOT");
  R.out = W.h2;
  launch_orth<UPD_DOT>(nvmax, grid, st, sel, V, ldv_sys, ldv_vec, nv, w, ldw, n, W.h1, kmax + 1, W.partial,
                       pstride, W.ticket, R);
  MDP_LAUNCH_CHECK("orth_pass UPD_DOT");
  R.out = W.nrm2;
  R.ostride = 1;
  R.mode = 2;
  R.h1 = W.h1;
  R.h2 = W.h2;
  R.hcol = hcol;
  R.kmax = kmax;
  R.nvs = nv;
  launch_orth<UPD_NORM>(nvmax, grid, st, sel, V, ldv_sys, ldv_vec, nv, w, ldw, n, W.h2, kmax + 1, W.partial,
                        pstride, W.ticket, R);
  MDP_LAUNCH_CHECK("orth_pass UPD_NORM");
  ::mdp::launch_k(arnoldi_next_kernel, ew_grid(n, nsel), 256, 0, st, sel, V, ldv_sys, ldv_vec, nv, kmax, w, ldw, n,
                                                         hcol, vcur, ldc, GA, J);
  MDP_LAUNCH_CHECK("mdp_arnoldi");
  return MDP_OK;
}

extern "C" int mdp_norms(int32_t nsel, const int32_t* sel, const double* x, int64_t ldx, int64_t n,
                         double* out, void* work, void* stream) {
  if (nsel == 0) return MDP_OK;
  MDP_REQUIRE(n > 0, "empty vectors");
  MDP_REQUIRE((uintptr_t)x % 16 == 0 && ldx % 2 == 0, "x must be 16-byte aligned with an even stride");
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = red_blocks(n);
  Work W = carve(work, nsel, 1, n);
  RedOut R{};
  R.out = out;
  R.ostride = 1;
  R.mode = 1;
  ::mdp::launch_k(orth_pass_kernel<0, NORM>, dim3(nb, nsel), 128, 0, st, sel, nullptr, 0, 0, nullptr, const_cast<double*>(x),
                                                            ldx, n, nullptr, 0, W.partial, 1, W.ticket, R, red_chunk(n));
  MDP_LAUNCH_CHECK("mdp_norms");
  return MDP_OK;
}

extern "C" int mdp_scale(int32_t nsel, const int32_t* sel, const double* x, int64_t ldx,
                         const double* num, const double* den, double* y, int64_t ldy, int64_t n,
                         void* stream) {
  if (nsel == 0) return MDP_OK;
  MDP_REQUIRE(num || den, "scale needs num or den");
  ::mdp::launch_k(scale_kernel, ew_grid(n, nsel), 256, 0, (cudaStream_t)stream, sel, x, ldx, num, den, y, ldy, n);
  MDP_LAUNCH_CHECK("mdp_scale");
  return MDP_OK;
}

extern "C" int mdp_basis_update(int32_t nsel, const int32_t* sel, double* x, int64_t ldx,
                                const double* Z, int64_t ldz_sys, int64_t ldz_vec, const int32_t* cnt,
                                const double* y, int32_t ystride, int64_t n, void* stream) {
  if (nsel == 0) return MDP_OK;
  ::mdp::launch_k(basis_update_kernel, ew_grid(n, nsel), 256, 0, (cudaStream_t)stream, sel, x, ldx, Z, ldz_sys,
                                                                          ldz_vec, cnt, y, ystride, n);
  MDP_LAUNCH_CHECK("mdp_basis_update");
  return MDP_OK;
}

extern "C" int mdp_residual(int32_t nsel, const int32_t* sel, const double* b, const double* y,
                            double* r, int64_t ld, int64_t n, double* rn, void* work, void* stream) {
  if (nsel == 0) return MDP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = red_blocks(n);
  Work W = carve(work, nsel, 1, n);
  RedOut R{};
  R.out = rn;
  R.ostride = 1;
  R.nk = 1;
  R.mode = 1;
  ::mdp::launch_k(residual_kernel, dim3(nb, nsel), 128, 0, st, sel, b, y, r, ld, n, W.partial, W.ticket, R,
                  red_chunk(n));
  MDP_LAUNCH_CHECK("mdp_residual");
  return MDP_OK;
}

extern "C" int mdp_axpby(int32_t nsel, const int32_t* sel, double a, const double* x, double b,
                         double* y, int64_t ld, int64_t n, void* stream) {
  if (nsel == 0) return MDP_OK;
  ::mdp::launch_k(axpby_kernel, ew_grid(n, nsel), 256, 0, (cudaStream_t)stream, sel, a, x, b, y, ld, n);
  MDP_LAUNCH_CHECK("mdp_axpby");
  return MDP_OK;
}

extern "C" int mdp_copy_vec(int32_t nsel, const int32_t* sel, const double* src, int64_t lds,
                            double* dst, int64_t ldd, const int32_t* dst_slot, int64_t slot_stride,
                            int64_t n, void* stream) {
  if (nsel == 0) return MDP_OK;
  ::mdp::launch_k(copy_vec_kernel, ew_grid(n, nsel), 256, 0, (cudaStream_t)stream, sel, src, lds, dst, ldd, dst_slot,
                                                                      slot_stride, n);
  MDP_LAUNCH_CHECK("mdp_copy_vec");
  return MDP_OK;
}

extern "C" int mdp_fixed_start(int32_t nsel, const int32_t* sel, int32_t k, const double* b, int64_t ldb,
                               const double* beta, double* v0, int64_t ldv, double* vcur, int64_t ldc, int64_t n,
                               double* H, double* cs, double* sn, double* g, double* flag, double* jac_out,
                               double omega, const double* diag, void* stream) {
  if (nsel == 0) return MDP_OK;
  MDP_REQUIRE(!jac_out || diag, "the fused first Jacobi sweep needs diag");
  ::mdp::launch_k(fixed_start_kernel, ew_grid(n, nsel), 256, 0, (cudaStream_t)stream, sel, b, ldb, beta, v0, ldv,
                  vcur, ldc, n, FixedState{k, H, cs, sn, g, flag}, JacPre{jac_out, omega, diag});
  MDP_LAUNCH_CHECK("fixed_start_kernel");
  return MDP_OK;
}

extern "C" int mdp_fixed_finish(int32_t nsel, const int32_t* sel, int32_t k, int32_t m, const double* Z,
                                int64_t ldz_sys, int64_t ldz_vec, double* x, int64_t ldx, int64_t n,
                                double* H, double* g, double* flag, void* stream) {
  MDP_REQUIRE(m >= 0 && m <= k && k <= 64, "fixed-step finish: m %d, k %d", m, k);
  if (nsel == 0) return MDP_OK;
  ::mdp::launch_k(fixed_finish_kernel, ew_grid(n, nsel), 256, 0, (cudaStream_t)stream, sel, m, Z, ldz_sys, ldz_vec,
                  x, ldx, n, FixedState{k, H, nullptr, nullptr, g, flag});
  MDP_LAUNCH_CHECK("fixed_finish_kernel");
  return MDP_OK;
}

extern "C" int mdp_fixed_init(int32_t nsel, int32_t k, const double* beta, double* H, double* cs, double* sn,
                              double* g, double* flag, void* stream) {
  if (nsel == 0) return MDP_OK;
  ::mdp::launch_k(fixed_init_kernel, ceil_div(nsel, 64), 64, 0, (cudaStream_t)stream, nsel, k, beta, H, cs, sn, g, flag);
  MDP_LAUNCH_CHECK("fixed_init_kernel");
  return MDP_OK;
}

extern "C" int mdp_givens_step(int32_t nsel, int32_t k, int32_t j, const double* hcol, double* H, double* cs,
                               double* sn, double* g, double* flag, void* stream) {
  MDP_REQUIRE(j >= 0 && j < k, "givens column %d outside [0, %d)", j, k);
  if (nsel == 0) return MDP_OK;
  ::mdp::launch_k(givens_step_kernel, ceil_div(nsel, 64), 64, 0, (cudaStream_t)stream, nsel, k, j, hcol, H, cs, sn, g, flag);
  MDP_LAUNCH_CHECK("givens_step_kernel");
  return MDP_OK;
}

extern "C" int mdp_backsub(int32_t nsel, int32_t k, int32_t m, const double* H, const double* g,
                           const double* flag, double* y, void* stream) {
  MDP_REQUIRE(m >= 0 && m <= k, "back substitution size %d outside [0, %d]", m, k);
  if (nsel == 0) return MDP_OK;
  ::mdp::launch_k(backsub_kernel, ceil_div(nsel, 64), 64, 0, (cudaStream_t)stream, nsel, k, m, H, g, flag, y);
  MDP_LAUNCH_CHECK("backsub_kernel");
  return MDP_OK;
}

extern "C" int mdp_copy_slot(int32_t nsel, const int32_t* sel, const double* src, int64_t lds,
                             const int32_t* slot, int64_t slot_stride, double* dst, int64_t ldd, int64_t n,
                             void* stream) {
  if (nsel == 0) return MDP_OK;
  ::mdp::launch_k(copy_slot_kernel, ew_grid(n, nsel), 256, 0, (cudaStream_t)stream, sel, src, lds, slot, slot_stride, dst, ldd,
                                                                       n);
  MDP_LAUNCH_CHECK("copy_slot_kernel");
  return MDP_OK;
}

extern "C" int mdp_fill(int32_t nsel, const int32_t* sel, double* y, int64_t ld, int64_t n, double v,
                        void* stream) {
  if (nsel == 0) return MDP_OK;
  ::mdp::launch_k(fill_kernel, ew_grid(n, nsel), 256, 0, (cudaStream_t)stream, sel, y, ld, n, v);
  MDP_LAUNCH_CHECK("fill_kernel");
  return MDP_OK;
}

extern "C" int mdp_ilu0_apply(const mdp_ilu* f, int32_t nsel, const int32_t* sel, const double* r,
                              double* z, int64_t ld, void* stream) {
  MDP_REQUIRE(f != nullptr, "null ILU descriptor");
  if (nsel == 0) return MDP_OK;
  const size_t cap = 200 * 1024;
  const size_t base = (size_t)f->max_rows * sizeof(double);
  const size_t full = base + (size_t)f->max_nnz * (sizeof(double) + sizeof(int)) +
                      (size_t)(4 * f->max_rows + 1 + 2 * f->lev_stride) * sizeof(int);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ilu0_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap);
    attr = true;
  }
  if (base > cap) {  // large (3D) factors: x lives in z, 1024 threads per level
    MDP_REQUIRE(f->perm == nullptr, "permuted (direct) factors must fit the shared-memory sweep");
    MDP_REQUIRE(r != z, "the global-memory ILU sweep needs r and z distinct");
    ::mdp::launch_k(ilu0_apply_kernel, nsel, 1024, 0, (cudaStream_t)stream, *f, sel, r, z, ld, -1);
    MDP_LAUNCH_CHECK("mdp_ilu0_apply");
    return MDP_OK;
  }
  const int staged = full <= cap;
  ::mdp::launch_k(ilu0_apply_kernel, nsel, 256, staged ? full : base, (cudaStream_t)stream, *f, sel, r, z, ld, staged);
  MDP_LAUNCH_CHECK("mdp_ilu0_apply");
  return MDP_OK;
}
